/*
 * srmra_oracle.c — float64 CPU ORACLE for one projected-EM iteration of 2-D SR-MRA.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2204_04754_b200/, libsrmra.so) never links, imports or calls it, and shares no
 * code, header, table or constant with it.
 *
 * What it computes is the plain definition of one EM iteration of the paper, evaluated by
 * brute force in float64:
 *
 *   log-likelihood   PAPER.md:228-233  (eq:likelihood_EM)
 *       LL = sum_i log sum_s rho1[s1] rho2[s2] exp(-||y_i - P R_s x||^2 / (2 sigma^2))
 *   E-step weights   PAPER.md:247-250  (eq:weights_EM)
 *       w^{i,s} = C^i rho[s] exp(-||y_i - P R_s x||^2/(2 sigma^2)),  sum_s w^{i,s} = 1
 *   M-step for x     PAPER.md:255-263  (eq:x_EM), A x = b with P^{-1} read as P^T
 *       (reading R1), so A is diagonal:
 *       A[p] = sum_{i,s,n: p = P R_s-sampled pixel of n} w^{i,s},  b[p] = same sum of w^{i,s} y_i[n]
 *   M-step for rho   PAPER.md:266-268  (eq:rho_EM) in its separable-marginal form
 *       (reading R2): rho1'[s1] = sum_{s2} sum_i w^{i,s} / sum_i sum_s' w^{i,s'}, same for rho2.
 *   projection       PAPER.md:384-388 (Algorithm 2 step 2) with the north_star stand-in
 *       denoiser: 3x3 circular box filter, then clamp to [-1, 1] (reading R7).
 *
 * Index convention, PAPER.md:37-38 (explicit form of eq:model_1):
 *       (P R_s x)[n1,n2] = x[(n1 K - s1) mod L, (n2 K - s2) mod L],  s = (s1, s2), s1 on the
 *       first (row) index, flattened s = s1*L + s2 (reading R3).
 *
 * Parallel over observations with OpenMP (static schedule, thread-local float64 accumulators
 * reduced in thread-index order: deterministic for a fixed thread count).  The modular column
 * index is hoisted by materialising, for each s2, the K-decimated columns of x (a gather table;
 * no arithmetic of the method is changed by it).
 *
 * Parity status: every exported function is pinned by tests/test_oracle_pins.py (brute-force
 * dense-matrix construction, closed forms, invariances, monotone LL, sigma->0 recovery).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int imod(int64_t a, int64_t m) { int64_t r = a % m; return (int)(r < 0 ? r + m : r); }

static double safe_log(double p) { return p > 0.0 ? log(p) : -INFINITY; }

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* table xs[s2][row][n2] = x[row][(n2*K - s2) mod L] */
static double* build_col_table(const double* x, int L, int Ll, int K) {
    double* xs = (double*)malloc(sizeof(double) * (size_t)L * L * Ll);
    if (!xs) return NULL;
    for (int s2 = 0; s2 < L; ++s2)
        for (int row = 0; row < L; ++row)
            for (int n2 = 0; n2 < Ll; ++n2)
                xs[((size_t)s2 * L + row) * Ll + n2] = x[(size_t)row * L + imod((int64_t)n2 * K - s2, L)];
    return xs;
}

/* ell[s] = log rho1[s1] + log rho2[s2] - ||y_i - P R_s x||^2 / (2 sigma^2) for all s;
 * returns lse = log sum_s exp(ell[s])  (eq:likelihood_EM inner term). */
static double obs_logits(const float* yi, int L, int Ll, int K, double inv2s2,
                         const double* xs, const double* lr1, const double* lr2, const double* lrj,
                         double* ell) {
    for (int s1 = 0; s1 < L; ++s1) {
        for (int s2 = 0; s2 < L; ++s2) {
            double d = 0.0;
            const double* xt = xs + (size_t)s2 * L * Ll;
            for (int n1 = 0; n1 < Ll; ++n1) {
                const double* xr = xt + (size_t)imod((int64_t)n1 * K - s1, L) * Ll;
                const float* yr = yi + (size_t)n1 * Ll;
                for (int n2 = 0; n2 < Ll; ++n2) {
                    double e = (double)yr[n2] - xr[n2];
                    d += e * e;
                }
            }
            /* log prior: separable log rho1[s1] + log rho2[s2], or the joint log rho[s] (NEXT-3) */
            ell[s1 * L + s2] = (lrj ? lrj[s1 * L + s2] : lr1[s1] + lr2[s2]) - d * inv2s2;
        }
    }
    int L2 = L * L;
    double m = -INFINITY;
    for (int s = 0; s < L2; ++s) if (ell[s] > m) m = ell[s];
    double acc = 0.0;
    for (int s = 0; s < L2; ++s) acc += exp(ell[s] - m);
    return m + log(acc);
}

/* 3x3 circular box filter then clamp to [-1,1] (north_star stand-in for D(x, sigma)). */
void oracle_project(const double* x, int L, double* out) {
    for (int p1 = 0; p1 < L; ++p1)
        for (int p2 = 0; p2 < L; ++p2) {
            double acc = 0.0;
            for (int d1 = -1; d1 <= 1; ++d1)
                for (int d2 = -1; d2 <= 1; ++d2)
                    acc += x[(size_t)imod(p1 + d1, L) * L + imod(p2 + d2, L)];
            double v = acc / 9.0;
            out[(size_t)p1 * L + p2] = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        }
}

/* Posterior w^{i,.} (eq:weights_EM) of ONE observation; returns its log-likelihood term. */
double oracle_posterior(const float* yi, int L, int Ll, int K, double sigma,
                        const double* x, const double* rho1, const double* rho2,
                        double* w_out) {
    double* xs = build_col_table(x, L, Ll, K);
    double* lr1 = (double*)malloc(sizeof(double) * L);
    double* lr2 = (double*)malloc(sizeof(double) * L);
    for (int k = 0; k < L; ++k) { lr1[k] = safe_log(rho1[k]); lr2[k] = safe_log(rho2[k]); }
    double lse = obs_logits(yi, L, Ll, K, 1.0 / (2.0 * sigma * sigma), xs, lr1, lr2, NULL, w_out);
    for (int s = 0; s < L * L; ++s) w_out[s] = exp(w_out[s] - lse);
    free(xs); free(lr1); free(lr2);
    return lse;
}

/* Per-observation log-likelihood terms for a list of observation indices (sampled parity). */
int oracle_loglik_obs(const float* y, const int64_t* idx, int64_t n_idx,
                      int L, int Ll, int K, double sigma,
                      const double* x, const double* rho1, const double* rho2, double* ll_out) {
    double* xs = build_col_table(x, L, Ll, K);
    if (!xs) return -5;
    double lr1[4096], lr2[4096];
    if (L > 4096) { free(xs); return -1; }
    for (int k = 0; k < L; ++k) { lr1[k] = safe_log(rho1[k]); lr2[k] = safe_log(rho2[k]); }
    double inv2s2 = 1.0 / (2.0 * sigma * sigma);
    int L2 = L * L;
#pragma omp parallel
    {
        double* ell = (double*)malloc(sizeof(double) * L2);
#pragma omp for schedule(dynamic, 1)
        for (int64_t j = 0; j < n_idx; ++j)
            ll_out[j] = obs_logits(y + (size_t)idx[j] * Ll * Ll, L, Ll, K, inv2s2, xs, lr1, lr2, NULL, ell);
        free(ell);
    }
    free(xs);
    return 0;
}

/*
 * One EM iteration (E-step, M-step, optional projection) over all N observations.
 * Inputs : y [N][Ll][Ll] float32 (promoted exactly to float64), x [L][L], rho1/rho2 [L].
 * Outputs: x_out [L][L], rho1_out/rho2_out [L], *ll_out = LL at the INPUT theta (reading R4).
 * Optional (NULL to skip): b_out [L*L], A_out [L*L], colsum_out [L*L] (= sum_i w^{i,s}),
 *                          ll_obs_out [N] (per-observation log-likelihood terms).
 * tau: pixel p keeps x[p] when A[p] <= tau (reading R6).  project: apply the stand-in D.
 * Returns 0, or -1 on invalid sizes, -5 on allocation failure.
 */
static int em_iter_impl(const float* y, int64_t N, int L, int Ll, int K, double sigma,
                        const double* x, const double* rho1, const double* rho2, const double* rhoj,
                        int project, double tau,
                        double* x_out, double* rho1_out, double* rho2_out, double* rhoj_out, double* ll_out,
                        double* b_out, double* A_out, double* colsum_out, double* ll_obs_out) {
    if (N < 0 || L <= 0 || Ll <= 0 || K <= 0 || Ll * K != L || !(sigma > 0.0) || L > 4096) return -1;
    const int L2 = L * L, Ll2 = Ll * Ll;
    double lr1[4096], lr2[4096];
    double* lrj = NULL;
    if (rhoj) {  /* joint prior rho[s] (NEXT-3): its log per shift */
        lrj = (double*)malloc(sizeof(double) * L2);
        if (!lrj) return -5;
        for (int s = 0; s < L2; ++s) lrj[s] = safe_log(rhoj[s]);
    } else {
        for (int k = 0; k < L; ++k) { lr1[k] = safe_log(rho1[k]); lr2[k] = safe_log(rho2[k]); }
    }
    const double inv2s2 = 1.0 / (2.0 * sigma * sigma);
    double* xs = build_col_table(x, L, Ll, K);
    if (!xs) return -5;
    int* colidx = (int*)malloc(sizeof(int) * (size_t)L * Ll);   /* (n2 K - s2) mod L */
    for (int s2 = 0; s2 < L; ++s2)
        for (int n2 = 0; n2 < Ll; ++n2) colidx[(size_t)s2 * Ll + n2] = imod((int64_t)n2 * K - s2, L);

    int nt = oracle_max_threads();
    double* acc = (double*)calloc((size_t)nt * (3 * (size_t)L2 + 1), sizeof(double));
    if (!acc) { free(xs); return -5; }

#pragma omp parallel
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num();
#else
        int tid = 0;
#endif
        double* b = acc + (size_t)tid * (3 * (size_t)L2 + 1);
        double* A = b + L2;
        double* cs = A + L2;
        double* ll = cs + L2;
        double* ell = (double*)malloc(sizeof(double) * L2);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < N; ++i) {
            const float* yi = y + (size_t)i * Ll2;
            /* E-step: logits and normaliser C^i (eq:weights_EM) */
            double lse = obs_logits(yi, L, Ll, K, inv2s2, xs, lr1, lr2, lrj, ell);
            *ll += lse;
            if (ll_obs_out) ll_obs_out[i] = lse;
            /* M-step accumulation (eq:x_EM with P^{-1} := P^T, eq:rho_EM) */
            for (int s1 = 0; s1 < L; ++s1)
                for (int s2 = 0; s2 < L; ++s2) {
                    double w = exp(ell[s1 * L + s2] - lse);
                    if (w == 0.0) continue;           /* bit-identical skip */
                    cs[s1 * L + s2] += w;
                    const int* ci = colidx + (size_t)s2 * Ll;
                    for (int n1 = 0; n1 < Ll; ++n1) {
                        const size_t row = (size_t)imod((int64_t)n1 * K - s1, L) * L;
                        const float* yr = yi + (size_t)n1 * Ll;
                        for (int n2 = 0; n2 < Ll; ++n2) {
                            const size_t p = row + ci[n2];   /* (n1 K - s1, n2 K - s2) mod L */
                            b[p] += w * (double)yr[n2];
                            A[p] += w;
                        }
                    }
                }
        }
        free(ell);
    }
    free(xs);
    free(colidx);

    /* fixed-order reduction over thread-local accumulators */
    double* b = (double*)calloc((size_t)3 * L2 + 1, sizeof(double));
    double* A = b + L2;
    double* cs = A + L2;
    double ll = 0.0;
    for (int t = 0; t < nt; ++t) {
        const double* src = acc + (size_t)t * (3 * (size_t)L2 + 1);
        for (int k = 0; k < 3 * L2; ++k) b[k] += src[k];
        ll += src[3 * L2];
    }
    free(acc);

    /* rho update: marginals of eq:rho_EM (separable), or eq:rho_EM as written (joint, NEXT-3) with the
     * marginals of the new joint prior reported in rho1_out / rho2_out */
    double tot = 0.0;
    for (int s = 0; s < L2; ++s) tot += cs[s];
    for (int k = 0; k < L; ++k) { rho1_out[k] = 0.0; rho2_out[k] = 0.0; }
    for (int s1 = 0; s1 < L; ++s1)
        for (int s2 = 0; s2 < L; ++s2) {
            rho1_out[s1] += cs[s1 * L + s2];
            rho2_out[s2] += cs[s1 * L + s2];
        }
    for (int k = 0; k < L; ++k) {
        rho1_out[k] = tot > 0 ? rho1_out[k] / tot : (rhoj ? 0.0 : rho1[k]);
        rho2_out[k] = tot > 0 ? rho2_out[k] / tot : (rhoj ? 0.0 : rho2[k]);
    }
    if (rhoj && rhoj_out)
        for (int s = 0; s < L2; ++s) rhoj_out[s] = tot > 0 ? cs[s] / tot : rhoj[s];
    free(lrj);

    /* x update: A x' = b, A diagonal */
    double* xn = (double*)malloc(sizeof(double) * L2);
    for (int p = 0; p < L2; ++p) xn[p] = A[p] > tau ? b[p] / A[p] : x[p];
    if (project) oracle_project(xn, L, x_out);
    else memcpy(x_out, xn, sizeof(double) * L2);
    free(xn);

    *ll_out = ll;
    if (b_out) memcpy(b_out, b, sizeof(double) * L2);
    if (A_out) memcpy(A_out, A, sizeof(double) * L2);
    if (colsum_out) memcpy(colsum_out, cs, sizeof(double) * L2);
    free(b);
    return 0;
}

int oracle_em_iter(const float* y, int64_t N, int L, int Ll, int K, double sigma,
                   const double* x, const double* rho1, const double* rho2,
                   int project, double tau,
                   double* x_out, double* rho1_out, double* rho2_out, double* ll_out,
                   double* b_out, double* A_out, double* colsum_out, double* ll_obs_out) {
    return em_iter_impl(y, N, L, Ll, K, sigma, x, rho1, rho2, NULL, project, tau, x_out, rho1_out, rho2_out,
                        NULL, ll_out, b_out, A_out, colsum_out, ll_obs_out);
}

/* NEXT-3: one EM iteration with a joint (non-separable) shift prior rho[s1 L + s2] (PAPER.md:230-231
 * with rho[s] as the weight of shift s; eq:rho_EM as written):
 * rho'[s] = sum_i w^{i,s} / sum_i sum_s' w^{i,s'}.  rho_out [L^2]; rho1_out / rho2_out its marginals. */
int oracle_em_iter_joint(const float* y, int64_t N, int L, int Ll, int K, double sigma,
                         const double* x, const double* rho, int project, double tau,
                         double* x_out, double* rho_out, double* rho1_out, double* rho2_out, double* ll_out,
                         double* b_out, double* A_out, double* colsum_out, double* ll_obs_out) {
    return em_iter_impl(y, N, L, Ll, K, sigma, x, NULL, NULL, rho, project, tau, x_out, rho1_out, rho2_out,
                        rho_out, ll_out, b_out, A_out, colsum_out, ll_obs_out);
}
