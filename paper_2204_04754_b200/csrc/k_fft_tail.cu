// k_fft_tail.cu — everything of an FFT-path iteration after the E/M kernel, as ONE cooperative
// kernel whose phases are separated by grid-wide barriers (one launch instead of four latency-bound
// single-block kernels).  All arithmetic is float64.
//
//   phase R  (a5)  fixed-order sum of the per-CTA float32 partials of k_fft_em (deterministic)
//   phase F  (a5, a7)  b_r = irfft2(Bhat_r) / L_low^2 scattered to b[(K m - r) mod L]   (eq:x_EM numerator,
//                  PAPER.md:255-263 with P^{-1} := P^T), Bhat_{2q} = (U_q+V_q)/2, Bhat_{2q+1} = i(U_q-V_q)/2,
//                  and in the same item x' = b / A: every pixel of b_r divides by the class mass of class r
//                  (A[p] is the mass of class (-p mod K) = r), keep x_t if A <= tau; the last item forms the
//                  class mass, marginals (eq:rho_EM), rho' and the LL
//   phase Q  (a8, a1)  projection x'' = clamp(box3x3(x'), -1, 1) (Algorithm 2 step 2) evaluated
//                  while staging each x''_r, then the next iteration's Xhat_r = rfft2(x''_r)/L_low^2
//                  (pair-interleaved hi + lo), E_r, mean(x''_r) and log2 rho (the E/M kernel derives
//                  the class bias from E_r)
// Two grid barriers per iteration.  With world > 1 the host runs phase R alone, all-reduces the
// accumulators over NCCL, then F and Q.
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "dft64.cuh"
#include "srmra_internal.cuh"

namespace cg = cooperative_groups;

// SRMRA_TAIL_ROLLED (A/B): every loop of the tail rolled, the smallest code (the tail runs once per iteration from a
// cold instruction cache)
#ifdef SRMRA_TAIL_ROLLED
#define TAIL_UNROLL _Pragma("unroll 1")
#define TAIL_INNER _Pragma("unroll 1")
#else
#define TAIL_UNROLL _Pragma("unroll")
#define TAIL_INNER
#endif

namespace srmra {

int fft_partial_bins(int KK, int Ll);
size_t fft_joint_bins(int KK, int Ll);

namespace ffttail {
using namespace dft64;

constexpr int kThreads = 256;
constexpr int kSlices = kThreads / 32;

struct TailArgs {
    unsigned long long* stamps;  // optional phase timestamps (globaltimer, block 0), 8 entries
    int mode;                 // TAIL_* bits
    int L, K, t, project, trace_cap;
    double tau, inv_2s2;
    const float2* part;       // [nparts][PB] float32 partials
    const double* llpart;     // [nparts]
    int nparts, PB;
    double* acc;              // [2 PB + 1] float64 accumulators (+ LL)
    const double* tw;         // cos | sin (2 pi j / L_low)
    double* pack;
    int64_t off_cm, off_m1, off_m2, off_ll;
    double *x64, *rho, *xtmp, *trace;
    float* x32;
    int* flag;
    float2* xhat;             // [2 (hi | lo)][NP][Ll][Lh][2]
    float* par32;             // log2 units: lr1 | lr2 | beta
    double* par64;            // E | E_min
    int nchunk;               // row chunks per class in phase F
    int nchunk_q, wq;         // phase Q: column chunks per class, columns per chunk
    int* iter;                // device iteration counter (t is read here, +1 after finalize) or NULL
    int* run;                 // srmra_run control: [0] stop flag (set here on convergence), [1] first t of the run
    const double* rtol;       // convergence tolerance of the run (0: none)
    int proj_every;           // F of Algorithm 2 (project after t when (t+1) % F == 0; 0 = never)
    // NEXT-3 joint prior (eq:rho_EM as written): per-CTA posterior mass per shift -> jacc -> rho'[s]
    int joint, JB;            // JB = KK Ll^2 bins [r][t1][t2]
    const float* jpart;       // [nparts][JB]
    double* jacc;             // [JB]
    double* rhoj;             // [L][L]
    float2* ljp;              // [NP][Ll n2][Ll n1] log2 rho of (class 2q, class 2q+1)
};

__device__ inline void grid_sync() { cg::this_grid().sync(); }
__device__ inline unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- phase R: bins in rounds of 32, kSlices threads per bin, two rounds per pass.  A thread issues the loads of
// all its partials of both rounds (up to kMaxP each, unrolled and predicated) before the first add: one L2 round
// trip per pass instead of one per group of four partials; the sum over them is a fixed-order chain.
constexpr int kMaxP = 20;
template <bool JOINT>
__device__ void phase_reduce(const TailArgs& a) {
    __shared__ double2 red[2][kSlices][33];
    const int b = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int step = gridDim.x * 32;
    for (int base = blockIdx.x * 32; base < a.PB; base += 2 * step) {
        const int k0 = base + b, k1 = base + step + b;
        double sx0 = 0.0, sy0 = 0.0, sx1 = 0.0, sy1 = 0.0;
        for (int c0 = sl; c0 < a.nparts; c0 += kMaxP * kSlices) {
            float2 v0[kMaxP], v1[kMaxP];
TAIL_UNROLL
            for (int u = 0; u < kMaxP; ++u) {
                const int c = c0 + u * kSlices;
                const float2* pc = a.part + (size_t)c * a.PB;
                v0[u] = (c < a.nparts && k0 < a.PB) ? __ldcg(pc + k0) : make_float2(0.f, 0.f);
                v1[u] = (c < a.nparts && k1 < a.PB) ? __ldcg(pc + k1) : make_float2(0.f, 0.f);
            }
TAIL_UNROLL
            for (int u = 0; u < kMaxP; ++u) {
                sx0 += v0[u].x;
                sy0 += v0[u].y;
                sx1 += v1[u].x;
                sy1 += v1[u].y;
            }
        }
        red[0][sl][b] = make_double2(sx0, sy0);
        red[1][sl][b] = make_double2(sx1, sy1);
        __syncthreads();
        if (sl < 2) {
            const int k = sl ? k1 : k0;
            if (k < a.PB) {
                double tx = 0.0, ty = 0.0;
                for (int j = 0; j < kSlices; ++j) {
                    tx += red[sl][j][b].x;
                    ty += red[sl][j][b].y;
                }
                a.acc[2 * k] = tx;
                a.acc[2 * k + 1] = ty;
            }
        }
        __syncthreads();
    }
    if constexpr (JOINT) {  // joint prior: the per-shift posterior mass, same fixed-order scheme (real bins)
        __shared__ double redj[kSlices][33];
        for (int base = blockIdx.x * 32; base < a.JB; base += gridDim.x * 32) {
            const int k = base + b;
            double sx = 0.0;
            if (k < a.JB) {
                for (int c0 = sl; c0 < a.nparts; c0 += kMaxP * kSlices) {
                    float v[kMaxP];
TAIL_UNROLL
                    for (int u = 0; u < kMaxP; ++u) {
                        const int c = c0 + u * kSlices;
                        v[u] = c < a.nparts ? __ldcg(a.jpart + (size_t)c * a.JB + k) : 0.f;
                    }
TAIL_UNROLL
                    for (int u = 0; u < kMaxP; ++u) sx += v[u];
                }
            }
            redj[sl][b] = sx;
            __syncthreads();
            if (sl == 0 && k < a.JB) {
                double tx = 0.0;
                for (int j = 0; j < kSlices; ++j) tx += redj[j][b];
                a.jacc[k] = tx;
            }
            __syncthreads();
        }
    }
    if (blockIdx.x == 0 && sl == 1) {  // LL partials: strided lanes then a fixed-order shuffle tree
        double s = 0.0;
        for (int c = b; c < a.nparts; c += 32) s += __ldcg(a.llpart + c);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (b == 0) a.acc[2 * a.PB] = s;
    }
}

// class mass: the sum of a line of Ll row sums, by one warp — lane sums of a stride-32 walk, then an xor shuffle
// tree (the same fixed order in every caller, and the same value in every lane).  `pre` holds this lane's values
// (t = lane + 32 j, j < 4, zero past Ll), loaded by the caller together with its other loads.
__device__ __forceinline__ double line_sum(const double (&pre)[4]) {
    double s = ((pre[0] + pre[1]) + pre[2]) + pre[3];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}
template <typename F>
__device__ __forceinline__ void line_load(double (&pre)[4], int Ll, F at) {
    const int lane = threadIdx.x & 31;
TAIL_UNROLL
    for (int j = 0; j < 4; ++j) pre[j] = lane + 32 * j < Ll ? at(lane + 32 * j) : 0.0;
}

// ---- phase F: item (r, ch) -> rows [ch R, ch R + R) of b_r (and x' there when `update`);
//      item KK*nchunk -> mass, marginals, LL (and rho', the LL trace when `update`)
template <bool JOINT>
__device__ void phase_fold(const TailArgs& a, double* sm, bool update) {
    __shared__ double red[32];
    __shared__ double cm_s;
    int bad = 0;
    const int L = a.L, K = a.K, Ll = L / K, Lh = Ll / 2 + 1, KK = K * K, M = Ll - 1, NP = (KK + 1) / 2;
    const int R = Ll / a.nchunk;
    double* cs = sm;
    double* sn = cs + Ll;
    double2* B = reinterpret_cast<double2*>(sn + Ll);  // [Ll][Lh]
    double2* T = B + Ll * Lh;                          // [R][Lh]
    load_tw(a.tw, cs, sn, Ll);
    const double2* A = reinterpret_cast<const double2*>(a.acc);
    const int nitems = KK * a.nchunk + 1;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        __syncthreads();
        if (item < KK * a.nchunk) {
            const int r = item / a.nchunk, ch = item - r * a.nchunk, r1 = r / K, r2 = r % K;
            const int m1a = ch * R;
            // class mass of class r (warp 0, summed as in the marginals item), its loads issued with the first
            // chunk of the B loads: one L2 round trip per chunk of kE bins per thread
            double pre[4] = {0.0, 0.0, 0.0, 0.0};
            const double2* Rr = A + (size_t)2 * NP * Ll * Lh + (size_t)r * Ll;
            if (update && threadIdx.x < 32) line_load(pre, Ll, [&](int t) { return __ldcg(&Rr[t].x); });
            const double2* U = A + (size_t)(r / 2) * 2 * Ll * Lh;
            const double2* V = U + (size_t)Ll * Lh;
            constexpr int kE = 4;
            for (int e0 = threadIdx.x; e0 < Ll * Lh; e0 += kE * blockDim.x) {
                double2 uu[kE], vv[kE];
TAIL_UNROLL
                for (int q = 0; q < kE; ++q) {
                    const int e = e0 + q * blockDim.x;
                    uu[q] = e < Ll * Lh ? __ldcg(U + e) : make_double2(0.0, 0.0);
                    vv[q] = e < Ll * Lh ? __ldcg(V + e) : make_double2(0.0, 0.0);
                }
TAIL_UNROLL
                for (int q = 0; q < kE; ++q) {
                    const int e = e0 + q * blockDim.x;
                    const double2 u = uu[q], v = vv[q];
                    if (e < Ll * Lh)
                        B[e] = (r & 1) ? make_double2(-0.5 * (u.y - v.y), 0.5 * (u.x - v.x))
                                       : make_double2(0.5 * (u.x + v.x), 0.5 * (u.y + v.y));
                }
            }
            if (update && threadIdx.x < 32) {
                const double cmr = line_sum(pre);
                if (threadIdx.x == 0) cm_s = cmr;
            }
            __syncthreads();
            for (int e = threadIdx.x; e < R * Lh; e += blockDim.x) {  // inverse along k1
                const int mm = e / Lh, k2 = e - mm * Lh, m1 = m1a + mm;
                double re = 0, im = 0;
                TAIL_INNER
                for (int k1 = 0; k1 < Ll; ++k1) {
                    const int j = (k1 * m1) & M;
                    const double2 t = B[k1 * Lh + k2];
                    re += t.x * cs[j] - t.y * sn[j];
                    im += t.y * cs[j] + t.x * sn[j];
                }
                T[e] = make_double2(re, im);
            }
            __syncthreads();
            const double inv = 1.0 / ((double)Ll * Ll);
            for (int e = threadIdx.x; e < R * Ll; e += blockDim.x) {  // c2r along k2
                const int mm = e / Ll, m2 = e - mm * Ll, m1 = m1a + mm;
                const double2* Tr = T + mm * Lh;
                double s = Tr[0].x + ((m2 & 1) ? -Tr[Ll / 2].x : Tr[Ll / 2].x);
                TAIL_INNER
                for (int k2 = 1; k2 < Ll / 2; ++k2) {
                    const int j = (k2 * m2) & M;
                    s += 2.0 * (Tr[k2].x * cs[j] - Tr[k2].y * sn[j]);
                }
                const size_t p = (size_t)imod(K * m1 - r1, L) * L + imod(K * m2 - r2, L);
                a.pack[p] = s * inv;
                if (update) {  // eq:x_EM: x' = b / A, keep x_t where the class is unobserved (A <= tau)
                    const double v = cm_s > a.tau ? (s * inv) / cm_s : a.x64[p];
                    bad |= !isfinite(v);
                    a.xtmp[p] = v;
                }
            }
        } else {
            // staged in shared memory (the B / T area is free in this item): row sums R [KK][Ll] (real
            // part) and the class row lines crow_r[k2], k2 <= Ll/2, separated from the pair lines
            // CU [NP][Ll]: crow_{2q} = (CU[k] + conj CU[-k])/2, crow_{2q+1} = (CU[k] - conj CU[-k])/(2i)
            const double2* Rg = A + (size_t)2 * NP * Ll * Lh;
            const double2* CU = Rg + (size_t)KK * Ll;
            double* Rs = reinterpret_cast<double*>(B);            // [KK][Ll]
            double2* crow = reinterpret_cast<double2*>(Rs + KK * Ll);  // [KK][Lh]
            // every load of the item first (chunks of kE elements per thread: one L2 round trip each)
            if (threadIdx.x == 0) a.pack[a.off_ll] = __ldcg(a.acc + 2 * (size_t)a.PB);
            double2 rho_pre[2];  // (rho1[k], rho2[k]) of the update's k = threadIdx.x + u blockDim.x
TAIL_UNROLL
            for (int u = 0; u < 2; ++u) {
                const int k = threadIdx.x + u * blockDim.x;
                rho_pre[u] = (update && !JOINT && k < L) ? make_double2(a.rho[k], a.rho[L + k]) : make_double2(0.0, 0.0);
            }
            constexpr int kE = 4;
            const int nR = KK * Ll, nC = KK * Lh;
            for (int e0 = threadIdx.x; e0 < nR + nC; e0 += kE * blockDim.x) {
                double2 zp[kE], zm[kE];
TAIL_UNROLL
                for (int q = 0; q < kE; ++q) {
                    const int e = e0 + q * blockDim.x;
                    zp[q] = zm[q] = make_double2(0.0, 0.0);
                    if (e < nR) {
                        zp[q].x = __ldcg(&Rg[e].x);
                    } else if (e < nR + nC) {
                        const int ec = e - nR, cls = ec / Lh, k2 = ec - cls * Lh, qq = cls / 2;
                        zp[q] = __ldcg(CU + (size_t)qq * Ll + k2);
                        zm[q] = __ldcg(CU + (size_t)qq * Ll + ((Ll - k2) & M));
                    }
                }
TAIL_UNROLL
                for (int q = 0; q < kE; ++q) {
                    const int e = e0 + q * blockDim.x;
                    if (e < nR) {
                        Rs[e] = zp[q].x;
                    } else if (e < nR + nC) {
                        const int ec = e - nR, cls = ec / Lh;
                        crow[ec] = (cls & 1) ? make_double2(0.5 * (zp[q].y + zm[q].y), 0.5 * (zm[q].x - zp[q].x))
                                             : make_double2(0.5 * (zp[q].x + zm[q].x), 0.5 * (zp[q].y - zm[q].y));
                    }
                }
            }
            __syncthreads();
            for (int rr = threadIdx.x >> 5; rr < KK; rr += blockDim.x >> 5) {  // one warp per class
                double pre[4];
                line_load(pre, Ll, [&](int t) { return Rs[rr * Ll + t]; });
                const double s = line_sum(pre);
                if ((threadIdx.x & 31) == 0) a.pack[a.off_cm + rr] = s;   // class mass sum_i sum_{s in class r} w^{i,s}
            }
            const double invL = 1.0 / Ll;
            // this thread's marginals stay in registers for the rho update (L <= 2 blockDim: at most 2 per thread)
            double m1v[2] = {0.0, 0.0}, m2v[2] = {0.0, 0.0};
TAIL_UNROLL
            for (int u = 0; u < 2; ++u) {
                const int s = threadIdx.x + u * blockDim.x;
                if (s >= L) break;
                const int rs = s % K, t = s / K;
                double a1 = 0.0, a2 = 0.0;
                for (int ro = 0; ro < K; ++ro) {
                    a1 += Rs[(rs * K + ro) * Ll + t];   // marg1[s] = sum_{r2} R_{(rs, r2)}[t]
                    const double2* cr = crow + (ro * K + rs) * Lh;  // marg2[s] = sum_{r1} C_{(r1, rs)}[t]
                    a2 += cr[0].x + ((t & 1) ? -cr[Ll / 2].x : cr[Ll / 2].x);
                    TAIL_INNER
                    for (int k2 = 1; k2 < Ll / 2; ++k2) {
                        const int j = (k2 * t) & M;
                        a2 += 2.0 * (cr[k2].x * cs[j] - cr[k2].y * sn[j]);
                    }
                }
                a.pack[a.off_m1 + s] = a1;
                a.pack[a.off_m2 + s] = a2 * invL;
                m1v[u] = a1;
                m2v[u] = a2 * invL;
            }
            if (JOINT && update) {
                // eq:rho_EM as written: rho'[s] = sum_i w^{i,s} / sum_i sum_s' w^{i,s'} (zero prior mass stays
                // zero); the reported marginals are its row / column sums
                __syncthreads();
                double tot = 0.0;
                for (int s = threadIdx.x; s < L * L; s += blockDim.x) {
                    const int s1 = s / L, s2 = s - s1 * L;
                    const int jb = ((s1 % K) * K + s2 % K) * Ll * Ll + (s1 / K) * Ll + s2 / K;
                    tot += a.rhoj[s] == 0.0 ? 0.0 : fmax(__ldcg(a.jacc + jb), 0.0);
                }
                tot = block_sum(tot, red);
                __syncthreads();
                if (tot > 0.0) {
                    for (int s = threadIdx.x; s < L * L; s += blockDim.x) {
                        const int s1 = s / L, s2 = s - s1 * L;
                        const int jb = ((s1 % K) * K + s2 % K) * Ll * Ll + (s1 / K) * Ll + s2 / K;
                        a.rhoj[s] = a.rhoj[s] == 0.0 ? 0.0 : fmax(__ldcg(a.jacc + jb), 0.0) / tot;
                    }
                }
                __syncthreads();
                for (int k = threadIdx.x; k < L; k += blockDim.x) {
                    double r1 = 0.0, r2 = 0.0;
                    for (int j = 0; j < L; ++j) {
                        r1 += a.rhoj[(size_t)k * L + j];
                        r2 += a.rhoj[(size_t)j * L + k];
                    }
                    a.rho[k] = r1;
                    a.rho[L + k] = r2;
                }
            } else if (update) {
                // eq:rho_EM marginals; zero prior mass stays exactly zero; per-axis normalisation (the marginals
                // from registers, rho prefetched at the top of the item, both sums in one block reduction)
                double m1s = 0.0, m2s = 0.0;
                double g1[2], g2[2];
TAIL_UNROLL
                for (int u = 0; u < 2; ++u) {
                    const int k = threadIdx.x + u * blockDim.x;
                    g1[u] = k < L && rho_pre[u].x != 0.0 ? fmax(m1v[u], 0.0) : 0.0;
                    g2[u] = k < L && rho_pre[u].y != 0.0 ? fmax(m2v[u], 0.0) : 0.0;
                    m1s += g1[u];
                    m2s += g2[u];
                }
                m1s = warp_sum(m1s);
                m2s = warp_sum(m2s);
                __shared__ double red2[2][32];
                if ((threadIdx.x & 31) == 0) {
                    red2[0][threadIdx.x >> 5] = m1s;
                    red2[1][threadIdx.x >> 5] = m2s;
                }
                __syncthreads();
                {
                    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
                    m1s = warp_sum(lane < nw ? red2[0][lane] : 0.0);
                    m2s = warp_sum(lane < nw ? red2[1][lane] : 0.0);
                }
                if (m1s > 0.0 && m2s > 0.0) {
TAIL_UNROLL
                    for (int u = 0; u < 2; ++u) {
                        const int k = threadIdx.x + u * blockDim.x;
                        if (k < L) {
                            a.rho[k] = g1[u] / m1s;
                            a.rho[L + k] = g2[u] / m2s;
                        }
                    }
                }
            }
            if (update && threadIdx.x == 0) {
                const double ll = a.pack[a.off_ll];
                if (a.t < a.trace_cap) a.trace[a.t] = ll;
                bad |= !isfinite(ll);
                // Algorithm 2 stopping rule (srmra_run): |LL_t - LL_{t-1}| <= rtol |LL_t| for t >= run start + 1;
                // the remaining enqueued iterations of the run become no-ops
                const double rt = *a.rtol;
                if (rt > 0.0 && a.t - a.run[1] >= 1 && a.t - 1 < a.trace_cap &&
                    fabs(ll - a.trace[a.t - 1]) <= rt * fabs(ll))
                    a.run[0] = 1;
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.flag, 1);
}

// ---- phase Q: Xhat of the new x (items (r, ch): columns k2 in chunk ch of class r) and the logit bias
// (last item).  Each item stages x_r (float64), transforms its k2 columns along n2 for every row, then
// along n1: no work is repeated across items and the shared memory stays below 227 KB at L_low = 128.
template <bool JOINT>
__device__ void phase_prep(const TailArgs& a, double* sm) {
    const int L = a.L, K = a.K, Ll = L / K, Lh = Ll / 2 + 1, KK = K * K, M = Ll - 1;
    const int Wq = a.wq, nck = a.nchunk_q;
    const int nitems = KK * nck + 1;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        __syncthreads();
        if (item < KK * nck) {
            const int r = item / nck, ch = item - r * nck, r1 = r / K, r2 = r % K;
            const int k2a = ch * Wq, nw = min(Wq, Lh - k2a);
            double* cs = sm;
            double* sn = cs + Ll;
            double* src = sn + Ll;
            double2* tmp = reinterpret_cast<double2*>(src + Ll * Ll);  // [Ll][Wq]
            load_tw(a.tw, cs, sn, Ll);
            // x''_r[m]: after an update, the projection of x' (or x' itself when this iteration does not
            // project); at load time, x_0.  The ch == 0 item of class r also stores x'' and E_r, mean(x''_r)
            const bool from_tmp = (a.mode & TAIL_FINALIZE) != 0;
            double e2 = 0.0, e1 = 0.0;
            // (4 pixels per thread with all 36 stencil loads issued before the first use, and x' stored polyphase by phase
            // F so that every stencil load of a warp is a contiguous run instead of a stride-K gather: neither was faster)
            for (int m = threadIdx.x; m < Ll * Ll; m += blockDim.x) {
                const int m1 = m / Ll, m2 = m - m1 * Ll;
                const int p1 = imod(K * m1 - r1, L), p2 = imod(K * m2 - r2, L);
                double v;
                if (!from_tmp) {
                    v = __ldcg(a.x64 + (size_t)p1 * L + p2);
                } else if (a.project) {
                    const int rm = (p1 == 0 ? L - 1 : p1 - 1) * L, r0 = p1 * L, rp = (p1 == L - 1 ? 0 : p1 + 1) * L;
                    const int cm1 = p2 == 0 ? L - 1 : p2 - 1, cp1 = p2 == L - 1 ? 0 : p2 + 1;
                    const double* xs = a.xtmp;
                    double acc = __ldcg(xs + rm + cm1) + __ldcg(xs + rm + p2) + __ldcg(xs + rm + cp1);
                    acc += __ldcg(xs + r0 + cm1) + __ldcg(xs + r0 + p2) + __ldcg(xs + r0 + cp1);
                    acc += __ldcg(xs + rp + cm1) + __ldcg(xs + rp + p2) + __ldcg(xs + rp + cp1);
                    v = acc / 9.0;
                    v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
                } else {
                    v = __ldcg(a.xtmp + (size_t)p1 * L + p2);
                }
                src[m] = v;
                if (ch == 0) {
                    e2 += v * v;
                    e1 += v;
                    if (from_tmp) a.x64[(size_t)p1 * L + p2] = v;
                    a.x32[(size_t)p1 * L + p2] = (float)v;
                }
            }
            if (ch == 0) {
                __shared__ double redq[32];
                e2 = block_sum(e2, redq);
                __syncthreads();
                e1 = block_sum(e1, redq);
                if (threadIdx.x == 0) {
                    a.par64[r] = e2;                            // E_r = ||x_r||^2
                    a.par64[KK + 1 + r] = e1 / ((double)Ll * Ll);  // mean of x_r (DC term, k_fft128.cu)
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < Ll * nw; e += blockDim.x) {  // along n2: tmp[n1][k2 - k2a]
                const int n1 = e / nw, kk = e - n1 * nw, k2 = k2a + kk;
                const double* row = src + n1 * Ll;
                double re = 0, im = 0;
                TAIL_INNER
                for (int n2 = 0; n2 < Ll; ++n2) {
                    const int j = (k2 * n2) & M;
                    re = fma(row[n2], cs[j], re);
                    im = fma(-row[n2], sn[j], im);
                }
                tmp[n1 * Wq + kk] = make_double2(re, im);
            }
            __syncthreads();
            const double scale = 1.0 / ((double)Ll * Ll);
            float2* out = a.xhat + (size_t)(r / 2) * Ll * Lh * 2 + (r & 1);   // pair-interleaved
            const size_t lo_plane = (size_t)((KK + 1) / 2) * Ll * Lh * 2;         // x_hat = hi + lo
            for (int e = threadIdx.x; e < Ll * nw; e += blockDim.x) {  // along n1: rows k1, columns of the chunk
                const int k1 = e / nw, kk = e - k1 * nw, k2 = k2a + kk;
                double re = 0, im = 0;
                TAIL_INNER
                for (int n1 = 0; n1 < Ll; ++n1) {
                    const int j = (k1 * n1) & M;
                    const double2 t = tmp[n1 * Wq + kk];
                    re += t.x * cs[j] + t.y * sn[j];
                    im += t.y * cs[j] - t.x * sn[j];
                }
                const double vr = re * scale, vi = im * scale;
                const float2 hi = make_float2((float)vr, (float)vi);
                out[((size_t)k1 * Lh + k2) * 2] = hi;
                out[lo_plane + ((size_t)k1 * Lh + k2) * 2] = make_float2((float)(vr - hi.x), (float)(vi - hi.y));
            }
        } else {
            // log2 of the shift marginals (log 0 = -inf); the class bias beta_r = (E_min - E_r) log2(e) /
            // (2 sigma^2) is formed by the E/M kernel from E_r (written by the ch == 0 items)
            for (int k = threadIdx.x; k < L; k += blockDim.x) {
                const double p1 = __ldcg(a.rho + k), p2 = __ldcg(a.rho + L + k);
                a.par32[k] = p1 > 0.0 ? (float)log2(p1) : -INFINITY;
                a.par32[L + k] = p2 > 0.0 ? (float)log2(p2) : -INFINITY;
            }
            if constexpr (JOINT) {  // per-shift log2 prior, pair-interleaved [q][n2][n1] (the E/M kernel's JOINT table)
                const int NPq = (KK + 1) / 2;
                for (int e = threadIdx.x; e < NPq * Ll * Ll; e += blockDim.x) {
                    const int qq = e / (Ll * Ll), rem = e - qq * Ll * Ll, n2 = rem / Ll, n1 = rem - n2 * Ll;
                    float lv[2] = {0.f, 0.f};
                    for (int h = 0; h < 2; ++h) {
                        const int r = 2 * qq + h;
                        if (r >= KK) break;
                        const int s1 = r / K + K * n1, s2 = r % K + K * n2;
                        const double pv = __ldcg(a.rhoj + (size_t)s1 * L + s2);
                        lv[h] = pv > 0.0 ? (float)log2(pv) : -INFINITY;
                    }
                    a.ljp[e] = make_float2(lv[0], lv[1]);
                }
            }
        }
    }
}

// debug (SRMRA_TAIL_STAMPS): the slowest block's item-loop duration of a phase (ns << 12 | its last item), slot k
__device__ inline void stamp_items(const TailArgs& a, int k, unsigned long long t0, int nitems) {
    if (!a.stamps) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        int last = -1;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) last = it;
        atomicMax(a.stamps + k, ((gtime() - t0) << 12) | (unsigned long long)(last & 0xfff));
    }
}

__device__ inline void stamp(const TailArgs& a, int k) {
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[k] = t;
    }
}

template <bool JOINT>
__global__ void __launch_bounds__(kThreads, 1) k_fft_tail(TailArgs a) {
    extern __shared__ double sm[];
    if (*reinterpret_cast<volatile int*>(a.run)) return;  // a converged srmra_run: nothing left to do
    {  // graph-replayable: the iteration index and the projection flag come from the device
        a.t = *reinterpret_cast<volatile int*>(a.iter);
        a.project = a.proj_every > 0 && ((a.t + 1) % a.proj_every == 0);
    }
    bool synced = true;
    stamp(a, 0);
    if (a.stamps && threadIdx.x == 0) {  // earliest block start
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        atomicMin(a.stamps + 6, t0);
    }
    if (a.mode & TAIL_REDUCE) {
        phase_reduce<JOINT>(a);
        synced = false;
    }
    if (a.mode & TAIL_FOLD) {
        if (!synced) grid_sync();
        stamp(a, 1);
        const unsigned long long t0 = a.stamps ? gtime() : 0ull;
        phase_fold<JOINT>(a, sm, (a.mode & TAIL_FINALIZE) != 0);
        stamp_items(a, 2, t0, a.K * a.K * a.nchunk + 1);
        synced = false;
    }
    if (a.mode & TAIL_PREP) {
        if (!synced) grid_sync();
        stamp(a, 4);
        const unsigned long long t0 = a.stamps ? gtime() : 0ull;
        phase_prep<JOINT>(a, sm);
        stamp_items(a, 3, t0, a.K * a.K * a.nchunk_q + 1);
    }
    if (a.stamps) {
        __syncthreads();
        stamp(a, 5);
        if (threadIdx.x == 0) {  // latest block end
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            atomicMax(a.stamps + 7, t1);
        }
    }
    // every block read the counter before its first grid barrier; block 0 passed at least one since
    if (a.iter && (a.mode & TAIL_FINALIZE) && blockIdx.x == 0 && threadIdx.x == 0) *a.iter = a.t + 1;
}

}  // namespace ffttail

using namespace ffttail;

int fft_tail_grid(const srmra_ctx* c) {
    const int PB = fft_partial_bins(c->KK, c->Ll);
    int g = (PB + 31) / 32;
    const int items = c->KK * (c->Ll >= 8 ? c->Ll / 8 : 1) + 1;
    if (g < items) g = items;
    if (g > c->num_sms) g = c->num_sms;
    return g < 1 ? 1 : g;
}

cudaError_t launch_fft_tail(srmra_ctx* c, int mode) {
    const int Ll = c->Ll, Lh = Ll / 2 + 1;
    TailArgs a;
    a.stamps = c->d_stamps;
    a.mode = mode;
    a.L = c->L;
    a.K = c->K;
    a.t = 0;        // both read from the device iteration counter by the kernel (graph-replayable)
    a.project = 0;
    a.iter = c->d_iter;
    a.run = c->d_run;
    a.rtol = c->d_rtol;
    a.proj_every = c->denoiser ? 0 : c->opt.proj_every;  // a denoiser hook replaces the built-in projection
    a.trace_cap = c->opt.trace_cap;
    a.tau = c->tau;
    a.inv_2s2 = c->inv_2s2;
    a.part = c->tail_nparts ? c->tail_part : c->d_part;
    a.llpart = c->tail_nparts ? c->tail_llpart : c->d_llpart;
    a.nparts = c->n_local > 0 ? (c->tail_nparts ? c->tail_nparts : c->fft_grid) : 0;
    a.PB = fft_partial_bins(c->KK, Ll);
    a.acc = c->d_bhat;
    a.tw = c->d_tw;
    a.pack = c->d_pack;
    a.off_cm = c->pk.cmass;
    a.off_m1 = c->pk.m1;
    a.off_m2 = c->pk.m2;
    a.off_ll = c->pk.ll;
    a.x64 = c->d_x64;
    a.rho = c->d_rho;
    a.xtmp = c->d_xtmp;
    a.trace = c->d_trace;
    a.x32 = c->d_x32;
    a.flag = c->d_flag;
    a.xhat = c->d_xhat;
    a.par32 = c->par.f32;
    a.par64 = c->par.f64;
    a.joint = c->fft_joint ? 1 : 0;
    a.JB = (int)fft_joint_bins(c->KK, Ll);
    a.jpart = c->d_jpart;
    a.jacc = c->d_jacc;
    a.rhoj = c->d_rhoj;
    a.ljp = c->d_ljp;
    a.nchunk = Ll >= 8 ? Ll / 8 : 1;
    a.wq = (Lh + a.nchunk - 1) / a.nchunk;
    a.nchunk_q = (Lh + a.wq - 1) / a.wq;
    const int R = Ll / a.nchunk;
    size_t sm_fold = sizeof(double) * 2 * Ll + sizeof(double2) * ((size_t)Ll * Lh + (size_t)R * Lh);
    const size_t sm_marg = sizeof(double) * (2 * Ll + (size_t)c->KK * (Ll + 2 * Lh));  // marginal item staging
    if (sm_marg > sm_fold) sm_fold = sm_marg;
    size_t sm_prep = sizeof(double) * (2 * Ll + (size_t)Ll * Ll) + sizeof(double2) * (size_t)Ll * a.wq;
    const size_t sm = sm_fold > sm_prep ? sm_fold : sm_prep;
    // the joint-prior work is a separate instantiation: the separable tail's code stays as small as before
    // (after an L2 flush its instructions are fetched from HBM)
    auto kern = c->fft_joint ? k_fft_tail<true> : k_fft_tail<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    // same L1 / shared-memory split as the E/M kernel before it: no carve-out reconfiguration between them
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const int grid = fft_tail_grid(c);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers; capturable in a CUDA graph
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace srmra
