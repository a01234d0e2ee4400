// k_gemm.cu — the tcgen05 tensor-core E/M path (SRMRA_PATH_GEMM), fp32-accurate 3xTF32.
//
//   GEMM1 (E-step)  S = Y T(x)^T : S[i,s] = <y_i, P R_s x> = sum_n y_i[n] x[(n1K - s1) mod L, (n2K - s2) mod L]
//                   (PAPER.md:37-38 and the residual expansion of eq:likelihood_EM).
//                   T(x) (L^2 x L_low^2) is never materialised: its rows are windows of the polyphase
//                   component x_r (s = r + K t: T[s][n] = x_r[n - t]); every 16-byte k-chunk of a row is a
//                   16-byte-aligned window of one of 4 pre-rotated, periodically extended copies of x_r
//                   (built by k_gemm_prep, L2-resident), copied into the canonical smem layout by cp.async.
//   softmax         per observation: posterior w^{i,s} (eq:weights_EM, logits as in k_common.cu), LL_i;
//                   writes W^T split into tf32 hi / lo, transposed ([L^2][N]) for GEMM2.
//   GEMM2 (M-step)  Z = W^T Y : Z[s][n] = sum_i w^{i,s} y_i[n]; an all-ones column appended to Y gives
//                   colsum[s] = sum_i w^{i,s} (eq:rho_EM numerator) in the same GEMM.
//   fold            b[p] = sum_n Z[(nK - p) mod L][n]  (eq:x_EM numerator with P^{-1} := P^T).
// The GEMM mainloop: 128x128 output tile per CTA in TMEM (128 columns), K in steps of 32 with a
// 3-stage cp.async ring; one elected thread issues 3 x 4 tcgen05.mma.kind::tf32 (hi*hi, hi*lo, lo*hi)
// per step and commits them to the stage's mbarrier, which the loads of the stage's next use wait on.
#include <math.h>
#include <stdlib.h>

#include "srmra_internal.cuh"
#include "tcgen05.cuh"

namespace srmra {
namespace gemmk {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, THREADS = 128;
// split-K: the K range is cut into KSPLIT contiguous parts accumulated in separate TMEM blocks and
// summed in float64 in the epilogue (fp32 tensor-core accumulation error shrinks ~KSPLIT-fold)
constexpr int KSPLIT = 4;
constexpr int TILE_BYTES = BM * BK * 4;               // one operand tile (16 KB)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;           // A_hi | A_lo | B_hi | B_lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr uint32_t IDESC = tc::idesc_tf32<BM, BN>();

struct GemmArgs {
    // A: rows [M][lda] fp32 hi / lo (K-major)
    const float* a_hi;
    const float* a_lo;
    int64_t lda;
    int M;
    int K;             // contraction length (multiple of 4)
    // B dense: rows [N][ldb] hi / lo
    const float* b_hi;
    const float* b_lo;
    int64_t ldb;
    int N;
    // B implicit T(x) (GEMM1): xe[hi|lo][KK][4 rot][Ll][2 Ll]
    const float* xe;
    int L, Ll, K_ds;
    // C: [M][ldc] fp32
    float* c;
    int64_t ldc;
};

// GEMM column order: j = (r Ll + t1) Ll + t2 for shift s = (r1 + K t1, r2 + K t2), class r = r1 K + r2 — the
// shifts of one class and one t1 are Ll consecutive columns (their T(x) rows are circular shifts of one
// row of x_r, which makes a B tile a rectangular box of the circulant factor used by the TMA mainloop)
__device__ __forceinline__ void j_to_s(int j, int Ll, int K, int& s1, int& s2) {
    const int t2 = j % Ll, rt = j / Ll, t1 = rt % Ll, r = rt / Ll;
    s1 = r / K + K * t1;
    s2 = r % K + K * t2;
}
__device__ __forceinline__ int s_to_j(int s1, int s2, int Ll, int K) {
    return (((s1 % K) * K + (s2 % K)) * Ll + s1 / K) * Ll + s2 / K;
}

// rotated, periodically extended polyphase copies: xe[h][r][rot][row][c] = x_r[row][(c + rot) mod Ll]
__device__ __forceinline__ size_t xe_index(int h, int r, int rot, int row, int c, int KK, int Ll) {
    return ((((size_t)h * KK + r) * 4 + rot) * Ll + row) * (2 * Ll) + c;
}

template <bool IMPLICIT_B>
__global__ void __launch_bounds__(THREADS, 1) k_gemm3(GemmArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned operand area
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t mbar[STAGES];
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

    if (warp == 0) tc::tmem_alloc<BN * KSPLIT>(&tmem_slot);
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) tc::mbar_init(tc::smem_u32(&mbar[s]), 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t taddr = tmem_slot;

    // ---- per-thread load plan: thread tid copies row tid of the A tile and row tid of the B tile
    const int arow = m0 + tid;
    const bool a_ok = arow < g.M;
    const float* a_hi_row = g.a_hi + (size_t)(a_ok ? arow : 0) * g.lda;
    const float* a_lo_row = g.a_lo + (size_t)(a_ok ? arow : 0) * g.lda;
    const int brow = n0 + tid;
    const bool b_ok = brow < g.N;
    const float* b_hi_row = nullptr;
    const float* b_lo_row = nullptr;
    // implicit T: row s = brow -> class r = (s1 mod K, s2 mod K), low-res shift t = (s1 div K, s2 div K);
    // T[s][n1 Ll + n2] = x_r[(n1 - t1) mod Ll][(n2 - t2) mod Ll]; the window of a chunk starting at n2
    // starts at st = (n2 - t2) mod Ll = (st0 + n2) mod Ll with st0 = (-t2) mod Ll; n2 advances by 4 so the
    // rotation rot = st0 & 3 is fixed per row and the extended column is c0 = (st0 & ~3) + n2.
    int t1 = 0, rot = 0, c0base = 0, rcls = 0;
    if (IMPLICIT_B) {
        const int j = b_ok ? brow : 0;  // column order j = (r Ll + t1) Ll + t2
        const int t2 = j % g.Ll;
        t1 = (j / g.Ll) % g.Ll;
        rcls = j / (g.Ll * g.Ll);
        const int st0 = (g.Ll - t2) % g.Ll;
        rot = st0 & 3;
        c0base = st0 - rot;
    } else {
        b_hi_row = g.b_hi + (size_t)(b_ok ? brow : 0) * g.ldb;
        b_lo_row = g.b_lo + (size_t)(b_ok ? brow : 0) * g.ldb;
    }
    const int KKc = g.K_ds * g.K_ds;

    auto load_tile = [&](int kt, int st) {
        unsigned char* sb = base + st * STAGE_BYTES;
        const uint32_t sa_hi = tc::smem_u32(sb), sa_lo = sa_hi + TILE_BYTES;
        const uint32_t sb_hi = sa_lo + TILE_BYTES, sb_lo = sb_hi + TILE_BYTES;
#pragma unroll
        for (int j = 0; j < BK / 4; ++j) {
            const int k = kt * BK + 4 * j;
            const bool kv = k < g.K;
            const uint32_t off = tc::kmajor_off<BK>(tid, 4 * j);
            tc::cp_async16_zfill(sa_hi + off, a_hi_row + (kv ? k : 0), a_ok && kv);
            tc::cp_async16_zfill(sa_lo + off, a_lo_row + (kv ? k : 0), a_ok && kv);
            if (IMPLICIT_B) {
                const int n1 = k / g.Ll, n2 = k - n1 * g.Ll;
                const int row = (n1 - t1 + g.Ll) % g.Ll;
                const size_t ih = xe_index(0, rcls, rot, row, c0base + n2, KKc, g.Ll);
                const size_t il = xe_index(1, rcls, rot, row, c0base + n2, KKc, g.Ll);
                tc::cp_async16_zfill(sb_hi + off, g.xe + (kv ? ih : 0), b_ok && kv);
                tc::cp_async16_zfill(sb_lo + off, g.xe + (kv ? il : 0), b_ok && kv);
            } else {
                tc::cp_async16_zfill(sb_hi + off, b_hi_row + (kv ? k : 0), b_ok && kv);
                tc::cp_async16_zfill(sb_lo + off, b_lo_row + (kv ? k : 0), b_ok && kv);
            }
        }
        tc::cp_async_commit();
    };

    const int nk = (g.K + BK - 1) / BK;
    const int kper = (nk + KSPLIT - 1) / KSPLIT;  // K tiles per split part
    load_tile(0, 0);
    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % STAGES;
        if (kt + 1 < nk) {
            const int st1 = (kt + 1) % STAGES;
            if (kt + 1 >= STAGES) tc::mbar_wait(tc::smem_u32(&mbar[st1]), ((kt + 1) / STAGES - 1) & 1);
            load_tile(kt + 1, st1);
            tc::cp_async_wait<1>();
        } else {
            tc::cp_async_wait<0>();
        }
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t sa = tc::smem_u32(base + st * STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
                const uint32_t o = kk * 256;  // two 16-byte k-chunks per MMA
                const uint64_t ah = tc::kmajor_desc<BK>(sa + o), al = tc::kmajor_desc<BK>(sa + TILE_BYTES + o);
                const uint64_t bh = tc::kmajor_desc<BK>(sa + 2 * TILE_BYTES + o);
                const uint64_t bl = tc::kmajor_desc<BK>(sa + 3 * TILE_BYTES + o);
                const int part = kt / kper;
                const uint32_t td = taddr + (uint32_t)(part * BN);
                tc::mma_tf32(td, ah, bh, IDESC, ((kt - part * kper) | kk) != 0);
                tc::mma_tf32(td, ah, bl, IDESC, 1u);
                tc::mma_tf32(td, al, bh, IDESC, 1u);
            }
            tc::commit(tc::smem_u32(&mbar[st]));
        }
    }
    tc::mbar_wait(tc::smem_u32(&mbar[(nk - 1) % STAGES]), ((nk - 1) / STAGES) & 1);
    tc::fence_after();

    // ---- epilogue: warp w owns TMEM lanes 32w..32w+31 = tile rows; 16 columns per load
    const int row = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < BN; cc += 16) {
        float v[16];
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        const int nparts = (nk + kper - 1) / kper;
        for (int part = 0; part < nparts; ++part) {
            tc::tmem_ld16(taddr + ((uint32_t)(warp * 32) << 16) + part * BN + cc, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] += (double)v[j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = (float)acc[j];
        if (row < g.M) {
            float* dst = g.c + (size_t)row * g.ldc + n0 + cc;
            if (n0 + cc + 16 <= g.N) {
#pragma unroll
                for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
                for (int j = 0; j < 16; ++j)
                    if (n0 + cc + j < g.N) dst[j] = v[j];
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<BN * KSPLIT>(taddr);
}

// ---------------------------------------------------------------- init: tf32 splits of Y and Y^T
// yhl: [2][n][Ll2] (hi | lo);  ythl: [2][Ll2 + 16][ldw] (hi | lo), row Ll2 = ones (colsum), rows beyond 0
__global__ void k_gemm_init(const float* __restrict__ y, int64_t n, int Ll2, int64_t ldw, float* __restrict__ yhl,
                            float* __restrict__ ythl) {
    __shared__ float tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int k0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const size_t plane_y = (size_t)n * Ll2, plane_t = (size_t)(Ll2 + 16) * ldw;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = i0 + r;
        const int k = k0 + tx;
        float v = 0.f;
        if (i < n && k < Ll2) {
            v = y[i * Ll2 + k];
            float hi, lo;
            tc::split_tf32(v, hi, lo);
            yhl[i * Ll2 + k] = hi;
            yhl[plane_y + i * Ll2 + k] = lo;
        }
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int k = k0 + r;
        const int64_t i = i0 + tx;
        if (k < Ll2 && i < ldw) {
            float hi, lo;
            tc::split_tf32(i < n ? tile[tx][r] : 0.f, hi, lo);
            ythl[(size_t)k * ldw + i] = hi;
            ythl[plane_t + (size_t)k * ldw + i] = lo;
        }
    }
}
__global__ void k_gemm_init_ones(int64_t n, int Ll2, int64_t ldw, float* __restrict__ ythl) {
    const size_t plane_t = (size_t)(Ll2 + 16) * ldw;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < 16 * ldw; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / ldw);
        const int64_t i = e - (int64_t)r * ldw;
        ythl[(size_t)(Ll2 + r) * ldw + i] = (r == 0 && i < n) ? 1.f : 0.f;
        ythl[plane_t + (size_t)(Ll2 + r) * ldw + i] = 0.f;
    }
}

// ---------------------------------------------------------------- prep: rotated extended polyphase copies
__global__ void k_gemm_prep(const float* __restrict__ x32, int L, int K, float* __restrict__ xe) {
    const int Ll = L / K, KK = K * K;
    const int total = KK * 4 * Ll * 2 * Ll;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int c = e % (2 * Ll);
        const int row = (e / (2 * Ll)) % Ll;
        const int rot = (e / (2 * Ll * Ll)) % 4;
        const int r = e / (2 * Ll * Ll * 4);
        const int r1 = r / K, r2 = r % K;
        const int m2 = (c + rot) % Ll;
        const float v = x32[(size_t)imod(K * row - r1, L) * L + imod(K * m2 - r2, L)];  // x_r[row][m2]
        float hi, lo;
        tc::split_tf32(v, hi, lo);
        xe[xe_index(0, r, rot, row, c, KK, Ll)] = hi;
        xe[xe_index(1, r, rot, row, c, KK, Ll)] = lo;
    }
}

// ---------------------------------------------------------------- softmax (posterior), transposed W^T
// Block: 8 observations, one warp per row.  Phase 1: the row maximum Sref, then ONE pass forming the
// logits (those of k_common.cu, natural units) with an online (max, argmax, sum); the LL is anchored at
// the argmax shift with an exact float64 residual.  Phase 2: one thread per GEMM column j writes
// w = exp(v - m) / Z of the block's 8 observations as 32 contiguous bytes of row j of W^T (hi and lo).
// Rows n..ldw-1 of the last block are zero (the padding of GEMM2's contraction).
__global__ void __launch_bounds__(256) k_gemm_softmax(const float* __restrict__ S, int64_t n, int L, int K,
                                                      const float* __restrict__ par32, const double* __restrict__ par64,
                                                      const double* __restrict__ ynorm, float inv_s2f, double inv_s2,
                                                      double inv_2s2, int64_t ldw, float* __restrict__ wthl,
                                                      double* __restrict__ llobs, double* __restrict__ ll_out,
                                                      const float* __restrict__ y, const double* __restrict__ x64,
                                                      const double* __restrict__ rho, const float* __restrict__ lrj,
                                                      const double* __restrict__ rhoj) {
    constexpr int R = 8;
    __shared__ float sref_s[R], m_s[R], iz_s[R];
    __shared__ double lls[R];
    const int L2 = L * L, Ll = L / K;
    const float* lr1 = par32;
    const float* lr2 = par32 + L;
    const float* beta = par32 + 2 * L;
    (void)par64;
    (void)ynorm;
    (void)inv_s2;
    const int64_t i0 = (int64_t)blockIdx.x * R;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {
        const int64_t i = i0 + warp;
        if (i < n) {
            const float4* Si4 = reinterpret_cast<const float4*>(S + (size_t)i * L2);
            float mx = -INFINITY;
            for (int q = lane; q < L2 / 4; q += 32) {
                const float4 v4 = __ldcg(Si4 + q);
                mx = fmaxf(fmaxf(mx, fmaxf(v4.x, v4.y)), fmaxf(v4.z, v4.w));
            }
            const float sref = warp_max(mx);
            float vm = -INFINITY, z = 0.f;
            int am = 0;
            for (int q = lane; q < L2 / 4; q += 32) {
                const float4 v4 = __ldcg(Si4 + q);
                const float sv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    int s1, s2;
                    j_to_s(4 * q + u, Ll, K, s1, s2);
                    const int sh = s2 + L * s1;
                    const float v = fmaf(sv[u] - sref, inv_s2f, lr1[s1] + lr2[s2] + beta[(s1 % K) * K + s2 % K] +
                                                                  (lrj ? __ldg(lrj + sh) : 0.f));
                    if (v > vm) {  // online max / sum; argmax ties: the smaller shift index
                        z = (vm == -INFINITY ? 0.f : z * expf(vm - v)) + 1.f;
                        vm = v;
                        am = sh;
                    } else if (v > -INFINITY) {  // zero prior mass (log 0 = -inf) contributes nothing
                        z += expf(v - vm);
                        if (v == vm && sh < am) am = sh;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float v2 = __shfl_xor_sync(0xffffffffu, vm, o), z2 = __shfl_xor_sync(0xffffffffu, z, o);
                const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
                const float M = fmaxf(vm, v2);
                const float zc = (vm == -INFINITY ? 0.f : z * expf(vm - M)) + (v2 == -INFINITY ? 0.f : z2 * expf(v2 - M));
                if (v2 > vm || (v2 == vm && a2 < am)) am = a2;
                vm = M;
                z = zc;
            }
            // log-sum-exp anchored at the argmax shift s*: lse = ell[s*] + log sum_s exp(v_s - v_s*), with
            // ell[s*] = log rho1 + log rho2 - ||y_i - P R_s* x||^2 / (2 sigma^2) from an exact float64 residual,
            // so the fp32 score error only enters through the (small) log-sum term (eq:likelihood_EM)
            const int a1 = am / L, a2 = am - a1 * L;
            double d = 0.0;
            for (int nn = lane; nn < Ll * Ll; nn += 32) {
                const int n1 = nn / Ll, n2 = nn - n1 * Ll;
                const double e = (double)y[(size_t)i * Ll * Ll + nn] - x64[(size_t)imod(n1 * K - a1, L) * L + imod(n2 * K - a2, L)];
                d += e * e;
            }
            d = warp_sum(d);
            if (lane == 0) {
                sref_s[warp] = sref;
                m_s[warp] = vm;
                iz_s[warp] = 1.f / z;
                const double lp = rhoj ? log(rhoj[am]) : log(rho[a1]) + log(rho[L + a2]);  // log prior at s*
                const double lse = lp - d * inv_2s2 + log((double)z);
                if (llobs) llobs[i] = lse;
                lls[warp] = lse;
            }
        } else if (lane == 0) {
            sref_s[warp] = 0.f;
            m_s[warp] = 0.f;
            iz_s[warp] = 0.f;  // padding rows: w = 0
            lls[warp] = 0.0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int r = 0; r < R; ++r) s += lls[r];
        atomicAdd(ll_out, s);
    }
    const size_t plane = (size_t)L2 * ldw;
    for (int j = threadIdx.x; j < L2; j += blockDim.x) {
        int s1, s2;
        j_to_s(j, Ll, K, s1, s2);
        const float bias = lr1[s1] + lr2[s2] + beta[(s1 % K) * K + s2 % K] + (lrj ? __ldg(lrj + s2 + L * s1) : 0.f);
        float hi[R], lo[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float w = 0.f;
            if (i0 + r < n) w = expf(fmaf(__ldcg(S + (size_t)(i0 + r) * L2 + j) - sref_s[r], inv_s2f, bias) - m_s[r]) * iz_s[r];
            tc::split_tf32(w, hi[r], lo[r]);
        }
        float4* dh = reinterpret_cast<float4*>(wthl + (size_t)j * ldw + i0);
        float4* dl = reinterpret_cast<float4*>(wthl + plane + (size_t)j * ldw + i0);
        dh[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
        dh[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
        dl[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
        dl[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
    }
}

// ---------------------------------------------------------------- fold: b[p] = sum_n Z[(nK - p) mod L][n]
__global__ void k_gemm_fold(const float* __restrict__ Z, int64_t ldz, int L, int K, double* __restrict__ b,
                            double* __restrict__ colsum) {
    const int Ll = L / K, Ll2 = Ll * Ll, L2 = L * L;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int p = warp; p < L2; p += nw) {
        const int p1 = p / L, p2 = p - p1 * L;
        double acc = 0.0;
        for (int nn = lane; nn < Ll2; nn += 32) {
            const int n1 = nn / Ll, n2 = nn - n1 * Ll;
            const int j = s_to_j(imod(n1 * K - p1, L), imod(n2 * K - p2, L), Ll, K);
            acc += (double)Z[(size_t)j * ldz + nn];
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            b[p] = acc;
            // colsum of shift s = p (the loop index doubles as a shift): column Ll2 = W^T . ones
            colsum[p] = (double)Z[(size_t)s_to_j(p1, p2, Ll, K) * ldz + Ll2];
        }
    }
}

}  // namespace gemmk

// ==================================================================== host side
using namespace gemmk;

bool gemm_tma_supported(int Ll);
size_t gemm_circ_floats(int L, int K);
cudaError_t launch_gemm_circ(const float* x32, int L, int K, float* cf, cudaStream_t st);

// TMA mainloop (k_gemm_tma.cu) for L_low in {32, 64}; SRMRA_GEMM_TMA=0 selects the cp.async mainloop
static bool use_tma(const srmra_ctx* c) {
    const char* e = getenv("SRMRA_GEMM_TMA");
    return gemm_tma_supported(c->Ll) && !(e && atoi(e) == 0);
}

// L_low <= 64: the fp32 tensor-core accumulation chains (L_low^2 / KSPLIT terms) keep the scores within the
// parity tolerance; at L_low = 128 the FFT path (k_fft128.cu) is the path.
bool gemm_supported(int L, int Ll, int K) { return Ll >= 4 && Ll <= 64 && (Ll % 4) == 0 && L <= 4096 && K * K <= 256; }

// observations padded to a multiple of 8 (the softmax writes 8 observations = 32 B per W^T row segment)
static int64_t ldw_of(int64_t n) { return ((n + 7) / 8) * 8 > 0 ? ((n + 7) / 8) * 8 : 8; }

size_t gemm_bytes(const srmra_ctx* c) {
    const int64_t n = c->n_local, ldw = ldw_of(n);
    size_t b = 0;
    b += sizeof(float) * 2 * (size_t)n * c->Ll2;                 // Y hi/lo
    b += sizeof(float) * 2 * (size_t)(c->Ll2 + 16) * ldw;        // Y^T hi/lo (+ ones row)
    b += sizeof(float) * (size_t)n * c->L2;                      // S
    b += sizeof(float) * 2 * (size_t)c->L2 * ldw;                // W^T hi/lo
    b += sizeof(float) * (size_t)c->L2 * (c->Ll2 + 16);          // Z
    b += sizeof(float) * 2 * (size_t)c->KK * 4 * c->Ll * 2 * c->Ll;  // rotated x copies
    b += sizeof(float) * gemm_circ_floats(c->L, c->K);              // circulant factor (TMA mainloop)
    return b;
}

cudaError_t gemm_alloc(srmra_ctx* c) {
    const int64_t n = c->n_local, ldw = ldw_of(n);
    cudaError_t e;
    if ((e = cudaMalloc(&c->g_yhl, sizeof(float) * (2 * (size_t)n * c->Ll2 + 4))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->g_ythl, sizeof(float) * 2 * (size_t)(c->Ll2 + 16) * ldw)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->g_s, sizeof(float) * ((size_t)n * c->L2 + 4))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->g_wthl, sizeof(float) * 2 * (size_t)c->L2 * ldw)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->g_z, sizeof(float) * (size_t)c->L2 * (c->Ll2 + 16))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->g_xe, sizeof(float) * 2 * (size_t)c->KK * 4 * c->Ll * 2 * c->Ll)) != cudaSuccess) return e;
    if (gemm_tma_supported(c->Ll) &&
        (e = cudaMalloc(&c->g_cf, sizeof(float) * gemm_circ_floats(c->L, c->K))) != cudaSuccess)
        return e;
    c->g_ldw = ldw;
    return cudaFuncSetAttribute(k_gemm3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess
               ? cudaGetLastError()
               : cudaFuncSetAttribute(k_gemm3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
}

void gemm_free(srmra_ctx* c) {
    void* bufs[] = {c->g_yhl, c->g_ythl, c->g_s, c->g_wthl, c->g_z, c->g_xe, c->g_cf};
    for (void* p : bufs)
        if (p) cudaFree(p);
}

cudaError_t launch_gemm_init(srmra_ctx* c) {
    const int64_t n = c->n_local;
    if (n == 0) return cudaSuccess;
    dim3 grid((unsigned)((c->g_ldw + 31) / 32), (unsigned)((c->Ll2 + 31) / 32));
    k_gemm_init<<<grid, 256, 0, c->stream>>>(c->d_y, n, c->Ll2, c->g_ldw, c->g_yhl, c->g_ythl);
    k_gemm_init_ones<<<64, 256, 0, c->stream>>>(n, c->Ll2, c->g_ldw, c->g_ythl);
    return cudaGetLastError();
}

// prep (k_prep of k_common.cu runs first) -> GEMM1 -> softmax -> GEMM2 -> fold; the pack kernel follows
cudaError_t launch_gemm_em(srmra_ctx* c, cudaEvent_t ev_em0, cudaEvent_t ev_em1) {
    const int64_t n = c->n_local;
    const bool tma = use_tma(c);
    if (tma) {
        cudaError_t e = launch_gemm_circ(c->d_x32, c->L, c->K, c->g_cf, c->stream);
        if (e != cudaSuccess) return e;
    } else {
        const int total = c->KK * 4 * c->Ll * 2 * c->Ll;
        k_gemm_prep<<<(total + 255) / 256, 256, 0, c->stream>>>(c->d_x32, c->L, c->K, c->g_xe);
    }
    if (n == 0) return cudaGetLastError();
    if (ev_em0) cudaEventRecord(ev_em0, c->stream);
    if (tma) {
        const size_t cfp = gemm_circ_floats(c->L, c->K) / 2;  // one plane
        cudaError_t e = launch_gemm_tma(c->g_yhl, c->g_yhl + (size_t)n * c->Ll2, n, c->Ll2, c->g_cf, c->g_cf + cfp,
                                        (int64_t)c->KK * c->Ll2, c->Ll, c->L2, c->Ll2, 1, c->Ll, c->g_s, c->L2, c->stream);
        if (e != cudaSuccess) return e;
        k_gemm_softmax<<<(unsigned)(c->g_ldw / 8), 256, 0, c->stream>>>(
            c->g_s, n, c->L, c->K, c->par.f32, c->par.f64, c->d_ynorm, (float)c->inv_s2, c->inv_s2, c->inv_2s2, c->g_ldw,
            c->g_wthl, c->d_llobs, c->d_pack + c->pk.ll, c->d_y, c->d_x64, c->d_rho,
            c->joint ? c->d_lrj : nullptr, c->joint ? c->d_rhoj : nullptr);
        e = launch_gemm_tma(c->g_wthl, c->g_wthl + (size_t)c->L2 * c->g_ldw, c->L2, c->g_ldw, c->g_ythl,
                            c->g_ythl + (size_t)(c->Ll2 + 16) * c->g_ldw, c->Ll2 + 16, c->g_ldw, c->Ll2 + 16, c->g_ldw,
                            0, c->Ll, c->g_z, c->Ll2 + 16, c->stream);
        if (e != cudaSuccess) return e;
        if (ev_em1) cudaEventRecord(ev_em1, c->stream);
        k_gemm_fold<<<(c->L2 * 32 + 255) / 256, 256, 0, c->stream>>>(c->g_z, c->Ll2 + 16, c->L, c->K,
                                                                      c->d_pack + c->pk.b, c->d_colsum);
        return cudaGetLastError();
    }
    GemmArgs g1{};
    g1.a_hi = c->g_yhl;
    g1.a_lo = c->g_yhl + (size_t)n * c->Ll2;
    g1.lda = c->Ll2;
    g1.M = (int)n;
    g1.K = c->Ll2;
    g1.N = c->L2;
    g1.xe = c->g_xe;
    g1.L = c->L;
    g1.Ll = c->Ll;
    g1.K_ds = c->K;
    g1.c = c->g_s;
    g1.ldc = c->L2;
    k_gemm3<true><<<dim3((c->L2 + BN - 1) / BN, (unsigned)((n + BM - 1) / BM)), THREADS, SMEM_BYTES, c->stream>>>(g1);
    k_gemm_softmax<<<(unsigned)(c->g_ldw / 8), 256, 0, c->stream>>>(
        c->g_s, n, c->L, c->K, c->par.f32, c->par.f64, c->d_ynorm, (float)c->inv_s2, c->inv_s2, c->inv_2s2, c->g_ldw,
        c->g_wthl, c->d_llobs, c->d_pack + c->pk.ll, c->d_y, c->d_x64, c->d_rho,
            c->joint ? c->d_lrj : nullptr, c->joint ? c->d_rhoj : nullptr);
    GemmArgs g2{};
    g2.a_hi = c->g_wthl;
    g2.a_lo = c->g_wthl + (size_t)c->L2 * c->g_ldw;
    g2.lda = c->g_ldw;
    g2.M = c->L2;
    g2.K = (int)c->g_ldw;
    g2.b_hi = c->g_ythl;
    g2.b_lo = c->g_ythl + (size_t)(c->Ll2 + 16) * c->g_ldw;
    g2.ldb = c->g_ldw;
    g2.N = c->Ll2 + 16;
    g2.c = c->g_z;
    g2.ldc = c->Ll2 + 16;
    k_gemm3<false><<<dim3((g2.N + BN - 1) / BN, (c->L2 + BM - 1) / BM), THREADS, SMEM_BYTES, c->stream>>>(g2);
    if (ev_em1) cudaEventRecord(ev_em1, c->stream);
    k_gemm_fold<<<(c->L2 * 32 + 255) / 256, 256, 0, c->stream>>>(c->g_z, c->Ll2 + 16, c->L, c->K,
                                                                  c->d_pack + c->pk.b, c->d_colsum);
    return cudaGetLastError();
}

}  // namespace srmra
