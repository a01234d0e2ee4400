// k_gemm_tma.cu — TMA-fed, warp-specialised tcgen05 3xTF32 mainloop of the GEMM path (L_low in {32, 64}).
//
// The cp.async mainloop of k_gemm.cu (k_gemm3) is bound by the L1TEX / LSU path its 16-byte operand
// copies take (ncu: L1TEX 80 % busy, L2 19 %, tensor pipe 14 % at c1).  Here every operand tile is
// one or a few TMA boxes (cp.async.bulk.tensor, 128-byte swizzle), which bypass the LSU:
//   GEMM1  S = Y T(x)^T:  A = Y hi / lo [N][Ll^2]; B = T(x) in the GEMM column order j = (r, t1, t2)
//          (k_gemm.cu): for one class r and one t1 the Ll rows t2 of T at k-row n1 are the circular
//          shifts of row rho = (n1 - t1) mod Ll of x_r, i.e. a rectangular box of the circulant factor
//          C[r][rho][t2][n2] = x_r[rho][(n2 - t2) mod Ll]  (L^2 Ll floats; T itself, L^2 Ll^2, is never formed)
//   GEMM2  Z = W^T Y:     A = W^T hi / lo [L^2][ldw]; B = Y^T hi / lo [Ll^2 + 16][ldw] (dense)
// Warp 0 issues the TMA loads of a 3-stage ring (full / empty mbarriers), warp 1 the 3 x 4 MMAs per
// 32-wide k-tile (hi.hi, hi.lo, lo.hi) into 4 split-K TMEM blocks of 128 columns, warps 2..5 drain TMEM
// and combine the split-K blocks in float64.  UMMA shared-memory descriptors: K-major, SWIZZLE_128B
// (LBO 16 B, SBO 1024 B, layout type 2 — cute/arch/mma_sm100_desc.hpp), advanced by 32 B per MMA.
#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "srmra_internal.cuh"
#include "tcgen05.cuh"

namespace srmra {
namespace gemmt {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, KSPLIT = 4, THREADS = 192;
constexpr int TILE_BYTES = BM * BK * 4;      // 16 KB: 128 rows x 128 B (one swizzle row each)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;  // A hi | A lo | B hi | B lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr uint32_t IDESC = tc::idesc_tf32<BM, BN>();

struct TmaArgs {
    int M, N, nk;   // C is M x N; nk k-tiles of 32
    int circ, Ll;   // B from the circulant factor (GEMM1) with L_low = Ll, else dense
    float* c;
    int64_t ldc;
    double* c64;    // non-null: float64 atomic accumulation into c64 (K split over blockIdx.z, kz k-tiles each)
    int kz;
    int sym;        // A == B: only the tiles n0 >= m0 are computed (C symmetric)
};

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;    // LBO: 16 B (unused for swizzled K-major)
    d |= (uint64_t)64 << 32;   // SBO: 1024 B between 8-row groups
    d |= (uint64_t)1 << 46;    // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;    // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tma(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
               const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo, TmaArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[STAGES], empty[STAGES], done;
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    if (g.sym && n0 < m0) return;  // the mirror tile holds the transpose
    const int kt0 = blockIdx.z * g.kz, nloc = min(g.nk - kt0, g.kz);

    if (warp == 1) tc::tmem_alloc<BN * KSPLIT>(&tmem_slot);
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(tc::smem_u32(&full[s]), 1);
            tc::mbar_init(tc::smem_u32(&empty[s]), 1);
        }
        tc::mbar_init(tc::smem_u32(&done), 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t taddr = tmem_slot;
    const int kper = (nloc + KSPLIT - 1) / KSPLIT;

    if (warp == 0 && lane == 0) {
        // ---- producer: TMA boxes of tile kt into stage kt % STAGES
        for (int lt = 0; lt < nloc; ++lt) {
            const int kt = kt0 + lt, st = lt % STAGES;
            if (lt >= STAGES) tc::mbar_wait(tc::smem_u32(&empty[st]), ((lt / STAGES) - 1) & 1);
            const uint32_t sb = tc::smem_u32(base + st * STAGE_BYTES), fb = tc::smem_u32(&full[st]);
            mbar_expect_tx(fb, STAGE_BYTES);
            tma_2d(sb, &ta_hi, kt * BK, m0, fb);
            tma_2d(sb + TILE_BYTES, &ta_lo, kt * BK, m0, fb);
            if (!g.circ) {
                tma_2d(sb + 2 * TILE_BYTES, &tb_hi, kt * BK, n0, fb);
                tma_2d(sb + 3 * TILE_BYTES, &tb_lo, kt * BK, n0, fb);
            } else {
                // k = n1 Ll + n2: this tile covers row n1, columns [c0, c0 + 32); the BN columns j are
                // BN / Ll groups (r, t1) of Ll shifts t2 -> box rows ((r Ll + rho) Ll + t2), rho = (n1 - t1) mod Ll
                const int Ll = g.Ll, n1 = (kt * BK) / Ll, c0 = (kt * BK) % Ll;
                for (int grp = 0; grp < BN / Ll; ++grp) {
                    const int rt = (n0 + grp * Ll) / Ll, r = rt / Ll, t1 = rt % Ll;
                    const int rho = (n1 - t1 + Ll) % Ll;
                    const int row = (r * Ll + rho) * Ll;
                    const uint32_t off = (uint32_t)(grp * Ll * BK * 4);
                    tma_2d(sb + 2 * TILE_BYTES + off, &tb_hi, c0, row, fb);
                    tma_2d(sb + 3 * TILE_BYTES + off, &tb_lo, c0, row, fb);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: 3 x 4 tcgen05.mma kind::tf32 per k-tile into split-K block kt / kper
        for (int lt = 0; lt < nloc; ++lt) {
            const int st = lt % STAGES;
            tc::mbar_wait(tc::smem_u32(&full[st]), (lt / STAGES) & 1);
            tc::fence_after();
            const uint32_t sa = tc::smem_u32(base + st * STAGE_BYTES);
            const int part = lt / kper;
            const uint32_t td = taddr + (uint32_t)(part * BN);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
                const uint32_t o = kk * 32;  // 8 tf32 = 32 B along K inside the 128-B swizzle row
                const uint64_t ah = sw128_desc(sa + o), al = sw128_desc(sa + TILE_BYTES + o);
                const uint64_t bh = sw128_desc(sa + 2 * TILE_BYTES + o), bl = sw128_desc(sa + 3 * TILE_BYTES + o);
                tc::mma_tf32(td, ah, bh, IDESC, ((lt - part * kper) | kk) != 0);
                tc::mma_tf32(td, ah, bl, IDESC, 1u);
                tc::mma_tf32(td, al, bh, IDESC, 1u);
            }
            tc::commit(tc::smem_u32(&empty[st]));  // frees the stage once these MMAs have read it
        }
        tc::commit(tc::smem_u32(&done));
    } else if (warp >= 2) {
        // ---- epilogue: warp w drains TMEM lanes 32 (w % 4) .. (tile rows), float64 split-K combine
        tc::mbar_wait(tc::smem_u32(&done), 0);
        tc::fence_after();
        const int q4 = warp & 3;
        const int row = m0 + q4 * 32 + lane;
        const int nparts = (nloc + kper - 1) / kper;
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 16) {
            float v[16];
            double acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0.0;
            for (int part = 0; part < nparts; ++part) {
                tc::tmem_ld16(taddr + ((uint32_t)(q4 * 32) << 16) + part * BN + cc, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] += (double)v[j];
            }
            if (row < g.M && g.c64) {
                double* dst = g.c64 + (size_t)row * g.ldc + n0 + cc;
                for (int j = 0; j < 16; ++j)
                    if (n0 + cc + j < g.N) atomicAdd(dst + j, acc[j]);
            } else if (row < g.M) {
                float* dst = g.c + (size_t)row * g.ldc + n0 + cc;
                if (n0 + cc + 16 <= g.N) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(dst + j) =
                            make_float4((float)acc[j], (float)acc[j + 1], (float)acc[j + 2], (float)acc[j + 3]);
                } else {
                    for (int j = 0; j < 16; ++j)
                        if (n0 + cc + j < g.N) dst[j] = (float)acc[j];
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<BN * KSPLIT>(taddr);
}

// ---------------------------------------------------------------- float64-accumulating variant (NEXT-2)
// C (float64) += A B^T with the float32 TMEM chains kept short: the MMA warp rotates over the 4 TMEM blocks
// of 128 columns, one block per chunk of CH k-tiles (CH x 4 x 3 = 48 MMA accumulations for CH = 4), and 8
// epilogue warps (2 per TMEM lane quadrant, 64 columns each) drain every finished chunk into float64
// registers while the MMA fills the next blocks.  A CTA covers kz k-tiles (blockIdx.z slice); slices are
// combined with float64 atomics (plain stores when there is one slice).  sym: only tiles n0 >= m0.
constexpr int CH = 4, ACC_THREADS = 320;

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

struct Acc64Args {
    int M, N, nk, kz, sym;
    double* c;
    int64_t ldc;
};

__global__ void __launch_bounds__(ACC_THREADS, 1)
    k_gemm_tma_acc64(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                     const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo, Acc64Args g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[STAGES], empty[STAGES], cfull[KSPLIT], cempty[KSPLIT];
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    if (g.sym && n0 < m0) return;
    const int kt0 = blockIdx.z * g.kz, nloc = min(g.nk - kt0, g.kz);
    const int nch = (nloc + CH - 1) / CH;

    if (warp == 1) tc::tmem_alloc<BN * KSPLIT>(&tmem_slot);
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(tc::smem_u32(&full[s]), 1);
            tc::mbar_init(tc::smem_u32(&empty[s]), 1);
        }
        for (int p = 0; p < KSPLIT; ++p) {
            tc::mbar_init(tc::smem_u32(&cfull[p]), 1);
            tc::mbar_init(tc::smem_u32(&cempty[p]), 8);  // one arrival per epilogue warp
        }
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t taddr = tmem_slot;

    if (warp == 0 && lane == 0) {
        for (int lt = 0; lt < nloc; ++lt) {
            const int kt = kt0 + lt, st = lt % STAGES;
            if (lt >= STAGES) tc::mbar_wait(tc::smem_u32(&empty[st]), ((lt / STAGES) - 1) & 1);
            const uint32_t sb = tc::smem_u32(base + st * STAGE_BYTES), fb = tc::smem_u32(&full[st]);
            mbar_expect_tx(fb, STAGE_BYTES);
            tma_2d(sb, &ta_hi, kt * BK, m0, fb);
            tma_2d(sb + TILE_BYTES, &ta_lo, kt * BK, m0, fb);
            tma_2d(sb + 2 * TILE_BYTES, &tb_hi, kt * BK, n0, fb);
            tma_2d(sb + 3 * TILE_BYTES, &tb_lo, kt * BK, n0, fb);
        }
    } else if (warp == 1 && lane == 0) {
        for (int lt = 0; lt < nloc; ++lt) {
            const int ch = lt / CH, part = ch % KSPLIT;
            if (lt % CH == 0 && ch >= KSPLIT) {  // the epilogue has drained this block's previous chunk
                tc::mbar_wait(tc::smem_u32(&cempty[part]), ((ch / KSPLIT) - 1) & 1);
                tc::fence_after();
            }
            const int st = lt % STAGES;
            tc::mbar_wait(tc::smem_u32(&full[st]), (lt / STAGES) & 1);
            tc::fence_after();
            const uint32_t sa = tc::smem_u32(base + st * STAGE_BYTES);
            const uint32_t td = taddr + (uint32_t)(part * BN);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
                const uint32_t o = kk * 32;
                const uint64_t ah = sw128_desc(sa + o), al = sw128_desc(sa + TILE_BYTES + o);
                const uint64_t bh = sw128_desc(sa + 2 * TILE_BYTES + o), bl = sw128_desc(sa + 3 * TILE_BYTES + o);
                tc::mma_tf32(td, ah, bh, IDESC, ((lt % CH) | kk) != 0);
                tc::mma_tf32(td, ah, bl, IDESC, 1u);
                tc::mma_tf32(td, al, bh, IDESC, 1u);
            }
            tc::commit(tc::smem_u32(&empty[st]));
            if (lt % CH == CH - 1 || lt == nloc - 1) tc::commit(tc::smem_u32(&cfull[part]));
        }
    } else if (warp >= 2) {
        const int q4 = warp & 3, half = (warp - 2) >> 2;  // lane quadrant, column half
        double acc[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) acc[j] = 0.0;
        for (int ch = 0; ch < nch; ++ch) {
            const int part = ch % KSPLIT;
            tc::mbar_wait(tc::smem_u32(&cfull[part]), (ch / KSPLIT) & 1);
            tc::fence_after();
            const uint32_t ta = taddr + ((uint32_t)(q4 * 32) << 16) + part * BN + half * 64;
#pragma unroll
            for (int cc = 0; cc < 64; cc += 32) {
                float va[16], vb[16];
                tc::tmem_ld16x2(ta + cc, va, ta + cc + 16, vb);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    acc[cc + j] += (double)va[j];
                    acc[cc + 16 + j] += (double)vb[j];
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tc::smem_u32(&cempty[part]));
        }
        const int row = m0 + q4 * 32 + lane;
        if (row < g.M) {
            double* dst = g.c + (size_t)row * g.ldc + n0 + half * 64;
            const int lim = g.N - (n0 + half * 64);
            const bool single = gridDim.z == 1;
#pragma unroll
            for (int j = 0; j < 64; ++j)
                if (j < lim) {
                    if (single) dst[j] = acc[j];
                    else atomicAdd(dst + j, acc[j]);
                }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<BN * KSPLIT>(taddr);
}

// circulant factor of the polyphase components: cf[h][(r Ll + rho) Ll + t2][n2] = x_r[rho][(n2 - t2) mod Ll],
// tf32 hi (h = 0) / lo (h = 1), x_r[m1][m2] = x[(K m1 - r1) mod L][(K m2 - r2) mod L]
__global__ void k_gemm_circ(const float* __restrict__ x32, int L, int K, float* __restrict__ cf) {
    const int Ll = L / K, KK = K * K;
    const int64_t total = (int64_t)KK * Ll * Ll * Ll;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int n2 = (int)(e % Ll);
        const int t2 = (int)((e / Ll) % Ll);
        const int rho = (int)((e / ((int64_t)Ll * Ll)) % Ll);
        const int r = (int)(e / ((int64_t)Ll * Ll * Ll));
        const int m2 = (n2 - t2 + Ll) % Ll;
        const float v = x32[(size_t)imod(K * rho - r / K, L) * L + imod(K * m2 - r % K, L)];
        float hi, lo;
        tc::split_tf32(v, hi, lo);
        cf[e] = hi;
        cf[total + e] = lo;
    }
}

}  // namespace gemmt

using namespace gemmt;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// row-major float32 [rows][cols] (row pitch `pitch` floats), box [box_rows][32 floats], 128-byte swizzle,
// out-of-range elements read as 0
static bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t pitch, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(pitch * sizeof(float))};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C (float64, zeroed by the caller when the K range is sliced) = A B^T, K sliced in kz k-tiles over
// blockIdx.z (kz <= 0: chosen so that about 2 waves of CTAs cover the SMs), sym as above
cudaError_t launch_gemm_tma_acc64(const float* a_hi, const float* a_lo, int64_t M, int64_t lda, const float* b_hi,
                                  const float* b_lo, int64_t nb_rows, int64_t ldb, int N, int64_t Kdim, double* c,
                                  int64_t ldc, int sym, int num_sms, cudaStream_t st, int* zslices) {
    static PerDeviceOnce attr;
    cudaError_t ea = attr.run([] { return cudaFuncSetAttribute(k_gemm_tma_acc64, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES); });
    if (ea != cudaSuccess) return ea;
    CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
    bool ok = make_map(&ta_hi, a_hi, M, Kdim, lda, BM) && make_map(&ta_lo, a_lo, M, Kdim, lda, BM) &&
              make_map(&tb_hi, b_hi, nb_rows, Kdim, ldb, BN) && make_map(&tb_lo, b_lo, nb_rows, Kdim, ldb, BN);
    if (!ok) return cudaErrorInvalidValue;
    Acc64Args g;
    g.M = (int)M;
    g.N = N;
    g.nk = (int)((Kdim + BK - 1) / BK);
    g.sym = sym;
    g.c = c;
    g.ldc = ldc;
    const int tm = (int)((M + BM - 1) / BM), tn = (N + BN - 1) / BN;
    const int tiles = sym ? tm * (tm + 1) / 2 : tm * tn;
    // z slices: at least ~2 waves of CTAs; among up to 4x that many, the count whose last wave is fullest
    const int want = std::max(1, (2 * num_sms + tiles - 1) / tiles);
    int zb = want;
    double eb = 0.0;
    for (int zz = want; zz <= 4 * want && zz <= std::max(1, g.nk / CH); ++zz) {
        const double ctas = (double)tiles * zz, waves = ceil(ctas / num_sms);
        const double eff = ctas / (waves * num_sms);
        if (eff > eb + 1e-9) { eb = eff; zb = zz; }
    }
    g.kz = std::max(CH, (g.nk + zb - 1) / zb);
    const int z = (g.nk + g.kz - 1) / g.kz;
    if (zslices) *zslices = z;
    dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)z);
    k_gemm_tma_acc64<<<grid, ACC_THREADS, SMEM_BYTES, st>>>(ta_hi, ta_lo, tb_hi, tb_lo, g);
    return cudaGetLastError();
}

bool gemm_tma_supported(int Ll) { return (Ll == 32 || Ll == 64) && encode_fn() != nullptr; }
size_t gemm_circ_floats(int L, int K) { const int Ll = L / K; return (size_t)2 * K * K * Ll * Ll * Ll; }

cudaError_t launch_gemm_circ(const float* x32, int L, int K, float* cf, cudaStream_t st) {
    const int64_t total = (int64_t)K * K * (L / K) * (L / K) * (L / K);
    k_gemm_circ<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(x32, L, K, cf);
    return cudaGetLastError();
}

// C[M][N] = A B^T (both K-major, hi / lo tf32 planes), 3xTF32 with float64 split-K combine.
// c64 != NULL: C is accumulated in float64 with atomics into c64 (zeroed by the caller), the K range split
// over blockIdx.z in slices of kz k-tiles (shorter float32 TMEM chains, more CTAs); sym: A == B, only the
// tiles with n0 >= m0 are computed.
cudaError_t launch_gemm_tma(const float* a_hi, const float* a_lo, int64_t M, int64_t lda, const float* b_hi,
                            const float* b_lo, int64_t nb_rows, int64_t ldb, int N, int64_t Kdim, int circ, int Ll,
                            float* c, int64_t ldc, cudaStream_t st, double* c64, int kz, int sym) {
    static PerDeviceOnce attr;
    cudaError_t ea = attr.run([] { return cudaFuncSetAttribute(k_gemm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES); });
    if (ea != cudaSuccess) return ea;
    CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
    bool ok = make_map(&ta_hi, a_hi, M, Kdim, lda, BM) && make_map(&ta_lo, a_lo, M, Kdim, lda, BM);
    if (circ) ok = ok && make_map(&tb_hi, b_hi, nb_rows, Ll, Ll, Ll) && make_map(&tb_lo, b_lo, nb_rows, Ll, Ll, Ll);
    else ok = ok && make_map(&tb_hi, b_hi, nb_rows, Kdim, ldb, BN) && make_map(&tb_lo, b_lo, nb_rows, Kdim, ldb, BN);
    if (!ok) return cudaErrorInvalidValue;
    TmaArgs g;
    g.M = (int)M;
    g.N = N;
    g.nk = (int)((Kdim + BK - 1) / BK);
    g.circ = circ;
    g.Ll = Ll;
    g.c = c;
    g.ldc = ldc;
    g.c64 = c64;
    g.kz = (c64 && kz > 0) ? kz : g.nk;
    g.sym = sym;
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)((g.nk + g.kz - 1) / g.kz));
    k_gemm_tma<<<grid, THREADS, SMEM_BYTES, st>>>(ta_hi, ta_lo, tb_hi, tb_lo, g);
    return cudaGetLastError();
}

}  // namespace srmra
