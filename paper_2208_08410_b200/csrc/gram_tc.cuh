// gram_tc.cuh — B0 = A^T A on the 5th-generation tensor cores (tcgen05, kind::tf32), for the
// explicit-Gram path (TSVD_OPT_METHOD = 1; Alg. 3's Gram, with the symmetric task schedule
// of P:347-348: only the tiles touching the upper triangle are computed, the rest is mirrored).
//
// C[i, j] = sum_r A[r, i] A[r, j]: M = the i columns, N = the j columns, K = the rows of the slab.
// Both operands are column blocks of the row-major slab, so both are MN-major in the MMA's terms.
// One persistent CTA per SM walks a tile list (BM x BN = 128 x 256 output tiles, grouped so that the
// SMs working at the same time share operand column blocks in L2); per tile the K loop streams
// BK-row chunks of the two column blocks through a ring of shared-memory stages:
//   warp 0  (one thread)  TMA producer: 2-D tensor loads (128-byte swizzle, 32-byte atoms) of the raw
//                         fp32 chunks
//   warps 2-5             converter: lo = a - tf32(a) for every element of the chunk (the tensor core
//                         reads fp32 bits and keeps the top 19, i.e. tf32(a) by truncation), written
//                         to the stage's lo buffers at the same (swizzled) offsets
//   warps 6-9             epilogue: each finished K chunk of the accumulator (TMEM -> registers) is
//                         added into the output, transposed into the lower triangle (gt_fold_t)
//   warp 1  (one thread)  MMA issuer: per 8-row k-group three tcgen05.mma (M=128, N=256, K=8):
//                         D += A·B, D += A·B_lo, D += A_lo·B  (3xTF32: hi·hi + hi·lo + lo·hi with
//                         hi = the truncation the MMA applies itself, so no hi copy exists) into a
//                         128 x 256 fp32 accumulator in tensor memory; tcgen05.commit frees the stage.
//                         The tensor core's accumulation rounds toward zero (measured: a relative bias
//                         ~K 2^-25 on sums of K positive terms, 1e-3 at K = 65536), so it only sums
//                         K chunks of 512 rows, into two accumulators used in turn; the epilogue warps
//                         add each finished chunk into the output in fp32 (round to nearest) while the
//                         tensor core fills the other one
// No copy of A (the round-1 path kept 8 GiB of TF32 hi / lo copies for cuBLAS at C2).
#pragma once
#include <cuda.h>

#include "gram_kernels.cuh"

namespace tsvd {

constexpr int kGtBM = 128, kGtBN = 256, kGtBK = 16, kGtStages = 4;
constexpr int kGtConvWarps = 4, kGtEpiWarps = 4;                   // warps 2-5 convert, 6-9 fold chunks
constexpr int kGtThreads = 32 * (2 + kGtConvWarps + kGtEpiWarps);
constexpr int kGtConv = 32 * kGtConvWarps;
constexpr int kGtChunkBytes = kGtBK * 128;                         // one 32-column x BK-row TMA box
constexpr int kGtABytes = (kGtBM / 32) * kGtChunkBytes;            // 8 KB
constexpr int kGtBBytes = (kGtBN / 32) * kGtChunkBytes;            // 16 KB
constexpr int kGtStageBytes = 2 * (kGtABytes + kGtBBytes);         // raw + lo: 48 KB
constexpr int kGtSmem = kGtStages * kGtStageBytes + 1024 + 256;    // + alignment + barriers
constexpr int kGtTmemCols = 512;                                   // two fp32 accumulators (N columns each)
constexpr int kGtChunkStages = 512 / kGtBK;  // K rows summed inside the tensor core per chunk: 512

struct GtParams {
    const int2 *tiles;   // (I, J) tile list, in schedule order
    int ntiles;
    int64_t n;           // B0 is n x n, row stride ldb
    int64_t ldb;
    int64_t m;           // rows of the slab (K)
    float *B;
};

__device__ __forceinline__ uint32_t gt_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void gt_tma_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(gt_smem(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(gt_smem(bar))
        : "memory");
}

// shared-memory matrix descriptor, MN-major tf32: the only smem layout the tensor core takes for
// 32-bit MN-major operands is the 128-byte swizzle with 32-byte atoms (layout type 1,
// "SWIZZLE_128B_BASE32B"; the TMA writes it with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 128-byte rows
// (32 elements along M / N) in groups of 4 rows.  LBO = stride between 32-element column chunks,
// SBO = stride between 4-row groups (512 B), version 1 (sm_100)
__device__ __forceinline__ uint64_t gt_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
    return d;
}

// instruction descriptor: D fp32, A / B tf32, both MN-major, M = 128, N = 256
constexpr uint32_t kGtIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                              ((uint32_t)(kGtBN >> 3) << 17) | ((uint32_t)(kGtBM >> 4) << 24);

__device__ __forceinline__ void gt_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kGtIdesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void gt_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(gt_smem(bar))
                 : "memory");
}

__device__ __forceinline__ void gt_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gt_smem(bar)) : "memory");
}

// shared-memory accesses by 32-bit shared address: the stage pointers are rounded up to the 1 KB
// swizzle alignment through an integer cast, after which the compiler no longer knows they point
// to shared memory and emits generic LD.E / ST.E (ncu: the converter's top stall)
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float lds32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

// lo = a - tf32_trunc(a) (exact in fp32): the part of a the tensor core drops
__device__ __forceinline__ float gt_lo(float a) { return a - __uint_as_float(__float_as_uint(a) & 0xFFFFE000u); }

// lo parts of `count` float4 of a stage: raw at [src + 16 i], lo to [dst + 16 i] for i = t, t + T, ...;
// U loads in flight before their stores (the volatile shared accesses keep program order)
template <int U>
__device__ __forceinline__ void gt_convert(uint32_t src, uint32_t dst, int t, int T, int count) {
    for (int i0 = t; i0 < count; i0 += U * T) {
        float4 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * T < count) a[u] = lds128(src + 16 * (i0 + u * T));
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * T < count)
                sts128(dst + 16 * (i0 + u * T), make_float4(gt_lo(a[u].x), gt_lo(a[u].y), gt_lo(a[u].z), gt_lo(a[u].w)));
    }
}

// the lo parts of a row slab in global memory (LO_GMEM)
__global__ void gram_lo_split(const float *__restrict__ A, int64_t rows, int64_t cols, int64_t ld,
                              float *__restrict__ lo) {
    const int64_t n4 = cols / 4, total = rows * n4;  // ld % 4 == 0 and 16-B aligned rows (TMA contract)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / n4, c = (i - r * n4) * 4;
        const float4 a = *reinterpret_cast<const float4 *>(A + r * ld + c);
        *reinterpret_cast<float4 *>(lo + r * ld + c) = make_float4(gt_lo(a.x), gt_lo(a.y), gt_lo(a.z), gt_lo(a.w));
    }
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows && (cols & 3); r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t c = n4 * 4; c < cols; ++c) lo[r * ld + c] = gt_lo(A[r * ld + c]);
}

// mbarrier phase test without blocking (the epilogue folds a finished chunk when it is ready)
__device__ __forceinline__ bool gt_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(gt_smem(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// 32 consecutive accumulator columns of this warp's TMEM lane quarter (lane = row), waited for
__device__ __forceinline__ void gt_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Fold one 32-column group of a finished accumulator chunk into B, TRANSPOSED.  Lane = row i of the
// tile (tcgen05.ld 32x32b: TMEM lane i, registers = columns jc .. jc + 31); it adds C[i][jc + e] into
// B[jc + e][i] — B is symmetric, so the tile lands in the other triangle and gram_mirror_to_upper
// completes B afterwards.  For each e the warp's 32 lanes touch 32 consecutive floats of one row of
// B: one 128-byte line per instruction (the row-per-thread float4 RMW touched 32 lines per instruction
// and was ~9 % of the single-CTA kernel's L1 wavefronts, ncu).  Each element is read, added (round to
// nearest) and written by one thread, chunk after chunk in order: deterministic.
__device__ __forceinline__ void gt_fold_t(float *__restrict__ B, int64_t ldb, int64_t n, int64_t i, int64_t jc,
                                          const uint32_t (&v)[32], bool first) {
    if (i >= n) return;
    float old[32];
    if (!first) {
#pragma unroll
        for (int e = 0; e < 32; ++e) old[e] = jc + e < n ? B[(jc + e) * ldb + i] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 32; ++e)
        if (jc + e < n) B[(jc + e) * ldb + i] = first ? __uint_as_float(v[e]) : old[e] + __uint_as_float(v[e]);
}

// LO_GMEM: the lo parts come from a precomputed copy in global memory (map_lo, one elementwise pass
// over A before the kernel) by TMA like the raw chunks, instead of the converter warps — less
// shared-memory traffic per stage (no converter read + write), one more copy of A in HBM
template <bool LO_GMEM>
__global__ void __launch_bounds__(kGtThreads, 1)
    gram_tc(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap map_lo, const GtParams p) {
    extern __shared__ unsigned char gt_raw[];
    unsigned char *smem = (unsigned char *)(((uintptr_t)gt_raw + 1023) & ~(uintptr_t)1023);  // swizzle: 1 KB
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kGtStages * kGtStageBytes);         // TMA landed
    uint64_t *conv = full + kGtStages;    // lo buffers written (kGtConv converter threads)
    uint64_t *empty = conv + kGtStages;   // the stage's MMAs completed
    uint64_t *dfull = empty + kGtStages;  // [2] accumulator buffer b holds a finished K chunk
    uint64_t *dempty = dfull + 2;         // [2] the epilogue has folded buffer b into the output
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(dempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (int)((p.m + kGtBK - 1) / kGtBK);
    const int nchunk = (nk + kGtChunkStages - 1) / kGtChunkStages;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kGtStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], kGtConv);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], 32 * kGtEpiWarps);
        }
        fence_barrier_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gt_smem(tmem_slot)),
                     "n"(kGtTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    // Work order: rounds of two tiles per CTA (t0 = r 2G + b, t1 = t0 + G, G = grid), and inside a round
    // K-chunk-major: chunk k of t0, chunk k of t1, chunk k + 1 of t0, ...  Every CTA is at about the
    // same K chunk of a compact block of tiles at the same time, so one chunk's operand rows (a few MB)
    // are read from DRAM once and served from L2 to all SMs; the two tiles alternate between the two
    // TMEM accumulators, so one tile's chunk is folded while the other's is multiplied.
    // job j (0, 1, 2, ... in that order) uses accumulator j & 1.
#define GT_FOR_JOBS(...)                                                                           \
    for (int r0 = blockIdx.x; r0 < p.ntiles; r0 += 2 * gridDim.x) {                                \
        const int nt = r0 + (int)gridDim.x < p.ntiles ? 2 : 1;                                     \
        const int2 tl[2] = {p.tiles[r0], p.tiles[nt == 2 ? r0 + gridDim.x : r0]};                  \
        for (int k = 0; k < nchunk; ++k)                                                           \
            for (int u = 0; u < nt; ++u) {                                                         \
                const int2 tile = tl[u];                                                           \
                const int kb0 = k * kGtChunkStages;                                                \
                const int kb1 = kb0 + kGtChunkStages < nk ? kb0 + kGtChunkStages : nk;             \
                __VA_ARGS__                                                                        \
            }                                                                                      \
    }

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer
            int s = 0;
            uint32_t ph = 0;
            GT_FOR_JOBS({
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char *st = smem + (size_t)s * kGtStageBytes;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)((LO_GMEM ? 2 : 1) * (kGtABytes + kGtBBytes)));
                    for (int c = 0; c < kGtBM / 32; ++c)
                        gt_tma_2d(st + c * kGtChunkBytes, &map, tile.x * kGtBM + 32 * c, kb * kGtBK, &full[s]);
                    for (int c = 0; c < kGtBN / 32; ++c)
                        gt_tma_2d(st + kGtABytes + c * kGtChunkBytes, &map, tile.y * kGtBN + 32 * c, kb * kGtBK,
                                  &full[s]);
                    if (LO_GMEM) {
                        unsigned char *sl = st + kGtABytes + kGtBBytes;
                        for (int c = 0; c < kGtBM / 32; ++c)
                            gt_tma_2d(sl + c * kGtChunkBytes, &map_lo, tile.x * kGtBM + 32 * c, kb * kGtBK, &full[s]);
                        for (int c = 0; c < kGtBN / 32; ++c)
                            gt_tma_2d(sl + kGtABytes + c * kGtChunkBytes, &map_lo, tile.y * kGtBN + 32 * c,
                                      kb * kGtBK, &full[s]);
                    }
                    if (++s == kGtStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            })
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer
            int s = 0;
            uint32_t ph = 0;
            uint32_t dph[2] = {0u, 0u};
            int buf = 0;
            GT_FOR_JOBS({
                const uint32_t dacc = tmem + (uint32_t)(buf * kGtBN);  // this job's accumulator columns
                mbar_wait(&dempty[buf], dph[buf] ^ 1u);  // the epilogue has folded this buffer's last job
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(LO_GMEM ? &full[s] : &conv[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t base = gt_smem(smem + (size_t)s * kGtStageBytes);
                    const uint32_t a_raw = base, b_raw = base + kGtABytes;
                    const uint32_t a_lo = base + kGtABytes + kGtBBytes, b_lo = a_lo + kGtABytes;
#pragma unroll
                    for (int kk = 0; kk < kGtBK / 8; ++kk) {
                        const uint32_t ko = kk * 1024;  // 8 rows of 128 B
                        const uint64_t da = gt_desc(a_raw + ko, kGtChunkBytes, 512);
                        const uint64_t db = gt_desc(b_raw + ko, kGtChunkBytes, 512);
                        const uint64_t dal = gt_desc(a_lo + ko, kGtChunkBytes, 512);
                        const uint64_t dbl = gt_desc(b_lo + ko, kGtChunkBytes, 512);
                        gt_mma(dacc, da, db, (kb > kb0 || kk > 0) ? 1u : 0u);  // hi·hi (a job's first overwrites)
                        gt_mma(dacc, da, dbl, 1u);                             // hi·lo
                        gt_mma(dacc, dal, db, 1u);                             // lo·hi
                    }
                    gt_commit(&empty[s]);  // frees the stage once these MMAs have read it
                    if (++s == kGtStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                gt_commit(&dfull[buf]);  // the job's partial sum is complete once every MMA above has finished
                dph[buf] ^= 1u;
                buf ^= 1;
            })
        }
    } else if (warp < 2 + kGtConvWarps) {  // ===== converter (warps 2-5)
        if (!LO_GMEM) {
            const int ct = threadIdx.x - 64;  // 0 .. kGtConv - 1
            int s = 0;
            uint32_t ph = 0;
            GT_FOR_JOBS({
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[s], ph);
                    const uint32_t raw = gt_smem(smem + (size_t)s * kGtStageBytes);
                    gt_convert<6>(raw, raw + kGtABytes + kGtBBytes, ct, kGtConv, (kGtABytes + kGtBBytes) / 16);
                    fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
                    gt_arrive(&conv[s]);
                    if (++s == kGtStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            })
        }
    } else {  // ===== epilogue (warps 6-9: TMEM lane quarter q = warp % 4, all 256 columns)
        // a finished job's partial sum (rows i0 + 32 q + lane, columns j0 .. j0 + 255) is added in fp32
        // (round to nearest) into the output, transposed (gt_fold_t) — chunk 0 of a tile stores.  The
        // tensor core's own
        // accumulation rounds toward zero, so its sums stay short (512 rows) and the chunks of a tile are
        // summed here, in chunk order, while the tensor core fills the other accumulator
        const int q = warp & 3;
        uint32_t dph[2] = {0u, 0u};
        int buf = 0;
        GT_FOR_JOBS({
            (void)kb1;
            const int64_t i = (int64_t)tile.x * kGtBM + 32 * q + lane;
            const int64_t j0 = (int64_t)tile.y * kGtBN;
            mbar_wait(&dfull[buf], dph[buf]);
            dph[buf] ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const bool first = k == 0;
#pragma unroll 1
            for (int c = 0; c < kGtBN / 32; ++c) {
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * kGtBN + 32 * c);
                gt_ld32(taddr, v);
                gt_fold_t(p.B, p.ldb, p.n, i, j0 + 32 * c, v, first);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            gt_arrive(&dempty[buf]);
            buf ^= 1;
        })
    }
#undef GT_FOR_JOBS
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGtTmemCols) : "memory");
}

// ---------------------------------------------------------------------------------------------
// gram_tc2: the same product on CTA pairs (2-CTA cluster, tcgen05.mma.cta_group::2, M = N = 256).
// The pair owns a 256 x 256 output tile; each CTA stages half of each operand (A: its 128 of the
// M columns, B: its 128 of the N columns) with the lo parts next to them, so per SM the shared
// memory carries half the B bytes of the single-CTA kernel per MMA and the L2 feeds 8 KB per 8-row
// k-group instead of 12 KB for 1.5x the products (smem: TMA write + converter read/write + MMA reads
// ~125 B/clk at the tensor core's tf32 rate, inside the 128 B/clk port; the single-CTA kernel
// needed ~190 and ran 1.5x above the MMA floor).  Leader = cluster rank 0:
//   both CTAs  warp 0: TMA producer (own halves, own `full` barrier); warps 2-5: converter (lo =
//              a - tf32(a) into own smem, then ONE remote arrive on the leader's `conv`);
//              warps 6-9: epilogue (own TMEM half = output rows 128 rank .. + 127 of the tile,
//              then ONE remote arrive on the leader's `dempty`)
//   leader     warp 1: MMA issuer (waits for both CTAs' converters, issues the pair MMAs, commits
//              multicast to both CTAs' `empty` / `dfull`)
// Summation order of the output is that of gram_tc (512-row chunks folded in chunk order).
constexpr int kG2Tile = 256;                                      // pair tile (M = N = 256)
constexpr int kG2Half = 128;                                      // columns of each operand per CTA
#ifndef TSVD_G2_BK
#define TSVD_G2_BK 16   // rows per ring stage (A/B: 32 with 3 stages)
#endif
constexpr int kG2BK = TSVD_G2_BK;                                 // the tensor map box is 32 x kG2BK
constexpr int kG2Stages = kG2BK == 16 ? 6 : 3;
constexpr int kG2HalfBytes = (kG2Half / 32) * kG2BK * 128;        // 8 KB: 4 TMA boxes of 32 x BK
constexpr int kG2StageBytes = 4 * kG2HalfBytes;                   // A raw, B raw, A lo, B lo: 32 KB
constexpr int kG2Smem = kG2Stages * kG2StageBytes + 1024 + 256;
constexpr int kG2ChunkStages = 512 / kG2BK;
// instruction descriptor: D fp32, A / B tf32, both MN-major, M = 256, N = 256
constexpr uint32_t kG2Idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                              ((uint32_t)(kG2Tile >> 3) << 17) | ((uint32_t)(kG2Tile >> 4) << 24);

__device__ __forceinline__ void g2_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kG2Idesc), "r"(accumulate)
        : "memory");
}
// arrive on the barrier at this CTA-local offset in both CTAs of the pair once the MMAs issued so
// far have completed
__device__ __forceinline__ void g2_commit_both(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            gt_smem(bar)),
        "h"((uint16_t)3)
        : "memory");
}
// arrive on the leader's mbarrier (shared::cluster address) with the default .release.cta semantics:
// the writer threads' fence.proxy.async + the named barrier before it order the stage's smem stores
// for the tensor core; a .release.cluster arrive compiles to MEMBAR.ALL + ERRBAR and, one per stage
// on the converter's critical path, measured 12 % of the pair kernel's stall samples (ncu)
__device__ __forceinline__ void g2_remote_arrive(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void g2_named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__global__ void __launch_bounds__(kGtThreads, 1)
    gram_tc2(const __grid_constant__ CUtensorMap map, const GtParams p) {
    extern __shared__ unsigned char g2_raw[];
    unsigned char *smem = (unsigned char *)(((uintptr_t)g2_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kG2Stages * kG2StageBytes);  // own TMA landed
    uint64_t *conv = full + kG2Stages;    // leader: both converters done with the stage (count 2)
    uint64_t *empty = conv + kG2Stages;   // the stage's MMAs completed (multicast commit)
    uint64_t *dfull = empty + kG2Stages;  // [2] accumulator b holds a finished job (multicast commit)
    uint64_t *dempty = dfull + 2;         // [2] leader: both epilogues folded accumulator b (count 2)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(dempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nk = (int)((p.m + kG2BK - 1) / kG2BK);
    const int nchunk = (nk + kG2ChunkStages - 1) / kG2ChunkStages;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kG2Stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 2);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], 2);
        }
        fence_barrier_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    }
    if (warp == 1) {  // both CTAs, same warp: one pair allocation (same TMEM address in both)
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gt_smem(tmem_slot)),
                     "n"(kGtTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / multicast
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

#define G2_FOR_JOBS(...)                                                                           \
    for (int r0 = pair; r0 < p.ntiles; r0 += 2 * npairs) {                                         \
        const int nt = r0 + npairs < p.ntiles ? 2 : 1;                                             \
        const int2 tl[2] = {p.tiles[r0], p.tiles[nt == 2 ? r0 + npairs : r0]};                     \
        for (int k = 0; k < nchunk; ++k)                                                           \
            for (int u = 0; u < nt; ++u) {                                                         \
                const int2 tile = tl[u];                                                           \
                const int kb0 = k * kG2ChunkStages;                                                \
                const int kb1 = kb0 + kG2ChunkStages < nk ? kb0 + kG2ChunkStages : nk;             \
                __VA_ARGS__                                                                        \
            }                                                                                      \
    }

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: this CTA's halves of both operands
            int s = 0;
            uint32_t ph = 0;
            G2_FOR_JOBS({
                const int ca = tile.x * kG2Tile + (int)rank * kG2Half;  // A: M columns of this CTA
                const int cb = tile.y * kG2Tile + (int)rank * kG2Half;  // B: N columns of this CTA
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char *st = smem + (size_t)s * kG2StageBytes;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * kG2HalfBytes));
                    for (int c = 0; c < kG2Half / 32; ++c) {
                        gt_tma_2d(st + c * (kG2BK * 128), &map, ca + 32 * c, kb * kG2BK, &full[s]);
                        gt_tma_2d(st + kG2HalfBytes + c * (kG2BK * 128), &map, cb + 32 * c, kb * kG2BK, &full[s]);
                    }
                    if (++s == kG2Stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            })
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {  // ===== MMA issuer (leader)
            int s = 0;
            uint32_t ph = 0;
            uint32_t dph[2] = {0u, 0u};
            int buf = 0;
            G2_FOR_JOBS({
                const uint32_t dacc = tmem + (uint32_t)(buf * kG2Tile);
                mbar_wait(&dempty[buf], dph[buf] ^ 1u);  // both epilogues folded its last job
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&conv[s], ph);  // both CTAs' raw and lo halves are in place
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t base = gt_smem(smem + (size_t)s * kG2StageBytes);
                    const uint32_t a_raw = base, b_raw = base + kG2HalfBytes;
                    const uint32_t a_lo = base + 2 * kG2HalfBytes, b_lo = base + 3 * kG2HalfBytes;
#pragma unroll
                    for (int kk = 0; kk < kG2BK / 8; ++kk) {
                        const uint32_t ko = kk * 1024;  // 8 rows of 128 B
                        const uint64_t da = gt_desc(a_raw + ko, kG2BK * 128, 512);
                        const uint64_t db = gt_desc(b_raw + ko, kG2BK * 128, 512);
                        const uint64_t dal = gt_desc(a_lo + ko, kG2BK * 128, 512);
                        const uint64_t dbl = gt_desc(b_lo + ko, kG2BK * 128, 512);
                        g2_mma(dacc, da, db, (kb > kb0 || kk > 0) ? 1u : 0u);  // hi·hi
                        g2_mma(dacc, da, dbl, 1u);                             // hi·lo
                        g2_mma(dacc, dal, db, 1u);                             // lo·hi
                    }
                    g2_commit_both(&empty[s]);  // frees the stage in both CTAs
                    if (++s == kG2Stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                g2_commit_both(&dfull[buf]);
                dph[buf] ^= 1u;
                buf ^= 1;
            })
        }
    } else if (warp < 2 + kGtConvWarps) {  // ===== converter (warps 2-5, both CTAs)
        const int ct = threadIdx.x - 64;
        const uint32_t conv_leader = map_to_rank(gt_smem(conv), 0u);
        int s = 0;
        uint32_t ph = 0;
        G2_FOR_JOBS({
            (void)tile;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[s], ph);
                const uint32_t raw = gt_smem(smem + (size_t)s * kG2StageBytes);
                gt_convert<8>(raw, raw + 2 * kG2HalfBytes, ct, kGtConv, (2 * kG2HalfBytes) / 16);
                fence_proxy_async_smem();  // generic stores -> visible to the tensor core (async proxy)
                g2_named_sync(1, kGtConv);
                if (ct == 0) g2_remote_arrive(conv_leader + (uint32_t)(s * sizeof(uint64_t)));
                if (++s == kG2Stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        })
    } else {  // ===== epilogue (warps 6-9, both CTAs): TMEM lane quarter q, all 256 columns
        const int q = warp & 3;
        const int et = threadIdx.x - 32 * (2 + kGtConvWarps);
        const uint32_t dempty_leader = map_to_rank(gt_smem(dempty), 0u);
        uint32_t dph[2] = {0u, 0u};
        int buf = 0;
        G2_FOR_JOBS({
            (void)kb1;
            const int64_t i = (int64_t)tile.x * kG2Tile + (int64_t)rank * kG2Half + 32 * q + lane;
            const int64_t j0 = (int64_t)tile.y * kG2Tile;
            mbar_wait(&dfull[buf], dph[buf]);
            dph[buf] ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const bool first = k == 0;
#pragma unroll 1
            for (int c = 0; c < kG2Tile / 32; ++c) {
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * kG2Tile + 32 * c);
                gt_ld32(taddr, v);
                gt_fold_t(p.B, p.ldb, p.n, i, j0 + 32 * c, v, first);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            g2_named_sync(2, 32 * kGtEpiWarps);
            if (et == 0) g2_remote_arrive(dempty_leader + (uint32_t)(buf * sizeof(uint64_t)));
            buf ^= 1;
        })
    }
#undef G2_FOR_JOBS
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // no multicast commit or remote arrive may target a CTA that has left
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGtTmemCols) : "memory");
}

// ---------------------------------------------------------------------------------------------
// gram_tc3: the CTA-pair product with the A operand in TENSOR MEMORY.  gram_tc2 is shared-memory
// bound (~127 of 128 B/clk per SM: TMA writes, converter reads/writes, and the tensor core reading
// both operands of three MMAs).  Here each CTA's converter reads its A half (M columns) once from a
// plain (unswizzled) shared-memory tile, and writes A and its lo part into a 4-slot TMEM ring with
// tcgen05.st; all three MMAs take A from TMEM (tcgen05.mma ... [d], [a_tmem], b_desc), so the
// shared-memory operand traffic is B only (raw twice, lo once).  TMEM: 2 accumulators of N = 192
// columns + 4 slots x 32 columns of A = 512.  Tiles are 256 (M) x 192 (N), those touching j >= i.
constexpr int kG3M = 256;                                          // pair tile rows (M)
constexpr int kG3AHalf = 128;                                      // per-CTA A columns
constexpr int kG3BK = 16;
static_assert(kG3BK == kGtBK, "the swizzled tensor map box is 32 x kGtBK");
constexpr int kG3Stages = 8;
constexpr int kG3ABytes = kG3AHalf * kG3BK * 4;                    // 8 KB plain [k][m]
constexpr int kG3SlotCols = 2 * (kG3BK / 8) * 8;                   // raw + lo per 8-row k-group: 32
constexpr int kG3ChunkStages = 512 / kG3BK;
// the N-dependent layout: N = 192 (two accumulators + a 4-slot A ring) or 128 (8 slots)
template <int N>
struct G3 {
    static constexpr int BHalf = N / 2;                            // per-CTA B columns
    static constexpr int BBytes = (BHalf / 32) * kG3BK * 128;      // swizzled boxes of 32 x BK
    static constexpr int StageBytes = kG3ABytes + 2 * BBytes;      // A raw, B raw, B lo
    static constexpr int Smem = kG3Stages * StageBytes + 1024 + 512;
    static constexpr int RingCol = 2 * N;                          // A ring after the two accumulators
    static constexpr int Slots = (512 - RingCol) / kG3SlotCols;
    static_assert(Slots >= 2 && BHalf % 32 == 0, "TMEM budget / TMA box width");
    // instruction descriptor: D fp32, A / B tf32, A from TMEM (K-major), B MN-major, M = 256, N
    static constexpr uint32_t Idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) |
                                      ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kG3M >> 4) << 24);
};

__device__ __forceinline__ void g3_mma(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void g3_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}

template <int N>
__global__ void __launch_bounds__(kGtThreads, 1)
    gram_tc3(const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_a, const GtParams p) {
    extern __shared__ unsigned char g3_raw[];
    unsigned char *smem = (unsigned char *)(((uintptr_t)g3_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kG3Stages * G3<N>::StageBytes);  // own TMA landed
    uint64_t *conv = full + kG3Stages;      // leader: both CTAs' B lo + TMEM A slot written (count 2)
    uint64_t *empty = conv + kG3Stages;     // the stage's MMAs completed (multicast commit): smem stage free
    uint64_t *tfree = empty + kG3Stages;    // [slots] the TMEM A slot's MMAs completed (multicast commit)
    uint64_t *dfull = tfree + G3<N>::Slots;     // [2] accumulator b holds a finished job (multicast commit)
    uint64_t *dempty = dfull + 2;           // [2] leader: both epilogues folded accumulator b (count 2)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(dempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nk = (int)((p.m + kG3BK - 1) / kG3BK);
    const int nchunk = (nk + kG3ChunkStages - 1) / kG3ChunkStages;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kG3Stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 2);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < G3<N>::Slots; ++s) mbar_init(&tfree[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], 2);
        }
        fence_barrier_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gt_smem(tmem_slot)),
                     "n"(kGtTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

#define G3_FOR_JOBS(...)                                                                           \
    for (int r0 = pair; r0 < p.ntiles; r0 += 2 * npairs) {                                         \
        const int nt = r0 + npairs < p.ntiles ? 2 : 1;                                             \
        const int2 tl[2] = {p.tiles[r0], p.tiles[nt == 2 ? r0 + npairs : r0]};                     \
        for (int k = 0; k < nchunk; ++k)                                                           \
            for (int u = 0; u < nt; ++u) {                                                         \
                const int2 tile = tl[u];                                                           \
                const int kb0 = k * kG3ChunkStages;                                                \
                const int kb1 = kb0 + kG3ChunkStages < nk ? kb0 + kG3ChunkStages : nk;             \
                __VA_ARGS__                                                                        \
            }                                                                                      \
    }

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: A half (plain), B half (swizzled)
            int s = 0;
            uint32_t ph = 0;
            G3_FOR_JOBS({
                const int ca = tile.x * kG3M + (int)rank * kG3AHalf;
                const int cb = tile.y * N + (int)rank * G3<N>::BHalf;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char *st = smem + (size_t)s * G3<N>::StageBytes;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(kG3ABytes + G3<N>::BBytes));
                    gt_tma_2d(st, &map_a, ca, kb * kG3BK, &full[s]);
                    for (int c = 0; c < G3<N>::BHalf / 32; ++c)
                        gt_tma_2d(st + kG3ABytes + c * (kG3BK * 128), &map_b, cb + 32 * c, kb * kG3BK, &full[s]);
                    if (++s == kG3Stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            })
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {  // ===== MMA issuer (leader)
            int s = 0, slot = 0;
            uint32_t ph = 0;
            uint32_t dph[2] = {0u, 0u};
            int buf = 0;
            G3_FOR_JOBS({
                const uint32_t dacc = tmem + (uint32_t)(buf * N);
                mbar_wait(&dempty[buf], dph[buf] ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&conv[s], ph);  // both CTAs: B lo in smem, A raw / lo in TMEM slot
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t b_raw = gt_smem(smem + (size_t)s * G3<N>::StageBytes + kG3ABytes);
                    const uint32_t b_lo = b_raw + G3<N>::BBytes;
                    const uint32_t ta = tmem + (uint32_t)(G3<N>::RingCol + slot * kG3SlotCols);
#pragma unroll
                    for (int kk = 0; kk < kG3BK / 8; ++kk) {
                        const uint32_t ko = kk * 1024;  // 8 rows of 128 B
                        const uint64_t db = gt_desc(b_raw + ko, kG3BK * 128, 512);
                        const uint64_t dbl = gt_desc(b_lo + ko, kG3BK * 128, 512);
                        const uint32_t a_raw = ta + (uint32_t)(kk * 16), a_lo = a_raw + 8;
                        g3_mma(dacc, a_raw, db, G3<N>::Idesc, (kb > kb0 || kk > 0) ? 1u : 0u);  // hi·hi
                        g3_mma(dacc, a_raw, dbl, G3<N>::Idesc, 1u);                             // hi·lo
                        g3_mma(dacc, a_lo, db, G3<N>::Idesc, 1u);                               // lo·hi
                    }
                    g2_commit_both(&empty[s]);     // smem stage free in both CTAs
                    g2_commit_both(&tfree[slot]);  // TMEM A slot free in both CTAs
                    if (++s == kG3Stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                    if (++slot == G3<N>::Slots) slot = 0;
                }
                g2_commit_both(&dfull[buf]);
                dph[buf] ^= 1u;
                buf ^= 1;
            })
        }
    } else if (warp < 2 + kGtConvWarps) {  // ===== converter (warps 2-5, both CTAs)
        // thread -> TMEM lane (A row m): warp w may only access lanes 32 (w % 4) .. + 31
        const int ct = threadIdx.x - 64;
        const int m = 32 * (warp & 3) + lane;
        const uint32_t conv_leader = map_to_rank(gt_smem(conv), 0u);
        int s = 0, slot = 0, seq = 0;
        uint32_t ph = 0;
        G3_FOR_JOBS({
            (void)tile;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[s], ph);
                const uint32_t st = gt_smem(smem + (size_t)s * G3<N>::StageBytes);
                // A: row m, k = 0..15 from the plain [k][m] tile (loads issued first)
                float r0[16], r1[16];  // per 8-row k-group: raw k0..7, lo k0..7
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    r0[e] = lds32(st + 4u * (uint32_t)(e * kG3AHalf + m));
                    r1[e] = lds32(st + 4u * (uint32_t)((8 + e) * kG3AHalf + m));
                }
                // B: lo parts next to the raw ones (same swizzled positions)
                gt_convert<(G3<N>::BBytes / 16 + kGtConv - 1) / kGtConv>(st + kG3ABytes, st + kG3ABytes + G3<N>::BBytes, ct, kGtConv, G3<N>::BBytes / 16);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    r0[8 + e] = gt_lo(r0[e]);
                    r1[8 + e] = gt_lo(r1[e]);
                }
                // the slot's previous MMAs must have completed before it is overwritten
                if (seq >= G3<N>::Slots) mbar_wait(&tfree[slot], (uint32_t)((seq / G3<N>::Slots - 1) & 1));
                const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(G3<N>::RingCol + slot * kG3SlotCols);
                g3_st16(ta, r0);
                g3_st16(ta + 16, r1);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                fence_proxy_async_smem();  // B lo (generic stores) -> visible to the tensor core
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                g2_named_sync(1, kGtConv);
                if (ct == 0) g2_remote_arrive(conv_leader + (uint32_t)(s * sizeof(uint64_t)));
                if (++s == kG3Stages) {
                    s = 0;
                    ph ^= 1u;
                }
                if (++slot == G3<N>::Slots) slot = 0;
                ++seq;
            }
        })
    } else {  // ===== epilogue (warps 6-9, both CTAs): TMEM lane quarter q, all N columns
        const int q = warp & 3;
        const int et = threadIdx.x - 32 * (2 + kGtConvWarps);
        const uint32_t dempty_leader = map_to_rank(gt_smem(dempty), 0u);
        uint32_t dph[2] = {0u, 0u};
        int buf = 0;
        G3_FOR_JOBS({
            (void)kb1;
            const int64_t i = (int64_t)tile.x * kG3M + (int64_t)rank * kG3AHalf + 32 * q + lane;
            const int64_t j0 = (int64_t)tile.y * N;
            mbar_wait(&dfull[buf], dph[buf]);
            dph[buf] ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const bool first = k == 0;
#pragma unroll 1
            for (int c = 0; c < N / 32; ++c) {
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * N + 32 * c);
                gt_ld32(taddr, v);
                gt_fold_t(p.B, p.ldb, p.n, i, j0 + 32 * c, v, first);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            g2_named_sync(2, 32 * kGtEpiWarps);
            if (et == 0) g2_remote_arrive(dempty_leader + (uint32_t)(buf * sizeof(uint64_t)));
            buf ^= 1;
        })
    }
#undef G3_FOR_JOBS
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGtTmemCols) : "memory");
}

// strictly-upper triangle from the lower one (the epilogues stored every tile transposed, so every
// (i, j) with i >= j holds its value); 32 x 32 tiles through shared memory, both sides coalesced
__global__ void gram_mirror_to_upper(float *__restrict__ B, int64_t n, int64_t ldb) {
    __shared__ float tile[32][33];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;  // destination tile (rows bi, columns bj), bi <= bj
    if (bi > bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {  // source: rows of tile (bj, bi)
        const int64_t r = bj * 32 + k, c = bi * 32 + tx;
        if (r < n && c < n) tile[k][tx] = B[r * ldb + c];
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = bi * 32 + k, c = bj * 32 + tx;  // B[r][c] = B[c][r] for r < c
        if (r < n && c < n && r < c) B[r * ldb + c] = tile[tx][k];
    }
}

}  // namespace tsvd
