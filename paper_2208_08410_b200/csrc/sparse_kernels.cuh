// sparse_kernels.cuh — the Gram-vector product for a CSR row slab (Alg. 4).
//
// Both products of an iteration are one kernel over "segments" (rows of the CSR for N2, columns of
// the slab's CSC for N3) — the gathered vector is read through an fp32 copy (reading R23) and every
// product and sum is fp64:
//   N2 (MODE_T)  t_r = (sum_k val_k y32[col_k]) / ||y_cur|| - U_r . c   (= (X' v)_r, v = y_cur/||y_cur||
//                folded in; deflation in the factored form of Eq. 2), t32[r] = fp32(t_r), per-thread
//                partials of w = U^T t;
//   N2 (MODE_U)  extraction u_r = (A v)_r and per-block sum u_r^2;
//   N3 (MODE_Y)  y_j = sum_k cval_k t32[row_k] over the CSC — the transpose product without atomics and
//                in a fixed order; block 0 also sums the w partials.  y and w land in yw = [y | w].
// The fp64 sums carried from one index block to the next are stored in slice-position order of the
// block that reads them (acc[phase & 1], ping-pong): the reader loads them coalesced at its own
// position, the writer stores at perm[phase][q] — for every block but the last, perm holds the
// segment's position in the NEXT block (rewritten by sell_next at build time), not the segment
// itself.  One scattered access per segment and block instead of two (the kernel is bound by the
// L1TEX unit's scattered sectors, ~1 per clock per SM: ncu).
// Layout (N4b, built once by tsvd_set_csr): the entries are split into K index blocks so that one
// launch's gathers stay inside an L2-resident block of the gathered vector (48 MiB of fp32).  Inside a
// block the segments are stored SELL-32-sigma: segments are sorted by length (descending, stable)
// inside windows of kSellW, cut into slices of 32 (one warp, one segment per lane), and a slice's
// entries are interleaved — entry u of lane l at slice_off + 32 u + l, short segments padded with
// idx = -1 — so every entry load of a warp is one coalesced 128-byte line (a plain CSR row per thread
// costs ~9 L1 wavefronts per load instruction; the random gathers, 1 wavefront per entry, are what
// is left).  perm[] maps a slice lane back to its segment.  The per-segment fp64 sums are carried
// across the K launches in block order (acc) and each segment sums its entries in their order, so
// every result is deterministic.
#pragma once
#include "fin_kernels.cuh"

namespace tsvd {

constexpr int kSpThreads = 256;
// fp32 gather block that stays L2-resident (126 MB L2).  c4n (n = 2^25, ms per Gram pass): 32 and 40 MiB
// (K = 4 blocks) 14.7, 48 and 56 MiB (K = 3) 13.9, 64 MiB (K = 2) 14.7 — fewer blocks carry fewer
// partial sums until the block no longer stays in L2
constexpr size_t kSpL2BlockBytes = 48u << 20;
constexpr int kSpWarps = kSpThreads / 32;
#ifndef TSVD_SP_BATCH
#define TSVD_SP_BATCH 8
#endif
constexpr int kSpBatch = TSVD_SP_BATCH;         // entries (gathers) in flight per lane
constexpr int kSpMaxL = 96;                     // deflation columns the per-thread w partials can hold
constexpr int kSellW = 1024;                    // segments per sorting window (sigma)

enum SpMode { MODE_T = 0, MODE_U = 1, MODE_Y = 2 };

// the random gather of the fp32 vector: TSVD_SP_GATHER = 1 (default) ld.global.cg (L2 only, 3.6 % faster
// per pass on c4n than 0 = the read-only path; ncu: the pass is bound by the L1TEX unit, ~1 scattered
// sector per clock per SM, and an L1 hit rate of 1 % buys nothing)
#ifndef TSVD_SP_GATHER
#define TSVD_SP_GATHER 1
#endif
__device__ __forceinline__ float sp_gather(const float *p) {
#if TSVD_SP_GATHER == 1
    return __ldcg(p);
#else
    return __ldg(p);
#endif
}

// One direction of the product: K blocks of `segs` segments over shared entry arrays, SELL-32-sigma.
struct SpView {
    const int32_t *soff;  // [K][nsl + 1] block-local entry offset of each slice (slice length = diff / 32)
    const int64_t *base;  // [K + 1] first entry of each block
    const int32_t *perm;  // [K][segs] slice lane (32 j + l) -> segment (last block) or its position in the next block
    const int32_t *idx;   // gathered indices (columns for the CSR, local rows for the CSC); -1 = padding
    const float *val;
    int64_t segs, nsl;    // segments, slices per block (ceil(segs / 32))
};

struct SpParams {
    SpView csr;       // rows of the slab by column block (N2)
    SpView csc;       // columns of the slab by row block (N3)
    int64_t rows;
    int64_t n;
    const float *U;   // rows x ldu fp32
    int ldu;
    int l;
    const double *c;
    const double *ybuf;
    int64_t ystride;
    const LoopState *st;
    double *t;        // [rows] MODE_U: u_r (fp64)
    float *t32;       // [rows] MODE_T: t_r rounded to fp32, gathered by N3
    const float *y32; // [n] y_cur rounded to fp32 (written by fin_iter), gathered by N2
    double *wpart;    // [gridDim.x][wpart_ld]
    int wpart_ld;
    double *sq_part;  // [gridDim.x] (MODE_U)
    double *yw;       // N3 output: y (n) | w (l) at wofs
    int64_t wofs;
    int parts;        // gridDim.x of N2 (rows of wpart)
    int phase, nphase;  // launch `phase` of `nphase` covers index block `phase`
    double *acc[2];   // [segs] carried fp64 partial sums when nphase > 1: block b reads acc[b & 1]
                      // (its own position order) and writes acc[(b + 1) & 1]
    int64_t sl0, sl1; // slices [sl0, sl1) of this launch (N3's last block: column chunks, kSellW-aligned)
    const int32_t *blk_idx;  // out of memory (degree 1): this block's entries in a device ring slot
    const float *blk_val;    // (nullptr: the view's resident arrays)
};

// N2 / N3.  LAST: the launch of the last index block (finishes the sums: outputs, deflation, w);
// the others only carry their partial sums.  Dynamic shared memory (MODE_T, LAST): l * (kSpThreads + 1)
// doubles (per-thread w partials, c).
template <int MODE, bool LAST>
#ifndef TSVD_SP_ACC_CS
#define TSVD_SP_ACC_CS 0
#endif
#ifndef TSVD_SP_MINB
#define TSVD_SP_MINB 1
#endif
__global__ void __launch_bounds__(kSpThreads, TSVD_SP_MINB) sp_pass(const SpParams p) {
    extern __shared__ double wsm[];
    __shared__ double red[kSpWarps];
    const LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop || (MODE != MODE_U && st->done)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SpView &V = MODE == MODE_Y ? p.csc : p.csr;
    const float *__restrict__ x = MODE == MODE_Y ? p.t32 : p.y32;
    const int l = (MODE == MODE_T && LAST) ? p.l : 0;
    const bool carry_in = p.phase > 0;
    double *csm = wsm + (int64_t)l * kSpThreads;
    if (MODE == MODE_T && LAST) {
        for (int i = 0; i < l; ++i) wsm[i * kSpThreads + tid] = 0.0;
        for (int i = tid; i < l; i += kSpThreads) csm[i] = p.c[i];
        __syncthreads();
    }
    const double inv = MODE == MODE_Y ? 1.0 : 1.0 / st->ny;
    const int32_t *__restrict__ soff = V.soff + (int64_t)p.phase * (V.nsl + 1);
    const int32_t *__restrict__ perm = V.perm + (int64_t)p.phase * V.segs;
    const int64_t b0 = V.base[p.phase];
    const int32_t *__restrict__ ip = (p.blk_idx ? p.blk_idx : V.idx + b0) + lane;
    const float *__restrict__ vp = (p.blk_val ? p.blk_val : V.val + b0) + lane;
    double sq = 0.0;
    const int64_t nw = (int64_t)gridDim.x * kSpWarps;
    for (int64_t j = p.sl0 + (int64_t)blockIdx.x * kSpWarps + warp; j < p.sl1; j += nw) {
        const int64_t q = 32 * j + lane;
        // this lane's segment (last block) or its position in the next block; -1: past the end
        const int32_t s = q < V.segs ? __ldcs(perm + q) : -1;
#if TSVD_SP_ACC_CS
        const double carried = (carry_in && s >= 0) ? __ldcs(p.acc[p.phase & 1] + q) : 0.0;  // coalesced
#else
        const double carried = (carry_in && s >= 0) ? __ldcg(p.acc[p.phase & 1] + q) : 0.0;  // coalesced
#endif
        const int32_t e0 = __ldg(soff + j), e1 = __ldg(soff + j + 1);  // slice entries [e0, e1), 32 wide
        double sum = 0.0;
        for (int32_t e = e0; e < e1; e += 32 * kSpBatch) {
            int32_t c[kSpBatch];
            float v[kSpBatch], g[kSpBatch];
#pragma unroll
            for (int u = 0; u < kSpBatch; ++u) {  // coalesced: 32 lanes read one 128-byte line
                const bool ok = e + 32 * u < e1;
                c[u] = ok ? __ldcs(ip + e + 32 * u) : -1;  // streaming: read once per pass
                v[u] = ok ? __ldcs(vp + e + 32 * u) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kSpBatch; ++u) g[u] = c[u] >= 0 ? sp_gather(x + c[u]) : 0.f;
#pragma unroll
            for (int u = 0; u < kSpBatch; ++u)
                if (c[u] >= 0) sum += (double)v[u] * (double)g[u];  // entry order
        }
        if (s < 0) continue;
        if (carry_in) sum = carried + sum;  // blocks in order
        if (!LAST) {
#if TSVD_SP_ACC_CS
            __stcs(p.acc[(p.phase + 1) & 1] + s, sum);  // evict-first: keep L2 for the gathered block
#else
            p.acc[(p.phase + 1) & 1][s] = sum;  // at the segment's position in the next block
#endif
            continue;
        }
        if (MODE == MODE_Y) {
            p.yw[s] = sum;
        } else if (MODE == MODE_U) {
            const double u = sum * inv;
            p.t[s] = u;
            sq += u * u;
        } else {
            double t = sum * inv;
            if (l > 0) {  // U_r . c: deflation without forming X' (Eq. 2, factored); w += t U_r
                const float *Ur = p.U + (int64_t)s * p.ldu;
                double corr = 0.0;
                for (int i = 0; i < l; ++i) corr += (double)Ur[i] * csm[i];
                t -= corr;
                for (int i = 0; i < l; ++i) wsm[i * kSpThreads + tid] += t * (double)Ur[i];
            }
            p.t32[s] = (float)t;
        }
    }
    if (!LAST) return;  // not the last block: only the carried sums were written
    if (MODE == MODE_U) {
        sq = warp_sum(sq);
        if (lane == 0) red[warp] = sq;
        __syncthreads();
        if (tid == 0) {
            double a = 0.0;
            for (int w = 0; w < kSpWarps; ++w) a += red[w];
            p.sq_part[blockIdx.x] = a;
        }
    } else if (MODE == MODE_T) {
        __syncthreads();
        for (int i = warp; i < l; i += kSpWarps) {  // threads' partials in thread order
            double a = 0.0;
            for (int jj = lane; jj < kSpThreads; jj += 32) a += wsm[i * kSpThreads + jj];
            a = warp_sum(a);
            if (lane == 0) p.wpart[(int64_t)blockIdx.x * p.wpart_ld + i] = a;
        }
    } else if (blockIdx.x == 0 && p.sl1 == V.nsl) {  // the launch that finishes y also finishes w
        for (int i = warp; i < p.l; i += kSpWarps) {
            double w = 0.0;
            for (int b = lane; b < p.parts; b += 32) w += p.wpart[(int64_t)b * p.wpart_ld + i];
            w = warp_sum(w);
            if (lane == 0) p.yw[p.wofs + i] = w;
        }
    }
}

// ---------------------------------------------------------------- N4b: SELL-32-sigma build (one time)
// one CTA (kSellW threads) per (block, window): sort the window's segments by length, descending and
// stable (bitonic sort of 64-bit keys (~len << 32 | index)), write perm, the inverse position ipos and
// the slice sizes (32 x the longest segment of each slice, the slice's first)
__global__ void __launch_bounds__(kSellW) sell_sort(const unsigned *__restrict__ cnt, int64_t segs,
                                                    int32_t *__restrict__ perm, int32_t *__restrict__ ipos,
                                                    unsigned *__restrict__ ssize, int64_t nsl) {
    __shared__ unsigned long long key[kSellW];
    const int b = blockIdx.y;
    const int64_t w0 = (int64_t)blockIdx.x * kSellW;
    const int i = threadIdx.x;
    const int64_t s = w0 + i;
    const unsigned len = s < segs ? cnt[(int64_t)b * segs + s] : 0u;
    key[i] = s < segs ? ((unsigned long long)(0xFFFFFFFFu - len) << 32) | (unsigned)i : ~0ull;
    __syncthreads();
    for (int k = 2; k <= kSellW; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            const int ixj = i ^ jj;
            if (ixj > i) {
                const unsigned long long a = key[i], c = key[ixj];
                if (((i & k) == 0) == (a > c)) {
                    key[i] = c;
                    key[ixj] = a;
                }
            }
            __syncthreads();
        }
    const unsigned long long kk = key[i];
    if (s < segs) {  // position w0 + i holds a real segment (padding keys sort last)
        const int64_t seg = w0 + (int64_t)(kk & 0xFFFFFFFFu);
        perm[(int64_t)b * segs + s] = (int32_t)seg;
        ipos[(int64_t)b * segs + seg] = (int32_t)s;
        if ((i & 31) == 0) ssize[(int64_t)b * nsl + s / 32] = 32u * (0xFFFFFFFFu - (unsigned)(kk >> 32));
    }
}

// perm[b][q] (b < K - 1) := position of that segment in block b + 1 (the carried sums' write index)
__global__ void sell_next(int32_t *__restrict__ perm, const int32_t *__restrict__ ipos, int K, int64_t segs) {
    const int64_t total = (int64_t)(K - 1) * segs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / segs;
        perm[i] = ipos[(b + 1) * segs + perm[i]];
    }
}

// entry u of the segment at position q (slice q / 32, lane q % 32) goes to soff[slice] + 32 u + lane
__device__ __forceinline__ int64_t sell_dst(const int64_t *flat_sl, int64_t b, int64_t nsl, int32_t q) {
    return flat_sl[b * nsl + q / 32] + (q & 31);
}

// CSR rows -> column-blocked SELL: thread per row, its pieces of block 0, 1, ... in row order
__global__ void sell_from_csr(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                              const float *__restrict__ val, int64_t rows, int K, const unsigned *__restrict__ cnt,
                              const int32_t *__restrict__ ipos, const int64_t *__restrict__ flat_sl, int64_t nsl,
                              int32_t *__restrict__ sidx, float *__restrict__ sval) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = row_ptr[r];
        for (int b = 0; b < K; ++b) {
            const unsigned len = cnt[(int64_t)b * rows + r];
            const int64_t d = sell_dst(flat_sl, b, nsl, ipos[(int64_t)b * rows + r]);
            for (unsigned u = 0; u < len; ++u, ++k) {
                sidx[d + 32 * (int64_t)u] = col[k];
                sval[d + 32 * (int64_t)u] = val[k];
            }
        }
    }
}

// compact blocked segments (flat [K][segs] offsets) -> SELL: thread per (block, segment)
__global__ void sell_from_flat(const int64_t *__restrict__ flat, const int32_t *__restrict__ idx,
                               const float *__restrict__ val, int K, int64_t segs, const int32_t *__restrict__ ipos,
                               const int64_t *__restrict__ flat_sl, int64_t nsl, int32_t *__restrict__ sidx,
                               float *__restrict__ sval) {
    const int64_t total = (int64_t)K * segs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / segs;
        const int64_t d = sell_dst(flat_sl, b, nsl, ipos[i]);
        for (int64_t k = flat[i], u = 0; k < flat[i + 1]; ++k, ++u) {
            sidx[d + 32 * u] = idx[k];
            sval[d + 32 * u] = val[k];
        }
    }
}

// ---------------------------------------------------------------- N4: CSR -> CSC (one time)
// blocked CSC (row block b = r / bwr): entries per [block][column]
__global__ void csc_blk_count(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rows,
                              int64_t n, int64_t bwr, unsigned *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nwarps) {
        unsigned *cb = cnt + (r / bwr) * n;
        for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) atomicAdd(&cb[col[k]], 1u);
    }
}

constexpr int kScanThreads = 1024, kScanItems = 4, kScanTile = kScanThreads * kScanItems;

// exclusive scan of a tile of counts into out (int64), tile total into bsum[blockIdx.x]
__global__ void __launch_bounds__(kScanThreads)
    scan_tiles(const unsigned *__restrict__ in, int64_t n, int64_t *__restrict__ out, int64_t *__restrict__ bsum) {
    __shared__ int64_t wsum[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)tid * kScanItems;
    int64_t v[kScanItems], run = 0;
    for (int q = 0; q < kScanItems; ++q) {
        v[q] = (base + q < n) ? (int64_t)in[base + q] : 0;
        run += v[q];
    }
    int64_t x = run;  // inclusive warp scan of thread totals
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    int64_t excl = x - run + (warp > 0 ? wsum[warp - 1] : 0);
    for (int q = 0; q < kScanItems; ++q) {
        if (base + q < n) out[base + q] = excl;
        excl += v[q];
    }
    if (tid == kScanThreads - 1) bsum[blockIdx.x] = excl;
}

// exclusive scan of the tile totals (one block, sequential chunks per thread), total -> out[n]
__global__ void __launch_bounds__(kScanThreads) scan_totals(int64_t *__restrict__ bsum, int64_t nb, int64_t *__restrict__ total) {
    __shared__ int64_t wsum[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t per = (nb + kScanThreads - 1) / kScanThreads;
    const int64_t b0 = tid * per, b1 = b0 + per < nb ? b0 + per : nb;
    int64_t run = 0;
    for (int64_t b = b0; b < b1; ++b) run += bsum[b];
    int64_t x = run;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    int64_t excl = x - run + (warp > 0 ? wsum[warp - 1] : 0);
    for (int64_t b = b0; b < b1; ++b) {
        const int64_t v = bsum[b];
        bsum[b] = excl;
        excl += v;
    }
    if (tid == kScanThreads - 1) *total = excl;
}

__global__ void scan_add(int64_t *__restrict__ out, int64_t n, const int64_t *__restrict__ bsum) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] += bsum[i / kScanTile];
}

// warp per row: claim a slot in each entry's [row block][column] segment (order inside a segment fixed
// afterwards by csc_sort); the stored row index is local to the slab
__global__ void csc_blk_scatter(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                const float *__restrict__ val, int64_t rows, int64_t n, int64_t bwr,
                                const int64_t *__restrict__ flat, unsigned *__restrict__ fill,
                                int32_t *__restrict__ row_idx, float *__restrict__ cval) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nwarps) {
        const int64_t sb = (r / bwr) * n;
        for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) {
            const int64_t seg = sb + col[k];
            const int64_t pos = flat[seg] + atomicAdd(&fill[seg], 1u);
            row_idx[pos] = (int32_t)r;
            cval[pos] = val[k];
        }
    }
}

// flat exclusive scan over [K][segs] (+ total) -> block bases and int32 block-local offsets
__global__ void flat_to_off(const int64_t *__restrict__ flat, int K, int64_t segs, int32_t *__restrict__ off,
                            int64_t *__restrict__ base) {
    const int64_t total = (int64_t)K * (segs + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / (segs + 1), s = i - b * (segs + 1);
        const int64_t b0 = flat[b * segs];
        off[i] = (int32_t)(flat[b * segs + s] - b0);  // s == segs: the next block's first entry (or the total)
        if (s == 0) base[b] = b0;
        if (i == 0) base[K] = flat[(int64_t)K * segs];
    }
}

// thread per column: insertion sort of the column segment by row index (CSR has unique columns
// per row, so keys are distinct and the result is unique)
__global__ void csc_sort(const int64_t *__restrict__ col_ptr, int64_t n, int32_t *__restrict__ row_idx,
                         float *__restrict__ cval) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k0 = col_ptr[j], k1 = col_ptr[j + 1];
        for (int64_t a = k0 + 1; a < k1; ++a) {
            const int32_t key = row_idx[a];
            const float v = cval[a];
            int64_t b = a - 1;
            while (b >= k0 && row_idx[b] > key) {
                row_idx[b + 1] = row_idx[b];
                cval[b + 1] = cval[b];
                --b;
            }
            row_idx[b + 1] = key;
            cval[b + 1] = v;
        }
    }
}

// ---------------------------------------------------------------- N4b: index blocking (one time)
// Compressed segments (rows of the CSR, columns of the CSC) with sorted indices, split into K
// blocks of width bw by index: thread per segment, binary search of the block boundaries.
// cnt[b * segs + s] = entries of segment s in block b.
__global__ void blk_count(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx, int64_t segs, int K,
                          int64_t bw, unsigned *__restrict__ cnt) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < segs; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k0 = ptr[s], k1 = ptr[s + 1];
        int64_t prev = k0;
        for (int b = 0; b < K; ++b) {
            int64_t lo = prev, hi = k1;  // first entry with idx >= (b + 1) bw
            const int64_t lim = (int64_t)(b + 1) * bw;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)idx[mid] < lim) lo = mid + 1;
                else hi = mid;
            }
            cnt[(int64_t)b * segs + s] = (unsigned)(lo - prev);
            prev = lo;
        }
    }
}

// scatter each segment's block pieces (order inside a piece kept) to the blocked layout
__global__ void blk_scatter(const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                            const float *__restrict__ val, int64_t segs, int K, const int64_t *__restrict__ bptr,
                            int32_t *__restrict__ bidx, float *__restrict__ bval) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < segs; s += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = ptr[s];
        for (int b = 0; b < K; ++b) {
            const int64_t d0 = bptr[(int64_t)b * segs + s], d1 = bptr[(int64_t)b * segs + s + 1];
            for (int64_t d = d0; d < d1; ++d, ++k) {
                bidx[d] = idx[k];
                bval[d] = val[k];
            }
        }
    }
}

// host-input validation helper on the device: count entries with a column outside [0, n) or a
// non-increasing column inside a row (CSR contract: sorted, unique columns)
__global__ void csr_check(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rows,
                          int64_t n, int64_t nnz, unsigned long long *__restrict__ bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long nb = 0;
    for (int64_t r = i; r < rows; r += stride) {
        const int64_t k0 = row_ptr[r], k1 = row_ptr[r + 1];
        if (k1 < k0 || k0 < 0 || k1 > nnz) {  // decreasing or out of [0, nnz]: never index col with it
            ++nb;
            continue;
        }
        for (int64_t k = k0; k < k1; ++k) {
            const int32_t c = col[k];
            if (c < 0 || c >= n || (k > k0 && c <= col[k - 1])) ++nb;
        }
    }
    if (nb) atomicAdd(bad, nb);
}

}  // namespace tsvd
