// sparse_kernels.cuh — the Gram-vector product for a CSR row slab (Alg. 4).
//
//   N2 csr_spmv   warp per row: t_r = (sum_k val_k y32[col_k]) / ||y_cur|| - U_r . c   (= (X' v)_r,
//                 v = y_cur / ||y_cur|| folded in, y32 = fp32 copy of the fp64 iterate written by the
//                 finalize kernel: reading R23); per-block partials of w = U^T t.  EXTRACT: u_r =
//                 (A v)_r and per-block sum u_r^2.
//   N3 csc_spmvT  warp per column over the slab's CSC: y_j = sum_k cval_k t[row_k] — the transpose
//                 product with no atomics and a fixed summation order; block 0 also sums the w
//                 partials.  y and w land in yw = [y | w] (then the all-reduce across ranks, if any,
//                 and fin_iter<SRC_YW>).
//   N4 csc_*      one-time CSR -> CSC of the slab on the device: column histogram, exclusive scan,
//                 scatter, per-column sort by row index (so the CSC, and every result, is
//                 deterministic).
// Products and sums are fp64; the gathered vectors are fp32 copies (the path is bound by the random
// gathers' DRAM traffic, not by arithmetic).
#pragma once
#include "fin_kernels.cuh"

namespace tsvd {

constexpr int kSpThreads = 256;
constexpr size_t kSpL2BlockBytes = 32u << 20;  // fp32 gather block that stays L2-resident (126 MB L2)
constexpr int kSpWarps = kSpThreads / 32;

struct SpParams {
    const int64_t *row_ptr;  // CSR of the slab, rows + 1 entries, row_ptr[0] == 0
    const int32_t *col;
    const float *val;
    int64_t rows;
    const int64_t *col_ptr;  // CSC of the same slab, n + 1 entries
    const int32_t *row_idx;
    const float *cval;
    int64_t n;
    const float *U;  // rows x ldu fp32
    int ldu;
    int l;
    const double *c;
    const double *ybuf;
    int64_t ystride;
    const LoopState *st;
    double *t;        // [rows] EXTRACT: u_r (fp64)
    float *t32;       // [rows] iteration: t_r rounded to fp32, gathered by N3
    const float *y32; // [n] y_cur rounded to fp32 (written by fin_iter), gathered by N2
    double *wpart;    // [gridDim.x][wpart_ld]
    int wpart_ld;
    double *sq_part;  // [gridDim.x] (EXTRACT)
    double *yw;       // N3 output: y (n) | w (l) at wofs
    int64_t wofs;
    int parts;        // gridDim.x of N2 (rows of wpart)
    // index blocking (an L2-sized block of the gathered vector per launch): launch `phase` of
    // `nphase` covers the entries whose gathered index lies in block `phase`; the per-row (column)
    // partial sums are carried across launches in fp64 and finished by the last launch.  The
    // blocked pointers of phase b start at row_ptr + b * rows (col_ptr + b * n): one exclusive scan
    // over [block][segment] counts.
    int phase, nphase;
    double *acc;      // [rows] (N2) or [n] (N3) carried partial sums when nphase > 1
};

// Memory-level parallelism: each warp works on kSpRows consecutive rows (columns) at once.  Per lane,
// the index/value loads of all of them are issued together (streaming, evict-first: they are read
// once per pass), then all their gathers, so a warp has kSpRows dependent chains in flight instead
// of one.  Lane `lane` of row q still sums k = k0 + lane, k0 + lane + 32, ... and the warp tree is
// the same, so every result is bitwise what one row per warp gives.
constexpr int kSpRows = 4;

// Lanes per segment: L (8, 16 or 32) lanes share a row (column), so a warp holds 32 / L groups of
// kSpRows consecutive segments.  The host picks L from the mean segment length (nnz per row per
// index block): short segments (blocked, or sparse rows) would otherwise leave most lanes idle.

// bounds of the group's kSpRows segments starting at rb: group lanes 0..kSpRows load
// ptr[min(rb + lane, segs)], broadcast within the group; segments past the end are empty
template <int L>
__device__ __forceinline__ void sp_bounds(const int64_t *ptr, int64_t rb, int64_t segs, int sl, int64_t (&kb)[kSpRows],
                                          int64_t (&ke)[kSpRows]) {
    int64_t v = 0;
    if (sl <= kSpRows) v = __ldcs(ptr + (rb + sl < segs ? rb + sl : segs));
#pragma unroll
    for (int q = 0; q < kSpRows; ++q) {
        kb[q] = __shfl_sync(0xffffffffu, v, q, L);
        ke[q] = __shfl_sync(0xffffffffu, v, q + 1, L);
    }
}

// fp64 sum over the L lanes of a group (butterfly inside the group: every lane gets the total)
template <int L>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// sum_k val[k] x[idx[k]] over [kb[q], ke[q]) for every q: group lane sl takes k = kb + sl, kb + sl
// + L, ...; fp64 products and sums; the index/value loads of all kSpRows segments are issued
// together (streaming, evict-first: read once per pass), then all their gathers.  x is an fp32
// copy of the gathered vector: a random gather costs a whole L2 sector (or line) of DRAM traffic
// whatever its width, and the fp32 copy is half the footprint, so more of it stays in L2
// (measured: L2 hit rate 10 % with the fp64 vector at n = 2^25, 24 % fp32, 72 % fp32 + blocks).
template <int L>
__device__ __forceinline__ void sp_rows_dot(const int64_t (&kb)[kSpRows], const int64_t (&ke)[kSpRows],
                                            const int32_t *idx, const float *val, const float *x, int sl,
                                            double (&s)[kSpRows]) {
    int64_t maxlen = 0;
#pragma unroll
    for (int q = 0; q < kSpRows; ++q) {
        s[q] = 0.0;
        maxlen = (ke[q] - kb[q]) > maxlen ? (ke[q] - kb[q]) : maxlen;
    }
    for (int64_t off = sl; off < maxlen; off += L) {
        int32_t ci[kSpRows];
        float vv[kSpRows];
#pragma unroll
        for (int q = 0; q < kSpRows; ++q) {
            const int64_t k = kb[q] + off;
            ci[q] = -1;
            vv[q] = 0.f;
            if (k < ke[q]) {
                ci[q] = __ldcs(idx + k);
                vv[q] = __ldcs(val + k);
            }
        }
        double g[kSpRows];
#pragma unroll
        for (int q = 0; q < kSpRows; ++q) g[q] = ci[q] >= 0 ? (double)__ldg(x + ci[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < kSpRows; ++q)
            if (ci[q] >= 0) s[q] += (double)vv[q] * g[q];
    }
#pragma unroll
    for (int q = 0; q < kSpRows; ++q) s[q] = group_sum<L>(s[q]);
}

// carry the kSpRows segment sums of a group across index blocks (fixed block order): group lane
// q < kSpRows owns segment rb + q; on the last block the totals are broadcast back into s[]
template <int L>
__device__ __forceinline__ bool sp_carry(const SpParams &p, double *acc, int64_t rb, int64_t segs, int sl,
                                         double (&s)[kSpRows]) {
    double v = s[0];
#pragma unroll
    for (int q = 1; q < kSpRows; ++q)
        if (sl == q) v = s[q];
    if (sl < kSpRows && rb + sl < segs) {
        if (p.phase > 0) v = acc[rb + sl] + v;
        if (p.phase < p.nphase - 1) acc[rb + sl] = v;
    }
    if (p.phase < p.nphase - 1) return false;  // totals not complete yet
#pragma unroll
    for (int q = 0; q < kSpRows; ++q) s[q] = __shfl_sync(0xffffffffu, v, q, L);
    return true;
}

// N2.  Dynamic shared memory: kSpWarps * (32 / L) * l doubles (per-group w accumulators).
template <bool EXTRACT, int L>
__global__ void __launch_bounds__(kSpThreads) csr_spmv(const SpParams p) {
    constexpr int G = 32 / L;
    extern __shared__ double wsm[];
    __shared__ double sqw[kSpWarps * G];
    const LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop || (!EXTRACT && st->done)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane / L, sl = lane % L;
    const int l = EXTRACT ? 0 : p.l;
    const double inv = 1.0 / st->ny;
    double *wme = wsm + (warp * G + grp) * (l > 0 ? l : 1);
    for (int i = sl; i < l; i += L) wme[i] = 0.0;
    double sq = 0.0;
    const int64_t nwarps = (int64_t)gridDim.x * kSpWarps;
    const int64_t *ptr = p.row_ptr + (int64_t)p.phase * p.rows;
    for (int64_t r0 = ((int64_t)blockIdx.x * kSpWarps + warp) * (G * kSpRows); r0 < p.rows;
         r0 += nwarps * (G * kSpRows)) {
        const int64_t rb = r0 + grp * kSpRows;
        int64_t kb[kSpRows], ke[kSpRows];
        sp_bounds<L>(ptr, rb, p.rows, sl, kb, ke);
        double sr[kSpRows];
        sp_rows_dot<L>(kb, ke, p.col, p.val, p.y32, sl, sr);
        if (p.nphase > 1 && !sp_carry<L>(p, p.acc, rb, p.rows, sl, sr)) continue;
#pragma unroll
        for (int q = 0; q < kSpRows; ++q) {
            const int64_t r = rb + q;
            const bool ok = r < p.rows;  // group-uniform; every lane still joins the shuffles
            double s = sr[q] * inv;
            if (!EXTRACT && l > 0) {
                const float *Ur = p.U + (ok ? r : 0) * p.ldu;
                double corr = 0.0;  // U_r . c: deflation without forming X' (Eq. 2, factored)
                if (ok)
                    for (int i = sl; i < l; i += L) corr += (double)Ur[i] * p.c[i];
                s -= group_sum<L>(corr);
                if (ok)
                    for (int i = sl; i < l; i += L) wme[i] += s * (double)Ur[i];
            }
            if (ok && sl == 0) {
                if (EXTRACT) p.t[r] = s;
                else p.t32[r] = (float)s;
                sq += s * s;
            }
        }
    }
    if (p.phase < p.nphase - 1) return;  // not the last block: only the carried sums were written
    if (sl == 0) sqw[warp * G + grp] = sq;
    __syncthreads();
    if (EXTRACT) {
        if (tid == 0) {
            double a = 0.0;
            for (int w = 0; w < kSpWarps * G; ++w) a += sqw[w];
            p.sq_part[blockIdx.x] = a;
        }
    } else {
        for (int i = tid; i < l; i += kSpThreads) {
            double a = 0.0;
            for (int w = 0; w < kSpWarps * G; ++w) a += wsm[w * l + i];  // groups in order
            p.wpart[(int64_t)blockIdx.x * p.wpart_ld + i] = a;
        }
    }
}

// N3.
template <int L>
__global__ void __launch_bounds__(kSpThreads) csc_spmvT(const SpParams p) {
    constexpr int G = 32 / L;
    const LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop || st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane / L, sl = lane % L;
    const int64_t nwarps = (int64_t)gridDim.x * kSpWarps;
    const int64_t *ptr = p.col_ptr + (int64_t)p.phase * p.n;
    for (int64_t j0 = ((int64_t)blockIdx.x * kSpWarps + warp) * (G * kSpRows); j0 < p.n;
         j0 += nwarps * (G * kSpRows)) {
        const int64_t jb = j0 + grp * kSpRows;
        int64_t kb[kSpRows], ke[kSpRows];
        sp_bounds<L>(ptr, jb, p.n, sl, kb, ke);
        double sc[kSpRows];
        sp_rows_dot<L>(kb, ke, p.row_idx, p.cval, p.t32, sl, sc);
        double v = sc[0];
#pragma unroll
        for (int q = 1; q < kSpRows; ++q)
            if (sl == q) v = sc[q];
        if (sl < kSpRows && jb + sl < p.n) {
            if (p.nphase > 1 && p.phase > 0) v = p.acc[jb + sl] + v;
            if (p.phase < p.nphase - 1) p.acc[jb + sl] = v;
            else p.yw[jb + sl] = v;
        }
    }
    if (blockIdx.x == 0 && p.phase == p.nphase - 1)
        for (int i = warp; i < p.l; i += kSpWarps) {
            double w = 0.0;
            for (int b = lane; b < p.parts; b += 32) w += p.wpart[(int64_t)b * p.wpart_ld + i];
            w = warp_sum(w);
            if (lane == 0) p.yw[p.wofs + i] = w;
        }
}

// ---------------------------------------------------------------- N4: CSR -> CSC (one time)
__global__ void csc_count(const int32_t *__restrict__ col, int64_t nnz, unsigned *__restrict__ cnt) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[col[k]], 1u);
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

// warp per row: claim a slot in each entry's column (order inside a column fixed by csc_sort)
__global__ void csc_scatter(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            const float *__restrict__ val, int64_t rows, const int64_t *__restrict__ col_ptr,
                            unsigned *__restrict__ fill, int32_t *__restrict__ row_idx, float *__restrict__ cval) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nwarps)
        for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) {
            const int32_t j = col[k];
            const int64_t pos = col_ptr[j] + atomicAdd(&fill[j], 1u);
            row_idx[pos] = (int32_t)r;
            cval[pos] = val[k];
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
                          int64_t n, unsigned long long *__restrict__ bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long nb = 0;
    for (int64_t r = i; r < rows; r += stride) {
        const int64_t k0 = row_ptr[r], k1 = row_ptr[r + 1];
        if (k1 < k0) ++nb;
        for (int64_t k = k0; k < k1; ++k) {
            const int32_t c = col[k];
            if (c < 0 || c >= n || (k > k0 && c <= col[k - 1])) ++nb;
        }
    }
    if (nb) atomicAdd(bad, nb);
}

}  // namespace tsvd
