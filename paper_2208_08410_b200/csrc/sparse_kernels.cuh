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
};

// Memory-level parallelism: each warp works on kSpRows consecutive rows (columns) at once.  Per lane,
// the index/value loads of all of them are issued together (streaming, evict-first: they are read
// once per pass), then all their gathers, so a warp has kSpRows dependent chains in flight instead
// of one.  Lane `lane` of row q still sums k = k0 + lane, k0 + lane + 32, ... and the warp tree is
// the same, so every result is bitwise what one row per warp gives.
constexpr int kSpRows = 4;

// row (column) pointers of kSpRows consecutive rows starting at r0: lanes 0..kSpRows load
// ptr[min(r0 + lane, rows)], the bounds are broadcast; rows past the end are empty
__device__ __forceinline__ void sp_bounds(const int64_t *ptr, int64_t r0, int64_t rows, int lane, int64_t (&kb)[kSpRows],
                                          int64_t (&ke)[kSpRows]) {
    int64_t v = 0;
    if (lane <= kSpRows) v = __ldcs(ptr + (r0 + lane < rows ? r0 + lane : rows));
#pragma unroll
    for (int q = 0; q < kSpRows; ++q) {
        kb[q] = __shfl_sync(0xffffffffu, v, q);
        ke[q] = __shfl_sync(0xffffffffu, v, q + 1);
    }
}

// sum_k val[k] x[idx[k]] over [kb[q], ke[q]) for every q, lane-strided, fp64 products and sums.
// x is an fp32 copy of the gathered vector: a random gather costs a whole L2 sector (or line) of
// DRAM traffic whatever its width, and the fp32 copy is half the footprint, so most of it stays in
// the 126 MB L2 (measured: L2 hit rate 10 % with the fp64 vector at n = 2^25).
__device__ __forceinline__ void sp_rows_dot(const int64_t (&kb)[kSpRows], const int64_t (&ke)[kSpRows],
                                            const int32_t *idx, const float *val, const float *x, int lane,
                                            double (&s)[kSpRows]) {
    int64_t maxlen = 0;
#pragma unroll
    for (int q = 0; q < kSpRows; ++q) {
        s[q] = 0.0;
        maxlen = (ke[q] - kb[q]) > maxlen ? (ke[q] - kb[q]) : maxlen;
    }
    for (int64_t off = lane; off < maxlen; off += 32) {
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
    for (int q = 0; q < kSpRows; ++q) s[q] = warp_sum(s[q]);
}

// N2.  Dynamic shared memory: kSpWarps * l doubles (per-warp w accumulators, lane-owned entries).
template <bool EXTRACT>
__global__ void __launch_bounds__(kSpThreads) csr_spmv(const SpParams p) {
    extern __shared__ double wsm[];
    __shared__ double sqw[kSpWarps];
    const LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop || (!EXTRACT && st->done)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l = EXTRACT ? 0 : p.l;
    const double inv = 1.0 / st->ny;
    double *wme = wsm + warp * (l > 0 ? l : 1);
    for (int i = lane; i < l; i += 32) wme[i] = 0.0;
    double sq = 0.0;
    const int64_t nwarps = (int64_t)gridDim.x * kSpWarps;
    for (int64_t r0 = ((int64_t)blockIdx.x * kSpWarps + warp) * kSpRows; r0 < p.rows; r0 += nwarps * kSpRows) {
        int64_t kb[kSpRows], ke[kSpRows];
        sp_bounds(p.row_ptr, r0, p.rows, lane, kb, ke);
        double sr[kSpRows];
        sp_rows_dot(kb, ke, p.col, p.val, p.y32, lane, sr);
#pragma unroll
        for (int q = 0; q < kSpRows; ++q) {
            const int64_t r = r0 + q;
            if (r >= p.rows) break;
            double s = sr[q] * inv;
            if (!EXTRACT && l > 0) {
                const float *Ur = p.U + r * p.ldu;
                double corr = 0.0;  // U_r . c: deflation without forming X' (Eq. 2, factored)
                for (int i = lane; i < l; i += 32) corr += (double)Ur[i] * p.c[i];
                s -= warp_sum(corr);
                for (int i = lane; i < l; i += 32) wme[i] += s * (double)Ur[i];
            }
            if (lane == 0) {
                if (EXTRACT) p.t[r] = s;
                else p.t32[r] = (float)s;
                sq += s * s;
            }
        }
    }
    if (lane == 0) sqw[warp] = sq;
    __syncthreads();
    if (EXTRACT) {
        if (tid == 0) {
            double a = 0.0;
            for (int w = 0; w < kSpWarps; ++w) a += sqw[w];
            p.sq_part[blockIdx.x] = a;
        }
    } else {
        for (int i = tid; i < l; i += kSpThreads) {
            double a = 0.0;
            for (int w = 0; w < kSpWarps; ++w) a += wsm[w * l + i];  // warps in order
            p.wpart[(int64_t)blockIdx.x * p.wpart_ld + i] = a;
        }
    }
}

// N3.
__global__ void __launch_bounds__(kSpThreads) csc_spmvT(const SpParams p) {
    const LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop || st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * kSpWarps;
    for (int64_t j0 = ((int64_t)blockIdx.x * kSpWarps + warp) * kSpRows; j0 < p.n; j0 += nwarps * kSpRows) {
        int64_t kb[kSpRows], ke[kSpRows];
        sp_bounds(p.col_ptr, j0, p.n, lane, kb, ke);
        double sc[kSpRows];
        sp_rows_dot(kb, ke, p.row_idx, p.cval, p.t32, lane, sc);
        if (lane < kSpRows && j0 + lane < p.n) {
            double v = sc[0];
#pragma unroll
            for (int q = 1; q < kSpRows; ++q)
                if (lane == q) v = sc[q];
            p.yw[j0 + lane] = v;
        }
    }
    if (blockIdx.x == 0)
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
