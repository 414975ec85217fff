// gram_kernels.cuh — sm_100a kernels of the Gram-vector hot path.
//
//   N1 gv_fused      one pass over the row slab of A per power iteration:
//                      t_r = A_r . v - U_r . c        (= (X' v)_r,  Alg. 4 lines 3-4 + 14)
//                      y  += t_r A_r^T                 (X'^T X' v before the V correction)
//                      w  += t_r U_r^T                 (U^T X' v)
//                    A and U rows are staged by TMA bulk copies (cp.async.bulk) into an S-stage
//                    shared-memory ring; each staged element is read from shared memory ONCE into
//                    registers and used for both the dot and the axpy, so A is read from HBM
//                    exactly once per iteration (the paper's Alg. 4 reads it twice).
//                    EXTRACT=true runs the same pipeline for u = A v and ||u||^2.
//   N7 reduce_partials   fixed-order fp64 sum of the per-CTA partials of y and w.
//   N5 fin_partial / fin_scalar / fin_normalize
//                    y -= V (S w); ||y||^2, v.y, V^T y in fp64; d = |v.y|/||y||, stop test
//                    |v0.v1| >= 1-eps, v1 = y/||y||, c_next = S V^T v1.
//   N6 ext_reduce / ext_scale   sigma = ||A v1||, U[:,l] = A v1 / sigma.
//
// Precision (reading R17): A, U and the copy of v fed to N1 are fp32; products are
// fp32 FMAs inside a thread, every cross-thread / cross-CTA / cross-GPU sum is fp64, and the
// per-CTA y accumulators are flushed to fp64 every `run_rows` rows.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsvd {

constexpr int kMaxStages = 8;

struct LoopState {
    double yy;      // ||y||^2 of the last product
    double ny;      // ||y||
    double d;       // |v0 . v1| of the last iteration
    int32_t it;     // iterations done in this component
    int32_t done;   // loop finished
    int32_t status; // 0 ok, 1 not converged, 2 rank exhausted, -7 numeric
    int32_t pad;
};

struct GvParams {
    const float *A;        // row slab base (row 0 of this launch)
    int64_t ld;            // leading dimension (floats), % 4 == 0
    int64_t rows;          // rows in this launch
    int32_t n;             // columns
    int32_t n4;            // ceil(n / 4): float4 per row
    const float *U;        // rows x ldu fp32 (row 0 aligned with A's row 0); may be null if l == 0
    int32_t ldu;           // % 4 == 0
    int32_t l;             // components already found (U columns used)
    const float *v32;      // fp32 copy of v, zero padded to >= 4*T*NV
    const double *c;       // c = S (V^T v), length l
    double *ypart;         // [gridDim.x][ypart_ld] fp64 per-CTA partial of A^T t
    int64_t ypart_ld;
    double *wpart;         // [gridDim.x][wpart_ld] fp64 per-CTA partial of U^T t
    int32_t wpart_ld;
    int32_t stages;        // S
    int32_t stage_bytes;   // bytes per ring slot (A row + U row, 128-B aligned)
    int32_t row_bytes;     // n4 * 16
    int32_t u_bytes;       // round4(l) * 4 (0 if l == 0 or EXTRACT)
    int32_t run_rows;      // fp32 run length before flushing to fp64
    double *u_out;         // EXTRACT: fp64 (A v)_r, indexed by launch row
    double *sq_part;       // EXTRACT: [gridDim.x] fp64 sum of (A v)_r^2
    const int32_t *done;   // optional: skip the launch when *done != 0 (speculative loops)
};

// ---------------------------------------------------------------- PTX helpers (mbarrier + TMA)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TSVD_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TSVD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk TMA global -> shared, completion counted on `bar` (bytes % 16 == 0, 16-B aligned).
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// ---------------------------------------------------------------- N1: fused Gram-vector pass
// Grid: one persistent CTA per (SM x CTAs/SM), each owning a contiguous row range.
// Block: T threads; thread `tid` owns float4 columns {k*T + tid : k < NV} of every row.
template <int T, int NV, bool EXTRACT>
__global__ void __launch_bounds__(T) gv_fused(const GvParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NW = T / 32;
    if (p.done != nullptr && *p.done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)p.stages * p.stage_bytes);
    double *red = reinterpret_cast<double *>(bars + kMaxStages);  // [2][NW]

    const int64_t r0 = p.rows * blockIdx.x / gridDim.x;
    const int64_t r1 = p.rows * (blockIdx.x + 1) / gridDim.x;
    const int nr = (int)(r1 - r0);
    const int S = p.stages;
    const int l = EXTRACT ? 0 : p.l;
    const uint32_t tx_bytes = (uint32_t)(p.row_bytes + (EXTRACT ? 0 : p.u_bytes));

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int slot, int64_t row) {
        unsigned char *dst = smem + (size_t)slot * p.stage_bytes;
        mbar_arrive_expect_tx(&bars[slot], tx_bytes);
        tma_load_1d(dst, p.A + row * p.ld, (uint32_t)p.row_bytes, &bars[slot]);
        if (!EXTRACT && p.u_bytes > 0)
            tma_load_1d(dst + p.row_bytes, p.U + row * p.ldu, (uint32_t)p.u_bytes, &bars[slot]);
    };
    if (tid == 0) {
        const int pre = nr < S ? nr : S;
        for (int s = 0; s < pre; ++s) issue(s, r0 + s);
    }

    // this thread's slice of v (fp32, zero padded) and c
    float4 vr[NV];
    const float4 *v4 = reinterpret_cast<const float4 *>(p.v32);
#pragma unroll
    for (int k = 0; k < NV; ++k) vr[k] = v4[k * T + tid];
    double cval = 0.0;
    if (!EXTRACT && tid < l) cval = p.c[tid];
    const int tail = p.n & 3;  // valid lanes of the last float4 (0 = full)

    float4 ya[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) ya[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    double wacc = 0.0, sq = 0.0;
    bool flushed = false;
    double *yp = p.ypart + (int64_t)blockIdx.x * p.ypart_ld;

    auto flush = [&]() {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = k * T + tid;
            if (idx < p.n4) {
                double2 *dst = reinterpret_cast<double2 *>(yp + 4 * (int64_t)idx);
                double2 lo = make_double2(ya[k].x, ya[k].y), hi = make_double2(ya[k].z, ya[k].w);
                if (flushed) {
                    const double2 olo = dst[0], ohi = dst[1];
                    lo.x += olo.x; lo.y += olo.y; hi.x += ohi.x; hi.y += ohi.y;
                }
                dst[0] = lo;
                dst[1] = hi;
            }
            ya[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        flushed = true;
    };

    int run = 0;
    for (int i = 0; i < nr; ++i) {
        const int s = i % S;
        mbar_wait(&bars[s], (uint32_t)((i / S) & 1));
        const unsigned char *slot = smem + (size_t)s * p.stage_bytes;
        const float4 *row = reinterpret_cast<const float4 *>(slot);

        float4 a[NV];
        float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = k * T + tid;
            if (idx < p.n4) {
                a[k] = row[idx];
                if (tail && idx == p.n4 - 1) {  // columns >= n of the last float4 may be garbage
                    if (tail < 2) a[k].y = 0.f;
                    if (tail < 3) a[k].z = 0.f;
                    a[k].w = 0.f;
                }
            } else {
                a[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            q0 = fmaf(a[k].x, vr[k].x, q0);
            q1 = fmaf(a[k].y, vr[k].y, q1);
            q2 = fmaf(a[k].z, vr[k].z, q2);
            q3 = fmaf(a[k].w, vr[k].w, q3);
        }
        double part = (double)((q0 + q1) + (q2 + q3));
        float ur = 0.f;
        if (!EXTRACT && tid < l) {
            ur = reinterpret_cast<const float *>(slot + p.row_bytes)[tid];
            part -= (double)ur * cval;  // - U_r . c  (deflation, never forming X')
        }
        part = warp_sum(part);
        if (lane == 0) red[(i & 1) * NW + warp] = part;
        __syncthreads();  // (a) partial dots visible, (b) every thread is done reading slot s
        if (tid == 0 && i + S < nr) {
            fence_proxy_async_smem();
            issue(s, r0 + i + S);
        }
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += red[(i & 1) * NW + w];  // same order in every thread

        if (EXTRACT) {
            if (tid == 0) {
                p.u_out[r0 + i] = t;
                sq += t * t;
            }
        } else {
            const float tf = (float)t;
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                ya[k].x = fmaf(tf, a[k].x, ya[k].x);
                ya[k].y = fmaf(tf, a[k].y, ya[k].y);
                ya[k].z = fmaf(tf, a[k].z, ya[k].z);
                ya[k].w = fmaf(tf, a[k].w, ya[k].w);
            }
            if (tid < l) wacc += t * (double)ur;
            if (++run == p.run_rows && i + 1 < nr) {
                flush();
                run = 0;
            }
        }
    }
    if (EXTRACT) {
        if (tid == 0) p.sq_part[blockIdx.x] = sq;
    } else {
        flush();
        if (tid < l) p.wpart[(int64_t)blockIdx.x * p.wpart_ld + tid] = wacc;
    }
}

// ---------------------------------------------------------------- N7: fixed-order partial sum
// y[j] = sum_{b < parts} ypart[b][j] (b ascending), w[i] likewise.  yw: [y (n) | pad | w (l)].
__global__ void reduce_partials(const double *__restrict__ ypart, int parts, int64_t ypart_ld, int n,
                                const double *__restrict__ wpart, int wpart_ld, int l, double *__restrict__ y,
                                double *__restrict__ w, const int32_t *done) {
    if (done != nullptr && *done) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) {
        double s0 = 0.0;
        int b = 0;
        for (; b < parts; ++b) s0 += ypart[(int64_t)b * ypart_ld + j];
        y[j] = s0;
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < l; i += blockDim.x) {
            double s = 0.0;
            for (int b = 0; b < parts; ++b) s += wpart[(int64_t)b * wpart_ld + i];
            w[i] = s;
        }
    }
}

// ---------------------------------------------------------------- N5a: correction + partial dots
// mode 0 (iterate): y_j -= sum_i V[j,i] S_i w_i.   mode 1 (init) / 2 (raw): no correction.
// Block partials part[b] = { sum y_j^2, sum v_j y_j, (V^T y)_0..l-1 } over the block's j range.
constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads)
    fin_partial(int mode, int n, int l, const double *__restrict__ S, const double *__restrict__ V, int ldv,
                const double *__restrict__ w, double *__restrict__ y, const double *__restrict__ v,
                double *__restrict__ part, int part_ld, const int32_t *done) {
    if (done != nullptr && *done) return;
    __shared__ double ys[kFinThreads];
    __shared__ double red[2][kFinThreads / 32];
    extern __shared__ double g[];  // l values of S_i w_i
    const int tid = threadIdx.x;
    for (int i = tid; i < l; i += kFinThreads) g[i] = (mode == 0) ? S[i] * w[i] : 0.0;
    __syncthreads();
    const int j0 = blockIdx.x * kFinThreads;
    const int j = j0 + tid;
    double yj = 0.0, vj = 0.0;
    if (j < n) {
        yj = y[j];
        if (mode == 0 && l > 0) {
            double corr = 0.0;
            for (int i = 0; i < l; ++i) corr += V[(int64_t)j * ldv + i] * g[i];
            yj -= corr;
            y[j] = yj;
        }
        vj = (mode == 0) ? v[j] : 0.0;
    }
    ys[tid] = yj;
    double a = warp_sum(yj * yj), b = warp_sum(vj * yj);
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = a;
        red[1][tid >> 5] = b;
    }
    __syncthreads();
    double *out = part + (int64_t)blockIdx.x * part_ld;
    if (tid == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int k = 0; k < kFinThreads / 32; ++k) {
            s0 += red[0][k];
            s1 += red[1][k];
        }
        out[0] = s0;
        out[1] = s1;
    }
    const int jn = (n - j0) < kFinThreads ? (n - j0) : kFinThreads;
    for (int i = tid; i < l; i += kFinThreads) {  // (V^T y)_i over this block's rows, coalesced in i
        double s = 0.0;
        for (int jj = 0; jj < jn; ++jj) s += V[(int64_t)(j0 + jj) * ldv + i] * ys[jj];
        out[2 + i] = s;
    }
}

// ---------------------------------------------------------------- N5b: scalars + stop test
// mode 0 iterate, 1 init (normalise x), 2 raw (no normalisation; gram_apply).
__global__ void __launch_bounds__(kFinThreads)
    fin_scalar(int mode, int parts, int part_ld, int l, const double *__restrict__ S, const double *__restrict__ part,
               double *__restrict__ c, LoopState *st, double eps, int fixed_T, int max_iter,
               unsigned long long cond_handle, int use_cond) {
    __shared__ double tot[2];
    __shared__ double inv_s;
    const int tid = threadIdx.x;
    if (st->done && mode == 0) return;
    for (int q = tid; q < 2 + l; q += kFinThreads) {
        double s = 0.0;
        for (int b = 0; b < parts; ++b) s += part[(int64_t)b * part_ld + q];  // fixed order
        if (q < 2) tot[q] = s;
        else c[q - 2] = s;  // raw V^T y for now
    }
    __syncthreads();
    if (tid == 0) {
        const double yy = tot[0];
        double ny = sqrt(yy);
        if (mode == 2) ny = 1.0;
        st->yy = yy;
        st->ny = ny;
        if (mode == 1) {
            st->it = 0;
            st->done = 0;
            st->status = (isfinite(ny) && ny > 0.0) ? 0 : -7;
            if (st->status) st->done = 1;
            st->d = 0.0;
        } else if (mode == 0) {
            const int it = st->it + 1;
            st->it = it;
            if (!isfinite(ny)) {
                st->status = -7;
                st->done = 1;
            } else if (ny == 0.0) {
                st->status = 2;
                st->done = 1;
            } else {
                const double d = fabs(tot[1]) / ny;  // |v0 . v1| with v1 = y / ||y||
                st->d = d;
                if (fixed_T > 0) {
                    if (it >= fixed_T) st->done = 1;
                } else if (d >= 1.0 - eps) {
                    st->done = 1;
                } else if (it >= max_iter) {
                    st->done = 1;
                    st->status = 1;
                }
            }
        }
        inv_s = (ny > 0.0 && isfinite(ny)) ? ny : 1.0;
#if CUDART_VERSION >= 12030
        if (use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, st->done ? 0u : 1u);
#endif
    }
    __syncthreads();
    for (int i = tid; i < l; i += kFinThreads) c[i] = S[i] * (c[i] / inv_s);  // c = S V^T v1
}

// ---------------------------------------------------------------- N5c: v1 = y / ||y||
// Writes the fp64 master (for the stop test) and the fp32 copy fed to N1.
__global__ void fin_normalize(int n, const double *__restrict__ y, const LoopState *st, double *__restrict__ v,
                              float *__restrict__ v32, int skip_when_failed) {
    const double ny = st->ny;
    if (skip_when_failed && (st->status < 0 || st->status == 2)) return;
    const double inv = (ny > 0.0 && isfinite(ny)) ? ny : 1.0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const double x = y[j] / inv;
        v[j] = x;
        v32[j] = (float)x;
    }
}

// ---------------------------------------------------------------- N6: extraction tail
__global__ void ext_reduce(const double *__restrict__ sq_part, int parts, double *__restrict__ sig2) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < parts; ++b) s += sq_part[b];
        *sig2 = s;
    }
}

// U[r, l] = u_r / sigma (fp32 storage), V[j, l] = v1_j, S[l] = sigma
__global__ void ext_scale(int64_t rows, int n, int l, const double *__restrict__ u, const double *__restrict__ sig2,
                          const double *__restrict__ v, float *__restrict__ U, int ldu, double *__restrict__ V,
                          int ldv, double *__restrict__ S) {
    const double sigma = sqrt(*sig2);
    const double inv = sigma > 0.0 ? sigma : 1.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t r = g; r < rows; r += stride) U[r * ldu + l] = (float)(u[r] / inv);
    for (int64_t j = g; j < n; j += stride) V[j * ldv + l] = v[j];
    if (g == 0) S[l] = sigma;
}

// fp64 -> fp32 copy of a vector (gram_apply input path)
__global__ void to_f32(int n, const double *__restrict__ x, float *__restrict__ y) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) y[j] = (float)x[j];
}

}  // namespace tsvd
