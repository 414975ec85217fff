// fin_kernels.cuh — everything after N1 in a power iteration, and the extraction tail.
//
//   N5 fin_iter<SRC>  per column j: y_j = (sum of the partial y's) - sum_i V[j,i] S_i w_i  (Eq. 2's
//                     2nd and 4th terms in exact factored form); per block ||y||^2, v.y, V^T y; the
//                     LAST block to arrive (arrival counter) sums the block partials in block order
//                     and takes the scalar decisions: ||y||, the stop test |v0 . v1| >= 1 - eps
//                     (P:123), c_next = S V^T v1, and the CUDA-graph WHILE condition.  y_new goes to
//                     the other half of a ping-pong buffer; the next N1 builds v = y_new / ||y_new||.
//   N6 ext_finish<SRC> sigma = ||A v1||, U[:,l] = A v1 / sigma, V[:,l] = v1, S[l].
//
// SRC selects where the partial sums come from:
//   SRC_PARTS  single GPU: the per-CTA partials of N1, summed here in CTA order.
//   SRC_YW     multi-GPU over NCCL: reduce_partials wrote [y_g | w_g], ncclAllReduce summed it.
//   SRC_PEER   multi-GPU over NVLink peer memory: every rank's publish() wrote its [y_g | w_g] into
//              its own symmetric buffer and raised a flag on every peer; fin_iter waits for all
//              flags of this epoch and sums the ranks' vectors in RANK ORDER straight from peer
//              memory (P2P loads over NVLink 5 / NVSwitch) — the all-reduce is fused into the
//              finalize kernel, bit-identical on every rank, and lives inside the CUDA graph.
// Every sum has a fixed order: results are bitwise reproducible for a fixed grid and world size.
#pragma once
#include "gram_kernels.cuh"

namespace tsvd {

constexpr int kFinCols = 32;                       // columns per fin block
constexpr int kFinGroups = kFinThreads / kFinCols;  // partial groups per column

enum FinMode { FIN_ITERATE = 0, FIN_INIT = 1, FIN_LOAD_RAW = 2, FIN_APPLY = 3, FIN_INIT_EXT = 4, FIN_ITERATE_EXT = 5 };
enum FinSrc { SRC_PARTS = 0, SRC_YW = 1, SRC_PEER = 2 };

// Called by one thread per block: wait until every rank has published epoch `target`.
// Gives up after 30 s (a dead peer) with status -6 instead of hanging the GPU.
__device__ __forceinline__ bool peer_wait(const PeerView &pv, unsigned target, LoopState *st) {
    const unsigned long long t0 = globaltimer_ns();
    for (int r = 0; r < pv.world; ++r) {
        while ((int)(ld_acquire_sys(pv.flags + r) - target) < 0) {
            if (globaltimer_ns() - t0 > 30000000000ull) {
                st->status = -6;
                st->stop = 1;
                return false;
            }
            __nanosleep(64);
        }
    }
    return true;
}

// ---------------------------------------------------------------- multi-GPU: local partial sums
// NCCL path: yw = [ y_g (n) | pad | w_g (l) ] (then ncclAllReduce).
__global__ void __launch_bounds__(kFinThreads)
    reduce_partials(const double *__restrict__ ypart, int parts, int64_t ypart_ld, int n,
                    const double *__restrict__ wpart, int wpart_ld, int l, double *__restrict__ yw, int64_t wofs,
                    const LoopState *st) {
    __shared__ double gsum[kFinGroups][kFinCols];
    griddep_launch();
    griddep_wait();
    if (st->stop || st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
    for (int64_t ch = blockIdx.x; ch * kFinCols < n; ch += gridDim.x) {
        const int64_t j = ch * kFinCols + lane;
        double s = 0.0;
        if (j < n)
            for (int b = grp; b < parts; b += kFinGroups) s += ypart[(int64_t)b * ypart_ld + j];
        gsum[grp][lane] = s;
        __syncthreads();
        if (grp == 0 && j < n) {
            double y = gsum[0][lane];
            for (int q = 1; q < kFinGroups; ++q) y += gsum[q][lane];
            yw[j] = y;
        }
        __syncthreads();
    }
    if (blockIdx.x == 0)
        for (int i = grp; i < l; i += kFinGroups) {
            double w = 0.0;
            for (int b = lane; b < parts; b += 32) w += wpart[(int64_t)b * wpart_ld + i];
            w = warp_sum(w);
            if (lane == 0) yw[wofs + i] = w;
        }
}

// Peer path: same local sums, written into this rank's symmetric slot (epoch & 1); the last block
// then raises flag = epoch + 1 on every rank (release, system scope).  mode 1: ||u||^2 only.
struct PubParams {
    int mode;  // 0: y and w of an iteration; 1: sum of the per-CTA ||u||^2 (extraction)
    const double *ypart;
    int parts;
    int64_t ypart_ld;
    const double *wpart;
    int wpart_ld;
    int n, l;
    const double *sq_part;
    PeerView pv;
    LoopState *st;
    int with_sq;  // mode 0 after a fused-extraction pass: also publish sum(u_r^2)
};

__global__ void __launch_bounds__(kFinThreads) publish(const PubParams p) {
    __shared__ double gsum[kFinGroups][kFinCols];
    __shared__ int am_last;
    LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop || (p.mode == 0 && st->done)) return;  // identical decision on every rank
    const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
    const unsigned e = st->epoch;
    double *slot = p.pv.buf[p.pv.rank] + (int64_t)(e & 1u) * p.pv.slot_stride;
    if (p.mode == 0) {
        for (int64_t ch = blockIdx.x; ch * kFinCols < p.n; ch += gridDim.x) {
            const int64_t j = ch * kFinCols + lane;
            double s = 0.0;
            if (j < p.n)
                for (int b = grp; b < p.parts; b += kFinGroups) s += p.ypart[(int64_t)b * p.ypart_ld + j];
            gsum[grp][lane] = s;
            __syncthreads();
            if (grp == 0 && j < p.n) {
                double y = gsum[0][lane];
                for (int q = 1; q < kFinGroups; ++q) y += gsum[q][lane];
                slot[j] = y;
            }
            __syncthreads();
        }
        if (blockIdx.x == 0)
            for (int i = grp; i < p.l; i += kFinGroups) {
                double w = 0.0;
                for (int b = lane; b < p.parts; b += 32) w += p.wpart[(int64_t)b * p.wpart_ld + i];
                w = warp_sum(w);
                if (lane == 0) slot[p.pv.wofs + i] = w;
            }
        if (p.with_sq && blockIdx.x == 0 && tid == 0) {
            double s = 0.0;
            for (int b = 0; b < p.parts; ++b) s += p.sq_part[b];
            slot[p.pv.sofs] = s;
        }
    } else if (blockIdx.x == 0 && tid == 0) {
        double s = 0.0;
        for (int b = 0; b < p.parts; ++b) s += p.sq_part[b];
        slot[p.pv.sofs] = s;
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) am_last = (atomicAdd(&st->pub_counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!am_last || tid != 0) return;
    __threadfence_system();
    st->pub_counter = 0;
    for (int r = 0; r < p.pv.world; ++r) st_release_sys(p.pv.rflags[r], e + 1u);
}

// ---------------------------------------------------------------- N5: fin_iter
struct FinParams {
    int mode;
    int n, l;
    const double *S;          // sigma[0..l)
    const double *V;          // n x ldv fp64 row-major
    int ldv;
    const double *ypart;      // SRC_PARTS: per-CTA partials of N1
    int parts;
    int64_t ypart_ld;
    const double *wpart;
    int wpart_ld;
    const double *yw;         // SRC_YW: all-reduced [y | w]
    int64_t wofs;
    PeerView pv;              // SRC_PEER
    const double *xsrc;       // FIN_INIT / FIN_LOAD_RAW: vector to load
    double *ybuf;             // [2][ystride]
    int64_t ystride;
    double *part;             // [gridDim.x][part_ld]
    int part_ld;
    double *c;                // out: c = S V^T v1
    LoopState *st;
    double eps;
    int fixed_T, max_iter;
    unsigned long long cond;
    int use_cond;
    unsigned long long *tl;   // debug timeline (TSVD_TIMELINE)
    // fused extraction (FIN_INIT_EXT / FIN_ITERATE_EXT): component `fresh` = l-1 was extracted by
    // the same N1 pass that ran the first iteration of component l; its sigma is only known here
    int fresh;                // -1 when unused
    double *Vout;             // FIN_INIT_EXT: V[:, fresh] = previous iterate
    float *vprev32;           // FIN_INIT_EXT: fp32 copy of it, staged by the next N1<TWO>
    CompStat *stat;           // stat[fresh]
    const double *sq_part;    // FIN_ITERATE_EXT (SRC_PARTS): per-CTA sums of u_r^2
    int sq_parts;
    float *U;                 // FIN_ITERATE_EXT: U[:, fresh] = u / sigma
    int ldu;
    const double *u_out;
    int64_t rows;
    float *y32;               // sparse path: fp32 copy of every vector written to ybuf (else null)
};

// FIN_ITERATE : y_new = sum(partials) - V (S w) -> ybuf[(it+1)&1]; stop test; it += 1
// FIN_INIT    : ybuf[0] = x; ||x||, c = S V^T (x/||x||); it = 0   (P:112 normalisation)
// FIN_LOAD_RAW: ybuf[0] = v, ny := 1, c = S V^T v                          (tsvd_gram_apply)
// FIN_APPLY   : ybuf[1] = sum(partials) - V (S w); no state change        (tsvd_gram_apply)
//
// Grid-stride over column chunks (grid <= a few blocks per SM, so the last block reduces a bounded
// number of block partials even at n = 1e8).  SRC_PARTS reductions use 32-column chunks: thread
// (c, g) sums the per-CTA partials b = g, g+8, ... of column c and the 8 group sums are added in g
// order.  Other sources use 256-column chunks, one column per thread.  (V^T y)_i for i < 16 is
// accumulated in registers by the thread that owns the column; components >= 16 go through a
// shared-memory tile.  Every sum has a fixed order.
constexpr int kVtReg = 16;

template <int SRC>
__global__ void __launch_bounds__(kFinThreads, 4) fin_iter(const FinParams p) {
    __shared__ double gsum[kFinGroups][kFinCols];
    __shared__ double wred[kFinThreads / 32][2 + kVtReg];
    __shared__ int am_last, peer_ok;
    __shared__ double inv_s;
    extern __shared__ double dyn[];  // g[l] | tot[2 + l] | vtx[max(0, l - 16)] | ys[256]
    const int l = p.l;
    const int lx = l > kVtReg ? l - kVtReg : 0;
    double *g = dyn;
    double *tot = g + l;
    double *vtx = tot + 2 + l;
    double *ys = vtx + lx;
    __shared__ double sigma_s;
    LoopState *st = p.st;
    const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
    const int mode = p.mode;
    const bool iterate = (mode == FIN_ITERATE || mode == FIN_ITERATE_EXT);
    griddep_launch();
    griddep_wait();
    if (st->stop || (iterate && st->done)) {
        if (blockIdx.x == 0 && tid == 0) set_cond(p.cond, p.use_cond, 0u);
        return;
    }
    const int64_t n = p.n;
    const int it = st->it;
    const double ny = st->ny;
    const unsigned e = st->epoch;
    const double *ycur = p.ybuf + (int64_t)(it & 1) * p.ystride;
    if (p.tl && iterate && blockIdx.x == 0 && tid == 0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 3] = globaltimer_ns();
    double *ynew = p.ybuf + (int64_t)(iterate ? ((it + 1) & 1) : (mode == FIN_APPLY ? 1 : 0)) * p.ystride;
    const bool reduce = (iterate || mode == FIN_APPLY);
    const int64_t slot_off = (int64_t)(e & 1u) * p.pv.slot_stride;
    // the fresh component's sigma is unknown until FIN_ITERATE_EXT: weight 1 in g and c meanwhile
    const int fresh = (mode == FIN_INIT_EXT || mode == FIN_ITERATE_EXT) ? p.fresh : -1;

    if (reduce) {
        if (SRC == SRC_PEER) {
            if (tid == 0) peer_ok = peer_wait(p.pv, e + 1u, st);
            __syncthreads();
            if (!peer_ok) {
                if (blockIdx.x == 0 && tid == 0) set_cond(p.cond, p.use_cond, 0u);
                return;
            }
        }
        if (SRC == SRC_PARTS) {  // g_i = S_i w_i, w = U^T X' v: warp per i, lanes stride the CTA partials
            for (int i = grp; i < l; i += kFinGroups) {
                double w = 0.0;
                for (int b = lane; b < p.parts; b += 32) w += p.wpart[(int64_t)b * p.wpart_ld + i];
                w = warp_sum(w);
                if (lane == 0) g[i] = (i == fresh ? 1.0 : p.S[i]) * w;
            }
        } else if (SRC == SRC_YW) {
            for (int i = tid; i < l; i += kFinThreads) g[i] = (i == fresh ? 1.0 : p.S[i]) * p.yw[p.wofs + i];
        } else {
            for (int i = tid; i < l; i += kFinThreads) {
                double w = 0.0;
                for (int r = 0; r < p.pv.world; ++r) w += __ldcg(p.pv.buf[r] + slot_off + p.pv.wofs + i);
                g[i] = (i == fresh ? 1.0 : p.S[i]) * w;
            }
        }
        if (mode == FIN_ITERATE_EXT) {  // sigma_fresh = ||A v_prev||, sums in a fixed order
            if (tid == 0) {
                double s2 = 0.0;
                if (SRC == SRC_PEER) {
                    for (int r = 0; r < p.pv.world; ++r) s2 += __ldcg(p.pv.buf[r] + slot_off + p.pv.sofs);
                } else {
                    for (int b = 0; b < p.sq_parts; ++b) s2 += p.sq_part[b];
                }
                sigma_s = sqrt(s2);
            }
            __syncthreads();
            const double sg = sigma_s;
            if (sg > 0.0 && isfinite(sg))  // U[:, fresh] = u / sigma, all blocks share the rows
                for (int64_t r = (int64_t)blockIdx.x * kFinThreads + tid; r < p.rows;
                     r += (int64_t)gridDim.x * kFinThreads)
                    p.U[r * p.ldu + fresh] = (float)(p.u_out[r] / sg);
        }
    }
    for (int i = tid; i < lx; i += kFinThreads) vtx[i] = 0.0;
    __syncthreads();

    const bool narrow = (SRC == SRC_PARTS) && reduce;  // 32-column chunks with the 8-group reduction
    const int cols = narrow ? kFinCols : kFinThreads;
    const int64_t nchunks = (n + cols - 1) / cols;
    double a_yy = 0.0, a_vy = 0.0;
    double acc[kVtReg];
#pragma unroll
    for (int i = 0; i < kVtReg; ++i) acc[i] = 0.0;

    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int64_t j0 = ch * cols;
        int64_t j;
        bool active;
        double yj = 0.0, vj = 0.0;
        if (narrow) {
            j = j0 + lane;
            double s = 0.0;
            if (j < n) {
                const double *col = p.ypart + j;
#pragma unroll 4
                for (int b = grp; b < p.parts; b += kFinGroups) s += col[(int64_t)b * p.ypart_ld];
            }
            gsum[grp][lane] = s;
            __syncthreads();
            active = (grp == 0) && (j < n);
            if (active) {
                yj = gsum[0][lane];
#pragma unroll
                for (int q = 1; q < kFinGroups; ++q) yj += gsum[q][lane];
            }
        } else {
            j = j0 + tid;
            active = j < n;
            if (active) {
                if (!reduce) {
                    yj = p.xsrc[j];
                } else if (SRC == SRC_YW) {
                    yj = p.yw[j];
                } else if (SRC == SRC_PEER) {
                    for (int r = 0; r < p.pv.world; ++r) yj += __ldcg(p.pv.buf[r] + slot_off + j);  // rank order
                }
            }
        }
        if (active) {
            const double *Vj = p.V + j * p.ldv;
            double vold = 0.0;
            if (reduce) {
                double corr = 0.0;  // (V (S w))_j: the 2nd / 4th terms of Eq. 2 in factored form
                for (int i = 0; i < l; ++i) corr += Vj[i] * g[i];
                yj -= corr;
                if (iterate) vj = ycur[j] / ny;
            } else if (mode == FIN_INIT_EXT) {  // the finished component's v becomes V[:, fresh]
                vold = ycur[j] / ny;
                p.Vout[j * p.ldv + fresh] = vold;
                p.vprev32[j] = (float)vold;
            }
            ynew[j] = yj;
            if (p.y32) p.y32[j] = (float)yj;  // sparse path: fp32 copy for N2's gathers
            a_yy += yj * yj;
            a_vy += vj * yj;
#pragma unroll
            for (int i = 0; i < kVtReg; ++i)
                if (i < l) acc[i] += (i == fresh && mode == FIN_INIT_EXT ? vold : Vj[i]) * yj;
        }
        if (lx > 0) {  // components >= 16: shared tile of this chunk's y, coalesced over i
            if (narrow) {
                if (grp == 0) ys[lane] = active ? yj : 0.0;
            } else {
                ys[tid] = active ? yj : 0.0;
            }
            __syncthreads();
            const int jn = (int)((n - j0) < cols ? (n - j0) : cols);
            for (int i = kVtReg + tid; i < l; i += kFinThreads) {
                double s = 0.0;
                for (int jj = 0; jj < jn; ++jj) s += p.V[(j0 + jj) * p.ldv + i] * ys[jj];
                vtx[i - kVtReg] += s;
            }
        }
        __syncthreads();
    }
    // ---- block partials: { sum y^2, sum v y, (V^T y)_0..l-1 } (warp shuffles, then warps in order)
    const int lr = l < kVtReg ? l : kVtReg;
    {
        double q = warp_sum(a_yy);
        if (lane == 0) wred[grp][0] = q;
        q = warp_sum(a_vy);
        if (lane == 0) wred[grp][1] = q;
#pragma unroll
        for (int i = 0; i < kVtReg; ++i) {  // static indices: acc stays in registers
            if (i < lr) {
                q = warp_sum(acc[i]);
                if (lane == 0) wred[grp][2 + i] = q;
            }
        }
    }
    __syncthreads();
    double *out = p.part + (int64_t)blockIdx.x * p.part_ld;
    if (tid < 2 + lr) {
        double s = 0.0;
        for (int w = 0; w < kFinThreads / 32; ++w) s += wred[w][tid];
        out[tid] = s;
    }
    for (int i = tid; i < lx; i += kFinThreads) out[2 + kVtReg + i] = vtx[i];
    // ---- the last block to arrive takes the scalar decisions (fixed-order sums: deterministic)
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = (atomicAdd(&st->counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    if (p.tl && iterate && tid == 0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 4] = globaltimer_ns();
    if (mode == FIN_APPLY) {
        if (tid == 0) {
            st->counter = 0;
            if (SRC == SRC_PEER) st->epoch = e + 1u;
        }
        return;
    }
    const int nb = (int)gridDim.x;
    for (int q = grp; q < 2 + l; q += kFinGroups) {  // warp per quantity, lanes stride the blocks
        double s = 0.0;
        for (int bb = lane; bb < nb; bb += 32) s += __ldcg(p.part + (int64_t)bb * p.part_ld + q);
        s = warp_sum(s);
        if (lane == 0) tot[q] = s;
    }
    __syncthreads();
    __shared__ double c_fresh_scale;  // S of the fresh column in c: 1 (INIT_EXT) or sigma (ITERATE_EXT)
    if (tid == 0) {
        st->counter = 0;
        const double yy = tot[0];
        const double nyn = sqrt(yy);
        c_fresh_scale = 1.0;
        if (mode == FIN_INIT_EXT) {  // close the finished component's record (sigma comes next pass)
            CompStat cs = p.stat[fresh];
            cs.it = it;
            cs.d = st->d;
            cs.status = st->status;
            p.stat[fresh] = cs;
        }
        if (mode == FIN_ITERATE_EXT) {
            const double sg = sigma_s;
            CompStat cs = p.stat[fresh];
            cs.sigma = sg;
            if (sg > 0.0 && isfinite(sg)) {
                const_cast<double *>(p.S)[fresh] = sg;  // (S is read-only elsewhere in this launch)
                cs.valid = 1;
                c_fresh_scale = sg;
            } else {  // the extracted component had no energy: rank exhausted (R14) / non-finite
                cs.status = isfinite(sg) ? 2 : -7;
                st->status = cs.status;
                st->stop = 1;
                st->done = 1;
            }
            p.stat[fresh] = cs;
        }
        if (mode == FIN_LOAD_RAW) {
            st->ny = 1.0;
            st->it = 0;
            st->done = 0;
            st->status = 0;
            inv_s = 1.0;
        } else if (mode == FIN_INIT || mode == FIN_INIT_EXT) {
            st->ny = nyn;
            st->it = 0;
            st->done = 0;
            st->d = 0.0;
            if (!(nyn > 0.0) || !isfinite(nyn)) {  // zero or non-finite initial sample
                st->status = -7;
                st->stop = 1;
                st->done = 1;
            } else {
                st->status = 0;
            }
            inv_s = (nyn > 0.0 && isfinite(nyn)) ? nyn : 1.0;
        } else {  // FIN_ITERATE / FIN_ITERATE_EXT
            if (SRC == SRC_PEER) st->epoch = e + 1u;
            const int itn = it + 1;
            st->it = itn;
            if (st->stop) {
                // the fused extraction found sigma == 0: nothing more to decide
            } else if (!isfinite(nyn)) {
                st->status = -7;
                st->stop = 1;
                st->done = 1;
            } else if (nyn == 0.0) {  // X'^T X' v = 0: rank exhausted (reading R14)
                st->status = 2;
                st->stop = 1;
                st->done = 1;
            } else {
                st->ny = nyn;
                const double d = fabs(tot[1]) / nyn;  // |v0 . v1| with v1 = y / ||y||
                st->d = d;
                if (p.fixed_T > 0) {
                    if (itn >= p.fixed_T) st->done = 1;
                } else if (d >= 1.0 - p.eps) {
                    st->done = 1;
                } else if (itn >= p.max_iter) {
                    st->done = 1;
                    st->status = 1;
                }
            }
            inv_s = (nyn > 0.0 && isfinite(nyn)) ? nyn : 1.0;
            set_cond(p.cond, p.use_cond, (st->done || st->stop) ? 0u : 1u);
            if (p.tl) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 2] = globaltimer_ns();  // debug timeline
        }
    }
    __syncthreads();
    for (int i = tid; i < l; i += kFinThreads)  // c = S V^T v1
        p.c[i] = (i == fresh ? c_fresh_scale : p.S[i]) * (tot[2 + i] / inv_s);
}

// ---------------------------------------------------------------- N6: extraction tail
// NCCL path: local sum of the per-CTA ||u||^2 partials (then ncclAllReduce).
__global__ void ext_reduce(const double *__restrict__ sq_part, int parts, double *__restrict__ sig2,
                           const LoopState *st) {
    griddep_launch();
    griddep_wait();
    if (st->stop) return;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < parts; ++b) s += sq_part[b];
        *sig2 = s;
    }
}

struct ExtParams {
    int64_t rows;
    int n, l;
    const double *u;         // (A v1)_r
    const double *sq_part;   // SRC_PARTS: per-CTA sums of u_r^2
    int parts;
    const double *sig2;      // SRC_YW: all-reduced ||u||^2
    PeerView pv;             // SRC_PEER
    const double *ybuf;
    int64_t ystride;
    float *U;                // m_g x ldu
    int ldu;
    double *V;               // n x ldv
    int ldv;
    double *S;
    CompStat *stat;          // stat[l]
    LoopState *st;
};

// sigma = ||A v1||, U[r,l] = (A v1)_r / sigma, V[j,l] = v1_j, S[l] = sigma
template <int SRC>
__global__ void ext_finish(const ExtParams p) {
    __shared__ int am_last, peer_ok;
    LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop) {  // a previous step hit rank exhaustion / non-finite: record and skip
        if (blockIdx.x == 0 && threadIdx.x == 0 && !p.stat[p.l].valid) {
            p.stat[p.l].status = st->status;
            p.stat[p.l].it = st->it;
        }
        return;
    }
    const unsigned e = st->epoch;
    double sig2 = 0.0;
    if (SRC == SRC_PARTS) {
        for (int b = 0; b < p.parts; ++b) sig2 += p.sq_part[b];  // every block, same order
    } else if (SRC == SRC_YW) {
        sig2 = *p.sig2;
    } else {
        if (threadIdx.x == 0) peer_ok = peer_wait(p.pv, e + 1u, st);
        __syncthreads();
        if (!peer_ok) return;
        const int64_t off = (int64_t)(e & 1u) * p.pv.slot_stride + p.pv.sofs;
        for (int r = 0; r < p.pv.world; ++r) sig2 += __ldcg(p.pv.buf[r] + off);  // rank order
    }
    const double sigma = sqrt(sig2);
    const bool ok = (sigma > 0.0) && isfinite(sigma);
    if (ok) {
        const double ny = st->ny;
        const double *ycur = p.ybuf + (int64_t)(st->it & 1) * p.ystride;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (int64_t r = g; r < p.rows; r += stride) p.U[r * p.ldu + p.l] = (float)(p.u[r] / sigma);
        for (int64_t j = g; j < p.n; j += stride) p.V[j * p.ldv + p.l] = ycur[j] / ny;
    }
    // last block: record the component, advance the peer epoch
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) am_last = (atomicAdd(&st->counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!am_last || threadIdx.x != 0) return;
    st->counter = 0;
    if (SRC == SRC_PEER) st->epoch = e + 1u;
    if (!ok) {
        st->status = isfinite(sigma) ? 2 : -7;
        st->stop = 1;
        p.stat[p.l].status = st->status;
        p.stat[p.l].it = st->it;
        return;
    }
    p.S[p.l] = sigma;
    CompStat cs;
    cs.d = st->d;
    cs.sigma = sigma;
    cs.it = st->it;
    cs.status = st->status;
    cs.valid = 1;
    cs.pad = 0;
    p.stat[p.l] = cs;
}

}  // namespace tsvd
