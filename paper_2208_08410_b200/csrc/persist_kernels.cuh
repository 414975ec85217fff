// persist_kernels.cuh — N7: the whole SVD_1D loop of one component in ONE persistent kernel.
//
// Alg. 2 lines 5-9: repeat { y = X'^T X' v (Eq. 2, factored form F2);
// v1 = y / ||y||; stop when |v0 . v1| >= 1 - eps }.  The separate-kernel path (N1 gv_fused +
// N5 fin_iter per iteration) pays two kernel boundaries per iteration (measured ~30 us of
// transition + ~20 us of finalize on a ~620 us pass).  Here a cooperative grid (one
// CTA per SM slot, all co-resident) runs every pass of the component:
//
//   pass:   stream the CTA's row range through the TMA ring exactly as N1 does (t_r, y += t_r A_r,
//           w += t_r U_r), flush the per-CTA fp64 partials ypart[b], wpart[b]
//   sync 1: grid barrier
//   reduce: CTA b sums a 32-aligned column slice of the partials over all CTAs in a fixed order,
//           applies the V (S w) correction (every CTA reduces w itself), writes y_new, and its
//           slice's partial scalars { sum y^2, sum v y, (V^T y)_0..l-1 } -> part[b]
//   publish: the slice of y_new (fp32) and the slice scalars as stamped words (value + pass stamp)
//   decide: every CTA polls the G slice scalars and sums them in the same fixed order (so every CTA
//           takes the same decision bit for bit), ||y||, d = |v . y| / ||y||, stop test, c = S V^T v1
//           for the next pass; CTA 0 publishes the loop state; the next pass polls the y_new words
//           it needs for v.  No second grid barrier: a stamped word carries its own readiness.
//
// The producer keeps feeding the ring across pass boundaries (A and the U rows do not change
// during a component), so the next pass's first S rows are in flight while the grid reduces.
// The row ranges are walked serpentine (odd passes backwards) when p.serpentine is set.
// Summation orders are fixed: the result is bitwise reproducible run to run.
#pragma once
#include "gram_kernels.cuh"

namespace tsvd {

struct PsParams {
    const float *A;          // row slab, ld floats per row
    int64_t ld;
    int64_t rows;
    int32_t n, n4;
    const float *U;          // rows x ldu fp32 (deflation rows staged with every A row)
    int32_t ldu;
    int32_t l;               // components already found
    int32_t u_bytes;         // round4(l) * 4, 0 if l == 0
    int32_t stages, stage_bytes, row_bytes, run_rows;
    double *ybuf;            // [2][ystride] fp64 iterates
    int64_t ystride;
    LoopState *st;
    double *c;               // c = S V^T v (in: from the init kernel; out: last value)
    const double *S;         // sigma[0..l)
    const double *V;         // n x ldv fp64
    int32_t ldv;
    double *ypart;           // [G][ypart_ld]
    int64_t ypart_ld;
    double *wpart;           // [G][wpart_ld]
    int32_t wpart_ld;
    double *part;            // [G][part_ld] slice scalars (tail_init)
    int32_t part_ld;
    ulonglong2 *pub;         // [G][part_ld] stamped slice scalars of every pass (ll_send words)
    unsigned long long *puby;  // [round4(n)] stamped fp32 y_new words {float bits | stamp << 32}
    unsigned *gbar;          // grid barrier state (2 words, zero-initialised)
    double eps;
    int32_t fixed_T, max_iter;
    int32_t serpentine;
    int32_t part32;          // every CTA's range is a single fp32 run (rows <= run_rows): fp32 partials
    unsigned long long *tl;  // debug timeline (TSVD_TIMELINE), same record layout as N1 + N5
    PxView px;               // world > 1: NVLink peer exchange of the column slices (one block)
    int32_t vcache;          // the CTA's column slice of V[:, :l] cached in shared memory for the
                             // launch (V does not change during a component): Vs[i (per + 1) + c]
    // component transitions inside the kernel (two-vector path, R21):
    // head_ext: the launch starts by reducing the partials of the two-vector pass (gv_fused<TWO>,
    //   fp64 partials, sq_part, u_out) that began this component: sigma_fresh = ||u||, U[:, fresh] =
    //   u / sigma, S[fresh], stat[fresh]; weight 1 on the fresh column in g, sigma in c
    // tail_init: after the stop decision, initialise component l + 1: V[:, l] = v, vprev32 = v,
    //   y_cur = x_{l+1} (V0n), ||x||, c = S V^T x / ||x|| (weight 1 on column l), stat[l]
    int32_t head_ext, tail_init;
    int32_t fresh;           // head_ext: the component being extracted (l - 1)
    double *Sw;              // writable S (head_ext)
    double *Vw;              // writable V (tail_init)
    float *Uw;               // writable U (head_ext)
    const double *u_out;     // head_ext: (A v_fresh)_r of this rank's rows, fp64
    const double *sq_part;   // head_ext: per-CTA sums of u_r^2 of the two-vector pass
    CompStat *stat;
    const double *V0n;       // tail_init: x_{l+1}
    float *vprev32;          // tail_init: fp32 copy of v_l for the next two-vector pass
};

constexpr int kPsLanesV = 4;  // (V^T y) accumulators per lane: components l <= 128
// doubles of slice-reduction scratch: T (one per thread) or, for T >= 128, [T/32 warps][128 columns]
// (fp32 partials are read as float4: a warp covers a 128-column block of one partial row)
__host__ __device__ constexpr int kPsGred(int T) { return T >= 128 ? 4 * T : T; }

// sum_{b = first, first + step, ... < count} base[b * ld], in that order, with U loads in flight at a
// time (these reductions are L2-latency bound: one round trip per batch instead of per element)
template <int U, typename E>
__device__ __forceinline__ double strided_sum(const E *base, int64_t ld, int first, int step, int count) {
    double acc = 0.0;
    for (int b0 = first; b0 < count; b0 += U * step) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int bb = b0 + u * step;
            v[u] = bb < count ? (double)__ldcg(base + (int64_t)bb * ld) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (b0 + u * step < count) acc += v[u];
    }
    return acc;
}

// Low-latency exchange word pair: {lo32 | stamp << 32, hi32 | stamp << 32}.  Each 8-byte word is
// written and read single-copy atomically, so a word whose stamp matches carries the right half.
__device__ __forceinline__ void ll_send(ulonglong2 *dst, unsigned stamp, double x) {
    const unsigned long long s = (unsigned long long)stamp << 32;
    const unsigned long long a = s | (unsigned)__double2loint(x), b = s | (unsigned)__double2hiint(x);
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ll_send_gpu(ulonglong2 *dst, unsigned stamp, double x) {
    const unsigned long long s = (unsigned long long)stamp << 32;
    const unsigned long long a = s | (unsigned)__double2loint(x), b = s | (unsigned)__double2hiint(x);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_volatile_u2(const void *src) {
    ulonglong2 v;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(src) : "memory");
    return v;
}
// Poll until both words carry `stamp`; after 30 s mark the run failed (status -6) and return 0.
__device__ __forceinline__ double ll_recv(const ulonglong2 *src, unsigned stamp, unsigned long long t0,
                                         LoopState *st) {
    for (unsigned spin = 0;; ++spin) {
        unsigned long long a, b;
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(src) : "memory");
        if ((unsigned)(a >> 32) == stamp && (unsigned)(b >> 32) == stamp)
            return __hiloint2double((int)(unsigned)b, (int)(unsigned)a);
        if ((spin & 1023) == 1023 && globaltimer_ns() - t0 > 30000000000ull) {  // a rank did not arrive
            st->status = -6;
            st->stop = 1;
            return 0.0;
        }
    }
}

// strided_sum over stamped words, one attempt: U loads in flight per batch, `ok` cleared if any
// word is not yet current (the caller waits and retries); the summation order is that of strided_sum
template <int U>
__device__ __forceinline__ double ll_try_sum(const ulonglong2 *base, int64_t ld, int first, int step, int count,
                                             unsigned stamp, bool &ok) {
    double acc = 0.0;
    for (int b0 = first; b0 < count; b0 += U * step) {
        ulonglong2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int bb = b0 + u * step;
            v[u] = bb < count ? ld_volatile_u2(base + (int64_t)bb * ld) : make_ulonglong2(0ull, 0ull);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (b0 + u * step < count) {
                ok &= (unsigned)(v[u].x >> 32) == stamp && (unsigned)(v[u].y >> 32) == stamp;
                acc += __hiloint2double((int)(unsigned)v[u].y, (int)(unsigned)v[u].x);
            }
    }
    return acc;
}

// FULL: n == 4 NV T (every thread's NV float4 columns exist, no tail): the row loop drops its
// per-element bounds checks (fewer instructions per row, which matters when the SM clock is capped)
template <int T, int NV, bool FULL = false>
__global__ void __launch_bounds__(T) gv_persist(const PsParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NW = T / 32;
    griddep_launch();
    griddep_wait();
    LoopState *st = p.st;
    if (st->stop || st->done) return;  // every CTA reads the same state: uniform exit
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int S = p.stages, l = p.l;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
    double *red = reinterpret_cast<double *>(bars + kMaxStages);  // [2][NW] row dot partials
    double *cvec = red + 2 * NW;                                   // [l] c = S V^T v
    double *gvec = cvec + p.wpart_ld;                              // [l] S w
    double *tot = gvec + p.wpart_ld;                               // [2 + l] decision sums
    double *gred = tot + 2 + p.wpart_ld;                           // [kPsGred(T)] slice reduction
    double *ys = gred + kPsGred(T);                                // [128] y of the column block
    double *Ssm = ys + 128;  // [l] sigma (the per-pass reductions read it twice: no L2 round trip)
    double *Vs = Ssm + p.wpart_ld;  // vcache: [l][per + 1] (odd stride: the column-owner reads and
                                    // the component-per-lane reads are both bank-conflict free)
    __shared__ int64_t slot_row[kMaxStages];
    __shared__ double ny_s;
    __shared__ int done_s;
    __shared__ int xfail_s;
    __shared__ int tout_s;   // the decision poll gave up (30 s): block-uniform exit flag  // world > 1: an exchange timed out (st->stop raised) before publication
    __shared__ double sred[2][32];
    // producer state (thread 0 only; kept in shared memory to leave the registers to the row loop):
    // next row index pk within pass pp of the range [plo, plo + pnr), next ring slot pslot
    __shared__ int64_t plo, pnr, pk;
    __shared__ int pp, pslot, pit0;
    // pass stamps (monotone across launches and runs: a stamp never repeats): the words published by
    // iteration `it` carry xeb_s + it + 1; kept in shared memory with it0_s to spare the row loop's
    // registers
    __shared__ unsigned xeb_s;
    __shared__ int it0_s;

    const int64_t nr = p.rows * (b + 1) / G - p.rows * b / G;
    const int it0 = st->it;
    int it = it0;

    auto feed = [&]() {  // thread 0: next row of the (endless) serpentine sequence into the ring
        const int64_t k = pk;
        const int64_t row = (p.serpentine && ((pit0 + pp) & 1)) ? plo + pnr - 1 - k : plo + k;
        if (k + 1 == pnr) {
            pk = 0;
            pp = pp + 1;
        } else {
            pk = k + 1;
        }
        const int slot = pslot;
        pslot = slot + 1 == S ? 0 : slot + 1;
        slot_row[slot] = row;
        unsigned char *dst = smem + (size_t)slot * p.stage_bytes;
        mbar_arrive_expect_tx(&bars[slot], (uint32_t)(p.n4 * 16 + (l > 0 ? p.u_bytes : 0)));
        tma_load_1d(dst, p.A + row * p.ld, (uint32_t)(p.n4 * 16), &bars[slot]);
        if (l > 0) tma_load_1d(dst + p.row_bytes, p.U + row * p.ldu, (uint32_t)p.u_bytes, &bars[slot]);
    };
    if (tid == 0) {
        plo = p.rows * b / G;
        pnr = nr;
        pk = 0;
        pp = 0;
        pslot = 0;
        pit0 = it0 + (p.head_ext ? 1 : 0);  // head: the first pass run here is iteration it0 + 1
        xeb_s = st->xepoch - (unsigned)it0;
        it0_s = it0;
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
        // head: the first rows are fed after the U column of the fresh component is written
        if (nr > 0 && !p.head_ext)
            for (int s = 0; s < S; ++s) feed();
    }
    for (int i = tid; i < l; i += T) {
        cvec[i] = p.c[i];
        Ssm[i] = p.S[i];  // (head: entry `fresh` is set from the head's own sigma below)
    }
    if (p.vcache) {  // this CTA's column slice of V[:, :l] (the slice geometry of the reduction below)
        const int Gs = p.px.world > 1 ? p.px.G : G;
        const int per = (int)(((p.n + Gs - 1) / Gs + 31) / 32 * 32);
        const int64_t j0 = b < Gs ? (int64_t)b * per : (int64_t)p.n;
        const int64_t j1 = (j0 + per) < (int64_t)p.n ? (j0 + per) : (int64_t)p.n;
        for (int idx = tid; idx < l * per; idx += T) {
            const int i = idx / per, c = idx - i * per;
            Vs[i * (per + 1) + c] = j0 + c < j1 ? p.V[(j0 + c) * p.ldv + i] : 0.0;
        }
    }
    if (tid == 0) ny_s = st->ny;
    __syncthreads();

    const int tail = p.n & 3;
    int cs = 0;         // consumer: ring slot of the next row
    uint32_t cph = 0;   // and the phase to wait for
    int rb = 0;         // parity of the dot-product scratch
    double *yp = p.ypart + (int64_t)b * p.ypart_ld;
    __shared__ double sigma_s;
    bool head = p.head_ext != 0;
    for (;;) {
      if (!head) {
        // ---- v = y_cur / ||y_cur|| in registers (fp64 master -> fp32), c for this pass
        float4 vr[NV];
        {
            const double inv = 1.0 / ny_s;
            const double *ycur = p.ybuf + (int64_t)(it & 1) * p.ystride;
            // y_new of the previous pass of this launch: the stamped fp32 words published by the slice
            // owners (p.puby); the first pass of a launch reads the fp64 ybuf of a prior kernel.  Both
            // are 8 bytes per column: one load sequence, the interpretation selected per word
            const bool pub = it != it0_s;
            const unsigned xe = xeb_s + (unsigned)it;
            const unsigned long long *src =
                pub ? p.puby : reinterpret_cast<const unsigned long long *>(ycur);
            auto build = [&]() -> bool {  // straight-line: loads, stamp checks, v; false if a word is stale
                bool ok = true;
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int idx = k * T + tid;
                    const int j = 4 * idx;
                    float f[4] = {0.f, 0.f, 0.f, 0.f};
                    if (FULL || idx < p.n4) {  // (both buffers hold round4(n) words)
                        // L2 loads (ld.cg: never a stale L1 line); a stale stamped word is re-polled
                        const ulonglong2 w0 = __ldcg(reinterpret_cast<const ulonglong2 *>(src) + 2 * (int64_t)idx);
                        const ulonglong2 w1 = __ldcg(reinterpret_cast<const ulonglong2 *>(src) + 2 * (int64_t)idx + 1);
                        const unsigned long long wd[4] = {w0.x, w0.y, w1.x, w1.y};
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (FULL || j + c < p.n) {
                                ok &= !pub || (unsigned)(wd[c] >> 32) == xe;
                                const double y = pub ? (double)__uint_as_float((unsigned)wd[c])
                                                     : __longlong_as_double((long long)wd[c]);
                                f[c] = (float)(y * inv);
                            }
                    }
                    vr[k] = make_float4(f[0], f[1], f[2], f[3]);
                }
                return ok;
            };
            // a stale word (its owner's y stores and scalar stores come from different threads, so the
            // scalars can be seen first) costs one more round of the same parallel loads
            const unsigned long long t0 = globaltimer_ns();
            for (unsigned spin = 1; !build(); ++spin) {
                if ((spin & 255) == 0 && globaltimer_ns() - t0 > 30000000000ull) {
                    st->status = -6;
                    st->stop = 1;
                    break;
                }
                __nanosleep(128);
            }
        }
        const double cval = tid < l ? cvec[tid] : 0.0;
        if (p.tl && b == 0 && tid == 0) {
            const unsigned long long idx = atomicAdd(p.tl, 1ull) % 4096;
            p.tl[2 + kTl * idx] = globaltimer_ns();
        }

        // ---- the pass over this CTA's rows (N1 body)
        float4 ya[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) ya[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        double wacc = 0.0;
        bool flushed = false;
        auto flush = [&]() {
            if (p.part32) {  // one fp32 run per pass: the partial IS an fp32 sum, store it as such
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int idx = k * T + tid;
                    if (FULL || idx < p.n4) reinterpret_cast<float4 *>(yp)[idx] = ya[k];
                    ya[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                return;
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int idx = k * T + tid;
                if (idx < p.n4) {
                    double2 *dst = reinterpret_cast<double2 *>(yp + 4 * (int64_t)idx);
                    double2 lo2 = make_double2(ya[k].x, ya[k].y), hi2 = make_double2(ya[k].z, ya[k].w);
                    if (flushed) {
                        const double2 olo = dst[0], ohi = dst[1];
                        lo2.x += olo.x; lo2.y += olo.y; hi2.x += ohi.x; hi2.y += ohi.y;
                    }
                    dst[0] = lo2;
                    dst[1] = hi2;
                }
                ya[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            flushed = true;
        };
        int run = 0;
        for (int64_t k = 0; k < nr; ++k) {
            mbar_wait(&bars[cs], cph);
            const unsigned char *slot = smem + (size_t)cs * p.stage_bytes;
            const float4 *row = reinterpret_cast<const float4 *>(slot);
            float4 a[NV];
            float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
            for (int kk = 0; kk < NV; ++kk) {
                const int idx = kk * T + tid;
                if (FULL || idx < p.n4) {
                    a[kk] = row[idx];
                    if (!FULL && tail && idx == p.n4 - 1) {
                        if (tail < 2) a[kk].y = 0.f;
                        if (tail < 3) a[kk].z = 0.f;
                        a[kk].w = 0.f;
                    }
                } else {
                    a[kk] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                q0 = fmaf(a[kk].x, vr[kk].x, q0);
                q1 = fmaf(a[kk].y, vr[kk].y, q1);
                q2 = fmaf(a[kk].z, vr[kk].z, q2);
                q3 = fmaf(a[kk].w, vr[kk].w, q3);
            }
            double part = (double)((q0 + q1) + (q2 + q3));
            float ur = 0.f;
            if (tid < l) {
                ur = reinterpret_cast<const float *>(slot + p.row_bytes)[tid];
                part -= (double)ur * cval;  // - U_r . c
            }
            part = warp_sum(part);
            if (lane == 0) red[rb * NW + warp] = part;
            __syncthreads();  // dots visible; every thread is done reading the slot
            if (tid == 0) {
                fence_proxy_async_smem();
                feed();  // keeps S rows in flight, across the pass boundary too
            }
            double t = 0.0;
            t = sum_warps<NW>(red + rb * NW, lane);
            rb ^= 1;
            if (++cs == S) {
                cs = 0;
                cph ^= 1u;
            }
            const float tf = (float)t;
#pragma unroll
            for (int kk = 0; kk < NV; ++kk) {
                ya[kk].x = fmaf(tf, a[kk].x, ya[kk].x);
                ya[kk].y = fmaf(tf, a[kk].y, ya[kk].y);
                ya[kk].z = fmaf(tf, a[kk].z, ya[kk].z);
                ya[kk].w = fmaf(tf, a[kk].w, ya[kk].w);
            }
            if (tid < l) wacc += t * (double)ur;
            if (++run == p.run_rows && !p.part32) {  // part32: the single run is flushed after the loop
                flush();
                run = 0;
            }
        }
        flush();
        if (tid < l) p.wpart[(int64_t)b * p.wpart_ld + tid] = wacc;
        grid_sync(p.gbar);  // sync 1: every partial is written
        if (p.tl && b == 0 && tid == 0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 1] = globaltimer_ns();
      }
        // head: the partials are those of the two-vector pass (an earlier kernel: fp64, visible)
        const bool ext = head;
        const bool p32 = p.part32 && !ext;
        const int fresh = ext ? p.fresh : -1;
        const bool xsq = ext && b == 0;  // CTA 0 (column slice 0 on every rank) carries ||u||^2

        // ---- g = S w (every CTA, fixed order), then this CTA's column slice of y_new.  world > 1:
        // gvec holds the local w until the exchange has delivered every rank's
        const bool multi = p.px.world > 1;
        const double *ycur = p.ybuf + (int64_t)(it & 1) * p.ystride;
        double *ynew = p.ybuf + (int64_t)((it + 1) & 1) * p.ystride;
        const double inv = 1.0 / ny_s;
        // column slices: G of them (world > 1: px.G, the smallest grid of any rank, so that every
        // rank cuts the columns the same way)
        const int Gs = multi ? p.px.G : G;
        const int64_t per = ((p.n + Gs - 1) / Gs + 31) / 32 * 32;
        const int64_t j0 = b < Gs ? (int64_t)b * per : (int64_t)p.n;
        const int64_t j1 = (j0 + per) < (int64_t)p.n ? (j0 + per) : (int64_t)p.n;
        // column blocks of CW columns: PG thread groups sum interleaved subsets of the G partials of
        // one column each (independent loads, unrolled), group sums added in group order
        constexpr int CW = T < 128 ? T : 128;
        constexpr int PG = T / CW;
        const int cc = tid % CW, cg = tid / CW;
        double a_yy = 0.0, a_vy = 0.0;
        double vacc[kPsLanesV];  // (V^T y)_i, i = lane + 32 q, partial over the columns of this warp
#pragma unroll
        for (int q = 0; q < kPsLanesV; ++q) vacc[q] = 0.0;
        for (int64_t c0 = j0; c0 < j1; c0 += CW) {
            const int64_t j = c0 + cc;
            constexpr bool kVec = CW == 128;  // fp32 partials as float4: warp w sums partials w, w+NW, ...
            const bool vec = kVec && p32;
            if (vec) {
                const int64_t jv = c0 + 4 * lane;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                if (jv < j1) {
                    const float *col = reinterpret_cast<const float *>(p.ypart) + jv;
                    const int64_t ld32 = 2 * p.ypart_ld;
                    constexpr int U = NW >= 16 ? 12 : 20;  // one round of loads for G <= U NW (148 CTAs)
                    for (int b0 = warp; b0 < G; b0 += U * NW) {
                        float4 v[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int bb = b0 + u * NW;
                            v[u] = bb < G ? __ldcg(reinterpret_cast<const float4 *>(col + (int64_t)bb * ld32))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (b0 + u * NW < G) {
                                s0 += (double)v[u].x;
                                s1 += (double)v[u].y;
                                s2 += (double)v[u].z;
                                s3 += (double)v[u].w;
                            }
                    }
                }
                double *gw = gred + warp * 128 + 4 * lane;
                gw[0] = s0;
                gw[1] = s1;
                gw[2] = s2;
                gw[3] = s3;
            } else {
                double sacc = 0.0;
                if (j < j1)
                    sacc = p32 ? strided_sum<40>(reinterpret_cast<const float *>(p.ypart) + j, 2 * p.ypart_ld, cg, PG, G)
                               : strided_sum<40>(p.ypart + j, p.ypart_ld, cg, PG, G);
                gred[cg * CW + cc] = sacc;
            }
            if (c0 == j0) {  // w = U^T t summed over the CTAs (issued after the slice loads: one more round)
                for (int i = warp; i < l; i += NW) {
                    const double w = warp_sum(strided_sum<8>(p.wpart + i, p.wpart_ld, lane, 32, G));
                    if (lane == 0) gvec[i] = multi ? w : (i == fresh ? 1.0 : Ssm[i]) * w;
                }
                if (xsq && warp == NW - 1) {  // ||u||^2 of this rank (sigma of the fresh component)
                    const double q = warp_sum(strided_sum<8>(p.sq_part, 1, lane, 32, G));
                    if (lane == 0) sigma_s = q;
                }
            }
            __syncthreads();
            if (p.tl && b == 0 && tid == 0 && c0 == j0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 3] = globaltimer_ns();
            double y = 0.0;
            if (tid < CW && j < j1) {
                if (vec) {
                    y = gred[tid];
#pragma unroll
                    for (int q = 1; q < NW; ++q) y += gred[q * 128 + tid];
                } else {
                    y = gred[tid];
#pragma unroll
                    for (int q = 1; q < PG; ++q) y += gred[q * CW + tid];
                }
            }
            if (multi) {  // push my slice (+ local w) to every rank, wait for every rank's, sum in rank order
                // low-latency protocol: every 8-byte word carries half of the value and the pass
                // stamp, so a receiver polls the data itself (no fence, no separate flag)
                const unsigned target = xeb_s + (unsigned)it + 1u;
                const int64_t so = ((int64_t)(target & 1u) * p.px.world * Gs + b) * p.px.SL;  // + src * Gs * SL
                const int64_t mine = so + (int64_t)p.px.rank * Gs * p.px.SL;
                for (int r = 0; r < p.px.world; ++r) {
                    ulonglong2 *dst = p.px.rbuf[r] + mine;
                    if (tid < CW && j < j1) ll_send(dst + tid, target, y);
                    if (tid < l) ll_send(dst + p.px.per + tid, target, gvec[tid]);
                    if (xsq && tid == T - 1) ll_send(dst + p.px.per + l, target, sigma_s);
                }
                const ulonglong2 *src = p.px.lbuf + so;
                const unsigned long long t0 = globaltimer_ns();
                // elements to receive: [rank][CW slice values | l w | ||u||^2 (head)]
                const int EL = CW + l + (xsq ? 1 : 0);
                const int E = p.px.world * EL;
                if (E <= kPsGred(T)) {  // one element per thread: all polls in flight at once
                    __syncthreads();    // gred (the local sums) and gvec (local w) have been read
                    for (int e = tid; e < E; e += T) {
                        const int r = e / EL, c = e - r * EL;
                        double v = 0.0;
                        if (c >= CW) v = ll_recv(src + (int64_t)r * Gs * p.px.SL + p.px.per + (c - CW), target, t0, st);
                        else if (c0 + c < j1) v = ll_recv(src + (int64_t)r * Gs * p.px.SL + c, target, t0, st);
                        gred[e] = v;
                    }
                    __syncthreads();
                    if (tid < CW && j < j1) {  // ranks in order
                        y = 0.0;
                        for (int r = 0; r < p.px.world; ++r) y += gred[r * EL + tid];
                    }
                    if (tid < l) {
                        double w = 0.0;
                        for (int r = 0; r < p.px.world; ++r) w += gred[r * EL + CW + tid];
                        gvec[tid] = (tid == fresh ? 1.0 : Ssm[tid]) * w;
                    }
                    if (xsq && tid == T - 1) {
                        double q = 0.0;
                        for (int r = 0; r < p.px.world; ++r) q += gred[r * EL + CW + l];
                        sigma_s = q;
                    }
                } else {
                    if (tid < CW && j < j1) {
                        y = 0.0;
                        for (int r = 0; r < p.px.world; ++r)
                            y += ll_recv(src + (int64_t)r * Gs * p.px.SL + tid, target, t0, st);
                    }
                    __syncthreads();  // every thread is done with gvec (local w) and sigma_s
                    if (tid < l) {
                        double w = 0.0;
                        for (int r = 0; r < p.px.world; ++r)
                            w += ll_recv(src + (int64_t)r * Gs * p.px.SL + p.px.per + tid, target, t0, st);
                        gvec[tid] = (tid == fresh ? 1.0 : Ssm[tid]) * w;
                    }
                    if (xsq && tid == T - 1) {
                        double q = 0.0;
                        for (int r = 0; r < p.px.world; ++r)
                            q += ll_recv(src + (int64_t)r * Gs * p.px.SL + p.px.per + l, target, t0, st);
                        sigma_s = q;
                    }
                }
                __syncthreads();
                if (p.tl && b == 0 && tid == 0 && c0 == j0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 4] = globaltimer_ns();
            }
            if (tid < CW) {
                if (j < j1) {
                    double corr = 0.0;  // (V (S w))_j
                    if (p.vcache) {
                        const double *Vj = Vs + (j - j0);
                        for (int i = 0; i < l; ++i) corr += Vj[i * (per + 1)] * gvec[i];
                    } else {
                        const double *Vj = p.V + j * p.ldv;
#pragma unroll 4
                        for (int i = 0; i < l; ++i) corr += Vj[i] * gvec[i];
                    }
                    y -= corr;
                    __stcg(ynew + j, y);
                    __stcg(p.puby + j, ((unsigned long long)(xeb_s + (unsigned)it + 1u) << 32) | __float_as_uint((float)y));
                    a_yy += y * y;
                    a_vy += (__ldcg(ycur + j) * inv) * y;
                }
                ys[tid] = y;
            }
            __syncthreads();
            if (l > 0) {  // warp w: columns w, w + NW, ... of the block; lane: components lane + 32 q
                const int jn = (int)((j1 - c0) < CW ? (j1 - c0) : CW);
                for (int jj = warp; jj < jn; jj += NW) {
                    const double yj = ys[jj];
                    if (p.vcache) {
                        const double *Vr = Vs + (c0 + jj - j0);
#pragma unroll
                        for (int q = 0; q < kPsLanesV; ++q)
                            if (lane + 32 * q < l) vacc[q] += Vr[(lane + 32 * q) * (per + 1)] * yj;
                    } else {
                        const double *Vr = p.V + (c0 + jj) * p.ldv;
#pragma unroll
                        for (int q = 0; q < kPsLanesV; ++q)
                            if (lane + 32 * q < l) vacc[q] += Vr[lane + 32 * q] * yj;
                    }
                }
            }
            __syncthreads();
        }
        if (p.tl && b == 0 && tid == 0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 5] = globaltimer_ns();
        const unsigned pst = xeb_s + (unsigned)it + 1u;  // this pass's stamp
        if (tid == 0) xfail_s = multi ? *reinterpret_cast<volatile int32_t *>(&st->stop) : 0;
        ulonglong2 *pb = p.pub + (int64_t)b * p.part_ld;
        {  // block sums in a fixed order: warps (of the CW column threads), then lanes; published as
           // stamped words (a CTA whose exchange timed out publishes -inf for ||y||^2)
            const double yy = warp_sum(a_yy), vy = warp_sum(a_vy);
            if (lane == 0 && warp < CW / 32) {
                sred[0][warp] = yy;
                sred[1][warp] = vy;
            }
            __syncthreads();
            if (tid < 2) {
                double acc = 0.0;
                for (int w = 0; w < CW / 32; ++w) acc += sred[tid][w];
                if (tid == 0 && xfail_s) acc = -INFINITY;
                ll_send_gpu(pb + tid, pst, acc);
            }
            if (ext && tid == 2) ll_send_gpu(pb + 2 + l, pst, xsq ? sigma_s : 0.0);  // ||u||^2 rides along
#pragma unroll
            for (int q = 0; q < kPsLanesV; ++q) {
                if (32 * q >= l) break;
                __syncthreads();
                gred[warp * 32 + lane] = vacc[q];
                __syncthreads();
                if (tid < 32 && 32 * q + tid < l) {
                    double acc = 0.0;
                    for (int w = 0; w < NW; ++w) acc += gred[w * 32 + tid];
                    ll_send_gpu(pb + 2 + 32 * q + tid, pst, acc);
                }
            }
        }
        if (p.tl && b == 0 && tid == 0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 6] = globaltimer_ns();

        // ---- decision: identical in every CTA (same data, same fixed order).  Polling every CTA's
        // stamped scalars is also the grid-wide ordering point: a CTA that has them all knows every
        // CTA has finished reading this pass's partials (its next flush may overwrite them)
        {  // half-warp per quantity, 16 lanes striding the CTAs: one round of loads for 2 + l <= 2 NW.
           // A CTA that finds a stale word (its peers are still reducing) does not keep the whole
           // block polling (that load storm slows the late CTAs down): warp 0 alone polls, with a
           // back-off, the word each CTA writes last, then the block loads everything again
            const int hl = lane & 15;
            const int nq = 2 + l + (ext ? 1 : 0);
            const int qlast = l > 0 ? 2 + l - 1 : 1;
            const unsigned long long t0 = globaltimer_ns();
            for (;;) {
                bool ok = true;
                for (int q0 = 2 * warp; q0 < nq; q0 += 2 * NW) {  // warp-uniform trip count
                    const int q = q0 + (lane >> 4);
                    double sq = q < nq ? ll_try_sum<10>(p.pub + q, p.part_ld, hl, 16, G, pst, ok) : 0.0;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                    if (hl == 0 && q < nq) tot[q] = sq;
                }
                if (__syncthreads_and(ok)) break;
                if (warp == 0) {
                    for (int bb = lane; bb < G; bb += 32)
                        for (unsigned spin = 0;; ++spin) {
                            const ulonglong2 w = ld_volatile_u2(p.pub + (int64_t)bb * p.part_ld + qlast);
                            if ((unsigned)(w.x >> 32) == pst && (unsigned)(w.y >> 32) == pst) break;
                            if ((spin & 255) == 255 && globaltimer_ns() - t0 > 30000000000ull) {
                                st->status = -6;  // a CTA never published: give up (the run fails)
                                st->stop = 1;
                                break;
                            }
                            __nanosleep(64);
                        }
                }
                // the give-up decision is taken once (thread 0) and shared, so every thread of the
                // block leaves the poll loop together (a per-thread clock read could split the block
                // between the __syncthreads_and above and the barrier below)
                __syncthreads();
                if (tid == 0) tout_s = globaltimer_ns() - t0 > 30000000000ull;
                __syncthreads();
                if (tout_s) break;
            }
        }
        __syncthreads();
        if (p.tl && b == 0 && tid == 0) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 7] = globaltimer_ns();
        const int itn = it + 1;
        if (tid == 0) {
            const double nyn = sqrt(tot[0]);
            int done = 0, status = 0;
            double d = 0.0;
            // a CTA whose exchange timed out (st->stop raised) published -inf: every CTA leaves
            const int peer_fail = multi && tot[0] < 0.0;
            const double sg = ext ? sqrt(tot[2 + l]) : 1.0;  // sigma of the fresh component
            sigma_s = sg;
            if (peer_fail) {
                done = 3;
            } else if (ext && !(sg > 0.0 && isfinite(sg))) {  // the extracted component had no energy
                status = isfinite(sg) ? 2 : -7;
                done = 2;
            } else if (!isfinite(nyn)) {
                status = -7;
                done = 2;
            } else if (nyn == 0.0) {  // X'^T X' v = 0: rank exhausted (reading R14)
                status = 2;
                done = 2;
            } else {
                d = fabs(tot[1]) / nyn;  // |v0 . v1| with v1 = y / ||y||
                if (p.fixed_T > 0) {
                    if (itn >= p.fixed_T) done = 1;
                } else if (d >= 1.0 - p.eps) {
                    done = 1;
                } else if (itn >= p.max_iter) {
                    done = 1;
                    status = 1;
                }
            }
            ny_s = (nyn > 0.0 && isfinite(nyn)) ? nyn : 1.0;
            // a CTA that gave up waiting (30 s) has already set status -6 and stop: keep them
            if (*reinterpret_cast<volatile int32_t *>(&st->status) == -6) done = 3;
            done_s = done;
            if (b == 0) {
                st->it = itn;
                if (done < 2) {
                    st->ny = nyn;
                    st->d = d;
                }
                if (done == 3) st->done = 1;  // status -6 / stop already set by the timed-out CTA
                if (done == 1 || done == 2) {
                    st->status = status;
                    st->done = 1;
                    if (done == 2) st->stop = 1;
                }
                st->xepoch = xeb_s + (unsigned)itn;
                if (ext) {  // the fresh component's sigma; its it/d/status came with tail_init
                    CompStat cs = p.stat[fresh];
                    cs.sigma = sg;
                    if (sg > 0.0 && isfinite(sg)) {
                        p.Sw[fresh] = sg;
                        cs.valid = 1;
                    } else {
                        cs.status = status;
                    }
                    p.stat[fresh] = cs;
                }
                if (p.tl) p.tl[2 + kTl * ((p.tl[0] - 1) % 4096) + 2] = globaltimer_ns();
            }
        }
        __syncthreads();
        for (int i = tid; i < l; i += T) {  // c = S V^T v1 for the next pass (sigma for the fresh column)
            cvec[i] = (i == fresh ? sigma_s : Ssm[i]) * (tot[2 + i] / ny_s);
            if (b == 0) p.c[i] = cvec[i];
        }
        if (ext) {  // U[:, fresh] = u / sigma on this CTA's rows, then start the row stream
            const double sg = sigma_s;
            if (tid == 0) Ssm[fresh] = sg;  // the cached sigma of the column extracted just now
            const int64_t r0 = p.rows * b / G;
            if (sg > 0.0 && isfinite(sg))
                for (int64_t r = r0 + tid; r < r0 + nr; r += T) p.Uw[r * p.ldu + fresh] = (float)(p.u_out[r] / sg);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // U rows are read by TMA next
            __syncthreads();
            if (tid == 0 && nr > 0)
                for (int s2 = 0; s2 < S; ++s2) feed();
        }
        head = false;
        it = itn;
        const int done = done_s;
        __syncthreads();
        if (done) break;
    }
    if (p.tail_init && done_s == 1) {
        // ---- component l + 1: V[:, l] = v, the fp32 copy for the next two-vector
        // pass, y_cur = x, ||x||, c = S V^T x / ||x|| with weight 1 on column l (its sigma comes with
        // the next pass, R21).  Same column slices as the reduction; V and x are replicated, so every
        // rank computes the same values without an exchange.
        constexpr int CW = T < 128 ? T : 128;
        const int Gs = p.px.world > 1 ? p.px.G : G;
        const int64_t per = ((p.n + Gs - 1) / Gs + 31) / 32 * 32;
        const int64_t j0 = b < Gs ? (int64_t)b * per : (int64_t)p.n;
        const int64_t j1 = (j0 + per) < (int64_t)p.n ? (j0 + per) : (int64_t)p.n;
        const double *yfin = p.ybuf + (int64_t)(it & 1) * p.ystride;
        double *x0 = p.ybuf;  // the next component starts at it = 0
        const double inv = 1.0 / ny_s;
        const int l1 = l + 1;
        double a_xx = 0.0;
        double vacc[kPsLanesV];
#pragma unroll
        for (int q = 0; q < kPsLanesV; ++q) vacc[q] = 0.0;
        for (int64_t c0 = j0; c0 < j1; c0 += CW) {
            if (tid < CW) {
                const int64_t j = c0 + tid;
                double x = 0.0;
                if (j < j1) {
                    const double v = __ldcg(yfin + j) * inv;  // read before x0 (maybe the same buffer) is written
                    p.Vw[j * p.ldv + l] = v;
                    p.vprev32[j] = (float)v;
                    x = p.V0n[j];
                    __stcg(x0 + j, x);
                    a_xx += x * x;
                }
                ys[tid] = x;
            }
            __syncthreads();
            const int jn = (int)((j1 - c0) < CW ? (j1 - c0) : CW);
            for (int jj = warp; jj < jn; jj += NW) {  // (V^T x)_i, columns 0..l (column l written above)
                const double *Vr = p.V + (c0 + jj) * p.ldv;
                const double xj = ys[jj];
#pragma unroll
                for (int q = 0; q < kPsLanesV; ++q)
                    if (lane + 32 * q < l1) vacc[q] += Vr[lane + 32 * q] * xj;
            }
            __syncthreads();
        }
        double *pp = p.part + (int64_t)b * p.part_ld;
        {
            const double xx = warp_sum(a_xx);
            if (lane == 0 && warp < CW / 32) sred[0][warp] = xx;
            __syncthreads();
            if (tid == 0) {
                double acc = 0.0;
                for (int w = 0; w < CW / 32; ++w) acc += sred[0][w];
                pp[0] = acc;
            }
#pragma unroll
            for (int q = 0; q < kPsLanesV; ++q) {
                if (32 * q >= l1) break;
                __syncthreads();
                gred[warp * 32 + lane] = vacc[q];
                __syncthreads();
                if (tid < 32 && 32 * q + tid < l1) {
                    double acc = 0.0;
                    for (int w = 0; w < NW; ++w) acc += gred[w * 32 + tid];
                    pp[2 + 32 * q + tid] = acc;
                }
            }
        }
        __threadfence();
        grid_sync(p.gbar);
        {
            const int hl = lane & 15;
            const int nq = 2 + l1;
            for (int q0 = 2 * warp; q0 < nq; q0 += 2 * NW) {
                const int q = q0 + (lane >> 4);
                double sq = (q < nq && q != 1) ? strided_sum<10>(p.part + q, p.part_ld, hl, 16, G) : 0.0;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                if (hl == 0 && q < nq) tot[q] = sq;
            }
        }
        __syncthreads();
        const double nyx = sqrt(tot[0]);
        const bool okx = nyx > 0.0 && isfinite(nyx);
        if (b == 0) {
            if (tid == 0) {
                CompStat cs = p.stat[l];  // the finished component (sigma comes with the next pass)
                cs.it = it;
                cs.d = st->d;
                cs.status = st->status;
                p.stat[l] = cs;
                st->it = 0;
                st->ny = okx ? nyx : 1.0;
                st->d = 0.0;
                st->done = okx ? 0 : 1;
                st->status = okx ? 0 : -7;
                if (!okx) st->stop = 1;
            }
            for (int i = tid; i < l1; i += T)
                p.c[i] = (i == l ? 1.0 : p.S[i]) * (tot[2 + i] / (okx ? nyx : 1.0));
        }
    }
    // drain the S rows fed ahead for a pass that will not run (no bulk copy may outlive the CTA)
    if (tid == 0 && nr > 0)
        for (int j = 0; j < S; ++j) {
            mbar_wait(&bars[cs], cph);
            if (++cs == S) {
                cs = 0;
                cph ^= 1u;
            }
        }
}

}  // namespace tsvd
