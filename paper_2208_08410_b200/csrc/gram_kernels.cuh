// gram_kernels.cuh — sm_100a kernels of the Gram-vector hot path.
//
// One power iteration (Alg. 2 lines 11-14) on one GPU is TWO kernels:
//
//   N1 gv_fused   one pass over the row slab of A:
//                   t_r = A_r . v - U_r . c        (= (X' v)_r,  Alg. 4 lines 3-4 + 14)
//                   y  += t_r A_r^T                 (A^T X' v)
//                   w  += t_r U_r^T                 (U^T X' v)
//                 A and U rows are staged by 1-D TMA bulk copies (cp.async.bulk) into an S-stage
//                 shared-memory ring; each staged element is read from shared memory ONCE into
//                 registers and used for both the dot and the axpy, so A is read from HBM exactly
//                 once per iteration (the paper's Alg. 4 reads it twice).  The
//                 prologue builds this thread's slice of v = y_cur / ||y_cur|| in registers (the
//                 normalisation of P:122 is folded here).  EXTRACT=true runs the same pipeline for
//                 u = A v and ||u||^2.
//   N5 fin_iter   (fin_kernels.cuh) reductions, V correction, stop test, c_next, WHILE condition.
//
// N6 extraction: gv_fused<EXTRACT> then ext_finish (fin_kernels.cuh).
//
// Precision (reading R17): A, U and the copy of v fed to N1 are fp32; products are fp32
// FMAs inside a thread, every cross-thread / cross-CTA / cross-GPU sum is fp64, and the per-CTA y
// accumulators are flushed to fp64 every `run_rows` rows.  The master iterate (y, ||y||) is fp64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsvd {

constexpr int kMaxStages = 8;
constexpr int kFinThreads = 256;

struct LoopState {
    double ny;             // ||y_cur||: the current iterate is v = y_cur / ny
    double d;              // |v0 . v1| of the last iteration
    int32_t it;            // iterations completed in this component; y_cur = ybuf[it & 1]
    int32_t done;          // this component's loop has finished
    int32_t status;        // 0 ok, 1 not converged (MAX_ITER), 2 rank exhausted, -7 non-finite, -6 peer timeout
    int32_t stop;          // sticky: rank exhausted / non-finite -> every later kernel is a no-op
    uint32_t counter;      // arrivals of the last-block-done reductions (returns to 0 after use)
    uint32_t epoch;        // peer-collective epoch: identical on all ranks, monotone across runs
    uint32_t pub_counter;  // arrivals of publish_partials
    uint32_t xepoch;       // persistent kernel's peer exchange: passes exchanged so far (identical
                           // on all ranks, monotone across runs)
};

constexpr int kMaxRanks = 8;

// Persistent kernel's cross-rank exchange (N7, world > 1): every rank owns a receive area
// [2 parity][world src][G slices][SL elements]; an element is one double sent with the
// low-latency protocol (two 8-byte words, each half of the value + the pass stamp).  CTA b pushes
// its local column-slice sums (and the local w) into slice b of every rank.
struct PxView {
    ulonglong2 *rbuf[kMaxRanks];  // rank r's receive area (IPC-mapped; [rank] is local)
    const ulonglong2 *lbuf;       // this rank's receive area
    int world, rank, G;
    int per, SL;                  // slice width (columns), slice stride (per + w slots, elements)
};

// Peer view of the symmetric reduction buffers (multi-GPU, NVLink peer memory).
struct PeerView {
    double *buf[kMaxRanks];       // each rank's symmetric buffer (IPC-mapped); buf[rank] is local
    unsigned *flags;              // local flag array: flags[q] = last epoch published by rank q
    unsigned *rflags[kMaxRanks];  // &(rank r's flags)[my rank]
    int world, rank;
    int64_t slot_stride;          // doubles per slot; slot (epoch & 1)
    int64_t wofs, sofs;           // offsets of w and of ||u||^2 inside a slot
};

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).  One arrival word: CTA 0 adds
// 2^31 - (G - 1), every other CTA adds 1, so bit 31 flips exactly when the last CTA arrives and the
// low bits return to zero (no reset, no generation read: one atomic round trip + the poll).
__device__ __forceinline__ void grid_sync(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(bar, nb);
        while (((old ^ ld_acquire_gpu(bar)) & 0x80000000u) == 0u) {
        }
        __threadfence();
    }
    __syncthreads();
}

struct CompStat {  // per component, written by ext_finish
    double d;
    double sigma;
    int32_t it;
    int32_t status;
    int32_t valid;
    int32_t pad;
};

struct GvParams {
    const float *A;          // row slab base (row 0 of this launch)
    int64_t ld;              // leading dimension (floats), % 4 == 0
    int64_t rows;            // rows in this launch
    int32_t n;               // columns
    int32_t n4;              // ceil(n / 4): float4 per row
    const float *U;          // rows x ldu fp32 (row 0 aligned with A's row 0)
    int32_t ldu;             // % 4 == 0
    int32_t l;               // components already found (U columns used)
    const double *ybuf;      // ping-pong fp64 iterate buffers, [2][ystride]
    int64_t ystride;
    const LoopState *st;     // it, ny, done, stop
    const double *c;         // c = S (V^T v), length l
    double *ypart;           // [gridDim.x][ypart_ld] fp64 per-CTA partial of A^T t
    int64_t ypart_ld;
    double *wpart;           // [gridDim.x][wpart_ld] fp64 per-CTA partial of U^T t
    int32_t wpart_ld;
    int32_t stages;          // S
    int32_t stage_bytes;     // bytes per ring slot (A row + U row, 128-B aligned)
    int32_t row_bytes;       // n4 * 16
    int32_t u_bytes;         // round4(l) * 4 (0 if l == 0 or EXTRACT)
    int32_t run_rows;        // fp32 run length before flushing to fp64
    double *u_out;           // EXTRACT: fp64 (A v)_r, indexed by launch row
    double *sq_part;         // EXTRACT: [gridDim.x] fp64 sum of (A v)_r^2
    int32_t accumulate;      // 1: add into the partials of an earlier launch of the same pass
                             //    (out-of-memory streaming: resident prefix, then ring batches)
    int32_t reduce_mode;     // 0: per-CTA partials only (fin_iter<SRC_PARTS> sums them)
                             // 1: cooperative launch; after a grid barrier each CTA sums a column
                             //    slice of the partials into yw = [y | w] (fin_iter<SRC_YW>)
                             // 2: as 1, into this rank's symmetric slot, then raise the peer flags
    double *yw;              // reduce_mode 1 target
    int64_t wofs;
    unsigned *gbar;          // grid barrier state (2 words)
    PeerView pv;             // reduce_mode 2
    unsigned long long *trace;  // debug (TSVD_TRACE): per CTA %globaltimer at entry, first row,
                                // end of the row loop, exit
    int32_t dynamic;            // 1: CTAs claim chunk_rows rows at a time from work[0]
    int32_t chunk_rows;
    unsigned long long *work;   // [0] next unclaimed row, [1] CTAs finished (reset by the last)
    unsigned long long *tl;     // debug timeline: [0] iterations, [1] exit count, then 3 per iteration
    const float *vprev;         // TWO: previous component's v (fp32, n4*4 floats, zero padded)
    int32_t vp_bytes;           // TWO: shared memory reserved for vprev (0 otherwise)
    int32_t serpentine;         // 1: odd iterations walk each CTA's row range backwards, so the
                                // rows the previous pass read last (still in L2) are read first
    int32_t store_t;            // explicit-Gram extraction: also store t_r in u_out and sum t_r^2
};

// Column-slice reduction of the per-CTA partials at the end of N1 (reduce_mode 1/2).  CTA c owns
// columns [c*per, (c+1)*per); warp w sums partials b = w, w+NW, ... of 32 columns and the warp sums
// are added in warp order (fixed order).  Partials written by other CTAs are read with ld.cg.
__device__ __forceinline__ double warp_sum(double x);

template <int T>
__device__ __forceinline__ void reduce_tail(const GvParams &p) {
    constexpr int NW = T / 32;
    __shared__ double red2[NW][32];
    grid_sync(p.gbar);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    LoopState *st = const_cast<LoopState *>(p.st);
    const unsigned e = st->epoch;
    double *yout = p.reduce_mode == 1 ? p.yw : p.pv.buf[p.pv.rank] + (int64_t)(e & 1u) * p.pv.slot_stride;
    const int64_t wofs = p.reduce_mode == 1 ? p.wofs : p.pv.wofs;
    const int64_t per = ((p.n + G - 1) / G + 31) / 32 * 32;
    const int64_t j0 = (int64_t)blockIdx.x * per;
    const int64_t j1 = (j0 + per) < (int64_t)p.n ? (j0 + per) : (int64_t)p.n;
    for (int64_t c0 = j0; c0 < j1; c0 += 32) {
        const int64_t j = c0 + lane;
        double s = 0.0;
        if (j < j1)
            for (int b = warp; b < G; b += NW) s += __ldcg(p.ypart + (int64_t)b * p.ypart_ld + j);
        red2[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && j < j1) {
            double y = red2[0][lane];
#pragma unroll
            for (int q = 1; q < NW; ++q) y += red2[q][lane];
            yout[j] = y;
        }
        __syncthreads();
    }
    if (blockIdx.x == 0)
        for (int i = warp; i < p.l; i += NW) {
            double w = 0.0;
            for (int b = lane; b < G; b += 32) w += __ldcg(p.wpart + (int64_t)b * p.wpart_ld + i);
            w = warp_sum(w);
            if (lane == 0) yout[wofs + i] = w;
        }
    if (p.reduce_mode == 2) {  // publish: last CTA raises flag = epoch + 1 on every rank
        __threadfence_system();
        __syncthreads();
        if (tid == 0 && atomicAdd(&st->pub_counter, 1u) == (unsigned)G - 1) {
            st->pub_counter = 0;
            __threadfence_system();
            for (int r = 0; r < p.pv.world; ++r) st_release_sys(p.pv.rflags[r], e + 1u);
        }
    }
}

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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// ---- 2-CTA cluster helpers (row split for n > 16384): DSMEM exchange of the half dot products
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_remote_arrive(uint32_t addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
// asynchronous 8-byte store into the partner CTA's shared memory that completes 8 tx-bytes on the
// partner's mbarrier (DSMEM message passing: one hop, no separate release/arrive)
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(remote_addr),
                 "d"(v), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TSVD_CWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TSVD_CWAIT_%=;\n}" ::"r"(smem_u32(bar)),
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

// debug timeline record per iteration: N1 start (block 0), N1 end (last CTA), fin end, fin start
// (block 0), fin tail start (last block), first N1 CTA out
constexpr int kTl = 8;

// Programmatic dependent launch: a kernel launched with the PDL attribute may start while its
// predecessor in the stream is still running; griddep_wait() blocks until that predecessor has
// completed and its memory is visible (a no-op without the attribute).  griddep_launch() lets the
// successor launch early; the successor still waits for this grid's completion before it reads.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Sum of the NW per-warp partials of a row, the same in every lane and every warp: lane i reads
// partial i mod NW and a butterfly over NW lanes adds them (commutative pairings: bitwise identical
// in all lanes).  One shared load + log2(NW) shuffle steps per warp instead of NW loads + NW - 1 adds
// per thread (the row loop's fp64 reduction was its largest instruction cost).
template <int NW>
__device__ __forceinline__ double sum_warps(const double *part, int lane) {
    double v = part[lane & (NW - 1)];
#pragma unroll
    for (int o = NW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void set_cond(unsigned long long h, int use, unsigned v) {
#if CUDART_VERSION >= 12040
    if (use) cudaGraphSetConditional((cudaGraphConditionalHandle)h, v);
#endif
}

// ---------------------------------------------------------------- N1: fused Gram-vector pass
// Grid: one persistent CTA per (SM x CTAs/SM), each owning a contiguous row range.
// Block: T threads; thread `tid` owns float4 columns {k*T + tid : k < NV} of every row.
#ifndef TSVD_TWO_TMEM_F4
#define TSVD_TWO_TMEM_F4 4   // float4 of v_prev per tcgen05.ld in the two-vector pass (2 or 4; A/B)
#endif
// SPLIT = 2 (n > 4*T*NV, up to 32768): a 2-CTA cluster shares each row range, CTA rank q staging
// and owning the q-th half of every row; the two half dot products are exchanged through
// distributed shared memory (remote store + remote mbarrier arrive) and added in rank order,
// so both CTAs use the same t_r.  Rank 0 alone handles the U (deflation) columns.
template <int T, int NV, bool EXTRACT, int SPLIT, bool TWO>
__global__ void __launch_bounds__(T) gv_fused(const GvParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NW = T / 32;
    const LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    // (store_t: the explicit path's extraction pass runs after its component is done)
    if (st->stop || (!EXTRACT && st->done && !p.store_t)) return;
    if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 4 + 0] = globaltimer_ns();
    if (!EXTRACT && p.tl && blockIdx.x == 0 && threadIdx.x == 0) {  // debug timeline (TSVD_TIMELINE)
        const unsigned long long idx = atomicAdd(p.tl, 1ull) % 4096;
        p.tl[2 + kTl * idx] = globaltimer_ns();
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float4 *vps = reinterpret_cast<float4 *>(smem + (size_t)p.stages * p.stage_bytes);  // TWO: v_prev
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)p.stages * p.stage_bytes + p.vp_bytes);
    double *red = reinterpret_cast<double *>(bars + kMaxStages);  // [2][NR][NW]

    __shared__ int64_t slot_row[kMaxStages];  // row held by each ring slot (-1: no more rows)
    // SPLIT: the partner's half dot product of row j in buffer j % kXb, completion on xbar[j % kXb]
    // (the lag-one loop reads row j's value one row later, so the partner may already be sending
    // rows j + 1, j + 2, j + 3: four buffers)
    constexpr int kXb = 4;
    __shared__ double xch[kXb];
    __shared__ __align__(8) uint64_t xbar[kXb];
    const int crank = SPLIT == 2 ? (int)cluster_ctarank() : 0;
    const int part_id = blockIdx.x / SPLIT;
    const int nparts = gridDim.x / SPLIT;
    const int half4 = (p.n4 + SPLIT - 1) / SPLIT;    // float4 columns per CTA (row_bytes = half4*16)
    const int c4_0 = crank * half4;                  // first float4 column of this CTA
    const int my_n4 = (p.n4 - c4_0) < half4 ? (p.n4 - c4_0) : half4;
    const bool owner = crank == 0;                   // handles U rows, w, u_out, sq
    const int S = p.stages;
    // TWO: the U column p.l-1 ("fresh") is not stored yet: its entries are u_r = A_r . v_prev,
    // computed in this same pass (the extraction of component p.l-1), with c_fresh = v_prev . v
    // (sigma cancels: U_r,f sigma_f (V_f . v) = (A_r . v_prev)(v_prev . v)).
    const int l = (EXTRACT || !owner) ? 0 : (TWO ? p.l - 1 : p.l);  // staged U columns
    const double c_fresh = TWO ? p.c[p.l - 1] : 0.0;
    constexpr int NR = TWO ? 2 : 1;                  // dot products per row
    const uint32_t tx_bytes = (uint32_t)(my_n4 * 16 + (l > 0 ? p.u_bytes : 0));

    // Row schedule (producer thread only).  Dynamic: claim chunks of chunk_rows rows from a
    // per-launch counter, so SMs that get less HBM bandwidth simply take fewer rows.  Static:
    // contiguous range per CTA (per cluster when SPLIT = 2), bitwise-reproducible sums.
    const bool dyn = p.dynamic && SPLIT == 1;
    int64_t cur = dyn ? 0 : p.rows * part_id / nparts;
    int64_t cur_end = dyn ? 0 : p.rows * (part_id + 1) / nparts;
    // serpentine order (static split): the row range is walked backwards on odd iterations
    const int64_t mirror = (!dyn && p.serpentine && (st->it & 1)) ? cur + cur_end - 1 : -1;
    auto next_row = [&]() -> int64_t {
        if (cur >= cur_end) {
            if (!dyn) return -1;
            const unsigned long long base = atomicAdd(p.work, (unsigned long long)p.chunk_rows);
            if (base >= (unsigned long long)p.rows) return -1;
            cur = (int64_t)base;
            cur_end = cur + p.chunk_rows < p.rows ? cur + p.chunk_rows : p.rows;
        }
        const int64_t r = cur++;
        return mirror >= 0 ? mirror - r : r;
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        if (SPLIT == 2)
            for (int b = 0; b < kXb; ++b) mbar_init(&xbar[b], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (SPLIT == 2) cluster_sync_all();  // the partner's exchange barriers exist before any arrive
    const uint32_t peer_xch = SPLIT == 2 ? map_to_rank(smem_u32(&xch[0]), crank ^ 1) : 0;
    const uint32_t peer_xbar = SPLIT == 2 ? map_to_rank(smem_u32(&xbar[0]), crank ^ 1) : 0;
    auto feed = [&](int slot) {  // producer: next row into `slot`, or close the slot
        const int64_t row = next_row();
        slot_row[slot] = row;
        if (row >= 0) {
            unsigned char *dst = smem + (size_t)slot * p.stage_bytes;
            mbar_arrive_expect_tx(&bars[slot], tx_bytes);
            tma_load_1d(dst, p.A + row * p.ld + (int64_t)c4_0 * 4, (uint32_t)(my_n4 * 16), &bars[slot]);
            if (l > 0 && p.u_bytes > 0)
                tma_load_1d(dst + p.row_bytes, p.U + row * p.ldu, (uint32_t)p.u_bytes, &bars[slot]);
        } else {
            mbar_arrive(&bars[slot]);
        }
    };
    if (tid == 0)
        for (int s = 0; s < S; ++s) feed(s);

    // this thread's slice of v = y_cur / ||y_cur|| (fp64 master -> fp32), while the ring fills
    float4 vr[NV];
    {
        const double inv = 1.0 / st->ny;
        const double *ycur = p.ybuf + (int64_t)(st->it & 1) * p.ystride;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int j = 4 * (c4_0 + k * T + tid);
            if (k * T + tid >= my_n4) {
                vr[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else if (j + 3 < p.n) {
                const double2 lo = *reinterpret_cast<const double2 *>(ycur + j);
                const double2 hi = *reinterpret_cast<const double2 *>(ycur + j + 2);
                vr[k] = make_float4((float)(lo.x * inv), (float)(lo.y * inv), (float)(hi.x * inv), (float)(hi.y * inv));
            } else {
                vr[k].x = j + 0 < p.n ? (float)(ycur[j + 0] * inv) : 0.f;
                vr[k].y = j + 1 < p.n ? (float)(ycur[j + 1] * inv) : 0.f;
                vr[k].z = j + 2 < p.n ? (float)(ycur[j + 2] * inv) : 0.f;
                vr[k].w = 0.f;
            }
        }
    }
    double cval = 0.0;
    if (!EXTRACT && tid < l) cval = p.c[tid];
    const int tail = p.n & 3;  // valid lanes of the last float4 (0 = full)
    // TWO: v_prev is read with every row.  Small n: staged once in shared memory.  n > 8192 (T = 512):
    // shared memory is taken by the ring, so each thread keeps its 4*NV floats of v_prev in tensor
    // memory (TMEM, 128 columns: lane quarter = warp % 4, column group = warp / 4) and reloads
    // them per row with tcgen05.ld — TMEM is otherwise unused by this memory-bound kernel.
    constexpr bool kTmemV = TWO && SPLIT == 1 && ((T == 512 && NV == 8) || (T == 256 && NV == 16));
    constexpr int kCpt = 4 * NV;  // TMEM columns per thread (32 or 64; 128 allocated per CTA)
    __shared__ uint32_t tm_base;
    uint32_t tm_addr = 0;
    if (kTmemV) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tm_base))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tm_addr = tm_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(kCpt * (warp >> 2));
        const float4 *src = reinterpret_cast<const float4 *>(p.vprev);
#pragma unroll
        for (int c = 0; c < kCpt / 32; ++c) {  // 8 float4 (32 columns) per tcgen05.st
        uint32_t r[32];
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
            const int idx = (8 * c + k8) * T + tid;
            const float4 v = idx < p.n4 ? src[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
            r[4 * k8 + 0] = __float_as_uint(v.x);
            r[4 * k8 + 1] = __float_as_uint(v.y);
            r[4 * k8 + 2] = __float_as_uint(v.z);
            r[4 * k8 + 3] = __float_as_uint(v.w);
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(tm_addr + (uint32_t)(32 * c)),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
            "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
            "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
            "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
            : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else if (TWO) {  // stage v_prev (fp32, zero padded to n4 float4) once; read per row from smem
        const float4 *src = reinterpret_cast<const float4 *>(p.vprev);
        for (int idx = tid; idx < p.n4; idx += T) vps[idx] = src[idx];
        __syncthreads();
    }
    const int tf_thread = TWO ? ((p.l - 1) & (T - 1)) : 0;  // accumulates w of the fresh column
    double wfresh = 0.0;

    float4 ya[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) ya[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    double wacc = 0.0, sq = 0.0;
    bool flushed = p.accumulate != 0;
    double *yp = p.ypart + (int64_t)part_id * p.ypart_ld + (int64_t)c4_0 * 4;

    auto flush = [&]() {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = k * T + tid;
            if (idx < my_n4) {
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
    // SPLIT = 2 Gram pass, lag one row: row i's half dot product goes to the partner right after
    // its local reduction, and the axpy of row i - 1 — whose partner half has had a whole row's time
    // to arrive — is done next, re-reading row i - 1 from its ring slot (freed after that axpy).  The
    // DSMEM round trip (~0.3-0.5 us per row in the exchange-then-wait order) leaves the critical path;
    // the slot is held one row longer (prefetch depth S - 1 rows).  Same values, same order.
    if constexpr (SPLIT == 2 && !EXTRACT && !TWO) {
        double th_prev = 0.0;   // row i - 1: my half dot product (U term included on the owner)
        float ur_prev = 0.f;    // its U_r entry of this thread's deflation column (owner, tid < l)
        int64_t grow_prev = -1;
        auto finish = [&](int j) {  // axpy of row j (slot j % S), then free the slot
            const int sj = j % S, b = j % kXb;
            if (tid == 0) mbar_wait_cluster(&xbar[b], (uint32_t)((j / kXb) & 1));
            __syncthreads();  // the partner's half of row j is in xch[b]
            const double other = *reinterpret_cast<volatile double *>(&xch[b]);
            const double t = owner ? th_prev + other : other + th_prev;
            const float tf = (float)t;
            const float4 *row = reinterpret_cast<const float4 *>(smem + (size_t)sj * p.stage_bytes);
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int idx = k * T + tid;
                float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
                if (idx < my_n4) {
                    a = row[idx];
                    if (tail && c4_0 + idx == p.n4 - 1) {
                        if (tail < 2) a.y = 0.f;
                        if (tail < 3) a.z = 0.f;
                        a.w = 0.f;
                    }
                }
                ya[k].x = fmaf(tf, a.x, ya[k].x);
                ya[k].y = fmaf(tf, a.y, ya[k].y);
                ya[k].z = fmaf(tf, a.z, ya[k].z);
                ya[k].w = fmaf(tf, a.w, ya[k].w);
            }
            if (tid < l) wacc += t * (double)ur_prev;
            if (p.store_t && tid == 0 && owner) {
                p.u_out[grow_prev] = t;
                sq += t * t;
            }
            if (++run == p.run_rows) {
                flush();
                run = 0;
            }
            __syncthreads();  // every thread is done with slot sj and xch[b]
            if (tid == 0) {
                fence_proxy_async_smem();
                feed(sj);
            }
        };
        for (int i = 0;; ++i) {
            const int s = i % S;
            mbar_wait(&bars[s], (uint32_t)((i / S) & 1));
            if (i == 0 && p.trace && tid == 0) p.trace[blockIdx.x * 4 + 1] = globaltimer_ns();
            const int64_t grow = slot_row[s];  // same value in every thread: uniform exit
            if (grow < 0) {
                if (i > 0) finish(i - 1);
                break;
            }
            const float4 *row = reinterpret_cast<const float4 *>(smem + (size_t)s * p.stage_bytes);
            float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int idx = k * T + tid;
                float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
                if (idx < my_n4) {
                    a = row[idx];
                    if (tail && c4_0 + idx == p.n4 - 1) {
                        if (tail < 2) a.y = 0.f;
                        if (tail < 3) a.z = 0.f;
                        a.w = 0.f;
                    }
                }
                q0 = fmaf(a.x, vr[k].x, q0);
                q1 = fmaf(a.y, vr[k].y, q1);
                q2 = fmaf(a.z, vr[k].z, q2);
                q3 = fmaf(a.w, vr[k].w, q3);
            }
            double part = (double)((q0 + q1) + (q2 + q3));
            float ur = 0.f;
            if (tid < l) {
                ur = reinterpret_cast<const float *>(reinterpret_cast<const unsigned char *>(row) + p.row_bytes)[tid];
                part -= (double)ur * cval;
            }
            part = warp_sum(part);
            if (lane == 0) red[(i & 1) * NW + warp] = part;
            __syncthreads();  // row i's partial dots visible
            const double th = sum_warps<NW>(red + (i & 1) * NW, lane);
            if (tid == 0) {
                const int b = i % kXb;
                mbar_arrive_expect_tx(&xbar[b], (uint32_t)sizeof(double));
                st_async_f64(peer_xch + b * (uint32_t)sizeof(double), th, peer_xbar + b * (uint32_t)sizeof(uint64_t));
            }
            if (i > 0) finish(i - 1);
            th_prev = th;
            ur_prev = ur;
            grow_prev = grow;
        }
    } else
    for (int i = 0;; ++i) {
        const int s = i % S;
        mbar_wait(&bars[s], (uint32_t)((i / S) & 1));
        if (i == 0 && p.trace && tid == 0) p.trace[blockIdx.x * 4 + 1] = globaltimer_ns();
        const int64_t grow = slot_row[s];  // same value in every thread: uniform exit
        if (grow < 0) break;
        const unsigned char *slot = smem + (size_t)s * p.stage_bytes;
        const float4 *row = reinterpret_cast<const float4 *>(slot);

        float4 a[NV];
        float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;  // TWO: dot with v_prev
        // kTmemV: KV float4 of v_prev per tcgen05.ld (one wait::ld per KV float4 of the row): 4 for the
        // 256 x 16 variant (240 registers, no spill; two-vector pass 699.7 -> 681.2 us in ncu at C2),
        // 2 for 512 x 8 (128-register budget: 4 spills)
        constexpr int KV = (T == 256 && NV == 16) ? TSVD_TWO_TMEM_F4 : 2;
        uint32_t vt8[4 * KV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = k * T + tid;
            if (idx < my_n4) {
                a[k] = row[idx];
                if (tail && c4_0 + idx == p.n4 - 1) {  // columns >= n of the last float4 may be garbage
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
            if (kTmemV) {  // columns 4k..4k+3 of this thread's v_prev, KV float4 per TMEM load
                if ((k % KV) == 0) {
                    if constexpr (KV == 4) {
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
                            "%12, %13, %14, %15}, [%16];\n\t"
                            "tcgen05.wait::ld.sync.aligned;"
                            : "=r"(vt8[0]), "=r"(vt8[1]), "=r"(vt8[2]), "=r"(vt8[3]), "=r"(vt8[4]), "=r"(vt8[5]),
                              "=r"(vt8[6]), "=r"(vt8[7]), "=r"(vt8[8]), "=r"(vt8[9]), "=r"(vt8[10]), "=r"(vt8[11]),
                              "=r"(vt8[12]), "=r"(vt8[13]), "=r"(vt8[14]), "=r"(vt8[15])
                            : "r"(tm_addr + (uint32_t)(4 * k))
                            : "memory");
                    } else {
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
                            "tcgen05.wait::ld.sync.aligned;"
                            : "=r"(vt8[0]), "=r"(vt8[1]), "=r"(vt8[2]), "=r"(vt8[3]), "=r"(vt8[4]), "=r"(vt8[5]),
                              "=r"(vt8[6]), "=r"(vt8[7])
                            : "r"(tm_addr + (uint32_t)(4 * k))
                            : "memory");
                    }
                }
                const int o = 4 * (k % KV);
                p0 = fmaf(a[k].x, __uint_as_float(vt8[o + 0]), p0);
                p1 = fmaf(a[k].y, __uint_as_float(vt8[o + 1]), p1);
                p2 = fmaf(a[k].z, __uint_as_float(vt8[o + 2]), p2);
                p3 = fmaf(a[k].w, __uint_as_float(vt8[o + 3]), p3);
            } else if (TWO && idx < my_n4) {
                const float4 vp = vps[idx];
                p0 = fmaf(a[k].x, vp.x, p0);
                p1 = fmaf(a[k].y, vp.y, p1);
                p2 = fmaf(a[k].z, vp.z, p2);
                p3 = fmaf(a[k].w, vp.w, p3);
            }
        }
        double part = (double)((q0 + q1) + (q2 + q3));
        float ur = 0.f;
        if (!EXTRACT && tid < l) {
            ur = reinterpret_cast<const float *>(slot + p.row_bytes)[tid];
            part -= (double)ur * cval;  // - U_r . c  (deflation, never forming X')
        }
        part = warp_sum(part);
        if (lane == 0) red[((i & 1) * NR) * NW + warp] = part;
        if (TWO) {
            const double pu = warp_sum((double)((p0 + p1) + (p2 + p3)));
            if (lane == 0) red[((i & 1) * NR + 1) * NW + warp] = pu;
        }
        __syncthreads();  // (a) partial dots visible, (b) every thread is done reading slot s
        if (tid == 0) {
            fence_proxy_async_smem();
            feed(s);
        }
        double t = 0.0, u = 0.0;
        t = sum_warps<NW>(red + ((i & 1) * NR) * NW, lane);  // same value in every thread
        if (TWO) {
            u = sum_warps<NW>(red + ((i & 1) * NR + 1) * NW, lane);
            t -= u * c_fresh;  // - U_r,fresh sigma_f (V_f . v) = - u_r (v_prev . v)
            if (tid == 0) {
                p.u_out[grow] = u;
                sq += u * u;
            }
        }
        if (SPLIT == 2) {  // half dot products: send mine, wait for the partner's, add in rank order
            const int b = i % kXb;
            if (tid == 0) {
                mbar_arrive_expect_tx(&xbar[b], (uint32_t)sizeof(double));  // my arrival + 8 bytes due
                st_async_f64(peer_xch + b * (uint32_t)sizeof(double), t, peer_xbar + b * (uint32_t)sizeof(uint64_t));
                mbar_wait_cluster(&xbar[b], (uint32_t)((i / kXb) & 1));
            }
            __syncthreads();
            const double other = *reinterpret_cast<volatile double *>(&xch[b]);
            t = owner ? t + other : other + t;
        }

        if (EXTRACT) {
            if (tid == 0 && owner) {
                p.u_out[grow] = t;
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
            if (TWO && tid == tf_thread) wfresh += t * u;  // sigma_f U_f^T t = u^T t
            if (!TWO && p.store_t && tid == 0 && owner) {
                p.u_out[grow] = t;
                sq += t * t;
            }
            if (++run == p.run_rows) {
                flush();
                run = 0;
            }
        }
    }
    if (p.trace && tid == 0) p.trace[blockIdx.x * 4 + 2] = globaltimer_ns();
    if (EXTRACT) {
        if (tid == 0 && owner) p.sq_part[part_id] = p.accumulate ? p.sq_part[part_id] + sq : sq;
    } else {
        flush();
        if (tid < l) {
            double *wp = p.wpart + (int64_t)part_id * p.wpart_ld + tid;
            *wp = p.accumulate ? *wp + wacc : wacc;
        }
        if (!TWO && p.store_t && tid == 0 && owner) p.sq_part[part_id] = p.accumulate ? p.sq_part[part_id] + sq : sq;
        if (TWO) {
            if (tid == tf_thread) {
                double *wp = p.wpart + (int64_t)part_id * p.wpart_ld + (p.l - 1);
                *wp = p.accumulate ? *wp + wfresh : wfresh;
            }
            if (tid == 0) p.sq_part[part_id] = p.accumulate ? p.sq_part[part_id] + sq : sq;
        }
        if (SPLIT == 1 && p.reduce_mode) reduce_tail<T>(p);
    }
    if (SPLIT == 2) cluster_sync_all();  // no CTA leaves while its partner may still address it
    if (kTmemV) {  // every warp is done with its TMEM columns
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm_base) : "memory");
    }
    if (p.trace) {
        __syncthreads();
        if (tid == 0) p.trace[blockIdx.x * 4 + 3] = globaltimer_ns();
    }
    if (!EXTRACT && p.tl && tid == 0) {
        __threadfence();
        const unsigned long long now = globaltimer_ns();
        unsigned long long *rec = p.tl + 2 + kTl * ((p.tl[0] - 1) % 4096);
        const unsigned long long old = atomicAdd(p.tl + 1, 1ull);
        if (old == 0) rec[5] = now;  // first CTA out
        if (old == gridDim.x - 1) {
            p.tl[1] = 0;
            rec[1] = now;
        }
    }
    if (p.dynamic && tid == 0) {  // last CTA out resets the row counter for the next launch
        __threadfence();
        if (atomicAdd(p.work + 1, 1ull) == gridDim.x - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
            __threadfence();
        }
    }
}

}  // namespace tsvd
