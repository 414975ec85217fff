// tsvd.cu — libtsvd.so: the C ABI of include/tsvd.h and the Alg. 1 / Alg. 2 driver.
//
// The driver is host code that only plans, allocates and launches; every arithmetic step of the
// power iteration (Gram-vector product, reductions, normalisation, stop test, extraction) runs
// in the kernels of gram_kernels.cuh / fin_kernels.cuh.  A whole tsvd_run (all k components:
// init, power-iteration WHILE loop, extraction) is ONE CUDA graph with one conditional WHILE node
// per component, so the host synchronises once per run.  One process per GPU; multi-GPU = row
// partition with one all-reduce of [y_g | w_g] per iteration (merges Alg. 4 lines 6,
// 8, 16), done inside the finalize kernel over NVLink peer memory (default) or by NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tsvd.h"
#include "fin_kernels.cuh"
#include "gram_kernels.cuh"
#include "sparse_kernels.cuh"
#include "persist_kernels.cuh"
#include "explicit_kernels.cuh"
#include "gram_tc.cuh"
#include <cublas_v2.h>

using namespace tsvd;

namespace {

constexpr int kMaxThreadsPerCta = 512;
constexpr int kRingTargetBytes = 192 * 1024;  // bytes in flight per SM (Little's law)
constexpr int kSmemBudget = 220 * 1024;       // per SM, leaves room for barriers/scratch
constexpr int kMaxK = 4096;                   // fin_iter keeps 2k+2 doubles in shared memory

enum Coll { COLL_NONE = 0, COLL_PEER = 1, COLL_NCCL = 2 };

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

using GvFn = void (*)(const GvParams);

template <int T, bool EX, bool TWO>
GvFn pick_nv(int nv) {
    switch (nv) {
    case 1: return gv_fused<T, 1, EX, 1, TWO>;
    case 2: return gv_fused<T, 2, EX, 1, TWO>;
    case 4: return gv_fused<T, 4, EX, 1, TWO>;
    case 8: return gv_fused<T, 8, EX, 1, TWO>;
    case 16:
        if constexpr (T == 256 && TWO && !EX) return gv_fused<256, 16, false, 1, true>;  // n = 16384, 8 warps
        return nullptr;
    default: return nullptr;
    }
}
// EX: extraction (dot only); TWO: extraction of the previous component fused into the first
// iteration of the next (split-free kernels only)
template <bool EX, bool TWO = false>
GvFn pick_gv(int T, int nv, int split = 1) {
    if (split == 2) return (!TWO && T == 512 && nv == 8) ? gv_fused<512, 8, EX, 2, false> : nullptr;
    switch (T) {
    case 32: return pick_nv<32, EX, TWO>(nv);
    case 64: return pick_nv<64, EX, TWO>(nv);
    case 128: return pick_nv<128, EX, TWO>(nv);
    case 256: return pick_nv<256, EX, TWO>(nv);
    case 512: return pick_nv<512, EX, TWO>(nv);
    default: return nullptr;
    }
}


using GbFn = void (*)(const GbParams);
template <int T>
GbFn pick_gb_nv(int nv) {
    return nv == 1 ? gb_persist<T, 1> : nv == 2 ? gb_persist<T, 2> : nv == 4 ? gb_persist<T, 4> : gb_persist<T, 8>;
}
inline GbFn pick_gb(int T, int nv) {
    switch (T) {
    case 32: return pick_gb_nv<32>(nv);
    case 64: return pick_gb_nv<64>(nv);
    case 128: return pick_gb_nv<128>(nv);
    case 256: return pick_gb_nv<256>(nv);
    default: return pick_gb_nv<512>(nv);
    }
}

using PsFn = void (*)(const PsParams);

template <int T>
PsFn pick_ps_nv(int nv) {
    switch (nv) {
    case 1: return gv_persist<T, 1>;
    case 2: return gv_persist<T, 2>;
    case 4: return gv_persist<T, 4>;
    case 8: return gv_persist<T, 8>;
    default: return nullptr;
    }
}
PsFn pick_ps(int T, int nv, bool full = false) {
    if (T == 256 && nv == 16) return full ? gv_persist<256, 16, true> : gv_persist<256, 16>;  // n = 16384, 8 warps
    if (full && T == 512 && nv == 8) return gv_persist<512, 8, true>;  // n = 16384
    if (full && T == 512 && nv == 4) return gv_persist<512, 4, true>;  // n = 8192
    switch (T) {
    case 32: return pick_ps_nv<32>(nv);
    case 64: return pick_ps_nv<64>(nv);
    case 128: return pick_ps_nv<128>(nv);
    case 256: return pick_ps_nv<256>(nv);
    case 512: return pick_ps_nv<512>(nv);
    default: return nullptr;
    }
}

// In-process rank groups (tsvd_get_inproc_id): W handles of ONE process, driven from W host threads,
// typically on one GPU with TSVD_OPT_SM_LIMIT splitting its SMs.  The setup-time agreements (min of
// an int, every rank's exchange-buffer pointer) go through this host rendezvous instead of NCCL, and
// the peer buffers are the other handles' device pointers (no IPC); the data path — the persistent
// kernel's stamped-word exchange and the per-iteration peer all-reduce — is the multi-GPU code as is.
struct InprocGroup {
    std::mutex mu;
    std::condition_variable cv;
    int world = 0, arrived = 0;
    unsigned long long gen = 0;
    std::vector<long long> v;
    std::vector<void *> p;
    long long rmin = 0;
    std::vector<void *> rp;
};
std::mutex g_grp_mu;
std::map<std::string, std::weak_ptr<InprocGroup>> g_grps;
constexpr char kInprocMagic[16] = "TSVD-INPROC-ID";  // first 16 bytes of an in-process group id

}  // namespace

struct tsvd_s {
    // problem
    int64_t m = 0, n = 0;
    int32_t k = 0, kpad = 4;
    double eps = 1e-6;
    // device / comm
    int dev = 0, sms = 148;
    cudaStream_t stream = nullptr, body_stream = nullptr;
    int32_t rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    std::shared_ptr<InprocGroup> grp;       // in-process ranks (instead of comm)
    void *ar_tmp = nullptr;                 // in-process all-reduce scratch
    size_t ar_bytes = 0;
    int sm_limit = 0;                       // TSVD_OPT_SM_LIMIT (0 = every SM of the device)
    int coll = COLL_NONE;
    int coll_opt = 0;
    double *sym = nullptr;                  // this rank's symmetric buffer (peer path)
    void *peer_map[kMaxRanks] = {};         // IPC-opened peer buffers
    void *px_map[kMaxRanks] = {};           // IPC-opened peer receive areas of the persistent kernel
    char *px_mem = nullptr;                 // this rank's receive area + flags (N7, world > 1)
    PxView px{};
    bool px_ok = false;
    PeerView pv{};
    std::string peer_error;
    // options
    int max_iter = 10000, fixed_T = 0, use_graph = 1, timing = 0, run_rows = 1024, cps_opt = 0, unroll = 2;
    uint64_t seed = 0;
    // input
    int64_t row_begin = 0, row_end = 0, m_g = 0;
    const float *A_user = nullptr;
    int64_t ld_user = 0;
    tsvd_mem mem = TSVD_MEM_DEVICE;
    bool have_A = false;
    float *A_own = nullptr;
    int64_t ld_own = 0;
    const float *A_use = nullptr;
    int64_t ld_use = 0;
    std::vector<double> V0;
    bool have_V0 = false;
    int64_t v0_version = 1, v0_uploaded = 0;
    // out-of-memory degree 1 (host input): resident prefix [0, m_res) + streamed batches
    // wide input (m < n): the handle runs the tall problem on A^T; U and V swap roles at the
    // boundary.  The user's buffer is A^T row-major in place when it is column-major (the CSVD column
    // partition across ranks: a rank's column slab of A is a row slab of A^T); a row-major wide A
    // (or a column-major tall one) is transposed once into a device copy (tcopy, single GPU)
    bool wide = false, tcopy = false;
    tsvd_layout layout = TSVD_ROW_MAJOR;
    int64_t m_user = 0, n_user = 0;
    float *At = nullptr;
    int placement = 0, qdepth = 3;
    int64_t work_bytes = 0;  // device workspace allocated by ensure_alloc (report: peak device bytes)
    int64_t resident_cap = -1, batch_rows_opt = 0;
    int64_t m_res = 0, batch_rows = 0, own_rows = 0;
    bool streaming = false, host_registered = false;
    std::vector<float *> ring;
    std::vector<cudaEvent_t> ev_full, ev_free;
    cudaStream_t copy_stream = nullptr;
    int64_t streamed_bytes = 0, streamed_batches = 0;
    double stream_pass_ms = 0.0;
    // sparse CSR slab: the input arrays (borrowed device arrays, or an owned copy of host
    // arrays, freed once the blocked views replace them) and the two blocked views built once on
    // the device (N4/N4b): spc = the CSR by column block (N2), spr = the CSC by row block (N3)
    bool sparse = false, csr_owned = false;
    int64_t nnz_g = 0;
    int64_t *row_ptr_d = nullptr;
    int32_t *col_d = nullptr;
    float *val_d = nullptr;
    SpView spc{}, spr{};
    std::vector<void *> sp_mem;  // device arrays owned by the blocked views
    int64_t sp_bytes = 0;        // their size (report)
    double csc_build_ms = 0.0;
    // in-kernel column-slice reduction of the N1 partials (cooperative launch), option 13
    int fused_opt = 0;
    unsigned *gbar = nullptr;
    // dynamic row scheduling in N1 (option 14 DETERMINISTIC = 1 switches to a static split)
    int dynamic_opt = 0;  // measured: the static split is faster on the dense C2 pass
    unsigned long long *work = nullptr;
    unsigned long long *tl_d = nullptr;  // debug: TSVD_TIMELINE=<file> (N1 start/end, fin end per iteration)
    // debug: TSVD_TRACE=<file> appends per-CTA N1 timestamps of host-loop iterations
    unsigned long long *trace_d = nullptr;
    FILE *trace_f = nullptr;
    int64_t trace_launch = 0;
    // factors (device)
    float *U32 = nullptr;   // m_g x kpad
    double *V64 = nullptr;  // n x k (TSVD_OPT_V_PLACEMENT = 1: the device alias of mapped pinned host memory)
    int v_host = 0;         // TSVD_OPT_V_PLACEMENT: the co-factor V and the initial samples V0 on the host
    double *V64_h = nullptr, *V0d_h = nullptr;  // their host allocations (v_host)
    double *S64 = nullptr;  // k
    int32_t l_found = 0;
    // vectors / workspaces (device)
    double *ybuf = nullptr, *yw = nullptr, *V0d = nullptr, *c64 = nullptr, *ypart = nullptr, *wpart = nullptr;
    double *part = nullptr, *u64 = nullptr, *sq_part = nullptr, *sig2 = nullptr;
    float *y32 = nullptr, *t32 = nullptr;  // sparse: fp32 copies of y_cur and t for the gathers
    // sparse index blocking (L2-sized blocks of the gathered vectors): kc column blocks for N2,
    // kr row blocks for N3
    int sp_kc = 1, sp_kr = 1;
    int64_t sp_block_opt = 0;  // TSVD_OPT_SPARSE_BLOCK: block width in elements (0 = auto)
    int sp_chunks = 4;         // world > 1: N3's last block in column chunks, each all-reduced at once
    int grid_nl = 0;           // grid of the carry-only sparse launches (not the last index block)
    double *acc_r = nullptr, *acc_c = nullptr;    // carried sums (ping-pong pairs: [2][segs])
    cudaStream_t sp_comm_stream = nullptr;
    std::vector<cudaEvent_t> sp_ev;
    // sparse out of memory (degree 1, PLACEMENT = 2 with host input): both views' entry arrays in
    // pinned host memory, each block copied into a q_s-slot device ring before its launch
    bool sp_stream = false;
    int32_t *sp_hidx[2] = {}; float *sp_hval[2] = {};
    std::vector<int64_t> sp_hbase[2];
    std::vector<void *> sp_ring;
    std::vector<cudaEvent_t> sp_full, sp_free;
    int64_t sp_slot_entries = 0;
    int64_t sp_launch = 0;
    LoopState *st = nullptr;
    CompStat *stats = nullptr;
    LoopState *st_host = nullptr;      // pinned
    ulonglong2 *pub = nullptr;         // persistent kernel: stamped slice scalars [grid][part_ld]
    unsigned long long *puby = nullptr;  // persistent kernel: stamped fp32 y words [round4(n)]
    CompStat *stats_host = nullptr;    // pinned
    double *vec_host = nullptr;        // pinned staging (n doubles)
    int64_t ystride = 0, wofs = 0, ypart_ld = 0;
    int fin_blocks = 0, part_ld = 0;
    bool allocated = false;
    // plan
    int T = 0, NV = 0, S = 0, grid = 0, cps = 0, stage_bytes = 0, row_bytes = 0;
    int split = 1, parts = 0;  // CTAs per row range (2-CTA cluster for n > 16384); partial slots
    // fused extraction (option 16): N1<TWO> = first iteration of component l + extraction of l-1
    int fuse_ext_opt = 1, S_two = 0, vp_bytes = 0, T_two = 0;
    size_t smem_two = 0;
    GvFn gv_two = nullptr;
    float *vprev32 = nullptr;
    bool fused_ext_used = false;
    int carveout_opt = 1;
    int pdl_opt = 1;       // TSVD_OPT_PDL
    int serp_opt = 1;      // TSVD_OPT_ROW_ORDER
    int persist_opt = 1;   // TSVD_OPT_PERSISTENT
    // explicit-Gram path (TSVD_OPT_METHOD = 1, NEXT#1): B0 = A^T A, P = A^T U, Q = U^T U
    int method = 0;
    GbFn gb = nullptr;
    int S_gb = 0;
    size_t smem_gb = 0;
    float *B0 = nullptr, *Pm = nullptr, *g_hi = nullptr, *g_lo = nullptr;  // Gram, A^T U, TF32 split of A
    double *Qm = nullptr, *gpart = nullptr, *zero64 = nullptr;
    int64_t ldb0 = 0;
    bool B0_ok = false;
    int pq_l = 0;          // components whose P / Q columns are valid
    double gram_ms = 0.0;  // B0 build time of the last build
    int gram_blocks = 0;   // n_b of the symmetric task schedule of the last build (tcgen05: tiles computed)
    int2 *gram_tiles = nullptr;  // tcgen05 Gram: the symmetric tile list
    int gram_pair = 0;           // ... of kernel variant 1 (single CTA), 2 (pair), 3 (pair, A in TMEM)
    int gram_ntiles = 0;
    int64_t gram_n = -1;
    cublasHandle_t cublas = nullptr;
    PsFn gv_ps = nullptr;  // N7: one persistent cooperative kernel per component (null: unsupported)
    int S_ps = 0;
    size_t smem_ps = 0;
    int64_t vcache_doubles = 0;  // shared-memory V slice cache of the persistent kernel (0: none)
    int grid_gb = 0;  // explicit-Gram iteration grid (from n, identical on every rank)
    int T_ps = 0, NV_ps = 0;  // persistent kernel's CTA width (may differ from the N1 kernels')
    char *gx_mem = nullptr;             // explicit Gram, world > 1: [y area 2n | sums area] (IPC)
    void *gx_map[kMaxRanks] = {};
    ulonglong2 *gx_y[kMaxRanks] = {}, *gx_s[kMaxRanks] = {};
    bool gx_ok = false;
    double ps_ms = 0.0;    // TIMING: event time of the persistent launches, and the passes they ran
    int64_t ps_passes = 0, ps_launches = 0;  // debug knob TSVD_CARVEOUT=0: leave the driver's per-kernel L1/shared split
    size_t smem = 0;
    GvFn gv = nullptr, gv_ex = nullptr;
    // run graph (cached by starting component)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int graph_l0 = -1;
    std::string graph_error;
    // results / report
    std::vector<int32_t> iters;
    std::vector<double> dots;
    int32_t k_found = 0;
    double n1_ms = 0.0, run_ms = 0.0, h2d_ms = 0.0;
    int64_t n1_launches = 0, total_iters = 0, launches = 0;
    std::string loop_mode = "none";
    std::string err;

    tsvd_status fail(tsvd_status s, const char *fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return s;
    }
};

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) return h->fail(TSVD_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)
#define NK(call)                                                                                    \
    do {                                                                                            \
        if (h->grp) return h->fail(TSVD_ERR_UNSUPPORTED, "%s: no NCCL communicator (in-process ranks "       \
                                   "run the peer collective only)", #call);                        \
        ncclResult_t r_ = (call);                                                                   \
        if (r_ != ncclSuccess) return h->fail(TSVD_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)
#define TRY(expr)                        \
    do {                                 \
        tsvd_status s_ = (expr);         \
        if (s_ < 0) return s_;           \
    } while (0)

static thread_local std::string g_err;

// N1 reduces its own partials (grid barrier + column slices) unless the pass is split into
// several launches (streaming) or the input is sparse (N3 writes y directly).
static bool fused_reduce(tsvd_t h) { return h->fused_opt && !h->sparse && !h->streaming && h->split == 1; }

static int fin_src(tsvd_t h) {
    if (h->sparse) return SRC_YW;  // N3 writes y straight into yw (then NCCL if world > 1)
    if (h->coll == COLL_PEER) return SRC_PEER;
    if (h->coll == COLL_NCCL) return SRC_YW;
    return fused_reduce(h) ? SRC_YW : SRC_PARTS;
}

// Every kernel of the loop asks for the same L1/shared split (maximum shared), so consecutive
// launches never wait for an SM to drain and re-partition its L1 (measured: the gap between the
// finalize kernel and the next fused pass).
template <class F>
static cudaError_t max_carveout(F *fn) {
    return cudaFuncSetAttribute((const void *)fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared);
}

static tsvd_status set_fin_attrs(tsvd_t h) {
    const int fin_dyn = (2 * h->k + 2 + std::max(0, h->k - kVtReg) + kFinThreads) * (int)sizeof(double);
    CK(cudaFuncSetAttribute(fin_iter<SRC_PARTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, fin_dyn));
    CK(cudaFuncSetAttribute(fin_iter<SRC_YW>, cudaFuncAttributeMaxDynamicSharedMemorySize, fin_dyn));
    CK(cudaFuncSetAttribute(fin_iter<SRC_PEER>, cudaFuncAttributeMaxDynamicSharedMemorySize, fin_dyn));
    if (h->carveout_opt) {
        CK(max_carveout(fin_iter<SRC_PARTS>));
        CK(max_carveout(fin_iter<SRC_YW>));
        CK(max_carveout(fin_iter<SRC_PEER>));
        CK(max_carveout(publish));
        CK(max_carveout(reduce_partials));
        CK(max_carveout(ext_reduce));
        CK(max_carveout(ext_finish<SRC_PARTS>));
        CK(max_carveout(ext_finish<SRC_YW>));
        CK(max_carveout(ext_finish<SRC_PEER>));
        // (the sparse kernels keep the driver's L1 / shared split: a thread's entry loads of a batch
        // hit the L1 lines its warp's neighbours brought in)
    }
    return TSVD_OK;
}

// ------------------------------------------------------------------------------------ planning
static tsvd_status plan(tsvd_t h) {
    const int64_t n = h->n;
    if (h->sparse) {  // N2/N3: one thread per segment, a grid of resident 256-thread blocks
        // l <= k deflation columns (tsvd_gram_apply may run with l = k injected factors)
        if (h->k > kSpMaxL)
            return h->fail(TSVD_ERR_UNSUPPORTED, "sparse path: k = %d > %d (per-thread w partials)", h->k, kSpMaxL);
        const int dyn = (int)((int64_t)std::max(h->k, 1) * (kSpThreads + 1) * sizeof(double));
        int occ = 0, occ_nl = 0;
        CK(cudaFuncSetAttribute(sp_pass<MODE_T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
        // one resident wave each: the last-block kernels (outputs, per-block w / u^2 partials: `parts`
        // rows) and the leaner carry-only kernels of the other index blocks
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sp_pass<MODE_T, true>, kSpThreads, dyn));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_nl, sp_pass<MODE_Y, false>, kSpThreads, 0));
        h->grid = h->sms * std::max(1, occ);
        h->grid_nl = h->sms * std::max(1, occ_nl);
        h->parts = h->grid;
        h->T = kSpThreads;
        return set_fin_attrs(h);
    }
    // thread tid owns deflation column tid of a staged U row (and its w / V^T y lane): T >= k
    if (h->k > kMaxThreadsPerCta)
        return h->fail(TSVD_ERR_UNSUPPORTED, "dense path: k = %d > %d components", h->k, kMaxThreadsPerCta);
    int T = 32;
    while (((int64_t)4 * T * 8 < n || T < h->k) && T < kMaxThreadsPerCta) T *= 2;
    int split = 1;
    if ((int64_t)4 * T * 8 < n) split = 2;  // 2-CTA cluster: each CTA stages and owns half a row
    if ((int64_t)4 * T * 8 * split < n)
        return h->fail(TSVD_ERR_UNSUPPORTED, "n = %lld > 32768 is not supported by the dense kernel", (long long)n);
    int NV = 1;
    while ((int64_t)4 * T * NV * split < n) NV *= 2;
    const int n4 = (int)((n + 3) / 4);
    h->split = split;
    h->row_bytes = ((n4 + split - 1) / split) * 16;
    h->stage_bytes = (int)round_up(h->row_bytes + h->kpad * 4, 128);
    int cps = h->cps_opt > 0 ? h->cps_opt : std::max(1, 512 / T);
    int S = (int)std::min<int64_t>(kMaxStages, std::max<int64_t>(2, (kRingTargetBytes + (int64_t)h->stage_bytes * cps - 1) /
                                                                     ((int64_t)h->stage_bytes * cps)));
    while ((int64_t)S * h->stage_bytes * cps > kSmemBudget && S > 2) --S;
    while ((int64_t)S * h->stage_bytes * cps > kSmemBudget && cps > 1) --cps;
    if ((int64_t)S * h->stage_bytes > kSmemBudget)
        return h->fail(TSVD_ERR_UNSUPPORTED, "k = %d too large for the shared-memory ring at n = %lld", h->k,
                       (long long)n);
    h->T = T;
    h->NV = NV;
    h->S = S;
    h->smem = (size_t)S * h->stage_bytes + kMaxStages * sizeof(uint64_t) + 2 * (T / 32) * sizeof(double);
    h->gv = pick_gv<false>(T, NV, split);
    h->gv_ex = pick_gv<true>(T, NV, split);
    CK(cudaFuncSetAttribute(h->gv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem));
    CK(cudaFuncSetAttribute(h->gv_ex, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem));
    if (h->carveout_opt) {
        CK(max_carveout(h->gv));
        CK(max_carveout(h->gv_ex));
    }
    if (split == 2) {
        CK(cudaFuncSetAttribute(h->gv, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
        CK(cudaFuncSetAttribute(h->gv_ex, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    }
    TRY(set_fin_attrs(h));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->gv, T, h->smem));
    if (occ < 1) return h->fail(TSVD_ERR_UNSUPPORTED, "fused kernel does not fit on an SM (T=%d smem=%zu)", T, h->smem);
    h->cps = std::min(cps, occ);
    // one row range per CTA (per 2-CTA cluster when split): at most one range per row
    // at least min_rows = 8 rows per CTA (A/B knob TSVD_MIN_ROWS_PER_CTA): a small matrix (C1, in
    // L2) is latency-bound by the per-pass reduction over the CTAs' partials, not by its rows.  C1
    // (512 x 256, k = 8): 66.6 us per iteration with one row per CTA (512 CTAs), 25.4 / 24.5 / 25.1 /
    // 32.6 us with 4 / 8 / 16 / 32 rows; large inputs are unaffected (m_g / 8 >> SMs)
    int64_t min_rows = 8;
    if (const char *e = getenv("TSVD_MIN_ROWS_PER_CTA")) min_rows = std::max<int64_t>(1, atoll(e));
    h->grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->sms * h->cps / split, (h->m_g + min_rows - 1) / min_rows)) * split;
    h->parts = h->grid / split;
    // fused-extraction variant: v_prev staged in shared memory, so fewer ring stages
    h->gv_two = nullptr;
    if (split == 1) {
        // n > 8192: v_prev lives in tensor memory, the ring keeps all its stages.  n = 16384: 256
        // threads x 16 float4 columns (as the persistent kernel; TSVD_TWO_T512 keeps 512 x 8)
        int Tt = T, NVt = NV;
        if (T == 512 && NV == 8 && !getenv("TSVD_TWO_T512")) {
            Tt = 256;
            NVt = 16;
        }
        h->T_two = Tt;
        h->vp_bytes = (T == 512 && NV == 8) ? 0 : (int)round_up((int64_t)n4 * 16, 128);
        const int64_t fixed = h->vp_bytes + kMaxStages * sizeof(uint64_t) + 4 * (Tt / 32) * sizeof(double) + 1024;
        int S2 = (int)std::min<int64_t>(S, (kSmemBudget / h->cps - fixed) / h->stage_bytes);
        if (S2 >= 2) {
            h->S_two = S2;
            h->smem_two = (size_t)S2 * h->stage_bytes + h->vp_bytes + kMaxStages * sizeof(uint64_t) +
                          4 * (Tt / 32) * sizeof(double);
            h->gv_two = pick_gv<false, true>(Tt, NVt);
            CK(cudaFuncSetAttribute(h->gv_two, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem_two));
            if (h->carveout_opt) CK(max_carveout(h->gv_two));
        }
    }
    // persistent per-component kernel: same ring, plus the reduction scratch; every CTA of the grid
    // must be co-resident (cooperative launch), and (V^T y)_i is owned by thread i (k <= T + 1)
    h->gv_ps = nullptr;
    // n = 16384: 8 warps x 16 float4 columns per thread (255 registers) instead of the N1 kernels'
    // 16 x 8 — half the per-row warp reductions (1 GPU 144.9 -> 143.9 ms, 4 GPUs 39.47 -> 39.27 ms,
    // interleaved A/B); TSVD_PS_T512 keeps 16 warps
    int Tp = T, NVp = NV;
    if (T == 512 && NV == 8 && !getenv("TSVD_PS_T512")) {
        Tp = 256;
        NVp = 16;
    }
    h->T_ps = Tp;
    h->NV_ps = NVp;
    if (split == 1 && h->k <= 32 * kPsLanesV + 1 && h->k <= Tp) {
        const int64_t extra = kMaxStages * 8 + (int64_t)(2 * (Tp / 32) + 4 * h->kpad + 2 + kPsGred(Tp) + 128) * 8;
        int Sp = S;
        while (Sp > 2 && ((int64_t)Sp * h->stage_bytes + extra) * h->cps > kSmemBudget) --Sp;
        PsFn fn = pick_ps(Tp, NVp, n == (int64_t)4 * NVp * Tp && !getenv("TSVD_NO_FULL"));
        if (fn && ((int64_t)Sp * h->stage_bytes + extra) * h->cps <= kSmemBudget) {
            // V[:, :k] of the CTA's column slice (k (per + 1) doubles) in the space left, if any:
            // the per-pass V correction and V^T y read it from shared memory instead of L2
            const int64_t per1 = ((n + h->grid - 1) / h->grid + 31) / 32 * 32;
            const int64_t vneed = (int64_t)h->k * (per1 + 1);
            h->vcache_doubles = ((int64_t)Sp * h->stage_bytes + extra + 8 * vneed) * h->cps <= kSmemBudget ? vneed : 0;
            const size_t sm = (size_t)Sp * h->stage_bytes + (size_t)extra + 8 * (size_t)h->vcache_doubles;
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            if (h->carveout_opt) CK(max_carveout(fn));
            int occ_ps = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_ps, fn, Tp, sm));
            if (occ_ps * h->sms >= h->grid) {
                h->gv_ps = fn;
                h->S_ps = Sp;
                h->smem_ps = sm;
            }
        }
    }
    // explicit-Gram iteration kernel: the same ring over rows of B0 (n x n)
    h->gb = nullptr;
    if (split == 1) {
        const int64_t extra = kMaxStages * 8 + (int64_t)(2 * (T / 32) + 4 * h->kpad + 2) * 8;
        int Sg = S;
        while (Sg > 2 && ((int64_t)Sg * h->stage_bytes + extra) * h->cps > kSmemBudget) --Sg;
        GbFn fn = pick_gb(T, NV);
        const size_t sm = (size_t)Sg * h->stage_bytes + (size_t)extra;
        if (((int64_t)Sg * h->stage_bytes + extra) * h->cps <= kSmemBudget) {
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T, sm));
            // grid from n and the device only (not from this rank's rows): with a row-partitioned A
            // every rank iterates on the same B0 with the same grid, so the results agree bit for bit
            const int64_t gg = std::min<int64_t>((int64_t)h->sms * std::min(h->cps, occ), h->n);
            if (occ > 0 && gg >= 1) {
                h->gb = fn;
                h->S_gb = Sg;
                h->smem_gb = sm;
                h->grid_gb = (int)gg;
            }
        }
    }
    return TSVD_OK;
}

// Kernel launch with programmatic dependent launch (PDL) when enabled: the kernel may be scheduled
// while its predecessor drains (every kernel of the loop calls griddep_wait() before it reads
// anything), which hides the launch latency between the fused pass and the finalize kernel.
// cluster > 1: thread-block cluster of that many CTAs (the split kernel).
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(tsvd_t h, void (*fn)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                            int cluster, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    int na = 0;
    // PDL lets a successor's CTAs become resident while this kernel runs: with an SM budget shared
    // by several handles (in-process ranks) that would take SMs another rank's cooperative grid
    // needs, so it is off under TSVD_OPT_SM_LIMIT
    if (h->pdl_opt && !h->sm_limit) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

// the fused pass: one CTA per row range, or a 2-CTA cluster per row range (split)
static cudaError_t launch_n1(tsvd_t h, GvFn fn, const GvParams &p, cudaStream_t s) {
    return launch_k(h, fn, h->grid, h->T, h->smem, s, h->split, p);
}

// Fresh loop state; the peer-collective epoch is kept (flags in peer memory are monotone).
static tsvd_status reset_state(tsvd_t h) {
    uint32_t epoch = 0, xepoch = 0;
    if (h->allocated) {
        CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        epoch = h->st_host->epoch;
        xepoch = h->st_host->xepoch;
    }
    LoopState s{};
    s.ny = 1.0;
    s.epoch = epoch;
    s.xepoch = xepoch;
    *h->st_host = s;
    CK(cudaMemcpyAsync(h->st, h->st_host, sizeof(LoopState), cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return TSVD_OK;
}

// ---- setup-time collectives: NCCL across processes, the host rendezvous for in-process ranks
// every rank contributes (val, ptr); returns the min of val and every rank's ptr in rank order
// (LLONG_MIN if a rank did not arrive within 60 s)
static long long grp_exchange(tsvd_t h, long long val, void *ptr, std::vector<void *> *all, const char *tag = "") {
    InprocGroup &g = *h->grp;
    static const bool dbg = getenv("TSVD_GRP_DEBUG") != nullptr;  // debug: rendezvous trace on stderr
    if (dbg)
        fprintf(stderr, "[grp %p rank %d enter %s gen %llu t %.3f]\n", (void *)&g, h->rank, tag, g.gen,
                std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count());
    std::unique_lock<std::mutex> lk(g.mu);
    g.v[h->rank] = val;
    g.p[h->rank] = ptr;
    const unsigned long long my = g.gen;
    if (++g.arrived == g.world) {
        g.rmin = *std::min_element(g.v.begin(), g.v.end());
        g.rp = g.p;
        g.arrived = 0;
        ++g.gen;
        g.cv.notify_all();
    } else if (!g.cv.wait_for(lk, std::chrono::seconds(60), [&] { return g.gen != my; })) {
        if (dbg) fprintf(stderr, "[grp %p rank %d TIMEOUT %s gen %llu]\n", (void *)&g, h->rank, tag, my);
        return LLONG_MIN;
    }
    if (all) *all = g.rp;
    return g.rmin;
}

// In-process ranks share one device: a host API call with an implicit device-wide synchronisation
// (cudaFree, some allocations) in one rank's thread would wait for another rank's kernel that is
// spinning for this rank's exchange words.  Every rank finishes its host-side preparation (buffers,
// graph capture and instantiation) before any rank launches the run.
static tsvd_status inproc_rendezvous(tsvd_t h) {
    if (!h->grp) return TSVD_OK;
    if (grp_exchange(h, 0, nullptr, nullptr, "rendezvous") == LLONG_MIN)
        return h->fail(TSVD_ERR_NCCL, "in-process group: a rank did not arrive within 60 s");
    return TSVD_OK;
}

// v = min over the ranks
static tsvd_status coll_min_int(tsvd_t h, int &v) {
    if (h->grp) {
        const long long r = grp_exchange(h, v, nullptr, nullptr, "min");
        if (r == LLONG_MIN) return h->fail(TSVD_ERR_NCCL, "in-process group: a rank did not arrive within 60 s");
        v = (int)r;
        return TSVD_OK;
    }
    int *d = nullptr;
    CK(cudaMalloc((void **)&d, sizeof(int)));
    CK(cudaMemcpy(d, &v, sizeof(int), cudaMemcpyHostToDevice));
    NK(ncclAllReduce(d, d, 1, ncclInt, ncclMin, h->comm, h->stream));
    CK(cudaMemcpyAsync(&v, d, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(d);
    return TSVD_OK;
}

// out[i] = sum over ranks of in_r[i], in rank order (in-process ranks: every rank's buffer is a
// device pointer of this process)
struct RankPtrs {
    const void *p[kMaxRanks];
};
template <typename F>
__global__ void sum_ranks(RankPtrs in, int world, F *__restrict__ out, int64_t count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        F acc = static_cast<const F *>(in.p[0])[i];
        for (int r = 1; r < world; ++r) acc += static_cast<const F *>(in.p[r])[i];
        out[i] = acc;
    }
}

// In-place sum all-reduce of `count` fp32 / fp64 elements on stream s: ncclAllReduce across
// processes; for in-process ranks a host rendezvous (every rank's partial complete), a rank-ordered
// sum of the ranks' buffers into a scratch buffer, a second rendezvous (every rank done reading),
// and the copy back — host-synchronous, used only where the multi-process path calls NCCL (sparse
// vectors, the explicit Gram's B0 and extraction sums)
static tsvd_status coll_allreduce(tsvd_t h, void *buf, size_t count, bool f64, cudaStream_t s) {
    if (!h->grp) {
        NK(ncclAllReduce(buf, buf, count, f64 ? ncclDouble : ncclFloat, ncclSum, h->comm, s));
        return TSVD_OK;
    }
    const size_t bytes = count * (f64 ? 8 : 4);
    if (bytes > h->ar_bytes) {
        CK(cudaStreamSynchronize(s));
        if (h->ar_tmp) CK(cudaFree(h->ar_tmp));
        h->ar_tmp = nullptr;
        CK(cudaMalloc(&h->ar_tmp, bytes));
        h->ar_bytes = bytes;
    }
    CK(cudaStreamSynchronize(s));
    std::vector<void *> all;
    if (grp_exchange(h, 0, buf, &all, "allreduce-1") == LLONG_MIN)
        return h->fail(TSVD_ERR_NCCL, "in-process group: a rank did not arrive within 60 s");
    RankPtrs rp{};
    for (int r = 0; r < h->world; ++r) rp.p[r] = all[r];
    const int blocks = (int)std::min<int64_t>(((int64_t)count + 255) / 256, (int64_t)h->sms * 8);
    if (count) {
        if (f64) sum_ranks<double><<<blocks, 256, 0, s>>>(rp, h->world, (double *)h->ar_tmp, (int64_t)count);
        else sum_ranks<float><<<blocks, 256, 0, s>>>(rp, h->world, (float *)h->ar_tmp, (int64_t)count);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s));
    if (grp_exchange(h, 0, nullptr, nullptr, "allreduce-2") == LLONG_MIN)
        return h->fail(TSVD_ERR_NCCL, "in-process group: a rank did not arrive within 60 s");
    if (count) CK(cudaMemcpyAsync(buf, h->ar_tmp, bytes, cudaMemcpyDeviceToDevice, s));
    return TSVD_OK;
}

// base[r] = rank r's copy of an exchange buffer (mine for r == rank).  Across processes: CUDA IPC
// handles all-gathered with NCCL and opened (maps[r] records what tsvd_destroy closes; ok = false if
// an open failed); in-process ranks: the other handles' device pointers themselves
static tsvd_status coll_share(tsvd_t h, void *mine, void **base, void **maps, bool &ok, std::string &err) {
    ok = true;
    if (h->grp) {
        std::vector<void *> all;
        if (grp_exchange(h, 0, mine, &all, "share") == LLONG_MIN)
            return h->fail(TSVD_ERR_NCCL, "in-process group: a rank did not arrive within 60 s");
        for (int r = 0; r < h->world; ++r) base[r] = all[r];
        return TSVD_OK;
    }
    cudaIpcMemHandle_t hm;
    CK(cudaIpcGetMemHandle(&hm, mine));
    char *dbuf = nullptr;
    CK(cudaMalloc((void **)&dbuf, sizeof(cudaIpcMemHandle_t) * (h->world + 1)));
    CK(cudaMemcpy(dbuf, &hm, sizeof(hm), cudaMemcpyHostToDevice));
    NK(ncclAllGather(dbuf, dbuf + sizeof(hm), sizeof(hm), ncclUint8, h->comm, h->stream));
    std::vector<cudaIpcMemHandle_t> all(h->world);
    CK(cudaMemcpyAsync(all.data(), dbuf + sizeof(hm), sizeof(hm) * h->world, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(dbuf);
    for (int r = 0; r < h->world; ++r) {
        base[r] = mine;
        if (r == h->rank) continue;
        void *q = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&q, all[r], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
            ok = false;
            base[r] = nullptr;
            continue;
        }
        maps[r] = q;
        base[r] = q;
    }
    return TSVD_OK;
}

// Receive areas of the persistent kernel's exchange (N7, world > 1): [2][world][G][SL] doubles +
// flags [world][G] per rank, mapped by coll_share.  Needs one column block per CTA
// (slice width <= 128 columns); otherwise the multi-GPU run keeps the per-iteration kernels.
static tsvd_status setup_px(tsvd_t h) {
    // the column slices must be the same on every rank: slice by the smallest grid of any rank
    // (a rank with fewer rows than CTA slots runs a smaller grid)
    int G = h->grid;
    TRY(coll_min_int(h, G));
    const int CW = std::min(h->T_ps, 128);
    const int per = (int)(((h->n + G - 1) / G + 31) / 32 * 32);
    if (per > CW || h->world > kMaxRanks) return TSVD_OK;
    const int SL = (int)round_up(per + h->kpad, 4);
    const size_t bytes = (size_t)2 * h->world * G * SL * sizeof(ulonglong2);
    CK(cudaMalloc((void **)&h->px_mem, bytes));
    // zeroed on the handle's stream and waited for BEFORE the pointer is shared: a plain cudaMemset
    // runs on the legacy stream, unordered with the peers' (non-blocking) streams, and a late memset
    // wiped stamped words a peer had already written (the receiver then waited out the 30 s timeout;
    // seen with in-process ranks, where the window is widest)
    CK(cudaMemsetAsync(h->px_mem, 0, bytes, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    void *base[kMaxRanks] = {};
    bool ok = true;
    std::string err;
    TRY(coll_share(h, h->px_mem, base, h->px_map, ok, err));
    if (!ok) h->peer_error = "persistent exchange: " + err;
    PxView px{};
    px.world = h->world;
    px.rank = h->rank;
    px.G = G;
    px.per = per;
    px.SL = SL;
    for (int r = 0; r < h->world; ++r) px.rbuf[r] = (ulonglong2 *)base[r];
    px.lbuf = (const ulonglong2 *)h->px_mem;
    // every rank must agree, or none uses the persistent exchange
    int agreed = ok ? 1 : 0;
    TRY(coll_min_int(h, agreed));
    h->px = px;
    h->px_ok = agreed == 1;
    return TSVD_OK;
}

static tsvd_status ensure_alloc(tsvd_t h) {
    if (h->allocated) return TSVD_OK;
    TRY(plan(h));
    const int64_t n = h->n, mg = h->m_g;
    h->ystride = round_up(n, 32);
    h->wofs = round_up(n, 32);
    // per-CTA partial rows: padded so the rows of different CTAs do not sit a power of two apart
    h->ypart_ld = round_up(n, 4) + (getenv("TSVD_NOPAD") ? 0 : 40);
    h->fin_blocks = (int)std::min<int64_t>((n + kFinCols - 1) / kFinCols, (int64_t)h->sms * 4);  // one wave
    h->part_ld = 2 + h->kpad;
    auto dm = [&](void **p, size_t bytes) -> cudaError_t {
        h->work_bytes += (int64_t)std::max<size_t>(bytes, 16);
        return cudaMalloc(p, std::max<size_t>(bytes, 16));
    };
    cudaError_t e = cudaSuccess;
    if (!e) e = dm((void **)&h->U32, (size_t)mg * h->kpad * sizeof(float));
    // the heavy co-factor V (n x k) and the initial samples (k x n): HBM by default; with
    // TSVD_OPT_V_PLACEMENT = 1 pinned host memory mapped into the device address space ("the
    // heavy co-factor V is stored on the host"), read by the kernels over the host link
    auto vm = [&](double **dptr, double **hptr, size_t bytes) -> cudaError_t {
        if (!h->v_host) return dm((void **)dptr, bytes);
        cudaError_t ee = cudaHostAlloc((void **)hptr, std::max<size_t>(bytes, 16), cudaHostAllocMapped);
        if (!ee) ee = cudaHostGetDevicePointer((void **)dptr, *hptr, 0);
        return ee;
    };
    if (!e) e = vm(&h->V64, &h->V64_h, (size_t)n * h->k * sizeof(double));
    if (!e) e = dm((void **)&h->S64, (size_t)h->k * sizeof(double));
    if (!e) e = dm((void **)&h->ybuf, (size_t)2 * h->ystride * sizeof(double));
    if (!e) e = dm((void **)&h->yw, (size_t)(h->wofs + h->kpad) * sizeof(double));
    if (!e) e = vm(&h->V0d, &h->V0d_h, (size_t)h->k * n * sizeof(double));
    if (!e) e = dm((void **)&h->c64, (size_t)h->kpad * sizeof(double));
    if (!e && !h->sparse) e = dm((void **)&h->ypart, (size_t)h->parts * h->ypart_ld * sizeof(double));
    if (!e) e = dm((void **)&h->wpart, (size_t)h->parts * h->kpad * sizeof(double));
    if (!e) e = dm((void **)&h->part, (size_t)std::max(h->fin_blocks, h->grid) * h->part_ld * sizeof(double));
    if (!e) e = dm((void **)&h->u64, (size_t)mg * sizeof(double));
    if (!e && h->sparse) e = dm((void **)&h->y32, (size_t)round_up(n, 4) * sizeof(float));
    if (!e && h->sparse) e = dm((void **)&h->t32, (size_t)mg * sizeof(float));
    if (!e) e = dm((void **)&h->sq_part, (size_t)h->parts * sizeof(double));
    if (!e) e = dm((void **)&h->sig2, sizeof(double));
    if (!e) e = dm((void **)&h->st, sizeof(LoopState));
    if (!e) e = dm((void **)&h->stats, (size_t)h->k * sizeof(CompStat));
    if (!e) e = dm((void **)&h->gbar, 2 * sizeof(unsigned));
    if (!e) e = cudaMemsetAsync(h->gbar, 0, 2 * sizeof(unsigned), h->stream);
    if (!e) e = dm((void **)&h->work, 2 * sizeof(unsigned long long));
    if (!e && !h->sparse) {  // persistent kernel's stamped publication words (zero: no stamp matches)
        e = dm((void **)&h->pub, (size_t)h->grid * h->part_ld * sizeof(ulonglong2));
        if (!e) e = cudaMemsetAsync(h->pub, 0, (size_t)h->grid * h->part_ld * sizeof(ulonglong2), h->stream);
        if (!e) e = dm((void **)&h->puby, (size_t)round_up(n, 4) * sizeof(unsigned long long));
        if (!e) e = cudaMemsetAsync(h->puby, 0, (size_t)round_up(n, 4) * sizeof(unsigned long long), h->stream);
    }
    if (!e && !h->sparse) {
        e = dm((void **)&h->vprev32, (size_t)round_up(n, 4) * sizeof(float));
        if (!e) e = cudaMemsetAsync(h->vprev32, 0, (size_t)round_up(n, 4) * sizeof(float), h->stream);
    }
    if (!e) e = cudaMemsetAsync(h->work, 0, 2 * sizeof(unsigned long long), h->stream);
    if (!e && getenv("TSVD_TRACE")) {
        e = dm((void **)&h->trace_d, (size_t)h->grid * 4 * sizeof(unsigned long long));
        char name[1024];
        snprintf(name, sizeof name, "%s.rank%d", getenv("TSVD_TRACE"), h->rank);
        h->trace_f = fopen(name, "a");
    }
    if (!e && getenv("TSVD_TIMELINE")) {
        e = dm((void **)&h->tl_d, (2 + kTl * 4096) * sizeof(unsigned long long));
        if (!e) e = cudaMemsetAsync(h->tl_d, 0, (2 + kTl * 4096) * sizeof(unsigned long long), h->stream);
    }
    if (!e) e = cudaMallocHost((void **)&h->st_host, sizeof(LoopState));
    if (!e) e = cudaMallocHost((void **)&h->stats_host, (size_t)h->k * sizeof(CompStat));
    if (!e) e = cudaMallocHost((void **)&h->vec_host, (size_t)n * sizeof(double));
    if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "device workspace allocation failed");
    CK(e);
    CK(cudaMemsetAsync(h->U32, 0, (size_t)mg * h->kpad * sizeof(float), h->stream));
    CK(cudaMemsetAsync(h->V64, 0, (size_t)n * h->k * sizeof(double), h->stream));
    CK(cudaMemsetAsync(h->S64, 0, (size_t)h->k * sizeof(double), h->stream));
    CK(cudaMemsetAsync(h->ybuf, 0, (size_t)2 * h->ystride * sizeof(double), h->stream));
    CK(cudaMemsetAsync(h->c64, 0, (size_t)h->kpad * sizeof(double), h->stream));
    CK(cudaMemsetAsync(h->yw, 0, (size_t)(h->wofs + h->kpad) * sizeof(double), h->stream));
    TRY(reset_state(h));
    h->allocated = true;
    if (h->world > 1 && h->coll == COLL_PEER && h->gv_ps && !h->sparse) TRY(setup_px(h));
    return TSVD_OK;
}

// Symmetric buffers for the in-kernel all-reduce: [2 slots x (y | w | ||u||^2)] + flags[world].
// Every rank cudaMallocs its own; coll_share maps every rank's (CUDA IPC across processes).
static tsvd_status setup_peer(tsvd_t h) {
    const int64_t wofs = round_up(h->n, 32), sofs = wofs + round_up(h->k, 4);
    const int64_t slot = round_up(sofs + 1, 32);
    const size_t flag_off = (size_t)2 * slot * sizeof(double);
    const size_t bytes = flag_off + 256;
    CK(cudaMalloc((void **)&h->sym, bytes));
    CK(cudaMemsetAsync(h->sym, 0, bytes, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    void *base[kMaxRanks] = {};
    bool ok = true;
    TRY(coll_share(h, h->sym, base, h->peer_map, ok, h->peer_error));
    if (!ok) return TSVD_ERR_CUDA;
    PeerView pv{};
    pv.world = h->world;
    pv.rank = h->rank;
    pv.slot_stride = slot;
    pv.wofs = wofs;
    pv.sofs = sofs;
    for (int r = 0; r < h->world; ++r) {
        pv.buf[r] = (double *)base[r];
        pv.rflags[r] = (unsigned *)((char *)base[r] + flag_off) + h->rank;
    }
    pv.flags = (unsigned *)((char *)h->sym + flag_off);
    h->pv = pv;
    return TSVD_OK;
}

static void free_ring(tsvd_t h) {
    for (float *p : h->ring) cudaFree(p);
    for (cudaEvent_t e : h->ev_full) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_free) cudaEventDestroy(e);
    h->ring.clear();
    h->ev_full.clear();
    h->ev_free.clear();
}

// Host input: decide the placement and make the resident rows device-resident for this
// run (H2D copy, counted in e2e timing).  Degree 0: the whole slab.  Degree 1: rows [0, m_res)
// resident, rows [m_res, m_g) streamed each pass through the ring (launch_pass).
static tsvd_status stage_A(tsvd_t h) {
    if (h->sparse) return TSVD_OK;  // CSR/CSC staged (and validated) by tsvd_set_csr
    if (h->mem == TSVD_MEM_DEVICE) {
        h->streaming = false;
        h->m_res = h->m_g;
        return TSVD_OK;
    }
    const int64_t n4 = (h->n + 3) / 4;
    const int64_t row_bytes = n4 * 16;
    h->ld_own = n4 * 4;
    if (!h->A_own || h->own_rows == 0) {  // first staging for this slab: decide the placement once
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const int64_t reserve = (int64_t)1 << 30;
        const int64_t avail = std::max<int64_t>(0, (int64_t)fr - reserve);
        const bool fits = row_bytes * h->m_g <= avail;
        if (h->placement == 1 && !fits)
            return h->fail(TSVD_ERR_NOMEM, "PLACEMENT=resident but the slab (%lld B) exceeds free HBM (%lld B)",
                           (long long)(row_bytes * h->m_g), (long long)avail);
        h->streaming = (h->placement == 2) || (h->placement == 0 && !fits);
        if (!h->streaming) {
            h->m_res = h->m_g;
        } else {
            h->batch_rows = h->batch_rows_opt > 0 ? h->batch_rows_opt
                                                  : std::max<int64_t>(1, (256ll << 20) / row_bytes);
            h->batch_rows = std::min(h->batch_rows, h->m_g);
            const int64_t ring_bytes = (int64_t)h->qdepth * h->batch_rows * row_bytes;
            if (ring_bytes > avail)
                return h->fail(TSVD_ERR_NOMEM, "no room for the %d-slot streaming ring (OOM degree 2, P:173)",
                               h->qdepth);
            int64_t res = (avail - ring_bytes) / row_bytes;
            if (h->resident_cap >= 0) res = std::min(res, h->resident_cap / row_bytes);
            h->m_res = std::min(res, h->m_g);
            for (int s = 0; s < h->qdepth; ++s) {
                float *p = nullptr;
                cudaEvent_t ef, eb;
                CK(cudaMalloc((void **)&p, (size_t)h->batch_rows * row_bytes));
                CK(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&eb, cudaEventDisableTiming));
                h->ring.push_back(p);
                h->ev_full.push_back(ef);
                h->ev_free.push_back(eb);
            }
            if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        }
        if (h->m_res > 0) {
            if (h->A_own) cudaFree(h->A_own);
            h->A_own = nullptr;
            cudaError_t e = cudaMalloc((void **)&h->A_own, (size_t)h->m_res * row_bytes);
            if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "A device buffer allocation failed");
            CK(e);
            if (h->ld_own != h->n) CK(cudaMemsetAsync(h->A_own, 0, (size_t)h->m_res * row_bytes, h->stream));
        }
        h->own_rows = std::max<int64_t>(h->m_res, 1);
        h->graph_l0 = -1;  // A pointer changed: the cached run graph is stale
    }
    if (h->streaming && h->mem == TSVD_MEM_HOST_PAGEABLE && !h->host_registered) {
        CK(cudaHostRegister((void *)h->A_user, (size_t)h->m_g * h->ld_user * sizeof(float), cudaHostRegisterDefault));
        h->host_registered = true;
    }
    if (h->m_res > 0) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, h->stream));
        CK(cudaMemcpy2DAsync(h->A_own, h->ld_own * sizeof(float), h->A_user, h->ld_user * sizeof(float),
                             h->n * sizeof(float), h->m_res, cudaMemcpyHostToDevice, h->stream));
        CK(cudaEventRecord(e1, h->stream));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        h->h2d_ms += ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    h->A_use = h->A_own;
    h->ld_use = h->ld_own;
    return TSVD_OK;
}

static tsvd_status unstage_A(tsvd_t h) {
    if (h->host_registered) {
        CK(cudaHostUnregister((void *)h->A_user));
        h->host_registered = false;
    }
    return TSVD_OK;
}

// ------------------------------------------------------------------------------------ launches
static GvParams gv_params(tsvd_t h, int l, bool extract) {
    GvParams p{};
    p.A = h->A_use;
    p.ld = h->ld_use;
    p.rows = h->m_res;
    p.n = (int32_t)h->n;
    p.n4 = (int32_t)((h->n + 3) / 4);
    p.U = h->U32;
    p.ldu = h->kpad;
    p.l = extract ? 0 : l;
    p.ybuf = h->ybuf;
    p.ystride = h->ystride;
    p.st = h->st;
    p.c = h->c64;
    p.ypart = h->ypart;
    p.ypart_ld = h->ypart_ld;
    p.wpart = h->wpart;
    p.wpart_ld = h->kpad;
    p.stages = h->S;
    p.stage_bytes = h->stage_bytes;
    p.row_bytes = h->row_bytes;
    p.u_bytes = (extract || l == 0) ? 0 : (int32_t)(round_up(l, 4) * 4);
    p.run_rows = h->run_rows;
    p.u_out = h->u64;
    p.sq_part = h->sq_part;
    p.reduce_mode = (!extract && fused_reduce(h)) ? (h->coll == COLL_PEER ? 2 : 1) : 0;
    p.yw = h->yw;
    p.wofs = h->wofs;
    p.gbar = h->gbar;
    p.pv = h->pv;
    p.trace = extract ? nullptr : h->trace_d;
    p.dynamic = h->dynamic_opt;
    p.chunk_rows = (int32_t)std::max<int64_t>(1, (256 << 10) / h->row_bytes);
    p.serpentine = h->serp_opt && !h->streaming;
    p.work = h->work;
    p.tl = extract ? nullptr : h->tl_d;
    return p;
}

// One pass of N1 over this rank's rows.  Resident slab: one launch.  Out of memory (degree 1): one
// launch over the resident prefix, then row batches copied host->device on the copy stream into a
// q_s-slot ring (slot reuse gated by events) and consumed by N1 launches that accumulate into the
// same per-CTA partials, so the H2D of batch b+1.. overlaps the kernel on batch b.
static SpParams sp_params(tsvd_t h, int l) {
    SpParams p{};
    p.phase = 0;
    p.nphase = 1;
    p.csr = h->spc;
    p.csc = h->spr;
    p.rows = h->m_g;
    p.n = h->n;
    p.U = h->U32;
    p.ldu = h->kpad;
    p.l = l;
    p.c = h->c64;
    p.ybuf = h->ybuf;
    p.ystride = h->ystride;
    p.st = h->st;
    p.t = h->u64;
    p.t32 = h->t32;
    p.y32 = h->y32;
    p.wpart = h->wpart;
    p.wpart_ld = h->kpad;
    p.sq_part = h->sq_part;
    p.yw = h->yw;
    p.wofs = h->wofs;
    p.parts = h->parts;
    return p;
}

// the sparse pass overlaps its cross-rank sum with N3 (column chunks of the last index block)
static bool sp_overlap(tsvd_t h) {
    return h->sparse && h->world > 1 && h->coll == COLL_NCCL && h->sp_chunks > 1 && !h->grp;
}

// Sparse pass: N2 (rows, one launch per column block) then N3 (columns, one launch per row block);
// N2 alone for the extraction.  world > 1: N3's last block runs in column chunks and each chunk's
// [y] (the last one with [w]) is all-reduced on a side stream while the next chunk computes.
// out of memory (degree 1): before a block launch of view v (0 = CSR, 1 = CSC), copy the block's entries
// into the next ring slot on the copy stream (slot reuse gated by the kernel that last read it)
static tsvd_status sp_stage_block(tsvd_t h, cudaStream_t s, int v, int b, SpParams &q) {
    q.blk_idx = nullptr;
    q.blk_val = nullptr;
    if (!h->sp_stream) return TSVD_OK;
    const int slot = (int)(h->sp_launch++ % (int64_t)h->sp_ring.size());
    const int64_t e0 = h->sp_hbase[v][b], cnt = h->sp_hbase[v][b + 1] - e0;
    int32_t *di = (int32_t *)h->sp_ring[slot];
    float *dv = (float *)(di + h->sp_slot_entries);
    CK(cudaStreamWaitEvent(h->copy_stream, h->sp_free[slot], 0));
    CK(cudaMemcpyAsync(di, h->sp_hidx[v] + e0, (size_t)cnt * sizeof(int32_t), cudaMemcpyHostToDevice, h->copy_stream));
    CK(cudaMemcpyAsync(dv, h->sp_hval[v] + e0, (size_t)cnt * sizeof(float), cudaMemcpyHostToDevice, h->copy_stream));
    CK(cudaEventRecord(h->sp_full[slot], h->copy_stream));
    CK(cudaStreamWaitEvent(s, h->sp_full[slot], 0));
    h->streamed_bytes += cnt * 8;
    h->streamed_batches += 1;
    q.blk_idx = di;
    q.blk_val = dv;
    q.phase = b;
    return TSVD_OK;
}
static tsvd_status sp_release_block(tsvd_t h, cudaStream_t s) {
    if (h->sp_stream)
        CK(cudaEventRecord(h->sp_free[(int)((h->sp_launch - 1) % (int64_t)h->sp_ring.size())], s));
    return TSVD_OK;
}

static tsvd_status launch_sparse(tsvd_t h, cudaStream_t s, int l, bool extract) {
    SpParams q = sp_params(h, l);  // one launch per index block (phase), partial sums carried in acc
    q.nphase = h->sp_kc;
    q.acc[0] = h->acc_r;
    q.acc[1] = h->acc_r ? h->acc_r + h->m_g : nullptr;
    q.sl0 = 0;
    q.sl1 = h->spc.nsl;
    const size_t dyn = (size_t)std::max(l, 0) * (kSpThreads + 1) * sizeof(double);
    for (int b = 0; b < h->sp_kc; ++b) {
        q.phase = b;
        TRY(sp_stage_block(h, s, 0, b, q));
        const bool last = b + 1 == h->sp_kc;
        if (!last) CK(launch_k(h, extract ? sp_pass<MODE_U, false> : sp_pass<MODE_T, false>, h->grid_nl, kSpThreads,
                               0, s, 1, q));
        else if (extract) CK(launch_k(h, sp_pass<MODE_U, true>, h->grid, kSpThreads, 0, s, 1, q));
        else CK(launch_k(h, sp_pass<MODE_T, true>, h->grid, kSpThreads, dyn, s, 1, q));
        TRY(sp_release_block(h, s));
    }
    if (!extract) {
        q.nphase = h->sp_kr;
        q.acc[0] = h->acc_c;
        q.acc[1] = h->acc_c ? h->acc_c + h->n : nullptr;
        q.sl0 = 0;
        q.sl1 = h->spr.nsl;
        for (int b = 0; b + 1 < h->sp_kr; ++b) {
            q.phase = b;
            TRY(sp_stage_block(h, s, 1, b, q));
            CK(launch_k(h, sp_pass<MODE_Y, false>, h->grid_nl, kSpThreads, 0, s, 1, q));
            TRY(sp_release_block(h, s));
        }
        q.phase = h->sp_kr - 1;
        TRY(sp_stage_block(h, s, 1, h->sp_kr - 1, q));
        if (!sp_overlap(h)) {
            CK(launch_k(h, sp_pass<MODE_Y, true>, h->grid, kSpThreads, 0, s, 1, q));
        } else {
            // column chunks on sorting-window boundaries (a window's slices hold only its columns)
            const int C = h->sp_chunks;
            const int64_t nwin = (h->n + kSellW - 1) / kSellW;
            for (int c = 0; c < C; ++c) {
                const int64_t w0 = nwin * c / C, w1 = nwin * (c + 1) / C;
                const int64_t c0 = w0 * kSellW, c1 = c + 1 == C ? h->n : w1 * kSellW;
                q.sl0 = c0 / 32;
                q.sl1 = c + 1 == C ? h->spr.nsl : c1 / 32;
                if (q.sl1 > q.sl0) CK(launch_k(h, sp_pass<MODE_Y, true>, h->grid, kSpThreads, 0, s, 1, q));
                CK(cudaEventRecord(h->sp_ev[c], s));
                CK(cudaStreamWaitEvent(h->sp_comm_stream, h->sp_ev[c], 0));
                const int64_t e1 = c + 1 == C ? h->wofs + h->kpad : c1;  // the last chunk carries w
                if (e1 > c0)
                    NK(ncclAllReduce(h->yw + c0, h->yw + c0, (size_t)(e1 - c0), ncclDouble, ncclSum, h->comm,
                                     h->sp_comm_stream));
            }
            CK(cudaEventRecord(h->sp_ev[C], h->sp_comm_stream));
            CK(cudaStreamWaitEvent(s, h->sp_ev[C], 0));
        }
        TRY(sp_release_block(h, s));
    }
    CK(cudaGetLastError());
    return TSVD_OK;
}

static tsvd_status launch_gv(tsvd_t h, cudaStream_t s, int l, bool extract) {
    if (h->sparse) return launch_sparse(h, s, l, extract);
    GvFn fn = extract ? h->gv_ex : h->gv;
    GvParams p = gv_params(h, l, extract);
    if (p.reduce_mode) {  // grid barrier inside: cooperative launch guarantees co-residency
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.gridDim = dim3(h->grid);
        cfg.blockDim = dim3(h->T);
        cfg.dynamicSmemBytes = h->smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, fn, p));
        return TSVD_OK;
    }
    if (!h->streaming || h->m_res > 0) CK(launch_n1(h, fn, p, s));
    if (!h->streaming) return TSVD_OK;
    const int64_t row_bytes = (int64_t)h->row_bytes;
    int b = 0;
    for (int64_t r0 = h->m_res; r0 < h->m_g; r0 += h->batch_rows, ++b) {
        const int slot = b % h->qdepth;
        const int64_t rows = std::min(h->batch_rows, h->m_g - r0);
        CK(cudaStreamWaitEvent(h->copy_stream, h->ev_free[slot], 0));
        CK(cudaMemcpy2DAsync(h->ring[slot], row_bytes, h->A_user + r0 * h->ld_user, h->ld_user * sizeof(float),
                             h->n * sizeof(float), rows, cudaMemcpyHostToDevice, h->copy_stream));
        CK(cudaEventRecord(h->ev_full[slot], h->copy_stream));
        CK(cudaStreamWaitEvent(s, h->ev_full[slot], 0));
        GvParams q = p;
        q.A = h->ring[slot];
        q.ld = row_bytes / 4;
        q.rows = rows;
        q.U = h->U32 + r0 * h->kpad;
        q.u_out = h->u64 + r0;
        q.accumulate = (r0 > 0 || h->m_res > 0) ? 1 : 0;
        CK(launch_n1(h, fn, q, s));
        CK(cudaEventRecord(h->ev_free[slot], s));
        h->streamed_bytes += rows * h->n * (int64_t)sizeof(float);
        h->streamed_batches += 1;
    }
    return TSVD_OK;
}

static FinParams fin_params(tsvd_t h, int mode, int l, const double *xsrc, unsigned long long cond, int use_cond) {
    FinParams p{};
    p.mode = mode;
    p.n = (int)h->n;
    p.l = l;
    p.S = h->S64;
    p.V = h->V64;
    p.ldv = h->k;
    p.ypart = h->ypart;
    p.parts = h->parts;
    p.ypart_ld = h->ypart_ld;
    p.wpart = h->wpart;
    p.wpart_ld = h->kpad;
    p.yw = h->yw;
    p.wofs = h->wofs;
    p.pv = h->pv;
    p.xsrc = xsrc;
    p.ybuf = h->ybuf;
    p.ystride = h->ystride;
    p.part = h->part;
    p.part_ld = h->part_ld;
    p.c = h->c64;
    p.st = h->st;
    p.eps = h->eps;
    p.fixed_T = h->fixed_T;
    p.max_iter = h->max_iter;
    p.cond = cond;
    p.use_cond = use_cond;
    p.tl = h->tl_d;
    p.fresh = l - 1;  // only read by the *_EXT modes
    p.y32 = h->sparse ? h->y32 : nullptr;
    p.Vout = h->V64;
    p.vprev32 = h->vprev32;
    p.stat = h->stats;
    p.sq_part = h->sq_part;
    p.sq_parts = h->parts;
    p.U = h->U32;
    p.ldu = h->kpad;
    p.u_out = h->u64;
    p.rows = h->m_g;
    return p;
}

static tsvd_status launch_fin(tsvd_t h, cudaStream_t s, const FinParams &p, int src) {
    const size_t dyn = (size_t)(2 * p.l + 2 + std::max(0, p.l - kVtReg) + kFinThreads) * sizeof(double);
    switch (src) {
    case SRC_PARTS: CK(launch_k(h, fin_iter<SRC_PARTS>, h->fin_blocks, kFinThreads, dyn, s, 1, p)); break;
    case SRC_YW: CK(launch_k(h, fin_iter<SRC_YW>, h->fin_blocks, kFinThreads, dyn, s, 1, p)); break;
    default: CK(launch_k(h, fin_iter<SRC_PEER>, h->fin_blocks, kFinThreads, dyn, s, 1, p)); break;
    }
    CK(cudaGetLastError());
    return TSVD_OK;
}

static PubParams pub_params(tsvd_t h, int mode, int l) {
    PubParams p{};
    p.mode = mode;
    p.ypart = h->ypart;
    p.parts = h->parts;
    p.ypart_ld = h->ypart_ld;
    p.wpart = h->wpart;
    p.wpart_ld = h->kpad;
    p.n = (int)h->n;
    p.l = l;
    p.sq_part = h->sq_part;
    p.pv = h->pv;
    p.st = h->st;
    return p;
}

// The cross-rank part of an iteration before fin_iter: nothing / publish / local sum + NCCL.
static tsvd_status launch_exchange(tsvd_t h, cudaStream_t s, int l) {
    if (h->sparse) {  // N3 already wrote [y_g | w_g]; the length-n sum is bandwidth-bound: NCCL
        if (h->world > 1 && !sp_overlap(h))
            TRY(coll_allreduce(h, h->yw, (size_t)(h->wofs + h->kpad), true, s));
        return TSVD_OK;
    }
    if (fused_reduce(h)) {  // N1 already summed its partials into yw / the symmetric slot
        if (h->coll == COLL_NCCL)
            TRY(coll_allreduce(h, h->yw, (size_t)(h->wofs + h->kpad), true, s));
        return TSVD_OK;
    }
    if (h->coll == COLL_PEER) {
        CK(launch_k(h, publish, h->fin_blocks, kFinThreads, 0, s, 1, pub_params(h, 0, l)));
    } else if (h->coll == COLL_NCCL) {
        CK(launch_k(h, reduce_partials, h->fin_blocks, kFinThreads, 0, s, 1, (const double *)h->ypart, h->parts,
                    h->ypart_ld, (int)h->n, (const double *)h->wpart, (int)h->kpad, l, h->yw, h->wofs,
                    (const LoopState *)h->st));
        TRY(coll_allreduce(h, h->yw, (size_t)(h->wofs + h->kpad), true, s));
    }
    return TSVD_OK;
}

// One power iteration: N1, [exchange], fin_iter.
static tsvd_status launch_iteration(tsvd_t h, cudaStream_t s, int l, unsigned long long cond, int use_cond,
                                    cudaEvent_t e0 = nullptr, cudaEvent_t e1 = nullptr) {
    if (e0) CK(cudaEventRecord(e0, s));
    TRY(launch_gv(h, s, l, false));
    if (e1) CK(cudaEventRecord(e1, s));
    TRY(launch_exchange(h, s, l));
    return launch_fin(h, s, fin_params(h, FIN_ITERATE, l, nullptr, cond, use_cond), fin_src(h));
}

// x_l (device, fp64) -> y_cur = x, ||x||, c = S V^T (x / ||x||)
static tsvd_status launch_init(tsvd_t h, cudaStream_t s, int l) {
    return launch_fin(h, s, fin_params(h, FIN_INIT, l, h->V0d + (size_t)l * h->n, 0ull, 0), SRC_PARTS);
}

// Fused extraction is used for dense, resident, unsplit slabs with an in-kernel reduction path.
static bool fuse_ext(tsvd_t h) {
    return h->fuse_ext_opt && h->gv_two && !h->sparse && !h->streaming && h->split == 1 && h->coll != COLL_NCCL &&
           !fused_reduce(h);
}

// Component l >= 1 with fused extraction.  FIN_INIT_EXT: V[:, l-1] = v_{l-1} (+ fp32 copy), load
// x_l, c = (S V^T x / ||x||) with weight 1 on column l-1.  Then ONE pass over A (N1<TWO>) does the
// first iteration of component l and u = A v_{l-1}; FIN_ITERATE_EXT finishes both:
// sigma_{l-1} = ||u||, U[:, l-1] = u / sigma_{l-1}, and the iterate of component l.
static tsvd_status launch_init_ext(tsvd_t h, cudaStream_t s, int l) {
    return launch_fin(h, s, fin_params(h, FIN_INIT_EXT, l, h->V0d + (size_t)l * h->n, 0ull, 0), SRC_PARTS);
}

// the two-vector pass alone (its partials are reduced by the next kernel)
static tsvd_status launch_two(tsvd_t h, cudaStream_t s, int l) {
    GvParams p = gv_params(h, l, false);
    p.l = l;
    p.u_bytes = l - 1 > 0 ? (int32_t)(round_up(l - 1, 4) * 4) : 0;
    p.stages = h->S_two;
    p.vprev = h->vprev32;
    p.vp_bytes = h->vp_bytes;
    p.reduce_mode = 0;
    p.tl = nullptr;
    p.trace = nullptr;
    CK(launch_k(h, h->gv_two, h->grid, h->T_two, h->smem_two, s, 1, p));
    return TSVD_OK;
}

static tsvd_status launch_fused_first(tsvd_t h, cudaStream_t s, int l, cudaEvent_t e0 = nullptr,
                                      cudaEvent_t e1 = nullptr) {
    if (e0) CK(cudaEventRecord(e0, s));
    GvParams p = gv_params(h, l, false);
    p.l = l;
    p.u_bytes = l - 1 > 0 ? (int32_t)(round_up(l - 1, 4) * 4) : 0;
    p.stages = h->S_two;
    p.vprev = h->vprev32;
    p.vp_bytes = h->vp_bytes;
    p.reduce_mode = 0;
    p.tl = nullptr;
    p.trace = nullptr;
    CK(launch_k(h, h->gv_two, h->grid, h->T_two, h->smem_two, s, 1, p));
    if (e1) CK(cudaEventRecord(e1, s));
    if (h->coll == COLL_PEER) {
        PubParams q = pub_params(h, 0, l);
        q.with_sq = 1;
        CK(launch_k(h, publish, h->fin_blocks, kFinThreads, 0, s, 1, q));
    }
    return launch_fin(h, s, fin_params(h, FIN_ITERATE_EXT, l, nullptr, 0ull, 0), fin_src(h));
}

// N7: the iterations of component l after the first (or all of them), in one cooperative launch.
static bool use_persist(tsvd_t h) {
    return h->persist_opt && h->gv_ps && !h->sparse && !h->streaming && h->split == 1 &&
           (h->coll == COLL_NONE || (h->coll == COLL_PEER && h->px_ok)) && !fused_reduce(h) && h->dynamic_opt == 0;
}

// head: the launch first reduces the two-vector pass of component l (extraction of l - 1);
// tail: after component l stops, it initialises component l + 1 (R21, DESIGN §6 N7)
static tsvd_status launch_persist(tsvd_t h, cudaStream_t s, int l, cudaEvent_t e0 = nullptr,
                                  cudaEvent_t e1 = nullptr, int head = 0, int tail = 0) {
    PsParams p{};
    p.head_ext = head;
    p.tail_init = tail;
    p.fresh = l - 1;
    p.Sw = h->S64;
    p.Vw = h->V64;
    p.Uw = h->U32;
    p.u_out = h->u64;
    p.sq_part = h->sq_part;
    p.stat = h->stats;
    p.V0n = tail ? h->V0d + (size_t)(l + 1) * h->n : nullptr;
    p.vprev32 = h->vprev32;
    p.A = h->A_use;
    p.ld = h->ld_use;
    p.rows = h->m_res;
    p.n = (int32_t)h->n;
    p.n4 = (int32_t)((h->n + 3) / 4);
    p.U = h->U32;
    p.ldu = h->kpad;
    p.l = l;
    p.u_bytes = l == 0 ? 0 : (int32_t)(round_up(l, 4) * 4);
    p.stages = h->S_ps;
    p.stage_bytes = h->stage_bytes;
    p.row_bytes = h->row_bytes;
    p.run_rows = h->run_rows;
    p.ybuf = h->ybuf;
    p.ystride = h->ystride;
    p.st = h->st;
    p.c = h->c64;
    p.S = h->S64;
    p.V = h->V64;
    p.ldv = h->k;
    p.ypart = h->ypart;
    p.ypart_ld = h->ypart_ld;
    p.wpart = h->wpart;
    p.wpart_ld = h->kpad;
    p.part = h->part;
    p.part_ld = h->part_ld;
    p.pub = h->pub;
    p.puby = h->puby;
    p.gbar = h->gbar;
    p.eps = h->eps;
    p.fixed_T = h->fixed_T;
    p.max_iter = h->max_iter;
    p.serpentine = h->serp_opt;
    // rows per CTA <= RUN_ROWS: each CTA's partial is one fp32 run, stored as fp32 (half the bytes;
    // the reduction widens to fp64 exactly as the fp64 store did)
    p.part32 = (h->m_res + h->grid - 1) / h->grid <= h->run_rows ? 1 : 0;
    if (const char *e = getenv("TSVD_PART32")) p.part32 &= atoi(e);  // debug A/B knob
    p.tl = h->tl_d;
    p.px.world = 1;
    if (h->world > 1) p.px = h->px;
    {  // the slice of V[:, :l] in shared memory when it fits the space plan() reserved
        const int Gs = h->world > 1 ? p.px.G : h->grid;
        const int64_t per = ((h->n + Gs - 1) / Gs + 31) / 32 * 32;
        p.vcache = (l > 0 && (int64_t)l * (per + 1) <= h->vcache_doubles && !getenv("TSVD_NO_VCACHE")) ? 1 : 0;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: grid barriers inside
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(h->grid);
    cfg.blockDim = dim3(h->T_ps);
    cfg.dynamicSmemBytes = h->smem_ps;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (e0) CK(cudaEventRecord(e0, s));
    CK(cudaLaunchKernelEx(&cfg, h->gv_ps, p));
    if (e1) CK(cudaEventRecord(e1, s));
    return TSVD_OK;
}

static tsvd_status launch_extract(tsvd_t h, cudaStream_t s, int l) {
    TRY(launch_gv(h, s, l, true));
    ExtParams p{};
    p.rows = h->m_g;
    p.n = (int)h->n;
    p.l = l;
    p.u = h->u64;
    p.sq_part = h->sq_part;
    p.parts = h->parts;
    p.sig2 = h->sig2;
    p.pv = h->pv;
    p.ybuf = h->ybuf;
    p.ystride = h->ystride;
    p.U = h->U32;
    p.ldu = h->kpad;
    p.V = h->V64;
    p.ldv = h->k;
    p.S = h->S64;
    p.stat = h->stats;
    p.st = h->st;
    const int64_t work = std::max<int64_t>(h->m_g, h->n);
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)h->sms * 8);
    if (h->coll == COLL_NONE) {
        CK(launch_k(h, ext_finish<SRC_PARTS>, blocks, 256, 0, s, 1, p));
    } else if (h->coll == COLL_PEER) {
        CK(launch_k(h, publish, 1, kFinThreads, 0, s, 1, pub_params(h, 1, l)));
        CK(launch_k(h, ext_finish<SRC_PEER>, blocks, 256, 0, s, 1, p));
    } else {
        CK(launch_k(h, ext_reduce, 1, 32, 0, s, 1, (const double *)h->sq_part, h->parts, h->sig2,
                    (const LoopState *)h->st));
        TRY(coll_allreduce(h, h->sig2, 1, true, s));
        ext_finish<SRC_YW><<<blocks, 256, 0, s>>>(p);
    }
    CK(cudaGetLastError());
    return TSVD_OK;
}

// Upload the initial samples x_l of every component once per V0 version.
static tsvd_status upload_v0(tsvd_t h) {
    if (h->v0_uploaded == h->v0_version) return TSVD_OK;
    const int64_t n = h->n;
    if (h->have_V0) {
        CK(cudaMemcpyAsync(h->V0d, h->V0.data(), (size_t)h->k * n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    } else {  // documented generator: splitmix64(seed, l, i) -> two 53-bit uniforms -> Box-Muller
        std::vector<double> x((size_t)h->k * n);
        const double two_pi = 6.283185307179586476925286766559;
        for (int l = 0; l < h->k; ++l) {
            const uint64_t key = splitmix64(splitmix64(h->seed) ^ (uint64_t)l);
            double *xl = x.data() + (size_t)l * n;
            for (int64_t i = 0; i < n; i += 2) {
                const double u1 = (double)(splitmix64(key ^ (uint64_t)i) >> 11) * 0x1.0p-53;
                const double u2 = (double)(splitmix64(key ^ (uint64_t)(i + 1)) >> 11) * 0x1.0p-53;
                const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
                xl[i] = r * std::cos(two_pi * u2);
                if (i + 1 < n) xl[i + 1] = r * std::sin(two_pi * u2);
            }
        }
        CK(cudaMemcpyAsync(h->V0d, x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    h->v0_uploaded = h->v0_version;
    return TSVD_OK;
}

static void drop_graph(tsvd_t h) {
    if (h->exec) cudaGraphExecDestroy(h->exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    h->exec = nullptr;
    h->graph = nullptr;
    h->graph_l0 = -1;
}

// Capture components l0..k-1 as one graph: [init, WHILE(iteration), extraction] per component.
static tsvd_status build_graph(tsvd_t h, int l0) {
#if CUDART_VERSION >= 12040
    drop_graph(h);
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
    tsvd_status s = TSVD_OK;
    cudaError_t ce = cudaSuccess;
    const bool fx = fuse_ext(h);
    const bool ps = use_persist(h);
    if (fx && ps) {  // chain: init, then per component [two-vector pass] + one persistent launch
        for (int l = l0; l < h->k && s >= 0; ++l) {
            s = l == l0 ? launch_init(h, h->stream, l) : launch_two(h, h->stream, l);
            if (s >= 0) s = launch_persist(h, h->stream, l, nullptr, nullptr, l > l0, l + 1 < h->k);
        }
        if (s >= 0) s = launch_extract(h, h->stream, h->k - 1);
    }
    for (int l = l0; l < h->k && s >= 0 && ce == cudaSuccess && !(fx && ps); ++l) {
        if (fx && l > l0) {  // extraction of l-1 rides on the first iteration of l
            s = launch_init_ext(h, h->stream, l);
            if (s >= 0) s = launch_fused_first(h, h->stream, l);
        } else {
            s = launch_init(h, h->stream, l);
        }
        if (s < 0) break;
        if (ps) {  // the iteration loop is one persistent kernel: no conditional node needed
            s = launch_persist(h, h->stream, l);
            if (s < 0) break;
            if (!fx || l == h->k - 1) s = launch_extract(h, h->stream, l);
            continue;
        }
        cudaStreamCaptureStatus cs;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        ce = cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &g, &deps, &nd);
        if (ce) break;
        cudaGraphConditionalHandle ch;
        ce = cudaGraphConditionalHandleCreate(&ch, g, 1, cudaGraphCondAssignDefault);
        if (ce) break;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = ch;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        ce = cudaGraphAddNode(&node, g, deps, nd, &cp);
        if (ce) break;
        ce = cudaStreamUpdateCaptureDependencies(h->stream, &node, 1, cudaStreamSetCaptureDependencies);
        if (ce) break;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        ce = cudaStreamBeginCaptureToGraph(h->body_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
        if (ce) break;
        // the body holds `unroll` iterations: every kernel of an iteration is a no-op once the
        // component is done, so this only saves WHILE-node turnarounds (~8 us each, measured)
        for (int u = 0; u < h->unroll && s >= 0; ++u)
            s = launch_iteration(h, h->body_stream, l, (unsigned long long)ch, 1);
        cudaGraph_t body_out = nullptr;
        cudaError_t ce2 = cudaStreamEndCapture(h->body_stream, &body_out);
        if (s < 0) break;
        ce = ce2;
        if (ce) break;
        if (!fx || l == h->k - 1) s = launch_extract(h, h->stream, l);
    }
    cudaGraph_t graph = nullptr;
    cudaError_t ce3 = cudaStreamEndCapture(h->stream, &graph);
    if (s < 0 || ce || ce3) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        if (s < 0) return s;
        return h->fail(TSVD_ERR_CUDA, "run-graph capture failed: %s", cudaGetErrorString(ce ? ce : ce3));
    }
    h->graph = graph;
    CK(cudaGraphInstantiate(&h->exec, graph, 0));
    h->graph_l0 = l0;
    return TSVD_OK;
#else
    return h->fail(TSVD_ERR_UNSUPPORTED, "CUDA graph conditional nodes need CUDA >= 12.4");
#endif
}

// Host-driven loop: one pinned D2H state read per iteration; optional CUDA events around N1.
// ---------------------------------------------------------------- explicit-Gram path (NEXT#1)
#define CB(x)                                                                                  \
    do {                                                                                       \
        cublasStatus_t cb_ = (x);                                                              \
        if (cb_ != CUBLAS_STATUS_SUCCESS) return h->fail(TSVD_ERR_CUDA, "cuBLAS error %d", (int)cb_); \
    } while (0)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The symmetric task schedule at tile granularity: the 128 x 256 tiles (I, J) that hold
// some (i, j) with j >= i, ordered in groups of 8 I blocks (an A column block is reused by the J
// tiles of its group; the SMs running at the same time share 8 A blocks and ~20 B blocks in L2)
static std::vector<int2> gram_tiles(int64_t n) {
    const int nI = (int)((n + kGtBM - 1) / kGtBM), nJ = (int)((n + kGtBN - 1) / kGtBN);
    std::vector<int2> t;
    for (int I0 = 0; I0 < nI; I0 += 8)
        for (int J = 0; J < nJ; ++J)
            for (int I = I0; I < std::min(nI, I0 + 8); ++I)
                if ((int64_t)kGtBN * J + kGtBN - 1 >= (int64_t)kGtBM * I) t.push_back(make_int2(I, J));
    return t;
}

// the same schedule for the CTA-pair kernel: 256 x 256 tiles (I, J) with J >= I, in groups of 4 I
// blocks (1024 A columns, as above)
static std::vector<int2> gram_tiles2(int64_t n) {
    const int nT = (int)((n + kG2Tile - 1) / kG2Tile);
    std::vector<int2> t;
    for (int I0 = 0; I0 < nT; I0 += 4)
        for (int J = I0; J < nT; ++J)
            for (int I = I0; I < std::min(nT, I0 + 4); ++I)
                if (J >= I) t.push_back(make_int2(I, J));
    return t;
}

// ... and for the A-in-TMEM pair kernel: 256 (M) x 192 (N) tiles touching j >= i
static std::vector<int2> gram_tiles3(int64_t n, int N) {
    const int nI = (int)((n + kG3M - 1) / kG3M), nJ = (int)((n + N - 1) / N);
    std::vector<int2> t;
    for (int I0 = 0; I0 < nI; I0 += 4)
        for (int J = 0; J < nJ; ++J)
            for (int I = I0; I < std::min(nI, I0 + 4); ++I)
                if ((int64_t)N * J + N - 1 >= (int64_t)kG3M * I) t.push_back(make_int2(I, J));
    return t;
}

// B0 = A^T A (Alg. 3's Gram) on the tcgen05 tensor cores, 3xTF32 (gram_tc.cuh), the
// symmetric tile schedule, then the strictly-lower triangle mirrored.  TSVD_GRAM_CUBLAS=1 keeps the
// round-1 path (three cuBLAS TF32 GEMMs of a hi/lo split of A per block product) for A/B timing.
static tsvd_status build_gram_cublas(tsvd_t h);
static tsvd_status build_gram(tsvd_t h) {
    if (getenv("TSVD_GRAM_CUBLAS")) return build_gram_cublas(h);
    auto t0 = std::chrono::steady_clock::now();
    const int64_t m = h->m_g, n = h->n;
    h->ldb0 = round_up(n, 4);
    if (!h->B0) {
        cudaError_t e = cudaMalloc((void **)&h->B0, (size_t)n * h->ldb0 * sizeof(float));
        if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "no room for the n x n Gram");
        CK(e);
        CK(cudaMemsetAsync(h->B0, 0, (size_t)n * h->ldb0 * sizeof(float), h->stream));
    }
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return h->fail(TSVD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = (EncodeTiledFn)fn;
    }
    const bool lo_gmem = getenv("TSVD_GRAM_LO_GMEM") != nullptr;  // A/B: the lo parts as a copy in HBM
    if (lo_gmem && !h->g_lo) {
        cudaError_t e = cudaMalloc((void **)&h->g_lo, (size_t)m * h->ld_use * sizeof(float));
        if (e) {
            cudaGetLastError();
            return h->fail(TSVD_ERR_NOMEM, "no room for the lo copy of A");
        }
    }
    if (lo_gmem) {
        gram_lo_split<<<h->sms * 8, 256, 0, h->stream>>>(h->A_use, m, n, h->ld_use, h->g_lo);
        CK(cudaGetLastError());
    }
    // default: the CTA-pair kernel (gram_tc2).  A/B: TSVD_GRAM_TC=3 (N = 192) / 4 (N = 128, 8 TMEM
    // slots) the pair kernel with A in TMEM
    // (fewer shared-memory bytes, but measured 5-10 % slower: 98 vs 88-93 ms at C2, the box's power
    // cap sets the clock under this tensor load), TSVD_GRAM_TC=1 (or LO_GMEM) the single-CTA kernel
    int variant = 2;
    if (const char *e = getenv("TSVD_GRAM_TC")) variant = atoi(e);
    if (getenv("TSVD_GRAM_TC1") || lo_gmem || h->sms < 2) variant = 1;
    const bool pair = variant >= 2;
    CUtensorMap map, map_lo;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
    const cuuint64_t strides[1] = {(cuuint64_t)h->ld_use * sizeof(float)};
    const cuuint32_t box[2] = {32, (cuuint32_t)(variant == 2 ? kG2BK : kGtBK)};  // 32 columns x the stage's rows
    const cuuint32_t estr[2] = {1, 1};
    for (int w = 0; w < 2; ++w) {
        CUresult r = encode(w ? &map_lo : &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                            (void *)(w && lo_gmem ? h->g_lo : h->A_use), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return h->fail(TSVD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    if (h->gram_n != n || h->gram_pair != variant) {
        const std::vector<int2> tiles = variant == 4 ? gram_tiles3(n, 128) : variant == 3 ? gram_tiles3(n, 192)
                                      : variant == 2 ? gram_tiles2(n) : gram_tiles(n);
        h->gram_pair = variant;
        cudaFree(h->gram_tiles);
        h->gram_tiles = nullptr;
        CK(cudaMalloc((void **)&h->gram_tiles, tiles.size() * sizeof(int2)));
        CK(cudaMemcpy(h->gram_tiles, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice));
        h->gram_ntiles = (int)tiles.size();
        h->gram_n = n;
        CK(cudaFuncSetAttribute(gram_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGtSmem));
        CK(cudaFuncSetAttribute(gram_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGtSmem));
        CK(cudaFuncSetAttribute(gram_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, kG2Smem));
        CK(cudaFuncSetAttribute(gram_tc2, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
        CK(cudaFuncSetAttribute(gram_tc3<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3<192>::Smem));
        CK(cudaFuncSetAttribute(gram_tc3<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3<128>::Smem));
    }
    GtParams p{};
    p.tiles = h->gram_tiles;
    p.ntiles = h->gram_ntiles;
    p.n = n;
    p.ldb = h->ldb0;
    p.m = m;
    p.B = h->B0;
    if (pair) {  // one CTA pair per TPC: an even grid of at most one CTA per SM
        const int G = 2 * std::max(1, std::min(h->sms / 2, h->gram_ntiles));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(kGtThreads);
        cfg.dynamicSmemBytes = variant == 4 ? G3<128>::Smem : variant == 3 ? G3<192>::Smem : kG2Smem;
        cfg.stream = h->stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (variant >= 3) {
            // A half: plain [k][m] boxes of 128 columns x 16 rows (read by the converter, not the MMA)
            CUtensorMap map_a;
            const cuuint32_t box_a[2] = {(cuuint32_t)kG3AHalf, (cuuint32_t)kG3BK};
            CUresult r = encode(&map_a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)h->A_use, dims, strides, box_a, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return h->fail(TSVD_ERR_CUDA, "cuTensorMapEncodeTiled (A half) failed (%d)", (int)r);
            if (variant == 4) CK(cudaLaunchKernelEx(&cfg, gram_tc3<128>, map, map_a, p));
            else CK(cudaLaunchKernelEx(&cfg, gram_tc3<192>, map, map_a, p));
        } else {
            CK(cudaLaunchKernelEx(&cfg, gram_tc2, map, p));
        }
    } else if (lo_gmem) {
        gram_tc<true><<<std::min(h->sms, h->gram_ntiles), kGtThreads, kGtSmem, h->stream>>>(map, map_lo, p);
    } else {
        gram_tc<false><<<std::min(h->sms, h->gram_ntiles), kGtThreads, kGtSmem, h->stream>>>(map, map_lo, p);
    }
    CK(cudaGetLastError());
    const int64_t nb = (n + 31) / 32;
    gram_mirror_to_upper<<<dim3((unsigned)nb, (unsigned)nb), dim3(32, 8), 0, h->stream>>>(h->B0, n, h->ldb0);
    CK(cudaGetLastError());
    h->gram_blocks = h->gram_ntiles;
    if (const char *dump = getenv("TSVD_GRAM_DUMP")) {  // debug: the Gram as n x ldb fp32 (tests, A/B)
        CK(cudaStreamSynchronize(h->stream));
        std::vector<float> hb((size_t)n * h->ldb0);
        CK(cudaMemcpy(hb.data(), h->B0, hb.size() * sizeof(float), cudaMemcpyDeviceToHost));
        if (FILE *f = fopen(dump, "wb")) {
            fwrite(hb.data(), sizeof(float), hb.size(), f);
            fclose(f);
        }
    }
    // row-partitioned A (world > 1): B0 = sum_g A_g^T A_g, one all-reduce over NVLink (Alg. 3's
    // Reduce_sum, as an all-reduce so that every rank iterates on the same B0)
    if (h->world > 1) TRY(coll_allreduce(h, h->B0, (size_t)n * h->ldb0, false, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->B0_ok = true;
    h->gram_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return TSVD_OK;
}

// B0 = A^T A (Alg. 3's Gram) with three TF32 tensor-core GEMMs of the hi/lo split of A:
// A^T A ~= Ah^T Ah + Ah^T Al + Al^T Ah (fp32-level products; cuBLAS for the plain library GEMM).
static tsvd_status build_gram_cublas(tsvd_t h) {
    auto t0 = std::chrono::steady_clock::now();
    const int64_t m = h->m_g, n = h->n;
    h->ldb0 = round_up(n, 4);
    if (!h->B0) {
        cudaError_t e = cudaMalloc((void **)&h->B0, (size_t)n * h->ldb0 * sizeof(float));
        if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "no room for the n x n Gram");
        CK(e);
        CK(cudaMemsetAsync(h->B0, 0, (size_t)n * h->ldb0 * sizeof(float), h->stream));
    }
    if (!h->g_hi) {  // kept for later builds (a new A of the same shape)
        cudaError_t e = cudaMalloc((void **)&h->g_hi, (size_t)m * n * sizeof(float));
        if (!e) e = cudaMalloc((void **)&h->g_lo, (size_t)m * n * sizeof(float));
        if (e) {
            cudaFree(h->g_hi);
            h->g_hi = h->g_lo = nullptr;
            cudaGetLastError();
            return h->fail(TSVD_ERR_NOMEM, "no room for the TF32 split of A");
        }
    }
    float *hi = h->g_hi, *lo = h->g_lo;
    split_tf32<<<h->sms * 8, 256, 0, h->stream>>>(h->A_use, m, n, h->ld_use, hi, lo);
    CK(cudaGetLastError());
    if (!h->cublas) CB(cublasCreate(&h->cublas));
    CB(cublasSetStream(h->cublas, h->stream));
    // column-major view: a row-major m x n slab is an n x m matrix A' (lda = n); A^T A = A' A'^T.
    // Symmetric task schedule: n_b column blocks of A', only the n_b(n_b + 1)/2 block
    // products (I <= J) are formed — each as three TF32 GEMMs of the hi/lo split — and the
    // strictly-lower blocks are mirrored.  n_b is the largest of 1..8 that keeps blocks >= 2048
    // wide (cuBLAS stays efficient).  (Full three GEMMs: 150-162 ms at C2; cuBLAS SYRK + SYR2K in
    // TF32 math mode: 785 ms.)  TSVD_GRAM_NB overrides n_b (A/B experiments).
    const float one = 1.f, zero = 0.f;
    const float *ops[3][2] = {{hi, hi}, {hi, lo}, {lo, hi}};
    int nb = (int)std::max<int64_t>(1, std::min<int64_t>(8, n / 2048));
    if (const char *e = getenv("TSVD_GRAM_NB")) nb = std::max(1, atoi(e));
    const int64_t bs = round_up((n + nb - 1) / nb, 32);
    h->gram_blocks = nb;
    for (int64_t I0 = 0; I0 < n; I0 += bs)
        for (int64_t J0 = I0; J0 < n; J0 += bs) {
            const int64_t bi = std::min(bs, n - I0), bj = std::min(bs, n - J0);
            for (int g = 0; g < 3; ++g)
                CB(cublasGemmEx(h->cublas, CUBLAS_OP_N, CUBLAS_OP_T, (int)bi, (int)bj, (int)m, &one, ops[g][0] + I0,
                                CUDA_R_32F, (int)n, ops[g][1] + J0, CUDA_R_32F, (int)n, g == 0 ? &zero : &one,
                                h->B0 + I0 + J0 * h->ldb0, CUDA_R_32F, (int)h->ldb0, CUBLAS_COMPUTE_32F_FAST_TF32,
                                CUBLAS_GEMM_DEFAULT));
        }
    if (bs < n) {
        const dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
        gram_mirror<<<grid, dim3(32, 8), 0, h->stream>>>(h->B0, n, h->ldb0, bs);
        CK(cudaGetLastError());
    }
    // row-partitioned A (world > 1): B0 = sum_g A_g^T A_g, one all-reduce over NVLink (Alg. 3's
    // Reduce_sum, as an all-reduce so that every rank iterates on the same B0)
    if (h->world > 1) TRY(coll_allreduce(h, h->B0, (size_t)n * h->ldb0, false, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->B0_ok = true;
    h->gram_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return TSVD_OK;
}

// Explicit Gram, world > 1: exchange areas of the row-partitioned iterations (gb_persist): every
// rank's [2][n] stamped y words + [2][world][G][2 + 2k] stamped sums, shared as setup_px does.  On
// any failure every rank falls back to replicated iterations.
static tsvd_status setup_gx(tsvd_t h) {
    if (h->gx_mem || h->world > kMaxRanks || h->k > 129) return TSVD_OK;
    const size_t ny = (size_t)2 * h->n, ns = (size_t)2 * h->world * h->grid_gb * (2 + 2 * h->k);
    CK(cudaMalloc((void **)&h->gx_mem, (ny + ns) * sizeof(ulonglong2)));
    CK(cudaMemsetAsync(h->gx_mem, 0, (ny + ns) * sizeof(ulonglong2), h->stream));
    CK(cudaStreamSynchronize(h->stream));
    void *base[kMaxRanks] = {};
    bool ok = true;
    std::string err;
    TRY(coll_share(h, h->gx_mem, base, h->gx_map, ok, err));
    for (int r = 0; r < h->world; ++r) {
        h->gx_y[r] = (ulonglong2 *)base[r];
        h->gx_s[r] = base[r] ? (ulonglong2 *)base[r] + ny : nullptr;
    }
    int agreed = ok ? 1 : 0;
    TRY(coll_min_int(h, agreed));
    h->gx_ok = agreed == 1 && !getenv("TSVD_GX_REPLICATED");  // env: A/B against replicated iterations
    return TSVD_OK;
}

static tsvd_status run_explicit(tsvd_t h, int l0) {
    if (h->sparse || h->streaming || h->split != 1 || !h->gb)
        return h->fail(TSVD_ERR_UNSUPPORTED, "METHOD=1 (explicit Gram) needs a dense, HBM-resident input "
                                             "with n <= 16384");
    if (l0 > h->pq_l)
        return h->fail(TSVD_ERR_UNSUPPORTED, "METHOD=1 resumes only from factors it computed itself");
    const int64_t n = h->n;
    if (!h->Pm) {
        CK(cudaMalloc((void **)&h->Pm, (size_t)n * h->kpad * sizeof(float)));
        CK(cudaMalloc((void **)&h->Qm, (size_t)h->k * h->k * sizeof(double)));
        CK(cudaMalloc((void **)&h->gpart, (size_t)2 * h->grid_gb * (2 + 2 * h->kpad) * sizeof(double)));
        CK(cudaMalloc((void **)&h->zero64, (size_t)h->kpad * sizeof(double)));
        CK(cudaMemsetAsync(h->Pm, 0, (size_t)n * h->kpad * sizeof(float), h->stream));
        CK(cudaMemsetAsync(h->Qm, 0, (size_t)h->k * h->k * sizeof(double), h->stream));
        CK(cudaMemsetAsync(h->zero64, 0, (size_t)h->kpad * sizeof(double), h->stream));
    }
    if (!h->B0_ok) TRY(build_gram(h));
    if (h->world > 1) TRY(setup_gx(h));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->timing) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
    }
    for (int l = l0; l < h->k; ++l) {
        TRY(launch_init(h, h->stream, l));  // x -> y_cur, ||x||
        GbParams g{};
        g.B = h->B0;
        g.ldb = h->ldb0;
        g.rows = n;
        g.row0 = 0;
        g.world = 1;
        if (h->world > 1 && h->gx_ok) {  // rows [n r / W, n (r + 1) / W) of B0 on rank r
            g.row0 = n * h->rank / h->world;
            g.rows = n * (h->rank + 1) / h->world - g.row0;
            g.world = h->world;
            g.rank = h->rank;
            for (int r = 0; r < h->world; ++r) {
                g.yx[r] = h->gx_y[r];
                g.sx[r] = h->gx_s[r];
            }
        }
        g.n = (int32_t)n;
        g.n4 = (int32_t)((n + 3) / 4);
        g.P = h->Pm;
        g.ldp = h->kpad;
        g.V = h->V64;
        g.ldv = h->k;
        g.S = h->S64;
        g.Q = h->Qm;
        g.ldq = h->k;
        g.l = l;
        g.stages = h->S_gb;
        g.stage_bytes = h->stage_bytes;
        g.row_bytes = h->row_bytes;
        g.ybuf = h->ybuf;
        g.ystride = h->ystride;
        g.st = h->st;
        g.c = h->c64;
        g.part = h->gpart;
        g.part_ld = 2 + 2 * h->kpad;
        g.gbar = h->gbar;
        g.eps = h->eps;
        g.fixed_T = h->fixed_T;
        g.max_iter = h->max_iter;
        g.serpentine = h->serp_opt;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.gridDim = dim3(h->grid_gb);
        cfg.blockDim = dim3(h->T);
        cfg.dynamicSmemBytes = h->smem_gb;
        cfg.stream = h->stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (e0) CK(cudaEventRecord(e0, h->stream));
        CK(cudaLaunchKernelEx(&cfg, h->gb, g));
        if (e1) CK(cudaEventRecord(e1, h->stream));
        // extraction + the new columns of P = A^T U and Q = U^T U: one fused pass, c = 0
        GvParams q = gv_params(h, l, false);
        q.c = h->zero64;
        q.store_t = 1;
        q.reduce_mode = 0;  // partials stay per CTA (world > 1: reduced and all-reduced below)
        q.tl = nullptr;
        q.trace = nullptr;
        CK(launch_n1(h, h->gv, q, h->stream));
        GxParams x{};
        x.rows = h->m_g;
        x.n = n;
        x.l = l;
        x.parts = h->parts;
        x.ldu = h->kpad;
        x.ldp = h->kpad;
        x.ldv = h->k;
        x.ldq = h->k;
        x.u_out = h->u64;
        x.ypart = h->ypart;
        x.wpart = h->wpart;
        x.sq_part = h->sq_part;
        x.ypart_ld = h->ypart_ld;
        x.wpart_ld = h->kpad;
        x.ybuf = h->ybuf;
        x.ystride = h->ystride;
        x.U = h->U32;
        x.P = h->Pm;
        x.V = h->V64;
        x.S = h->S64;
        x.Q = h->Qm;
        x.stat = h->stats;
        x.st = h->st;
        const int blocks = (int)std::min<int64_t>((std::max(h->m_g, n) + 255) / 256, (int64_t)h->sms * 8);
        if (h->world > 1) {  // [A_g^T u | U_g^T u | ||u_g||^2] summed over the ranks; identical on every rank
            CK(launch_k(h, gx_reduce, (int)std::min<int64_t>((n + l + 256) / 256, (int64_t)h->sms * 8), 256, 0,
                        h->stream, 1, x, h->yw, h->wofs));
            TRY(coll_allreduce(h, h->yw, (size_t)(h->wofs + h->kpad), true, h->stream));
            x.parts = 1;
            x.ypart = h->yw;
            x.ypart_ld = 0;
            x.wpart = h->yw + h->wofs;
            x.wpart_ld = 0;
            x.sq_part = h->yw + h->wofs + l;
        }
        CK(launch_k(h, gram_ext_finish, blocks, 256, 0, h->stream, 1, x));
        CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (getenv("TSVD_GRP_DEBUG"))
            fprintf(stderr, "[explicit rank %d component %d done: it %d status %d t %.3f]\n", h->rank, l,
                    h->st_host->it, h->st_host->status,
                    std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count());
        if (h->timing) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            h->ps_ms += ms;
            h->ps_launches += 1;
        }
        if (h->st_host->stop) break;
        h->pq_l = l + 1;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    h->loop_mode = h->timing ? "explicit-gram+events" : "explicit-gram";
    return TSVD_OK;
}

static tsvd_status run_host_loop(tsvd_t h, int l0) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->timing) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
    }
    const bool fx = fuse_ext(h);
    const bool ps = use_persist(h);
    if (fx && ps) {  // chain (as in the graph): one synchronisation per component
        for (int l = l0; l < h->k; ++l) {
            if (l == l0) TRY(launch_init(h, h->stream, l));
            else TRY(launch_two(h, h->stream, l));
            TRY(launch_persist(h, h->stream, l, e0, e1, l > l0, l + 1 < h->k));
            CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (h->timing) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                h->ps_ms += ms;
                h->ps_launches += 1;
            }
            if (h->st_host->stop) break;
        }
        if (!h->st_host->stop) TRY(launch_extract(h, h->stream, h->k - 1));
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        h->loop_mode = h->timing ? "host+events" : "host";
        return TSVD_OK;
    }
    for (int l = l0; l < h->k; ++l) {
        const bool fused_first = fx && l > l0;
        if (fused_first) TRY(launch_init_ext(h, h->stream, l));
        else TRY(launch_init(h, h->stream, l));
        if (ps) {  // fused first pass (if any), then the remaining iterations in one launch
            if (fused_first) TRY(launch_fused_first(h, h->stream, l));
            TRY(launch_persist(h, h->stream, l, e0, e1));
            CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (h->timing) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                h->ps_ms += ms;
                h->ps_launches += 1;
            }
            if (!fx || l == h->k - 1) TRY(launch_extract(h, h->stream, l));
            CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (h->st_host->stop) break;
            continue;
        }
        for (int pass = 0;; ++pass) {
            if (fused_first && pass == 0) TRY(launch_fused_first(h, h->stream, l, e0, e1));
            else TRY(launch_iteration(h, h->stream, l, 0ull, 0, e0, e1));
            CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (h->timing && !h->st_host->stop) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                h->n1_ms += ms;
                h->n1_launches += 1;
            }
            if (h->trace_d && h->trace_f) {  // debug: per-CTA timestamps of this N1 launch
                std::vector<unsigned long long> tr((size_t)h->grid * 4);
                CK(cudaMemcpy(tr.data(), h->trace_d, tr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                unsigned long long t0 = tr[0];
                for (int b = 0; b < h->grid; ++b) t0 = std::min(t0, tr[b * 4]);
                for (int b = 0; b < h->grid; ++b)
                    fprintf(h->trace_f, "%d,%lld,%d,%lld,%lld,%lld,%lld\n", h->rank, (long long)h->trace_launch, b,
                            (long long)(tr[b * 4] - t0), (long long)(tr[b * 4 + 1] - t0),
                            (long long)(tr[b * 4 + 2] - t0), (long long)(tr[b * 4 + 3] - t0));
                h->trace_launch++;
            }
            if (h->st_host->done || h->st_host->stop) break;
        }
        if (!fx || l == h->k - 1) TRY(launch_extract(h, h->stream, l));
        CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (h->st_host->stop) break;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    h->loop_mode = h->timing ? "host+events" : "host";
    return TSVD_OK;
}

// ------------------------------------------------------------------------------------ ABI
extern "C" {

tsvd_status tsvd_create(tsvd_t *out, int64_t m, int64_t n, int32_t k, double eps, tsvd_dtype dtype,
                        tsvd_layout layout) {
    if (!out) {
        g_err = "out == NULL";
        return TSVD_ERR_ARG;
    }
    *out = nullptr;
    const int64_t mn = std::min(m, n);
    if (m < 1 || n < 1 || k == 0 || k < -1 || (k > 0 && k > mn) || !(eps > 0.0 && eps < 1.0)) {
        g_err = "bad arguments: need m,n >= 1, k in [1, min(m,n)] or -1, 0 < eps < 1";
        return TSVD_ERR_ARG;
    }
    if (dtype != TSVD_F32) {
        g_err = "only fp32 in this version";
        return TSVD_ERR_UNSUPPORTED;
    }
    if (layout != TSVD_ROW_MAJOR && layout != TSVD_COL_MAJOR) {
        g_err = "layout must be TSVD_ROW_MAJOR or TSVD_COL_MAJOR";
        return TSVD_ERR_ARG;
    }
    const int64_t kk = k == -1 ? mn : k;
    if (kk > kMaxK) {
        g_err = "k > 4096 is not supported";
        return TSVD_ERR_UNSUPPORTED;
    }
    tsvd_t h = new tsvd_s();
    h->m_user = m;
    h->n_user = n;
    h->wide = m < n;
    h->layout = layout;
    // the internal problem is always tall (rows >= columns, V-first); it is stored row-major in
    // place when the user's major dimension is its row dimension, else through a transposed copy
    h->tcopy = (layout == TSVD_ROW_MAJOR) == h->wide;
    if (h->wide) std::swap(m, n);  // internal tall problem: A^T, n x m
    h->m = m;
    h->n = n;
    h->k = (int32_t)kk;
    h->kpad = (int32_t)round_up(h->k, 4);
    h->eps = eps;
    h->row_begin = 0;
    h->row_end = m;
    h->m_g = m;
    h->iters.assign(h->k, 0);
    h->dots.assign(h->k, 0.0);
    if (const char *c = getenv("TSVD_CARVEOUT")) h->carveout_opt = atoi(c);
    cudaError_t e = cudaGetDevice(&h->dev);
    if (!e) e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev);
    if (!e) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (!e) e = cudaStreamCreateWithFlags(&h->body_stream, cudaStreamNonBlocking);
    if (e) {
        g_err = std::string("CUDA: ") + cudaGetErrorString(e);
        delete h;
        return TSVD_ERR_CUDA;
    }
    *out = h;
    return TSVD_OK;
}

tsvd_status tsvd_get_inproc_id(void *out128) {
    if (!out128) return TSVD_ERR_ARG;
    static std::mutex mu;
    static unsigned long long counter = 0;
    unsigned long long c;
    {
        std::lock_guard<std::mutex> lk(mu);
        c = ++counter;
    }
    unsigned char id[128] = {};
    memcpy(id, kInprocMagic, sizeof(kInprocMagic));
    const unsigned long long t = (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count();
    memcpy(id + 16, &c, sizeof(c));
    memcpy(id + 24, &t, sizeof(t));
    memcpy(out128, id, sizeof(id));
    return TSVD_OK;
}

tsvd_status tsvd_get_unique_id(void *out128) {
    if (!out128) return TSVD_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return TSVD_ERR_NCCL;
    memcpy(out128, &id, sizeof(id));
    return TSVD_OK;
}

tsvd_status tsvd_set_comm(tsvd_t h, int32_t rank, int32_t world, const void *uid, int32_t device) {
    if (!h) return TSVD_ERR_ARG;
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world || (world > 1 && !uid))
        return h->fail(TSVD_ERR_ARG, "bad rank/world (world <= %d)", kMaxRanks);
    if (h->allocated || h->have_A) return h->fail(TSVD_ERR_STATE, "set_comm must precede set_dense");
    if (h->tcopy && world > 1)
        return h->fail(TSVD_ERR_UNSUPPORTED, "row-major wide (or column-major tall) inputs run on one GPU; pass a "
                                             "wide matrix column-major to partition its columns (CSVD, P:323)");
    if (device != h->dev) {
        CK(cudaSetDevice(device));
        if (h->stream) cudaStreamDestroy(h->stream);
        if (h->body_stream) cudaStreamDestroy(h->body_stream);
        h->dev = device;
        CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev));
        if (h->sm_limit > 0) h->sms = std::min(h->sms, h->sm_limit);
        CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->body_stream, cudaStreamNonBlocking));
    }
    h->rank = rank;
    h->world = world;
    h->coll = COLL_NONE;
    if (world > 1) {
        if (memcmp(uid, kInprocMagic, sizeof(kInprocMagic)) == 0) {  // in-process ranks (tsvd_get_inproc_id)
            if (h->coll_opt != 0)
                return h->fail(TSVD_ERR_UNSUPPORTED, "in-process ranks run the peer collective (COLLECTIVE = 0)");
            const std::string key((const char *)uid, 128);
            std::lock_guard<std::mutex> lk(g_grp_mu);
            for (auto it = g_grps.begin(); it != g_grps.end();)  // groups whose handles are all gone
                it = it->second.expired() ? g_grps.erase(it) : std::next(it);
            std::shared_ptr<InprocGroup> g = g_grps[key].lock();
            if (!g) {
                g = std::make_shared<InprocGroup>();
                g->world = world;
                g->v.assign(world, 0);
                g->p.assign(world, nullptr);
                g_grps[key] = g;
            }
            if (g->world != world) return h->fail(TSVD_ERR_ARG, "in-process group of %d ranks, not %d", g->world, world);
            h->grp = g;
        } else {
            ncclUniqueId id;
            memcpy(&id, uid, sizeof(id));
            NK(ncclCommInitRank(&h->comm, world, id, rank));
        }
        // every rank takes part in the handle exchange, then all agree on the collective to use
        const tsvd_status ps = setup_peer(h);
        int ok = (ps == TSVD_OK) ? 1 : 0;
        TRY(coll_min_int(h, ok));
        if (!ok && h->grp) return h->fail(TSVD_ERR_CUDA, "in-process group: %s", h->peer_error.c_str());
        h->coll = (ok && h->coll_opt == 0) ? COLL_PEER : COLL_NCCL;
    }
    return TSVD_OK;
}

tsvd_status tsvd_set_option(tsvd_t h, int32_t key, int64_t value) {
    if (!h) return TSVD_ERR_ARG;
    switch (key) {
    case TSVD_OPT_MAX_ITER:
        if (value < 1 || value > INT32_MAX) return h->fail(TSVD_ERR_ARG, "MAX_ITER must be >= 1");
        h->max_iter = (int)value;
        break;
    case TSVD_OPT_FIXED_ITERS:
        if (value < 0 || value > INT32_MAX) return h->fail(TSVD_ERR_ARG, "FIXED_ITERS must be >= 0");
        h->fixed_T = (int)value;
        break;
    case TSVD_OPT_SEED:
        h->seed = (uint64_t)value;
        if (!h->have_V0) h->v0_version++;
        break;
    case TSVD_OPT_GRAPH: h->use_graph = value != 0; break;
    case TSVD_OPT_TIMING: h->timing = value != 0; break;
    case TSVD_OPT_RUN_ROWS:
        if (value < 1 || value > INT32_MAX) return h->fail(TSVD_ERR_ARG, "RUN_ROWS must be >= 1");
        h->run_rows = (int)value;
        break;
    case TSVD_OPT_CTAS_PER_SM:
        if (value < 0 || value > 32) return h->fail(TSVD_ERR_ARG, "CTAS_PER_SM in [0, 32]");
        if (h->allocated) return h->fail(TSVD_ERR_STATE, "CTAS_PER_SM must precede the first run");
        h->cps_opt = (int)value;
        break;
    case TSVD_OPT_COLLECTIVE:
        if (value < 0 || value > 1) return h->fail(TSVD_ERR_ARG, "COLLECTIVE is 0 (peer) or 1 (nccl)");
        h->coll_opt = (int)value;
        if (h->world > 1) h->coll = (value == 1 || !h->sym || !h->pv.flags) ? COLL_NCCL : COLL_PEER;
        break;
    case TSVD_OPT_FUSED_REDUCE:
        h->fused_opt = value != 0;
        break;
    case TSVD_OPT_DETERMINISTIC:
        h->dynamic_opt = value == 0;
        break;
    case TSVD_OPT_GRAPH_UNROLL:
        if (value < 1 || value > 8) return h->fail(TSVD_ERR_ARG, "GRAPH_UNROLL in 1..8");
        h->unroll = (int)value;
        break;
    case TSVD_OPT_FUSED_EXTRACT:
        h->fuse_ext_opt = value != 0;
        break;
    case TSVD_OPT_PDL:
        h->pdl_opt = value != 0;
        break;
    case TSVD_OPT_ROW_ORDER:
        h->serp_opt = value != 0;
        break;
    case TSVD_OPT_PERSISTENT:
        h->persist_opt = value != 0;
        break;
    case TSVD_OPT_V_PLACEMENT:
        if (value < 0 || value > 1) return h->fail(TSVD_ERR_ARG, "V_PLACEMENT is 0 (HBM) or 1 (host)");
        if (h->allocated) return h->fail(TSVD_ERR_STATE, "V_PLACEMENT must precede the first run");
        h->v_host = (int)value;
        break;
    case TSVD_OPT_SM_LIMIT: {
        if (value < 0 || value > INT32_MAX) return h->fail(TSVD_ERR_ARG, "SM_LIMIT must be >= 0");
        if (h->allocated || h->have_A) return h->fail(TSVD_ERR_STATE, "SM_LIMIT must precede set_dense / set_csr");
        int dev_sms = 0;
        CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->dev));
        h->sm_limit = (int)value;
        h->sms = value > 0 ? std::min<int>(dev_sms, (int)value) : dev_sms;
        break;
    }
    case TSVD_OPT_METHOD:
        if (value < 0 || value > 1) return h->fail(TSVD_ERR_ARG, "METHOD in 0..1");
        h->method = (int)value;
        break;
    case TSVD_OPT_SPARSE_BLOCK:
        if (value < 0) return h->fail(TSVD_ERR_ARG, "SPARSE_BLOCK >= 0");
        h->sp_block_opt = value;
        break;
    case TSVD_OPT_PLACEMENT:
    case TSVD_OPT_RESIDENT_BYTES:
    case TSVD_OPT_BATCH_ROWS:
    case TSVD_OPT_QUEUE_DEPTH:
        if (key == TSVD_OPT_PLACEMENT && (value < 0 || value > 2)) return h->fail(TSVD_ERR_ARG, "PLACEMENT in 0..2");
        if (key == TSVD_OPT_RESIDENT_BYTES && value < -1) return h->fail(TSVD_ERR_ARG, "RESIDENT_BYTES >= -1");
        if (key == TSVD_OPT_BATCH_ROWS && value < 0) return h->fail(TSVD_ERR_ARG, "BATCH_ROWS >= 0");
        if (key == TSVD_OPT_QUEUE_DEPTH && (value < 1 || value > 8)) return h->fail(TSVD_ERR_ARG, "QUEUE_DEPTH in 1..8");
        if (key == TSVD_OPT_PLACEMENT) h->placement = (int)value;
        if (key == TSVD_OPT_RESIDENT_BYTES) h->resident_cap = value;
        if (key == TSVD_OPT_BATCH_ROWS) h->batch_rows_opt = value;
        if (key == TSVD_OPT_QUEUE_DEPTH) h->qdepth = (int)value;
        if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
        if (h->stream) cudaStreamSynchronize(h->stream);
        free_ring(h);
        h->own_rows = 0;  // re-decide the placement at the next staging
        break;
    default: return h->fail(TSVD_ERR_ARG, "unknown option %d", key);
    }
    h->graph_l0 = -1;  // options are baked into the captured kernel parameters
    return TSVD_OK;
}

tsvd_status tsvd_set_init(tsvd_t h, const double *V0) {
    if (!h) return TSVD_ERR_ARG;
    if (!V0) return h->fail(TSVD_ERR_ARG, "V0 == NULL");
    h->V0.assign(V0, V0 + (size_t)h->k * h->n);
    h->have_V0 = true;
    h->v0_version++;
    return TSVD_OK;
}

static tsvd_status set_dense_impl(tsvd_t h, const float *A, int64_t ld, int64_t row_begin, int64_t row_end,
                                  tsvd_mem mem);

// A^T into the handle's own buffer (n_user x round4(m_user)), from device or host A
__global__ void transpose_f32(const float *__restrict__ in, int64_t rows, int64_t cols, int64_t ldi,
                              float *__restrict__ out, int64_t ldo) {
    __shared__ float tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * ldi + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;  // out row = input column
        if (r < rows && c < cols) out[c * ldo + r] = tile[threadIdx.x][i];
    }
}

tsvd_status tsvd_set_dense(tsvd_t h, const float *A, int64_t ld, int64_t row_begin, int64_t row_end, tsvd_mem mem) {
    if (!h) return TSVD_ERR_ARG;
    // in place: the user's buffer IS the internal tall matrix, row-major (row-major tall A, or
    // column-major wide A = row-major A^T whose rows are A's columns; ranges count the major dimension)
    if (!h->tcopy) return set_dense_impl(h, A, ld, row_begin, row_end, mem);
    // transposed copy: the user's buffer is mu x nu row-major (mu < nu: row-major wide A; mu > nu:
    // column-major tall A viewed as its row-major transpose) and the tall solver runs on its transpose
    const int64_t mu = h->wide ? h->m_user : h->n_user, nu = h->wide ? h->n_user : h->m_user;
    if (!A || ld < nu) return h->fail(TSVD_ERR_ARG, "A == NULL or ld < the major dimension");
    if (row_begin != 0 || row_end != mu)
        return h->fail(TSVD_ERR_SHAPE, "this layout is passed whole (range [0, %lld))", (long long)mu);
    if (mem != TSVD_MEM_DEVICE && mem != TSVD_MEM_HOST_PINNED && mem != TSVD_MEM_HOST_PAGEABLE)
        return h->fail(TSVD_ERR_ARG, "bad mem kind");
    if (h->sparse) return h->fail(TSVD_ERR_STATE, "the input kind cannot change");
    CK(cudaSetDevice(h->dev));
    const int64_t ldt = round_up(mu, 4);
    if (!h->At) {
        cudaError_t e = cudaMalloc((void **)&h->At, (size_t)nu * ldt * sizeof(float));
        if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "no room for the transposed copy of A");
        CK(e);
        CK(cudaMemsetAsync(h->At, 0, (size_t)nu * ldt * sizeof(float), h->stream));
    }
    const float *src = A;
    float *tmp = nullptr;
    int64_t lds = ld;
    if (mem != TSVD_MEM_DEVICE) {  // stage the host matrix once, then transpose on the device
        cudaError_t e = cudaMalloc((void **)&tmp, (size_t)mu * nu * sizeof(float));
        if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "no room to stage the wide input");
        CK(e);
        CK(cudaMemcpy2DAsync(tmp, nu * sizeof(float), A, ld * sizeof(float), nu * sizeof(float), mu,
                             cudaMemcpyHostToDevice, h->stream));
        src = tmp;
        lds = nu;
    }
    dim3 grid((unsigned)((nu + 31) / 32), (unsigned)((mu + 31) / 32));
    transpose_f32<<<grid, dim3(32, 8), 0, h->stream>>>(src, mu, nu, lds, h->At, ldt);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    if (tmp) cudaFree(tmp);
    return set_dense_impl(h, h->At, ldt, 0, nu, TSVD_MEM_DEVICE);
}

static tsvd_status set_dense_impl(tsvd_t h, const float *A, int64_t ld, int64_t row_begin, int64_t row_end,
                                  tsvd_mem mem) {
    if (!A || ld < h->n) return h->fail(TSVD_ERR_ARG, "A == NULL or ld < n");
    if (row_begin < 0 || row_end > h->m || row_end <= row_begin)
        return h->fail(TSVD_ERR_SHAPE, "row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                       (long long)row_end, (long long)h->m);
    if (mem != TSVD_MEM_DEVICE && mem != TSVD_MEM_HOST_PINNED && mem != TSVD_MEM_HOST_PAGEABLE)
        return h->fail(TSVD_ERR_ARG, "bad mem kind");
    CK(cudaSetDevice(h->dev));
    if (h->allocated && ((row_end - row_begin) != h->m_g || h->sparse))
        return h->fail(TSVD_ERR_STATE, "the input kind / slab size cannot change after the first run");
    h->sparse = false;
    h->row_begin = row_begin;
    h->row_end = row_end;
    h->m_g = row_end - row_begin;
    h->A_user = A;
    h->ld_user = ld;
    h->mem = mem;
    h->have_A = true;
    h->graph_l0 = -1;
    h->B0_ok = false;  // explicit path: the Gram of the new A is built at the next run
    h->pq_l = 0;
    if (mem == TSVD_MEM_DEVICE) {
        const bool aligned = ((uintptr_t)A % 16 == 0) && (ld % 4 == 0);
        if (aligned) {
            h->A_use = A;
            h->ld_use = ld;
        } else {  // pack once into a 16-B aligned, ld % 4 == 0 copy (TMA bulk-copy alignment)
            const int64_t ldp = round_up(h->n, 4);
            if (h->A_own) cudaFree(h->A_own);
            h->A_own = nullptr;
            cudaError_t e = cudaMalloc((void **)&h->A_own, (size_t)h->m_g * ldp * sizeof(float));
            if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "no room for an aligned copy of A");
            CK(e);
            CK(cudaMemsetAsync(h->A_own, 0, (size_t)h->m_g * ldp * sizeof(float), h->stream));
            CK(cudaMemcpy2DAsync(h->A_own, ldp * sizeof(float), A, ld * sizeof(float), h->n * sizeof(float), h->m_g,
                                 cudaMemcpyDeviceToDevice, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            h->ld_own = ldp;
            h->A_use = h->A_own;
            h->ld_use = ldp;
        }
    }
    return TSVD_OK;
}

// device array owned by the sparse views (freed by free_sparse)
static cudaError_t sp_alloc(tsvd_t h, void **p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) {
        h->sp_mem.push_back(*p);
        h->sp_bytes += (int64_t)bytes;
    }
    return e;
}

// exclusive scan of K x segs counts into flat[0 .. len] (flat[len] = total), int64
static tsvd_status sp_scan(tsvd_t h, const unsigned *cnt, int64_t len, int64_t *flat) {
    const int64_t ntiles = (len + kScanTile - 1) / kScanTile;
    int64_t *bsum = nullptr;
    CK(cudaMalloc((void **)&bsum, (size_t)std::max<int64_t>(ntiles, 1) * sizeof(int64_t)));
    if (len > 0) {
        scan_tiles<<<(int)ntiles, kScanThreads, 0, h->stream>>>(cnt, len, flat, bsum);
        scan_totals<<<1, kScanThreads, 0, h->stream>>>(bsum, ntiles, flat + len);
        scan_add<<<h->sms * 8, 256, 0, h->stream>>>(flat, len, bsum);
    } else {
        CK(cudaMemsetAsync(flat, 0, sizeof(int64_t), h->stream));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(bsum);
    return TSVD_OK;
}

// SELL-32-sigma view of one direction from its entry counts cnt[K][segs] (N4b): sort every window's
// segments by length, slice sizes, scan, int32 block-local slice offsets + int64 block bases, and the
// padded entry arrays (idx = -1 / val = 0 where a lane's segment is shorter than its slice).  Leaves the
// flat slice scan (flat_sl, [K][nsl] + 1) and the inverse positions (ipos, [K][segs]) for the caller's
// scatter (caller frees).  TSVD_ERR_UNSUPPORTED if a block holds 2^31 or more (padded) entries.
static tsvd_status sell_view(tsvd_t h, const unsigned *cnt, int K, int64_t segs, SpView *v, int64_t **flat_sl,
                             int32_t **ipos) {
    const int64_t nsl = (segs + 31) / 32, len = (int64_t)K * nsl;
    int32_t *perm = nullptr, *soff = nullptr;
    int64_t *base = nullptr;
    unsigned *ssize = nullptr;
    *flat_sl = nullptr;
    *ipos = nullptr;
    cudaError_t e = sp_alloc(h, (void **)&perm, (size_t)K * segs * sizeof(int32_t));
    if (!e) e = cudaMalloc((void **)ipos, std::max<size_t>((size_t)K * segs * sizeof(int32_t), 16));
    if (!e) e = cudaMalloc((void **)&ssize, std::max<size_t>((size_t)len * sizeof(unsigned), 16));
    if (!e) e = cudaMalloc((void **)flat_sl, (size_t)(len + 1) * sizeof(int64_t));
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        cudaFree(ssize);
        return h->fail(TSVD_ERR_NOMEM, "sparse layout: no room for the slice tables");
    }
    CK(e);
    if (segs > 0) {
        const dim3 grid((unsigned)((segs + kSellW - 1) / kSellW), (unsigned)K);
        sell_sort<<<grid, kSellW, 0, h->stream>>>(cnt, segs, perm, *ipos, ssize, nsl);
        CK(cudaGetLastError());
    }
    tsvd_status st = sp_scan(h, ssize, len, *flat_sl);
    cudaFree(ssize);
    if (st != TSVD_OK) return st;
    // blocks 0 .. K-2 carry their sums to the next block: perm -> the next block's positions (the
    // layout itself is built from ipos, which keeps every block's own positions)
    if (K > 1 && segs > 0) {
        sell_next<<<h->sms * 8, 256, 0, h->stream>>>(perm, *ipos, K, segs);
        CK(cudaGetLastError());
    }
    std::vector<int64_t> starts(K + 1);
    for (int b = 0; b <= K; ++b)
        CK(cudaMemcpy(&starts[b], *flat_sl + (int64_t)b * nsl, sizeof(int64_t), cudaMemcpyDeviceToHost));
    for (int b = 0; b < K; ++b)
        if (starts[b + 1] - starts[b] > (int64_t)INT32_MAX) return TSVD_ERR_UNSUPPORTED;
    e = sp_alloc(h, (void **)&soff, (size_t)K * (nsl + 1) * sizeof(int32_t));
    if (!e) e = sp_alloc(h, (void **)&base, (size_t)(K + 1) * sizeof(int64_t));
    int32_t *sidx = nullptr;
    float *sval = nullptr;
    const int64_t total = starts[K];
    if (!e) e = sp_alloc(h, (void **)&sidx, (size_t)total * sizeof(int32_t));
    if (!e) e = sp_alloc(h, (void **)&sval, (size_t)total * sizeof(float));
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return h->fail(TSVD_ERR_NOMEM, "sparse layout: no room for the sliced entries (%lld)", (long long)total);
    }
    CK(e);
    CK(cudaMemsetAsync(sidx, 0xFF, (size_t)total * sizeof(int32_t), h->stream));  // padding: idx = -1
    CK(cudaMemsetAsync(sval, 0, (size_t)total * sizeof(float), h->stream));
    flat_to_off<<<h->sms * 8, 256, 0, h->stream>>>(*flat_sl, K, nsl, soff, base);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    v->soff = soff;
    v->base = base;
    v->perm = perm;
    v->idx = sidx;
    v->val = sval;
    v->segs = segs;
    v->nsl = nsl;
    return TSVD_OK;
}

// N4b (CSR by column block): per row, the entries of block b (columns [b bw, (b + 1) bw)) are a
// contiguous piece of the row; counted by binary search, then written straight into the SELL layout
static tsvd_status build_csr_view(tsvd_t h, int K, int64_t bw) {
    const int64_t mg = h->m_g;
    unsigned *cnt = nullptr;
    CK(cudaMalloc((void **)&cnt, std::max<size_t>((size_t)K * mg * sizeof(unsigned), 16)));
    blk_count<<<h->sms * 8, 256, 0, h->stream>>>(h->row_ptr_d, h->col_d, mg, K, bw, cnt);
    CK(cudaGetLastError());
    int64_t *flat_sl = nullptr;
    int32_t *ipos = nullptr;
    tsvd_status st = sell_view(h, cnt, K, mg, &h->spc, &flat_sl, &ipos);
    if (st == TSVD_OK && h->nnz_g > 0) {
        sell_from_csr<<<h->sms * 8, 256, 0, h->stream>>>(h->row_ptr_d, h->col_d, h->val_d, mg, K, cnt, ipos, flat_sl,
                                                         h->spc.nsl, const_cast<int32_t *>(h->spc.idx),
                                                         const_cast<float *>(h->spc.val));
        if (cudaGetLastError() != cudaSuccess) st = h->fail(TSVD_ERR_CUDA, "sell_from_csr launch failed");
        else if (cudaStreamSynchronize(h->stream) != cudaSuccess) st = h->fail(TSVD_ERR_CUDA, "sell_from_csr failed");
    }
    cudaFree(cnt);
    cudaFree(flat_sl);
    cudaFree(ipos);
    return st;
}

// N4 (CSC by row block, straight from the CSR): counts per [row block][column], scan, scatter into a
// compact temporary, each (block, column) segment sorted by row (so the layout — and every result —
// is deterministic), then the SELL layout
static tsvd_status build_csc_view(tsvd_t h, int K, int64_t bw) {
    const int64_t mg = h->m_g, n = h->n, nnz = h->nnz_g;
    const int64_t len = (int64_t)K * n;
    unsigned *cnt = nullptr, *fill = nullptr;
    int64_t *flat = nullptr;
    int32_t *cidx = nullptr;
    float *cval = nullptr;
    cudaError_t e = cudaMalloc((void **)&cnt, std::max<size_t>((size_t)len * sizeof(unsigned), 16));
    if (!e) e = cudaMalloc((void **)&fill, std::max<size_t>((size_t)len * sizeof(unsigned), 16));
    if (!e) e = cudaMalloc((void **)&flat, (size_t)(len + 1) * sizeof(int64_t));
    if (!e) e = cudaMalloc((void **)&cidx, std::max<size_t>((size_t)nnz * sizeof(int32_t), 16));
    if (!e) e = cudaMalloc((void **)&cval, std::max<size_t>((size_t)nnz * sizeof(float), 16));
    tsvd_status st = TSVD_OK;
    if (e) {
        cudaGetLastError();
        st = h->fail(e == cudaErrorMemoryAllocation ? TSVD_ERR_NOMEM : TSVD_ERR_CUDA, "CSC build: %s",
                     cudaGetErrorString(e));
    }
    if (st == TSVD_OK) {
        cudaMemsetAsync(cnt, 0, (size_t)len * sizeof(unsigned), h->stream);
        cudaMemsetAsync(fill, 0, (size_t)len * sizeof(unsigned), h->stream);
        if (nnz) csc_blk_count<<<h->sms * 8, 256, 0, h->stream>>>(h->row_ptr_d, h->col_d, mg, n, bw, cnt);
        st = sp_scan(h, cnt, len, flat);
    }
    if (st == TSVD_OK && nnz) {
        csc_blk_scatter<<<h->sms * 8, 256, 0, h->stream>>>(h->row_ptr_d, h->col_d, h->val_d, mg, n, bw, flat, fill,
                                                           cidx, cval);
        csc_sort<<<h->sms * 8, 256, 0, h->stream>>>(flat, len, cidx, cval);
        if (cudaGetLastError() != cudaSuccess) st = h->fail(TSVD_ERR_CUDA, "CSC scatter / sort launch failed");
    }
    cudaFree(fill);
    int64_t *flat_sl = nullptr;
    int32_t *ipos = nullptr;
    if (st == TSVD_OK) st = sell_view(h, cnt, K, n, &h->spr, &flat_sl, &ipos);
    if (st == TSVD_OK && nnz) {
        sell_from_flat<<<h->sms * 8, 256, 0, h->stream>>>(flat, cidx, cval, K, n, ipos, flat_sl, h->spr.nsl,
                                                          const_cast<int32_t *>(h->spr.idx),
                                                          const_cast<float *>(h->spr.val));
        if (cudaGetLastError() != cudaSuccess) st = h->fail(TSVD_ERR_CUDA, "sell_from_flat launch failed");
        else if (cudaStreamSynchronize(h->stream) != cudaSuccess) st = h->fail(TSVD_ERR_CUDA, "CSC layout failed");
    }
    cudaFree(cnt);
    cudaFree(flat);
    cudaFree(cidx);
    cudaFree(cval);
    cudaFree(flat_sl);
    cudaFree(ipos);
    return st;
}

static void free_sparse_stream(tsvd_t h) {
    if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
    for (int v = 0; v < 2; ++v) {
        if (h->sp_hidx[v]) cudaFreeHost(h->sp_hidx[v]);
        if (h->sp_hval[v]) cudaFreeHost(h->sp_hval[v]);
        h->sp_hidx[v] = nullptr;
        h->sp_hval[v] = nullptr;
        h->sp_hbase[v].clear();
    }
    for (void *q : h->sp_ring) cudaFree(q);
    for (cudaEvent_t e : h->sp_full) cudaEventDestroy(e);
    for (cudaEvent_t e : h->sp_free) cudaEventDestroy(e);
    h->sp_ring.clear();
    h->sp_full.clear();
    h->sp_free.clear();
    h->sp_stream = false;
}

// Sparse out of memory (degree 1): move both views' entry arrays (the bulk: 8 bytes per entry)
// to pinned host memory and size a q_s-slot device ring for the largest index block; every block
// launch then copies its block first (sp_stage_block).  The slice tables stay in HBM.
static tsvd_status sp_to_host(tsvd_t h) {
    int64_t slot = 0;
    for (int v = 0; v < 2; ++v) {
        SpView *view = v == 0 ? &h->spc : &h->spr;
        const int K = v == 0 ? h->sp_kc : h->sp_kr;
        h->sp_hbase[v].resize(K + 1);
        CK(cudaMemcpy(h->sp_hbase[v].data(), view->base, (K + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
        const int64_t T = h->sp_hbase[v][K];
        for (int b = 0; b < K; ++b) slot = std::max(slot, h->sp_hbase[v][b + 1] - h->sp_hbase[v][b]);
        CK(cudaHostAlloc((void **)&h->sp_hidx[v], std::max<size_t>((size_t)T * 4, 16), cudaHostAllocDefault));
        CK(cudaHostAlloc((void **)&h->sp_hval[v], std::max<size_t>((size_t)T * 4, 16), cudaHostAllocDefault));
        CK(cudaMemcpy(h->sp_hidx[v], view->idx, (size_t)T * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(h->sp_hval[v], view->val, (size_t)T * 4, cudaMemcpyDeviceToHost));
        for (const void *q : {(const void *)view->idx, (const void *)view->val}) {
            auto it = std::find(h->sp_mem.begin(), h->sp_mem.end(), q);
            if (it != h->sp_mem.end()) {
                cudaFree(*it);
                h->sp_mem.erase(it);
            }
        }
        h->sp_bytes -= 8 * T;
        view->idx = nullptr;
        view->val = nullptr;
    }
    h->sp_slot_entries = round_up(std::max<int64_t>(slot, 1), 32);
    for (int q = 0; q < h->qdepth; ++q) {
        void *p = nullptr;
        cudaEvent_t ef, eb;
        cudaError_t e = cudaMalloc(&p, (size_t)h->sp_slot_entries * 8);
        if (e == cudaErrorMemoryAllocation) return h->fail(TSVD_ERR_NOMEM, "no room for the %d-slot ring", h->qdepth);
        CK(e);
        CK(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&eb, cudaEventDisableTiming));
        h->sp_ring.push_back(p);
        h->sp_full.push_back(ef);
        h->sp_free.push_back(eb);
    }
    if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    h->sp_stream = true;
    h->streaming = true;  // host-driven loop (the copies are not captured in the run graph)
    return TSVD_OK;
}

static void free_sparse_views(tsvd_t h) {
    for (void *q : h->sp_mem) cudaFree(q);
    h->sp_mem.clear();
    h->sp_bytes = 0;
    h->spc = SpView{};
    h->spr = SpView{};
}

static void free_sparse(tsvd_t h) {
    free_sparse_stream(h);
    h->streaming = false;
    if (h->csr_owned) {
        cudaFree(h->row_ptr_d);
        cudaFree(h->col_d);
        cudaFree(h->val_d);
    }
    free_sparse_views(h);
    for (void *q : {(void *)h->acc_r, (void *)h->acc_c})
        if (q) cudaFree(q);
    h->acc_r = h->acc_c = nullptr;
    h->sp_kc = h->sp_kr = 1;
    h->row_ptr_d = nullptr;
    h->col_d = nullptr;
    h->val_d = nullptr;
    h->csr_owned = false;
}

tsvd_status tsvd_set_csr(tsvd_t h, const int64_t *row_ptr, const int32_t *col_idx, const float *val, int64_t nnz,
                         int64_t row_begin, int64_t row_end, tsvd_mem mem) {
    if (!h) return TSVD_ERR_ARG;
    if (!row_ptr || nnz < 0 || (nnz > 0 && (!col_idx || !val))) return h->fail(TSVD_ERR_ARG, "NULL CSR array");
    if (h->wide) return h->fail(TSVD_ERR_UNSUPPORTED, "sparse inputs must have m >= n (V-first branch) in this version");
    if (row_begin < 0 || row_end > h->m || row_end <= row_begin)
        return h->fail(TSVD_ERR_SHAPE, "row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                       (long long)row_end, (long long)h->m);
    if (h->n > INT32_MAX || (row_end - row_begin) > INT32_MAX)
        return h->fail(TSVD_ERR_UNSUPPORTED, "int32 column / local row indices");
    if (mem != TSVD_MEM_DEVICE && mem != TSVD_MEM_HOST_PINNED && mem != TSVD_MEM_HOST_PAGEABLE)
        return h->fail(TSVD_ERR_ARG, "bad mem kind");
    if (h->allocated && ((row_end - row_begin) != h->m_g || !h->sparse))
        return h->fail(TSVD_ERR_STATE, "the input kind / slab size cannot change after the first run");
    CK(cudaSetDevice(h->dev));
    const int64_t mg = row_end - row_begin, n = h->n;
    int64_t ends[2] = {0, nnz};
    if (mem == TSVD_MEM_DEVICE) {  // two small reads: the CSC build trusts [row_ptr[0], row_ptr[rows])
        CK(cudaMemcpy(&ends[0], row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&ends[1], row_ptr + mg, sizeof(int64_t), cudaMemcpyDeviceToHost));
    } else {
        ends[0] = row_ptr[0];
        ends[1] = row_ptr[mg];
    }
    if (ends[0] != 0 || ends[1] != nnz)
        return h->fail(TSVD_ERR_ARG, "row_ptr[0] must be 0 and row_ptr[rows] == nnz (got %lld, %lld; nnz %lld)",
                       (long long)ends[0], (long long)ends[1], (long long)nnz);
    free_sparse(h);
    h->sparse = true;
    h->row_begin = row_begin;
    h->row_end = row_end;
    h->m_g = mg;
    h->nnz_g = nnz;
    h->have_A = true;
    h->graph_l0 = -1;
    h->streaming = false;
    h->m_res = mg;
    if (h->world > 1) h->coll = COLL_NCCL;  // the length-n vector: coll_allreduce (NCCL; bandwidth-bound)
    auto t0 = std::chrono::steady_clock::now();
    if (mem == TSVD_MEM_DEVICE) {
        h->row_ptr_d = const_cast<int64_t *>(row_ptr);
        h->col_d = const_cast<int32_t *>(col_idx);
        h->val_d = const_cast<float *>(val);
    } else {
        h->csr_owned = true;
        CK(cudaMalloc((void **)&h->row_ptr_d, (size_t)(mg + 1) * sizeof(int64_t)));
        CK(cudaMalloc((void **)&h->col_d, std::max<size_t>((size_t)nnz * sizeof(int32_t), 16)));
        CK(cudaMalloc((void **)&h->val_d, std::max<size_t>((size_t)nnz * sizeof(float), 16)));
        CK(cudaMemcpyAsync(h->row_ptr_d, row_ptr, (size_t)(mg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
        if (nnz) {
            CK(cudaMemcpyAsync(h->col_d, col_idx, (size_t)nnz * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(h->val_d, val, (size_t)nnz * sizeof(float), cudaMemcpyHostToDevice, h->stream));
        }
    }
    // validate the CSR contract on the device (sorted unique columns in range)
    unsigned long long *bad = nullptr, bad_h = 0;
    CK(cudaMalloc((void **)&bad, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), h->stream));
    csr_check<<<h->sms * 8, 256, 0, h->stream>>>(h->row_ptr_d, h->col_d, mg, n, nnz, bad);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&bad_h, bad, sizeof(bad_h), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(bad);
    if (bad_h) {
        free_sparse(h);
        h->have_A = false;
        return h->fail(TSVD_ERR_ARG, "CSR has %llu bad rows / entries (row_ptr decreasing or outside [0, nnz], column out of range or not strictly increasing)",
                       bad_h);
    }
    // N4 / N4b: the two blocked views.  Index blocks keep each launch's gathers inside an L2-resident
    // block of the fp32 gathered vector (y32 for N2 by column, t32 for N3 by row); every block must
    // hold < 2^31 entries (int32 block-local offsets): the block count doubles until it does.
    const int64_t bw_auto = (int64_t)kSpL2BlockBytes / (int64_t)sizeof(float);
    const int64_t bwc = h->sp_block_opt > 0 ? h->sp_block_opt : bw_auto;
    const int64_t bwr = h->sp_block_opt > 0 ? h->sp_block_opt : bw_auto;
    int kc = (int)std::min<int64_t>(64, (n + bwc - 1) / bwc), kr = (int)std::min<int64_t>(64, (mg + bwr - 1) / bwr);
    tsvd_status bs = TSVD_OK;
    for (;; kr *= 2) {  // the CSC first: it is built from the CSR, which the CSR view may replace
        bs = build_csc_view(h, kr, (mg + kr - 1) / kr);
        if (bs != TSVD_ERR_UNSUPPORTED || kr >= mg) break;
        free_sparse_views(h);
    }
    if (bs == TSVD_OK)
        for (;; kc *= 2) {
            bs = build_csr_view(h, kc, (n + kc - 1) / kc);
            if (bs != TSVD_ERR_UNSUPPORTED || kc >= n) break;
        }
    if (bs != TSVD_OK) {
        free_sparse(h);
        h->have_A = false;
        return bs == TSVD_ERR_UNSUPPORTED ? h->fail(bs, "sparse slab: an index block would exceed 2^31 entries") : bs;
    }
    h->sp_kc = kc;
    h->sp_kr = kr;
    if (kc > 1) CK(cudaMalloc((void **)&h->acc_r, (size_t)2 * mg * sizeof(double)));
    if (kr > 1) CK(cudaMalloc((void **)&h->acc_c, (size_t)2 * n * sizeof(double)));
    // both views are the library's own (sliced) copies: an owned input copy is dropped (2 copies of the
    // entries remain); borrowed device arrays are not read after tsvd_set_csr returns
    if (h->csr_owned) {
        cudaFree(h->row_ptr_d);
        cudaFree(h->col_d);
        cudaFree(h->val_d);
        h->csr_owned = false;
    }
    h->row_ptr_d = nullptr;
    h->col_d = nullptr;
    h->val_d = nullptr;
    if (h->placement == 2) TRY(sp_to_host(h));  // out of memory, degree 1
    if (h->world > 1 && !h->sp_comm_stream) {
        CK(cudaStreamCreateWithFlags(&h->sp_comm_stream, cudaStreamNonBlocking));
        for (int c = 0; c <= h->sp_chunks; ++c) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            h->sp_ev.push_back(e);
        }
    }
    h->csc_build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return TSVD_OK;
}

tsvd_status tsvd_set_factors(tsvd_t h, int32_t l, const float *U, const double *S, const double *V) {
    if (!h) return TSVD_ERR_ARG;
    if (l < 0 || l > h->k || (l > 0 && (!U || !S || !V))) return h->fail(TSVD_ERR_ARG, "bad factors");
    if (!h->have_A) return h->fail(TSVD_ERR_STATE, "set_dense first");
    CK(cudaSetDevice(h->dev));
    TRY(ensure_alloc(h));
    std::vector<float> uw;
    std::vector<double> vw;
    if (h->wide && l > 0) {  // the caller's U (m_user x l) is the tall V, its V (n_user x l) the tall U
        uw.resize((size_t)h->m_g * l);
        vw.resize((size_t)h->n * l);
        for (size_t i = 0; i < uw.size(); ++i) uw[i] = (float)V[i];
        for (size_t i = 0; i < vw.size(); ++i) vw[i] = (double)U[i];
        U = uw.data();
        V = vw.data();
    }
    if (l > 0) {
        CK(cudaMemcpy2DAsync(h->U32, h->kpad * sizeof(float), U, l * sizeof(float), l * sizeof(float), h->m_g,
                             cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(h->S64, S, l * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpy2DAsync(h->V64, h->k * sizeof(double), V, l * sizeof(double), l * sizeof(double), h->n,
                             cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    for (int i = l; i < h->k; ++i) {
        h->iters[i] = 0;
        h->dots[i] = 0.0;
    }
    h->l_found = l;
    h->k_found = l;
    // explicit Gram (METHOD = 1): P = A^T U and Q = U^T U were built for the factors this handle
    // computed; injected factors invalidate them (a METHOD = 1 run then restarts from l = 0 only)
    if (l > 0) h->pq_l = 0;
    return TSVD_OK;
}

tsvd_status tsvd_gram_apply(tsvd_t h, const double *v, double *y) {
    if (!h) return TSVD_ERR_ARG;
    if (!v || !y) return h->fail(TSVD_ERR_ARG, "NULL vector");
    if (!h->have_A) return h->fail(TSVD_ERR_STATE, "set_dense first");
    CK(cudaSetDevice(h->dev));
    TRY(ensure_alloc(h));
    TRY(stage_A(h));
    TRY(reset_state(h));
    const int n = (int)h->n, l = h->l_found;
    memcpy(h->vec_host, v, (size_t)n * sizeof(double));
    CK(cudaMemcpyAsync(h->yw, h->vec_host, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    // y_cur = v (unnormalised), c = S V^T v
    TRY(inproc_rendezvous(h));
    TRY(launch_fin(h, h->stream, fin_params(h, FIN_LOAD_RAW, l, h->yw, 0ull, 0), SRC_PARTS));
    TRY(launch_gv(h, h->stream, l, false));
    TRY(launch_exchange(h, h->stream, l));
    TRY(launch_fin(h, h->stream, fin_params(h, FIN_APPLY, l, nullptr, 0ull, 0), fin_src(h)));
    CK(cudaMemcpyAsync(h->vec_host, h->ybuf + h->ystride, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->st_host->status == -6) return h->fail(TSVD_ERR_NCCL, "peer all-reduce timed out (a rank did not arrive)");
    memcpy(y, h->vec_host, (size_t)n * sizeof(double));
    TRY(unstage_A(h));
    return TSVD_OK;
}

tsvd_status tsvd_run(tsvd_t h) {
    if (!h) return TSVD_ERR_ARG;
    if (!h->have_A) return h->fail(TSVD_ERR_STATE, "set_dense first");
    CK(cudaSetDevice(h->dev));
    auto t0 = std::chrono::steady_clock::now();
    TRY(ensure_alloc(h));
    TRY(stage_A(h));
    TRY(upload_v0(h));
    h->n1_ms = 0.0;
    h->n1_launches = 0;
    h->ps_ms = 0.0;
    h->ps_launches = 0;
    h->ps_passes = 0;
    h->total_iters = 0;
    h->launches = 0;
    const int l0 = h->l_found;
    if (l0 >= h->k) return TSVD_OK;
    CK(cudaMemsetAsync(h->stats, 0, (size_t)h->k * sizeof(CompStat), h->stream));
    TRY(reset_state(h));
    // the graph needs every collective to be a kernel: single GPU or the peer all-reduce
    h->streamed_bytes = 0;
    h->streamed_batches = 0;
    // the graph needs every step to be a device kernel: no NCCL call, no host->device streaming
    const bool explicit_gram = h->method == 1;
    const bool graph = !explicit_gram && h->use_graph && !h->timing && h->coll != COLL_NCCL && !h->streaming;
    bool ran = false;
    if (explicit_gram) {
        TRY(run_explicit(h, l0));
        ran = true;
    }
    if (graph) {
        tsvd_status gs = TSVD_OK;
        if (!h->exec || h->graph_l0 != l0) gs = build_graph(h, l0);
        if (gs >= 0) {
            TRY(inproc_rendezvous(h));
            CK(cudaGraphLaunch(h->exec, h->stream));
            h->loop_mode = use_persist(h) ? "graph-persistent" : "graph-while";
            ran = true;
        } else {
            h->graph_error = h->err;  // fall back to the host loop, keep the reason for the report
            TRY(reset_state(h));
        }
    }
    if (!ran) {
        TRY(inproc_rendezvous(h));
        TRY(run_host_loop(h, l0));
    }
    if (!ran && use_persist(h)) h->loop_mode = h->timing ? "host-persistent+events" : "host-persistent";
    CK(cudaMemcpyAsync(h->stats_host, h->stats, (size_t)h->k * sizeof(CompStat), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(LoopState), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->st_host->status == -6) return h->fail(TSVD_ERR_NCCL, "peer all-reduce timed out (a rank did not arrive)");
    if (h->st_host->status == -7 && h->st_host->stop)
        return h->fail(TSVD_ERR_NUMERIC, "non-finite value or zero initial vector");
    tsvd_status result = TSVD_OK;
    h->fused_ext_used = !explicit_gram && fuse_ext(h) && h->k - l0 > 1;
    // our kernels per iteration / extraction (NCCL calls not counted)
    int64_t per_pass = 1;
    if (h->streaming && !h->sparse)
        per_pass = (h->m_res > 0 ? 1 : 0) + (h->m_g - h->m_res + h->batch_rows - 1) / h->batch_rows;
    if (h->sparse) per_pass = h->sp_kc + h->sp_kr;
    const int64_t per_iter = per_pass + (h->coll == COLL_NONE || h->sparse || fused_reduce(h) ? 1 : 2);
    const int64_t per_ext = (h->sparse ? h->sp_kc : per_pass) + (h->coll == COLL_NONE ? 1 : 2);
    for (int l = l0; l < h->k; ++l) {
        const CompStat &cs = h->stats_host[l];
        // fused extraction: component l > l0 starts with init_ext + the fused first iteration (which
        // also extracts l-1); only the last component keeps a separate extraction
        const bool ff = h->fused_ext_used && l > l0;
        const int64_t body_it = ff ? std::max<int64_t>(cs.it - 1, 0) : cs.it;
        const int64_t issued = h->loop_mode == "graph-while"
                                   ? std::max<int64_t>(1, (body_it + h->unroll - 1) / h->unroll) * h->unroll
                                   : body_it;
        const bool ps = !explicit_gram && use_persist(h);
        if (ps || explicit_gram) h->ps_passes += body_it;
        if (explicit_gram)  // init + the B0 iteration kernel + the extraction pass + its finish
            h->launches += 4;
        else if (ps && h->fused_ext_used)  // chain: [init | two-vector pass] + one persistent launch
            h->launches += 2 + (l == h->k - 1 ? per_ext : 0);
        else
            h->launches += 1 + (ff ? per_iter : 0) + (ps ? 1 : per_iter * issued) +
                           (!h->fused_ext_used || l == h->k - 1 ? per_ext : 0);
        if (cs.status == -7) return h->fail(TSVD_ERR_NUMERIC, "non-finite value or zero initial vector at component %d", l);
        if (!cs.valid || cs.status == 2) {
            result = TSVD_WARN_RANK_EXHAUSTED;
            break;
        }
        h->iters[l] = cs.it;
        h->dots[l] = cs.d;
        h->total_iters += cs.it;
        if (cs.status == 1 && result == TSVD_OK) result = TSVD_WARN_NOT_CONVERGED;
        h->l_found = l + 1;
        h->k_found = l + 1;
    }
    if (h->tl_d) {  // debug timeline dump: iteration, N1 start, N1 end, fin end, fin start, fin tail,
                    // first N1 CTA out (ns, relative; -1 = not recorded)
        std::vector<unsigned long long> tl(2 + kTl * 4096);
        CK(cudaMemcpy(tl.data(), h->tl_d, tl.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        char name[1024];
        snprintf(name, sizeof name, "%s.rank%d", getenv("TSVD_TIMELINE"), h->rank);
        if (FILE *f = fopen(name, "a")) {
            const int64_t cnt = std::min<int64_t>((int64_t)tl[0], 4096);
            const unsigned long long base = cnt ? tl[2] : 0;
            for (int64_t i = 0; i < cnt; ++i)
            {
                const unsigned long long *r = tl.data() + 2 + kTl * i;
                auto rel = [&](unsigned long long t) { return t ? (long long)(t - base) : -1ll; };
                fprintf(f, "%lld", (long long)i);
                for (int q = 0; q < kTl; ++q) fprintf(f, ",%lld", rel(r[q]));
                fprintf(f, "\n");
            }
            fclose(f);
        }
        CK(cudaMemsetAsync(h->tl_d, 0, tl.size() * sizeof(unsigned long long), h->stream));
    }
    TRY(unstage_A(h));
    h->run_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (result == TSVD_WARN_RANK_EXHAUSTED) h->err = "rank exhausted before k components";
    return result;
}

tsvd_status tsvd_get_U_S_V(tsvd_t h, float *U, double *S, float *V) {
    if (!h) return TSVD_ERR_ARG;
    if (!h->allocated) return h->fail(TSVD_ERR_STATE, "nothing computed yet");
    CK(cudaSetDevice(h->dev));
    if (h->wide) {  // A^T = V S U^T: the caller's U is the tall V (m_user x k), its V the tall U
        std::vector<double> vt((size_t)h->n * h->k);
        std::vector<float> ut((size_t)h->m_g * h->kpad);
        CK(cudaMemcpyAsync(vt.data(), h->V64, vt.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(ut.data(), h->U32, ut.size() * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
        if (S) CK(cudaMemcpyAsync(S, h->S64, h->k * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        for (int64_t r = 0; U && r < h->n; ++r)
            for (int c = 0; c < h->k; ++c) U[r * h->k + c] = c < h->k_found ? (float)vt[r * h->k + c] : 0.f;
        for (int64_t r = 0; V && r < h->m_g; ++r)
            for (int c = 0; c < h->k; ++c) V[r * h->k + c] = c < h->k_found ? ut[r * h->kpad + c] : 0.f;
        for (int c = h->k_found; S && c < h->k; ++c) S[c] = 0.0;
        return TSVD_OK;
    }
    if (U)
        CK(cudaMemcpy2DAsync(U, h->k * sizeof(float), h->U32, h->kpad * sizeof(float), h->k * sizeof(float), h->m_g,
                             cudaMemcpyDeviceToHost, h->stream));
    if (S) CK(cudaMemcpyAsync(S, h->S64, h->k * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    std::vector<double> vt;
    if (V) {
        vt.resize((size_t)h->n * h->k);
        CK(cudaMemcpyAsync(vt.data(), h->V64, vt.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    if (V)
        for (size_t i = 0; i < vt.size(); ++i) V[i] = (float)vt[i];
    // columns >= k_found are zero (contract), whatever a partial run left on the device
    for (int64_t r = 0; U && r < h->m_g; ++r)
        for (int c = h->k_found; c < h->k; ++c) U[r * h->k + c] = 0.f;
    for (int c = h->k_found; S && c < h->k; ++c) S[c] = 0.0;
    for (int64_t r = 0; V && r < h->n; ++r)
        for (int c = h->k_found; c < h->k; ++c) V[r * h->k + c] = 0.f;
    return TSVD_OK;
}

tsvd_status tsvd_get_info(tsvd_t h, int32_t *k_found, int32_t *iters, double *dots) {
    if (!h) return TSVD_ERR_ARG;
    if (k_found) *k_found = h->k_found;
    if (iters) memcpy(iters, h->iters.data(), h->k * sizeof(int32_t));
    if (dots) memcpy(dots, h->dots.data(), h->k * sizeof(double));
    return TSVD_OK;
}

tsvd_status tsvd_get_report(tsvd_t h, char *buf, size_t cap) {
    if (!h || !buf || cap == 0) return TSVD_ERR_ARG;
    std::string s = "{";
    char tmp[768];
    static const char *colls[] = {"none", "peer-nvlink", "nccl"};
    snprintf(tmp, sizeof tmp,
             "\"m\": %lld, \"n\": %lld, \"k\": %d, \"eps\": %.3g, \"rank\": %d, \"world\": %d, \"rows\": [%lld, %lld], "
             "\"wide\": %s, \"layout\": \"%s\", \"transposed_copy\": %s, \"k_found\": %d, \"total_iters\": %lld, \"run_ms\": %.4f, \"h2d_ms\": %.4f, \"n1_ms\": %.6f, "
             "\"n1_launches\": %lld, \"kernel_launches\": %lld, \"loop\": \"%s\", \"collective\": \"%s\", ",
             (long long)h->m_user, (long long)h->n_user, h->k, h->eps, h->rank, h->world, (long long)h->row_begin,
             (long long)h->row_end, h->wide ? "true" : "false", h->layout == TSVD_COL_MAJOR ? "col" : "row",
             h->tcopy ? "true" : "false", h->k_found, (long long)h->total_iters, h->run_ms, h->h2d_ms,
             h->n1_ms,
             (long long)h->n1_launches, (long long)h->launches, h->loop_mode.c_str(), colls[h->coll]);
    s += tmp;
    snprintf(tmp, sizeof tmp,
             "\"persistent\": {\"enabled\": %s, \"T\": %d, \"NV\": %d, \"stages\": %d, \"smem\": %zu, \"ms\": %.6f, "
             "\"launches\": %lld, \"passes\": %lld}, \"method\": \"%s\", \"gram_ms\": %.3f, \"gram_blocks\": %d, ",
             (use_persist(h) || h->method == 1) ? "true" : "false", h->method == 1 ? h->T : h->T_ps,
             h->method == 1 ? h->NV : h->NV_ps, h->method == 1 ? h->S_gb : h->S_ps,
             h->method == 1 ? h->smem_gb : h->smem_ps, h->ps_ms, (long long)h->ps_launches, (long long)h->ps_passes,
             h->method == 1 ? "explicit-gram" : "gram-vector", h->gram_ms, h->gram_blocks);
    s += tmp;
    snprintf(tmp, sizeof tmp,
             "\"plan\": {\"T\": %d, \"NV\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"grid\": %d, \"smem\": %zu, "
             "\"stage_bytes\": %d, \"run_rows\": %d, \"split\": %d, \"two_T\": %d, \"fused_extract\": %s, \"pdl\": %s, "
             "\"serpentine\": %s}, ",
             h->T, h->NV, h->S, h->cps, h->grid, h->smem, h->stage_bytes, h->run_rows, h->split, h->T_two,
             h->fused_ext_used ? "true" : "false", (h->pdl_opt && !h->sm_limit) ? "true" : "false",
             h->serp_opt && !h->streaming ? "true" : "false");
    s += tmp;
    snprintf(tmp, sizeof tmp,
             "\"placement\": {\"streaming\": %s, \"resident_rows\": %lld, \"batch_rows\": %lld, \"queue_depth\": %d, "
             "\"streamed_bytes\": %lld, \"streamed_batches\": %lld, \"device_bytes\": %lld, \"v_on_host\": %s}, ",
             h->streaming ? "true" : "false", (long long)h->m_res, (long long)h->batch_rows, h->qdepth,
             (long long)h->streamed_bytes, (long long)h->streamed_batches,
             (long long)(h->work_bytes + (h->mem == TSVD_MEM_DEVICE || h->sparse ? 0 : h->m_res * ((h->n + 3) / 4) * 16) +
                         (h->streaming ? (int64_t)h->qdepth * h->batch_rows * ((h->n + 3) / 4) * 16 : 0) +
                         h->sp_bytes + (h->acc_r ? 16 * h->m_g : 0) + (h->acc_c ? 16 * h->n : 0) +
                         (int64_t)h->sp_ring.size() * h->sp_slot_entries * 8),
             h->v_host ? "true" : "false");
    s += tmp;
    snprintf(tmp, sizeof tmp,
             "\"sparse\": {\"enabled\": %s, \"nnz\": %lld, \"csc_build_ms\": %.3f, \"col_blocks\": %d, \"row_blocks\": %d, "
             "\"view_bytes\": %lld, \"input_kept\": %s, \"chunks\": %d}, ",
             h->sparse ? "true" : "false", (long long)h->nnz_g, h->csc_build_ms, h->sp_kc, h->sp_kr,
             (long long)h->sp_bytes, h->sparse && h->sp_kc == 1 ? "true" : "false", sp_overlap(h) ? h->sp_chunks : 1);
    s += tmp;
    std::string ge = h->graph_error + (h->peer_error.empty() ? "" : " | " + h->peer_error);
    for (char &c : ge)
        if (c == '"' || c == '\\') c = '\'';
    s += "\"graph_error\": \"" + ge + "\", \"iters\": [";
    for (int i = 0; i < h->k; ++i) {
        snprintf(tmp, sizeof tmp, "%s%d", i ? ", " : "", h->iters[i]);
        s += tmp;
    }
    s += "]}";
    snprintf(buf, cap, "%s", s.c_str());
    return TSVD_OK;
}

tsvd_status tsvd_time_gram_kernel(tsvd_t h, int32_t reps, double *ms) {
    if (!h || !ms || reps < 1) return TSVD_ERR_ARG;
    if (!h->have_A) return h->fail(TSVD_ERR_STATE, "set_dense first");
    CK(cudaSetDevice(h->dev));
    TRY(ensure_alloc(h));
    TRY(stage_A(h));
    TRY(reset_state(h));  // the kernel skips itself when a loop is done; invalidates iteration state
    const int l = std::min(h->l_found, h->k - 1);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    TRY(launch_gv(h, h->stream, l, false));  // warm-up
    CK(cudaEventRecord(e0, h->stream));
    for (int r = 0; r < reps; ++r) TRY(launch_gv(h, h->stream, l, false));
    CK(cudaEventRecord(e1, h->stream));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = (double)t / reps;
    return TSVD_OK;
}

void *tsvd_get_stream(tsvd_t h) { return h ? (void *)h->stream : nullptr; }

const char *tsvd_last_error(tsvd_t h) { return h ? h->err.c_str() : g_err.c_str(); }

void tsvd_destroy(tsvd_t h) {
    if (!h) return;
    cudaSetDevice(h->dev);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->grp) {  // barrier: no rank may still read our exchange buffers when they are freed
        grp_exchange(h, 0, nullptr, nullptr, "destroy");
    } else if (h->comm) {  // barrier: no peer may still read our symmetric buffer when it is freed
        int *d = nullptr;
        if (cudaMalloc((void **)&d, sizeof(int)) == cudaSuccess) {
            ncclAllReduce(d, d, 1, ncclInt32, ncclSum, h->comm, h->stream);
            cudaStreamSynchronize(h->stream);
            cudaFree(d);
        }
    }
    drop_graph(h);
    if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
    free_ring(h);
    free_sparse(h);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->sp_comm_stream) {
        cudaStreamSynchronize(h->sp_comm_stream);
        cudaStreamDestroy(h->sp_comm_stream);
    }
    for (cudaEvent_t e : h->sp_ev) cudaEventDestroy(e);
    if (h->host_registered) cudaHostUnregister((void *)h->A_user);
    for (int r = 0; r < kMaxRanks; ++r) {
        if (h->peer_map[r]) cudaIpcCloseMemHandle(h->peer_map[r]);
        if (h->px_map[r]) cudaIpcCloseMemHandle(h->px_map[r]);
        if (h->gx_map[r]) cudaIpcCloseMemHandle(h->gx_map[r]);
    }
    if (h->V64_h) cudaFreeHost(h->V64_h);
    if (h->V0d_h) cudaFreeHost(h->V0d_h);
    if (h->v_host) h->V64 = h->V0d = nullptr;
    void *dev_ptrs[] = {h->A_own, h->U32, h->V64, h->S64, h->ybuf, h->yw, h->V0d, h->c64, h->ypart,
                        h->wpart, h->part, h->u64, h->sq_part, h->sig2, h->st, h->stats, h->sym, h->gbar,
                        h->trace_d, h->work, h->tl_d, h->vprev32, h->px_mem, h->y32, h->t32, h->At,
                        h->B0, h->Pm, h->Qm, h->gpart, h->zero64, h->g_hi, h->g_lo, h->pub, h->puby, h->gx_mem,
                        h->gram_tiles, h->ar_tmp};
    if (h->cublas) cublasDestroy(h->cublas);
    if (h->trace_f) fclose(h->trace_f);
    for (void *p : dev_ptrs)
        if (p) cudaFree(p);
    if (h->st_host) cudaFreeHost(h->st_host);
    if (h->stats_host) cudaFreeHost(h->stats_host);
    if (h->vec_host) cudaFreeHost(h->vec_host);
    if (h->comm) ncclCommDestroy(h->comm);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->body_stream) cudaStreamDestroy(h->body_stream);
    delete h;
}

}  // extern "C"
