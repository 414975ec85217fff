/*
 * tsvd.h — C ABI of libtsvd.so, the B200-native (sm_100a) hot path of the power-method
 * truncated SVD of arXiv 2208.08410 ("Distributed Out-of-Memory SVD on CPU/GPU
 * Architectures").  Citations "P:nnn" are lines of the paper text.
 *
 * What the library computes:
 *   Alg. 1: for l = 0..k-1, with the first l components (U, S, V) found,
 *   Alg. 2 SVD_1D on the deflated X' = A - U diag(S) V^T: starting from
 *   v = x / ||x|| (x ~ N(0, I)), repeat
 *        y  = X'^T (X' v)          implicit Gram-vector product, Eq. 2 in the exact
 *                                   factored form  c = S (V^T v); t = A v - U c;
 *                                   w = S (U^T t); y = A^T t - V w   (X' never formed)
 *        v1 = y / ||y||
 *   until |v . v1| >= 1 - eps, then extracts u = A v1 / sigma, sigma = ||A v1||
 *   with the ORIGINAL A.
 *
 * Orientation (Alg. 1): m >= n runs the V-first (X'^T X') branch (square inputs too);
 * m < n runs the U-first (X' X'^T) branch of P:88-92 / Eq. 3 as the V-first branch of
 * A^T, with U and V swapped at the boundary.  Layout (tsvd_create): a row-major tall A and a
 * column-major wide A (= A^T row-major) are used in place; a row-major wide A or a column-major
 * tall A is transposed once into a device copy (one GPU).
 *
 * Conventions for every function:
 *   - No exceptions cross the ABI.  Every call returns a tsvd_status (warnings > 0, errors < 0)
 *     and stores a message retrievable with tsvd_last_error(h).
 *   - Input pointers are BORROWED: they must stay valid and unmodified until the call that
 *     consumes them (tsvd_run / tsvd_gram_apply) returns.  Outputs are copied into caller-owned
 *     buffers.  The handle owns every device buffer, stream, graph and communicator it creates.
 *   - A handle is not thread-safe; one host thread per handle.  One handle per GPU per process,
 *     except the ranks of an in-process group (tsvd_get_inproc_id), which share a GPU.
 *   - Multi-GPU, one process per GPU, or in-process ranks (tsvd_get_inproc_id: the
 *     same code path with every rank a handle of one process).  Row partition (RSVD/HSVD, row-major tall A):
 *     each rank owns rows [row_begin, row_end) of A and of U; S and V are replicated.  Column
 *     partition (CSVD, column-major wide A): each rank owns columns [row_begin, row_end)
 *     of A and those rows of V; S and U are replicated.  Every rank calls every function with
 *     the same (m, n, k, eps) and options.  Per iteration ONE reduction of [y_g | w_g] across ranks
 *     (Alg. 4 lines 6, 8, 16, merged): by default inside the kernels over NVLink peer
 *     memory (CUDA IPC-mapped buffers, stamped words, no library call; TSVD_OPT_COLLECTIVE = 0);
 *     ncclAllReduce with TSVD_OPT_COLLECTIVE = 1 and for sparse inputs.
 */
#ifndef TSVD_H
#define TSVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsvd_s *tsvd_t; /* opaque handle */

typedef enum { TSVD_F32 = 0 /* A, U stored fp32, all cross-thread sums fp64 */, TSVD_F64 = 1 /* reserved */ } tsvd_dtype;
typedef enum {
    TSVD_ROW_MAJOR = 0,  /* A[i, j] at A[i * ld + j]; range arguments count rows                       */
    TSVD_COL_MAJOR = 1   /* A[i, j] at A[i + j * ld]; range arguments count columns (the major dim.)    */
} tsvd_layout;
typedef enum { TSVD_MEM_DEVICE = 0, TSVD_MEM_HOST_PINNED = 1, TSVD_MEM_HOST_PAGEABLE = 2 } tsvd_mem;

typedef enum {
    TSVD_OK = 0,
    TSVD_WARN_NOT_CONVERGED = 1,   /* some component hit MAX_ITER (not fatal)              */
    TSVD_WARN_RANK_EXHAUSTED = 2,  /* ||X'^T X' v|| == 0 or sigma == 0: fewer than k found */
    TSVD_ERR_ARG = -1,             /* k > min(m,n), eps not in (0,1), null pointer, ...    */
    TSVD_ERR_SHAPE = -2,           /* row range / leading dimension inconsistent          */
    TSVD_ERR_UNSUPPORTED = -3,     /* layout / orientation / size not in this version     */
    TSVD_ERR_NOMEM = -4,           /* device allocation failed (incl. OOM degree 2) */
    TSVD_ERR_CUDA = -5,
    TSVD_ERR_NCCL = -6,
    TSVD_ERR_NUMERIC = -7,         /* non-finite value or zero initial vector              */
    TSVD_ERR_STATE = -8            /* call out of order (e.g. run before set_dense)        */
} tsvd_status;

typedef enum {
    TSVD_OPT_MAX_ITER = 1,       /* iterations cap per component; default 10000 (reading R5)       */
    TSVD_OPT_FIXED_ITERS = 2,    /* > 0: exactly T iterations, convergence test off */
    TSVD_OPT_SEED = 3,           /* seed of the internal x ~ N(0,1) generator (used when no
                                    tsvd_set_init): splitmix64(seed, l, i) + Box-Muller, fp64     */
    TSVD_OPT_GRAPH = 4,          /* 1 (default): iteration loop as a CUDA-graph WHILE node;
                                    0: host-driven loop (one D2H flag read per iteration)         */
    TSVD_OPT_TIMING = 5,         /* 1: host loop with CUDA events around every fused-kernel launch;
                                    totals appear in tsvd_get_report                              */
    TSVD_OPT_RUN_ROWS = 6,       /* rows per fp32 accumulation run before an fp64 flush (def 1024) */
    TSVD_OPT_CTAS_PER_SM = 7,    /* 0 = auto (occupancy); testing knob                              */
    TSVD_OPT_COLLECTIVE = 8,     /* world > 1: 0 (default) = all-reduce fused into the finalize kernel
                                    over NVLink peer memory (CUDA IPC, in-graph); 1 = ncclAllReduce
                                    with a host-driven loop (fallback / cross-check)                 */
    TSVD_OPT_PLACEMENT = 9,      /* host input only: 0 auto (resident if the slab fits in HBM, else
                                    OOM degree 1), 1 resident, 2 stream (resident prefix +
                                    batches streamed host->device every pass)                        */
    TSVD_OPT_RESIDENT_BYTES = 10,/* stream mode: cap on the HBM-resident prefix of A (-1 = as much as
                                    fits; 0 = stream every row)                                       */
    TSVD_OPT_BATCH_ROWS = 11,    /* stream mode: rows per H2D batch (0 = ~256 MiB batches)            */
    TSVD_OPT_QUEUE_DEPTH = 12,   /* stream mode: device ring slots q_s, 1..8, def. 3
                                    (1: copy and compute of consecutive batches serialise)            */
    TSVD_OPT_FUSED_REDUCE = 13,  /* 1: the fused kernel sums its per-CTA partials itself (cooperative
                                    launch, grid barrier, column slices) and, multi-GPU, publishes them
                                    to the peers; 0 (default): separate reduction kernel (measured
                                    faster)                                                */
    TSVD_OPT_DETERMINISTIC = 14, /* 1 (default): static contiguous row split per CTA, bitwise-
                                    reproducible results; 0: CTAs claim row chunks dynamically (sums
                                    reproducible only to rounding; measured slower on dense C2)        */
    TSVD_OPT_GRAPH_UNROLL = 15,  /* iterations per CUDA-graph WHILE body (1..8, default 2): later ones
                                    are no-ops once the component has stopped                        */
    TSVD_OPT_FUSED_EXTRACT = 16, /* dense resident input: 1 (default) = the extraction u = A v (Alg. 1
                                    lines 12-14) of component l-1 rides in the same pass over A
                                    as the first iteration of component l (one read of A saved per
                                    component); 0 = separate extraction pass. Same results to
                                    rounding (DESIGN R21)                                             */
    TSVD_OPT_PDL = 17,           /* 1 (default): kernels of the loop are launched with programmatic
                                    dependent launch (each waits for its predecessor in-kernel, so
                                    launch latency overlaps the predecessor's drain); 0: plain
                                    stream order. Bitwise-identical results either way             */
    TSVD_OPT_ROW_ORDER = 18,     /* resident input: 1 (default) = serpentine, each CTA walks its row
                                    range backwards on odd iterations so the rows last read by the
                                    previous pass (still in the 126 MB L2) are read first; 0 = always
                                    forward. Changes only the fp32 summation order (rounding)       */
    TSVD_OPT_PERSISTENT = 19,    /* dense resident, n <= 16384, one GPU or several with the peer
                                    collective: 1 (default) = the iterations of a component run inside
                                    ONE cooperative kernel (grid barrier, in-kernel reduction, cross-
                                    rank exchange and stop test; no per-iteration kernel boundaries);
                                    0 = one fused pass + finalize kernel per iteration                */
    TSVD_OPT_SPARSE_BLOCK = 20,  /* sparse: width (elements) of the index blocks the gathers are
                                    split into so that each launch's block of the fp32 gathered
                                    vector stays in L2; 0 (default) = 48 MiB of fp32 (n > 12.6M
                                    columns / rows => several blocks). Read by tsvd_set_csr          */
    TSVD_OPT_METHOD = 21,        /* 0 (default): implicit Gram-vector products (Eq. 2, the north star);
                                    1: explicit Gram (Alg. 2 lines 6-9 with Alg. 3's Gram, P:114-121,
                                    P:220-249): B0 = A^T A once (a tcgen05 3xTF32 kernel on CTA
                                    pairs over the symmetric tile schedule of P:348), then per iteration
                                    y = B0 v - P c - V g with P = A^T U, Q = U^T U (exact deflation,
                                    no U^T U = I assumption); dense, resident, n <= 16384.  World > 1:
                                    B0 all-reduced once, iterations row-partitioned over B0 (y rows
                                    exchanged over NVLink inside the kernel; k <= 129, else
                                    replicated).  Pays off when iterations per component are many */
    TSVD_OPT_V_PLACEMENT = 22,   /* 0 (default): the co-factor V (n x k fp64) and the initial samples
                                    (k x n fp64) in HBM; 1: in pinned host memory mapped into the
                                    device address space ("the heavy co-factor V is stored on the
                                    host"): the kernels read and write them over the host link
                                    (frees 16 n k bytes of HBM; every iteration pays n l reads over
                                    PCIe).  Must precede the first run                               */
    TSVD_OPT_SM_LIMIT = 23       /* run on at most this many SMs (0, default: all).  Lets several
                                    handles share one GPU at the same time — the in-process ranks of
                                    tsvd_get_inproc_id, whose persistent grids must be co-resident.
                                    Must precede tsvd_set_dense / tsvd_set_csr                        */
} tsvd_option;

/*
 * tsvd_create — new handle for an m x n fp32 problem, k components (k == -1 -> min(m, n),
 * P:71-72), stop rule |v0 . v1| >= 1 - eps.  Binds the current CUDA device.
 * m < n (wide, Alg. 1 else-branch P:88-92, Eq. 3): the U-first branch, run as the tall
 * (V-first) problem on A^T; the iterate and V0 have length m, U and V keep their meaning for A.
 * layout = TSVD_COL_MAJOR with m < n: A^T is the caller's buffer read row-major, used in place, and
 * may be column-partitioned across ranks (CSVD).  layout = TSVD_ROW_MAJOR with m < n, or
 * TSVD_COL_MAJOR with m >= n: the whole matrix is passed to tsvd_set_dense and transposed once into
 * a device copy (single GPU; the copy doubles the footprint).
 * Errors: TSVD_ERR_ARG (m, n < 1; k < -1 or 0 or > min(m,n); eps not in (0,1); out == NULL; unknown
 *         layout), TSVD_ERR_UNSUPPORTED (dtype != F32; k > 4096), TSVD_ERR_CUDA.
 */
tsvd_status tsvd_create(tsvd_t *out, int64_t m, int64_t n, int32_t k, double eps, tsvd_dtype dtype,
                        tsvd_layout layout);

/* tsvd_get_unique_id — writes a 128-byte ncclUniqueId into out128 (rank 0 calls it and
 * broadcasts the bytes, e.g. through torch.distributed).  Errors: TSVD_ERR_NCCL. */
tsvd_status tsvd_get_unique_id(void *out128);

/* tsvd_get_inproc_id — writes a 128-byte id of a NEW in-process rank group into out128: `world`
 * handles of this one process, each driven from its own host thread (tsvd_run blocks), pass it to
 * tsvd_set_comm instead of an NCCL id.  The setup-time agreements then use a host rendezvous and
 * the exchange buffers are the other handles' device pointers; the data path is the multi-GPU
 * peer path unchanged (row partition; one reduction per iteration, Alg. 4).
 * Typical use: several ranks on ONE GPU (TSVD_OPT_SM_LIMIT = about 3/4 of SMs / world each, one
 * CTA per SM), which runs the multi-GPU exchange protocol where only one GPU exists.  The ranks'
 * kernels wait for each other, so each rank's stream needs its own hardware queue: set
 * CUDA_DEVICE_MAX_CONNECTIONS >= 2 world before the process creates its CUDA context, and no other
 * thread of the process may make a device-synchronising CUDA call (cudaFree, cudaDeviceSynchronize,
 * tsvd_destroy of an unrelated handle, ...) while the ranks run.  Where the
 * multi-process path calls ncclAllReduce (sparse length-n vectors, METHOD = 1's B0 and extraction
 * sums) in-process ranks sum the ranks' buffers in rank order between two host rendezvous
 * (host-synchronous; a test vehicle, not a fast path).  TSVD_OPT_COLLECTIVE = 1 is refused with
 * TSVD_ERR_UNSUPPORTED.  Errors: TSVD_ERR_ARG. */
tsvd_status tsvd_get_inproc_id(void *out128);

/* tsvd_set_comm — join an NCCL communicator of `world` ranks (this rank = `rank`, world <= 8, one
 * node) on CUDA device `device`, and map every rank's symmetric reduction buffer into this process
 * (CUDA IPC handles exchanged with ncclAllGather) for the in-kernel NVLink all-reduce.  Collective:
 * every rank must call it.  Optional; world == 1 needs no call.  Must precede tsvd_set_dense.
 * If the peer mapping fails the handle falls back to ncclAllReduce (TSVD_OPT_COLLECTIVE = 1).
 * With an id from tsvd_get_inproc_id the ranks are handles of this process (no NCCL, see above);
 * a rank that does not arrive within 60 s fails the others with TSVD_ERR_NCCL.
 * Errors: TSVD_ERR_ARG (bad rank/world, world > 8, group size mismatch), TSVD_ERR_NCCL,
 * TSVD_ERR_CUDA, TSVD_ERR_UNSUPPORTED (in-process ranks with COLLECTIVE = 1). */
tsvd_status tsvd_set_comm(tsvd_t h, int32_t rank, int32_t world, const void *nccl_unique_id, int32_t device);

/* tsvd_set_option — see tsvd_option.  Errors: TSVD_ERR_ARG (unknown key / bad value). */
tsvd_status tsvd_set_option(tsvd_t h, int32_t key, int64_t value);

/* tsvd_set_init — host fp64 initial samples x, k x n row-major (= n x k column-major:
 * row l is component l's x, NOT normalised; the library normalises it).  Copied.
 * Errors: TSVD_ERR_ARG (NULL). */
tsvd_status tsvd_set_init(tsvd_t h, const double *V0);

/*
 * tsvd_set_dense — this rank's slab of A, fp32.  ROW_MAJOR: rows A[row_begin:row_end, 0:n] with
 * leading dimension ld >= n (elements between rows).  COL_MAJOR: columns A[0:m, row_begin:row_end]
 * (the range counts columns) with ld >= m (elements between columns).  Layouts that need the
 * transposed copy (see tsvd_create) take the whole matrix (range [0, major dimension)).
 * mem = DEVICE: the pointer is used in place when it
 * is 16-byte aligned and ld % 4 == 0, otherwise copied once into a padded device buffer.
 * mem = HOST_*: copied host->device inside every tsvd_run (end-to-end semantics).  If the slab
 * does not fit in HBM (or TSVD_OPT_PLACEMENT = 2) the run is out of memory of degree 1:
 * a prefix of rows stays resident and the remaining rows are streamed every pass in row batches
 * (collinear batching) through a q_s-slot device ring on a copy stream, overlapped with
 * the fused kernel.  Pageable input is page-locked (cudaHostRegister) for the
 * duration of a streamed run.
 * The union of all ranks' slabs must be [0, m) ([0, n) for COL_MAJOR) with contiguous, disjoint
 * ranges.
 * Errors: TSVD_ERR_ARG (NULL, ld too small), TSVD_ERR_SHAPE (range outside the major dimension or empty),
 *         TSVD_ERR_NOMEM (device input that is unaligned and has no room for an aligned copy).
 */
tsvd_status tsvd_set_dense(tsvd_t h, const float *A, int64_t ld, int64_t row_begin, int64_t row_end, tsvd_mem mem);

/*
 * tsvd_set_csr — this rank's sparse row slab rows [row_begin, row_end) in CSR: row_ptr
 * int64[rows + 1] with row_ptr[0] == 0 and row_ptr[rows] == nnz, col_idx int32[nnz] (strictly
 * increasing inside a row, in [0, n)), val fp32[nnz].  mem = DEVICE: borrowed in place; HOST_*:
 * copied once.  The CSR is validated on the device, then its CSC is built once on the device
 * (histogram, scan, scatter, per-column sort: deterministic), so every iteration runs the
 * row-wise product t = A v - U c and the column-wise, atomics-free y = A^T t.  The CSC doubles
 * the slab's footprint.  Multi-GPU: the length-n partial y is summed with ncclAllReduce.
 * row_ptr's ends are read back and checked for device input too (two 8-byte copies) before any
 * kernel indexes col_idx / val with them.
 * Errors: TSVD_ERR_ARG (NULL arrays, row_ptr[0] != 0 or row_ptr[rows] != nnz, decreasing row_ptr,
 *         columns out of range or unsorted), TSVD_ERR_SHAPE, TSVD_ERR_UNSUPPORTED (m < n; n or rows >
 *         2^31 - 1), TSVD_ERR_CUDA / NOMEM.
 */
tsvd_status tsvd_set_csr(tsvd_t h, const int64_t *row_ptr, const int32_t *col_idx, const float *val, int64_t nnz,
                         int64_t row_begin, int64_t row_end, tsvd_mem mem);

/*
 * tsvd_set_factors — resume / inject the deflation state: the first l components
 * (checkpoint after component l).  Host buffers: U this rank's slab, (row_end -
 * row_begin) x l fp32 row-major; S fp64[l]; V n x l fp64 row-major (m < n: U is m x l fp32,
 * replicated, and V this rank's slab of rows, fp64).  A later tsvd_run starts at component l.
 * With l > 0 the explicit-Gram state (TSVD_OPT_METHOD = 1: P = A^T U, Q = U^T U) is invalidated,
 * so a METHOD = 1 run after an injection fails with TSVD_ERR_UNSUPPORTED unless it restarts from
 * l = 0.  Errors: TSVD_ERR_ARG (l < 0 or > k, NULL with l > 0), TSVD_ERR_STATE.
 */
tsvd_status tsvd_set_factors(tsvd_t h, int32_t l, const float *U, const double *S, const double *V);

/*
 * tsvd_gram_apply — ONE implicit Gram-vector product y = X'^T (X' v) for the current l
 * factors (Eq. 2 in exact factored form; includes the cross-rank all-reduce).  v, y: host
 * fp64[min(m, n)] (m < n: y = X' X'^T v, Eq. 3; v is used as given, not normalised).  Blocking.
 * Errors: TSVD_ERR_STATE, CUDA/NCCL.
 */
tsvd_status tsvd_gram_apply(tsvd_t h, const double *v, double *y);

/*
 * tsvd_run — Alg. 1 from the current component to k (blocking, internal stream).
 * Returns TSVD_OK, TSVD_WARN_NOT_CONVERGED, TSVD_WARN_RANK_EXHAUSTED (k_found < k) or an error.
 */
tsvd_status tsvd_run(tsvd_t h);

/* tsvd_get_U_S_V — copy results to caller-owned host buffers (any may be NULL):
 * U: (row_end-row_begin) x k fp32 row-major (this rank's slab), S: fp64[k], V: n x k fp32
 * row-major.  m < n: U is m x k (replicated) and V is this rank's slab, (row_end-row_begin) x k.
 * Columns >= k_found are zero. */
tsvd_status tsvd_get_U_S_V(tsvd_t h, float *U, double *S, float *V);

/* tsvd_get_info — k_found, per-component iteration counts iters[k] and final |v0 . v1| dots[k]
 * (any pointer may be NULL). */
tsvd_status tsvd_get_info(tsvd_t h, int32_t *k_found, int32_t *iters, double *dots);

/* tsvd_get_report — JSON report (plan, iterations, timings, bytes) into buf (NUL-terminated,
 * truncated to cap).  Returns TSVD_ERR_ARG if cap == 0. */
tsvd_status tsvd_get_report(tsvd_t h, char *buf, size_t cap);

/* tsvd_time_gram_kernel — average duration (ms) of `reps` back-to-back launches of the fused
 * Gram-vector kernel on the current state, timed with CUDA events on the library stream. */
tsvd_status tsvd_time_gram_kernel(tsvd_t h, int32_t reps, double *ms_per_launch);

/* tsvd_get_stream — the handle's CUDA stream (cudaStream_t) on which every kernel of the path is
 * launched; lets a caller bracket calls with CUDA events on the launching stream.  NULL if h is. */
void *tsvd_get_stream(tsvd_t h);

/* tsvd_last_error — message of the last failing call on h (static string if h == NULL). */
const char *tsvd_last_error(tsvd_t h);

/* tsvd_destroy — free everything the handle owns.  Safe on NULL. */
void tsvd_destroy(tsvd_t h);

#ifdef __cplusplus
}
#endif
#endif /* TSVD_H */
