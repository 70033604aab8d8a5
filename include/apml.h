/*
 * apml.h -- C ABI of libapml.so, the B200 (sm_100a) sparse APML / CUDA-APML hot path.
 *
 * The method: Sharifipour et al., "From Theory to Throughput: CUDA-Optimized APML for
 * Large-Batch 3D Learning" (arXiv 2512.19743).  Citations are PAPER.md line numbers,
 * written P:<line>, with the section / equation / algorithm they fall in.
 *
 * What one call computes, per (pred, gt) pair b of a batch (Algorithm 1):
 *   C_ij = ||x_i - y_j||_2                                  (section III-A)
 *   per row i (K = M) and per column j (K = N): min, second minimum of the multiset,
 *   g = max(c~(2) + delta, eps_g), T = -log((1-p_min)/((K-1) p_min)) / g
 *                                                          (Eq. (1); clamp P:140)
 *   s = exp(-T (C - C_min)), keep s >= tau                  (section III-B)
 *   normalise each line by its kept sum                     (section III-C)
 *   P0 = (P_row + P_col) / 2 on the union support           (a missing
 *                                                            direction counts as 0)
 *   L_iter x { column scaling Eq. (3), row scaling Eq. (4) } with eps_stab
 *   loss_b = sum_t v_t ||x_i - y_j||                        (section III-D)
 * and its gradient with respect to pred (Eq. (5)).  No N x M buffer is ever
 * allocated: memory is O(B (capacity + N + M)).
 *
 * Conventions for every entry point
 *   - Point buffers are fp32, xyz-interleaved (array of structs): pred [B][N][3],
 *     gt [B][M][3]; d = 3 is fixed.  Pointers to point / loss / gradient buffers are
 *     CUDA DEVICE pointers unless the function name ends in _host.
 *   - All device work is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *     the legacy default stream).  No entry point synchronises the device unless its
 *     comment says so.
 *   - Ownership: the caller owns every buffer it passes; the library owns the context's
 *     internals (allocated through the caller's apml_allocator, or cudaMallocAsync when
 *     the allocator is NULL) and releases them in apml_ctx_destroy.
 *   - Errors: every function returning apml_status validates its arguments on the host
 *     before launching anything; on a non-OK status nothing has been written to caller
 *     buffers and apml_last_error() returns a thread-local message.
 *   - Threading: re-entrant; one context per forward call.
 */
#ifndef APML_H
#define APML_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APML_ABI_VERSION 3

#if defined(__GNUC__)
#define APML_API __attribute__((visibility("default")))
#else
#define APML_API
#endif

typedef enum {
    APML_OK = 0,
    APML_ERR_INVALID_ARG = 1, /* hyper-parameter outside its domain, NULL pointer */
    APML_ERR_SHAPE = 2,       /* B, N or M < 1, B > 32767, N, M >= 2^30, capacity >= 2^31 */
    APML_ERR_NONFINITE = 3,   /* non-finite coordinate (only with APML_FLAG_CHECK_FINITE) */
    APML_ERR_CAPACITY = 4,    /* support exceeded the emit capacity and could not be retried,
                                 or a pair's support reached 2^31 entries (the saturated count) */
    APML_ERR_CUDA = 5,        /* a CUDA runtime call failed */
    APML_ERR_OOM = 6,         /* the allocator returned NULL */
    APML_ERR_STATE = 7        /* backward on a context without saved state, or called twice */
} apml_status;

typedef enum {
    APML_GRAD_FULL = 0,          /* through softmax (incl. T via the gap), symmetrisation and
                                    Sinkhorn: "differentiates through the same sparse
                                    computation graph" */
    APML_GRAD_PLAN_DETACHED = 1  /* transport weights held constant: Eq. (5) only */
} apml_grad_mode;

/* flags */
#define APML_FLAG_SYNC_CHECK   1u /* after emission, read the per-pair support counts back
                                     (one device->host sync) and re-run with an exact
                                     capacity if any pair overflowed.  Without it the call is
                                     sync-free / graph-capturable and an overflowed pair gets
                                     a NaN loss (reported by apml_ctx_stats). */
#define APML_FLAG_CHECK_FINITE 2u /* scan the inputs for NaN/Inf first (one extra pass + sync) */
#define APML_FLAG_STAGE_TIMING 4u /* record CUDA events between the stages below (on the launch
                                     stream); read them with apml_ctx_stage_times */
#define APML_FLAG_MARKS_SHIFT 8  /* bits 8..16: with APML_FLAG_STAGE_TIMING, record only the stage
                                     marks k whose bit (8 + k) is set (0 = all nine).  Stage s
                                     (0..5) spans marks s, s+1 (Pass A, both directions in one
                                     launch: marks 1, 3); the backward spans marks 7, 8.  Each
                                     mark inside a captured CUDA graph is an event-record node
                                     that costs a few microseconds of pipelining (measured: all
                                     nine add ~40 us to a 306 us C2 step), so a timed loop
                                     brackets only the kernel it needs. */
#define APML_FLAG_MARKS(mask) ((uint32_t)(mask) << APML_FLAG_MARKS_SHIFT)
#define APML_FLAG_UNIFORM_FALLBACK 8u /* stability mode of dense APML (the sparse kernel
                                     "writes a uniform distribution over the corresponding row
                                     or column") instead of the gap clamp of CUDA-APML
                                     (the default): a line whose gap c~(2) = c2 - m is
                                     below eps_g keeps all K entries with P = 1/K and passes no
                                     gradient through its softmax.  Opt-in, for parity studies:
                                     such a line is dense (K entries), outside the O(nnz) memory
                                     contract; the capacity retry (APML_FLAG_SYNC_CHECK) sizes
                                     for it. */

/* Stages timed with APML_FLAG_STAGE_TIMING (indices into apml_ctx_stage_times' output). */
enum {
    APML_STAGE_STAGING = 0,     /* S0: AoS -> padded SoA + float4 copies */
    APML_STAGE_PASSA_ROWS = 1,  /* S1: row min / second min sweep (k_line_top2, B N M pairs) */
    APML_STAGE_PASSA_COLS = 2,  /* S1: column min / second min sweep (k_line_top2, B N M pairs);
                                   0 when both directions ran in one launch (counted under ROWS) */
    APML_STAGE_LINE_INFO = 3,   /* S2: line constants */
    APML_STAGE_EMIT = 4,        /* S3: emit sweep (k_emit, B N M pairs) */
    APML_STAGE_SPARSE_FWD = 5,  /* S4-S7: CSR/CSC, normalisation, Sinkhorn, loss (k_sparse_fwd) */
    APML_STAGE_SPARSE_BWD = 6,  /* S8: reverse pass (k_sparse_bwd) */
    APML_NUM_STAGES = 7
};

typedef struct {
    float   p_min;        /* Eq. (1); 0 < p_min < 1 and p_min > 1/K for every line
                             length K in {N, M} with K > 1; default 0.9 (paper defers) */
    float   tau;          /* pruning threshold on the UNNORMALISED similarity, keep s >= tau,
                             0 <= tau <= 1; default 1e-8 */
    int32_t l_iter;       /* Sinkhorn iterations, >= 0; default 10 */
    float   eps_stab;     /* Sinkhorn stability constant, > 0; default 1e-8 */
    float   delta;        /* g = c~(2) + delta, >= 0; default 1e-6 */
    float   eps_g;        /* gap clamp g = max(g, eps_g), > 0; default 1e-8 */
    float   eps_dist;     /* Eq. (5) denominator, > 0; default 1e-8 */
    int32_t grad_mode;    /* apml_grad_mode; default APML_GRAD_FULL */
    int32_t capacity;     /* emit capacity per pair in entries per point: cap = capacity*(N+M),
                             clipped to N*M; 0 = default: plans 6; eager calls 6 / 5 / 4 / 3
                             for N+M < 2048 / 8192 / 65536 / larger (Fig. 2's falling support
                             per point; an overflow is retried with the exact count) */
    uint32_t flags;       /* APML_FLAG_*; default APML_FLAG_SYNC_CHECK */
} apml_config;

/* Stream-ordered allocator used for all library-owned device memory. */
typedef struct {
    void* (*alloc)(size_t bytes, void* stream, void* user);
    void  (*free)(void* ptr, size_t bytes, void* stream, void* user);
    void* user;
} apml_allocator;

/* Per-call diagnostics (SPEC LossResult analogue). */
typedef struct {
    int64_t nnz_total;      /* |Omega_tau| summed over pairs (entries carrying a row or column flag) */
    int64_t emitted_total;  /* emitted entries incl. second-argmin-only entries (tau > tau*) */
    int64_t clamp_count;    /* lines whose gap was clamped to eps_g */
    int64_t capacity;       /* per-entry capacity per pair actually used (entries; after the
                               support read-back: the largest pair's count, + 64) */
    int64_t overflow_pairs; /* pairs whose support exceeded capacity (their loss is NaN) */
    int64_t bytes_ctx;      /* device bytes owned by the context (both allocations) */
    int64_t launches;       /* kernels launched so far by this context (forward + backward) */
    int64_t sweep_evals[3]; /* (i, j) distance evaluations executed by the sweeps of the last
                               forward: [0] Pass A rows, [1] Pass A columns, [2] emit.  Full
                               sweeps: every padded pair (B Np Mp); spatially culled sweeps:
                               counted on the device (cell-grid sweeps: the (own point, staged
                               point) pairs evaluated, both emit passes in [2]; the tile walk,
                               APML_CULL_MODE=0: the 32 x 32 blocks evaluated) */
    int64_t uniform_count;  /* lines given the uniform fallback (APML_FLAG_UNIFORM_FALLBACK) */
} apml_stats;

/* Caller-supplied, stream-ordered collectives for the row-sharded mode (torch.distributed /
 * NCCL over NVLink in practice).  Both must be called by every rank in the same order with
 * the same n; they return 0 on success.
 *   allreduce_sum_f32: buf[0..n) <- sum over ranks of buf[0..n), in place, device memory.
 *   allgather_f32:     recv[r*n .. (r+1)*n) <- rank r's send[0..n), device memory (the
 *                      library also moves int32 bit patterns through it; no arithmetic). */
typedef struct apml_nvls apml_nvls; /* opaque: an NVLink SHARP (NVLS) multicast team, below */

typedef struct {
    int32_t rank, world;
    int (*allreduce_sum_f32)(float* buf, int64_t n, void* stream, void* user);
    int (*allgather_f32)(const float* send, float* recv, int64_t n, void* stream, void* user);
    void* user;
    /* ABI 3.  Optional (NULL = unused):
     *   allgather_bytes: HOST all-gather of n bytes per rank, recv[r*n ..) <- rank r's send;
     *                    blocking; used only by apml_nvls_create to exchange handles.
     *   nvls:            a team from apml_nvls_create; when set, every per-iteration Sinkhorn
     *                    column sum (Eq. (3) forward and its reverse, X3) is reduced INSIDE the
     *                    library's kernels through NVSwitch multicast memory (multimem
     *                    ld_reduce) instead of the allreduce_sum_f32 callback. */
    int (*allgather_bytes)(const void* send, void* recv, int64_t n, void* user);
    apml_nvls* nvls;
} apml_comm;

/* NVLS team for the row-sharded mode (north_star "per-iteration column sums
 * are allreduced over NVLink"): one multicast object of `bytes` bytes bound to a buffer on
 * every rank's device (driver API: cuMulticastCreate / AddDevice / BindMem; rank 0 creates it
 * and passes its POSIX file descriptor to the other ranks of the node over a Unix socket,
 * SCM_RIGHTS; comm->allgather_bytes carries the rendezvous).  Each rank writes its partial
 * column sums into its own copy; a kernel then reads the sum over all ranks with ONE
 * multimem.ld_reduce per value, after a cross-GPU barrier made of a multicast red.add on a
 * flag word in the same memory -- compute and collective in one stream-ordered pair of
 * kernels, no NCCL call and no host involvement per iteration.  Collective over comm (every
 * rank, same bytes); ranks must share one node.  bytes >= 8 * B * M + 256 for a problem of B
 * pairs with M gt points.  Errors: APML_ERR_INVALID_ARG (no allgather_bytes for world > 1),
 * APML_ERR_CUDA (no multicast support, driver failure); *out = NULL then. */
APML_API apml_status apml_nvls_create(const apml_comm* comm, size_t bytes, apml_nvls** out);
/* 1 when the team is a real multicast object; 0 for a one-device team that the driver would
 * not build as one (a one-GPU box: cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE for
 * numDevices = 1), which then lives in plain device memory and runs the same kernels with
 * ordinary atomics and loads (the sum over one rank; APML_NVLS_STRICT=1 makes it an error). */
APML_API int apml_nvls_is_multicast(const apml_nvls* team);
/* Collective: unmap and release (every rank). */
APML_API void apml_nvls_destroy(apml_nvls* team);

typedef struct apml_ctx apml_ctx; /* opaque: state saved by forward for backward */

APML_API int apml_abi_version(void);

/* Paper / DESIGN.md defaults into *cfg. */
APML_API void apml_config_default(apml_config* cfg);

/* Forward, Algorithm 1 lines 1-8 for B independent pairs.
 *   pred   device [B][N][3] fp32 (x_i, predicted points)
 *   gt     device [B][M][3] fp32 (y_j, reference points)
 *   cfg    NULL -> apml_config_default
 *   alloc  NULL -> cudaMallocAsync / cudaFreeAsync on `stream`
 *   loss   device [B] fp32, per-pair <P, C> (unreduced; the caller reduces)
 *   ctx_out NULL -> no backward state is kept; else *ctx_out receives a context that the
 *          caller must release with apml_ctx_destroy (also on the error path it is NULL).
 * Synchronises the host only with APML_FLAG_SYNC_CHECK / APML_FLAG_CHECK_FINITE. */
APML_API apml_status apml_forward(const float* pred, const float* gt, int64_t B, int64_t N, int64_t M,
                         const apml_config* cfg, const apml_allocator* alloc, void* stream,
                         float* loss, apml_ctx** ctx_out);

/* Ragged batches (MM-Fi clouds of varying size): pair b uses only its first
 * n_sizes[b] pred points and m_sizes[b] gt points of the padded [B][N][3] / [B][M][3] buffers
 * (the padding is never read), every line length K in Eq. (1) is the PAIR's (m_b for rows,
 * n_b for columns), and the result per pair equals apml_forward on that pair alone.
 * n_sizes, m_sizes: HOST arrays [B] with 1 <= n_b <= N, 1 <= m_b <= M (else APML_ERR_SHAPE).
 * apml_backward writes zeros into the padding rows of grad_pred (and of grad_gt).
 * Ragged contexts run the full (non-culled) sweeps and the per-pair cluster sparse stage.
 * Errors as apml_forward. */
APML_API apml_status apml_forward_ragged(const float* pred, const float* gt, int64_t B, int64_t N, int64_t M,
                                         const int64_t* n_sizes, const int64_t* m_sizes, const apml_config* cfg,
                                         const apml_allocator* alloc, void* stream, float* loss, apml_ctx** ctx_out);

/* Forward with one cloud's pred rows SHARDED over the ranks of `comm` (north_star: "pred
 * rows shard and per-iteration column sums are all-reduced").  This rank holds pred rows
 * [row_offset, row_offset + N_local) of every pair (pred_local device [B][N_local][3]) and
 * the whole gt (device [B][M][3]); N_global = sum of N_local over ranks (the column line
 * length K of Eq. (1)).  Row statistics, the row softmax and the row scaling are local;
 * column statistics are merged with one all-gather (X2), and the column softmax sum, the
 * column argmin, every Sinkhorn column sum (Eq. (3), X3) and the loss are all-reduced.
 * loss (device [B]) receives the GLOBAL per-pair loss on every rank.  The returned context
 * drives the matching sharded backward through apml_backward (grad_pred = this rank's rows).
 * Collective and synchronising like apml_forward; all ranks must pass the same B, M, cfg. */
APML_API apml_status apml_forward_rowsharded(const float* pred_local, const float* gt, int64_t B,
                                             int64_t N_local, int64_t row_offset, int64_t N_global,
                                             int64_t M, const apml_config* cfg,
                                             const apml_allocator* alloc, const apml_comm* comm,
                                             void* stream, float* loss, apml_ctx** ctx_out);

/* Backward: grad_pred [B][N][3] (device, overwritten) = sum_b grad_loss[b] *
 * d loss_b / d pred_b.  grad_loss device [B].  One backward per context (ERR_STATE after). */
APML_API apml_status apml_backward(apml_ctx* ctx, const float* grad_loss, float* grad_pred, void* stream);

/* apml_backward plus, when grad_gt != NULL, the gradient with respect to gt (SURVEY 8(f)-3,
 * for settings where gt is itself predicted).  The loss depends on gt only through the costs
 * c_ij, so by Eq. (5) with x and y exchanged:
 *     grad_gt[b][j] = - sum_i w_ij (x_i - y_j),  w_ij = cbar_ij / (c_ij + eps_dist),
 * the same per-entry adjoints cbar as grad_pred (full or plan-detached mode).
 * grad_gt: device [B][M][3] fp32, caller-owned, overwritten (NaN rows for overflowed pairs).
 * Row-sharded contexts: every rank passes a full [B][M][3] buffer and receives the sum over
 * ranks (one allreduce_sum_f32 of 3 B M floats through the context's apml_comm).
 * Errors as apml_backward. */
APML_API apml_status apml_backward_ex(apml_ctx* ctx, const float* grad_loss, float* grad_pred, float* grad_gt,
                                      void* stream);

/* Reusable plans (CUDA-graph capturable steps).  apml_plan_create allocates, once, every
 * device buffer of a B x N x M problem (emit capacity = cfg->capacity x (N + M) entries per
 * pair) and returns a context; apml_plan_forward then runs the forward on new pred / gt with
 * NO allocation, NO host synchronisation and NO host read (APML_FLAG_SYNC_CHECK and
 * APML_FLAG_CHECK_FINITE are ignored), so a training step `apml_plan_forward +
 * apml_backward[_ex]` can be captured into a CUDA graph and replayed.  Exception: with
 * cfg->capacity == 0 (the default) the per-entry arrays (CSR / CSC, ~64 B per entry) are
 * sized by the plan's FIRST forward -- 1.25 x the largest per-pair support it emits, one count
 * read-back and one allocation in that call only -- so that memory follows the support, not
 * the emit capacity; if that first forward is itself being captured they take the emit
 * capacity.  A later input whose support exceeds that size is reported like a capacity
 * overflow (below).  A pair whose support
 * exceeds the capacity gets a NaN loss / gradient (apml_ctx_stats reports it).  Each
 * apml_plan_forward allows one backward; the introspection calls read the last forward.
 * Destroy with apml_ctx_destroy.  Errors: as apml_forward; APML_ERR_STATE for a context that
 * is not a plan. */
APML_API apml_status apml_plan_create(int64_t B, int64_t N, int64_t M, const apml_config* cfg,
                                      const apml_allocator* alloc, void* stream, apml_ctx** plan_out);
APML_API apml_status apml_plan_forward(apml_ctx* plan, const float* pred, const float* gt, void* stream,
                                       float* loss);

/* Forward AND backward of a plan in one call (a training step whose grad_loss -- device [B],
 * e.g. ones for a sum reduction -- is known before the call; JAX-style value-and-grad).
 * loss device [B], grad_pred device [B][N][3] overwritten; results equal apml_plan_forward +
 * apml_backward bit for bit.  With APML_FUSED=1 in the environment the sparse forward and
 * backward of each pair run in ONE cluster kernel (k_sparse_fwdbwd2: no kernel boundary
 * between them) -- measured no faster (C2 201 vs 90 + 106 us; C3 equal), so off by default.
 * Capturable in a CUDA graph.  Errors as apml_plan_forward / apml_backward. */
APML_API apml_status apml_plan_forward_backward(apml_ctx* plan, const float* pred, const float* gt,
                                                const float* grad_loss, void* stream, float* loss,
                                                float* grad_pred);

/* One training step of a plan on HOST buffers -- the end-to-end call: copies pred_host
 * [B][N][3] and gt_host [B][M][3] (fp32, host; pinned memory gives async copies) into
 * plan-owned device buffers, runs the forward and the backward with grad_loss = 1 for every
 * pair (sum reduction, the plan's grad_mode), and copies loss [B] and grad_pred [B][N][3]
 * back to loss_host / grad_pred_host.  The device part is captured once into a CUDA graph
 * owned by the plan and replayed on later calls (not on the legacy NULL stream, nor with
 * APML_HOST_GRAPH=0 in the environment).  Synchronises `stream` (NULL: the plan's stream)
 * before returning.  A pair whose support exceeds the plan's capacity gets NaN outputs.
 * Errors: APML_ERR_STATE (not a plan), APML_ERR_INVALID_ARG (NULL buffer), APML_ERR_OOM,
 * APML_ERR_CUDA; nothing is written to the host outputs on error. */
APML_API apml_status apml_plan_step_host(apml_ctx* plan, const float* pred_host, const float* gt_host,
                                         void* stream, float* loss_host, float* grad_pred_host);

/* Diagnostics; SYNCHRONISES the context's stream.  nnz_per_pair: host [B] or NULL. */
APML_API apml_status apml_ctx_stats(const apml_ctx* ctx, int64_t* nnz_per_pair, apml_stats* out);

/* Introspection (tests / diagnostics).  Copies pair b's support to the host in CSR order
 * (row-major, j ascending); SYNCHRONISES.  *count: in = capacity of the arrays, out =
 * number of entries (APML_ERR_CAPACITY if the arrays are too small; *count is still set).
 * flags: 1 = kept by the row softmax, 2 = kept by the column softmax, 0 = second-argmin
 * entry emitted only for the T-gradient (tau > tau*, reading R14).  p0 = P0, v = the final
 * plan a_i P0_ij b_j.  Any array pointer may be NULL. */
APML_API apml_status apml_ctx_support(const apml_ctx* ctx, int64_t b, int64_t* count, int32_t* i,
                                      int32_t* j, int32_t* flags, float* p0, float* v);

/* Per-line statistics of pair b (dir 0: rows, length N; dir 1: columns, length M), host
 * arrays, SYNCHRONISES: m = min distance, c2 = second smallest distance, T = Eq. (1)
 * temperature (0 for K = 1 lines), argmin / second = index of the other cloud (-1 if none).
 * Any pointer may be NULL. */
APML_API apml_status apml_ctx_lines(const apml_ctx* ctx, int64_t b, int32_t dir, float* m,
                                    float* c2, float* T, int32_t* argmin, int32_t* second);

/* Per-stage device durations in milliseconds (ms[APML_NUM_STAGES]; stages not run are 0)
 * for a context created with APML_FLAG_STAGE_TIMING.  SYNCHRONISES on the last event. */
APML_API apml_status apml_ctx_stage_times(const apml_ctx* ctx, float* ms, int32_t n);

/* Release a context (stream-ordered free on the context's stream).  NULL is a no-op. */
APML_API void apml_ctx_destroy(apml_ctx* ctx);

/* End-to-end convenience on HOST buffers: copies pred/gt host->device, runs forward and
 * backward with grad_loss = 1 for every pair (sum reduction), copies loss [B] and
 * grad_pred [B][N][3] back to the host.  Pinned host memory gives async copies.
 * Synchronises `stream` before returning. */
APML_API apml_status apml_loss_grad_host(const float* pred_host, const float* gt_host, int64_t B,
                                int64_t N, int64_t M, const apml_config* cfg,
                                const apml_allocator* alloc, void* stream, float* loss_host,
                                float* grad_pred_host);

/* Thread-local message describing the last non-OK status on this thread. */
APML_API const char* apml_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* APML_H */
