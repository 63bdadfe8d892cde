/*
 * cavs.h — C-ABI of the B200-native level-batched vertex-function engine.
 *
 * The hot path of Cavs (Zhang et al., arXiv 1712.04048; PAPER.md = the paper's
 * LaTeX at /root/reference/PAPER.md, "P:Lnnn" = its line nnn): a static vertex
 * function F is declared once and evaluated, forward and backward, over a
 * minibatch of K instance-specific input graphs G (§1; Fig. 1c P:L120-125;
 * P:L226-234 §3), batching all "activated" vertices of all K graphs into one
 * task per step (Algorithm 1, §3.2).
 *
 * Calls, in order:  cavs_create -> cavs_workspace_bytes -> cavs_set_workspace
 *   -> per batch: cavs_load_graphs -> cavs_schedule -> cavs_forward -> cavs_backward
 *
 * Conventions
 *  - Every call returns a cavs_status; CAVS_OK == 0.  No exceptions, abort or
 *    exit cross this boundary.  cavs_last_error() gives a message.
 *  - All device work is enqueued on the context's CUDA stream (cavs_create /
 *    cavs_set_stream) and is asynchronous, EXCEPT: cavs_schedule with T_out != NULL
 *    waits for a small header (status word, T, level_ptr[0..T]) read back from the
 *    device; with T_out == NULL the header is read back asynchronously and consumed by
 *    the next cavs_forward (after it has enqueued the pull, so the wait overlaps device
 *    work) or cavs_get_schedule; the *_host entry points synchronise at the end.
 *  - The library never allocates device memory: all scratch is carved from one
 *    caller-owned device buffer (cavs_set_workspace).  The caller (PyTorch in
 *    this repo) owns memory, streams and process groups.
 *  - A context is single-threaded; use one per GPU / rank.
 *  - "Global vertex id" of local vertex u of graph k = graph_ptr[k] + u
 *    (SPEC S:L251).  The child order inside a CSR row is the gather index k of
 *    Fig. 5 (`gather(k)`) — reading Z3 of DESIGN.md.
 *
 * Packed fp32 parameters (caller memory, same layout for dparams):
 *  Tree-LSTM / LSTM (cell CAVS_CELL_TREE_LSTM; LSTM is N = 1), Fig. 5 P:L321-328:
 *     W[4h x d] rows (i,f,o,u) | U_iou[3h x h] rows (i,o,u) | U_f[h x h] | b[4h] (i,f,o,u)
 *     (child-sum form with one U_f shared by all k, reading Z6)
 *  Tree-FC (CAVS_CELL_TREE_FC, N = 2), "a single fully-connected layer" P:L608,
 *  reading Z7: h = tanh(W_c [h_l ; h_r] + W_x x + b):
 *     W_c[h x 2h] (cols h_l | h_r) | W_x[h x d] | b[h]
 *  Row-major everywhere.
 */
#ifndef CAVS_H_
#define CAVS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum cavs_status {
  CAVS_OK = 0,
  CAVS_E_INVALID = 1,     /* bad argument / malformed graph (K<1, empty graph, id out of range, sizes) */
  CAVS_E_ARITY = 2,       /* a vertex has more than N children */
  CAVS_E_CYCLE = 3,       /* G is not a DAG: some vertex is never activated */
  CAVS_E_FANOUT = 4,      /* reserved (round 1: fan-out rejected).  DAG inputs -- a vertex with
                             several parents, or a child listed twice -- are accepted since
                             round 2 (NEXT-3); this code is no longer returned */
  CAVS_E_STATE = 5,       /* call out of order (e.g. backward before forward) */
  CAVS_E_CAPACITY = 6,    /* batch exceeds the context's max_* or the workspace is too small */
  CAVS_E_CUDA = 7,        /* a CUDA runtime/driver error; see cavs_last_error */
  CAVS_E_UNSUPPORTED = 8  /* e.g. bf16 tensor-core mode with h or d not a multiple of 64 */
} cavs_status;

typedef enum cavs_cell { CAVS_CELL_TREE_LSTM = 0, CAVS_CELL_TREE_FC = 1 } cavs_cell;

typedef enum cavs_precision {
  CAVS_FP32 = 0,   /* fp32 operands, FFMA GEMMs, accurate expf/tanhf: parity 1e-5 */
  CAVS_BF16 = 1    /* bf16 GEMM operands (RN-even), fp32 accumulate on tcgen05 tensor
                      cores, all elementwise math and state in fp32: parity 2e-2 */
} cavs_precision;

typedef struct cavs_desc {
  int32_t cell;          /* cavs_cell */
  int32_t N;             /* arity: max children per vertex (gather slots); Tree-FC requires 2 */
  int32_t h;             /* hidden size */
  int32_t d;             /* input (pull) size */
  int32_t precision;     /* cavs_precision */
  int32_t max_graphs;    /* capacity: K per batch */
  int32_t max_vertices;  /* capacity: V per batch (sum over graphs) */
  int32_t max_x;         /* capacity: pull records n_x per batch */
} cavs_desc;

typedef struct cavs_ctx cavs_ctx;

/* Number of fp32 entries of the packed parameter vector (layout above). */
size_t cavs_param_count(int32_t cell, int32_t N, int32_t h, int32_t d);

/* Fix F (cell, N, h, d, precision) and capacities ("declared ... and optimized once").
 * `cuda_stream` is a cudaStream_t (NULL = legacy default stream).  The context
 * owns no device memory until cavs_set_workspace.
 * Errors: CAVS_E_INVALID (N<1, h<1, d<1, unknown cell/precision, capacities < 1),
 *         CAVS_E_UNSUPPORTED (BF16 with h % 64 or d % 64 != 0; Tree-FC with N != 2),
 *         CAVS_E_CUDA (bad device). */
cavs_status cavs_create(const cavs_desc* desc, int device, void* cuda_stream, cavs_ctx** out);

/* Change the stream subsequent calls are enqueued on. */
cavs_status cavs_set_stream(cavs_ctx* ctx, void* cuda_stream);

/* Bytes of device scratch the context needs for its capacities (all arenas of
 * the dynamic-tensor plan, Fig. 7, plus schedule arrays and weight copies). */
size_t cavs_workspace_bytes(const cavs_ctx* ctx);

/* Hand the context its scratch: `dev` must be device memory of >= cavs_workspace_bytes,
 * 256-byte aligned, kept alive (and not used by anyone else) until cavs_destroy.
 * The buffer is zeroed here (stream-ordered).  Errors: CAVS_E_CAPACITY, CAVS_E_INVALID. */
cavs_status cavs_set_workspace(cavs_ctx* ctx, void* dev, size_t bytes);

/* Load the K input graphs of one minibatch as CSR child lists per instance
 * ("reads training samples and their associated graphs", §4).
 *   graph_ptr [K+1]: global vertex offsets, graph_ptr[0] = 0, graph_ptr[K] = V
 *   child_ptr [V+1]: CSR row pointers over global vertices, child_ptr[V] = E
 *   child_idx [E]  : children as INSTANCE-LOCAL ids (0 .. n_k-1); row order = gather index k.
 *                    A vertex may be the child of several parents and may appear twice in one
 *                    row (DAG inputs): its h / c are then gathered into every slot
 *                    that lists it and the gradients of all those slots are ADDED in a
 *                    fixed order (ascending parent position, then slot), so results are
 *                    deterministic.  E <= N * max_vertices.
 * `on_device` != 0: the three arrays are device pointers, read (and copied into the
 * workspace) by the first kernel of the next cavs_schedule — keep them alive and unmodified
 * until that kernel ran (stream order), i.e. until any later call on the stream completes.
 * `on_device` == 0: host pointers, copied host->device here (stream-ordered; borrowed until
 * that copy completes).
 * Host-side checks: K, V, E within capacity (CAVS_E_CAPACITY), K >= 1 (CAVS_E_INVALID).
 * Content checks run on the device and are reported by cavs_schedule.
 * Resets the state to LOADED. */
cavs_status cavs_load_graphs(cavs_ctx* ctx, int32_t K, int32_t V, int32_t E,
                             const int32_t* graph_ptr, const int32_t* child_ptr,
                             const int32_t* child_idx, int on_device);

/* Algorithm 1's task partition on the device: level(v) = 0 without
 * children, else 1 + max over children; V_t = {v : level(v) = t} ordered by ascending
 * global id; T = number of tasks.  Also builds the dynamic-tensor plan (positions,
 * child/parent slots; Fig. 7, Alg. 2).  Validates the graphs.
 * T_out != NULL: waits for the header (status, T, level_ptr) and returns T and the graphs'
 * validation errors here.  T_out == NULL: returns after enqueueing; the validation errors
 * are then returned by the next cavs_forward / cavs_get_schedule (which consume the header)
 * and the context falls back to LOADED.
 * A batch with fan-out anywhere runs the DAG path: per-task gather in the forward and a
 * pull-reduce over a parent CSR before each task's dF in the backward (the fused tree path,
 * where each child's dF runs inside its unique parent's epilogue, needs a single parent).
 * Errors: CAVS_E_STATE (nothing loaded), CAVS_E_INVALID, CAVS_E_ARITY, CAVS_E_CYCLE, CAVS_E_CUDA. */
cavs_status cavs_schedule(cavs_ctx* ctx, int32_t* T_out);

/* Copy the schedule into HOST buffers (any may be NULL):
 *   level [V], level_ptr [T+1], order [V] (position -> global vertex id).  Synchronous. */
cavs_status cavs_get_schedule(cavs_ctx* ctx, int32_t* level, int32_t* level_ptr, int32_t* order);

/* Forward pass over all K graphs (Alg. 1 FORWARD + Alg. 2): the eager pull/input
 * projection for all vertices with a record, then one batched task per level
 * t = 0..T-1 (gather -> cell -> scatter/push fused in one kernel per level).
 *   params  [P]      device fp32, packed layout above
 *   x       [n_x, d] device fp32 pull records
 *   x_row   [V]      device int32: record of each global vertex, -1 = none (pull() -> 0).  Several
 *                    vertices may pull the same record (an embedding row): their dx rows are ADDED.
 *                    An entry outside [-1, n_x) is an input error found on the device: the vertex
 *                    pulls nothing and the next cavs_sync returns CAVS_E_INVALID.
 *   h_out   [V, h]   device fp32 output: push(h) of every vertex, global id order (Fig. 5)
 * Activations stay in the workspace for cavs_backward.
 * Errors: CAVS_E_STATE (not scheduled), CAVS_E_CAPACITY (n_x > max_x), CAVS_E_INVALID (NULL). */
cavs_status cavs_forward(cavs_ctx* ctx, const float* params, int32_t n_x, const float* x,
                         const int32_t* x_row, float* h_out);

/* Inference-only forward: the same pass as cavs_forward (same h_out,
 * bit for bit); the level-0 cells (the pull projection's epilogue, half the vertices of a tree
 * batch) skip the activations only dF needs (gates, memory cells) — the level kernels keep
 * their stores (a runtime check there costs the register-bound persistent kernel ~5 us).
 * A following cavs_backward fails with CAVS_E_STATE until a training cavs_forward ran.
 * Arguments, layouts, ownership and errors as cavs_forward. */
cavs_status cavs_forward_inference(cavs_ctx* ctx, const float* params, int32_t n_x, const float* x,
                                   const int32_t* x_row, float* h_out);

/* Backward pass (Alg. 1 BACKWARD): tasks in reverse order, gradients
 * ADDED; scatter is gather's adjoint, push is pull's; parameter
 * gradients are lazily batched over all vertices once after the level loop (§3.5).
 *   dh_out  [V, h]   device fp32: dL/d(push h) of every vertex (the external loss's cotangent)
 *   dparams [P]      device fp32, OVERWRITTEN with dL/dparams summed over all K graphs
 *   dx      [n_x, d] device fp32, OVERWRITTEN with dL/dx (may be NULL): row r = the sum over the
 *                    vertices that pull record r of their pull adjoint W^T dz; rows
 *                    of records no vertex pulls are 0.  Deterministic when each record is pulled at
 *                    most once (then every row is written by one store; records pulled by several
 *                    vertices are accumulated with atomic adds after a zero fill).
 * Errors: CAVS_E_STATE (no forward since the last schedule), CAVS_E_INVALID. */
cavs_status cavs_backward(cavs_ctx* ctx, const float* dh_out, float* dparams, float* dx);

/* One whole training step from HOST buffers (the end-to-end entry point): stages the
 * CSR, params, x, x_row and dh_out host->device, runs load/schedule/forward/backward,
 * and copies dparams (and dx if non-NULL, and h_out if non-NULL) device->host.
 * Host buffers should be pinned for asynchronous copies.  Synchronises at the end. */
cavs_status cavs_train_step_host(cavs_ctx* ctx, int32_t K, int32_t V, int32_t E,
                                 const int32_t* graph_ptr, const int32_t* child_ptr,
                                 const int32_t* child_idx, const float* params, int32_t n_x,
                                 const float* x, const int32_t* x_row, const float* dh_out,
                                 float* dparams, float* dx, float* h_out);

/* Pipelined end-to-end training step from HOST buffers (r02): the same work as
 * cavs_train_step_host (H2D of this step's inputs, load / schedule / forward / backward, D2H of
 * dparams) but ASYNCHRONOUS: the H2D copies run on the context's own copy stream and overlap the
 * previous step's compute, the D2H of dparams on a second copy stream; two staging slots, so at most
 * two steps are in flight and a slot is reused only after the step that last used it has copied
 * its dparams out.  The call returns after enqueueing (it may wait for the previous step's
 * schedule header, see cavs_schedule); call cavs_sync before reading `dparams` or reusing the host
 * input buffers of the last two steps.  Host buffers must be pinned.
 *   gamma_rows != NULL: the push cotangent is given for n_gamma vertices only (e.g. the roots that
 *                       carry a loss): gamma [n_gamma, h] rows of dL/dh at global vertex ids
 *                       gamma_rows[i]; every other vertex has dL/dh = 0.
 *   gamma_rows == NULL: gamma is the dense [V, h] cotangent (n_gamma = V), or n_gamma = 0 (all zero).
 *   dparams [P] host fp32: dL/dparams of this step (valid after cavs_sync).
 * Errors: as cavs_train_step_host; CAVS_E_INVALID for inconsistent gamma arguments. */
cavs_status cavs_train_step_host_async(cavs_ctx* ctx, int32_t K, int32_t V, int32_t E,
                                       const int32_t* graph_ptr, const int32_t* child_ptr,
                                       const int32_t* child_idx, const float* params, int32_t n_x,
                                       const float* x, const int32_t* x_row, int32_t n_gamma,
                                       const int32_t* gamma_rows, const float* gamma, float* dparams);

/* Next-word softmax head (§5 P:L606 "predicts the next word"): the
 * loss lives outside (F, G) (reading Z9) and is wired to F through push (h_out) and push's adjoint
 * (dh_out = dL/dh).  This is its fused softmax / cross-entropy / gradient pass over the logits of
 * M rows (the head's contractions logits = H W^T + b and dH = dlogits W are plain GEMMs):
 *   logits  [M, vocab] device fp32 (row-major)
 *   target  [M]        device int32: class of each row, < 0 = no loss at this row
 *   loss    [M]        device fp32 (nullable): logsumexp(logits_m) - logits_m[target_m] (0 without target)
 *   dlogits [M, vocab] device fp32: scale * (softmax(logits_m) - onehot(target_m)) (0 without target);
 *                      may alias logits (in place)
 * Enqueued on `stream` (a cudaStream_t, NULL = legacy default).  No context needed.
 * Errors: CAVS_E_INVALID (sizes / null pointers), CAVS_E_CUDA (launch). */
cavs_status cavs_softmax_xent(const float* logits, int32_t M, int32_t vocab, const int32_t* target, float* loss,
                              float* dlogits, float scale, void* stream);

/* Sync-free mode (r02): with `on` != 0 the host never reads the schedule header -- cavs_schedule
 * (with T_out == NULL), cavs_forward and cavs_backward only enqueue work; the kernels take the
 * number of tasks T, the first internal position level_ptr[1] and the number of roots from the
 * device, so a whole step (load on device, schedule, forward, backward) can be captured in one
 * CUDA graph and replayed.  Requires the BF16 persistent path (h % 64 == 0, h <= 512; not with
 * the opt-in K-split backward).  Forests only: an invalid batch or a DAG batch makes every kernel
 * of the step skip its work, and the next cavs_sync returns its error (CAVS_E_INVALID / ARITY /
 * CYCLE, or CAVS_E_UNSUPPORTED for a DAG).  FLOP / byte accounting of cavs_profile_read is not
 * kept in this mode (phase times are).  Errors: CAVS_E_UNSUPPORTED, CAVS_E_STATE. */
cavs_status cavs_set_sync_free(cavs_ctx* ctx, int on);

/* Data-parallel overlap hook (SURVEY §8(e) "Overlap"): `cuda_event` (a cudaEvent_t created by the
 * caller, or NULL to clear) is recorded on the context's stream by every later cavs_backward as soon
 * as all WEIGHT blocks of dparams (W, U_iou, U_f / W_c, W_x) are final -- right after the lazily
 * batched weight-gradient GEMMs, before dX and db -- so a caller can start the all-reduce
 * of those blocks on another stream while the rest of the backward runs.  The bias block is final
 * when cavs_backward's work completes.  The event stays owned by the caller.  Errors: CAVS_E_INVALID. */
cavs_status cavs_set_grad_event(cavs_ctx* ctx, void* cuda_event);

/* Wait for all work enqueued on the context's stream and report the deferred device-side input
 * errors of the calls since the last cavs_schedule: CAVS_E_INVALID if a forward met an x_row
 * entry outside [-1, n_x).  CAVS_E_CUDA on a CUDA error.  cavs_train_step_host does this itself. */
cavs_status cavs_sync(cavs_ctx* ctx);

/* Number of kernels the library launched since the context was created (diagnostic). */
int64_t cavs_kernel_launches(const cavs_ctx* ctx);

/* Per-phase device timing: with profiling on, the library records one CUDA event on its
 * stream at every phase boundary of schedule/forward/backward (no extra synchronisation)
 * and accumulates, per phase, the elapsed time, the kernel launches and the ALGORITHMIC
 * FLOPs / bytes of that phase.
 * cavs_profile(ctx, 1) resets the accumulators and starts recording; (ctx, 0) stops.
 * cavs_profile_read synchronises the stream and returns the totals of one phase. */
typedef enum cavs_phase {
  CAVS_PH_SCHEDULE = 0,   /* graph validation + level sweep + task lists (Alg. 1) */
  CAVS_PH_PREP = 1,       /* parameter repack + pull gather */
  CAVS_PH_XPROJ = 2,      /* eager pull projection fused with task 0 */
  CAVS_PH_FWD_LEVELS = 3, /* forward tasks t = 1..T-1 (level GEMM + fused cell) */
  CAVS_PH_BWD_ROOTS = 4,  /* dF at the roots */
  CAVS_PH_BWD_LEVELS = 5, /* backward tasks t = T-1..1 (dH GEMM + fused dF of the children) */
  CAVS_PH_LAZY = 6,       /* lazily batched weight-gradient GEMMs */
  CAVS_PH_DX = 7,         /* pull's adjoint dx */
  CAVS_PH_REDUCE = 8,     /* db column sums + dparams packing */
  CAVS_PH_COUNT = 9
} cavs_phase;
cavs_status cavs_profile(cavs_ctx* ctx, int enable);
cavs_status cavs_profile_read(cavs_ctx* ctx, int32_t phase, double* ms, double* flops, double* bytes,
                              int64_t* launches);

const char* cavs_last_error(const cavs_ctx* ctx);

/* Which kernel path the context runs its batching tasks on (diagnostic string, owned by the
 * context, valid until the next call on it), e.g. "levels: persistent: grid 144 ...".  Only
 * meaningful after cavs_set_workspace; never NULL. */
const char* cavs_path_info(const cavs_ctx* ctx);
void cavs_destroy(cavs_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* CAVS_H_ */
