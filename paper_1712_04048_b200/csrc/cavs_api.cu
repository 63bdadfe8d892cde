// cavs_api.cu — the C-ABI (include/cavs.h): context, state machine, workspace carve-up
// (the dynamic-tensor memory plan, Fig. 7) and launch orchestration
// of Algorithm 1: schedule -> forward tasks t = 0..T-1 -> backward tasks
// t = T-1..1 -> lazily batched parameter gradients (§3.5).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "tc.h"

using namespace cavs;

enum { S_CREATED = 0, S_READY, S_LOADED, S_SCHEDULED, S_FORWARDED };

struct cavs_ctx {
  cavs_desc desc{};
  int device = 0;
  cudaStream_t stream = nullptr;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  int state = S_CREATED;
  Dev D{};
  std::vector<int> lp;          // host copy of level_ptr[0..T]
  int T = 0, n_roots = 0;
  int* h_hdr = nullptr;         // pinned readback buffer
  std::string err;
  std::string info;             // cavs_path_info buffer
  Prof prof;                    // phase marks + launch counts
  // lazy scratch layout
  float* lazy_db = nullptr;
  // staging for cavs_train_step_host
  float *s_params = nullptr, *s_x = nullptr, *s_dh = nullptr, *s_dp = nullptr, *s_dx = nullptr, *s_hout = nullptr;
  int *s_xrow = nullptr, *s_gp = nullptr, *s_cp = nullptr, *s_ci = nullptr;
  TcState* tc = nullptr;        // tensor-core (BF16) path state: TMA descriptors
  cudaEvent_t ev_hdr = nullptr; // recorded after the schedule header's device->host copy
  cudaEvent_t ev_wgrad = nullptr;   // caller's event: recorded once dparams' weight blocks are final
  XStream xs;                   // streaming ablation: side stream + per-task events
  // db (k_colsum) beside the lazy GEMMs and dX: side stream forked after the level tasks, joined at the
  // end of the backward (CAVS_DB_SIDE=0: on the main stream)
  cudaStream_t db_s = nullptr;
  cudaEvent_t ev_lv = nullptr, ev_db = nullptr;
  bool db_side = true;
  bool dx_side = true;                  // dX = dZ W on db_s too (CAVS_DX_SIDE=0: on the main stream)
  // pipelined host-buffer steps (cavs_train_step_host_async): two staging slots, H2D / D2H streams
  struct Slot {
    int *gp = nullptr, *cp = nullptr, *ci = nullptr, *xrow = nullptr, *grow = nullptr;
    float *params = nullptr, *x = nullptr, *gval = nullptr, *dp = nullptr;
    cudaEvent_t copied = nullptr, done = nullptr;
    bool used = false;
  } slot[2];
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_bwd = nullptr;
  int64_t n_async = 0;
  unsigned pull_gen = 0;
  bool hdr_pending = false;     // header copied asynchronously, not parsed yet
};

static constexpr int kReadback = 1024;

static cavs_status fail(cavs_ctx* c, cavs_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

static cavs_status cuda_check(cavs_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return CAVS_OK;
  return fail(c, CAVS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(expr) do { cavs_status _s = cuda_check(ctx, (expr), #expr); if (_s) return _s; } while (0)

static bool is_lstm(const cavs_desc& d) { return d.cell == CAVS_CELL_TREE_LSTM; }
static int gates(const cavs_desc& d) { return is_lstm(d) ? 3 + d.N : 1; }
// bytes per operand element as stored: bf16, fp32, or (FP32 split mode) three bf16 planes
static size_t esize(const cavs_ctx* c) { return c->desc.precision == CAVS_BF16 ? 2 : c->D.split ? 6 : 4; }

// Carve the workspace; with base == nullptr only computes the size.
static size_t carve(cavs_ctx* c, char* base) {
  const cavs_desc& d = c->desc;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    off = (off + 255) & ~(size_t)255;
    char* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  };
  const size_t V = d.max_vertices, K = d.max_graphs, X = d.max_x, N = d.N, h = d.h, dd = d.d;
  const size_t Vp = V + kPadRows, G = gates(d), es = esize(c);
  Dev& D = c->D;
  auto I = [&](size_t n) { return reinterpret_cast<int*>(take(n * 4)); };
  auto F = [&](size_t n) { return reinterpret_cast<float*>(take(n * 4)); };
  D.graph_ptr = I(K + 1); D.child_ptr = I(V + 1); D.child_idx = I(N * V + 1);   // DAGs: up to N V edges
  D.level = I(V); D.pos = I(V); D.graph_of = I(V); D.parent_v = I(V); D.slot_v = I(V);
  D.pending = I(V); D.queue = I(V);
  D.hdr = I(kHdrWords + V + 1); D.level_ptr = base ? D.hdr + kHdrWords : nullptr;
  D.roots = I(V); D.cnt = I(V + 1); D.lrank = I(V); D.goff = I(V + 1); D.gT = I(K); D.lcount = I(V + 1);
  D.gsync = reinterpret_cast<unsigned*>(I(64));
  D.tile_cnt = I(kLazyMaxTiles + kDbMaxBlocks + 1);   // + the schedule's last-CTA counter
  D.crow = I((V + 1) * (kMaxClusters + 1));
  D.order = I(V); D.child_pos = I(V * N); D.parent_pos = I(V); D.slot = I(V); D.deg = I(V);
  D.xrow_pos = I(Vp); D.tile_x = I(Vp / 64 + 2); D.xseen = I(X + 1);
  D.Hk = take(Vp * N * h * es);
  D.Hs = nullptr;                              // U h~ is accumulated as sum_k U h_k: no h~ arena
  D.Xp = take(Vp * dd * es);
  D.dZ = take(Vp * G * h * es);
  // FP32 split mode: plane q of an arena / weight copy starts q * (plane elements) after plane 0
  const size_t sp = D.split ? 1 : 0;
  D.ps_hk = sp * Vp * N * h; D.ps_xp = sp * Vp * dd; D.ps_dz = sp * Vp * G * h;
  D.Ck = is_lstm(d) ? F(Vp * N * h) : nullptr;
  D.XW = F(Vp * (is_lstm(d) ? 4 : 1) * h);
  D.gates = F(Vp * G * h);
  D.cst = is_lstm(d) ? F(Vp * h) : nullptr;
  D.dcb = is_lstm(d) ? F(Vp * h) : nullptr;
  D.bias = F(4 * h);
  if (is_lstm(d)) {
    D.Wa = take(4 * h * h * es); D.Wb = take(4 * h * dd * es); D.Wc = take(3 * h * h * es);
    D.Wd = take(h * h * es); D.We = take(dd * G * h * es);
    const size_t pw[5] = {4 * h * h, 4 * h * dd, 3 * h * h, h * h, dd * G * h};
    for (int i = 0; i < 5; ++i) D.ps_w[i] = sp * pw[i];
  } else {
    D.Wa = take(2 * h * h * es); D.Wb = take(h * dd * es); D.Wc = take(2 * h * h * es);
    D.Wd = nullptr; D.We = take(dd * h * es);
    const size_t pw[5] = {2 * h * h, h * dd, 2 * h * h, 0, dd * h};
    for (int i = 0; i < 5; ++i) D.ps_w[i] = sp * pw[i];
  }
  D.pptr = I(V + 1); D.pent = I(N * V + 1); D.pcur = I(V);          // DAG parent CSR (NEXT-3)
  D.dHg = F(Vp * N * h); D.dCg = is_lstm(d) ? F(Vp * N * h) : nullptr;
  D.rawld = (is_lstm(d) ? 3 + kMaxN : 2) * (int)h;
  D.raw = D.unfused ? F(Vp * D.rawld) : nullptr;     // unfused ablation only
  D.lazy = F(lazy_floats(D));
  // row-tiled level GEMMs (h > 512, BF16): split-K partial slots [296 items][acc columns][128 rows]
  const char* pe = std::getenv("CAVS_PERSIST");
  const bool rows_path = d.precision == CAVS_BF16 && (h > 512 || (pe && pe[0] == '0'));
  const size_t acc_cols = is_lstm(d) ? std::max<size_t>(256 * std::min<size_t>(N, 2), 128 * (1 + std::min<size_t>(N, 2))) : 256;
  D.rows_part = rows_path ? F((size_t)296 * acc_cols * 128) : nullptr;
  D.rows_cnt = rows_path ? I(1024) : nullptr;
  c->lazy_db = F((size_t)kDbChunks * d.N * 4 * h);   // db partials [(slot, chunk)][logical column]
  const size_t P = cavs_param_count(d.cell, d.N, d.h, d.d);
  c->s_params = F(P); c->s_dp = F(P);
  c->s_x = F(X * dd); c->s_dx = F(X * dd);
  c->s_dh = F(V * h); c->s_hout = F(V * h);
  c->s_xrow = I(V); c->s_gp = I(K + 1); c->s_cp = I(V + 1); c->s_ci = I(V + 1);
  for (auto& sl : c->slot) {                  // cavs_train_step_host_async staging
    sl.gp = I(K + 1); sl.cp = I(V + 1); sl.ci = I(N * V + 1); sl.xrow = I(V); sl.grow = I(V);
    sl.params = F(P); sl.x = F(X * dd); sl.gval = F(V * h); sl.dp = F(P);
  }
  return (off + 255) & ~(size_t)255;
}

#define CAVS_API extern "C" __attribute__((visibility("default")))

CAVS_API size_t cavs_param_count(int32_t cell, int32_t N, int32_t h, int32_t d) {
  (void)N;
  const size_t H = h, Dd = d;
  if (cell == CAVS_CELL_TREE_LSTM) return 4 * H * Dd + 3 * H * H + H * H + 4 * H;
  if (cell == CAVS_CELL_TREE_FC) return 2 * H * H + H * Dd + H;
  return 0;
}

CAVS_API cavs_status cavs_create(const cavs_desc* desc, int device, void* stream, cavs_ctx** out) {
  if (!desc || !out) return CAVS_E_INVALID;
  *out = nullptr;
  const cavs_desc& d = *desc;
  if ((d.cell != CAVS_CELL_TREE_LSTM && d.cell != CAVS_CELL_TREE_FC) || d.N < 1 || d.h < 1 || d.d < 1 ||
      (d.precision != CAVS_FP32 && d.precision != CAVS_BF16) || d.max_graphs < 1 || d.max_vertices < 1 ||
      d.max_x < 0)
    return CAVS_E_INVALID;
  if (d.N > kMaxN) return CAVS_E_UNSUPPORTED;
  if (d.cell == CAVS_CELL_TREE_FC && d.N != 2) return CAVS_E_UNSUPPORTED;
  if ((int64_t)4 * d.h > 256 * kDbMaxBlocks) return CAVS_E_UNSUPPORTED;     // db column blocks (k_colsum)
  if (d.precision == CAVS_BF16 && ((d.h % 64) || (d.d % 64))) return CAVS_E_UNSUPPORTED;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return CAVS_E_CUDA;
  cavs_ctx* c = new cavs_ctx();
  c->desc = d;
  c->device = device;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  c->D.cell = d.cell; c->D.N = d.N; c->D.h = d.h; c->D.d = d.d; c->D.prec = d.precision;
  {  // engine ablations (NEXT-1), fixed for the context's lifetime
    const char* lz = std::getenv("CAVS_LAZY_BATCH");
    const char* uf = std::getenv("CAVS_UNFUSED");
    const char* sx = std::getenv("CAVS_STREAMING");
    const char* dbs = std::getenv("CAVS_DB_SIDE");
    c->db_side = !(dbs && dbs[0] == '0');
    const char* dxs = std::getenv("CAVS_DX_SIDE");
    c->dx_side = !(dxs && dxs[0] == '0');
    c->D.lazy_off = lz && lz[0] == '0';
    c->D.unfused = uf && uf[0] == '1';
    c->D.stream_x = sx && sx[0] == '1';
    // FP32 mode on the tensor cores (bf16x3 split operands, six MMAs per product) unless the shape
    // or an ablation needs the FFMA path, or CAVS_FP32_FFMA=1 asks for it
    const char* ff = std::getenv("CAVS_FP32_FFMA");
    c->D.split = d.precision == CAVS_FP32 && !(ff && ff[0] == '1') && d.h % 64 == 0 && d.d % 64 == 0 &&
                 !c->D.lazy_off && !c->D.unfused && !c->D.stream_x;
  }
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaMallocHost(&c->h_hdr, sizeof(int) * (kHdrWords + kReadback)) != cudaSuccess) {
    delete c;
    return CAVS_E_CUDA;
  }
  c->ws_bytes = carve(c, nullptr);
  const char* tr = std::getenv("CAVS_TRACE");
  if (tr && tr[0] == '1') c->ws_bytes += 4u << 20;     // debug trace ring at the end of the workspace
  *out = c;
  return CAVS_OK;
}

CAVS_API cavs_status cavs_set_stream(cavs_ctx* ctx, void* stream) {
  if (!ctx) return CAVS_E_INVALID;
  ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  return CAVS_OK;
}

CAVS_API size_t cavs_workspace_bytes(const cavs_ctx* ctx) { return ctx ? ctx->ws_bytes : 0; }

CAVS_API cavs_status cavs_set_workspace(cavs_ctx* ctx, void* dev, size_t bytes) {
  if (!ctx || !dev) return fail(ctx, CAVS_E_INVALID, "null workspace");
  if ((reinterpret_cast<uintptr_t>(dev) & 255) != 0) return fail(ctx, CAVS_E_INVALID, "workspace not 256B aligned");
  if (bytes < ctx->ws_bytes) return fail(ctx, CAVS_E_CAPACITY, "workspace too small");
  CK(cudaSetDevice(ctx->device));
  ctx->ws = reinterpret_cast<char*>(dev);
  carve(ctx, ctx->ws);
  const char* tr = std::getenv("CAVS_TRACE");
  ctx->D.trace = (tr && tr[0] == '1') ? reinterpret_cast<unsigned long long*>(ctx->ws + ctx->ws_bytes - (4u << 20))
                                      : nullptr;
  CK(cudaMemsetAsync(ctx->ws, 0, ctx->ws_bytes, ctx->stream));   // arenas start finite (zero)
  if (ctx->desc.precision == CAVS_BF16 || ctx->D.split) {
    cavs_status s = tc_init(ctx->D, ctx->desc.max_vertices, &ctx->tc, &ctx->err);
    if (s) return s;
    ctx->D.ncl = tc_clusters(ctx->tc);
  }
  ctx->state = S_READY;
  return CAVS_OK;
}

CAVS_API cavs_status cavs_load_graphs(cavs_ctx* ctx, int32_t K, int32_t V, int32_t E, const int32_t* graph_ptr,
                             const int32_t* child_ptr, const int32_t* child_idx, int on_device) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_READY) return fail(ctx, CAVS_E_STATE, "set_workspace first");
  if (K < 1 || V < 1 || E < 0 || !graph_ptr || !child_ptr || (E > 0 && !child_idx))
    return fail(ctx, CAVS_E_INVALID, "bad sizes or null pointers");
  if (K > ctx->desc.max_graphs || V > ctx->desc.max_vertices || (int64_t)E > (int64_t)ctx->desc.N * ctx->desc.max_vertices)
    return fail(ctx, CAVS_E_CAPACITY, "batch exceeds context capacity");
  CK(cudaSetDevice(ctx->device));
  Dev& D = ctx->D;
  if (on_device) {            // read (and copied into the workspace) by cavs_schedule's first kernel
    D.src_gp = graph_ptr; D.src_cp = child_ptr; D.src_ci = child_idx;
  } else {
    CK(cudaMemcpyAsync((void*)D.graph_ptr, graph_ptr, sizeof(int) * (K + 1), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync((void*)D.child_ptr, child_ptr, sizeof(int) * (V + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (E > 0) CK(cudaMemcpyAsync((void*)D.child_idx, child_idx, sizeof(int) * E, cudaMemcpyHostToDevice, ctx->stream));
    D.src_gp = D.graph_ptr; D.src_cp = D.child_ptr; D.src_ci = D.child_idx;
  }
  D.K = K; D.V = V; D.E = E;
  ctx->state = S_LOADED;
  ctx->hdr_pending = false;
  return CAVS_OK;
}

// Wait for the schedule header (status, T, #roots, level_ptr) copied by cavs_schedule and
// parse it; reports the graphs' validation errors.  No-op when already parsed.
static cavs_status finish_schedule(cavs_ctx* ctx) {
  if (!ctx->hdr_pending) return CAVS_OK;
  ctx->hdr_pending = false;
  CK(cudaEventSynchronize(ctx->ev_hdr));
  Dev& D = ctx->D;
  const int nread = kHdrWords + std::min(D.V + 1, kReadback);
  const int st = ctx->h_hdr[0];
  if (st) {
    ctx->state = S_LOADED;
    if (st & ST_INVALID) return fail(ctx, CAVS_E_INVALID, "malformed graph (range/shape)");
    if (st & ST_ARITY) return fail(ctx, CAVS_E_ARITY, "a vertex has more than N children");
    return fail(ctx, CAVS_E_CYCLE, "input graph has a cycle");
  }
  const int T = ctx->h_hdr[1];
  ctx->T = T;
  D.dag = (ctx->h_hdr[3] & ST_DAG) ? 1 : 0;          // fan-out somewhere in the batch (NEXT-3)
  if (D.dag) {
    launch_dag_parents(D, ctx->stream);
    ctx->prof.count(4);
  }
  ctx->n_roots = ctx->h_hdr[2];
  ctx->lp.assign(T + 1, 0);
  if (T + 1 <= nread - kHdrWords) {
    std::memcpy(ctx->lp.data(), ctx->h_hdr + kHdrWords, sizeof(int) * (T + 1));
  } else {
    CK(cudaMemcpy(ctx->lp.data(), D.level_ptr, sizeof(int) * (T + 1), cudaMemcpyDeviceToHost));
  }
  D.T = T;
  D.lp1 = T > 1 ? ctx->lp[1] : D.V;
  return CAVS_OK;
}

CAVS_API cavs_status cavs_schedule(cavs_ctx* ctx, int32_t* T_out) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_LOADED) return fail(ctx, CAVS_E_STATE, "no graphs loaded");
  CK(cudaSetDevice(ctx->device));
  Dev& D = ctx->D;
  CK(cudaMemsetAsync(D.hdr, 0, sizeof(int) * kHdrWords, ctx->stream));
  ctx->prof.mark(CAVS_PH_SCHEDULE, ctx->stream);
  launch_schedule(D, ctx->stream);
  ctx->prof.count(3);
  ctx->prof.mark(-1, ctx->stream);
  CK(cudaGetLastError());
  ctx->state = S_SCHEDULED;
  if (D.sync_free && !T_out) {                  // sync-free mode: the header stays on the device
    ctx->hdr_pending = false;
    ctx->T = -1;
    ctx->lp.clear();
    D.dag = 0;
    return CAVS_OK;
  }
  const int nread = kHdrWords + std::min(D.V + 1, kReadback);
  CK(cudaMemcpyAsync(ctx->h_hdr, D.hdr, sizeof(int) * nread, cudaMemcpyDeviceToHost, ctx->stream));
  if (!ctx->ev_hdr) CK(cudaEventCreateWithFlags(&ctx->ev_hdr, cudaEventDisableTiming));
  CK(cudaEventRecord(ctx->ev_hdr, ctx->stream));
  ctx->hdr_pending = true;
  if (T_out) {
    const cavs_status st = finish_schedule(ctx);
    if (st) return st;
    *T_out = ctx->T;
  }
  return CAVS_OK;
}

CAVS_API cavs_status cavs_get_schedule(cavs_ctx* ctx, int32_t* level, int32_t* level_ptr, int32_t* order) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_SCHEDULED) return fail(ctx, CAVS_E_STATE, "not scheduled");
  CK(cudaSetDevice(ctx->device));
  if (ctx->T < 0) {                             // sync-free mode: fetch the header now (synchronous call)
    const int nread = kHdrWords + std::min(ctx->D.V + 1, kReadback);
    CK(cudaMemcpyAsync(ctx->h_hdr, ctx->D.hdr, sizeof(int) * nread, cudaMemcpyDeviceToHost, ctx->stream));
    if (!ctx->ev_hdr) CK(cudaEventCreateWithFlags(&ctx->ev_hdr, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->ev_hdr, ctx->stream));
    ctx->hdr_pending = true;
  }
  const cavs_status st = finish_schedule(ctx);
  if (st) return st;
  CK(cudaStreamSynchronize(ctx->stream));
  const Dev& D = ctx->D;
  if (level) CK(cudaMemcpy(level, D.level, sizeof(int) * D.V, cudaMemcpyDeviceToHost));
  if (level_ptr) std::memcpy(level_ptr, ctx->lp.data(), sizeof(int) * (ctx->T + 1));
  if (order) CK(cudaMemcpy(order, D.order, sizeof(int) * D.V, cudaMemcpyDeviceToHost));
  return CAVS_OK;
}

// --------------------------------------------------------------------------- roofline accounting
// ALGORITHMIC work per phase: FLOPs of the contractions the
// method must do (2 per MAC; a vertex with c children needs U h~ (3h^2 MACs, Tree-LSTM) and
// one U_f h_k per existing child; leaves no recurrent term), bytes = minimal HBM traffic of
// the phase's operands/results in the precision they are stored in.
static void account_forward(cavs_ctx* ctx) {
  Prof& P = ctx->prof;
  const Dev& D = ctx->D;
  const double h = D.h, d = D.d, I = D.V - D.lp1, E = D.E, nx = D.n_x, O = esize(ctx), S = 4;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const double G = lstm ? 3 + D.N : 1;
  if (lstm) {
    P.flops[CAVS_PH_XPROJ] += 2.0 * 4 * h * d * nx;
    P.flops[CAVS_PH_FWD_LEVELS] += 2.0 * h * h * (3 * I + E);
    // read child h (O) and c (S) per edge; write c, gates, h_out, parent slot h (O) + c (S), h~ (O)
    P.bytes[CAVS_PH_FWD_LEVELS] += E * h * (O + S) + I * h * (S + G * S + S + O + S + O) +
                                   (ctx->T - 1) * 4 * h * h * O;
    P.bytes[CAVS_PH_XPROJ] += nx * d * O + 4 * h * d * O + nx * h * (S + G * S + S + O + S);
  } else {
    P.flops[CAVS_PH_XPROJ] += 2.0 * h * d * nx;
    P.flops[CAVS_PH_FWD_LEVELS] += 2.0 * h * h * E;
    P.bytes[CAVS_PH_FWD_LEVELS] += E * h * O + I * h * (S + S + O) + (ctx->T - 1) * 2 * h * h * O;
    P.bytes[CAVS_PH_XPROJ] += nx * d * O + h * d * O + nx * h * (S + S + O);
  }
}

static void account_backward(cavs_ctx* ctx) {
  Prof& P = ctx->prof;
  const Dev& D = ctx->D;
  const double h = D.h, d = D.d, I = D.V - D.lp1, E = D.E, nx = D.n_x, O = esize(ctx), S = 4;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const double G = lstm ? 3 + D.N : 1;
  if (lstm) {
    P.flops[CAVS_PH_BWD_LEVELS] += 2.0 * h * h * (3 * I + E);
    P.flops[CAVS_PH_LAZY] += 2.0 * h * h * (3 * I + E) + 2.0 * 4 * h * d * nx;
    P.flops[CAVS_PH_DX] += 2.0 * 4 * h * d * nx;
    // read parent dZ (O), dc-bar, gates; per child: dh_out, gates, c, child c slots; write child dZ, dc-bar
    P.bytes[CAVS_PH_BWD_LEVELS] += I * h * (G * O + S + G * S) + E * h * (S + G * S + S + D.N * S + G * O + S) +
                                   (ctx->T - 1) * 4 * h * h * O;
    P.bytes[CAVS_PH_LAZY] += I * h * (3 * O + O) + E * h * 2 * O + nx * (G * h + d) * O +
                             (3 * h * h + h * h + G * h * d) * S;
  } else {
    P.flops[CAVS_PH_BWD_LEVELS] += 2.0 * h * h * E;
    P.flops[CAVS_PH_LAZY] += 2.0 * h * h * E + 2.0 * h * d * nx;
    P.flops[CAVS_PH_DX] += 2.0 * h * d * nx;
    P.bytes[CAVS_PH_BWD_LEVELS] += I * h * O + E * h * (S + S + O) + (ctx->T - 1) * 2 * h * h * O;
    P.bytes[CAVS_PH_LAZY] += I * h * (O + 2 * O) + nx * (h + d) * O + (2 * h * h + h * d) * S;
  }
}

// --------------------------------------------------------------------------- forward
static cavs_status forward_impl(cavs_ctx* ctx, const float* params, int32_t n_x, const float* x,
                                const int32_t* x_row, float* h_out, bool infer) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_SCHEDULED) return fail(ctx, CAVS_E_STATE, "cavs_schedule first");
  if (!params || !x_row || !h_out || (n_x > 0 && !x)) return fail(ctx, CAVS_E_INVALID, "null pointer");
  if (n_x < 0 || n_x > ctx->desc.max_x) return fail(ctx, CAVS_E_CAPACITY, "n_x exceeds max_x");
  CK(cudaSetDevice(ctx->device));
  Dev& D = ctx->D;
  D.params = params; D.x = x; D.x_row = x_row; D.h_out = h_out; D.n_x = n_x;
  D.infer = infer ? 1 : 0;                 // (a DAG batch gathers c from the leaves' saved state: see below)
  D.xgen = ++ctx->pull_gen;                // k_pull stamps every record it pulls (duplicates -> hdr[5])
  Prof& P = ctx->prof;
  P.mark(CAVS_PH_PREP, ctx->stream);
  // the parameter repack (weights only) runs on a side stream beside the pull; the forward's tensor-core
  // kernels wait for both (fork / join: a parallel branch in a CUDA-graph capture)
  const bool side = ctx->db_side;
  if (side && !ctx->db_s) {
    CK(cudaStreamCreateWithFlags(&ctx->db_s, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_lv, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_db, cudaEventDisableTiming));
  }
  if (side) {
    CK(cudaEventRecord(ctx->ev_lv, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->db_s, ctx->ev_lv, 0));
    launch_prep(D, ctx->db_s);
    if (ctx->tc) tc_zero_dz_tail(D, ctx->tc, ctx->db_s);
    CK(cudaEventRecord(ctx->ev_db, ctx->db_s));
  } else {
    launch_prep(D, ctx->stream);
    if (ctx->tc) tc_zero_dz_tail(D, ctx->tc, ctx->stream);
  }
  CK(cudaMemsetAsync(D.hdr + 4, 0, 2 * sizeof(int), ctx->stream));   // k_pull's statistics of this forward
  launch_pull(D, ctx->stream);
  if (side) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_db, 0));
  P.count(2);
  {  // a deferred schedule header is consumed here, while prep / pull run on the device
    const cavs_status st = finish_schedule(ctx);
    if (st) return st;
  }
  if (D.dag) D.infer = 0;                  // the per-task gather reads every child's saved c
  P.mark(CAVS_PH_XPROJ, ctx->stream);
  if (D.stream_x && !ctx->xs.s) {
    CK(cudaStreamCreateWithFlags(&ctx->xs.s, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->xs.start, cudaEventDisableTiming));
  }
  if (ctx->tc) tc_forward(D, ctx->tc, ctx->lp, ctx->stream, P, &ctx->xs);
  else simt_forward<float>(D, ctx->lp, ctx->stream, P, &ctx->xs);
  P.mark(-1, ctx->stream);
  if (ctx->T >= 0) account_forward(ctx);        // (sync-free mode: the host does not know I / T)
  CK(cudaGetLastError());
  ctx->state = infer ? S_SCHEDULED : S_FORWARDED;   // no activations for dF after an inference pass
  return CAVS_OK;
}

CAVS_API cavs_status cavs_forward(cavs_ctx* ctx, const float* params, int32_t n_x, const float* x,
                                  const int32_t* x_row, float* h_out) {
  return forward_impl(ctx, params, n_x, x, x_row, h_out, false);
}

CAVS_API cavs_status cavs_forward_inference(cavs_ctx* ctx, const float* params, int32_t n_x, const float* x,
                                            const int32_t* x_row, float* h_out) {
  return forward_impl(ctx, params, n_x, x, x_row, h_out, true);
}

// --------------------------------------------------------------------------- backward
CAVS_API cavs_status cavs_backward(cavs_ctx* ctx, const float* dh_out, float* dparams, float* dx) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_FORWARDED) return fail(ctx, CAVS_E_STATE, "cavs_forward first");
  if (!dh_out || !dparams) return fail(ctx, CAVS_E_INVALID, "null pointer");
  CK(cudaSetDevice(ctx->device));
  Dev& D = ctx->D;
  D.dh_out = dh_out; D.dparams = dparams; D.dx = dx;
  Prof& P = ctx->prof;
  // dx rows receive plain stores when every record is pulled exactly once (the usual case); the
  // zeroing + atomic adds only run when some record is pulled by several vertices or by none
  // (k_pull.s duplicate flag / pull count; decided on the device by k_dx_zero and the DX epilogue)
  if (dx && D.n_x > 0 && !ctx->tc) { launch_dx_zero(D, ctx->stream); P.count(1); }   // (tc: in tc_backward)
  P.mark(CAVS_PH_BWD_ROOTS, ctx->stream);
  if (!D.dag) {                                // DAG batches: every vertex's dF runs in launch_dag_df
    launch_roots(D, ctx->T >= 0 ? ctx->n_roots : -1, D.roots, ctx->stream);   // -1: count on the device
    P.count(1);
  }
  P.mark(CAVS_PH_BWD_LEVELS, ctx->stream);
  int split[3] = {1, 1, 1};
  if (ctx->tc) {
    if (ctx->db_side && !ctx->db_s) {
      CK(cudaStreamCreateWithFlags(&ctx->db_s, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->ev_lv, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_db, cudaEventDisableTiming));
    }
    // dX on the side stream (before db there) beside the lazy GEMMs unless CAVS_DX_SIDE=0
    tc_backward(D, ctx->tc, ctx->lp, ctx->stream, split, P, ctx->ev_wgrad, ctx->db_side ? ctx->ev_lv : nullptr,
                ctx->db_side && ctx->dx_side ? ctx->db_s : nullptr);
  } else {
    simt_backward<float>(D, ctx->lp, ctx->stream, P);
  }
  P.mark(CAVS_PH_REDUCE, ctx->stream);
  if (split[0] >= 0) {                         // split-K slots of the fallback lazy GEMMs -> dparams
    launch_pack(D, split, ctx->stream);
    P.count(1);
    if (ctx->ev_wgrad) CK(cudaEventRecord(ctx->ev_wgrad, ctx->stream));
  }
  if (ctx->tc && ctx->db_side) {                 // db -> dparams, beside the lazy GEMMs / dX (same dZ, disjoint outputs)
    CK(cudaStreamWaitEvent(ctx->db_s, ctx->ev_lv, 0));
    launch_colsum(D, ctx->lazy_db, ctx->db_s);
    CK(cudaEventRecord(ctx->ev_db, ctx->db_s));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_db, 0));
  } else {
    launch_colsum(D, ctx->lazy_db, ctx->stream);
  }
  P.count(1);
  P.mark(-1, ctx->stream);
  if (ctx->T >= 0) account_backward(ctx);
  CK(cudaGetLastError());
  return CAVS_OK;
}

CAVS_API cavs_status cavs_train_step_host(cavs_ctx* ctx, int32_t K, int32_t V, int32_t E, const int32_t* graph_ptr,
                                 const int32_t* child_ptr, const int32_t* child_idx, const float* params,
                                 int32_t n_x, const float* x, const int32_t* x_row, const float* dh_out,
                                 float* dparams, float* dx, float* h_out) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_READY) return fail(ctx, CAVS_E_STATE, "set_workspace first");
  if (n_x < 0 || n_x > ctx->desc.max_x || V > ctx->desc.max_vertices || V < 1)
    return fail(ctx, CAVS_E_CAPACITY, "batch exceeds capacity");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const cavs_desc& d = ctx->desc;
  const size_t P = cavs_param_count(d.cell, d.N, d.h, d.d);
  cavs_status st = cavs_load_graphs(ctx, K, V, E, graph_ptr, child_ptr, child_idx, 0);
  if (st) return st;
  CK(cudaMemcpyAsync(ctx->s_params, params, sizeof(float) * P, cudaMemcpyHostToDevice, s));
  if (n_x) CK(cudaMemcpyAsync(ctx->s_x, x, sizeof(float) * n_x * d.d, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->s_xrow, x_row, sizeof(int) * V, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->s_dh, dh_out, sizeof(float) * V * d.h, cudaMemcpyHostToDevice, s));
  st = cavs_schedule(ctx, nullptr);
  if (st) return st;
  st = cavs_forward(ctx, ctx->s_params, n_x, ctx->s_x, ctx->s_xrow, ctx->s_hout);
  if (st) return st;
  st = cavs_backward(ctx, ctx->s_dh, ctx->s_dp, dx ? ctx->s_dx : nullptr);
  if (st) return st;
  CK(cudaMemcpyAsync(dparams, ctx->s_dp, sizeof(float) * P, cudaMemcpyDeviceToHost, s));
  if (dx && n_x) CK(cudaMemcpyAsync(dx, ctx->s_dx, sizeof(float) * n_x * d.d, cudaMemcpyDeviceToHost, s));
  if (h_out) CK(cudaMemcpyAsync(h_out, ctx->s_hout, sizeof(float) * V * d.h, cudaMemcpyDeviceToHost, s));
  return cavs_sync(ctx);
}

// Pipelined end-to-end step (include/cavs.h): H2D of step i+1 on its own stream overlaps step i's
// compute, D2H of dparams on a third stream; two staging slots, reused once the step that last
// used the slot finished its D2H.  Cotangents may come as rows + values (the loss vertices).
CAVS_API cavs_status cavs_train_step_host_async(cavs_ctx* ctx, int32_t K, int32_t V, int32_t E,
                                                const int32_t* graph_ptr, const int32_t* child_ptr,
                                                const int32_t* child_idx, const float* params, int32_t n_x,
                                                const float* x, const int32_t* x_row, int32_t n_gamma,
                                                const int32_t* gamma_rows, const float* gamma, float* dparams) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_READY) return fail(ctx, CAVS_E_STATE, "set_workspace first");
  const cavs_desc& d = ctx->desc;
  if (n_x < 0 || n_x > d.max_x || V > d.max_vertices || V < 1 || K < 1 || K > d.max_graphs || E < 0 ||
      (int64_t)E > (int64_t)d.N * d.max_vertices)
    return fail(ctx, CAVS_E_CAPACITY, "batch exceeds capacity");
  if (!graph_ptr || !child_ptr || (E && !child_idx) || !params || !x_row || !dparams || (n_x && !x) ||
      n_gamma < 0 || n_gamma > V || (n_gamma && !gamma) || (!gamma_rows && n_gamma != V && n_gamma != 0))
    return fail(ctx, CAVS_E_INVALID, "null pointer or bad sizes");
  CK(cudaSetDevice(ctx->device));
  if (!ctx->h2d) {
    CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_bwd, cudaEventDisableTiming));
    for (auto& sl : ctx->slot) {
      CK(cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
  }
  const size_t P = cavs_param_count(d.cell, d.N, d.h, d.d);
  auto& sl = ctx->slot[ctx->n_async & 1];
  ++ctx->n_async;
  // ---- H2D of this step's inputs (waits only for the step that last used this slot) ----
  if (sl.used) CK(cudaStreamWaitEvent(ctx->h2d, sl.done, 0));
  sl.used = true;
  cudaStream_t c = ctx->h2d;
  CK(cudaMemcpyAsync(sl.gp, graph_ptr, sizeof(int) * (K + 1), cudaMemcpyHostToDevice, c));
  CK(cudaMemcpyAsync(sl.cp, child_ptr, sizeof(int) * (V + 1), cudaMemcpyHostToDevice, c));
  if (E) CK(cudaMemcpyAsync(sl.ci, child_idx, sizeof(int) * E, cudaMemcpyHostToDevice, c));
  CK(cudaMemcpyAsync(sl.params, params, sizeof(float) * P, cudaMemcpyHostToDevice, c));
  if (n_x) CK(cudaMemcpyAsync(sl.x, x, sizeof(float) * n_x * d.d, cudaMemcpyHostToDevice, c));
  CK(cudaMemcpyAsync(sl.xrow, x_row, sizeof(int) * V, cudaMemcpyHostToDevice, c));
  if (n_gamma) CK(cudaMemcpyAsync(sl.gval, gamma, sizeof(float) * n_gamma * d.h, cudaMemcpyHostToDevice, c));
  if (n_gamma && gamma_rows) CK(cudaMemcpyAsync(sl.grow, gamma_rows, sizeof(int) * n_gamma, cudaMemcpyHostToDevice, c));
  CK(cudaEventRecord(sl.copied, c));
  // ---- compute on the context's stream ----
  cudaStream_t s = ctx->stream;
  CK(cudaStreamWaitEvent(s, sl.copied, 0));
  cavs_status st = cavs_load_graphs(ctx, K, V, E, sl.gp, sl.cp, sl.ci, 1);
  if (st) return st;
  st = cavs_schedule(ctx, nullptr);
  if (st) return st;
  float* dh = ctx->s_dh;                       // dense push cotangent (a single buffer: stream-ordered)
  if (gamma_rows) {
    CK(cudaMemsetAsync(dh, 0, sizeof(float) * (size_t)V * d.h, s));
    launch_scatter_rows(dh, sl.gval, sl.grow, n_gamma, d.h, s);
  } else if (n_gamma) {
    dh = sl.gval;
  } else {
    CK(cudaMemsetAsync(dh, 0, sizeof(float) * (size_t)V * d.h, s));
  }
  st = cavs_forward(ctx, sl.params, n_x, sl.x, sl.xrow, ctx->s_hout);
  if (st) return st;
  st = cavs_backward(ctx, dh, sl.dp, nullptr);
  if (st) return st;
  CK(cudaEventRecord(ctx->ev_bwd, s));
  // ---- D2H of the step's result ----
  CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_bwd, 0));
  CK(cudaMemcpyAsync(dparams, sl.dp, sizeof(float) * P, cudaMemcpyDeviceToHost, ctx->d2h));
  CK(cudaEventRecord(sl.done, ctx->d2h));
  return CAVS_OK;
}

CAVS_API cavs_status cavs_set_sync_free(cavs_ctx* ctx, int on) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_READY) return fail(ctx, CAVS_E_STATE, "set_workspace first");
  if (on && !(ctx->desc.precision == CAVS_BF16 && tc_sync_free_capable(ctx->tc)))
    return fail(ctx, CAVS_E_UNSUPPORTED, "sync-free mode needs the BF16 persistent path (h % 64 == 0, h <= 512)");
  ctx->D.sync_free = on ? 1 : 0;
  return CAVS_OK;
}

CAVS_API cavs_status cavs_set_grad_event(cavs_ctx* ctx, void* cuda_event) {
  if (!ctx) return CAVS_E_INVALID;
  ctx->ev_wgrad = static_cast<cudaEvent_t>(cuda_event);
  return CAVS_OK;
}

CAVS_API cavs_status cavs_sync(cavs_ctx* ctx) {
  if (!ctx) return CAVS_E_INVALID;
  if (ctx->state < S_READY) return CAVS_OK;
  CK(cudaSetDevice(ctx->device));
  if (ctx->d2h) CK(cudaStreamSynchronize(ctx->d2h));   // pipelined host-buffer steps
  CK(cudaMemcpyAsync(ctx->h_hdr + kHdrWords + kReadback - 1, ctx->D.hdr + 3, sizeof(int), cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (ctx->D.sync_free) {                       // the schedule's own status, never read on the host before
    CK(cudaMemcpyAsync(ctx->h_hdr + kHdrWords + kReadback - 2, ctx->D.hdr, sizeof(int), cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->D.sync_free) {
    const int st = ctx->h_hdr[kHdrWords + kReadback - 2], fl = ctx->h_hdr[kHdrWords + kReadback - 1];
    if (st & ST_INVALID) return fail(ctx, CAVS_E_INVALID, "malformed graph (range/shape); the step did nothing");
    if (st & ST_ARITY) return fail(ctx, CAVS_E_ARITY, "a vertex has more than N children; the step did nothing");
    if (st & ST_CYCLE) return fail(ctx, CAVS_E_CYCLE, "input graph has a cycle; the step did nothing");
    if (fl & ST_DAG)
      return fail(ctx, CAVS_E_UNSUPPORTED, "DAG batch (fan-out) in sync-free mode; the step did nothing");
  }
  if (ctx->h_hdr[kHdrWords + kReadback - 1] & ST_XROW)
    return fail(ctx, CAVS_E_INVALID, "x_row entry outside [-1, n_x) (the vertex pulled nothing)");
  return CAVS_OK;
}

CAVS_API int64_t cavs_kernel_launches(const cavs_ctx* ctx) { return ctx ? ctx->prof.total : 0; }

static void drain_marks(cavs_ctx* ctx) {
  Prof& P = ctx->prof;
  if (P.marks.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (size_t i = 0; i + 1 < P.marks.size(); ++i) {
    const int ph = P.marks[i].first;
    if (ph < 0) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, P.marks[i].second, P.marks[i + 1].second);
    P.ms[ph] += ms;
  }
  for (auto& m : P.marks) cudaEventDestroy(m.second);
  P.marks.clear();
}

CAVS_API cavs_status cavs_profile(cavs_ctx* ctx, int enable) {
  if (!ctx) return CAVS_E_INVALID;
  CK(cudaSetDevice(ctx->device));
  drain_marks(ctx);
  Prof& P = ctx->prof;
  for (int i = 0; i < CAVS_PH_COUNT; ++i) { P.ms[i] = 0; P.flops[i] = 0; P.bytes[i] = 0; P.launches[i] = 0; }
  P.on = enable != 0;
  return CAVS_OK;
}

CAVS_API cavs_status cavs_profile_read(cavs_ctx* ctx, int32_t phase, double* ms, double* flops, double* bytes,
                                       int64_t* launches) {
  if (!ctx || phase < 0 || phase >= CAVS_PH_COUNT) return CAVS_E_INVALID;
  CK(cudaSetDevice(ctx->device));
  drain_marks(ctx);
  const Prof& P = ctx->prof;
  if (ms) *ms = P.ms[phase];
  if (flops) *flops = P.flops[phase];
  if (bytes) *bytes = P.bytes[phase];
  if (launches) *launches = P.launches[phase];
  return CAVS_OK;
}

CAVS_API const char* cavs_last_error(const cavs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

CAVS_API const char* cavs_path_info(const cavs_ctx* ctx) {
  if (!ctx) return "null context";
  cavs_ctx* c = const_cast<cavs_ctx*>(ctx);
  c->info = ctx->state < S_READY ? std::string("no workspace yet")
                                 : ctx->tc ? tc_describe(ctx->tc) : std::string("levels: FP32 FFMA") +
                                       (ctx->D.unfused ? "; ablation: unfused cell epilogues" : "") +
                                       (ctx->D.stream_x ? "; ablation: streamed x-projection" : "") +
                                       (ctx->D.lazy_off ? "; lazy batching OFF (ablation: per-task weight-gradient GEMMs)" : "");
  return c->info.c_str();
}

CAVS_API void cavs_destroy(cavs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream); else cudaDeviceSynchronize();
  tc_destroy(ctx->tc);
  if (ctx->xs.s) {
    cudaStreamSynchronize(ctx->xs.s);
    cudaStreamDestroy(ctx->xs.s);
    cudaEventDestroy(ctx->xs.start);
    for (cudaEvent_t e : ctx->xs.ev) cudaEventDestroy(e);
  }
  if (ctx->ev_hdr) cudaEventDestroy(ctx->ev_hdr);
  if (ctx->db_s) {
    cudaStreamSynchronize(ctx->db_s);
    cudaStreamDestroy(ctx->db_s);
    cudaEventDestroy(ctx->ev_lv);
    cudaEventDestroy(ctx->ev_db);
  }
  if (ctx->h2d) {
    cudaStreamSynchronize(ctx->d2h);
    cudaStreamDestroy(ctx->h2d);
    cudaStreamDestroy(ctx->d2h);
    cudaEventDestroy(ctx->ev_bwd);
    for (auto& sl : ctx->slot) { cudaEventDestroy(sl.copied); cudaEventDestroy(sl.done); }
  }
  if (ctx->h_hdr) cudaFreeHost(ctx->h_hdr);
  delete ctx;
}

