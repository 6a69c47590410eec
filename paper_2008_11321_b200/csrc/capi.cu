// capi.cu -- the C ABI declared in include/pgc.h: argument validation,
// workspace carving, thread-local error/statistics/tuning, phase sequencing.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "pgc.h"
#include "pgc_debug.h"
#include "pgc_internal.cuh"

namespace pgc {

static thread_local char g_err[512] = "";
static thread_local pgc_stats g_stats = {};
static thread_local Tuning g_tune;
static thread_local State* g_hstate = nullptr;
static thread_local unsigned long long* g_trace_grab = nullptr;
static thread_local unsigned long long* g_trace_done = nullptr;
static thread_local int64_t g_trace_n = -1;

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(PGC_ECUDA, "CUDA error '%s' (%s) at %s", cudaGetErrorString(e), cudaGetErrorName(e),
              where);
}

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

// Resident blocks per SM of a kernel on a device (cached per thread; a
// handful of entries).
int occupancy_cached(int dev, const void* kernel, int block, size_t smem) {
  struct E { int dev; const void* k; int block; size_t smem; int occ; };
  static thread_local std::vector<E> cache;
  for (const E& e : cache)
    if (e.dev == dev && e.k == kernel && e.block == block && e.smem == smem) return e.occ;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    occ = 1;
  }
  cache.push_back({dev, kernel, block, smem, occ});
  return occ;
}

bool& once_flag(int dev, int slot) {
  static thread_local bool flags[kMaxDevices][kOnceSlots] = {};
  static thread_local bool spill = false;  // out-of-range ordinals: never "done"
  if (dev < 0 || dev >= kMaxDevices || slot < 0 || slot >= kOnceSlots) {
    spill = false;
    return spill;
  }
  return flags[dev][slot];
}

Layout make_layout(int64_t n, int64_t nnz) {
  Layout L = {};
  size_t a = 0;
  auto take = [&](size_t bytes) {
    size_t o = a;
    a = a256(a + (bytes ? bytes : 1));
    return o;
  };
  const size_t un = (size_t)n, unnz = (size_t)nnz;
  L.state = take(sizeof(State));
  L.per_round = take(sizeof(long long) * 3 * kMaxRoundStats);
  L.D = take(4 * un);
  L.rs = take(un);
  L.npred = take(4 * un);
  L.P = take(4 * unnz);
  L.U0 = take(4 * un);
  L.U1 = take(4 * un);
  L.Rl = take(4 * un);
  // chunked vertices have degree > heavy_degree >= kMinHeavyDeg (at most
  // nnz/(kMinHeavyDeg+1) of them) and need ceil(deg/chunk) <= deg/kMinChunk + 1
  // items each; a chunk record is 2 x int4
  L.chunk_cap = nnz / kMinChunk + (nnz / (kMinHeavyDeg + 1) < n ? nnz / (kMinHeavyDeg + 1) : n) + 2;
  L.chunks = take(32 * (size_t)L.chunk_cap);
  // hub descriptors: vertices with more than kExpandMin chunks have degree
  // > kExpandMin * kMinChunk
  L.cexp_cap = nnz / ((int64_t)kExpandMin * kMinChunk) + 2;
  L.cexp = take(32 * (size_t)L.cexp_cap);
  L.range_cap = n + 65536;
  L.hist1 = take(4 * (size_t)(2 * L.range_cap));
  L.base1 = take(4 * (size_t)(2 * L.range_cap + 1));
  // sum over keys of pow2ceil(ceil(cnt/T)) <= 2n/T + 2 * (nonempty keys) <= 2n/T + 2n
  L.nb_cap = 2 * n / kBucketTarget + 2 * n + 2;
  L.bcnt = take(4 * (size_t)(L.nb_cap + 1));
  L.bstart = take(4 * (size_t)(L.nb_cap + 1));
  const int64_t big = L.nb_cap > 2 * L.range_cap + 1 ? L.nb_cap : 2 * L.range_cap + 1;
  L.scan_tmp_cap = big / kScanTile + 4;
  L.scan_tmp = take(4 * (size_t)L.scan_tmp_cap);
  // JP records: n in priority order, then the bulk's heavy work
  // list (> 62 preds, so at most nnz / 63 of them; a mega vertex adds at most
  // |pred| / jp_mega_chunk items, nnz / kMinMegaChunk in all) and light list (< n)
  L.rec_heavy_cap = (nnz / 63 < n ? nnz / 63 : n) + nnz / kMinMegaChunk + 1;
  L.rec = take(16 * (size_t)(L.rec_heavy_cap + 2 * n));
  // per heavy item {mega index or -1, chunks}; per mega vertex (> kMinMegaPred
  // preds: at most nnz / (kMinMegaPred + 1)) its used-color words and a counter
  L.hmeta = take(8 * (size_t)L.rec_heavy_cap);
  L.mega_cap = nnz / (kMinMegaPred + 1) + 1;
  L.mega = take(4 * (size_t)(kMegaWords + 1) * L.mega_cap);
  L.filt = take(2 * (size_t)kFilterBytes);
  L.total = a;
  return L;
}

static bool sizes_ok(int64_t n, int64_t nnz) {
  return n >= 0 && n < ((int64_t)1 << 29) && nnz >= 0 && nnz < ((int64_t)1 << 40);
}

static int check_graph_args(const pgc_graph* g) {
  if (!g) return fail(PGC_EINVAL, "graph is NULL");
  if (!sizes_ok(g->n, g->nnz))
    return fail(PGC_EINVAL, "bad sizes n=%lld nnz=%lld (need 0 <= n < 2^29, 0 <= nnz < 2^40)",
                (long long)g->n, (long long)g->nnz);
  if (!g->row_offsets) return fail(PGC_EINVAL, "row_offsets is NULL");
  if (g->nnz > 0 && !g->col_indices) return fail(PGC_EINVAL, "col_indices is NULL");
  return 0;
}

static int check_ws(const pgc_graph* g, void* ws, size_t bytes) {
  if (!ws) return fail(PGC_EWORKSPACE, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(PGC_EWORKSPACE, "workspace not 256-byte aligned");
  const size_t need = make_layout(g->n, g->nnz).total;
  if (bytes < need)
    return fail(PGC_EWORKSPACE, "workspace too small: %zu < %zu bytes", bytes, need);
  return 0;
}

static int make_ctx(Ctx& c, const pgc_graph* g, void* ws, void* stream) {
  c.n = g->n;
  c.nnz = g->nnz;
  c.off = g->row_offsets;
  c.col = g->col_indices;
  c.st = (cudaStream_t)stream;
  c.tune = g_tune;
  cudaGetLastError();  // a stale error of earlier, unrelated work must not be blamed on this call
  int dev = 0;
  PGC_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(PGC_EINTERNAL, "device ordinal %d out of range", dev);
  c.dev = dev;
  PGC_CUDA(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, dev));
  c.lay = make_layout(g->n, g->nnz);
  char* b = (char*)ws;
  c.state = (State*)(b + c.lay.state);
  c.per_round = (long long*)(b + c.lay.per_round);
  c.D = (int32_t*)(b + c.lay.D);
  c.rs = (uint8_t*)(b + c.lay.rs);
  c.npred = (int32_t*)(b + c.lay.npred);
  c.P = (int32_t*)(b + c.lay.P);
  c.U[0] = (int32_t*)(b + c.lay.U0);
  c.U[1] = (int32_t*)(b + c.lay.U1);
  c.Rl = (int32_t*)(b + c.lay.Rl);
  c.chunks = (int4*)(b + c.lay.chunks);
  c.cexp = (int4*)(b + c.lay.cexp);
  c.hist1 = (int32_t*)(b + c.lay.hist1);
  c.base1 = (int32_t*)(b + c.lay.base1);
  c.bcnt = (int32_t*)(b + c.lay.bcnt);
  c.bstart = (int32_t*)(b + c.lay.bstart);
  c.scan_tmp = (int32_t*)(b + c.lay.scan_tmp);
  c.rec = (int4*)(b + c.lay.rec);
  c.filt = (uint32_t*)(b + c.lay.filt);
  c.hmeta = (int2*)(b + c.lay.hmeta);
  c.mega = (uint32_t*)(b + c.lay.mega);
  c.lrec = c.rec;  // ADG and JP never use their records at the same time
  // pinned host mirror of State (portable: usable from every device's streams)
  if (!g_hstate) PGC_CUDA(cudaHostAlloc((void**)&g_hstate, sizeof(State), cudaHostAllocPortable));
  c.h_state = g_hstate;
  if (g_trace_grab && g_trace_n == g->n) {
    c.trace_grab = g_trace_grab;
    c.trace_done = g_trace_done;
  }
  return 0;
}

// Per-group device timing: one event pair around every launch when enabled.
// Events are pooled per thread AND device (an event belongs to the device it
// was created on) and reused across calls.
struct EventLog {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<int> groups;
  cudaEvent_t total[2] = {nullptr, nullptr};
  cudaError_t get(cudaEvent_t* e) {
    if (used == pool.size()) {
      cudaEvent_t x = nullptr;
      if (cudaError_t r = cudaEventCreate(&x)) return r;
      pool.push_back(x);
    }
    *e = pool[used++];
    return cudaSuccess;
  }
  void reset(bool on_) {
    on = on_;
    used = 0;
    groups.clear();
  }
};
static thread_local EventLog g_logs[kMaxDevices];

int log_begin(Ctx& c, int group) {
  EventLog& L = g_logs[c.dev];
  if (!L.on) return 0;
  L.groups.push_back(group);
  cudaEvent_t e;
  PGC_CUDA(L.get(&e));
  PGC_CUDA(cudaEventRecord(e, c.st));
  return 0;
}
int log_end(Ctx& c) {
  EventLog& L = g_logs[c.dev];
  if (!L.on) return 0;
  cudaEvent_t e;
  PGC_CUDA(L.get(&e));
  PGC_CUDA(cudaEventRecord(e, c.st));
  return 0;
}

int sync_state(Ctx& c) {
  PGC_CUDA(cudaMemcpyAsync(c.h_state, c.state, sizeof(State), cudaMemcpyDeviceToHost, c.st));
  PGC_CUDA(cudaStreamSynchronize(c.st));
  ++c.syncs;
  return 0;
}

static int call_begin(Ctx& c) {
  EventLog& L = g_logs[c.dev];
  L.reset(c.tune.timing != 0);
  if (L.on) {
    if (!L.total[0]) {
      PGC_CUDA(cudaEventCreate(&L.total[0]));
      PGC_CUDA(cudaEventCreate(&L.total[1]));
    }
    PGC_CUDA(cudaEventRecord(L.total[0], c.st));
  }
  return 0;
}

// Called after the call's final synchronisation.
static void call_end(Ctx& c, int rounds, int colors, long long sum_active,
                     unsigned long long cross, unsigned long long preds, int ncore) {
  g_stats.rounds = rounds;
  g_stats.num_colors = colors;
  g_stats.sum_active = sum_active;
  g_stats.cross_edges = (int64_t)cross;
  g_stats.pred_arcs = (int64_t)preds;
  g_stats.core_vertices = ncore;
  g_stats.core_ctas = c.core_ctas;
  g_stats.kernel_launches = c.launches;
  g_stats.host_syncs = c.syncs;
  g_stats.sim_col_passes = 0;
  g_stats.jp_levels = c.jp_levels;
  g_stats.small_path = c.small;
  float t[kNumGroups] = {-1.f, -1.f, -1.f, -1.f, -1.f, -1.f};
  float total = -1.f;
  EventLog& L = g_logs[c.dev];
  if (L.on && cudaEventRecord(L.total[1], c.st) == cudaSuccess &&
      cudaEventSynchronize(L.total[1]) == cudaSuccess) {
    for (int g = 0; g < kNumGroups; ++g) t[g] = 0.f;
    for (size_t i = 0; i < L.groups.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, L.pool[2 * i], L.pool[2 * i + 1]);
      t[L.groups[i]] += ms;
    }
    cudaEventElapsedTime(&total, L.total[0], L.total[1]);
  }
  cudaGetLastError();  // timing is best effort: never leave an error behind
  g_stats.t_select_ms = t[kGSelect];
  g_stats.t_update_ms = t[kGUpdate];
  g_stats.t_adg_other_ms = t[kGAdgOther];
  g_stats.t_order_ms = t[kGOrder];
  g_stats.t_core_ms = t[kGCore];
  g_stats.t_jp_ms = t[kGJp];
  g_stats.t_total_ms = total;
}

}  // namespace pgc

using namespace pgc;

extern "C" {

size_t pgc_workspace_bytes(int64_t n, int64_t nnz) {
  if (!sizes_ok(n, nnz)) return 0;
  return make_layout(n, nnz).total;
}

int pgc_adg_order(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, int32_t* round_out,
                  int32_t* num_rounds, void* workspace, size_t workspace_bytes, void* cuda_stream) {
  return pgc_adg_order_mode(g, eps_num, eps_den, PGC_UPDATE_PUSH, round_out, num_rounds, workspace,
                            workspace_bytes, cuda_stream);
}

int pgc_adg_order_mode(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, int update_mode,
                       int32_t* round_out, int32_t* num_rounds, void* workspace,
                       size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (update_mode != PGC_UPDATE_PUSH && update_mode != PGC_UPDATE_PULL)
    return fail(PGC_EINVAL, "update_mode must be PGC_UPDATE_PUSH or PGC_UPDATE_PULL");
  if (eps_num == 0 || eps_den == 0) return fail(PGC_EINVAL, "eps must be num/den with num, den >= 1");
  if (!num_rounds || (g->n > 0 && !round_out)) return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  if (int e = adg_run(c, eps_num, eps_den, 0, round_out,
                      update_mode == PGC_UPDATE_PULL ? kAdgPull : kAdgOnly, nullptr))
    return e;
  *num_rounds = c.h_state->T;
  call_end(c, c.h_state->T, 0, c.h_state->sum_active, c.h_state->cross, 0, 0);
  return PGC_OK;
}

int pgc_jp_color(const pgc_graph* g, const int32_t* round, uint64_t seed, int32_t* color_out,
                 int32_t* num_colors, void* workspace, size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (!num_colors || (g->n > 0 && (!color_out || !round)))
    return fail(PGC_EINVAL, "input/output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  c.round_key = round;
  c.seed = seed;
  if (int e = jp_setup_run(c, round, seed, color_out)) return e;
  if (int e = jp_order_run(c, round, seed, false, false, true)) return e;
  if (int e = jp_color_run(c, color_out)) return e;
  *num_colors = c.h_state->K;
  call_end(c, 0, c.h_state->K, 0, 0, c.h_state->pred_arcs, c.core_n);
  return PGC_OK;
}

// JP-ADG; the host entry point adds `col_ready` (UPDATE of round 1 waits for
// col[], init and the first selection overlap its copy) and `side`/`h_round`
// (round[] is final after ADG: its device->host copy overlaps JP).
static int color_jp_adg_impl(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, uint64_t seed,
                             int32_t* round_out, int32_t* color_out, int32_t* num_rounds,
                             int32_t* num_colors, void* workspace, size_t workspace_bytes,
                             void* cuda_stream, cudaEvent_t col_ready, cudaStream_t side,
                             cudaEvent_t adg_done, int32_t* h_round) {
  if (int e = check_graph_args(g)) return e;
  if (eps_num == 0 || eps_den == 0) return fail(PGC_EINVAL, "eps must be num/den with num, den >= 1");
  if (!num_rounds || !num_colors || (g->n > 0 && (!round_out || !color_out)))
    return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  c.col_ready = col_ready;
  if (int e = call_begin(c)) return e;
  if (small_path_wanted(c)) {  // the whole method in one launch (small.cu)
    if (int e = small_run(c, eps_num, eps_den, seed, round_out, color_out)) return e;
    if (h_round) PGC_CUDA(cudaMemcpyAsync(h_round, round_out, 4 * (size_t)g->n, cudaMemcpyDeviceToHost, c.st));
    *num_rounds = c.h_state->T;
    *num_colors = c.h_state->K;
    call_end(c, c.h_state->T, c.h_state->K, c.h_state->sum_active, c.h_state->cross,
             c.h_state->pred_arcs, 0);
    return PGC_OK;
  }
  if (int e = adg_run(c, eps_num, eps_den, seed, round_out, kAdgFused, color_out)) return e;
  if (h_round && g->n > 0) {
    PGC_CUDA(cudaEventRecord(adg_done, c.st));
    PGC_CUDA(cudaStreamWaitEvent(side, adg_done, 0));
    PGC_CUDA(cudaMemcpyAsync(h_round, round_out, 4 * (size_t)g->n, cudaMemcpyDeviceToHost, side));
  }
  const int T = c.h_state->T;
  const long long sum_active = c.h_state->sum_active;
  const unsigned long long cross = c.h_state->cross, preds = c.h_state->pred_arcs;
  c.round_key = round_out;
  c.seed = seed;
  if (int e = jp_order_run(c, round_out, seed, true, false, true)) return e;
  if (int e = jp_color_run(c, color_out)) return e;
  *num_rounds = T;
  *num_colors = c.h_state->K;
  call_end(c, T, c.h_state->K, sum_active, cross, preds, c.core_n);
  return PGC_OK;
}

int pgc_color_jp_adg(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, uint64_t seed,
                     int32_t* round_out, int32_t* color_out, int32_t* num_rounds,
                     int32_t* num_colors, void* workspace, size_t workspace_bytes,
                     void* cuda_stream) {
  return color_jp_adg_impl(g, eps_num, eps_den, seed, round_out, color_out, num_rounds, num_colors,
                           workspace, workspace_bytes, cuda_stream, nullptr, nullptr, nullptr,
                           nullptr);
}

int pgc_adg_m_order(const pgc_graph* g, int32_t* round_out, int32_t* num_rounds, void* workspace,
                    size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (!num_rounds || (g->n > 0 && !round_out)) return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  if (int e = adg_run(c, 1, 1, 0, round_out, kAdgOnly, nullptr, kRuleMedian)) return e;
  *num_rounds = c.h_state->T;
  call_end(c, c.h_state->T, 0, c.h_state->sum_active, c.h_state->cross, 0, 0);
  return PGC_OK;
}

int pgc_color_jp_adg_m(const pgc_graph* g, uint64_t seed, int32_t* round_out, int32_t* color_out,
                       int32_t* num_rounds, int32_t* num_colors, void* workspace,
                       size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (!num_rounds || !num_colors || (g->n > 0 && (!round_out || !color_out)))
    return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  if (int e = adg_run(c, 1, 1, seed, round_out, kAdgFused, color_out, kRuleMedian)) return e;
  const int T = c.h_state->T;
  const long long sum_active = c.h_state->sum_active;
  const unsigned long long cross = c.h_state->cross, preds = c.h_state->pred_arcs;
  c.round_key = round_out;
  c.seed = seed;
  if (int e = jp_order_run(c, round_out, seed, true, false, true)) return e;
  if (int e = jp_color_run(c, color_out)) return e;
  *num_rounds = T;
  *num_colors = c.h_state->K;
  call_end(c, T, c.h_state->K, sum_active, cross, preds, c.core_n);
  return PGC_OK;
}

int pgc_color_jp_adg_o(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, int32_t* round_out,
                       int32_t* color_out, int32_t* num_rounds, int32_t* num_colors,
                       void* workspace, size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (eps_num == 0 || eps_den == 0) return fail(PGC_EINVAL, "eps must be num/den with num, den >= 1");
  if (!num_rounds || !num_colors || (g->n > 0 && (!round_out || !color_out)))
    return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  if (int e = adg_run(c, eps_num, eps_den, 0, round_out, kAdgFusedO, color_out)) return e;
  const int T = c.h_state->T;
  const long long sum_active = c.h_state->sum_active;
  const unsigned long long cross = c.h_state->cross, preds = c.h_state->pred_arcs;
  int32_t* key1 = c.U[0];  // ADG's lists are free after the last round
  if (int e = adg_o_keys(c, round_out, key1)) return e;
  if (int e = jp_order_run(c, key1, 0, false, true, true)) return e;
  if (c.h_state->err == 6)
    return fail(PGC_EINVAL, "ADG-O: sum over rounds of (max residual degree + 1) exceeds INT32_MAX");
  c.round_key = round_out;  // the bulk's watch heuristic (never a result)
  c.seed = 0;
  if (int e = jp_color_run(c, color_out)) return e;
  *num_rounds = T;
  *num_colors = c.h_state->K;
  call_end(c, T, c.h_state->K, sum_active, cross, preds, c.core_n);
  return PGC_OK;
}

int pgc_jp_baseline(const pgc_graph* g, int kind, uint64_t seed, int32_t* color_out,
                    int32_t* num_colors, void* workspace, size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (kind < PGC_JP_R || kind > PGC_JP_LLF) return fail(PGC_EINVAL, "unknown JP baseline %d", kind);
  if (!num_colors || (g->n > 0 && !color_out)) return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  int32_t* key = c.U[0];  // free until the bulk split (after the order)
  if (int e = baseline_key_run(c, kind, key)) return e;
  c.round_key = nullptr;  // U0 is reused by the bulk split: the bulk watches by hash alone
  c.seed = seed;
  if (int e = jp_setup_run(c, key, seed, color_out)) return e;
  if (int e = jp_order_run(c, key, seed, false, false, true)) return e;
  if (int e = jp_color_run(c, color_out)) return e;
  *num_colors = c.h_state->K;
  call_end(c, 0, c.h_state->K, 0, 0, c.h_state->pred_arcs, c.core_n);
  return PGC_OK;
}

int pgc_color_dec_adg_itr(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, uint64_t seed,
                          int32_t* round_out, int32_t* color_out, int32_t* num_rounds,
                          int32_t* num_colors, void* workspace, size_t workspace_bytes,
                          void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (eps_num == 0 || eps_den == 0) return fail(PGC_EINVAL, "eps must be num/den with num, den >= 1");
  if (!num_rounds || !num_colors || (g->n > 0 && (!round_out || !color_out)))
    return fail(PGC_EINVAL, "output pointer is NULL");
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  if (int e = call_begin(c)) return e;
  if (int e = adg_run(c, eps_num, eps_den, seed, round_out, kAdgOnly, color_out)) return e;
  const int T = c.h_state->T;
  const long long sum_active = c.h_state->sum_active;
  const unsigned long long cross = c.h_state->cross;
  // the partitions R(T), ..., R(1) as ranges of the priority order
  if (int e = jp_order_run(c, round_out, seed, true)) return e;
  PGC_CUDA(cudaMemsetAsync(&c.state->K, 0, sizeof(int), c.st));
  if (g->n > 0) {  // nonempty graph: K >= 1 (isolated vertices already hold color 1)
    const int one = 1;
    PGC_CUDA(cudaMemcpyAsync(&c.state->K, &one, sizeof(int), cudaMemcpyHostToDevice, c.st));
  }
  long long passes = 0;
  if (int e = dec_itr_run(c, round_out, seed, color_out, &passes)) return e;
  *num_rounds = T;
  *num_colors = c.h_state->K;
  call_end(c, T, c.h_state->K, sum_active, cross, 0, 0);
  g_stats.sim_col_passes = (int32_t)(passes > 0x7fffffff ? 0x7fffffff : passes);
  return PGC_OK;
}

size_t pgc_host_workspace_bytes(int64_t n, int64_t nnz) {
  if (!sizes_ok(n, nnz)) return 0;
  return a256(8 * (size_t)(n + 1)) + a256(4 * (size_t)nnz) + 2 * a256(4 * (size_t)n) +
         make_layout(n, nnz).total;
}

int pgc_color_jp_adg_host(int64_t n, int64_t nnz, const int64_t* h_row_offsets,
                          const int32_t* h_col_indices, uint32_t eps_num, uint32_t eps_den,
                          uint64_t seed, int32_t* h_round_out, int32_t* h_color_out,
                          int32_t* num_rounds, int32_t* num_colors, void* workspace,
                          size_t workspace_bytes, void* cuda_stream) {
  if (!sizes_ok(n, nnz)) return fail(PGC_EINVAL, "bad sizes n=%lld nnz=%lld", (long long)n, (long long)nnz);
  if (!h_row_offsets || (nnz > 0 && !h_col_indices) || (n > 0 && (!h_round_out || !h_color_out)))
    return fail(PGC_EINVAL, "host pointer is NULL");
  if (!workspace) return fail(PGC_EWORKSPACE, "workspace is NULL");
  if (((uintptr_t)workspace & 255) != 0) return fail(PGC_EWORKSPACE, "workspace not 256-byte aligned");
  if (workspace_bytes < pgc_host_workspace_bytes(n, nnz))
    return fail(PGC_EWORKSPACE, "workspace too small: %zu < %zu bytes", workspace_bytes,
                pgc_host_workspace_bytes(n, nnz));
  char* b = (char*)workspace;
  int64_t* d_off = (int64_t*)b;
  b += a256(8 * (size_t)(n + 1));
  int32_t* d_col = (int32_t*)b;
  b += a256(4 * (size_t)nnz);
  int32_t* d_round = (int32_t*)b;
  b += a256(4 * (size_t)n);
  int32_t* d_color = (int32_t*)b;
  b += a256(4 * (size_t)n);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  // a side stream (per thread, created once) carries col[] host->device and
  // round[] device->host, overlapping the first ADG kernels and JP
  // (per thread and device: streams and events belong to one device)
  static thread_local cudaStream_t sides[64] = {};
  static thread_local cudaEvent_t evs[64][3] = {};
  int dev = 0;
  PGC_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(PGC_EINTERNAL, "device ordinal %d out of range", dev);
  cudaStream_t& side = sides[dev];
  cudaEvent_t* ev = evs[dev];
  if (!side) {
    PGC_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i) PGC_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  }
  PGC_CUDA(cudaEventRecord(ev[0], st));  // the side stream starts after st's earlier work
  PGC_CUDA(cudaStreamWaitEvent(side, ev[0], 0));
  PGC_CUDA(cudaMemcpyAsync(d_off, h_row_offsets, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, st));
  if (nnz > 0)
    PGC_CUDA(cudaMemcpyAsync(d_col, h_col_indices, 4 * (size_t)nnz, cudaMemcpyHostToDevice, side));
  PGC_CUDA(cudaEventRecord(ev[1], side));
  pgc_graph g = {n, nnz, d_off, d_col};
  int rc = color_jp_adg_impl(&g, eps_num, eps_den, seed, d_round, d_color, num_rounds, num_colors,
                             b, workspace_bytes - (size_t)(b - (char*)workspace), cuda_stream,
                             ev[1], side, ev[2], n > 0 ? h_round_out : nullptr);
  if (rc == PGC_OK && n > 0)
    PGC_CUDA(cudaMemcpyAsync(h_color_out, d_color, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
  PGC_CUDA(cudaStreamSynchronize(side));  // also on error: nothing may stay in flight
  PGC_CUDA(cudaStreamSynchronize(st));
  return rc;
}

int pgc_check_graph(const pgc_graph* g, void* workspace, size_t workspace_bytes, void* cuda_stream) {
  if (int e = check_graph_args(g)) return e;
  if (int e = check_ws(g, workspace, workspace_bytes)) return e;
  Ctx c;
  if (int e = make_ctx(c, g, workspace, cuda_stream)) return e;
  int64_t bad = -1;
  if (int e = check_graph_run(c, &bad)) return e;
  if (bad >= 0)
    return fail(PGC_EINVAL, "CSR invariant violated at vertex %lld (offsets, range, order, self-loop or symmetry)",
                (long long)bad);
  return PGC_OK;
}

int pgc_last_stats(pgc_stats* out) {
  if (!out) return fail(PGC_EINVAL, "out is NULL");
  *out = g_stats;
  return PGC_OK;
}

const char* pgc_last_error(void) { return g_err; }

int pgc_set_tuning(const char* key, int64_t value) {
  if (!key) return fail(PGC_EINVAL, "key is NULL");
  if (!strcmp(key, "timing") && (value == 0 || value == 1)) {
    g_tune.timing = (int)value;
    return PGC_OK;
  }
  if (!strcmp(key, "rounds_per_sync") && value >= 1 && value <= 1 << 16) {
    g_tune.rounds_per_sync = (int)value;
    return PGC_OK;
  }
  if (!strcmp(key, "heavy_degree") && value >= kMinHeavyDeg && value <= (1 << 30)) {
    g_tune.heavy_degree = (int)value;
    return PGC_OK;
  }
  if (!strcmp(key, "jp_mega_pred") && (value == 0 || (value >= kMinMegaPred && value <= (1 << 30)))) {
    g_tune.jp_mega_pred = (int)value;
    return PGC_OK;
  }
  if (!strcmp(key, "chunk_arcs") && value >= kMinChunk && value <= (1 << 24)) {
    g_tune.chunk_arcs = (int)value;
    return PGC_OK;
  }
  struct Key { const char* name; long long lo, hi; long long* l; int* i; };
  const Key keys[] = {
      {"jp_watchdog_ms", 1, 3600000, nullptr, &g_tune.jp_watchdog_ms},
      {"filter_ratio", 0, 1 << 20, nullptr, &g_tune.filter_ratio},
      {"jp_heavy_warps", 1, 4, nullptr, &g_tune.jp_heavy_warps},
      {"jp_heavy_batch", 1, 64, nullptr, &g_tune.jp_heavy_batch},
      {"jp_heavy_stripes", 1, kMaxHeavyStripes, nullptr, &g_tune.jp_heavy_stripes},
      {"jp_mega_chunk", kMinMegaChunk, kMegaBits, nullptr, &g_tune.jp_mega_chunk},
      {"jp_heavy_sleep_max", 0, 1000000, nullptr, &g_tune.jp_heavy_sleep_max},
      {"jp_light_sleep_max", 0, 1000000, nullptr, &g_tune.jp_light_sleep_max},
      {"core_max", 0, 65535, nullptr, &g_tune.core_max},
      {"core_min_avg", 0, 1 << 30, nullptr, &g_tune.core_min_avg},
      {"core_div", 0, 1 << 30, nullptr, &g_tune.core_div},
      {"core_dmul", 0, 1 << 20, nullptr, &g_tune.core_dmul},
      {"core_min_n", 1, 65535, nullptr, &g_tune.core_min_n},
      {"core_ctas", 0, 16, nullptr, &g_tune.core_ctas},
      {"core_spin_ns", 0, 100000, nullptr, &g_tune.core_spin_ns},
      {"core_tail_ns", 0, 100000, nullptr, &g_tune.core_tail_ns},
      {"core_pass_ns", 0, 100000, nullptr, &g_tune.core_pass_ns},
      {"core_near", 0, 512, nullptr, &g_tune.core_near},
      {"core_tier2", 0, 65535, nullptr, &g_tune.core_tier2},
      {"itr_blocks_per_sm", 0, 64, nullptr, &g_tune.itr_blocks_per_sm},
      {"itr_members_per_warp", 1, 1024, nullptr, &g_tune.itr_members_per_warp},
      {"jp_split_overlap", 0, 1, nullptr, &g_tune.jp_split_overlap},
      {"update_atom", 0, 1, nullptr, &g_tune.update_atom},
      {"fuse_init", 0, 1, nullptr, &g_tune.fuse_init},
      {"top_list", 0, 1, nullptr, &g_tune.top_list},
      {"levels", 0, 1, nullptr, &g_tune.levels},
      {"core_arc_cap", 0, 1ll << 40, &g_tune.core_arc_cap, nullptr},
      {"small_max_arcs", 0, 1ll << 40, &g_tune.small_max_arcs, nullptr},
      {"small_max_avg", 0, 1 << 30, nullptr, &g_tune.small_max_avg},
      {"small_blocks_per_sm", 0, 64, nullptr, &g_tune.small_blocks_per_sm},
      {"tiny_max_n", 0, 1ll << 30, &g_tune.tiny_max_n, nullptr},
      {"tiny_max_arcs", 0, 1ll << 40, &g_tune.tiny_max_arcs, nullptr},
      {"tiny_dataflow", 0, 1, nullptr, &g_tune.tiny_dataflow},
      {"core_arcs_per_cta", 1, 1ll << 40, &g_tune.core_arcs_per_cta, nullptr},
  };
  for (const Key& k : keys)
    if (!strcmp(key, k.name) && value >= k.lo && value <= k.hi) {
      if (k.l) *k.l = value;
      else *k.i = (int)value;
      return PGC_OK;
    }
  if (!strcmp(key, "block_threads") && value >= 64 && value <= 1024 && value % 32 == 0) {
    g_tune.block_threads = (int)value;
    return PGC_OK;
  }
  return fail(PGC_EINVAL, "unknown tuning key or value out of range: %s=%lld", key, (long long)value);
}

int pgc_version(void) { return PGC_VERSION; }

int pgc_debug_set_trace(uint64_t* t_grab, uint64_t* t_done, int64_t n) {
  if (n < 0 || (!t_grab) != (!t_done)) return fail(PGC_EINVAL, "trace: need both pointers and n >= 0");
  g_trace_grab = (unsigned long long*)t_grab;
  g_trace_done = (unsigned long long*)t_done;
  g_trace_n = t_grab ? n : -1;
  return PGC_OK;
}

}  // extern "C"
