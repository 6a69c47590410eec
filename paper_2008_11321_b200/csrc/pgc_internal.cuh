// pgc_internal.cuh -- shared internals of the B200 JP-ADG library (product path).
//
// Nothing here is shared with oracle/ (the CPU oracle is test infrastructure;
// the two share no code, header or constant table).
#pragma once

#include <cstddef>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys/ncu (no-ops without a tool)

namespace pgc {

constexpr int kWarp = 32;
constexpr int kExpandMin = 8;        // a vertex with more chunks gets one descriptor; k_round_aux writes its records
constexpr int kMinChunk = 256;        // smallest allowed arcs-per-work-item for chunked vertices
constexpr int kMinHeavyDeg = 128;     // smallest allowed heavy_degree (sizes the chunk records)
// JP bulk mega vertices (jp.cu): a vertex with more than jp_mega_pred preds is
// colored by ceil(|pred| / jp_mega_chunk) warps, one per chunk of its pred
// list, which OR their preds' colors into a kMegaBits-bit used-color set
constexpr int kMegaBits = 2048;       // = the heavy byte-map window: colors 1..2048
constexpr int kMegaWords = kMegaBits / 32;
constexpr int kMinMegaPred = 1024;    // smallest allowed jp_mega_pred (sizes the mega state)
constexpr int kMaxHeavyStripes = 8;   // JP bulk: heavy ticket counters (jp_heavy_stripes)
constexpr int kMinMegaChunk = 256;    // smallest allowed jp_mega_chunk (sizes the heavy list)
constexpr int kMaxRoundStats = 4096;  // per-round statistics kept in the workspace
constexpr int kCoreCap = 65536;       // JP core: at most this many vertices (u16 positions)
#ifndef PGC_BUCKET_TARGET
#define PGC_BUCKET_TARGET 8
#endif
constexpr int kBucketTarget = PGC_BUCKET_TARGET;  // mean bucket occupancy target of the priority-order sort
constexpr int kScanTile = 4096;       // elements per block in the device-wide scan

// Device-resident scalars of one call.  Lives at the head of the workspace.
// Counters that many blocks or warps hit with atomics sit on their own
// 128-byte lines (alignas): one L2 slice serves one line, so two hot counters
// sharing a line would make that slice the bottleneck of both (the JP bulk's
// light and heavy tickets and K were one line in round 1: 91 % tag rate on
// the max slice vs 52 % mean).
struct State {
  // ADG round state (Alg. 1)
  unsigned long long S;        // sum_{v in U} D[v] for the current round
  long long nU;                // |U| for the current round
  int done;                    // 1 once U is empty
  int err;                     // internal invariant failure code (0 = none)
  int T;                       // rounds completed
  int pad0;
  // totals
  long long sum_active;        // sum_l |U_l|
  unsigned long long cross;    // X
  long long avg_max;           // max over the rounds so far of floor(S_l / |U_l|): the densest U_l's mean degree
  // counters of the current round, reset by k_adg_finalize: the compaction
  // reservations of k_adg_select (one atomic per block step each)
  alignas(128) int nChunks;
  int nLight, nUnext;
  int nExp;                    // hub descriptors of this round (k_round_aux writes their chunk records)
  // ... the selection's block sums
  alignas(128) unsigned long long sumDR;  // sum of D over R_l
  int nR;
  int nOrdR;                   // non-isolated vertices of R_l (the priority order's round histogram)
  // ... UPDATE's block sums
  alignas(128) unsigned long long cut;    // arcs from R_l into U_{l+1}
  unsigned long long pred_arcs;  // sum_v |pred(v)|
  alignas(128) int top_n;      // length of the saved top-round list (k_round_aux; 0 = none)
  // priority-order sort
  int rmin, rmax;              // range of the first priority key
  int nbuckets;                // buckets in use
  int sorted;                  // total placed by the scan (== n_order)
  int n_order;                 // vertices in the priority order: all but the isolated ones
  int ord_ktop;                // split order: keys 0..ord_ktop (the top rounds) placed first
  int ord_btop;                // ... their buckets are 0..ord_btop-1
  int ord_ptop;                // ... and positions 0..ord_ptop-1
  int sorted_bot;              // split order: placed by the bottom part
  // JP
  int core_n;                  // |core| = length of the priority prefix colored by k_jp_core
                               // (both tiers)
  int core_n1;                 // tier 1 of the core: positions [0, core_n1) (u16 lists);
                               // tier 2: [core_n1, core_n) (int32 codes, after tier 1)
  long long core_arcs;         // sum of |pred| over the core
  int nheavy;                  // bulk heavy work items (vertices with |pred| > kLightPredMax;
                               // a mega vertex counts once per pred chunk)
  int nmega;                   // bulk mega vertices (|pred| > jp_mega_pred), split into chunks
  int nlight;                  // bulk vertices with 1 <= |pred| <= kLightPredMax
  int jp_levels;               // J, when the levels knob is on (k_jp_levels)
  alignas(128) int K;          // max color (atomicMax per warp)
  alignas(128) int ticket_heavy;  // next bulk tickets per class (heavy: stripe 0)
  // heavy stripes 1..kMaxHeavyStripes-1 (jp_heavy_stripes), 128 bytes apart
  alignas(128) int ticket_hs[(kMaxHeavyStripes - 1) * 32];
  alignas(128) int ticket_light;
  alignas(128) int ticket_levels;  // k_jp_levels' tickets
  // ADG-M radix select of the ceil(|U|/2)-th smallest key (D[v] << 32) | v
  alignas(128) unsigned long long msel_key;  // key bits found so far (the full key after the last pass)
  unsigned long long msel_mask;  // which key bits msel_key determines
  long long msel_rank;           // rank still to find among keys matching msel_key (1-based)
  int msel_done;                 // blocks finished in the current pass (last-block pick)
  int maxdeg;                    // maximum degree (ADG-M's radix schedule)
};

// Byte offsets of every workspace region (each 256-byte aligned).
struct Layout {
  size_t state, per_round, D, rs, npred, P, U0, U1, Rl, chunks, cexp, hist1, base1, bcnt, bstart,
      scan_tmp, rec, hmeta, mega, filt, total;
  int64_t chunk_cap, cexp_cap, range_cap, nb_cap, scan_tmp_cap, rec_heavy_cap, mega_cap;
};

Layout make_layout(int64_t n, int64_t nnz);

struct Tuning {
  int timing = 0;
  int rounds_per_sync = 8;
  int heavy_degree = 128;   // vertices with more arcs are split into edge chunks
  int chunk_arcs = 1024;    // arcs per chunk work item
  int filter_ratio = 4;     // UPDATE: filtered heavy kernel once |U_l| * ratio <= filter bits (0 = off)
  int jp_heavy_warps = 4;         // warps per 8-warp bulk JP block serving heavy vertices (1..4)
  int jp_heavy_batch = 1;         // heavy tickets per atomic (consecutive, per warp)
  int jp_heavy_stripes = 1;       // heavy list dealt round-robin to this many ticket counters
  int jp_mega_pred = 2048;        // bulk vertices with more preds are split into pred chunks,
                                  // colored by several warps (0 = off; else >= kMinMegaPred)
  int jp_mega_chunk = 512;        // preds per chunk (kMinMegaChunk .. kMegaBits)
  int jp_heavy_sleep_max = 256;   // ns, exponential backoff cap of waiting heavy warps
  int jp_light_sleep_max = 8192;  // ns, same for light warps
  int jp_watchdog_ms = 20000;     // JP kernel reports a stall after this long
  int core_max = 65535;           // JP core: max vertices (0 disables the core engine)
  int core_dmul = 20;             // JP core (after ADG): at most max(16 384, core_dmul * max_l mean degree of G[U_l]) vertices (0 = off)
  int core_div = 32;              // JP core: at most max(16 384, n_order / core_div) vertices (0 = no such cap)
  int core_min_avg = 32;          // JP core: min mean |pred| over the prefix
  int core_min_n = 256;           // JP core: smaller cores are left to the bulk kernel
  int core_ctas = 0;              // JP core: cluster size (0 = from core_arcs_per_cta)
  int core_spin_ns = 1024;        // JP core: backoff cap (ns) of a warp still several preds away
  int core_tail_ns = 0;           // JP core: sleep (ns) per poll of a warp in the tail
  int core_pass_ns = 0;           // JP core: min sleep (ns) between passes of a warp far from its tail
  int core_near = 0;              // JP core: warps with at most this many pending preds poll without backoff
  int core_tier2 = 0;             // JP core: a second cluster pass over the next <= this many
                                  // positions when tier 1 is capped (0 = off; measured slower
                                  // on R-MAT 24 / Chung-Lu / R-MAT 20)
  int itr_blocks_per_sm = 0;      // DEC-ADG-ITR: blocks per SM of the cooperative kernel (0 = occupancy)
  int itr_members_per_warp = 1;   // DEC-ADG-ITR: partition members per warp of the pass grid
  int jp_split_overlap = 1;       // JP: run the bulk split on a side stream beside the core kernel
  int top_list = 1;               // JP-ADG: ADG saves the top rounds' list for the split order
  int fuse_init = 1;              // ADG: round 1's selection also initialises D, rs, round, color
  int update_atom = 1;            // ADG round 1: one atomic per arc instead of gather + RED (Arc::atom)
  int levels = 0;                 // JP: also compute J = the longest path of G_rho (k_jp_levels;
                                  // diagnostics, off in timed runs)
  // JP-ADG on small / low-degree graphs: one persistent cooperative kernel
  // (small.cu) when nnz <= small_max_arcs and nnz <= small_max_avg * n
  long long small_max_arcs = 1ll << 24;    // 0 disables the one-kernel path
  int small_max_avg = 20;
  int small_blocks_per_sm = 0;             // blocks per SM of that kernel (0 = occupancy)
  // ... on ONE thread-block cluster with the per-vertex state in distributed
  // shared memory (k_tiny_jp_adg) when n <= tiny_max_n (and it fits) and
  // nnz <= tiny_max_arcs; tiny_max_n = 0 disables
  long long tiny_max_n = 1ll << 17;
  long long tiny_max_arcs = 1ll << 22;
  int tiny_dataflow = 1;                   // ... its JP as a barrier-free dataflow (else by levels)
  long long core_arc_cap = 1ll << 30;      // JP core: max sum |pred|
  long long core_arcs_per_cta = 2 << 20;   // JP core: pred arcs per cluster CTA
  int block_threads = 256;
};

// Positions the JP core engine may cover (tier 1 + tier 2): the split
// priority order sorts at least this many before the core starts.
inline int core_reach(const Tuning& t) {
  const long long r = (long long)t.core_max + (t.core_max > 0 ? t.core_tier2 : 0);
  return r > 0x7fffffff ? 0x7fffffff : (int)r;
}

// Kernel groups for per-group device timing (pgc_stats.t_*_ms).
enum Group { kGSelect = 0, kGUpdate = 1, kGAdgOther = 2, kGOrder = 3, kGCore = 4, kGJp = 5,
             kNumGroups = 6 };

// Everything a phase needs; built by the C-ABI layer from the caller's arguments.
struct Ctx {
  int launches = 0;  // kernels launched by this call
  int syncs = 0;     // host synchronisations by this call
  int dev = 0;       // the device of this call (cudaGetDevice at entry)
  int jp_levels = 0; // J of the last JP (levels knob), else 0
  int small = 0;     // the one-kernel small-graph path ran (small.cu): 1 grid, 2 one cluster
  int64_t n, nnz;
  const int64_t* off;
  const int32_t* col;
  cudaStream_t st;
  int nsm;
  Tuning tune;
  Layout lay;
  State* state;
  long long* per_round;  // [kMaxRoundStats][3] = (|U_l|, S_l, |R_l|)
  int32_t* D;
  uint8_t* rs;  // 1-byte round state: 0 = alive, else ((round-1) % 255) + 1 (L2-resident)
  int32_t* npred;
  int32_t* P;
  int32_t* U[2];
  int32_t* Rl;
  uint32_t* filt;  // 2 x kFilterWords: UPDATE membership filters of U_l (double-buffered)
  int4* lrec;      // UPDATE light work records (aliases the JP bulk record region)
  int4* chunks;    // UPDATE edge-chunk records, 2 x int4 each
  int4* cexp;      // hub descriptors (2 x int4 each) of vertices with > kExpandMin chunks
  int32_t* hist1;
  int32_t* base1;
  int32_t* bcnt;
  int32_t* bstart;
  int32_t* scan_tmp;
  int4* rec;       // JP records {v, |pred|, P slot}: n in priority order, then the
                   // bulk's heavy and light lists
  int2* hmeta;     // per heavy item: {mega index (-1: a whole vertex), chunks}
  uint32_t* mega;  // per mega vertex: kMegaWords used-color words, then (after all
                   // mega_cap of them) one finished-chunk counter each
  const int32_t* round_key = nullptr;  // JP first priority key (rho_ADG for JP-ADG)
  uint64_t seed = 0;                   // JP tie-break seed
  int core_ctas = 0;                   // cluster size used by the last k_jp_core (0 = none)
  int core_n = 0;                      // core vertices colored by k_jp_core (0 = none)
  // split order (jp_order_run with defer): the bottom part still to place
  bool ord_pending = false;
  bool ord_deferred = false;
  bool top_list = false;  // ADG saved U_l (the last with |U_l| >= core_max) in Rl
  const int32_t* ord_round = nullptr;
  uint64_t ord_seed = 0;
  int ord_idshift = 0;
  State* h_state;  // pinned host mirror
  cudaEvent_t col_ready = nullptr;  // host entry point: col[] still in flight until this event
  unsigned long long* trace_grab = nullptr;  // pgc_debug_set_trace (diagnostics)
  unsigned long long* trace_done = nullptr;
};

// UPDATE membership filter (adg.cu): 1 M bits (128 KB) per buffer
constexpr int kFilterBytes = 128 * 1024;
constexpr int kFilterWords = kFilterBytes / 4;

// ---- phases (host orchestration; return 0 or a PGC_* code) -----------------
// kAdgFusedO: JP Part 1 for ADG-O's total order (round, D_rem, id) (Q22)
// kAdgPull: ADG only, with the pull (CREW) UPDATE
enum AdgMode { kAdgOnly = 0, kAdgFused = 1, kAdgFusedO = 3, kAdgPull = 4 };
// selection rule of a round: ADG's mean threshold (Alg. 1) or ADG-M's median
//
enum AdgRule { kRuleMean = 0, kRuleMedian = 1 };
int adg_run(Ctx& c, uint32_t num, uint32_t den, uint64_t seed, int32_t* round, int mode,
            int32_t* color_zero, int rule = kRuleMean);
int jp_setup_run(Ctx& c, const int32_t* round, uint64_t seed, int32_t* color);
int adg_o_keys(Ctx& c, const int32_t* round, int32_t* key1);
int baseline_key_run(Ctx& c, int kind, int32_t* key);
int dec_itr_run(Ctx& c, const int32_t* round, uint64_t seed, int32_t* color, long long* passes);
// defer: place only the top rounds' records (enough for the JP core's prefix)
// and leave the rest to jp_color_run, which places them beside the core kernel
int jp_order_run(Ctx& c, const int32_t* round, uint64_t seed, bool range_known, bool idkey = false,
                 bool defer = false);
int jp_color_run(Ctx& c, int32_t* color);
int check_graph_run(Ctx& c, int64_t* bad_vertex);
// JP-ADG in one persistent kernel for small / low-degree graphs (small.cu)
bool small_path_wanted(const Ctx& c);
int small_run(Ctx& c, uint32_t num, uint32_t den, uint64_t seed, int32_t* round, int32_t* color);

// error reporting helper implemented in capi.cu
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);
// per-group event timing (no-ops unless timing is enabled; a failed event
// record returns PGC_ECUDA naming the event, not the next kernel); capi.cu
int log_begin(Ctx& c, int group);
int log_end(Ctx& c);
// A per-thread, per-device "done once" flag (function attributes such as the
// dynamic shared memory opt-in apply to the device they were set on, so a
// thread that drives two GPUs must set them on each).  slot < kOnceSlots.
// Slots: 0-4 k_update_heavy_f per Arc mode (adg.cu), 8 k_jp_core attributes,
// 9 side-stream kernels loaded (jp.cu), 10 k_tiny_jp_adg attributes,
// 11 k_small_jp_adg loaded (small.cu).
constexpr int kOnceSlots = 16;
constexpr int kMaxDevices = 64;
bool& once_flag(int dev, int slot);
// copy State to the pinned host mirror and wait for the stream; capi.cu
int sync_state(Ctx& c);

// Checked builds: the graph's sizes in device globals of each translation
// unit (set by its host phases), for vertex / arc bounds in PGC_DCHECKs.
#ifdef PGC_CHECKED
static __device__ long long g_chk_n = 0, g_chk_nnz = 0;
inline void chk_sizes(const Ctx& c) {
  cudaMemcpyToSymbolAsync(g_chk_n, &c.n, sizeof(long long), 0, cudaMemcpyHostToDevice, c.st);
  cudaMemcpyToSymbolAsync(g_chk_nnz, &c.nnz, sizeof(long long), 0, cudaMemcpyHostToDevice, c.st);
}
#define PGC_CHK_SIZES(c) ::pgc::chk_sizes(c)
#define PGC_DCHECK_V(u) PGC_DCHECK((long long)(u) >= 0 && (long long)(u) < ::pgc::g_chk_n, u, ::pgc::g_chk_n)
#define PGC_DCHECK_A(e) PGC_DCHECK((long long)(e) >= 0 && (long long)(e) < ::pgc::g_chk_nnz, e, ::pgc::g_chk_nnz)
#else
#define PGC_CHK_SIZES(c) \
  do {                   \
  } while (0)
#define PGC_DCHECK_V(u) \
  do {                  \
  } while (0)
#define PGC_DCHECK_A(e) \
  do {                  \
  } while (0)
#endif

// An NVTX range over a host phase (entry points, ADG, the priority order,
// the JP kernels): the phases show up by name in nsys / ncu --nvtx.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Launch a kernel (variadic so the <<<...>>> commas survive), check the launch,
// account it and time it in `group`.
#define PGC_LAUNCH(c, group, name, ...)                         \
  do {                                                          \
    if (int le_ = ::pgc::log_begin(c, group)) return le_;       \
    __VA_ARGS__;                                                \
    cudaError_t e_ = cudaGetLastError();                        \
    if (e_ != cudaSuccess) return ::pgc::cuda_fail(e_, name);   \
    if (int le_ = ::pgc::log_end(c)) return le_;                \
    ++(c).launches;                                             \
  } while (0)

#define PGC_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return ::pgc::cuda_fail(e_, #call); \
  } while (0)

#define PGC_LAUNCHED(name)                                        \
  do {                                                            \
    cudaError_t e_ = cudaGetLastError();                          \
    if (e_ != cudaSuccess) return ::pgc::cuda_fail(e_, name);     \
  } while (0)

// ---- checked builds ---------------------------------------------------------
// compute-sanitizer is closed on the GPU pool, so the checked library
// (tools/micro/build_checked.sh, -DPGC_CHECKED; never the product build)
// turns every PGC_DCHECK into a device assertion: a failed bound or invariant
// prints its file, line and values and traps (the call returns PGC_ECUDA).
#ifdef PGC_CHECKED
#define PGC_DCHECK(cond, a, b)                                                            \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("PGC_CHECKED failed: %s at %s:%d (%lld, %lld) block %d thread %d\n", #cond, \
             __FILE__, __LINE__, (long long)(a), (long long)(b), (int)blockIdx.x,         \
             (int)threadIdx.x);                                                           \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define PGC_DCHECK(cond, a, b) \
  do {                         \
  } while (0)
#endif

// ---- device helpers ---------------------------------------------------------
// rho_R(v) = splitmix64(seed ^ v): the first output of a SplitMix64 generator
// whose state is seed^v (published constants).
__device__ __forceinline__ uint64_t prio_hash(uint64_t seed, uint32_t v) {
  uint64_t z = (seed ^ (uint64_t)v) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int32_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.relaxed.gpu.global.u16 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u16(uint16_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}

// streaming (evict-first) accesses for data touched once: keeps the L2 for the
// randomly gathered per-vertex state (rs, D, colors).
__device__ __forceinline__ int ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(int32_t* p, int v) { __stcs(p, v); }

// Per-vertex ADG state that UPDATE hits at random (D[] by RED, rs[] by gather)
// is marked L2 evict-last, so the streams that pass through the L2 once (col,
// records, P) do not push it out (PGC_NO_L2HINT builds the plain accesses for A/B).
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// D[u] -= 1 with the result unused (a RED), evict-last
__device__ __forceinline__ void red_dec_keep(int32_t* a) {
#ifdef PGC_NO_L2HINT
  atomicSub(a, 1);
#else
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(a), "r"(-1),
               "l"(l2_keep_policy())
               : "memory");
#endif
}
// DecrementAndFetch with the old value returned (round 1's
// classifying atomic, Arc::atom), evict-last like the RED: an ATOM that misses
// the L2 waits for DRAM, and the probe (tools/micro/footprint_probe.cu) puts
// the ATOM rate at 126 G/s while the state stays in the L2 and 55 G/s once it
// does not
__device__ __forceinline__ int atom_dec_keep(int32_t* a) {
#if defined(PGC_NO_L2HINT) || defined(PGC_NO_ATOMHINT)
  return atomicAdd(a, -1);
#else
  int old;
  asm volatile("atom.relaxed.gpu.global.add.L2::cache_hint.s32 %0, [%1], %2, %3;"
               : "=r"(old)
               : "l"(a), "r"(-1), "l"(l2_keep_policy())
               : "memory");
  return old;
#endif
}
// plain int load / int and byte stores with the evict-last policy (the ADG
// per-vertex state, so the first UPDATE finds D and rs in L2)
__device__ __forceinline__ int ld_i32_keep(const int32_t* a) {
#ifdef PGC_NO_L2HINT
  return *a;
#else
  int v;
  asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(l2_keep_policy()));
  return v;
#endif
}
__device__ __forceinline__ void st_i32_keep(int32_t* a, int v) {
#ifdef PGC_NO_L2HINT
  *a = v;
#else
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(l2_keep_policy())
               : "memory");
#endif
}
__device__ __forceinline__ void st_u8_keep(uint8_t* a, int v) {
#ifdef PGC_NO_L2HINT
  *a = (uint8_t)v;
#else
  asm volatile("st.global.L2::cache_hint.b8 [%0], %1, %2;" ::"l"(a), "h"((unsigned short)v),
               "l"(l2_keep_policy())
               : "memory");
#endif
}
// read-only byte gather (rs is immutable during UPDATE), evict-last
__device__ __forceinline__ int ld_u8_keep(const uint8_t* a) {
#ifdef PGC_NO_L2HINT
  return __ldg(a);
#else
  unsigned short v;
  asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(a), "l"(l2_keep_policy()));
  return v;
#endif
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ int warp_max(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Block-wide stream compaction: every thread with `flag` appends `val` to
// out[] at a position reserved with ONE atomicAdd per block (order inside the
// list is arbitrary -- all consumers treat the lists as sets).  Must be called
// by all threads of the block; `sm` needs (blockDim/32 + 1) ints.
__device__ __forceinline__ void block_append(bool flag, int val, int32_t* out, int* counter,
                                             int* sm) {
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned b = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sm[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < nw; ++w) {
      int c = sm[w];
      sm[w] = tot;
      tot += c;
    }
    sm[nw] = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  if (flag) out[sm[nw] + sm[warp] + __popc(b & lanemask_lt())] = val;
  __syncthreads();
}

// block_append for 16-byte records (the UPDATE work lists).
__device__ __forceinline__ void block_append_rec(bool flag, int4 val, int4* out, int* counter,
                                                 int* sm) {
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned b = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sm[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < nw; ++w) {
      int c = sm[w];
      sm[w] = tot;
      tot += c;
    }
    sm[nw] = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  if (flag) __stcs(out + sm[nw] + sm[warp] + __popc(b & lanemask_lt()), val);  // read once
  __syncthreads();
}

// UPDATE work records (written by the select / classify kernels, one coalesced
// load per item in the UPDATE kernels):
//   light vertex: {v, deg, off_lo, off_hi}
//   edge chunk  : {v, len, start_lo, start_hi}, {base_lo, base_hi, 0, 0}
__device__ __forceinline__ int64_t lo_hi(int lo, int hi) {
  return (int64_t)(((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo);
}
__device__ __forceinline__ int4 light_rec(int v, int deg, int64_t o) {
  return make_int4(v, deg, (int)(uint32_t)o, (int)(o >> 32));
}

// Block-wide reservation: each thread asks for `cnt` slots; returns the
// thread's first slot, reserved with ONE atomicAdd per block.  All threads of
// the block must call it; `sm` needs (blockDim/32 + 1) ints.
__device__ __forceinline__ int block_reserve(int cnt, int* counter, int* sm) {
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= s) incl += y;
  }
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < nw; ++w) {
      int c = sm[w];
      sm[w] = tot;
      tot += c;
    }
    sm[nw] = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  const int base = sm[nw] + sm[warp] + incl - cnt;
  __syncthreads();
  return base;
}

template <typename T>
__device__ __forceinline__ T block_sum(T x, T* sm) {
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_sum(x);
  if (lane == 0) sm[warp] = x;
  __syncthreads();
  T t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nw; ++w) t += sm[w];
  __syncthreads();
  return t;  // valid in thread 0
}

// Grid of exactly one wave: SMs x resident blocks of `kernel` (cached per
// kernel and device).  Grid-stride kernels sized this way never run a second,
// serialised wave.
int occupancy_cached(int dev, const void* kernel, int block, size_t smem);  // capi.cu
template <typename K>
inline int wave_grid(const Ctx& c, K kernel, int block, size_t smem = 0) {
  return c.nsm * occupancy_cached(c.dev, (const void*)kernel, block, smem);
}

// ---- shared kernels (defined in adg.cu) -----------------------------------
__global__ void k_zero_i32(int32_t* p, int64_t len);
__global__ void k_zero_i32_dev(int32_t* p, const int* len, int extra);


}  // namespace pgc
