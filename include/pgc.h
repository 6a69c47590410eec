/*
 * pgc.h -- C ABI of the B200-native JP-ADG graph-coloring library.
 *
 * Method: Besta et al., "High-Performance Parallel Graph Coloring with Strong
 * Guarantees on Work, Depth, and Quality", SC'20 (arXiv 2008.11321);
 * /root/reference/PAPER.md.  This library implements the data-parallel hot
 * path of JP-ADG on one NVIDIA B200 (sm_100a):
 *
 *   ADG  (Algorithm 1): approximate degeneracy ordering.
 *        Round l removes every remaining vertex whose residual degree is at
 *        most (1+eps) times the remaining graph's average degree
 *        (PAPER.md:685), then decrements its neighbours' degrees (UPDATE,
 *        PAPER.md:692-696).  rho_ADG(v) = l.
 *   JP   (Algorithm 3) with the priority
 *        rho = <rho_ADG, rho_R>: a vertex is colored
 *        with the smallest color (>= 1) not used by any higher-priority
 *        neighbour (GetColor).
 *
 * Conventions shared by every entry point:
 *   - eps = eps_num / eps_den with eps_num >= 1, eps_den >= 1; the selection
 *     test is the exact integer form  den*D[v]*|U| <= (den+num)*sum_U D
 *     ("<=" per Alg. 1).  No floating point anywhere.
 *   - Rounds are 1-based.  A later round is a HIGHER priority
 *     (the dense core is colored first).  Inside a round the larger
 *     h(v) = splitmix64(seed ^ (uint64)v) wins (unsigned compare); h is a
 *     bijection, so the priority is a total order.
 *   - Colors are 1-based; num_colors = K = max color.
 *
 * Graph input (all entry points): an undirected simple graph in CSR,
 *   row_offsets : int64[n+1], row_offsets[0] = 0, nondecreasing, [n] = nnz
 *   col_indices : int32[nnz], each row strictly ascending, symmetric
 *                 (v in N(u) <=> u in N(v)), no self-loops.
 * These invariants are NOT checked on the hot path (pgc_check_graph checks
 * them in O(n+m)); results on an invalid graph are undefined.
 *
 * Memory ownership: the caller owns the graph, every output and the
 * workspace.  The library allocates nothing on the device, keeps no pointer
 * after a call returns, and has no global mutable state besides the
 * thread-local error string, statistics and tuning values.  Calls with
 * distinct workspaces on distinct streams are independent.
 *
 * Synchrony: work is enqueued on `cuda_stream` (a cudaStream_t, NULL = the
 * legacy default stream); each call blocks until its work has finished,
 * because T and K are returned in host memory.
 *
 * Errors: every entry point returns one of the PGC_* codes below; on a
 * nonzero return the contents of the outputs are unspecified and
 * pgc_last_error() describes the failure.  No C++ exception crosses the ABI.
 */
#ifndef PGC_H
#define PGC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGC_VERSION 3

enum pgc_status {
  PGC_OK = 0,          /* success                                                  */
  PGC_EINVAL = 1,      /* NULL pointer, n < 0, n >= 2^29, nnz < 0, nnz >= 2^40,
                          eps_num == 0 or eps_den == 0, bad round[] range           */
  PGC_EWORKSPACE = 2,  /* workspace too small or not 256-byte aligned              */
  PGC_ECUDA = 3,       /* a CUDA runtime error (message in pgc_last_error)         */
  PGC_EINTERNAL = 4    /* an internal invariant failed (a bug): e.g. an empty ADG
                          round, a round that broke Lemma 1's exact shrink
                          n_{l+1}(den+num) < n_l den, more
                          rounds than T0 = min{t : (den+num)^t >= n den^t}, an
                          inconsistent compaction count, or a JP stall         */
};

/* Graph in caller-owned DEVICE memory (see "Graph input" above). */
typedef struct pgc_graph {
  int64_t n;                   /* number of vertices, 0 <= n < 2^29 (the workspace
                                  layout indexes 2n + 65536 entries with int32)       */
  int64_t nnz;                 /* number of arcs = 2m = row_offsets[n], < 2^40        */
  const int64_t* row_offsets;  /* device, n+1 entries                                 */
  const int32_t* col_indices;  /* device, nnz entries                                 */
} pgc_graph;

/* Statistics of this thread's last successful call (pgc_last_stats). */
typedef struct pgc_stats {
  int32_t rounds;          /* T, number of ADG rounds (0 for pgc_jp_color)                */
  int32_t num_colors;      /* K (0 for pgc_adg_order)                                     */
  int64_t sum_active;      /* sum over rounds of |U_l| (Lemma 2 work term)  */
  int64_t cross_edges;     /* X: decrements applied to surviving vertices, over all rounds */
  int64_t pred_arcs;       /* sum_v |pred(v)|; equals m for a valid graph                 */
  int64_t core_vertices;   /* JP: length of the priority prefix colored by the cluster
                              "core" engine (0 = everything by the bulk dataflow)         */
  int32_t kernel_launches; /* CUDA kernels this call launched                             */
  int32_t host_syncs;      /* stream synchronisations this call performed                 */
  int32_t core_ctas;       /* JP: thread-block cluster size of the core engine (0 = none) */
  int32_t sim_col_passes;  /* DEC-ADG-ITR: SIM-COL passes over all partitions (else 0)    */
  int32_t jp_levels;       /* J = the number of vertices on a longest path of the JP DAG
                              G_rho (level[v] = 1 + max level over pred(v); Alg. 3's
                              depth term, Lemma 6 1192-1294).
                              Computed only with pgc_set_tuning("levels", 1) (an extra
                              dataflow pass after JP, off in timed runs; the one-kernel
                              small-graph path counts its levels for free), else 0.  */
  /* Device time per kernel group, from CUDA events on the call's stream; all -1
   * unless pgc_set_tuning("timing", 1).  Groups: ADG select (a2/a3), ADG UPDATE
   * with fused JP Part 1 (a4/a7), other ADG kernels (init, finalize), the
   * priority-order sort, the JP core (selection, list rewrite, cluster kernel),
   * the JP bulk dataflow (a8/a9), and the whole call. */
  float t_select_ms, t_update_ms, t_adg_other_ms, t_order_ms, t_core_ms, t_jp_ms, t_total_ms;
  int32_t small_path;      /* 1 if pgc_color_jp_adg ran as ONE persistent cooperative kernel
                              (2: as ONE thread-block cluster, state in DSMEM; core_ctas
                              then holds its size)
                              (small / low-degree graphs: nnz <= tuning "small_max_arcs"
                              and nnz <= "small_max_avg" * n; ADG rounds and JP levels
                              separated by grid barriers, JP frontier-driven with
                              count[] decrements, Alg. 3 l.1128-1133); same results.
                              Its device time is reported in t_select_ms.          */
} pgc_stats;

/* Bytes of device workspace the entry points below need for a graph with n
 * vertices and nnz arcs (the same size serves all three).  The workspace must
 * be 256-byte aligned.  Returns 0 for invalid sizes. */
size_t pgc_workspace_bytes(int64_t n, int64_t nnz);

/* ADG ordering only (Algorithm 1).
 *   round_out  : device int32[n], receives rho_ADG(v) in [1, T]
 *   num_rounds : host int32*, receives T (0 for n = 0)
 * ADG uses no randomness, so there is no seed. */
int pgc_adg_order(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, int32_t* round_out,
                  int32_t* num_rounds, void* workspace, size_t workspace_bytes,
                  void* cuda_stream);

/* How ADG's UPDATE applies the decrements ("Push vs. Pull").
 *   PGC_UPDATE_PUSH : iterate over R_l's arcs and decrement D[u] of every
 *                     surviving neighbour u (atomic RED per arc; Alg. 1 lines
 *                     692-696).  Each arc is scanned once over the whole run.
 *   PGC_UPDATE_PULL : iterate over the survivors U_{l+1} and subtract from D[v]
 *                     the number of v's neighbours in R_l (the CREW UPDATE,
 *                     PAPER.md:979-986): no concurrent writes per arc (a vertex
 *                     split over several warps adds one atomic per 512 arcs),
 *                     but every survivor rescans its whole adjacency each round.
 * Both give the identical round[] (the decrements are the same integers). */
enum pgc_update_mode { PGC_UPDATE_PUSH = 0, PGC_UPDATE_PULL = 1 };

/* pgc_adg_order with an explicit UPDATE style (pgc_adg_order = PGC_UPDATE_PUSH).
 * Arguments and errors as pgc_adg_order; an update_mode outside the enum is
 * PGC_EINVAL.  Stats: rounds, sum_active, cross_edges (identical for both
 * modes). */
int pgc_adg_order_mode(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, int update_mode,
                       int32_t* round_out, int32_t* num_rounds, void* workspace,
                       size_t workspace_bytes, void* cuda_stream);

/* JP coloring (Algorithm 3) for the priority
 * <round[v], splitmix64(seed ^ v)>, lexicographic.  round[] may be ANY int32
 * array whose value range (max - min) is below n + 65536, e.g. rho_ADG
 * (JP-ADG), a constant (JP-R) or the degree (JP-LF).
 *   round      : device int32[n], read only
 *   color_out  : device int32[n], receives colors in [1, K]
 *   num_colors : host int32*, receives K */
int pgc_jp_color(const pgc_graph* g, const int32_t* round, uint64_t seed, int32_t* color_out,
                 int32_t* num_colors, void* workspace, size_t workspace_bytes, void* cuda_stream);

/* JP-ADG, the whole hot path: ADG then JP with <rho_ADG, rho_R>.  JP Part 1
 * (pred counts / DAG) is fused into ADG's UPDATE.
 *   round_out, color_out : device int32[n]
 *   num_rounds, num_colors : host int32* */
int pgc_color_jp_adg(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, uint64_t seed,
                     int32_t* round_out, int32_t* color_out, int32_t* num_rounds,
                     int32_t* num_colors, void* workspace, size_t workspace_bytes,
                     void* cuda_stream);

/* ADG-M ordering only (the median variant of ADG; its
 * analysis: O(log n) rounds, a partial 4-approximate
 * degeneracy ordering).  Each round removes the vertices of U whose residual
 * degree is at most the median degree of U, limited to half of |U| (+1 if |U|
 * is odd).  Readings (Q19-Q21): U is ordered by (residual degree
 * ascending, id ascending) -- a stable integer sort of U; the median is the
 * degree of the ceil(|U|/2)-th vertex of that order; the cap keeps the first
 * ceil(|U|/2) vertices.  So |U_{l+1}| = floor(|U_l| / 2) and T = floor(log2 n)
 * + 1 exactly.  No eps, no seed.
 *   round_out  : device int32[n], receives rho_ADG-M(v) in [1, T]
 *   num_rounds : host int32*, receives T (0 for n = 0)
 * Same workspace, errors and ownership as pgc_adg_order. */
int pgc_adg_m_order(const pgc_graph* g, int32_t* round_out, int32_t* num_rounds, void* workspace,
                    size_t workspace_bytes, void* cuda_stream);

/* JP-ADG-M: ADG-M then JP with <rho_ADG-M, rho_R>
 * (rho_R(v) = splitmix64(seed ^ v) as in pgc_color_jp_adg); at most 4d + 1
 * colors.  JP Part 1 is fused into UPDATE as in pgc_color_jp_adg.
 *   round_out, color_out : device int32[n]
 *   num_rounds, num_colors : host int32* */
int pgc_color_jp_adg_m(const pgc_graph* g, uint64_t seed, int32_t* round_out, int32_t* color_out,
                       int32_t* num_rounds, int32_t* num_colors, void* workspace,
                       size_t workspace_bytes, void* cuda_stream);

/* JP-ADG-O: the ADG-O listing (explicit ordering of R,
 * 2231-2252) then JP with its total order rho_ADG-O.  The rounds are ADG's
 * (same eps rule); inside a round R is sorted by increasing residual degree
 * at selection, ties by increasing id (reading Q22), and rho(v) = its position
 * in the concatenated removal order.  JP gives the higher rho priority (no
 * random tie-break); JP Part 1 is fused into UPDATE (UPDATEandPRIORITIZE,
 * PAPER.md:2440-2452).
 *   round_out, color_out : device int32[n]
 *   num_rounds, num_colors : host int32*
 * PGC_EINVAL also if the sum over rounds of (max residual degree at selection
 * + 1) exceeds n + 65536 (the priority-order key range). */
int pgc_color_jp_adg_o(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, int32_t* round_out,
                       int32_t* color_out, int32_t* num_rounds, int32_t* num_colors,
                       void* workspace, size_t workspace_bytes, void* cuda_stream);

/* JP with the classic orderings the paper compares against,
 * each a first key plus the random tie-break rho_R(v) = splitmix64(seed ^ v):
 *   PGC_JP_R   rho = rho_R                      (JP-R, Jones-Plassmann)
 *   PGC_JP_FF  rho = <-v, rho_R>                (JP-FF: the natural vertex order)
 *   PGC_JP_LF  rho = <deg(v), rho_R>            (JP-LF: largest degree first)
 *   PGC_JP_LLF rho = <ceil(log2 deg(v)), rho_R> (JP-LLF: largest log-degree first)
 * (= pgc_jp_color with that first key, computed on the device.)
 *   color_out : device int32[n];  num_colors : host int32* */
enum pgc_jp_kind { PGC_JP_R = 0, PGC_JP_FF = 1, PGC_JP_LF = 2, PGC_JP_LLF = 3 };
int pgc_jp_baseline(const pgc_graph* g, int kind, uint64_t seed, int32_t* color_out,
                    int32_t* num_colors, void* workspace, size_t workspace_bytes, void* cuda_stream);

/* DEC-ADG-ITR: ADG's rounds as partitions R(T), ..., R(1),
 * colored in that order by SIM-COL with ITR's Part 1: each
 * uncolored vertex of the partition takes the smallest color no colored
 * neighbour uses; a vertex keeps it unless an uncolored same-partition
 * neighbour took the same color and has a larger splitmix64(seed ^ v) (the
 * conflict rule, reading Q23); repeat until the partition is colored.  At most
 * floor(2(1+eps)d) + 1 colors (the bound of JP-ADG).
 *   round_out, color_out : device int32[n]
 *   num_rounds, num_colors : host int32*;  pgc_last_stats().sim_col_passes */
int pgc_color_dec_adg_itr(const pgc_graph* g, uint32_t eps_num, uint32_t eps_den, uint64_t seed,
                          int32_t* round_out, int32_t* color_out, int32_t* num_rounds,
                          int32_t* num_colors, void* workspace, size_t workspace_bytes,
                          void* cuda_stream);

/* JP-ADG end to end from HOST memory: copies the CSR host->device on
 * `cuda_stream`, runs pgc_color_jp_adg, copies round[] and color[] back.
 * Host buffers should be pinned (cudaHostAlloc) for full copy bandwidth.
 *   h_row_offsets : host int64[n+1];  h_col_indices : host int32[nnz]
 *   h_round_out, h_color_out : host int32[n]
 *   workspace : DEVICE buffer of pgc_host_workspace_bytes(n, nnz) bytes */
size_t pgc_host_workspace_bytes(int64_t n, int64_t nnz);
int pgc_color_jp_adg_host(int64_t n, int64_t nnz, const int64_t* h_row_offsets,
                          const int32_t* h_col_indices, uint32_t eps_num, uint32_t eps_den,
                          uint64_t seed, int32_t* h_round_out, int32_t* h_color_out,
                          int32_t* num_rounds, int32_t* num_colors, void* workspace,
                          size_t workspace_bytes, void* cuda_stream);

/* O(n+m) validation of the CSR invariants on the device.  Returns PGC_OK or
 * PGC_EINVAL with the first offending vertex named in pgc_last_error(). */
int pgc_check_graph(const pgc_graph* g, void* workspace, size_t workspace_bytes,
                    void* cuda_stream);

/* Statistics of this thread's last successful call; PGC_EINVAL if out is NULL. */
int pgc_last_stats(pgc_stats* out);

/* Thread-local, NUL-terminated description of the last nonzero return. */
const char* pgc_last_error(void);

/* Thread-local tuning knobs (results never depend on them; tests sweep them to
 * prove it).  Keys and ranges:
 *   "timing" 0/1 (per-kernel-group CUDA events), "rounds_per_sync" >= 1,
 *   "heavy_degree" >= 128 (ADG UPDATE edge-chunks rows longer than this),
 *   "chunk_arcs" >= 256, "block_threads" 64..1024 (multiple of 32),
 *   "jp_heavy_warps" 1..4 (warps per 8-warp bulk JP block serving vertices with
 *   more than 62 preds), "jp_heavy_batch" 1..64 (heavy tickets per atomic),
 *   "jp_heavy_sleep_max" / "jp_light_sleep_max" ns >= 0
 *   (backoff caps of waiting bulk JP warps), "jp_watchdog_ms"
 *   (a stalled JP kernel returns PGC_EINTERNAL after this long; default 20000),
 *   "core_max" 0..65535 (JP core size cap; 0 disables the core engine),
 *   "core_min_avg" (min mean |pred| of the core prefix), "core_min_n",
 *   "core_ctas" 0..16 (cluster size; 0 = automatic), "core_spin_ns" (backoff cap
 *   of a core warp several preds away from ready), "core_arc_cap",
 *   "core_arcs_per_cta", "itr_blocks_per_sm" 0..64 (DEC-ADG-ITR pass kernel;
 *   0 = occupancy), "jp_split_overlap" 0/1 (JP: the bulk's work-list split runs
 *   on a second stream while the core kernel, one cluster of <= 16 SMs, runs;
 *   default 1), "update_atom" 0/1 (ADG round 1 classifies each arc by the old
 *   value of ONE atomic decrement instead of a state gather plus a RED;
 *   default 1), "fuse_init" 0/1 (ADG's first selection also initialises the
 *   per-vertex state; default 1), "top_list" 0/1 (JP-ADG: ADG keeps the top
 *   rounds' vertex list so the split order's top part skips a pass over n;
 *   default 1), "filter_ratio", "core_tail_ns", "core_pass_ns", "core_near",
 *   "core_tier2" 0..65535 (JP core: when the first cluster pass is capped at
 *   core_max, a second pass over the next <= core_tier2 positions; 0 = off),
 *   "small_max_arcs" (pgc_color_jp_adg runs as one persistent kernel when
 *   nnz <= this and nnz <= "small_max_avg" * n; 0 disables; defaults 2^24, 20),
 *   "small_blocks_per_sm" 0..64 (that kernel's grid; 0 = occupancy),
 *   "tiny_max_n" / "tiny_max_arcs" (that path runs on ONE thread-block cluster
 *   with the per-vertex state in distributed shared memory when n and nnz are
 *   at most these and the state fits; tiny_max_n = 0 disables; 2^17, 2^22),
 *   "tiny_dataflow" 0/1 (that kernel's JP as a barrier-free dataflow, a thread
 *   per own vertex; 0: frontier levels with cluster barriers; default 1).
 * Returns PGC_EINVAL for an unknown key or out-of-range value. */
int pgc_set_tuning(const char* key, int64_t value);

/* PGC_VERSION of the loaded library. */
int pgc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PGC_H */
