// small.cu -- JP-ADG for small and low-degree graphs in ONE persistent
// cooperative kernel (the latency path).
//
// The multi-kernel path (adg.cu + jp.cu) launches ~4 kernels per ADG round,
// syncs the host every 8 rounds, and spends ~10 launches and 2 host syncs on
// the priority order and the core/bulk split.  On graphs whose whole step is a
// few hundred microseconds of work (ER 16K: 0.26 M arcs, the 2048^2 grid:
// 12 M arcs, J = 16) those launches ARE the step.  Here the whole method runs
// in one launch, phases separated by grid barriers:
//
//   ADG (Algorithm 1), per round l -- 2 barriers:
//     select   Dmax_l = floor((den+num) S_l / (den |U_l|)) (exact, 128-bit,
//              readings Q1/Q2); R_l = {v in U_l : D[v] <= Dmax_l} (l.685),
//              round[v] = l (688-689); R_l and U_{l+1} = U_l \ R_l (687)
//              compacted with one atomic per warp; round 1 also initialises
//              D[v] = deg(v), color[v] = 0 (a1, l.676-677).
//     update   for v in R_l, u in N(v): u alive (round[u] == 0): D[u] -= 1
//              (l.692-696), cut += 1.  JP Part 1 fused (PAPER.md:2259-2271,
//              Alg. 3 l.1116-1121): count[v] = |pred(v)| = #alive neighbours
//              (they get a later round) + #same-round neighbours u with
//              h(u) > h(v) (Q8/Q10); count[v] == 0 puts v in the first
//              frontier.  Warp-flattened over the arcs of 32 vertices.
//     then every thread reads the round's block sums and carries
//     S_{l+1} = S_l - sum_{R_l} D - cut_l, |U_{l+1}| (degree-sum caching,
//     PAPER.md:2353-2365; Q5), and checks Lemma 1's per-round shrink exactly.
//   JP (Algorithm 3) frontier by frontier -- 1 barrier
//   per level, J levels (J = the JP DAG depth, reported with the levels knob):
//     for v in the frontier: color[v] = GetColor = the smallest color no pred
//     uses (l.1135-1138; 64-color bit-mask windows, OR-ed per owner lane in
//     shared memory); then for every succ u (lower priority): count[u] -= 1,
//     the vertex that takes it to 0 appends u to the next frontier (the Join
//     of l.1128-1133).  The next frontier is colored after the barrier, so
//     every pred color it reads is final.
//
// Results are the same integers as the multi-kernel path (the same Alg. 1 and
// the same priority); the choice is a host heuristic on (n, nnz) with a knob
// (pgc_set_tuning "small_max_arcs", "small_max_avg"; 0 disables the path).
// Data that other blocks wrote in an earlier phase is read with ld.cg (the L1
// is not coherent inside one kernel).
#include <cooperative_groups.h>

#include "pgc_internal.cuh"

namespace pgc {

namespace cg = cooperative_groups;

constexpr int kSmallBlock = 512;
constexpr int kSmallWarps = kSmallBlock / 32;
constexpr int kSmallUnroll = 4;  // flattened arc steps per warp iteration (loads in flight)
constexpr int kSelK = 4;         // selection: vertices per lane per step
// counter ring: 4 slots (round or level mod 4) x fields, each field on its own
// 128-byte line (16 x u64): the fields are hit by one atomic per warp
constexpr int kSmallSlots = 4;
enum { kSfUout = 0, kSfR = 1, kSfSumD = 2, kSfCut = 3, kSfPreds = 4, kSfF = 5, kSmallFields = 6 };
constexpr int kSmallLine = 16;
constexpr size_t kSmallCtrBytes = sizeof(unsigned long long) * kSmallSlots * kSmallFields * kSmallLine;

struct SmallArgs {
  int64_t n, nnz;
  const int64_t* off;
  const int32_t* col;
  uint32_t num, den;
  uint64_t seed;
  int32_t* round;
  int32_t* color;
  int32_t* D;
  int32_t* cnt;       // count[v] = |pred(v)|, then decremented by JP's Join
  int32_t* U[2];      // U_l lists (U_1 = every vertex, implicit)
  int32_t* R;         // R_l
  int32_t* F[2];      // JP frontiers
  unsigned long long* ctr;  // [kSmallSlots][kSmallFields][kSmallLine]
  State* st;
  long long* per_round;
};

__device__ __forceinline__ unsigned long long* sctr(unsigned long long* c, int slot, int f) {
  return c + ((slot & (kSmallSlots - 1)) * kSmallFields + f) * kSmallLine;
}
__device__ __forceinline__ unsigned long long ld_ctr(const unsigned long long* p) {
  return __ldcg(p);
}

// Per-warp append queues in shared memory: a list append is staged in the
// warp's queue and the queue goes out with ONE global atomic per kSmallQ
// entries (per-warp atomics on one list counter made that counter's L2 slice
// the bottleneck of a phase: ~1 atomic per 32 vertices from every warp).
// `fill` is warp-uniform; all 32 lanes call.
constexpr int kSmallQ = 256;
__device__ __forceinline__ void wq_flush(int32_t* q, int& fill, int32_t* out,
                                         unsigned long long* counter, int64_t cap) {
  __syncwarp();
  if (fill) {
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(counter, (unsigned long long)fill);
    base = __shfl_sync(0xffffffffu, base, 0);
    PGC_DCHECK(base + fill <= (unsigned long long)cap, base, fill);
    for (int i = lane_id(); i < fill; i += 32) out[base + i] = q[i];
  }
  fill = 0;
  __syncwarp();
}
__device__ __forceinline__ void wq_push(int32_t* q, int& fill, bool flag, int val, int32_t* out,
                                        unsigned long long* counter, int64_t cap) {
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  if (!b) return;
  if (fill + __popc(b) > kSmallQ) wq_flush(q, fill, out, counter, cap);
  if (flag) q[fill + __popc(b & lanemask_lt())] = val;
  fill += __popc(b);
}

// L2 policy for the grid kernel: the per-vertex state it gathers at random
// (round, color, D, count) is kept (evict-last) and the arrays it streams
// through (col, the lists) go first -- on the 2048^2 grid the state plus the
// CSR exceed the 126 MB L2 (ncu: 1.4 GB DRAM per step against 0.59 GB of
// algorithmic bytes before the hints).  Loads bypass L1 (.cg): other blocks
// wrote the state in earlier phases.
__device__ __forceinline__ int ldcg_keep(const int32_t* a) {
#ifdef PGC_NO_L2HINT
  return __ldcg(a);
#else
  int v;
  asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(l2_keep_policy()));
  return v;
#endif
}
__device__ __forceinline__ int atom_sub_keep(int32_t* a) {
#ifdef PGC_NO_L2HINT
  return atomicSub(a, 1);
#else
  int v;
  asm volatile("atom.global.add.L2::cache_hint.s32 %0, [%1], %2, %3;"
               : "=r"(v)
               : "l"(a), "r"(-1), "l"(l2_keep_policy())
               : "memory");
  return v;
#endif
}

// Owner lane of flattened arc j: the largest lane s with start_s <= j (lanes
// with no arcs share the next lane's start and are never picked for j < total).
__device__ __forceinline__ int owner_of(int start, int j) {
  int s = 0;
#pragma unroll
  for (int b = 16; b; b >>= 1) {
    const int t = s + b;
    const int st_t = __shfl_sync(0xffffffffu, start, t);
    if (st_t <= j) s = t;
  }
  return s;
}

// Vertices per warp for a list of `cnt` vertices (a power of two in 1..32):
// few enough that every warp of the grid gets work, so a phase costs a few
// dependent L2 round trips rather than a long per-warp arc loop.
__device__ __forceinline__ int verts_per_warp(long long cnt, long long nwarps) {
  const long long per = (cnt + nwarps - 1) / nwarps;
  int v = 1;
  while (v < 32 && v < per) v <<= 1;
  return v;
}

// Dmax = floor((den+num) S / (den |U|)) exactly (readings Q1/Q2), clamped to
// INT32_MAX; 64-bit division when the numerator fits (the software 128-bit
// division costs microseconds on a latency-bound phase).
__device__ __forceinline__ long long dmax_of(uint32_t num, uint32_t den, unsigned long long S,
                                             long long nU) {
  const unsigned long long dn = (unsigned long long)den + num;
  const unsigned long long denom = (unsigned long long)den * (unsigned long long)nU;
  unsigned long long q;
  if (S <= 0xffffffffffffffffull / dn) {
    q = (S * dn) / denom;
  } else {
    const unsigned __int128 q128 = ((unsigned __int128)dn * S) / denom;
    q = q128 > (unsigned __int128)0x7fffffff ? 0x7fffffffull : (unsigned long long)q128;
  }
  return q > 0x7fffffffull ? 0x7fffffffLL : (long long)q;
}

// Higher JP priority: <round, h> lexicographic (Q8, Q10; h is a bijection).
__device__ __forceinline__ bool prio_gt(int ra, uint64_t ha, int rb, uint64_t hb) {
  return ra > rb || (ra == rb && ha > hb);
}

#ifdef PGC_PROBE
// phase timeline (probe builds only): block 0 thread 0 stamps %globaltimer
// after every grid barrier and prints the phase lengths at the end
#define SMALL_STAMP()                                                   \
  do {                                                                  \
    if (tid == 0 && nstamp < 512) stamps[nstamp++] = globaltimer();     \
  } while (0)
#else
#define SMALL_STAMP() \
  do {                \
  } while (0)
#endif

__global__ void __launch_bounds__(kSmallBlock) k_small_jp_adg(SmallArgs a) {
  cg::grid_group grid = cg::this_grid();
#ifdef PGC_PROBE
  unsigned long long stamps[512];
  int nstamp = 0;
#endif
  __shared__ int s_acc[kSmallWarps][32];
  __shared__ unsigned s_mask[kSmallWarps][32][2];  // GetColor windows (two 32-bit halves: native smem atomics)
  __shared__ unsigned long long s_red[kSmallWarps];
  __shared__ int32_t s_q[kSmallWarps][2][kSmallQ];  // per-warp append queues
  int32_t* q0 = s_q[threadIdx.x >> 5][0];
  int32_t* q1 = s_q[threadIdx.x >> 5][1];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const long long tid = (long long)blockIdx.x * kSmallBlock + threadIdx.x;
  const long long nth = (long long)gridDim.x * kSmallBlock;
  const long long gwarp = tid >> 5, nwarps = nth >> 5;
  const int64_t n = a.n;
  s_acc[warp][lane] = 0;
  s_mask[warp][lane][0] = s_mask[warp][lane][1] = 0;
  for (long long i = tid; i < kSmallSlots * kSmallFields * kSmallLine; i += nth) a.ctr[i] = 0;
  if (tid == 0) a.st->K = 0;
  grid.sync();
  SMALL_STAMP();

  // ---------------------------------------------------------------- ADG
  unsigned long long S = (unsigned long long)a.nnz;  // S_1 = sum of degrees
  long long nU = n, sum_active = 0;
  unsigned long long cross = 0, preds_total = 0;
  int l = 0, err = 0;
  unsigned long long* f_first = sctr(a.ctr, 1, kSfF);  // JP level 1's frontier count
  while (nU > 0) {
    ++l;
    // the round fields of round l+2's slot (last read in round l-2; the
    // frontier field is JP's, reset per level)
    if (tid < kSfF) *sctr(a.ctr, l + 2, (int)tid) = 0;
    // select (a2/a3): exact threshold
    const long long dmax = dmax_of(a.num, a.den, S, nU);
    const int32_t* Uin = l == 1 ? nullptr : a.U[l & 1];
    int32_t* Uout = a.U[(l + 1) & 1];
    unsigned long long sumD = 0;
    // kSelK vertices per lane per step, loads first (the step is latency-bound)
    int fr = 0, fu = 0;
    for (long long base = gwarp * 32 * kSelK; base < nU; base += nwarps * 32 * kSelK) {
      int v[kSelK], d[kSelK];
      bool valid[kSelK];
#pragma unroll
      for (int k = 0; k < kSelK; ++k) {
        const long long i = base + 32 * k + lane;
        valid[k] = i < nU;
        v[k] = valid[k] ? (Uin ? __ldcg(Uin + i) : (int)i) : 0;
        PGC_DCHECK(!valid[k] || (v[k] >= 0 && v[k] < n), v[k], i);
      }
      if (l == 1) {
        int64_t o0[kSelK], o1[kSelK];
#pragma unroll
        for (int k = 0; k < kSelK; ++k) {
          o0[k] = valid[k] ? a.off[v[k]] : 0;
          o1[k] = valid[k] ? a.off[v[k] + 1] : 0;
        }
#pragma unroll
        for (int k = 0; k < kSelK; ++k) {
          d[k] = (int)(o1[k] - o0[k]);
          if (valid[k]) {
            st_i32_keep(a.D + v[k], d[k]);
            st_i32_keep(a.color + v[k], 0);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < kSelK; ++k) d[k] = valid[k] ? ldcg_keep(a.D + v[k]) : 0;
      }
#pragma unroll
      for (int k = 0; k < kSelK; ++k) {
        const bool sel = valid[k] && d[k] <= dmax;
        if (valid[k] && (sel || l == 1)) st_i32_keep(a.round + v[k], sel ? l : 0);
        if (sel) sumD += (unsigned long long)d[k];
        wq_push(q0, fr, sel, v[k], a.R, sctr(a.ctr, l, kSfR), n);
        wq_push(q1, fu, valid[k] && !sel, v[k], Uout, sctr(a.ctr, l, kSfUout), n);
      }
    }
    wq_flush(q0, fr, a.R, sctr(a.ctr, l, kSfR), n);
    wq_flush(q1, fu, Uout, sctr(a.ctr, l, kSfUout), n);
    sumD = warp_sum(sumD);
    if (lane == 0 && sumD) atomicAdd(sctr(a.ctr, l, kSfSumD), sumD);
    grid.sync();
    SMALL_STAMP();
    // update (a4) with fused JP Part 1 (a7)
    const long long nR = (long long)ld_ctr(sctr(a.ctr, l, kSfR));
    unsigned long long cut = 0, preds = 0;
    const int vpw = verts_per_warp(nR, nwarps);
    int ff = 0;
    for (long long base = gwarp * vpw; base < nR; base += nwarps * vpw) {
      const long long i = base + lane;
      const bool valid = lane < vpw && i < nR;
      const int v = valid ? __ldcg(a.R + i) : 0;
      PGC_DCHECK(!valid || (v >= 0 && v < n), v, i);
      const int64_t o = valid ? a.off[v] : 0;
      const int deg = valid ? (int)(a.off[v + 1] - o) : 0;
      const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
      int incl = deg;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
      }
      const int start = incl - deg;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int j0 = 0; j0 < total; j0 += 32 * kSmallUnroll) {
        int own[kSmallUnroll], u[kSmallUnroll], ru[kSmallUnroll];
#pragma unroll
        for (int k = 0; k < kSmallUnroll; ++k) {
          const int j = j0 + 32 * k + lane;
          own[k] = owner_of(start, j);
          const int64_t os = __shfl_sync(0xffffffffu, o, own[k]);
          const int ss = __shfl_sync(0xffffffffu, start, own[k]);
          PGC_DCHECK(j >= total || (os + (j - ss) >= 0 && os + (j - ss) < a.nnz), os + (j - ss), j);
          u[k] = j < total ? __ldcs(a.col + os + (j - ss)) : -1;
          PGC_DCHECK(u[k] < n, u[k], j);
        }
#pragma unroll
        for (int k = 0; k < kSmallUnroll; ++k) ru[k] = u[k] >= 0 ? ldcg_keep(a.round + u[k]) : -1;
#pragma unroll
        for (int k = 0; k < kSmallUnroll; ++k) {
          const uint64_t hs = __shfl_sync(0xffffffffu, hv, own[k]);
          bool pred = false;
          PGC_DCHECK(ru[k] <= l, u[k], ru[k] * 1000000ll + l);  // no round from the future
          if (ru[k] == 0) {  // alive: D[u] -= 1, u is a pred of v (later round)
            red_dec_keep(a.D + u[k]);
            ++cut;
            pred = true;
          } else if (ru[k] == l) {
            pred = prio_hash(a.seed, (uint32_t)u[k]) > hs;
          }
          // one shared add per (owner, step): owners hold contiguous lanes (an
          // atomic: the leaders of one owner in consecutive steps are different lanes)
          const unsigned same = __match_any_sync(0xffffffffu, own[k]);
          const int c = __popc(__ballot_sync(0xffffffffu, pred) & same);
          if (c && lane == __ffs(same) - 1) atomicAdd(&s_acc[warp][own[k]], c);
        }
      }
      __syncwarp();
      const int p = s_acc[warp][lane];
      s_acc[warp][lane] = 0;
      if (valid) {
        st_i32_keep(a.cnt + v, p);
        preds += (unsigned long long)p;
      }
      wq_push(q0, ff, valid && p == 0, v, a.F[1], f_first, n);
      __syncwarp();
    }
    wq_flush(q0, ff, a.F[1], f_first, n);
    cut = warp_sum(cut);
    preds = warp_sum(preds);
    if (lane == 0) {
      if (cut) atomicAdd(sctr(a.ctr, l, kSfCut), cut);
      if (preds) atomicAdd(sctr(a.ctr, l, kSfPreds), preds);
    }
    grid.sync();
    SMALL_STAMP();
    // finalize (every thread, same values): S_{l+1}, |U_{l+1}|, Lemma 1
    const long long nU1 = (long long)ld_ctr(sctr(a.ctr, l, kSfUout));
    const unsigned long long sumDR = ld_ctr(sctr(a.ctr, l, kSfSumD));
    const unsigned long long cut_l = ld_ctr(sctr(a.ctr, l, kSfCut));
    preds_total += ld_ctr(sctr(a.ctr, l, kSfPreds));
    if (tid == 0 && l - 1 < kMaxRoundStats) {
      a.per_round[3 * (l - 1) + 0] = nU;
      a.per_round[3 * (l - 1) + 1] = (long long)S;
      a.per_round[3 * (l - 1) + 2] = nR;
    }
    sum_active += nU;
    cross += cut_l;
    if (nR == 0) err = 1;
    if (nU1 != nU - nR) err = 2;
    if (!((unsigned __int128)nU1 * ((unsigned long long)a.den + a.num) <
          (unsigned __int128)nU * a.den))
      err = 7;  // Lemma 1
    S = S - sumDR - cut_l;
    nU = nU1;
    if (err) break;
  }

  // ---------------------------------------------------------------- JP
  int J = 0, kmax = 0;
#ifdef PGC_CHECKED
  // count[v] == |pred(v)| recomputed from the final rounds, vertex by vertex
  for (long long v = tid; v < n && !err; v += nth) {  // (err is uniform)
    int p = 0;
    const int rv = __ldcg(a.round + v);
    const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
    for (int64_t e = a.off[v]; e < a.off[v + 1]; ++e) {
      const int u = a.col[e];
      p += prio_gt(__ldcg(a.round + u), prio_hash(a.seed, (uint32_t)u), rv, hv);
    }
    if (p != __ldcg(a.cnt + v)) {
      printf("count mismatch v=%lld round=%d deg=%lld cnt=%d p=%d\n", v, rv,
             (long long)(a.off[v + 1] - a.off[v]), __ldcg(a.cnt + v), p);
      __trap();
    }
  }
  grid.sync();  // JP's Join decrements count[]: the check must finish first
  SMALL_STAMP();
#endif
  if (!err) {
    long long nF = (long long)ld_ctr(f_first);
    for (int j = 1; nF > 0; ++j) {
      J = j;
      if (tid < 1) *sctr(a.ctr, j + 2, kSfF) = 0;  // frontier counter of level j+2 (last read at level j-2)
      const int32_t* Fin = a.F[j & 1];
      int32_t* Fout = a.F[(j + 1) & 1];
      unsigned long long* fnext = sctr(a.ctr, j + 1, kSfF);
      const int vpw = verts_per_warp(nF, nwarps);
      int ff = 0;
      for (long long base = gwarp * vpw; base < nF; base += nwarps * vpw) {
        const long long i = base + lane;
        const bool valid = lane < vpw && i < nF;
        const int v = valid ? __ldcg(Fin + i) : 0;
        PGC_DCHECK(!valid || (v >= 0 && v < n), v, i);
        PGC_DCHECK(!valid || __ldcg(a.cnt + v) == 0, v, __ldcg(a.cnt + v));
        const int64_t o = valid ? a.off[v] : 0;
        const int deg = valid ? (int)(a.off[v + 1] - o) : 0;
        const int rv = valid ? ldcg_keep(a.round + v) : 0;
        const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
        int incl = deg;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, s);
          if (lane >= s) incl += y;
        }
        const int start = incl - deg;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        // One pass over the arcs does both halves of the level: a pred's color
        // goes into the owner's GetColor window, a succ's
        // count is decremented (the Join, l.1128-1133) -- v's color is read by
        // its succs only after the barrier.  Level 1 holds exactly the
        // vertices with no pred: color 1, nothing to mark.  A vertex whose
        // first 64-color window is full rescans its preds for the next window.
        bool need = valid && j > 1;
        int mycolor = valid ? 1 : 0;
        for (int wbase = 0, first = 1; first || __ballot_sync(0xffffffffu, need); wbase += 64, first = 0) {
          for (int j0 = 0; j0 < total; j0 += 32 * kSmallUnroll) {
            int own[kSmallUnroll], u[kSmallUnroll], ru[kSmallUnroll], on[kSmallUnroll];
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              const int jj = j0 + 32 * k + lane;
              own[k] = owner_of(start, jj);
              const int64_t os = __shfl_sync(0xffffffffu, o, own[k]);
              const int ss = __shfl_sync(0xffffffffu, start, own[k]);
              on[k] = __shfl_sync(0xffffffffu, (int)need, own[k]);  // every lane shuffles
              const bool scan = jj < total && (first || on[k]);
              PGC_DCHECK(!scan || os + (jj - ss) < a.nnz, os + (jj - ss), jj);
              u[k] = scan ? __ldcs(a.col + os + (jj - ss)) : -1;
              PGC_DCHECK(u[k] < n, u[k], jj);
            }
            // the neighbour's color is loaded beside its round (one dependent
            // L2 trip less; used only if it turns out to be a pred)
            int cu[kSmallUnroll];
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              ru[k] = u[k] >= 0 ? ldcg_keep(a.round + u[k]) : -1;
              cu[k] = u[k] >= 0 && on[k] ? ldcg_keep(a.color + u[k]) : 0;
            }
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              const int rs = __shfl_sync(0xffffffffu, rv, own[k]);
              const uint64_t hs = __shfl_sync(0xffffffffu, hv, own[k]);
              bool freed = false;
              if (u[k] >= 0) {
                if (prio_gt(ru[k], prio_hash(a.seed, (uint32_t)u[k]), rs, hs)) {
                  if (on[k]) {  // pred: colored in an earlier level
                    const int cb = cu[k] - 1 - wbase;
                    PGC_DCHECK(cb + wbase >= 0, u[k], cb + wbase);
                    if (cb >= 0 && cb < 64) atomicOr(&s_mask[warp][own[k]][cb >> 5], 1u << (cb & 31));
                  }
                } else if (first) {  // succ: count[u] -= 1; the last pred frees u
                  const int old = atom_sub_keep(a.cnt + u[k]);
                  PGC_DCHECK(old >= 1, u[k], old);
                  freed = old == 1;
                }
              }
              wq_push(q0, ff, freed, u[k], Fout, fnext, n);
            }
          }
          __syncwarp();
          const unsigned long long m =
              ((unsigned long long)s_mask[warp][lane][1] << 32) | s_mask[warp][lane][0];
          s_mask[warp][lane][0] = s_mask[warp][lane][1] = 0;
          if (need && ~m) {
            mycolor = wbase + __ffsll((long long)~m);
            need = false;
          }
          __syncwarp();
        }
        if (valid) {
          st_i32_keep(a.color + v, mycolor);
          kmax = max(kmax, mycolor);
        }
      }
      wq_flush(q0, ff, Fout, fnext, n);
      grid.sync();
      SMALL_STAMP();
      nF = (long long)ld_ctr(fnext);
    }
  }
  kmax = warp_max(kmax);
  if (lane == 0) s_red[warp] = (unsigned long long)kmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    int bm = 0;
    for (int w = 0; w < kSmallWarps; ++w) bm = max(bm, (int)s_red[w]);
    if (bm) atomicMax(&a.st->K, bm);
  }
#ifdef PGC_PROBE
  if (tid == 0) {
    printf("small phases (us):");
    for (int k = 1; k < nstamp; ++k) printf(" %.1f", (stamps[k] - stamps[k - 1]) * 1e-3);
    printf("\ntotal %.1f us, %d phases, grid %d\n", (stamps[nstamp - 1] - stamps[0]) * 1e-3, nstamp,
           (int)gridDim.x);
  }
#endif
  if (tid == 0) {
    State* st = a.st;
    st->T = l;
    st->rmax = l;
    st->sum_active = sum_active;
    st->cross = cross;
    st->pred_arcs = preds_total;
    st->jp_levels = J;
    st->err = err;
    st->done = 1;
    st->nU = nU;
    st->S = S;
  }
}


// ============================================================ tiny graphs
// The same method on ONE thread-block cluster (<= 16 CTAs x 1024 threads) with
// every per-vertex array in distributed shared memory: vertex v lives in CTA
// v mod C at index v / C (D, round, count, color, the U/R lists and the JP
// frontiers).  A phase then costs a cluster barrier (hardware, well under a
// microsecond) and DSMEM / L1 accesses instead of a grid barrier and L2 round
// trips; the CSR is read through the read-only path (each CTA's rows stay in
// its L1 across the phases).  Rounds and levels run as in k_small_jp_adg:
// select (own vertices, local lists) | cluster barrier | UPDATE + JP Part 1
// (decrements into the owners' D by DSMEM atomics) | cluster barrier; JP
// levels push a freed succ into its OWNER's next frontier (one DSMEM atomic
// per owner group of a warp).  Global sums (|U|, S terms) are per-CTA
// partials in a 2-slot ring read by warp 0 of every CTA after the barrier.
constexpr int kTinyBlock = 1024;
constexpr int kTinyWarps = kTinyBlock / 32;
static_assert(kTinyWarps == 32, "block sums: one lane of warp 0 per warp");
constexpr int kTinyMaxC = 16;
constexpr int kTinyPer = 8;     // dataflow JP: own vertices per thread (nloc <= 8 x 1024)
constexpr int kTinyArrays = 9;  // D, rnd, cnt, clr, U0, U1, R, F0, F1 (+ row starts, rows)
enum { kTpUout = 0, kTpR = 1, kTpSumD = 2, kTpCut = 3, kTpPreds = 4, kTpFields = 5 };

struct TinyArgs {
  int64_t n, nnz;
  const int64_t* off;
  const int32_t* col;
  uint32_t num, den;
  uint64_t seed;
  int32_t* round;
  int32_t* color;
  State* st;
  long long* per_round;
  int nloc;     // per-CTA capacity of every array (>= ceil(n / C))
  int cshift;   // C = 1 << cshift
  long long adj_cap;  // per-CTA capacity of the copied rows (ints)
  int dataflow;       // JP as a barrier-free dataflow (thread per own vertex), else by levels
  int levels;         // compute J (the levels knob)
  unsigned long long watchdog_ns;
};

__global__ void __launch_bounds__(kTinyBlock, 1) k_tiny_jp_adg(TinyArgs a) {
  cg::cluster_group cl = cg::this_cluster();
#ifdef PGC_PROBE
  unsigned long long stamps[512];
  int nstamp = 0;
  const long long tid = (long long)cl.block_rank() * kTinyBlock + threadIdx.x;
#endif
  extern __shared__ __align__(16) int32_t t_dyn[];
  __shared__ unsigned long long s_part[2][kTpFields];  // this CTA's partial sums (ring: round parity)
  __shared__ unsigned long long s_tot[kTpFields];
  __shared__ int s_nR, s_nUo;
  __shared__ int s_fcnt[3];  // frontier lengths (ring: level mod 3); other CTAs push into them
  __shared__ int s_acc[kTinyWarps][32];
  __shared__ unsigned s_mask[kTinyWarps][32][2];
  __shared__ unsigned long long s_wsum[kTinyWarps][2];
  const int C = 1 << a.cshift, cs = a.cshift, me = (int)cl.block_rank();
  const int nloc = a.nloc;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  int32_t* D = t_dyn;
  int32_t* rnd = D + nloc;
  int32_t* cnt = rnd + nloc;
  int32_t* clr = cnt + nloc;
  int32_t* Ul[2] = {clr + nloc, clr + 2 * nloc};
  int32_t* Rl = clr + 3 * nloc;
  int32_t* Fb[2] = {clr + 4 * nloc, clr + 5 * nloc};
  // the own rows of the CSR, copied once: cluster.sync invalidates the L1, so
  // a row read from global memory would cost an L2 round trip in every phase
  int32_t* loff = clr + 6 * nloc;  // [nloc + 1] local row starts into ladj
  int32_t* ladj = loff + nloc + 1; // [a.adj_cap]
  // an array element of vertex u in its owner's shared memory (generic address)
  auto at = [&](int32_t* local_array, int u) -> int32_t* {
    return cl.map_shared_rank(local_array, u & (C - 1)) + (u >> cs);
  };
  const int nown = me < n ? (int)((n - me + C - 1) >> cs) : 0;  // own vertices me, me + C, ...
  if (threadIdx.x == 0) {
    s_fcnt[0] = s_fcnt[1] = s_fcnt[2] = 0;
    s_nR = s_nUo = 0;
    if (me == 0) {
      a.st->K = 0;
      a.st->jp_levels = 0;
    }
  }
  s_acc[warp][lane] = 0;
  s_mask[warp][lane][0] = s_mask[warp][lane][1] = 0;
  // local row starts: a block scan of the own degrees (thread t: a contiguous chunk)
  {
    const int per = (nown + kTinyBlock - 1) / kTinyBlock;
    const int b0 = min(nown, (int)threadIdx.x * per), b1 = min(nown, b0 + per);
    long long sum = 0;
    for (int i = b0; i < b1; ++i) {
      const int v = (i << cs) + me;
      sum += __ldg(a.off + v + 1) - __ldg(a.off + v);
    }
    long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __shared__ long long s_w[kTinyWarps + 1];
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const long long w = s_w[lane];
      long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_w[lane] = wi - w;
      if (lane == 31) s_w[kTinyWarps] = wi;
    }
    __syncthreads();
    const long long tot = s_w[kTinyWarps];
    long long run = s_w[warp] + incl - sum;
    if (tot <= a.adj_cap) {
      for (int i = b0; i < b1; ++i) {
        const int v = (i << cs) + me;
        loff[i] = (int)run;
        const int d = (int)(__ldg(a.off + v + 1) - __ldg(a.off + v));
        D[i] = d;
        clr[i] = 0;
        run += d;
      }
      if (threadIdx.x == 0) loff[nown] = (int)tot;
    }
    if (threadIdx.x == 0) s_part[0][0] = tot > a.adj_cap ? 1ull : 0ull;  // does not fit
    __syncthreads();
    // copy the rows: a warp per row, coalesced
    if (tot <= a.adj_cap)
      for (int i = warp; i < nown; i += kTinyWarps) {
        const int v = (i << cs) + me;
        const int64_t o = __ldg(a.off + v);
        const int d = loff[i + 1] - loff[i];
        for (int k = lane; k < d; k += 32) ladj[loff[i] + k] = __ldg(a.col + o + k);
      }
  }
  cl.sync();
  SMALL_STAMP();
  // every CTA's rows must fit: otherwise all leave, the host runs the grid kernel
  {
    int bad = 0;
    if (warp == 0) bad = __any_sync(0xffffffffu, lane < C && *cl.map_shared_rank(&s_part[0][0], lane) != 0);
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = bad;
    __syncthreads();
    if (s_bad) {
      if (me == 0 && threadIdx.x == 0) a.st->err = 11;
      cl.sync();  // the peers' flags are read before anyone leaves
      return;
    }
  }
  cl.sync();  // the flags are read before round 1 reuses s_part

  unsigned long long S = (unsigned long long)a.nnz;
  long long nU = n, sum_active = 0;
  unsigned long long cross = 0, preds_total = 0;
  int l = 0, err = 0, nUloc = nown;
  while (nU > 0) {
    ++l;
    const int par = l & 1;
    const long long dmax = dmax_of(a.num, a.den, S, nU);
    const int32_t* Uin = Ul[l & 1];
    int32_t* Uout = Ul[(l + 1) & 1];
    // this round's partial-sum slot: last read by the peers in round l-2
    if (threadIdx.x < kTpFields) s_part[par][threadIdx.x] = 0;
    __syncthreads();
    // select (own vertices; local lists)
    unsigned long long sumD = 0;
    for (int base = warp * 32; base < nUloc; base += kTinyBlock) {
      const int i = base + lane;
      const bool valid = i < nUloc;
      const int v = valid ? (l == 1 ? (i << cs) + me : Uin[i]) : 0;
      const int iv = v >> cs;
      int d = 0;
      if (valid) d = D[iv];
      const bool sel = valid && d <= dmax;
      if (valid && (sel || l == 1)) rnd[iv] = sel ? l : 0;
      if (sel) sumD += (unsigned long long)d;
      const unsigned bs = __ballot_sync(0xffffffffu, sel), bu = __ballot_sync(0xffffffffu, valid && !sel);
      int ps = 0, pu = 0;
      if (lane == 0) {
        if (bs) ps = atomicAdd(&s_nR, __popc(bs));
        if (bu) pu = atomicAdd(&s_nUo, __popc(bu));
      }
      ps = __shfl_sync(0xffffffffu, ps, 0);
      pu = __shfl_sync(0xffffffffu, pu, 0);
      if (sel) Rl[ps + __popc(bs & lanemask_lt())] = v;
      if (valid && !sel) Uout[pu + __popc(bu & lanemask_lt())] = v;
    }
    sumD = warp_sum(sumD);
    if (lane == 0) s_wsum[warp][0] = sumD;
    __syncthreads();
    if (warp == 0) {  // the warp sums of the block, one lane each
      const unsigned long long t = warp_sum(s_wsum[lane][0]);
      if (lane == 0) {
        s_part[par][kTpSumD] = t;
        s_part[par][kTpR] = (unsigned long long)s_nR;
        s_part[par][kTpUout] = (unsigned long long)s_nUo;
      }
    }
    cl.sync();
    SMALL_STAMP();
    // UPDATE + JP Part 1 over the own R_l; decrements go to the owners' D
    const int nR = s_nR;
    unsigned long long cut = 0, preds = 0;
    const int vpwR = verts_per_warp(nR, kTinyWarps);
    for (int base = warp * vpwR; base < nR; base += kTinyWarps * vpwR) {
      const int i = base + lane;
      const bool valid = lane < vpwR && i < nR;
      const int v = valid ? Rl[i] : 0;
      const int o = valid ? loff[v >> cs] : 0;
      const int deg = valid ? loff[(v >> cs) + 1] - o : 0;
      const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
      int incl = deg;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
      }
      const int start = incl - deg;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int j0 = 0; j0 < total; j0 += 32 * kSmallUnroll) {
        int own[kSmallUnroll], u[kSmallUnroll], ru[kSmallUnroll];
#pragma unroll
        for (int k = 0; k < kSmallUnroll; ++k) {
          const int j = j0 + 32 * k + lane;
          own[k] = owner_of(start, j);
          const int os = __shfl_sync(0xffffffffu, o, own[k]);
          const int ss = __shfl_sync(0xffffffffu, start, own[k]);
          u[k] = j < total ? ladj[os + (j - ss)] : -1;
          PGC_DCHECK(j >= total || (u[k] >= 0 && u[k] < n), u[k], j);
        }
#pragma unroll
        for (int k = 0; k < kSmallUnroll; ++k) ru[k] = u[k] >= 0 ? *at(rnd, u[k]) : -1;
#pragma unroll
        for (int k = 0; k < kSmallUnroll; ++k) {
          const uint64_t hs = __shfl_sync(0xffffffffu, hv, own[k]);
          bool pred = false;
          if (ru[k] == 0) {
            atomicSub(at(D, u[k]), 1);
            ++cut;
            pred = true;
          } else if (ru[k] == l) {
            pred = prio_hash(a.seed, (uint32_t)u[k]) > hs;
          }
          const unsigned same = __match_any_sync(0xffffffffu, own[k]);
          const int c = __popc(__ballot_sync(0xffffffffu, pred) & same);
          if (c && lane == __ffs(same) - 1) atomicAdd(&s_acc[warp][own[k]], c);
        }
      }
      __syncwarp();
      const int p = s_acc[warp][lane];
      s_acc[warp][lane] = 0;
      if (valid) {
        cnt[v >> cs] = p;
        preds += (unsigned long long)p;
      }
      const unsigned bf = __ballot_sync(0xffffffffu, valid && p == 0);
      int pf = 0;
      if (lane == 0 && bf) pf = atomicAdd(&s_fcnt[1], __popc(bf));
      pf = __shfl_sync(0xffffffffu, pf, 0);
      if (valid && p == 0) Fb[1][pf + __popc(bf & lanemask_lt())] = v;
      __syncwarp();
    }
    cut = warp_sum(cut);
    preds = warp_sum(preds);
    if (lane == 0) {
      s_wsum[warp][0] = cut;
      s_wsum[warp][1] = preds;
    }
    __syncthreads();
    if (warp == 0) {
      const unsigned long long t0 = warp_sum(s_wsum[lane][0]), t1 = warp_sum(s_wsum[lane][1]);
      if (lane == 0) {
        s_part[par][kTpCut] = t0;
        s_part[par][kTpPreds] = t1;
      }
    }
    cl.sync();
    SMALL_STAMP();
    // every CTA sums the C partials (warp 0, one lane per CTA)
    if (warp == 0) {
      unsigned long long x[kTpFields];
#pragma unroll
      for (int f = 0; f < kTpFields; ++f)  // all C x fields loads in flight
        x[f] = lane < C ? *cl.map_shared_rank(&s_part[par][f], lane) : 0ull;
#pragma unroll
      for (int f = 0; f < kTpFields; ++f) {
        x[f] = warp_sum(x[f]);
        if (lane == 0) s_tot[f] = x[f];
      }
    }
    __syncthreads();
    const long long nU1 = (long long)s_tot[kTpUout];
    const long long nRg = (long long)s_tot[kTpR];
    const unsigned long long sumDR = s_tot[kTpSumD], cut_l = s_tot[kTpCut];
    preds_total += s_tot[kTpPreds];
    if (me == 0 && threadIdx.x == 0 && l - 1 < kMaxRoundStats) {
      a.per_round[3 * (l - 1) + 0] = nU;
      a.per_round[3 * (l - 1) + 1] = (long long)S;
      a.per_round[3 * (l - 1) + 2] = nRg;
    }
    sum_active += nU;
    cross += cut_l;
    if (nRg == 0) err = 1;
    if (nU1 != nU - nRg) err = 2;
    if (!((unsigned __int128)nU1 * ((unsigned long long)a.den + a.num) <
          (unsigned __int128)nU * a.den))
      err = 7;
    S = S - sumDR - cut_l;
    nU = nU1;
    nUloc = s_nUo;
    __syncthreads();  // every thread has read s_nR / s_nUo / s_tot
    if (threadIdx.x == 0) {
      s_nR = 0;
      s_nUo = 0;
    }
    __syncthreads();
    if (err) break;
  }

  // ---------------------------------------------------------------- JP
  int J = 0, kmax = 0;
  __shared__ int s_stall;
  if (threadIdx.x == 0) s_stall = 0;
  __syncthreads();
  if (!err && a.dataflow) {
    // Dataflow JP (Alg. 3 with its count[] Join, no level barriers): thread t
    // owns the local vertices t, t + 1024, ... and colors them in decreasing
    // priority, each once its count reaches 0 -- deadlock-free: the
    // highest-priority uncolored vertex always has all preds colored and is
    // the current vertex of its thread (a thread's earlier vertices have
    // higher priority, so they are colored).  A pred's color (and level) is
    // released before its decrement (cluster-scope fences); the decrement
    // is a DSMEM atomic on the succ's count.
    int32_t* lvl = Ul[0];  // JP levels (free after ADG)
    int mine[kTinyPer];
    int nm = 0;
    for (int i = threadIdx.x; i < nown && nm < kTinyPer; i += kTinyBlock) mine[nm++] = i;
    for (int x = 1; x < nm; ++x) {  // insertion sort, priority descending
      const int y = mine[x];
      const int ry = rnd[y];
      const uint64_t hy = prio_hash(a.seed, (uint32_t)((y << cs) + me));
      int z = x - 1;
      while (z >= 0 && prio_gt(ry, hy, rnd[mine[z]], prio_hash(a.seed, (uint32_t)((mine[z] << cs) + me)))) {
        mine[z + 1] = mine[z];
        --z;
      }
      mine[z + 1] = y;
    }
    // warp-synchronous: every lane checks its current vertex's count, then the
    // whole warp processes the ready ones one by one (lanes over the arcs):
    // no divergent spinning inside a warp
    const unsigned long long deadline = globaltimer() + a.watchdog_ns;
    int q = 0;
    unsigned ns = 0;
    for (;;) {
      const bool have = q < nm;
      bool ready = false;
      if (have) {  // acquire: a pred's color precedes its (release) decrement
        int cv;
        asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(cv) : "l"(cnt + mine[q]) : "memory");
        ready = cv == 0;
      }
      unsigned rb = __ballot_sync(0xffffffffu, ready);
      if (!__any_sync(0xffffffffu, have)) break;
      if (!rb) {
        if (__shfl_sync(0xffffffffu, (int)(globaltimer() > deadline), 0)) {
          if (lane == 0) s_stall = 1;
          break;
        }
        if (ns) __nanosleep(ns);
        ns = ns ? min(ns * 2, 128u) : 16u;
        continue;
      }
      ns = 0;
      while (rb) {
        const int src = __ffs(rb) - 1;
        rb &= rb - 1;
        const int i = __shfl_sync(0xffffffffu, have ? mine[q < nm ? q : 0] : 0, src);
        const int v = (i << cs) + me;
        const int rv = rnd[i];
        const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
        const int o = loff[i], d = loff[i + 1] - o;
        int color = 0, lv = 0;
        // the first 32 arcs' (u, pred?) stay in registers for the Join below
        int u0 = -1;
        bool pr0 = false;
        for (int wbase = 0; !color; wbase += 64) {
          unsigned long long m = 0;
          for (int e0 = 0; e0 < d; e0 += 32) {
            const int e = e0 + lane;
            const int u = e < d ? ladj[o + e] : -1;
            // round and color loaded together (one DSMEM round trip; the color
            // is used only if u turns out to be a pred)
            const int ru = u >= 0 ? *at(rnd, u) : -1;
            const int cl_u = u >= 0 ? *at(clr, u) : 0;
            const bool pr = u >= 0 && prio_gt(ru, prio_hash(a.seed, (uint32_t)u), rv, hv);
            if (e0 == 0 && wbase == 0) {
              u0 = u;
              pr0 = pr;
            }
            const int cu = pr ? cl_u : 0;
            if (pr && a.levels && wbase == 0) lv = max(lv, *at(lvl, u));
            PGC_DCHECK(!pr || cu > 0, u, cu);  // every pred is colored
            const int cb = cu - 1 - wbase;
            const bool in = pr && cb >= 0 && cb < 64;
            // OR of the lanes' color bits: shuffle-reduce the 64-bit word
            unsigned long long bit = in ? (1ull << cb) : 0ull;
#pragma unroll
            for (int s2 = 16; s2 > 0; s2 >>= 1) bit |= __shfl_xor_sync(0xffffffffu, bit, s2);
            m |= bit;
          }
          if (~m) color = wbase + __ffsll((long long)~m);
        }
        lv = warp_max(lv);
        if (lane == src) {
          clr[i] = color;
          if (a.levels) lvl[i] = lv + 1;
        }
        kmax = max(kmax, color);
        J = max(J, lv + 1);
        // Join: release decrements (the color store above precedes them)
        __syncwarp();
        for (int e0 = 0; e0 < d; e0 += 32) {
          const int e = e0 + lane;
          int u;
          bool succ;
          if (e0 == 0) {
            u = u0;
            succ = u0 >= 0 && !pr0;
          } else {
            u = e < d ? ladj[o + e] : -1;
            const int ru = u >= 0 ? *at(rnd, u) : -1;
            succ = u >= 0 && prio_gt(rv, hv, ru, prio_hash(a.seed, (uint32_t)u));
          }
          if (succ)
            asm volatile("red.release.cluster.add.s32 [%0], %1;" ::"l"(at(cnt, u)), "r"(-1) : "memory");
        }
        if (lane == src) ++q;
      }
    }
    J = a.levels ? J : 0;
    cl.sync();  // every vertex colored; the peers' stall flags below
    SMALL_STAMP();
    if (threadIdx.x < 32) {
      const int x = lane < C ? *cl.map_shared_rank(&s_stall, lane) : 0;
      if (__any_sync(0xffffffffu, x != 0) && lane == 0) err = 9;
    }
    if (threadIdx.x == 0 && err == 9) s_stall = 2;
    __syncthreads();
    if (s_stall == 2) err = 9;
  } else if (!err) {
    long long nF = 0;
    if (warp == 0) {
      long long x = lane < C ? *cl.map_shared_rank(&s_fcnt[1], lane) : 0;
      x = warp_sum(x);
      if (lane == 0) s_tot[0] = (unsigned long long)x;
    }
    __syncthreads();
    nF = (long long)s_tot[0];
    for (int j = 1; nF > 0; ++j) {
      J = j;
      const int nFl = s_fcnt[j % 3];
      const int32_t* Fin = Fb[j & 1];
      int32_t* Fout = Fb[(j + 1) & 1];
      const int nslot = (j + 1) % 3;
      __syncthreads();  // every thread has read s_fcnt[j % 3] and s_tot
      if (threadIdx.x == 0) s_fcnt[(j + 2) % 3] = 0;  // level j+2's (pushed into at level j+1)
      const int vpwF = verts_per_warp(nFl, kTinyWarps);
      for (int base = warp * vpwF; base < nFl; base += kTinyWarps * vpwF) {
        const int i = base + lane;
        const bool valid = lane < vpwF && i < nFl;
        const int v = valid ? Fin[i] : 0;
        const int o = valid ? loff[v >> cs] : 0;
        const int deg = valid ? loff[(v >> cs) + 1] - o : 0;
        const int rv = valid ? rnd[v >> cs] : 0;
        const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
        int incl = deg;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, s);
          if (lane >= s) incl += y;
        }
        const int start = incl - deg;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        bool need = valid && j > 1;
        int mycolor = valid ? 1 : 0;
        for (int wbase = 0, first = 1; first || __ballot_sync(0xffffffffu, need); wbase += 64, first = 0) {
          for (int j0 = 0; j0 < total; j0 += 32 * kSmallUnroll) {
            int own[kSmallUnroll], u[kSmallUnroll], ru[kSmallUnroll], cu[kSmallUnroll], on[kSmallUnroll];
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              const int jj = j0 + 32 * k + lane;
              own[k] = owner_of(start, jj);
              const int os = __shfl_sync(0xffffffffu, o, own[k]);
              const int ss = __shfl_sync(0xffffffffu, start, own[k]);
              on[k] = __shfl_sync(0xffffffffu, (int)need, own[k]);
              const bool scan = jj < total && (first || on[k]);
              u[k] = scan ? ladj[os + (jj - ss)] : -1;
            }
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              ru[k] = u[k] >= 0 ? *at(rnd, u[k]) : -1;
              cu[k] = u[k] >= 0 && on[k] ? *at(clr, u[k]) : 0;
            }
            // classify every step, all count decrements in flight together
            int oldc[kSmallUnroll];
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              const int rs = __shfl_sync(0xffffffffu, rv, own[k]);
              const uint64_t hs = __shfl_sync(0xffffffffu, hv, own[k]);
              oldc[k] = 0;
              if (u[k] >= 0) {
                if (prio_gt(ru[k], prio_hash(a.seed, (uint32_t)u[k]), rs, hs)) {
                  if (on[k]) {
                    const int cb = cu[k] - 1 - wbase;
                    PGC_DCHECK(cb + wbase >= 0, u[k], cb + wbase);
                    if (cb >= 0 && cb < 64) atomicOr(&s_mask[warp][own[k]][cb >> 5], 1u << (cb & 31));
                  }
                } else if (first) {
                  oldc[k] = atomicSub(at(cnt, u[k]), 1);
                  PGC_DCHECK(oldc[k] >= 1, u[k], oldc[k]);
                }
              }
            }
            // a freed u goes to its owner's next frontier: one DSMEM atomic per
            // (step, owner) group, all issued before any position is used
            unsigned grp[kSmallUnroll];
            int pos[kSmallUnroll], key[kSmallUnroll];
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              key[k] = oldc[k] == 1 ? (u[k] & (C - 1)) : -1;
              grp[k] = __match_any_sync(0xffffffffu, key[k]);
              pos[k] = 0;
              if (key[k] >= 0 && lane == __ffs(grp[k]) - 1)
                pos[k] = atomicAdd(cl.map_shared_rank(&s_fcnt[nslot], key[k]), __popc(grp[k]));
            }
#pragma unroll
            for (int k = 0; k < kSmallUnroll; ++k) {
              const int p0 = __shfl_sync(0xffffffffu, pos[k], __ffs(grp[k]) - 1);
              if (key[k] >= 0)
                *cl.map_shared_rank(Fout + p0 + __popc(grp[k] & lanemask_lt()), key[k]) = u[k];
            }
          }
          __syncwarp();
          const unsigned long long m =
              ((unsigned long long)s_mask[warp][lane][1] << 32) | s_mask[warp][lane][0];
          s_mask[warp][lane][0] = s_mask[warp][lane][1] = 0;
          if (need && ~m) {
            mycolor = wbase + __ffsll((long long)~m);
            need = false;
          }
          __syncwarp();
        }
        if (valid) {
          clr[v >> cs] = mycolor;
          kmax = max(kmax, mycolor);
        }
      }
      cl.sync();
      SMALL_STAMP();
      if (warp == 0) {
        long long x = lane < C ? *cl.map_shared_rank(&s_fcnt[nslot], lane) : 0;
        x = warp_sum(x);
        if (lane == 0) s_tot[0] = (unsigned long long)x;
      }
      __syncthreads();
      nF = (long long)s_tot[0];
    }
  }
#ifdef PGC_PROBE
  if (tid == 0) {
    printf("tiny phases (us):");
    for (int k = 1; k < nstamp; ++k) printf(" %.1f", (stamps[k] - stamps[k - 1]) * 1e-3);
    printf("\ntotal %.1f us, %d phases, cluster %d\n", (stamps[nstamp - 1] - stamps[0]) * 1e-3, nstamp, C);
  }
#endif
  // outputs: every CTA writes its own vertices
  for (int i = threadIdx.x; i < nown; i += kTinyBlock) {
    const int v = (i << cs) + me;
    a.round[v] = rnd[i];
    a.color[v] = err ? 0 : clr[i];
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&a.st->K, kmax);
  if (a.dataflow) {  // J: a per-thread max here
    J = warp_max(J);
    if (lane == 0 && J) atomicMax(&a.st->jp_levels, J);
  }
  if (me == 0 && threadIdx.x == 0) {
    State* st = a.st;
    st->T = l;
    st->rmax = l;
    st->sum_active = sum_active;
    st->cross = cross;
    st->pred_arcs = preds_total;
    if (!a.dataflow) st->jp_levels = J;
    st->err = err;
    st->done = 1;
    st->nU = nU;
    st->S = S;
  }
  cl.sync();  // no CTA leaves while a peer may still access its shared memory
}

// Host side: one cooperative launch, one state read-back.
bool small_path_wanted(const Ctx& c) {
  if (c.tune.small_max_arcs <= 0 || c.n <= 0) return false;
  if (c.nnz > c.tune.small_max_arcs) return false;
  return c.nnz <= (long long)c.tune.small_max_avg * c.n;
}

static_assert(kSmallCtrBytes <= 2 * (size_t)kFilterBytes, "counter ring must fit the filter region");

// The one-cluster variant when the graph fits the cluster's shared memory:
// returns -1 when it ran (and succeeded), 0 when not applicable, else an error.
static int tiny_try(Ctx& c, uint32_t num, uint32_t den, uint64_t seed, int32_t* round, int32_t* color) {
  if (c.tune.tiny_max_n <= 0 || c.n > c.tune.tiny_max_n || c.nnz > c.tune.tiny_max_arcs) return 0;
  if (c.n >= (1ll << 30)) return 0;
  bool& attr = once_flag(c.dev, 10);
  static thread_local int max_smem[kMaxDevices] = {};
  if (!attr) {
    int optin = 0;
    PGC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.dev));
    cudaFuncAttributes fa;
    PGC_CUDA(cudaFuncGetAttributes(&fa, k_tiny_jp_adg));
    max_smem[c.dev] = optin - (int)fa.sharedSizeBytes;
    if (cudaFuncSetAttribute(k_tiny_jp_adg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_smem[c.dev]) != cudaSuccess ||
        cudaFuncSetAttribute(k_tiny_jp_adg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess) {
      cudaGetLastError();
      max_smem[c.dev] = 0;  // no tiny path on this device
    }
    attr = true;
  }
  int C = 0;
  size_t smem = 0;
  int nloc = 0;
  for (int cand = kTinyMaxC; cand >= 2; cand >>= 1) {
    nloc = (int)((c.n + cand - 1) / cand);
    // the arrays, the row starts and at least the mean row share of the CSR
    const long long need = 4ll * ((long long)kTinyArrays * (nloc > 0 ? nloc : 1) + nloc + 1) +
                           4ll * ((c.nnz + cand - 1) / cand);
    if (need > max_smem[c.dev]) break;  // a smaller cluster holds less per cluster
    smem = (size_t)max_smem[c.dev];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cand);
    cfg.blockDim = dim3(kTinyBlock);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cand;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k_tiny_jp_adg, &cfg) == cudaSuccess && ncl >= 1) {
      C = cand;
      break;
    }
    cudaGetLastError();
  }
  if (!C) return 0;
  TinyArgs a;
  a.n = c.n;
  a.nnz = c.nnz;
  a.off = c.off;
  a.col = c.col;
  a.num = num;
  a.den = den;
  a.seed = seed;
  a.round = round;
  a.color = color;
  a.st = c.state;
  a.per_round = c.per_round;
  a.nloc = nloc;
  a.cshift = __builtin_ctz((unsigned)C);
  a.adj_cap = ((long long)smem - 4ll * ((long long)kTinyArrays * nloc + nloc + 1)) / 4;
  a.dataflow = c.tune.tiny_dataflow && nloc <= kTinyPer * kTinyBlock;
  a.levels = c.tune.levels;
  a.watchdog_ns = (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kTinyBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (c.col_ready) PGC_CUDA(cudaStreamWaitEvent(c.st, c.col_ready, 0));
  PGC_LAUNCH(c, kGSelect, "k_tiny_jp_adg", PGC_CUDA(cudaLaunchKernelEx(&cfg, k_tiny_jp_adg, a)));
  if (int e = sync_state(c)) return e;
  const State* h = c.h_state;
  if (h->err == 11) return 0;  // a CTA's rows did not fit its shared memory: the grid kernel
  if (h->err == 9)
    return fail(4, "JP (one-cluster dataflow) stalled: no progress within %d ms (watchdog)",
                c.tune.jp_watchdog_ms);
  if (h->err == 7)
    return fail(4, "ADG round %d broke Lemma 1's per-round shrink (PAPER.md:761-771)", h->T);
  if (h->err) return fail(4, "ADG internal invariant failed (code %d)", h->err);
  c.jp_levels = c.tune.levels ? h->jp_levels : 0;
  c.small = 2;
  c.core_ctas = C;
  return -1;
}

int small_run(Ctx& c, uint32_t num, uint32_t den, uint64_t seed, int32_t* round, int32_t* color) {
  NvtxRange nvtx_("pgc one-kernel JP-ADG");
  PGC_CHK_SIZES(c);
  if (!once_flag(c.dev, 11)) {  // load the kernel before the first timed launch
    cudaFuncAttributes fa;
    PGC_CUDA(cudaFuncGetAttributes(&fa, k_small_jp_adg));
    once_flag(c.dev, 11) = true;
  }
  if (int e = tiny_try(c, num, den, seed, round, color)) return e < 0 ? 0 : e;  // done on one cluster
  SmallArgs a;
  a.n = c.n;
  a.nnz = c.nnz;
  a.off = c.off;
  a.col = c.col;
  a.num = num;
  a.den = den;
  a.seed = seed;
  a.round = round;
  a.color = color;
  a.D = c.D;
  a.cnt = c.npred;
  a.U[0] = c.U[0];
  a.U[1] = c.U[1];
  a.R = c.Rl;
  int32_t* fr = reinterpret_cast<int32_t*>(c.rec);  // 16 (2n + ...) bytes: two n-int frontiers
  a.F[0] = fr;
  a.F[1] = fr + c.n;
  a.ctr = reinterpret_cast<unsigned long long*>(c.filt);  // the UPDATE filter is unused here
  a.st = c.state;
  a.per_round = c.per_round;
  // grid: enough warps for a wave of the largest phase, at most one wave of
  // resident blocks (a grid barrier needs every block resident)
  const int occ = occupancy_cached(c.dev, (const void*)k_small_jp_adg, kSmallBlock, 0);
  const int cap = c.nsm * (c.tune.small_blocks_per_sm > 0 && c.tune.small_blocks_per_sm < occ
                               ? c.tune.small_blocks_per_sm
                               : occ);
  const long long want = (c.n + kSmallBlock - 1) / kSmallBlock;
  const int G = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  if (c.col_ready) PGC_CUDA(cudaStreamWaitEvent(c.st, c.col_ready, 0));
  void* args[] = {&a};
  PGC_LAUNCH(c, kGSelect, "k_small_jp_adg",
             PGC_CUDA(cudaLaunchCooperativeKernel((const void*)k_small_jp_adg, dim3(G),
                                                  dim3(kSmallBlock), args, 0, c.st)));
  if (int e = sync_state(c)) return e;
  const State* h = c.h_state;
  if (h->err == 7)
    return fail(4, "ADG round %d broke Lemma 1's per-round shrink (PAPER.md:761-771)", h->T);
  if (h->err) return fail(4, "ADG internal invariant failed (code %d)", h->err);
  c.jp_levels = c.tune.levels ? h->jp_levels : 0;  // (free here; reported like the other path)
  c.small = 1;
  return 0;
}

}  // namespace pgc
