// adg.cu -- ADG (Algorithm 1) on the B200, plus the arc
// classification kernels shared with JP Part 1 (Algorithm 3).
//
// Per round l (host loop, kernels read every size from device memory):
//   k_adg_select   Count/Reduce are cached (S_l, |U_l| carried in State,
//                  PAPER.md:2353-2365); Dmax_l = floor((den+num)*S_l/(den*|U_l|))
//                  once per block in 128-bit; R_l = {v in U_l : D[v] <= Dmax_l}
//                  (exact); round[v] = l (688-689); block-level
//                  ballot compaction of R_l (light list + heavy edge chunks)
//                  and U_{l+1} (U = U \ R, 687).
//   k_update_*     UPDATE (692-696): for v in R_l, u in N(v) with round[u]==0:
//                  D[u] -= 1 (RED, result unused), cut += 1.  Fused JP Part 1
//                  (PAPER.md:2259-2271): pred(v) = {u alive} U {u in R_l :
//                  h(u) > h(v)} is written into v's own CSR slot of P[] and
//                  npred[v] = |pred(v)| (= count[v] of Alg. 3).
//   k_adg_finalize S_{l+1} = S_l - sum_{R_l} D - cut_l; |U_{l+1}| = |U_l| - |R_l|.
#include <cstdio>
#include <utility>
#include <vector>

#include "pgc_internal.cuh"

namespace pgc {

__global__ void k_zero_i32(int32_t* p, int64_t len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}
__global__ void k_zero_i32_dev(int32_t* p, const int* len, int extra) {
  int64_t L = (int64_t)*len + extra;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

// a1: D[v] = deg(v); round[v] = 0 (v in U); optional color[v] = 0 (uncolored,
// PAPER.md:1115).  Thread 0 initialises the round state: S_1 = nnz, |U_1| = n.
// An isolated vertex (deg 0) is settled here: it counts in |U| (Q12) and gets
// its round from the select kernel like any vertex (with ADG's mean rule that
// is round 1: D = 0 <= Dmax_1), but it has no arc to scan and is no pred of
// any vertex, so it gets no work record; with JP its color is GetColor of the empty
// pred set, 1, and npred = -1 keeps it out of the priority
// order (it can neither wait nor be waited on).
__global__ void k_adg_init(int64_t n, int64_t nnz, const int64_t* __restrict__ off,
                           int32_t* __restrict__ D, uint8_t* __restrict__ rs,
                           int32_t* __restrict__ round, int32_t* __restrict__ color,
                           int32_t* __restrict__ npred, uint32_t* __restrict__ filt, State* st) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = (int32_t)(off[v + 1] - off[v]);
    st_i32_keep(D + v, d);
    st_u8_keep(rs + v, 0);
    round[v] = 0;
    if (color) {
      color[v] = d == 0 ? 1 : 0;
      npred[v] = d == 0 ? -1 : 0;  // (the fused UPDATE overwrites it with |pred(v)|)
    }
  }
  if (filt)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * kFilterWords;
         i += gridDim.x * blockDim.x)
      filt[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    State s = {};
    s.S = (unsigned long long)nnz;
    s.nU = n;
    s.done = (n == 0);
    s.rmin = 1;
    s.rmax = 0;
    *st = s;
  }
}

// The state part of k_adg_init alone: with the mean rule, round 1's
// selection initialises the per-vertex arrays itself (first = 1).
__global__ void k_adg_state_init(int64_t n, int64_t nnz, State* st) {
  State s = {};
  s.S = (unsigned long long)nnz;
  s.nU = n;
  s.done = (n == 0);
  s.rmin = 1;
  s.rmax = 0;
  *st = s;
}

// a2+a3: threshold, select, compact.
constexpr int kSelItems = 4;
__global__ void k_adg_select(int l, int rule, uint32_t num, uint32_t den, const int64_t* __restrict__ off,
                             int32_t* __restrict__ D, int32_t* __restrict__ round,
                             uint8_t* __restrict__ rs,
                             const int32_t* __restrict__ Uin, int32_t* __restrict__ Uout,
                             int4* __restrict__ lrec, int4* __restrict__ chunks,
                             int32_t* __restrict__ npred, State* st, int heavy_deg, int chunk,
                             int64_t chunk_cap, int pull, int mark_removed, int first,
                             int32_t* __restrict__ color, uint32_t* __restrict__ filt,
                             int4* __restrict__ cexp) {
  __shared__ int sm[33];
  __shared__ long long s_dmax;
  __shared__ unsigned long long s_red[32];
  if (st->done) return;
  const long long count = st->nU;
  if (threadIdx.x == 0) {
    // Dmax = floor((den+num) * S / (den * |U|)); den*|U| < 2^63, numerator < 2^97.
    unsigned __int128 numer = (unsigned __int128)((unsigned long long)den + num) * st->S;
    unsigned long long denom = (unsigned long long)den * (unsigned long long)count;
    unsigned __int128 q = numer / denom;
    s_dmax = q > (unsigned __int128)0x7fffffff ? 0x7fffffffLL : (long long)q;
  }
  __syncthreads();
  const long long dmax = s_dmax;
  const unsigned long long mkey = st->msel_key;
  if (first && filt)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * kFilterWords;
         i += gridDim.x * blockDim.x)
      filt[i] = 0;  // ADG-M: the ceil(|U|/2)-th smallest key
  unsigned long long my_sumD = 0;
  unsigned long long my_nR = 0, my_nOrd = 0;
  // kSelItems vertices per thread per step (coalesced: item j of thread t is
  // base + j * blockDim + t); the three output lists (edge chunks, light
  // records, U_{l+1}) are compacted with ONE block scan of packed counts and
  // one atomicAdd per list per step
  constexpr int K = kSelItems;
  const long long step = (long long)gridDim.x * blockDim.x * K;
  for (long long base = (long long)blockIdx.x * blockDim.x * K; base < count; base += step) {
    int v[K], d[K], nch[K];
    long long o[K], deg[K];
    bool valid[K], sel[K], light[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const long long i = base + (long long)j * blockDim.x + threadIdx.x;
      valid[j] = i < count;
      v[j] = valid[j] ? (Uin ? Uin[i] : (int)i) : 0;
    }
    long long o0[K] = {}, e0[K] = {};
    if (first) {  // round 1 fused with init: D[v] = deg(v) from the offsets
#pragma unroll
      for (int j = 0; j < K; ++j) {
        o0[j] = valid[j] ? off[v[j]] : 0;
        e0[j] = valid[j] ? off[v[j] + 1] : 0;
      }
#pragma unroll
      for (int j = 0; j < K; ++j) d[j] = (int)(e0[j] - o0[j]);
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) d[j] = valid[j] ? ld_i32_keep(D + v[j]) : 0;
    }
    unsigned long long packed = 0;  // chunks | light << 32 | unext << 48
#pragma unroll
    for (int j = 0; j < K; ++j) {
      // ADG: D <= (1+eps) * mean (exact integer form);  ADG-M: the
      // ceil(|U|/2) smallest keys (D, id) of U (median rule)
      sel[j] = valid[j] && (rule == kRuleMedian
                                ? ((((unsigned long long)(uint32_t)d[j]) << 32) | (uint32_t)v[j]) <= mkey
                                : d[j] <= dmax);
      light[j] = false;
      nch[j] = 0;
      o[j] = 0;
      deg[j] = 0;
      if (first && valid[j]) {  // k_adg_init's per-vertex state (a1), then round 1's
        st_i32_keep(D + v[j], sel[j] && mark_removed ? -1 : d[j]);
        st_u8_keep(rs + v[j], sel[j] ? 1 : 0);
        round[v[j]] = sel[j] ? l : 0;
        if (color) {
          color[v[j]] = d[j] == 0 ? 1 : 0;
          npred[v[j]] = d[j] == 0 ? -1 : 0;
        }
      } else if (sel[j]) {
        round[v[j]] = l;
        st_u8_keep(rs + v[j], (l - 1) % 255 + 1);
        if (mark_removed) st_i32_keep(D + v[j], -1);  // round 1's atomic UPDATE (Arc::atom)
      }
      if (sel[j]) {
        my_sumD += (unsigned long long)d[j];
        my_nR += 1;
      }
      // UPDATE's work records: push scans R_l's arcs, pull the survivors' (U_{l+1})
      if (pull ? (valid[j] && !sel[j]) : sel[j]) {
        o[j] = first ? o0[j] : off[v[j]];
        deg[j] = first ? e0[j] - o0[j] : off[v[j] + 1] - o[j];
        light[j] = deg[j] > 0 && deg[j] <= heavy_deg;  // isolated: settled by k_adg_init
        if (deg[j] > heavy_deg) {
          nch[j] = (int)((deg[j] + chunk - 1) / chunk);
          if (!pull) npred[v[j]] = 0;
        }
      }
      packed += (unsigned long long)nch[j] + ((unsigned long long)light[j] << 32) +
                ((unsigned long long)(valid[j] && !sel[j]) << 48);
      my_nOrd += (!pull && (light[j] || nch[j] > 0)) ? 1 : 0;  // removed, not isolated
    }
    // block exclusive scan of the packed counts
    const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long incl = packed;
#pragma unroll
    for (int o_ = 1; o_ < 32; o_ <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o_);
      if (lane >= o_) incl += y;
    }
    if (lane == 31) s_red[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long run = 0;
      for (int w = 0; w < nw; ++w) {
        const unsigned long long c = s_red[w];
        s_red[w] = run;
        run += c;
      }
      const unsigned tch = (unsigned)(run & 0xffffffffull), tl = (unsigned)((run >> 32) & 0xffff),
                     tu = (unsigned)(run >> 48);
      sm[0] = tch ? atomicAdd(&st->nChunks, (int)tch) : 0;
      sm[1] = tl ? atomicAdd(&st->nLight, (int)tl) : 0;
      sm[2] = tu ? atomicAdd(&st->nUnext, (int)tu) : 0;
    }
    __syncthreads();
    const unsigned long long ex = s_red[warp] + incl - packed;
    long long cpos = sm[0] + (long long)(ex & 0xffffffffull);
    int lpos = sm[1] + (int)((ex >> 32) & 0xffff), upos = sm[2] + (int)(ex >> 48);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (nch[j]) {
        if (cpos + nch[j] > chunk_cap) st->err = 3;
        else if (nch[j] > kExpandMin) {
          // a hub: one descriptor; k_round_aux writes its records, a warp per
          // hub (one thread writing a late round's ~10^2 records per hub made
          // the selection of the last rounds 20-40 us each)
          const int e = atomicAdd(&st->nExp, 1);
          cexp[2 * e] = make_int4(v[j], nch[j], (int)cpos, (int)deg[j]);
          cexp[2 * e + 1] = make_int4((int)(uint32_t)o[j], (int)(o[j] >> 32), 0, 0);
        } else
          for (int k = 0; k < nch[j]; ++k) {
            const long long s0 = o[j] + (long long)k * chunk;
            const int len = (int)min((long long)chunk, o[j] + deg[j] - s0);
            __stcs(chunks + 2 * (cpos + k), make_int4(v[j], len, (int)(uint32_t)s0, (int)(s0 >> 32)));
            __stcs(chunks + 2 * (cpos + k) + 1, make_int4((int)(uint32_t)o[j], (int)(o[j] >> 32), 0, 0));
          }
        cpos += nch[j];
      }
      if (light[j]) PGC_DCHECK_V(lpos);  // light records: at most n
      if (light[j]) __stcs(lrec + lpos++, light_rec(v[j], (int)deg[j], o[j]));
      if (valid[j] && !sel[j]) {
        PGC_DCHECK_V(upos);  // |U_{l+1}| < n
        PGC_DCHECK_V(v[j]);
        Uout[upos++] = v[j];
      }
    }
    __syncthreads();  // s_red / sm are reused by the next step
  }
  unsigned long long t = block_sum(my_sumD, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(&st->sumDR, t);
  t = block_sum(my_nR, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(&st->nR, (int)t);
  t = block_sum(my_nOrd, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(&st->nOrdR, (int)t);
}

// Arc classifier.  MODE 0: ADG only; 1: ADG with fused JP Part 1; 2: JP Part 1
// for an arbitrary first key (pgc_jp_color); 3: ADG with fused JP Part 1 for
// ADG-O's total order (round, D_rem, id) (UPDATEandPRIORITIZE);
// 4: ADG's pull (CREW) UPDATE: the records are the
// survivors U_{l+1}, an arc is counted iff its target was removed in round l,
// and the owner subtracts its count from its own D (no per-arc atomics).
template <int MODE>
struct Arc {
  static constexpr bool kPreds = MODE != 0 && MODE != 4;  // stores pred slots (JP Part 1)
  int l;
  uint64_t seed;
  const int32_t* __restrict__ round;
  int32_t* __restrict__ D;
  const uint8_t* __restrict__ rs;
  // Round 1 of MODES 0/1 (knob update_atom): ONE atomic per arc instead of a
  // state gather plus a RED.  k_adg_select has set D = -1 on R_1, so the
  // DecrementAndFetch's old value classifies the target (>= 0: alive, < 0:
  // removed this round; no vertex was removed earlier); the decrement of a
  // removed vertex is harmless (its D is never read again in these modes and
  // stays negative: at most deg < 2^31 decrements).
  int atom = 0;
  // Round state of u.  MODE 0/1: 0 = alive (u in U), 1 = removed in this
  // round, 2 = removed earlier; read from the 1-byte rs[] while l <= 255
  // (exact: rs = ((round-1) mod 255) + 1), from round[] afterwards.  MODE 2:
  // the key round[u].  Split in two so a kernel issues all of a strip's gathers
  // before it consumes any (raw() on a clamped address is unconditional; a
  // gather whose use sits in the same branch would serialise on its latency).
  __device__ __forceinline__ int raw(int u) const {
    if ((MODE == 0 || MODE == 1) && atom) return u >= 0 ? atom_dec_keep(&D[u]) : 0;
    const int uu = u >= 0 ? u : 0;
    if (MODE != 2 && l <= 255) return ld_u8_keep(rs + uu);  // read-only, L2 evict-last
    return round[uu];
  }
  __device__ __forceinline__ int decode(int u, int x) const {
    if (u < 0) return 0;
    if (MODE == 2) return x;
    if ((MODE == 0 || MODE == 1) && atom) return x < 0 ? 1 : 0;
    return x == 0 ? 0 : (x == l ? 1 : 2);  // for l <= 255, rs == round of every removed u
  }
  __device__ __forceinline__ int state(int u) const { return decode(u, raw(u)); }
  __device__ __forceinline__ int gather(int u) const { return state(u); }
  // v's own second key: rho_R(v) (MODES 1, 2) or (D_rem[v], v) packed (MODE 3;
  // D of a vertex removed this round no longer changes: only alive vertices
  // are decremented)
  __device__ __forceinline__ uint64_t own(int v) const {
    if (MODE == 3) return (((uint64_t)(uint32_t)D[v]) << 32) | (uint32_t)v;
    if (MODE == 4) return 0;
    return prio_hash(seed, (uint32_t)v);
  }
  // true iff u in pred(v); performs UPDATE's decrement and counts cut arcs.
  // g = gather(u).
  // MODE 3: a same-round neighbour's D_rem, loaded for a whole strip before
  // any classify (a load consumed in its own branch would serialise)
  __device__ __forceinline__ int same_round_d(int u, int g) const {
    if (MODE != 3) return 0;
    return g == 1 ? D[u] : 0;
  }
  __device__ __forceinline__ bool classify(int u, int g, int rv, uint64_t hv,
                                          unsigned long long& cut, int du = 0) const {
    if (MODE == 4) {                    // pull: u in N(v) ∩ R_l
      if (g != 1) return false;
      cut += 1;
      return true;
    }
    if (MODE == 2) {
      if (g != rv) return g > rv;
      return prio_hash(seed, (uint32_t)u) > hv;
    }
    const int su = g;
    if (su == 0) {                      // u in U \ R: DecrementAndFetch(D[u])
      if (!((MODE == 0 || MODE == 1) && atom))
        red_dec_keep(&D[u]);            // result unused -> RED (the atom path has decremented)
      cut += 1;
      return MODE == 1 || MODE == 3;    // u gets a later round: higher priority
    }
    if (MODE == 1 && su == 1) return prio_hash(seed, (uint32_t)u) > hv;  // same round: hash
    if (MODE == 3 && su == 1)  // same round: (D_rem, id)
      return ((((uint64_t)(uint32_t)du) << 32) | (uint32_t)u) > hv;
    return false;                       // removed earlier: lower priority
  }
};

// UPDATE for light vertices (deg <= heavy_deg): a warp takes 32 list entries
// and walks their concatenated adjacencies (warp-level merge path: each arc
// finds its owner by a 5-step shuffle search over the inclusive degree scan),
// kStrips strips of 32 arcs in flight (col loads, then state gathers, then
// classification) so each warp keeps kStrips independent requests outstanding.
// Pred slots: the arcs of one owner are contiguous in a strip, so an arc's
// rank among its owner's preds is a popc of the pred ballot over the owner's
// segment; each lane keeps its own vertex's running count in a register (no
// shared-memory atomics).
constexpr int kStrips = 8;
#ifndef PGC_LIGHT_STRIPS
#define PGC_LIGHT_STRIPS 8
#endif
#ifndef PGC_LIGHT_MINB
#define PGC_LIGHT_MINB 1
#endif
constexpr int kLStrips = PGC_LIGHT_STRIPS;
template <int MODE>
__global__ void __launch_bounds__(256, PGC_LIGHT_MINB) k_update_light(Arc<MODE> A, const int32_t* __restrict__ col,
                                                      const int4* __restrict__ lrec,
                                                      int32_t* __restrict__ npred,
                                                      int32_t* __restrict__ P, State* st) {
  __shared__ unsigned long long s_red[32];
  __shared__ int s_next;
  if (MODE != 2 && st->done) return;
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  const int nL = st->nLight;
  // each block owns a contiguous range of 32-vertex groups; its warps take
  // groups from it dynamically (shared-memory ticket), which evens out the
  // degree variance between groups without a contended global counter.  The
  // next group's records are loaded one group ahead.
  const int ngroups = (nL + 31) >> 5;
  const int g_lo = (int)((long long)ngroups * blockIdx.x / gridDim.x);
  const int g_hi = (int)((long long)ngroups * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) s_next = g_lo;
  __syncthreads();
  unsigned long long cut = 0, preds = 0;
  auto take = [&](int& g, int4& r) {
    g = 0;
    if (lane == 0) g = atomicAdd(&s_next, 1);
    g = __shfl_sync(0xffffffffu, g, 0);
    const int i = g * 32 + lane;
    r = (g < g_hi && i < nL) ? __ldcs(lrec + i) : make_int4(0, 0, 0, 0);
  };
  // (records one group ahead; two and three groups ahead measured no faster on
  // R-MAT 24 and 4-6 % slower UPDATE on Chung-Lu / R-MAT 20: 85 registers)
  int g_nx;
  int4 r_nx;
  take(g_nx, r_nx);
  for (;;) {
    const int g = g_nx;
    if (g >= g_hi) break;
    const int4 r = r_nx;
    take(g_nx, r_nx);
    const bool valid = g * 32 + lane < nL;
    const int v = r.x, deg = r.y;
    const long long o = lo_hi(r.z, r.w);
    const int rv = (MODE == 2 && valid) ? A.round[v] : 0;
    const uint64_t hv = (MODE != 0 && valid) ? A.own(v) : 0;
    int incl = deg;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, s);
      if (lane >= s) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - deg;
    int cnt = 0;  // preds of this lane's vertex found so far
    for (int t0 = 0; t0 < total; t0 += 32 * kLStrips) {
      int u[kLStrips], ow[kLStrips], gs[kLStrips];
#pragma unroll
      for (int k = 0; k < kLStrips; ++k) {
        const int a = t0 + 32 * k + lane;
        // owner = number of lanes whose inclusive prefix is <= a
        int lo = 0;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          int x = __shfl_sync(0xffffffffu, incl, lo + s - 1);
          if (x <= a) lo += s;
        }
        ow[k] = lo > 31 ? 31 : lo;
        const long long oo = __shfl_sync(0xffffffffu, o, ow[k]);
        const int oe = __shfl_sync(0xffffffffu, excl, ow[k]);
        if (a < total) PGC_DCHECK_A(oo + (a - oe));
        u[k] = a < total ? ld_stream(col + oo + (a - oe)) : -1;
        if (a < total) PGC_DCHECK_V(u[k]);
      }
#pragma unroll
      for (int k = 0; k < kLStrips; ++k) gs[k] = A.raw(u[k]);  // all gathers in flight
#pragma unroll
      for (int k = 0; k < kLStrips; ++k) gs[k] = A.decode(u[k], gs[k]);
      int du[kLStrips];
#pragma unroll
      for (int k = 0; k < kLStrips; ++k) du[k] = A.same_round_d(u[k], gs[k]);
#pragma unroll
      for (int k = 0; k < kLStrips; ++k) {
        const int ts = t0 + 32 * k;  // first arc of this strip
        const uint64_t oh = MODE != 0 ? __shfl_sync(0xffffffffu, hv, ow[k]) : 0;
        const int orv = MODE == 2 ? __shfl_sync(0xffffffffu, rv, ow[k]) : 0;
        const bool pred = u[k] >= 0 && A.classify(u[k], gs[k], orv, oh, cut, du[k]);
        if (MODE != 0) {
          const unsigned pb = __ballot_sync(0xffffffffu, pred);
          const int base = __shfl_sync(0xffffffffu, cnt, ow[k]);
          const int oe = __shfl_sync(0xffffffffu, excl, ow[k]);
          const long long oo = __shfl_sync(0xffffffffu, o, ow[k]);
          const int seg0 = max(0, oe - ts);  // first lane of the owner's segment
#ifdef PGC_CHECKED
          const int odeg = __shfl_sync(0xffffffffu, deg, ow[k]);
#endif
          if (Arc<MODE>::kPreds && pred) {
            const int rank = __popc(pb & lt & ~((1u << seg0) - 1u));
            PGC_DCHECK(base + rank < odeg, base + rank, odeg);  // pred(v) fits v's CSR slot
            PGC_DCHECK_A(oo + base + rank);
            st_stream(P + oo + base + rank, u[k]);
          }
          // own segment in this strip: lanes [lo, hi)
          const int lo = min(32, max(0, excl - ts)), hi = min(32, max(0, incl - ts));
          const unsigned mhi = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
          const unsigned mlo = lo >= 32 ? 0xffffffffu : ((1u << lo) - 1u);
          cnt += __popc(pb & mhi & ~mlo);
        }
      }
    }
    if (MODE == 4 && valid && cnt) A.D[v] -= cnt;  // v's own counter: one writer
    if (Arc<MODE>::kPreds && valid) {
      npred[v] = cnt;
      preds += (unsigned long long)cnt;
    }
  }
  unsigned long long t = block_sum(cut, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(&st->cut, t);
  if (Arc<MODE>::kPreds) {
    t = block_sum(preds, s_red);
    if (threadIdx.x == 0 && t) atomicAdd(&st->pred_arcs, t);
  }
}

constexpr uint32_t kFilterBitsFwd = kFilterBytes * 8u;
// true iff round l runs the filtered heavy UPDATE (k_update_heavy_f)
__device__ __forceinline__ bool filter_round(const State* st, int ratio) {
  return ratio > 0 && st->nU * (long long)ratio <= (long long)kFilterBitsFwd;
}

// UPDATE for chunked vertices: one warp per `chunk`-arc work item.  The preds
// found in each 512-arc sub-chunk are staged in shared memory and written as
// one coalesced run after a single atomicAdd on npred[v] (no per-strip atomic
// round trip on the critical path).
constexpr int kSub = 512;
template <int MODE>
__global__ void __launch_bounds__(256) k_update_heavy(Arc<MODE> A, const int32_t* __restrict__ col,
                                                      const int4* __restrict__ chunks,
                                                      int32_t* __restrict__ npred,
                                                      int32_t* __restrict__ P, State* st,
                                                      int filter_ratio) {
  __shared__ unsigned long long s_red[32];
  __shared__ int s_buf[Arc<MODE>::kPreds ? 8 : 1][Arc<MODE>::kPreds ? kSub : 1];
  __shared__ int s_next;
  if (MODE != 2 && st->done) return;
  if (MODE != 2 && filter_round(st, filter_ratio)) return;  // k_update_heavy_f's round
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int nC = st->nChunks;
  const int c_lo = (int)((long long)nC * blockIdx.x / gridDim.x);
  const int c_hi = (int)((long long)nC * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) s_next = c_lo;
  __syncthreads();
  unsigned long long cut = 0, preds = 0;
  // chunk records are fetched one item ahead (lanes 0/1 load the two halves)
  auto take = [&](int& ci, int4& r) {
    ci = 0;
    if (lane == 0) ci = atomicAdd(&s_next, 1);
    ci = __shfl_sync(0xffffffffu, ci, 0);
    r = (ci < c_hi && lane < 2) ? __ldcs(chunks + 2 * ci + lane) : make_int4(0, 0, 0, 0);
  };
  int ci_nx;
  int4 r_nx;
  take(ci_nx, r_nx);
  for (;;) {
    const int ci = ci_nx;
    if (ci >= c_hi) break;
    const int4 r0 = r_nx;
    take(ci_nx, r_nx);
    const int v = __shfl_sync(0xffffffffu, r0.x, 0);
    const int len = __shfl_sync(0xffffffffu, r0.y, 0);
    const long long s = lo_hi(__shfl_sync(0xffffffffu, r0.z, 0), __shfl_sync(0xffffffffu, r0.w, 0));
    const long long o = lo_hi(__shfl_sync(0xffffffffu, r0.x, 1), __shfl_sync(0xffffffffu, r0.y, 1));
    const long long e = s + len;
    const uint64_t hv = MODE != 0 ? A.own(v) : 0;
    const int rv = MODE == 2 ? A.round[v] : 0;
    for (long long s0 = s; s0 < e; s0 += kSub) {
      const long long e0 = min(e, s0 + kSub);
      int cnt = 0;  // preds staged in s_buf[warp]
      for (long long a0 = s0; a0 < e0; a0 += 32 * kStrips) {
        // kStrips strips of 32 arcs: independent col loads, then state gathers in flight
        int u[kStrips], g[kStrips];
#pragma unroll
        for (int k = 0; k < kStrips; ++k) {
          const long long a = a0 + 32 * k + lane;
          if (a < e0) PGC_DCHECK_A(a);
          u[k] = a < e0 ? ld_stream(col + a) : -1;
          if (a < e0) PGC_DCHECK_V(u[k]);
        }
#pragma unroll
        for (int k = 0; k < kStrips; ++k) g[k] = A.raw(u[k]);  // all gathers in flight
#pragma unroll
        for (int k = 0; k < kStrips; ++k) g[k] = A.decode(u[k], g[k]);
        int du[kStrips];
#pragma unroll
        for (int k = 0; k < kStrips; ++k) du[k] = A.same_round_d(u[k], g[k]);
#pragma unroll
        for (int k = 0; k < kStrips; ++k) {
          const bool pred = u[k] >= 0 && A.classify(u[k], g[k], rv, hv, cut, du[k]);
          if (MODE != 0) {
            const unsigned bal = __ballot_sync(0xffffffffu, pred);
            if (Arc<MODE>::kPreds && pred) s_buf[warp][cnt + __popc(bal & lanemask_lt())] = u[k];
            cnt += __popc(bal);
          }
        }
      }
      if (MODE == 4 && cnt && lane == 0) atomicSub(&A.D[v], cnt);  // one per sub-chunk
      if (Arc<MODE>::kPreds && cnt) {
        __syncwarp();
        int base = 0;
        if (lane == 0) base = atomicAdd(&npred[v], cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < cnt; i += 32) {
          PGC_DCHECK_A(o + base + i);
          st_stream(P + o + base + i, s_buf[warp][i]);
        }
        if (lane == 0) preds += (unsigned long long)cnt;
        __syncwarp();
      }
    }
  }
  unsigned long long t = block_sum(cut, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(&st->cut, t);
  if (Arc<MODE>::kPreds) {
    t = block_sum(preds, s_red);
    if (threadIdx.x == 0 && t) atomicAdd(&st->pred_arcs, t);
  }
}

// UPDATE for chunked vertices in the late rounds, with a membership filter.
// Once |U_l| is small, most arcs of R_l lead to vertices removed in earlier
// rounds (on R-MAT 24, 171 M of the 236 M arcs of rounds 4-7): their state
// gather is a wasted random access, and UPDATE is bound by the random-access
// rate.  Each CTA (one per SM, 1024 threads) copies a one-hash Bloom filter of
// U_l (the round's input list: alive or removed this round; built once per
// round by k_round_aux) into shared memory; an arc whose target misses the
// filter is "removed earlier" for certain.  A warp first filters a 256-arc
// step and compacts the hits (members of U_l plus <= 1/ratio false positives)
// into shared memory, then gathers, classifies and decrements only those, 32
// per pass: the per-arc work of a dead arc is a load, a hash and one shared
// load.  The result is identical: the filter only skips gathers whose answer
// it already knows.  The plain kernel runs the rounds with |U_l| > bits /
// ratio (each of the two kernels exits if the round is not its).
constexpr int kFilterThreads = 1024;
constexpr int kFilterSub = 256;                       // arcs per step; staged preds / hits per warp
constexpr uint32_t kFilterBits = kFilterBytes * 8u;   // filter bits
constexpr size_t kFilterSmem = kFilterBytes + 2 * (kFilterThreads / 32) * kFilterSub * 4;
static_assert(kFilterBits == kFilterBitsFwd, "filter size");
__device__ __forceinline__ uint32_t filter_slot(int u) {
  return __umulhi((uint32_t)u * 0x9E3779B1u, kFilterBits);
}

// Between round l's selection and its UPDATE, one launch (k_round_aux):
// (a) the membership filter: set the bits of U_l (the round's input list) in
//     the global filter buffer l&1 -- one RED per member, once per round, not
//     per CTA -- and clear buffer (l+1)&1 for the next round (its last reader,
//     UPDATE of round l-1, has finished).  Buffers start zeroed (k_adg_init).
// (b) the saved top list: in the round where |U| drops below target (|U_l| >=
//     target > |U_{l+1}|), keep a copy of U_l -- the smallest U holding every
//     vertex of the top rounds the JP core's prefix is drawn from (with the
//     mean rule U_l, l >= 2, holds no isolated vertex) -- so the priority
//     order's top part need not pass over all n vertices.  U_1 (every vertex)
//     is not kept.
// (c) the chunk records of this round's hubs (k_adg_select's descriptors), a
//     warp per hub.
__global__ void __launch_bounds__(1024) k_round_aux(int l, const int32_t* __restrict__ Uin,
                                                    uint32_t* __restrict__ filt, State* st, int ratio,
                                                    int32_t* __restrict__ save, int target,
                                                    int4* __restrict__ chunks,
                                                    const int4* __restrict__ cexp, int chunk) {
  if (st->done) return;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  const long long nU = st->nU;
  if (filt) {
    uint32_t* nxt = filt + (size_t)((l + 1) & 1) * kFilterWords;
    for (int i = tid; i < kFilterWords / 4; i += nt) reinterpret_cast<uint4*>(nxt)[i] = make_uint4(0, 0, 0, 0);
    if (filter_round(st, ratio)) {
      uint32_t* cur = filt + (size_t)(l & 1) * kFilterWords;
      for (long long i = tid; i < nU; i += nt) {
        const int u = Uin ? Uin[i] : (int)i;
        const uint32_t b = filter_slot(u);
        atomicOr(&cur[b >> 5], 1u << (b & 31));
      }
    }
  }
  if (save && l >= 2 && nU >= target && st->nUnext < target) {
    if (tid == 0) st->top_n = (int)nU;
    for (long long i = tid; i < nU; i += nt) save[i] = Uin[i];
  }
  const int nE = st->nExp;
  const int lane = lane_id();
  for (int e = tid >> 5; e < nE; e += nt >> 5) {
    const int4 d0 = cexp[2 * e], d1 = cexp[2 * e + 1];
    const long long o = lo_hi(d1.x, d1.y);
    const int4 tail = make_int4(d1.x, d1.y, 0, 0);
    for (int k = lane; k < d0.y; k += 32) {
      const long long s0 = o + (long long)k * chunk;
      const int len = (int)min((long long)chunk, o + d0.w - s0);
      __stcs(chunks + 2 * ((long long)d0.z + k), make_int4(d0.x, len, (int)(uint32_t)s0, (int)(s0 >> 32)));
      __stcs(chunks + 2 * ((long long)d0.z + k) + 1, tail);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFilterThreads, 1)
    k_update_heavy_f(Arc<MODE> A, const int32_t* __restrict__ col, const int4* __restrict__ chunks,
                     const uint32_t* __restrict__ gfilt, int32_t* __restrict__ npred,
                     int32_t* __restrict__ P, State* st, int ratio) {
  extern __shared__ __align__(16) unsigned char f_smem[];
  uint32_t* filt = reinterpret_cast<uint32_t*>(f_smem);
  int* s_buf_all = reinterpret_cast<int*>(f_smem + kFilterBytes);
  __shared__ unsigned long long s_red[32];
  __shared__ int s_next;
  if (st->done || !filter_round(st, ratio)) return;
  const int nC = st->nChunks;
  if (nC == 0) return;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  int* s_buf = s_buf_all + warp * kFilterSub;
  int* s_hit = s_buf_all + (kFilterThreads / 32 + warp) * kFilterSub;
  {  // the round's filter (built by k_round_aux) -> shared memory
    const uint4* src = reinterpret_cast<const uint4*>(gfilt + (size_t)(A.l & 1) * kFilterWords);
    uint4* dst = reinterpret_cast<uint4*>(filt);
    for (int i = threadIdx.x; i < kFilterWords / 4; i += blockDim.x) dst[i] = __ldcg(src + i);
  }
  const int c_lo = (int)((long long)nC * blockIdx.x / gridDim.x);
  const int c_hi = (int)((long long)nC * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) s_next = c_lo;
  __syncthreads();
  unsigned long long cut = 0, preds = 0;
  auto take = [&](int& ci, int4& r) {
    ci = 0;
    if (lane == 0) ci = atomicAdd(&s_next, 1);
    ci = __shfl_sync(0xffffffffu, ci, 0);
    r = (ci < c_hi && lane < 2) ? __ldcs(chunks + 2 * ci + lane) : make_int4(0, 0, 0, 0);
  };
  int ci_nx;
  int4 r_nx;
  take(ci_nx, r_nx);
  for (;;) {
    const int ci = ci_nx;
    if (ci >= c_hi) break;
    const int4 r0 = r_nx;
    take(ci_nx, r_nx);
    const int v = __shfl_sync(0xffffffffu, r0.x, 0);
    const int len = __shfl_sync(0xffffffffu, r0.y, 0);
    const long long s = lo_hi(__shfl_sync(0xffffffffu, r0.z, 0), __shfl_sync(0xffffffffu, r0.w, 0));
    const long long o = lo_hi(__shfl_sync(0xffffffffu, r0.x, 1), __shfl_sync(0xffffffffu, r0.y, 1));
    const long long e = s + len;
    const uint64_t hv = MODE != 0 ? A.own(v) : 0;
    for (long long s0 = s; s0 < e; s0 += kFilterSub) {
      const long long e0 = min(e, s0 + kFilterSub);
      // 1. filter the step's arcs; compact the hits into s_hit (arc order kept)
      int nh = 0;
      {
        static_assert(32 * kStrips == kFilterSub, "one filter pass per step");
        int u[kStrips];
        uint32_t fw[kStrips];
#pragma unroll
        for (int k = 0; k < kStrips; ++k) {
          const long long a = s0 + 32 * k + lane;
          u[k] = a < e0 ? ld_stream(col + a) : -1;
        }
#pragma unroll
        for (int k = 0; k < kStrips; ++k) fw[k] = filt[filter_slot(u[k] >= 0 ? u[k] : 0) >> 5];
#pragma unroll
        for (int k = 0; k < kStrips; ++k) {
          const bool hit = u[k] >= 0 && ((fw[k] >> (filter_slot(u[k]) & 31)) & 1u);
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (hit) s_hit[nh + __popc(bal & lt)] = u[k];
          nh += __popc(bal);
        }
      }
      __syncwarp();
      // 2. the hits, 64 per pass (two gathers in flight per lane): the real
      //    state, UPDATE's decrement, the pred test
      int cnt = 0;
      for (int j0 = 0; j0 < nh; j0 += 64) {
        int u[2], g[2], du[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) u[k] = j0 + 32 * k + lane < nh ? s_hit[j0 + 32 * k + lane] : -1;
#pragma unroll
        for (int k = 0; k < 2; ++k) g[k] = A.raw(u[k]);
#pragma unroll
        for (int k = 0; k < 2; ++k) g[k] = A.decode(u[k], g[k]);
#pragma unroll
        for (int k = 0; k < 2; ++k) du[k] = A.same_round_d(u[k], g[k]);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const bool pred = u[k] >= 0 && A.classify(u[k], g[k], 0, hv, cut, du[k]);
          if (MODE != 0) {
            const unsigned bal = __ballot_sync(0xffffffffu, pred);
            if (pred) s_buf[cnt + __popc(bal & lt)] = u[k];
            cnt += __popc(bal);
          }
        }
      }
      if (MODE != 0 && cnt) {
        __syncwarp();
        int base = 0;
        if (lane == 0) base = atomicAdd(&npred[v], cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < cnt; i += 32) st_stream(P + o + base + i, s_buf[i]);
        if (lane == 0) preds += (unsigned long long)cnt;
        __syncwarp();
      }
    }
  }
  unsigned long long t = block_sum(cut, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(&st->cut, t);
  if (Arc<MODE>::kPreds) {
    t = block_sum(preds, s_red);
    if (threadIdx.x == 0 && t) atomicAdd(&st->pred_arcs, t);
  }
}

// ADG-M's median (readings Q19-Q21): the ceil(|U|/2)-th
// smallest key (D[v] << 32) | v over U by a radix select, most significant
// digit first.  Only bits that can be nonzero are visited: the D field's
// bit length comes from the maximum degree, the id field's from n - 1, in
// digits of <= 12 bits (so R-MAT 24 needs 2 + 2 passes).  A pass is ONE
// kernel: every block histograms the keys that match the bits found so far
// (shared memory), adds it to the global histogram, and the last block to
// finish picks the digit holding the wanted rank and clears the histogram.
// Keys are distinct (the id is in the low word), so R = {v in U : key <=
// selected key} has exactly ceil(|U|/2) vertices: the first half of U in
// (D, id) order.
constexpr int kMselBits = 12;
constexpr int kMselBins = 1 << kMselBits;
__global__ void k_maxdeg(int64_t n, const int64_t* __restrict__ off, State* st) {
  int m = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)(off[v + 1] - off[v]));
  m = warp_max(m);
  if (lane_id() == 0 && m) atomicMax(&st->maxdeg, m);
}
// first == 2: the round's first pass bins min(D, kMselBins - 1) (the median's
// D is exact after one pass unless it is >= kMselBins - 1, which leaves the
// key undetermined for the digit passes); a digit pass whose bits are already
// determined returns at once.
__global__ void __launch_bounds__(1024) k_msel_pass(int first, int shift, int bits,
                                                    const int32_t* __restrict__ Uin,
                                                    const int32_t* __restrict__ D,
                                                    int32_t* __restrict__ hist, State* st) {
  __shared__ int sh[kMselBins];
  __shared__ long long s_w[32];
  __shared__ int s_last, s_digit;
  __shared__ long long s_before;
  if (st->done) return;
  const unsigned long long pkey = st->msel_key, pmask = st->msel_mask;
  const unsigned dmask = (1u << bits) - 1u;
  const bool clampD = first == 2;
  if (!clampD && ((pmask >> shift) & dmask) == dmask) return;  // digit known
  for (int i = threadIdx.x; i < kMselBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const long long nU = st->nU;
  for (long long i0 = blockIdx.x * (long long)blockDim.x; i0 < nU; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    int bin = -1;
    if (i < nU) {
      const int v = Uin ? Uin[i] : (int)i;
      const unsigned long long key = (((unsigned long long)(uint32_t)ld_i32_keep(D + v)) << 32) | (uint32_t)v;
      if (clampD) bin = (int)min((uint32_t)(key >> 32), (uint32_t)(kMselBins - 1));
      else if ((key & pmask) == pkey) bin = (int)((unsigned)(key >> shift) & dmask);
    }
    // degrees concentrate on few bins: one shared atomic per distinct bin per warp
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && lane_id() == __ffs(peers) - 1) atomicAdd(&sh[bin], __popc(peers));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMselBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&st->msel_done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  // last block: block scan of the histogram (4 bins per thread), the digit
  // whose inclusive count first reaches the rank; clear for the next pass
  __threadfence();
  const long long rank = first ? (nU + 1) / 2 : st->msel_rank;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  long long c4[4], tot = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c4[k] = __ldcg(hist + 4 * t + k);
    tot += c4[k];
  }
  long long incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
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
  }
  __syncthreads();
  long long before = s_w[warp] + incl - tot;  // keys in bins < 4t
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (before < rank && rank <= before + c4[k]) {
      s_digit = 4 * t + k;
      s_before = before;
    }
    before += c4[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) hist[4 * t + k] = 0;
  __syncthreads();
  if (t == 0) {
    if (clampD && s_digit == kMselBins - 1) {  // D >= kMselBins - 1: digit passes from scratch
      st->msel_key = 0;
      st->msel_mask = 0;
      st->msel_rank = rank;
    } else if (clampD) {                         // D = s_digit exactly
      st->msel_key = (unsigned long long)s_digit << 32;
      st->msel_mask = 0xffffffffull << 32;
      st->msel_rank = rank - s_before;
    } else {
      st->msel_key = pkey | ((unsigned long long)s_digit << shift);
      st->msel_mask = pmask | ((unsigned long long)dmask << shift);
      st->msel_rank = rank - s_before;
    }
    st->msel_done = 0;
  }
}
// before a round's first pass: nothing determined yet
__global__ void k_msel_reset(State* st) {
  st->msel_key = 0;
  st->msel_mask = 0;
  st->msel_done = 0;
}

// a2/a5: carry the cached degree sum and |U| to the next round (Q5 reading of
// PAPER.md:2359-2361), record statistics, detect termination.
// ord_cnt[l-1] = the non-isolated vertices of R_l (capacity cap): the
// priority order's round histogram, so the order needs no counting pass.
// Every round is checked against the exact integer form of Lemma 1's
// per-round shrink: the mean rule leaves
// n_{l+1} (den+num) < n_l den survivors (at most a 1/(1+eps) fraction); the
// median rule (ADG-M) exactly floor(n_l / 2).  A round that
// breaks it is a bug (err 7 -> PGC_EINTERNAL), which also bounds T by T0.
// (per_round keeps the first kMaxRoundStats rounds' (|U_l|, S_l, |R_l|): a
// diagnostic record, never read by the method.)
__global__ void k_adg_finalize(int l, int rule, uint32_t num, uint32_t den, State* st,
                               long long* per_round, int32_t* ord_cnt, int64_t cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st->done) return;
  const int nR = st->nR;
  if (nR == 0) {            // impossible for eps > 0 (Lemma 1): min degree <= mean
    st->err = 1;
    st->done = 1;
    return;
  }
  if (l - 1 < kMaxRoundStats) {
    per_round[3 * (l - 1) + 0] = st->nU;
    per_round[3 * (l - 1) + 1] = (long long)st->S;
    per_round[3 * (l - 1) + 2] = nR;
  }
  {  // the mean degree of G[U_l]: S_l = 2 |E[U_l]| (Q3); its maximum sizes the JP core
    const long long a = (long long)(st->S / (unsigned long long)(st->nU > 0 ? st->nU : 1));
    if (a > st->avg_max) st->avg_max = a;
  }
  st->sum_active += st->nU;
  st->cross += st->cut;
  if (l - 1 < cap) ord_cnt[l - 1] = st->nOrdR;
  st->nOrdR = 0;
  const long long nU1 = st->nU - nR;
  if (st->nUnext != nU1) st->err = 2;
  const bool shrink_ok =
      rule == kRuleMedian
          ? nU1 == st->nU / 2
          : (unsigned __int128)nU1 * ((unsigned long long)den + num) <
                (unsigned __int128)st->nU * den;
  if (!shrink_ok) st->err = 7;
  st->S = st->S - st->sumDR - st->cut;
  st->nU = nU1;
  st->T = l;
  st->rmax = l;
  st->sumDR = 0;
  st->cut = 0;
  st->nR = 0;
  st->nLight = 0;
  st->nUnext = 0;
  st->nChunks = 0;
  st->nExp = 0;
  if (nU1 == 0 || st->err) st->done = 1;
}

// T0 = min{t : (den+num)^t >= n den^t}, the exact round bound implied by
// Lemma 1's per-round shrink, for the host
// loop guard; ADG-M: floor(log2 n) + 1.  Exact: ceil(n (den/(den+num))^t)
// is tracked as a rational bound in 128-bit, rounding up at every step
// (each round leaves an integer count of survivors).
static long long round_bound(int64_t n, uint32_t num, uint32_t den, int rule) {
  if (n <= 0) return 0;
  if (rule == kRuleMedian) {
    long long t = 0;
    for (int64_t x = n; x > 0; x >>= 1) ++t;
    return t;
  }
  // survivors after t rounds <= s_t with s_0 = n, s_{t+1} = max integer s with
  // s (den+num) < s_t den, i.e. s_{t+1} = ceil(s_t den / (den+num)) - 1
  long long t = 0;
  unsigned __int128 s = (unsigned __int128)n;
  const unsigned __int128 a = den, b = (unsigned __int128)den + num;
  while (s > 0) {
    s = (s * a + b - 1) / b - 1;
    ++t;
  }
  return t;
}

// JP Part 1 work lists for an arbitrary key (pgc_jp_color): every vertex is
// classified, light ones into Rl, heavy ones into edge chunks; color[v] = 0
// (uncolored) except isolated vertices, settled as in
// k_adg_init (color 1, npred -1: outside the priority order).
__global__ void k_jp_classify(int64_t n, const int64_t* __restrict__ off, int4* __restrict__ lrec,
                              int4* __restrict__ chunks, int32_t* __restrict__ npred,
                              int32_t* __restrict__ color, State* st,
                              int heavy_deg, int chunk, int64_t chunk_cap) {
  __shared__ int sm[33];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {
    const long long i = base + threadIdx.x;
    const bool valid = i < n;
    bool light = false;
    int nch = 0;
    long long o = 0, deg = 0;
    if (valid) {
      const int v = (int)i;
      o = off[v];
      deg = off[v + 1] - o;
      light = deg > 0 && deg <= heavy_deg;
      if (deg > heavy_deg) {
        nch = (int)((deg + chunk - 1) / chunk);
        npred[v] = 0;
      }
      color[v] = deg == 0 ? 1 : 0;
      if (deg == 0) npred[v] = -1;
    }
    const int cb = block_reserve(nch, &st->nChunks, sm);
    if (nch) {
      if (cb + (long long)nch > chunk_cap) st->err = 3;
      else
        for (int k = 0; k < nch; ++k) {
          const long long s0 = o + (long long)k * chunk;
          const int len = (int)min((long long)chunk, o + deg - s0);
          chunks[2 * (cb + k)] = make_int4((int)i, len, (int)(uint32_t)s0, (int)(s0 >> 32));
          chunks[2 * (cb + k) + 1] = make_int4((int)(uint32_t)o, (int)(o >> 32), 0, 0);
        }
    }
    block_append_rec(light, light_rec((int)i, (int)deg, o), lrec, &st->nLight, sm);
  }
}

__global__ void k_state_reset_jp(State* st) {
  State s = {};
  s.rmin = 0x7fffffff;
  s.rmax = (int)0x80000000;
  *st = s;
}

static int grid_for(const Ctx& c, int per_sm) { return c.nsm * per_sm; }

template <int MODE>
static int launch_update(Ctx& c, const Arc<MODE>& A, const int32_t* Uin = nullptr) {
  const int GL = wave_grid(c, k_update_light<MODE>, 256);
  PGC_LAUNCH(c, kGUpdate, "k_update_light",
             k_update_light<MODE><<<GL, 256, 0, c.st>>>(A, c.col, c.lrec, c.npred, c.P, c.state));
  const int ratio = (MODE == 2 || MODE == 4) ? 0 : c.tune.filter_ratio;
  const int GH = wave_grid(c, k_update_heavy<MODE>, 256);
  PGC_LAUNCH(c, kGUpdate, "k_update_heavy",
             k_update_heavy<MODE><<<GH, 256, 0, c.st>>>(A, c.col, c.chunks, c.npred, c.P, c.state,
                                                        ratio));
  if constexpr (MODE != 2 && MODE != 4) {
    if (ratio > 0) {
      bool& attr = once_flag(c.dev, MODE);  // the attribute is per function AND device
      if (!attr) {
        PGC_CUDA(cudaFuncSetAttribute(k_update_heavy_f<MODE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kFilterSmem));
        attr = true;
      }
      PGC_LAUNCH(c, kGUpdate, "k_update_heavy_f",
                 k_update_heavy_f<MODE><<<c.nsm, kFilterThreads, kFilterSmem, c.st>>>(
                     A, c.col, c.chunks, c.filt, c.npred, c.P, c.state, ratio));
    }
  }
  return 0;
}

int adg_run(Ctx& c, uint32_t num, uint32_t den, uint64_t seed, int32_t* round, int mode,
            int32_t* color_zero, int rule) {
  NvtxRange nvtx_("pgc ADG (Alg. 1)");
  PGC_CHK_SIZES(c);
  const int B = 256;
  const int G = grid_for(c, 8);
  // mean rule: round 1's selection does init's per-vertex work (one pass less)
  const bool fuse_init = rule == kRuleMean && c.tune.fuse_init;
  // JP-ADG: keep the top rounds' vertex list for the split priority order
  const bool save_top = mode == kAdgFused && rule == kRuleMean && c.tune.jp_split_overlap &&
                        c.tune.core_max > 0 && c.tune.top_list;
  c.top_list = save_top;
  if (fuse_init)
    PGC_LAUNCH(c, kGAdgOther, "k_adg_state_init",
               k_adg_state_init<<<1, 1, 0, c.st>>>(c.n, c.nnz, c.state));
  else
    PGC_LAUNCH(c, kGAdgOther, "k_adg_init",
               k_adg_init<<<G, B, 0, c.st>>>(c.n, c.nnz, c.off, c.D, c.rs, round, color_zero,
                                             c.npred, c.tune.filter_ratio > 0 ? c.filt : nullptr,
                                             c.state));
  if (c.n == 0) return sync_state(c);
  int32_t* mhist = c.hist1;  // the order's histograms are free during ADG
  // ADG-M's radix schedule: (shift, bits) digits over the bits of (D << 32) | v
  // that can be nonzero (D < 2^bitlen(maxdeg), v < 2^bitlen(n-1))
  std::vector<std::pair<int, int>> digits;
  if (rule == kRuleMedian) {
    PGC_LAUNCH(c, kGAdgOther, "k_zero_i32", k_zero_i32<<<4, 512, 0, c.st>>>(mhist, kMselBins));
    PGC_LAUNCH(c, kGAdgOther, "k_maxdeg", k_maxdeg<<<grid_for(c, 8), 256, 0, c.st>>>(c.n, c.off, c.state));
    if (int e = sync_state(c)) return e;
    auto bitlen = [](long long x) { int b = 1; while (b < 62 && (1ll << b) <= x) ++b; return b; };
    const int dbits = bitlen(c.h_state->maxdeg), ibits = bitlen(c.n - 1);
    for (int hi = 32 + dbits; hi > 32; hi -= kMselBits) {
      const int lo = hi - kMselBits > 32 ? hi - kMselBits : 32;
      digits.push_back({lo, hi - lo});
    }
    for (int hi = ibits; hi > 0; hi -= kMselBits) {
      const int lo = hi - kMselBits > 0 ? hi - kMselBits : 0;
      digits.push_back({lo, hi - lo});
    }
  }
  int l = 1;
  const int batch = c.tune.rounds_per_sync < 1 ? 1 : c.tune.rounds_per_sync;
  const long long T0 = round_bound(c.n, num, den, rule);
  for (;;) {
    for (int j = 0; j < batch; ++j, ++l) {
      const int32_t* Uin = l == 1 ? nullptr : c.U[l & 1];
      int32_t* Uout = c.U[(l + 1) & 1];
      const int atom = l == 1 && c.tune.update_atom && (mode == kAdgOnly || mode == kAdgFused);
      if (rule == kRuleMedian) {
        PGC_LAUNCH(c, kGSelect, "k_msel_reset", k_msel_reset<<<1, 1, 0, c.st>>>(c.state));
        // the clamped-D pass first, then the digit passes (those of D return
        // at once when the clamped pass fixed D)
        PGC_LAUNCH(c, kGSelect, "k_msel_pass",
                   k_msel_pass<<<c.nsm * 2, 1024, 0, c.st>>>(2, 32, kMselBits, Uin, c.D, mhist,
                                                            c.state));
        for (size_t p = 0; p < digits.size(); ++p)
          PGC_LAUNCH(c, kGSelect, "k_msel_pass",
                     k_msel_pass<<<c.nsm * 2, 1024, 0, c.st>>>(0, digits[p].first,
                                                              digits[p].second, Uin, c.D, mhist,
                                                              c.state));
      }
      PGC_LAUNCH(c, kGSelect, "k_adg_select",
                 k_adg_select<<<G, B, 0, c.st>>>(l, rule, num, den, c.off, c.D, round, c.rs, Uin, Uout,
                                                 c.lrec, c.chunks, c.npred, c.state,
                                                 c.tune.heavy_degree, c.tune.chunk_arcs,
                                                 c.lay.chunk_cap, mode == kAdgPull, atom,
                                                 fuse_init && l == 1, color_zero,
                                                 c.tune.filter_ratio > 0 ? c.filt : nullptr,
                                                 c.cexp));
      if (l == 1 && c.col_ready) PGC_CUDA(cudaStreamWaitEvent(c.st, c.col_ready, 0));
      PGC_LAUNCH(c, kGUpdate, "k_round_aux",
                 k_round_aux<<<c.nsm * 2, 1024, 0, c.st>>>(
                     l, Uin, c.tune.filter_ratio > 0 && mode != kAdgPull ? c.filt : nullptr, c.state,
                     c.tune.filter_ratio, save_top ? c.Rl : nullptr, core_reach(c.tune), c.chunks,
                     c.cexp, c.tune.chunk_arcs));
      if (mode == kAdgFused) {
        if (int e = launch_update(c, Arc<1>{l, seed, round, c.D, c.rs, atom}, Uin)) return e;
      } else if (mode == kAdgFusedO) {
        if (int e = launch_update(c, Arc<3>{l, seed, round, c.D, c.rs}, Uin)) return e;
      } else if (mode == kAdgPull) {
        if (int e = launch_update(c, Arc<4>{l, seed, round, c.D, c.rs}, Uin)) return e;
      } else {
        if (int e = launch_update(c, Arc<0>{l, seed, round, c.D, c.rs, atom}, Uin)) return e;
      }
      PGC_LAUNCH(c, kGAdgOther, "k_adg_finalize",
                 k_adg_finalize<<<1, 32, 0, c.st>>>(l, rule, num, den, c.state, c.per_round,
                                                    c.hist1 + c.lay.range_cap, c.lay.range_cap));
    }
    if (int e = sync_state(c)) return e;
    if (c.h_state->err == 7)
      return fail(4, "ADG round %d broke Lemma 1's per-round shrink (PAPER.md:761-771)", c.h_state->T);
    if (c.h_state->err) return fail(4, "ADG internal invariant failed (code %d)", c.h_state->err);
    if (c.h_state->done) break;
    if ((long long)l - 1 >= T0)  // rounds 1..l-1 ran, U is not empty: T > T0
      return fail(4, "ADG did not terminate within T0 = %lld rounds (Lemma 1)", T0);
  }
  return 0;
}

// ADG-O's priority as one int32 key per vertex for the order: key1[v] =
// goff[round[v]] + D_rem[v], goff[r] = sum over earlier rounds r' of
// (max D_rem in r' + 1); with the id as the second key (Key2::idkey) the
// order is (round, D_rem, id) descending = rho_ADG-O descending (Q22).
__global__ void k_o_dmax(int64_t n, const int32_t* __restrict__ round, const int32_t* __restrict__ D,
                         int32_t* __restrict__ dmaxr) {
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x; v0 < n; v0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = v0 + threadIdx.x;
    const int r = v < n ? round[v] : -1;
    const int d = v < n ? D[v] : 0;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    const int dm = __reduce_max_sync(peers, d);
    if (r >= 0 && lane_id() == __ffs(peers) - 1) atomicMax(&dmaxr[r], dm);
  }
}
// one block: goff[r] = exclusive prefix of (dmaxr[r] + 1) over r = 1..T
__global__ void __launch_bounds__(1024) k_o_goff(int T, const int32_t* __restrict__ dmaxr,
                                                 int32_t* __restrict__ goff, State* st) {
  __shared__ long long s_w[32];
  __shared__ long long s_carry;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_carry = 0;
  __syncthreads();
  for (int r0 = 1; r0 <= T; r0 += 1024) {
    const int r = r0 + t;
    const long long x = r <= T ? (long long)dmaxr[r] + 1 : 0;
    long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
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
    }
    __syncthreads();
    const long long ex = s_carry + s_w[warp] + incl - x;
    if (r <= T) goff[r] = ex > 0x7fffffffLL ? 0x7fffffff : (int)ex;
    __syncthreads();
    if (t == 1023) s_carry = ex + x;
    __syncthreads();
  }
  if (t == 0 && s_carry > 0x7fffffffLL) st->err = 6;  // key range does not fit int32
}
__global__ void k_o_key(int64_t n, const int32_t* __restrict__ round, const int32_t* __restrict__ D,
                        const int32_t* __restrict__ goff, int32_t* __restrict__ key1) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    key1[v] = goff[round[v]] + D[v];
}

int adg_o_keys(Ctx& c, const int32_t* round, int32_t* key1) {
  PGC_CHK_SIZES(c);
  const int T = c.h_state->T;
  if (c.n == 0) return 0;
  // the order's histogram space (2(n + 65536) ints >= 2(T + 2)) is free until jp_order_run
  int32_t* dmaxr = c.hist1;
  int32_t* goff = c.hist1 + T + 2;
  const int G = grid_for(c, 8);
  PGC_LAUNCH(c, kGOrder, "k_zero_i32", k_zero_i32<<<G, 256, 0, c.st>>>(dmaxr, (int64_t)T + 2));
  PGC_LAUNCH(c, kGOrder, "k_o_dmax", k_o_dmax<<<G, 256, 0, c.st>>>(c.n, round, c.D, dmaxr));
  PGC_LAUNCH(c, kGOrder, "k_o_goff", k_o_goff<<<1, 1024, 0, c.st>>>(T, dmaxr, goff, c.state));
  PGC_LAUNCH(c, kGOrder, "k_o_key", k_o_key<<<G, 256, 0, c.st>>>(c.n, round, c.D, goff, key1));
  return 0;
}

// JP baseline first keys: FF = natural order (-v), LF =
// degree, LLF = ceil(log2 deg) (deg 0 -> 0: isolated vertices are outside
// the order anyway), R = constant (the hash alone).
__global__ void k_baseline_key(int64_t n, const int64_t* __restrict__ off, int kind,
                               int32_t* __restrict__ key) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = off[v + 1] - off[v];
    int k = 0;
    if (kind == 1) k = -(int)v;
    else if (kind == 2) k = (int)d;
    else if (kind == 3) k = d <= 1 ? 0 : 64 - __clzll((unsigned long long)(d - 1));  // ceil(log2 d)
    key[v] = k;
  }
}

int baseline_key_run(Ctx& c, int kind, int32_t* key) {
  PGC_CHK_SIZES(c);
  if (c.n == 0) return 0;
  PGC_LAUNCH(c, kGAdgOther, "k_baseline_key",
             k_baseline_key<<<grid_for(c, 8), 256, 0, c.st>>>(c.n, c.off, kind, key));
  return 0;
}

int jp_setup_run(Ctx& c, const int32_t* round, uint64_t seed, int32_t* color) {
  NvtxRange nvtx_("pgc JP Part 1");
  PGC_CHK_SIZES(c);
  const int G = grid_for(c, 8);
  PGC_LAUNCH(c, kGAdgOther, "k_state_reset_jp", k_state_reset_jp<<<1, 1, 0, c.st>>>(c.state));
  if (c.n == 0) return 0;
  PGC_LAUNCH(c, kGUpdate, "k_jp_classify",
             k_jp_classify<<<G, 256, 0, c.st>>>(c.n, c.off, c.lrec, c.chunks, c.npred, color,
                                                c.state,
                                                c.tune.heavy_degree, c.tune.chunk_arcs,
                                                c.lay.chunk_cap));
  return launch_update(c, Arc<2>{0, seed, round, nullptr, nullptr});
}

}  // namespace pgc
