// jp.cu -- Jones-Plassmann coloring (Algorithm 3) for the
// priority rho = <round, splitmix64(seed ^ v)>.
//
// JP Part 1 (pred[v], count[v] = |pred[v]|, lines 1116-1121) is produced by
// ADG's fused UPDATE (adg.cu) or by jp_setup_run: pred(v) lives in v's own
// CSR slot P[off[v] .. off[v] + npred[v]).
//
// JP Part 2 runs as a sync-free dataflow instead of level-synchronous
// frontiers: vertices are placed in one priority order (a topological order
// of the DAG G_rho) and handed to warps by an atomic
// ticket; a vertex is colored by GetColor (1135-1138) as soon as every
// predecessor's color is nonzero -- the Join of line 1132 observed by polling
// the predecessor's color instead of decrementing a counter.  Deadlock
// freedom: tickets are taken in priority order and a warp never blocks, so the
// highest-priority uncolored vertex always belongs to a running warp whose
// predecessors are all colored.
//
// Priority order = stable two-level bucket sort by key
//   (class, round desc, h desc), class 0 = |pred| > kLightPredMax ("heavy").
// Both classes are priority-ordered; heavy vertices are colored warp-per-
// vertex (bitmap windows in shared memory), light ones lane-per-vertex (a
// 64-bit used-color mask in registers).
#include <climits>
#include <cstdio>

#include "pgc_internal.cuh"

namespace pgc {

// ------------------------------------------------------------- scan ---------
__global__ void k_scan_reduce(const int32_t* __restrict__ in, const int* len_ptr, int64_t len_h,
                              int32_t* __restrict__ tmp) {
  __shared__ int sm[32];
  const int64_t len = len_h >= 0 ? len_h : (int64_t)*len_ptr;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  int s = 0;
  if (t0 < len) {
    for (int k = threadIdx.x; k < kScanTile; k += blockDim.x) {
      const int64_t i = t0 + k;
      if (i < len) s += in[i];
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    int x = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0;
    x = warp_sum(x);
    if (threadIdx.x == 0) tmp[blockIdx.x] = x;
  }
}

// single block: exclusive scan of tmp[0..ntiles), writes total to out[len] and *total
__global__ void k_scan_tmp(int32_t* __restrict__ tmp, int64_t ntiles_cap, const int* len_ptr,
                           int64_t len_h, int32_t* __restrict__ out, int* total_out) {
  __shared__ int sm[32];
  __shared__ int carry;
  const int64_t len = len_h >= 0 ? len_h : (int64_t)*len_ptr;
  const int64_t ntiles = (len + kScanTile - 1) / kScanTile;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t b0 = 0; b0 < ntiles && b0 < ntiles_cap; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const int x = i < ntiles ? tmp[i] : 0;
    int incl = x;
    for (int s = 1; s < 32; s <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, s);
      if (lane >= s) incl += y;
    }
    if (lane == 31) sm[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? sm[lane] : 0;
      int wi = w;
      for (int s = 1; s < 32; s <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, wi, s);
        if (lane >= s) wi += y;
      }
      if (lane < nw) sm[lane] = wi - w;
    }
    __syncthreads();
    const int c0 = carry;
    if (i < ntiles) tmp[i] = c0 + sm[warp] + incl - x;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c0 + sm[warp] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[len] = carry;
    if (total_out) *total_out = carry;
  }
}

__global__ void __launch_bounds__(1024) k_scan_down(const int32_t* in, const int* len_ptr,
                                                    int64_t len_h, const int32_t* __restrict__ tmp,
                                                    int32_t* out) {
  __shared__ int sm[32];
  const int64_t len = len_h >= 0 ? len_h : (int64_t)*len_ptr;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  if (t0 >= len) return;
  constexpr int PER = kScanTile / 1024;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int v[PER];
  int s = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int64_t i = t0 + threadIdx.x * PER + k;
    v[k] = i < len ? in[i] : 0;
    s += v[k];
  }
  int incl = s;
  for (int d = 1; d < 32; d <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = sm[lane];
    int wi = w;
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += y;
    }
    sm[lane] = wi - w;
  }
  __syncthreads();
  int run = tmp[blockIdx.x] + sm[warp] + incl - s;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int64_t i = t0 + threadIdx.x * PER + k;
    if (i < len) out[i] = run;
    run += v[k];
  }
}

static int scan_ex(Ctx& c, const int32_t* in, int32_t* out, const int* len_ptr, int64_t len_h,
                   int64_t cap, int* total_out) {
  const int64_t ntiles_cap = (cap + kScanTile - 1) / kScanTile + 1;
  if (ntiles_cap > c.lay.scan_tmp_cap) return fail(4, "scan temp too small");
  const int64_t grid = len_h >= 0 ? (len_h + kScanTile - 1) / kScanTile : ntiles_cap;
  if (grid > 0)
    PGC_LAUNCH(c, kGOrder, "k_scan_reduce",
               k_scan_reduce<<<(unsigned)grid, 256, 0, c.st>>>(in, len_ptr, len_h, c.scan_tmp));
  PGC_LAUNCH(c, kGOrder, "k_scan_tmp",
             k_scan_tmp<<<1, 1024, 0, c.st>>>(c.scan_tmp, ntiles_cap, len_ptr, len_h, out, total_out));
  if (grid > 0)
    PGC_LAUNCH(c, kGOrder, "k_scan_down",
               k_scan_down<<<(unsigned)grid, 1024, 0, c.st>>>(in, len_ptr, len_h, c.scan_tmp, out));
  return 0;
}

// ------------------------------------------------------------- order --------
__global__ void k_key_range(int64_t n, const int32_t* __restrict__ round, State* st) {
  int mn = INT_MAX, mx = INT_MIN;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int r = round[v];
    mn = min(mn, r);
    mx = max(mx, r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->rmin, mn);
    atomicMax(&st->rmax, mx);
  }
}

__device__ __forceinline__ int key_index(int cls, int r, int rmax, int range) {
  return cls * range + (rmax - r);  // class-major, then round descending
}
__device__ __forceinline__ int bucket_count_for(int cnt) {
  if (cnt <= 0) return 0;
  int want = (cnt + kBucketTarget - 1) / kBucketTarget;
  int b = 1;
  while (b < want) b <<= 1;
  return b;
}

// hist1[key index] += 1; privatised in shared memory when the key range is small.
__global__ void k_hist1(int64_t n, const int32_t* __restrict__ round,
                        const int32_t* __restrict__ npred, const State* st, int range,
                        int32_t* __restrict__ hist1, int* nheavy) {
  extern __shared__ int sh[];
  const int rmax = st->rmax;
  const int L = 2 * range;
  const bool priv = L <= 8192;
  if (priv)
    for (int i = threadIdx.x; i < L; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  int heavy = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int cls = npred[v] > kLightPredMax ? 0 : 1;
    heavy += 1 - cls;
    const int k = key_index(cls, round[v], rmax, range);
    if (priv) atomicAdd(&sh[k], 1);
    else atomicAdd(&hist1[k], 1);
  }
  heavy = warp_sum(heavy);
  if ((threadIdx.x & 31) == 0 && heavy) atomicAdd(nheavy, heavy);
  __syncthreads();
  if (priv)
    for (int i = threadIdx.x; i < L; i += blockDim.x)
      if (sh[i]) atomicAdd(&hist1[i], sh[i]);
}

__global__ void k_bucket_sizes(int L, const int32_t* __restrict__ hist1, int32_t* __restrict__ bsz) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x)
    bsz[i] = bucket_count_for(hist1[i]);
}

__device__ __forceinline__ int bucket_of(int v, int r, int cls, uint64_t seed, int rmax, int range,
                                         const int32_t* __restrict__ hist1,
                                         const int32_t* __restrict__ base1) {
  const int k = key_index(cls, r, rmax, range);
  const int B = bucket_count_for(hist1[k]);
  const int lg = 31 - __clz(B);
  const uint64_t h = prio_hash(seed, (uint32_t)v);
  const int hb = lg ? (int)(h >> (64 - lg)) : 0;
  return base1[k] + (B - 1 - hb);  // larger hash -> earlier bucket
}

__global__ void k_hist2(int64_t n, const int32_t* __restrict__ round,
                        const int32_t* __restrict__ npred, uint64_t seed, const State* st,
                        int range, const int32_t* __restrict__ hist1,
                        const int32_t* __restrict__ base1, int32_t* __restrict__ bcnt) {
  const int rmax = st->rmax;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int cls = npred[v] > kLightPredMax ? 0 : 1;
    const int b = bucket_of((int)v, round[v], cls, seed, rmax, range, hist1, base1);
    atomicAdd(&bcnt[b], 1);
  }
}

__global__ void k_scatter(int64_t n, const int32_t* __restrict__ round,
                          const int32_t* __restrict__ npred, uint64_t seed, const State* st,
                          int range, const int32_t* __restrict__ hist1,
                          const int32_t* __restrict__ base1, int32_t* __restrict__ bcnt,
                          const int32_t* __restrict__ bstart, int32_t* __restrict__ order) {
  const int rmax = st->rmax;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int cls = npred[v] > kLightPredMax ? 0 : 1;
    const int b = bucket_of((int)v, round[v], cls, seed, rmax, range, hist1, base1);
    const int pos = bstart[b] + atomicSub(&bcnt[b], 1) - 1;
    order[pos] = (int)v;
  }
}

// Sort every bucket by h descending (bucket = same class and round, same top
// hash bits).  One lane per bucket (insertion sort in registers, <= 16
// entries, the common case at mean occupancy 4..8); larger buckets are
// ranked by a whole warp afterwards.
constexpr int kLaneSortMax = 16;
__global__ void k_bucket_sort(const State* st, const int32_t* __restrict__ bstart,
                              int32_t* __restrict__ order, uint64_t seed) {
  const int lane = lane_id();
  const int nb = st->nbuckets;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = gridDim.x * blockDim.x;
  for (int b0 = tid - lane; b0 < nb; b0 += nthreads) {
    const int b = b0 + lane;
    int s0 = 0, s = 0;
    if (b < nb) {
      s0 = bstart[b];
      s = bstart[b + 1] - s0;
    }
    if (s >= 2 && s <= kLaneSortMax) {
      int vv[kLaneSortMax];
      uint64_t hh[kLaneSortMax];
#pragma unroll
      for (int i = 0; i < kLaneSortMax; ++i)
        if (i < s) {
          vv[i] = order[s0 + i];
          hh[i] = prio_hash(seed, (uint32_t)vv[i]);
        }
#pragma unroll
      for (int i = 1; i < kLaneSortMax; ++i) {
        if (i < s) {
          const int x = vv[i];
          const uint64_t hx = hh[i];
          int j = i - 1;
#pragma unroll
          for (int k = kLaneSortMax - 2; k >= 0; --k) {  // shift larger-priority-later entries
            if (k <= j && k < i && hh[k] < hx) {
              hh[k + 1] = hh[k];
              vv[k + 1] = vv[k];
              hh[k] = hx;
              vv[k] = x;
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kLaneSortMax; ++i)
        if (i < s) order[s0 + i] = vv[i];
    }
    // rare large buckets: the whole warp ranks them, one bucket at a time
    unsigned big = __ballot_sync(0xffffffffu, s > kLaneSortMax);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int bs0 = __shfl_sync(0xffffffffu, s0, src);
      const int bs = __shfl_sync(0xffffffffu, s, src);
      if (bs <= 32) {
        const int v = lane < bs ? order[bs0 + lane] : 0;
        const uint64_t h = lane < bs ? prio_hash(seed, (uint32_t)v) : 0;
        int rank = 0;
        for (int j = 0; j < bs; ++j) rank += __shfl_sync(0xffffffffu, h, j) > h;
        __syncwarp();
        if (lane < bs) order[bs0 + rank] = v;
        __syncwarp();
      } else if (lane == 0) {  // very rare: insertion sort in place
        for (int i = 1; i < bs; ++i) {
          const int x = order[bs0 + i];
          const uint64_t hx = prio_hash(seed, (uint32_t)x);
          int j = i - 1;
          while (j >= 0 && prio_hash(seed, (uint32_t)order[bs0 + j]) < hx) {
            order[bs0 + j + 1] = order[bs0 + j];
            --j;
          }
          order[bs0 + j + 1] = x;
        }
      }
      __syncwarp();
    }
  }
}

__global__ void k_order_setup(State* st, int rmax_host, int use_host) {
  if (use_host) {
    st->rmin = 1;
    st->rmax = rmax_host;
  }
  st->nheavy = 0;
  st->nbuckets = 0;
  st->sorted = 0;
}

int jp_order_run(Ctx& c, const int32_t* round, uint64_t seed, bool range_known) {
  const int G = c.nsm * 8;
  if (c.n == 0) return 0;
  int rmin, rmax;
  if (range_known) {
    rmin = 1;
    rmax = c.h_state->T;
    PGC_LAUNCH(c, kGOrder, "k_order_setup", k_order_setup<<<1, 1, 0, c.st>>>(c.state, rmax, 1));
  } else {
    PGC_LAUNCH(c, kGOrder, "k_key_range", k_key_range<<<G, 256, 0, c.st>>>(c.n, round, c.state));
    PGC_LAUNCH(c, kGOrder, "k_order_setup", k_order_setup<<<1, 1, 0, c.st>>>(c.state, 0, 0));
    if (int e = sync_state(c)) return e;
    rmin = c.h_state->rmin;
    rmax = c.h_state->rmax;
  }
  const int64_t range = (int64_t)rmax - rmin + 1;
  if (range < 1 || range > c.lay.range_cap)
    return fail(1, "round[] value range %lld exceeds n + 65536", (long long)range);
  const int L = (int)(2 * range);
  PGC_LAUNCH(c, kGOrder, "k_zero_i32", k_zero_i32<<<G, 256, 0, c.st>>>(c.hist1, L));
  const size_t shb = L <= 8192 ? (size_t)L * sizeof(int) : 0;
  PGC_LAUNCH(c, kGOrder, "k_hist1",
             k_hist1<<<G, 256, shb, c.st>>>(c.n, round, c.npred, c.state, (int)range, c.hist1,
                                            &c.state->nheavy));
  PGC_LAUNCH(c, kGOrder, "k_bucket_sizes",
             k_bucket_sizes<<<G, 256, 0, c.st>>>(L, c.hist1, c.base1));
  if (int e = scan_ex(c, c.base1, c.base1, nullptr, L, L, &c.state->nbuckets)) return e;
  PGC_LAUNCH(c, kGOrder, "k_zero_i32_dev",
             k_zero_i32_dev<<<G, 256, 0, c.st>>>(c.bcnt, &c.state->nbuckets, 1));
  PGC_LAUNCH(c, kGOrder, "k_hist2",
             k_hist2<<<G, 256, 0, c.st>>>(c.n, round, c.npred, seed, c.state, (int)range, c.hist1,
                                          c.base1, c.bcnt));
  if (int e = scan_ex(c, c.bcnt, c.bstart, &c.state->nbuckets, -1, c.lay.nb_cap,
                      &c.state->sorted))
    return e;
  PGC_LAUNCH(c, kGOrder, "k_scatter",
             k_scatter<<<G, 256, 0, c.st>>>(c.n, round, c.npred, seed, c.state, (int)range, c.hist1,
                                            c.base1, c.bcnt, c.bstart, c.order));
  PGC_LAUNCH(c, kGOrder, "k_bucket_sort",
             k_bucket_sort<<<G, 256, 0, c.st>>>(c.state, c.bstart, c.order, seed));
  return 0;
}

// ------------------------------------------------------------- color --------
constexpr int kJpBlock = 256;
constexpr int kJpWarps = kJpBlock / 32;
constexpr int kPendCap = 256;          // pending-pred list capacity per heavy warp (smem)
constexpr int kLightBatch = 8;         // pred loads in flight per light lane

// OR color cc into the window bitmap (colors wbase+1 .. wbase+kHeavyWin).
__device__ __forceinline__ void bm_set(unsigned* bm, int cc, int wbase) {
  if (cc > wbase && cc <= wbase + kHeavyWin) {
    const int bit = cc - wbase - 1;
    atomicOr(&bm[bit >> 5], 1u << (bit & 31));
  }
}

__device__ __forceinline__ int vload(const int* p) { return *(volatile const int*)p; }

// Watchdog: a JP kernel running past its budget reports a stall (st->err = 5)
// instead of hanging the device.  Idle spin iterations check only the local
// %globaltimer (no memory traffic on the polling path).
__device__ __forceinline__ bool stalled(State* st, unsigned long long deadline) {
  if (globaltimer() > deadline) {
    st->err = 5;
    return true;
  }
  return false;
}

// Heavy path, one warp per vertex: examine preds [from, np) in strips of 4x32
// (4 independent loads in flight per lane), OR colored ones into the window,
// queue pending ones in the warp's list.  Returns the index to resume from when
// the pending list is full, np when every pred was examined.
__device__ __forceinline__ int heavy_scan(const int32_t* __restrict__ P, int64_t pb, int np,
                                          int from, const int32_t* color, unsigned* bm, int wbase,
                                          int* plist, int& npend) {
  const int lane = lane_id();
  for (int i0 = from; i0 < np; i0 += 128) {
    int u[4], cc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + 32 * k + lane;
      u[k] = i < np ? __ldg(P + pb + i) : -1;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) cc[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool pend = u[k] >= 0 && cc[k] == 0;
      if (u[k] >= 0 && cc[k]) bm_set(bm, cc[k], wbase);
      const unsigned bal = __ballot_sync(0xffffffffu, pend);
      const int cnt = __popc(bal);
      if (npend + cnt > kPendCap) return i0 + 32 * k;  // strips before k are complete
      if (pend) plist[npend + __popc(bal & lanemask_lt())] = u[k];
      npend += cnt;
    }
  }
  return np;
}

__global__ void __launch_bounds__(kJpBlock) k_jp_color(int64_t n, const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ P,
                                                      const int32_t* __restrict__ npred,
                                                      const int32_t* __restrict__ order,
                                                      int32_t* color, State* st,
                                                      int heavy_warps,
                                                      unsigned heavy_sleep_max,
                                                      unsigned light_sleep_max,
                                                      unsigned long long* tr_grab,
                                                      unsigned long long* tr_done,
                                                      unsigned long long watchdog_ns) {
  const unsigned long long deadline = globaltimer() + watchdog_ns;
  // heavy-warp state: window bitmap + pending preds, per warp
  __shared__ unsigned s_bm[kJpWarps][kHeavyWin / 32];
  __shared__ int s_pend[kJpWarps][kPendCap];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int nheavy = st->nheavy;
  int kmax = 0;
  if (warp < heavy_warps) {
    unsigned* bm = s_bm[warp];
    int* plist = s_pend[warp];
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&st->ticket_heavy, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= nheavy) break;
      const int v = order[t];
      const int np = npred[v];
      const int64_t pb = off[v];
      if (tr_grab && lane == 0) tr_grab[v] = globaltimer();
      int found = 0;
      for (int wbase = 0; !found; wbase += kHeavyWin) {
        bm[lane] = 0;
        bm[lane + 32] = 0;
        __syncwarp();
        int npend = 0;
        int over = heavy_scan(P, pb, np, 0, color, bm, wbase, plist, npend);
        // poll the pending preds until every one is colored (never blocks: a
        // pass either makes progress or sleeps briefly and retries)
        unsigned sleep_ns = 16;
        while (npend > 0 || over < np) {
          bool progress = false;
          int keep = 0;
          for (int j0 = 0; j0 < npend; j0 += 32) {
            const int j = j0 + lane;
            int u = 0, cc = 1;
            if (j < npend) {
              u = plist[j];
              cc = ld_relaxed(color + u);
            }
            const bool still = j < npend && cc == 0;
            if (j < npend && cc) bm_set(bm, cc, wbase);
            const unsigned bal = __ballot_sync(0xffffffffu, still);
            if (__ballot_sync(0xffffffffu, j < npend && cc != 0)) progress = true;
            __syncwarp();
            if (still) plist[keep + __popc(bal & lanemask_lt())] = u;
            keep += __popc(bal);
          }
          npend = keep;
          __syncwarp();
          if (over < np) {
            const int before = over;
            over = heavy_scan(P, pb, np, over, color, bm, wbase, plist, npend);
            if (over != before) progress = true;
          }
          if (npend == 0 && over >= np) break;
          if (progress) {
            sleep_ns = 16;
          } else {
            if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) {
              found = -1;
              break;
            }
            __nanosleep(sleep_ns);
            sleep_ns = min(sleep_ns * 2, heavy_sleep_max);
          }
        }
        __syncwarp();
        if (found < 0) break;  // stalled (watchdog)
        // GetColor inside this window: the first zero bit
        const unsigned z0 = ~bm[lane], z1 = ~bm[lane + 32];
        const unsigned b0 = __ballot_sync(0xffffffffu, z0 != 0);
        const unsigned b1 = __ballot_sync(0xffffffffu, z1 != 0);
        if (b0) {
          const int w = __ffs(b0) - 1;
          const unsigned z = __shfl_sync(0xffffffffu, z0, w);
          found = wbase + 32 * w + __ffs(z);
        } else if (b1) {
          const int w = __ffs(b1) - 1;
          const unsigned z = __shfl_sync(0xffffffffu, z1, w);
          found = wbase + 32 * (w + 32) + __ffs(z);
        }
        __syncwarp();
      }
      if (found < 0) break;  // stalled: the host reports PGC_EINTERNAL
      if (lane == 0) {
        st_relaxed(color + v, found);
        if (tr_done) tr_done[v] = globaltimer();
      }
      kmax = max(kmax, found);
    }
  } else {
    const int64_t nlight = n - nheavy;
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&st->ticket_light, 32);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= nlight || globaltimer() > deadline) break;
      const int64_t pos = nheavy + (int64_t)t + lane;
      const bool valid = pos < n;
      int v = 0, np = 0;
      int64_t pb = 0;
      unsigned long long mask = 1ull;  // used colors; bit 0 reserved (colors start at 1)
      unsigned long long pend = 0ull;  // indices of preds still uncolored (np <= 62)
      if (valid) {
        v = order[pos];
        np = npred[v];
        pb = off[v];
        if (tr_grab) tr_grab[v] = globaltimer();
      }
      // first pass over every pred, kLightBatch loads in flight
      for (int j0 = 0; j0 < np; j0 += kLightBatch) {
        int u[kLightBatch], cc[kLightBatch];
#pragma unroll
        for (int k = 0; k < kLightBatch; ++k) u[k] = j0 + k < np ? __ldg(P + pb + j0 + k) : -1;
#pragma unroll
        for (int k = 0; k < kLightBatch; ++k) cc[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 1;
#pragma unroll
        for (int k = 0; k < kLightBatch; ++k) {
          if (u[k] < 0) continue;
          if (cc[k] == 0) pend |= 1ull << (j0 + k);
          else if (cc[k] < 64) mask |= 1ull << cc[k];
        }
      }
      // Waiting: each lane watches ONE pending pred (its lowest pending index)
      // with a single load per poll; only when the watched pred is colored does
      // it re-examine the remaining pending preds in one batched pass.
      int watch_j = pend ? __ffsll((long long)pend) - 1 : -1;
      int watch_u = watch_j >= 0 ? __ldg(P + pb + watch_j) : -1;
      bool done = !valid;
      unsigned sleep_ns = 32;
      for (;;) {
        bool progress = false;
        if (!done && watch_u >= 0) {
          const int cw = ld_relaxed(color + watch_u);
          if (cw) {
            if (cw < 64) mask |= 1ull << cw;
            pend &= ~(1ull << watch_j);
            progress = true;
            // batched re-poll of the other pending preds
            unsigned long long p = pend;
            while (p) {
              int js[kLightBatch], u[kLightBatch], cc[kLightBatch];
#pragma unroll
              for (int k = 0; k < kLightBatch; ++k) {
                js[k] = p ? __ffsll((long long)p) - 1 : -1;
                p &= p - 1;
              }
#pragma unroll
              for (int k = 0; k < kLightBatch; ++k) u[k] = js[k] >= 0 ? __ldg(P + pb + js[k]) : -1;
#pragma unroll
              for (int k = 0; k < kLightBatch; ++k) cc[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 0;
#pragma unroll
              for (int k = 0; k < kLightBatch; ++k)
                if (cc[k]) {
                  if (cc[k] < 64) mask |= 1ull << cc[k];
                  pend &= ~(1ull << js[k]);
                }
            }
            watch_j = pend ? __ffsll((long long)pend) - 1 : -1;
            watch_u = watch_j >= 0 ? __ldg(P + pb + watch_j) : -1;
          }
        }
        if (!done && watch_u < 0) {  // GetColor: smallest color unused by the preds
          const int cc = __ffsll((long long)~mask) - 1;
          st_relaxed(color + v, cc);
          if (tr_done) tr_done[v] = globaltimer();
          kmax = max(kmax, cc);
          done = true;
          progress = true;
        }
        if (__ballot_sync(0xffffffffu, !done) == 0) break;
        if (__ballot_sync(0xffffffffu, progress)) {
          sleep_ns = 32;
        } else {
          if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) break;
          __nanosleep(sleep_ns);
          sleep_ns = min(sleep_ns * 2, light_sleep_max);
        }
      }
    }
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&st->K, kmax);
}

__global__ void k_jp_reset(State* st) {
  st->ticket_heavy = 0;
  st->ticket_light = 0;
  st->K = 0;
}

int jp_color_run(Ctx& c, int32_t* color) {
  PGC_LAUNCH(c, kGJp, "k_jp_reset", k_jp_reset<<<1, 1, 0, c.st>>>(c.state));
  if (c.n > 0) {
    static thread_local int occ = 0;
    if (occ == 0) {
      PGC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_jp_color, kJpBlock, 0));
      if (occ < 1) occ = 1;
    }
    PGC_LAUNCH(c, kGJp, "k_jp_color",
               k_jp_color<<<c.nsm * occ, kJpBlock, 0, c.st>>>(
                   c.n, c.off, c.P, c.npred, c.order, color, c.state, c.tune.jp_heavy_warps,
                   (unsigned)c.tune.jp_heavy_sleep_max, (unsigned)c.tune.jp_light_sleep_max,
                   c.trace_grab, c.trace_done, (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull));
  }
  if (int e = sync_state(c)) return e;
  if (c.h_state->err == 5)
    return fail(4, "JP coloring stalled: no progress within %d ms (watchdog)", c.tune.jp_watchdog_ms);
  if (c.n > 0 && c.h_state->sorted != c.n)
    return fail(4, "priority order placed %d of %lld vertices", c.h_state->sorted,
                (long long)c.n);
  return 0;
}

// ------------------------------------------------------------- check --------
__global__ void k_check_graph(int64_t n, int64_t nnz, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ col, unsigned long long* bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = off[v], b = off[v + 1];
    bool ok = a >= 0 && b >= a && b <= nnz && (v > 0 || a == 0) && (v < n - 1 || b == nnz);
    for (int64_t e = a; ok && e < b; ++e) {
      const int u = col[e];
      if (u < 0 || u >= n || u == v || (e > a && col[e - 1] >= u)) {
        ok = false;
        break;
      }
      // symmetry: v must appear in N(u) (binary search in the sorted row)
      int64_t lo = off[u], hi = off[u + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < v) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= off[u + 1] || col[lo] != v) ok = false;
    }
    if (!ok) atomicMin(bad, (unsigned long long)v);
  }
}

int check_graph_run(Ctx& c, int64_t* bad_vertex) {
  unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(&c.state->S);
  PGC_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), c.st));
  if (c.n > 0)
    PGC_LAUNCH(c, kGAdgOther, "k_check_graph",
               k_check_graph<<<c.nsm * 8, 256, 0, c.st>>>(c.n, c.nnz, c.off, c.col, d_bad));
  if (int e = sync_state(c)) return e;
  const unsigned long long h = c.h_state->S;
  *bad_vertex = h == ~0ull ? -1 : (int64_t)h;
  return 0;
}

}  // namespace pgc
