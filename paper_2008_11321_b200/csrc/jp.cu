// jp.cu -- Jones-Plassmann coloring (Algorithm 3) for the
// priority rho = <round, splitmix64(seed ^ v)>.
//
// JP Part 1 (pred[v], count[v] = |pred[v]|, lines 1116-1121) is produced by
// ADG's fused UPDATE (adg.cu) or by jp_setup_run: pred(v) lives in v's own
// CSR slot P[off[v] .. off[v] + npred[v]).
//
// JP Part 2 (lines 1123-1133) runs without level barriers:
//   1. jp_order_run  -- the exact priority order (a topological order of the
//                       DAG G_rho) by a two-level bucket sort.
//   2. k_jp_core     -- the dense priority prefix ("core", where the long
//                       dependency chains live) on one thread-block cluster
//                       with a shared-memory color replica per CTA (DSMEM).
//   3. k_jp_bulk     -- everything else as a lane-per-vertex dataflow: the
//                       Join of line 1132 is observed by polling the
//                       predecessors' colors instead of decrementing a counter.
// GetColor (lines 1135-1138) = first zero bit of a used-color bitmap window.
#include <climits>
#include <cstdio>

#include <cooperative_groups.h>

#include "pgc_internal.cuh"

namespace pgc {

namespace cg = cooperative_groups;

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
// Exact priority order: round descending, then h = splitmix64(seed ^ v)
// descending (a topological order of G_rho).
// Two-level bucket sort: key (round) histogram -> per-round bucket count ~
// |round| / kBucketTarget (a power of two, indexed by the top hash bits) ->
// scatter -> sort every bucket by h.
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

__device__ __forceinline__ int bucket_count_for(int cnt) {
  if (cnt <= 0) return 0;
  int want = (cnt + kBucketTarget - 1) / kBucketTarget;
  int b = 1;
  while (b < want) b <<= 1;
  return b;
}

// hist1[rmax - round[v]] += 1; privatised in shared memory when the key range is small.
__global__ void k_hist1(int64_t n, const int32_t* __restrict__ round, const State* st, int range,
                        int32_t* __restrict__ hist1) {
  extern __shared__ int sh[];
  const int rmax = st->rmax;
  const bool priv = range <= 8192;
  if (priv)
    for (int i = threadIdx.x; i < range; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int k = rmax - round[v];
    if (priv) atomicAdd(&sh[k], 1);
    else atomicAdd(&hist1[k], 1);
  }
  __syncthreads();
  if (priv)
    for (int i = threadIdx.x; i < range; i += blockDim.x)
      if (sh[i]) atomicAdd(&hist1[i], sh[i]);
}

__global__ void k_bucket_sizes(int L, const int32_t* __restrict__ hist1, int32_t* __restrict__ bsz) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x)
    bsz[i] = bucket_count_for(hist1[i]);
}

__device__ __forceinline__ int bucket_of(int v, int r, uint64_t seed, int rmax,
                                         const int32_t* __restrict__ hist1,
                                         const int32_t* __restrict__ base1) {
  const int k = rmax - r;
  const int B = bucket_count_for(hist1[k]);
  const int lg = 31 - __clz(B);
  const uint64_t h = prio_hash(seed, (uint32_t)v);
  const int hb = lg ? (int)(h >> (64 - lg)) : 0;
  return base1[k] + (B - 1 - hb);  // larger hash -> earlier bucket
}

__global__ void k_hist2(int64_t n, const int32_t* __restrict__ round, uint64_t seed,
                        const State* st, const int32_t* __restrict__ hist1,
                        const int32_t* __restrict__ base1, int32_t* __restrict__ bcnt) {
  const int rmax = st->rmax;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int b = bucket_of((int)v, round[v], seed, rmax, hist1, base1);
    atomicAdd(&bcnt[b], 1);
  }
}

__global__ void k_scatter(int64_t n, const int32_t* __restrict__ round, uint64_t seed,
                          const State* st, const int32_t* __restrict__ hist1,
                          const int32_t* __restrict__ base1, int32_t* __restrict__ bcnt,
                          const int32_t* __restrict__ bstart, int32_t* __restrict__ order) {
  const int rmax = st->rmax;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int b = bucket_of((int)v, round[v], seed, rmax, hist1, base1);
    const int pos = bstart[b] + atomicSub(&bcnt[b], 1) - 1;
    order[pos] = (int)v;
  }
}

// Sort every bucket by h descending (bucket = same round, same top hash
// bits).  One lane per bucket (insertion sort in registers, <= 16 entries, the
// common case at mean occupancy 4..8); larger buckets are ranked by a whole
// warp afterwards.
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
  const int L = (int)range;
  PGC_LAUNCH(c, kGOrder, "k_zero_i32", k_zero_i32<<<G, 256, 0, c.st>>>(c.hist1, L));
  const size_t shb = L <= 8192 ? (size_t)L * sizeof(int) : 0;
  PGC_LAUNCH(c, kGOrder, "k_hist1",
             k_hist1<<<G, 256, shb, c.st>>>(c.n, round, c.state, L, c.hist1));
  PGC_LAUNCH(c, kGOrder, "k_bucket_sizes",
             k_bucket_sizes<<<G, 256, 0, c.st>>>(L, c.hist1, c.base1));
  if (int e = scan_ex(c, c.base1, c.base1, nullptr, L, L, &c.state->nbuckets)) return e;
  PGC_LAUNCH(c, kGOrder, "k_zero_i32_dev",
             k_zero_i32_dev<<<G, 256, 0, c.st>>>(c.bcnt, &c.state->nbuckets, 1));
  PGC_LAUNCH(c, kGOrder, "k_hist2",
             k_hist2<<<G, 256, 0, c.st>>>(c.n, round, seed, c.state, c.hist1, c.base1, c.bcnt));
  if (int e = scan_ex(c, c.bcnt, c.bstart, &c.state->nbuckets, -1, c.lay.nb_cap,
                      &c.state->sorted))
    return e;
  PGC_LAUNCH(c, kGOrder, "k_scatter",
             k_scatter<<<G, 256, 0, c.st>>>(c.n, round, seed, c.state, c.hist1, c.base1, c.bcnt,
                                            c.bstart, c.order));
  PGC_LAUNCH(c, kGOrder, "k_bucket_sort",
             k_bucket_sort<<<G, 256, 0, c.st>>>(c.state, c.bstart, c.order, seed));
  return 0;
}

// ------------------------------------------------------------- shared -------
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

// ------------------------------------------------------------- core ---------
// JP on the "core": the longest prefix of the priority order whose vertices
// average >= core_min_avg preds (the dense, deep part of G_rho: on R-MAT 24 the
// top 55K vertices carry 4 146 of the 4 625 JP levels).  A priority prefix is
// closed under pred (preds have higher priority), so the core is colored
// before and independently of everything else.  It runs on ONE thread-block
// cluster: every CTA keeps a u16 replica of all core colors in shared memory;
// a vertex is colored by a warp of CTA (p mod C) (p = its core position), which
// reads its pred list -- rewritten to u16 core positions by k_core_lists -- and
// looks every pred color up in its LOCAL replica, waits on uncolored preds by
// polling local shared memory, takes GetColor from a
// 2048-color bitmap window, and publishes the color to all C replicas with
// DSMEM stores (plus the global color[]).  A dependency hop thus costs one
// DSMEM store + a local shared-memory poll instead of an L2 round trip.
constexpr int kCoreBlock = 1024;
constexpr int kCoreWarps = kCoreBlock / 32;
constexpr int kCoreWin = 2048;   // colors per bitmap window (64 x u32)
constexpr int kCorePend = 256;   // pending-pred list capacity per warp

// One block: NC = the longest prefix p <= min(n, core_max) of the priority
// order with sum(npred) >= min_avg * p and sum(npred) <= arc_cap.
__global__ void __launch_bounds__(1024) k_core_select(int64_t n, const int32_t* __restrict__ order,
                                                      const int32_t* __restrict__ npred, State* st,
                                                      int core_max, int min_avg,
                                                      long long arc_cap) {
  __shared__ long long s_w[32];
  __shared__ unsigned long long s_best;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int L = (int)(n < (int64_t)core_max ? n : (int64_t)core_max);
  const int per = (L + blockDim.x - 1) / blockDim.x;
  const int t0 = threadIdx.x * per;
  if (threadIdx.x == 0) s_best = 0;
  long long loc = 0;
  for (int k = 0; k < per; ++k)
    if (t0 + k < L) loc += npred[order[t0 + k]];
  long long incl = loc;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= s) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
    long long wi = w;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, wi, s);
      if (lane >= s) wi += y;
    }
    s_w[lane] = wi - w;
  }
  __syncthreads();
  long long run = s_w[warp] + incl - loc;
  unsigned long long best = 0;
  for (int k = 0; k < per; ++k) {
    const int p = t0 + k;
    if (p >= L) break;
    run += npred[order[p]];  // sum over the prefix of length p + 1
    if (run >= (long long)min_avg * (p + 1) && run <= arc_cap)
      best = ((unsigned long long)(p + 1) << 32) | (unsigned long long)run;
  }
  atomicMax(&s_best, best);
  __syncthreads();
  if (threadIdx.x == 0) {
    st->core_n = (int)(s_best >> 32);
    st->core_arcs = (long long)(s_best & 0xffffffffull);
  }
}

__global__ void k_core_pos(const int32_t* __restrict__ order, const State* st,
                           int32_t* __restrict__ pos) {
  const int NC = st->core_n;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < NC; p += gridDim.x * blockDim.x)
    pos[order[p]] = p;
}

// Warp per core vertex: rewrite its pred list in place (P slot, int32 ids ->
// u16 core positions at the start of the same slot) and record (slot, |pred|).
__global__ void k_core_lists(const int64_t* __restrict__ off, const int32_t* __restrict__ order,
                             const int32_t* __restrict__ npred, const int32_t* __restrict__ pos,
                             int32_t* P, int64_t* __restrict__ cbase, int32_t* __restrict__ cnp,
                             const State* st) {
  const int lane = lane_id();
  const int NC = st->core_n;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < NC; p += nw) {
    const int v = order[p];
    const int np = npred[v];
    const int64_t b = off[v];
    if (lane == 0) {
      cbase[p] = b;
      cnp[p] = np;
    }
    uint16_t* L = reinterpret_cast<uint16_t*>(P + b);
    for (int i0 = 0; i0 < np; i0 += 32) {
      const int i = i0 + lane;
      const int y = i < np ? pos[P[b + i]] : 0;
      __syncwarp();  // every lane has read its int32 entry before any u16 lands
      if (i < np) L[i] = (uint16_t)y;
      __syncwarp();
    }
  }
}

__device__ __forceinline__ int ld_vol_u16(const uint16_t* p) {
  return *(volatile const uint16_t*)p;
}

// OR color cc into the window bitmap (colors wbase+1 .. wbase+kCoreWin).
__device__ __forceinline__ void bm_set(unsigned* bm, int cc, int wbase) {
  const int bit = cc - wbase - 1;
  if (bit >= 0 && bit < kCoreWin) atomicOr(&bm[bit >> 5], 1u << (bit & 31));
}

// Examine core preds [from, np) in strips of 4x32: colored ones go into the
// window, uncolored ones into the warp's pending list.  Returns where to resume
// when the list is full, np when every pred was examined.
__device__ __forceinline__ int core_scan(const uint16_t* __restrict__ L, int np, int from,
                                         const uint16_t* cc, unsigned* bm, int wbase,
                                         uint16_t* plist, int& npend) {
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  for (int i0 = from; i0 < np; i0 += 128) {
    int q[4], c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + 32 * k + lane;
      q[k] = i < np ? (int)__ldg(L + i) : -1;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = q[k] >= 0 ? ld_vol_u16(cc + q[k]) : 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool pend = q[k] >= 0 && c[k] == 0;
      if (q[k] >= 0 && c[k]) bm_set(bm, c[k], wbase);
      const unsigned bal = __ballot_sync(0xffffffffu, pend);
      const int cnt = __popc(bal);
      if (npend + cnt > kCorePend) return i0 + 32 * k;  // strips before k are complete
      if (pend) plist[npend + __popc(bal & lt)] = (uint16_t)q[k];
      npend += cnt;
    }
  }
  return np;
}

__global__ void __launch_bounds__(kCoreBlock, 1) k_jp_core(const int32_t* __restrict__ order,
                                                           const int64_t* __restrict__ cbase,
                                                           const int32_t* __restrict__ cnp,
                                                           const int32_t* __restrict__ P,
                                                           int32_t* color, State* st,
                                                           unsigned long long watchdog_ns) {
  extern __shared__ __align__(16) uint16_t s_cc[];  // [NC] color replica (0 = uncolored)
  __shared__ unsigned s_bm[kCoreWarps][kCoreWin / 32];
  __shared__ uint16_t s_pend[kCoreWarps][kCorePend];
  __shared__ int s_ticket;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int NC = st->core_n;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  for (int i = threadIdx.x; i < NC; i += blockDim.x) s_cc[i] = 0;
  if (threadIdx.x == 0) s_ticket = 0;
  cl.sync();  // every replica is zeroed before any color is published
  uint16_t* remote = lane < C ? cl.map_shared_rank(s_cc, lane) : nullptr;
  const unsigned long long deadline = globaltimer() + watchdog_ns;
  unsigned* bm = s_bm[warp];
  uint16_t* plist = s_pend[warp];
  int kmax = 0;
  bool stall = false;
  while (!stall) {
    int k = 0;
    if (lane == 0) k = atomicAdd(&s_ticket, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    const int p = rank + C * k;
    if (p >= NC) break;
    const int np = cnp[p];
    const uint16_t* L = reinterpret_cast<const uint16_t*>(P + cbase[p]);
    int found = 0;
    for (int wbase = 0; !found && !stall; wbase += kCoreWin) {
      bm[lane] = 0;
      bm[lane + 32] = 0;
      __syncwarp();
      int npend = 0;
      int over = core_scan(L, np, 0, s_cc, bm, wbase, plist, npend);
      unsigned sleep_ns = 0;
      while (npend > 0 || over < np) {
        bool progress = false;
        int keep = 0;
        for (int j0 = 0; j0 < npend; j0 += 32) {
          const int j = j0 + lane;
          int q = 0, cc = 1;
          if (j < npend) {
            q = plist[j];
            cc = ld_vol_u16(s_cc + q);
          }
          const bool still = j < npend && cc == 0;
          if (j < npend && cc) bm_set(bm, cc, wbase);
          const unsigned bal = __ballot_sync(0xffffffffu, still);
          if (__ballot_sync(0xffffffffu, j < npend && cc != 0)) progress = true;
          __syncwarp();
          if (still) plist[keep + __popc(bal & lt)] = (uint16_t)q;
          keep += __popc(bal);
        }
        npend = keep;
        __syncwarp();
        if (over < np) {
          const int before = over;
          over = core_scan(L, np, over, s_cc, bm, wbase, plist, npend);
          if (over != before) progress = true;
        }
        if (npend == 0 && over >= np) break;
        if (progress) {
          sleep_ns = 0;
        } else {
          if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) {
            stall = true;
            break;
          }
          if (sleep_ns) __nanosleep(sleep_ns);
          sleep_ns = sleep_ns ? min(sleep_ns * 2, 64u) : 8u;
        }
      }
      __syncwarp();
      if (stall) break;
      // GetColor inside this window: the first zero bit
      const unsigned z0 = ~bm[lane], z1 = ~bm[lane + 32];
      const unsigned b0 = __ballot_sync(0xffffffffu, z0 != 0);
      const unsigned b1 = __ballot_sync(0xffffffffu, z1 != 0);
      if (b0) {
        const int w = __ffs(b0) - 1;
        found = wbase + 32 * w + __ffs(__shfl_sync(0xffffffffu, z0, w));
      } else if (b1) {
        const int w = __ffs(b1) - 1;
        found = wbase + 32 * (w + 32) + __ffs(__shfl_sync(0xffffffffu, z1, w));
      }
      __syncwarp();
    }
    if (stall) break;
    if (lane < C) *(volatile uint16_t*)(remote + p) = (uint16_t)found;  // publish to every replica
    if (lane == 0) st_relaxed(color + order[p], found);
    kmax = max(kmax, found);
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&st->K, kmax);
  cl.sync();  // no CTA leaves while a peer may still store into its replica
}

// ------------------------------------------------------------- bulk ---------
// JP on the rest of the priority order as a sync-free dataflow, one vertex per
// lane.  Tickets are taken in priority order (a topological order of G_rho) by
// free lanes; a lane scans its vertex's preds once (colors of colored preds go
// into a lane-private 512-color bitmap in shared memory, uncolored preds are
// compacted in place at the front of the vertex's own P slot), then watches
// the lowest-priority pending pred with one load per poll; when it is colored
// the pending list is re-examined.  With no pending pred, GetColor is the
// first zero bit; the lane stores the color and takes a
// new ticket.  Deadlock freedom: the highest-priority uncolored vertex has all
// preds colored, and if it is not held by a lane then no later ticket was
// handed out either, so some lane is free to take it; no lane ever blocks.
constexpr int kBulkBlock = 256;
constexpr int kBulkWords = 16;  // 512-color window per lane
constexpr int kBulkWin = 32 * kBulkWords;
constexpr int kBulkBatch = 8;   // pred loads in flight per lane

struct BulkLane {
  int v = -1, np = 0, wbase = 0, npend = 0, watch = -1;
  int64_t pb = 0;
  bool scan = false;
};

// priority key of u (larger = higher priority): round, then hash
__device__ __forceinline__ bool lower_prio(int ru, uint64_t hu, int rw, uint64_t hw) {
  return ru != rw ? ru < rw : hu < hw;
}

__global__ void __launch_bounds__(kBulkBlock) k_jp_bulk(int64_t n, const int64_t* __restrict__ off,
                                                       int32_t* P, const int32_t* __restrict__ npred,
                                                       const int32_t* __restrict__ order,
                                                       const int32_t* __restrict__ round,
                                                       uint64_t seed, int32_t* color, State* st,
                                                       unsigned sleep_max,
                                                       unsigned long long* tr_grab,
                                                       unsigned long long* tr_done,
                                                       unsigned long long watchdog_ns) {
  __shared__ unsigned s_bm[kBulkWords][kBulkBlock];  // word-major: lane-private, conflict-free
  const unsigned long long deadline = globaltimer() + watchdog_ns;
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  const int NC = st->core_n;
  const int64_t nb = n - NC;
  BulkLane s;
  bool exhausted = false;
  int kmax = 0;
  unsigned sleep_ns = 32;
  auto bm = [&](int w) -> unsigned& { return s_bm[w][threadIdx.x]; };
  // Re-examine pending preds P[pb, pb+npend): OR colored ones into the
  // window, compact the rest in place, watch the lowest-priority one.
  auto recheck = [&]() {
    int keep = 0, wr = 0x7fffffff;
    uint64_t wh = ~0ull;
    s.watch = -1;
    for (int j0 = 0; j0 < s.npend; j0 += kBulkBatch) {
      int u[kBulkBatch], c[kBulkBatch];
#pragma unroll
      for (int k = 0; k < kBulkBatch; ++k) u[k] = j0 + k < s.npend ? P[s.pb + j0 + k] : -1;
#pragma unroll
      for (int k = 0; k < kBulkBatch; ++k) c[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 1;
#pragma unroll
      for (int k = 0; k < kBulkBatch; ++k) {
        if (u[k] < 0) continue;
        if (c[k]) {
          const int bit = c[k] - s.wbase - 1;
          if (bit >= 0 && bit < kBulkWin) bm(bit >> 5) |= 1u << (bit & 31);
        } else {
          P[s.pb + keep++] = u[k];
          const int ru = round[u[k]];
          const uint64_t hu = prio_hash(seed, (uint32_t)u[k]);
          if (s.watch < 0 || lower_prio(ru, hu, wr, wh)) {
            s.watch = u[k];
            wr = ru;
            wh = hu;
          }
        }
      }
    }
    s.npend = keep;
  };
  for (;;) {
    // 1. free lanes take the next tickets (one atomic per warp)
    const unsigned want = __ballot_sync(0xffffffffu, s.v < 0 && !exhausted);
    if (want) {
      const int leader = __ffs(want) - 1;
      long long t0 = 0;
      if (lane == leader) t0 = atomicAdd(&st->ticket, (unsigned long long)__popc(want));
      t0 = __shfl_sync(0xffffffffu, t0, leader);
      if (s.v < 0 && !exhausted) {
        const long long t = t0 + __popc(want & lt);
        if (t < nb) {
          s.v = order[NC + t];
          s.np = npred[s.v];
          s.pb = off[s.v];
          s.wbase = 0;
          s.scan = true;
          if (tr_grab) tr_grab[s.v] = globaltimer();
        } else {
          exhausted = true;
        }
      }
    }
    if (__ballot_sync(0xffffffffu, s.v >= 0) == 0) break;  // all lanes free and out of tickets
    bool progress = false;
    // 2. first pass over every pred (or a new color window)
    if (s.v >= 0 && s.scan) {
#pragma unroll
      for (int w = 0; w < kBulkWords; ++w) bm(w) = 0;
      s.npend = s.np;  // every pred is "pending" until examined
      recheck();
      s.scan = false;
      progress = true;
    }
    // 3. poll the watched pred; when it is colored, re-examine the others
    if (s.v >= 0 && s.npend > 0) {
      if (ld_relaxed(color + s.watch)) {
        recheck();
        progress = true;
      }
    }
    // 4. GetColor once nothing is pending
    if (s.v >= 0 && !s.scan && s.npend == 0) {
      int found = 0;
#pragma unroll
      for (int w = 0; w < kBulkWords; ++w) {
        const unsigned z = ~bm(w);
        if (!found && z) found = s.wbase + 32 * w + __ffs(z);
      }
      if (found) {
        st_relaxed(color + s.v, found);
        if (tr_done) tr_done[s.v] = globaltimer();
        kmax = max(kmax, found);
        s.v = -1;
      } else {  // all kBulkWin colors of this window used: next window
        s.wbase += kBulkWin;
        s.scan = true;
      }
      progress = true;
    }
    if (__ballot_sync(0xffffffffu, progress)) {
      sleep_ns = 32;
    } else {
      if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) break;
      __nanosleep(sleep_ns);
      sleep_ns = min(sleep_ns * 2, sleep_max);
    }
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&st->K, kmax);
}

__global__ void k_jp_reset(State* st) {
  st->ticket = 0;
  st->K = 0;
  st->core_n = 0;
  st->core_arcs = 0;
}

// Largest cluster size (power of two <= want) that k_jp_core can launch with
// `smem` dynamic bytes; 0 if none.
static int core_cluster_size(int want, size_t smem) {
  static thread_local int attr_done = 0;
  if (!attr_done) {
    cudaFuncSetAttribute(k_jp_core, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_done = 1;
  }
  if (cudaFuncSetAttribute(k_jp_core, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int C = want; C >= 1; C >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kCoreBlock);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k_jp_core, &cfg) == cudaSuccess && nclusters >= 1)
      return C;
    cudaGetLastError();
  }
  return 0;
}

static int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

int jp_color_run(Ctx& c, int32_t* color) {
  PGC_LAUNCH(c, kGJp, "k_jp_reset", k_jp_reset<<<1, 1, 0, c.st>>>(c.state));
  if (c.n > 0) {
    // --- core ---
    if (c.tune.core_max > 0) {
      PGC_LAUNCH(c, kGCore, "k_core_select",
                 k_core_select<<<1, 1024, 0, c.st>>>(c.n, c.order, c.npred, c.state,
                                                      c.tune.core_max, c.tune.core_min_avg,
                                                      c.tune.core_arc_cap));
      if (int e = sync_state(c)) return e;
      const int NC = c.h_state->core_n;
      const long long arcs = c.h_state->core_arcs;
      int C = 0;
      const size_t smem = ((size_t)NC * 2 + 15) & ~(size_t)15;
      if (NC >= c.tune.core_min_n) {
        int want = c.tune.core_ctas > 0
                       ? c.tune.core_ctas
                       : (int)((arcs + c.tune.core_arcs_per_cta - 1) / c.tune.core_arcs_per_cta);
        want = pow2_floor(want < 1 ? 1 : (want > 16 ? 16 : want));
        C = core_cluster_size(want, smem);
      }
      if (C == 0) {
        PGC_CUDA(cudaMemsetAsync(&c.state->core_n, 0, sizeof(int), c.st));
      } else {
        c.core_ctas = C;
        const int G = c.nsm * 4;
        PGC_LAUNCH(c, kGCore, "k_core_pos", k_core_pos<<<G, 256, 0, c.st>>>(c.order, c.state, c.D));
        PGC_LAUNCH(c, kGCore, "k_core_lists",
                   k_core_lists<<<G * 2, 256, 0, c.st>>>(c.off, c.order, c.npred, c.D, c.P,
                                                         c.cbase, c.cnp, c.state));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(kCoreBlock);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = c.st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const unsigned long long wd = (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull;
        PGC_LAUNCH(c, kGCore, "k_jp_core",
                   PGC_CUDA(cudaLaunchKernelEx(&cfg, k_jp_core, (const int32_t*)c.order,
                                               (const int64_t*)c.cbase, (const int32_t*)c.cnp,
                                               (const int32_t*)c.P, color, c.state, wd)));
      }
    }
    // --- bulk ---
    const int G = wave_grid(c, k_jp_bulk, kBulkBlock);
    PGC_LAUNCH(c, kGJp, "k_jp_bulk",
               k_jp_bulk<<<G, kBulkBlock, 0, c.st>>>(
                   c.n, c.off, c.P, c.npred, c.order, c.round_key, c.seed, color, c.state,
                   (unsigned)c.tune.jp_sleep_max, c.trace_grab, c.trace_done,
                   (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull));
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
