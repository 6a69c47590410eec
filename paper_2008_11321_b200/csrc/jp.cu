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

// PGC_PROBE builds (tools/micro/build_probe.sh, never the product library)
// stamp per-vertex phase times (%globaltimer) into the trace arrays ([8*v + k])
// for the core engine hop breakdown (tools/micro/hop_probe.py, core_probe.py).
#ifdef PGC_PROBE
#define PROBE_STAMP(arr, v, k) \
  do {                          \
    if ((arr) && lane == 0) (arr)[8 * (v) + (k)] = globaltimer(); \
  } while (0)
#else
#define PROBE_STAMP(arr, v, k) \
  do {                          \
  } while (0)
#endif

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
                   int64_t cap, int* total_out, int group = kGOrder) {
  const int64_t ntiles_cap = (cap + kScanTile - 1) / kScanTile + 1;
  if (ntiles_cap > c.lay.scan_tmp_cap) return fail(4, "scan temp too small");
  const int64_t grid = len_h >= 0 ? (len_h + kScanTile - 1) / kScanTile : ntiles_cap;
  if (grid > 0)
    PGC_LAUNCH(c, group, "k_scan_reduce",
               k_scan_reduce<<<(unsigned)grid, 256, 0, c.st>>>(in, len_ptr, len_h, c.scan_tmp));
  PGC_LAUNCH(c, group, "k_scan_tmp",
             k_scan_tmp<<<1, 1024, 0, c.st>>>(c.scan_tmp, ntiles_cap, len_ptr, len_h, out, total_out));
  if (grid > 0)
    PGC_LAUNCH(c, group, "k_scan_down",
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

// The priority order holds every vertex except the isolated ones (npred < 0,
// settled with color 1 before JP: no pred, no succ).
__device__ __forceinline__ bool in_order(const int32_t* __restrict__ npred, int64_t v) {
  return npred[v] >= 0;
}

// hist1[rmax - round[v]] += 1; privatised in shared memory when the key range is
// small.  Also counts the ordered vertices (st->n_order).
__global__ void k_hist1(int64_t n, const int32_t* __restrict__ round,
                        const int32_t* __restrict__ npred, State* st, int range,
                        int32_t* __restrict__ hist1) {
  extern __shared__ int sh[];
  __shared__ int s_cnt;
  const int rmax = st->rmax;
  const bool priv = range <= 8192;
  if (priv)
    for (int i = threadIdx.x; i < range; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int cnt = 0;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x; v0 < n; v0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = v0 + threadIdx.x;
    const bool in = v < n && in_order(npred, v);
    const int k = in ? rmax - round[v] : -1;
    cnt += in;
    // few distinct keys: one atomic per key per warp (lanes with equal keys)
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    if (in && lane_id() == __ffs(peers) - 1) {
      if (priv) atomicAdd(&sh[k], __popc(peers));
      else atomicAdd(&hist1[k], __popc(peers));
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s_cnt, cnt);
  __syncthreads();
  if (priv)
    for (int i = threadIdx.x; i < range; i += blockDim.x)
      if (sh[i]) atomicAdd(&hist1[i], sh[i]);
  if (threadIdx.x == 0 && s_cnt) atomicAdd(&st->n_order, s_cnt);
}

// hist1[k] = cnt[T-1-k] (key k = rmax - round = T - round), n_order = sum:
// the ADG selection counted every round's ordered (non-isolated) vertices.
__global__ void __launch_bounds__(1024) k_hist1_rounds(int T, const int32_t* __restrict__ cnt,
                                                       int32_t* __restrict__ hist1, State* st) {
  __shared__ int s_w[32];
  int sum = 0;
  for (int k = threadIdx.x; k < T; k += blockDim.x) {
    const int x = cnt[T - 1 - k];
    hist1[k] = x;
    sum += x;
  }
  sum = __reduce_add_sync(0xffffffffu, sum);
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
    st->n_order = t;
  }
}

__global__ void k_bucket_sizes(int L, const int32_t* __restrict__ hist1, int32_t* __restrict__ bsz) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x)
    bsz[i] = bucket_count_for(hist1[i]);
}

// Second priority key: rho_R(v) = splitmix64(seed ^ v) (JP-ADG, JP-ADG-M,
// pgc_jp_color), or the id itself for ADG-O's total order (Q22: inside a
// (round, D_rem) group the larger id has the larger rho), shifted so that the
// ids 0..n-1 span the top bits the buckets are indexed by (idkey = 64 minus
// the bit length of n-1; 0 selects the hash).
struct Key2 {
  uint64_t seed;
  int idkey;
  __device__ __forceinline__ uint64_t operator()(uint32_t v) const {
    return idkey ? ((uint64_t)v << idkey) : prio_hash(seed, v);
  }
};

__device__ __forceinline__ int bucket_of(int v, int r, Key2 seed, int rmax,
                                         const int32_t* __restrict__ hist1,
                                         const int32_t* __restrict__ base1) {
  const int k = rmax - r;
  const int B = bucket_count_for(hist1[k]);
  const int lg = 31 - __clz(B);
  const uint64_t h = seed((uint32_t)v);
  const int hb = lg ? (int)(h >> (64 - lg)) : 0;
  return base1[k] + (B - 1 - hb);  // larger hash -> earlier bucket
}

#ifndef PGC_ORD_ITEMS
#define PGC_ORD_ITEMS 4
#endif
constexpr int kOrdItems = PGC_ORD_ITEMS;
__global__ void k_hist2(int64_t n, const int32_t* __restrict__ round, Key2 seed,
                        const int32_t* __restrict__ npred,
                        const State* st, const int32_t* __restrict__ hist1,
                        const int32_t* __restrict__ base1, int32_t* __restrict__ bcnt,
                        int part, const int32_t* __restrict__ list) {
  const int rmax = st->rmax;
  const int ktop = st->ord_ktop;
  // `list` (part 0): a superset of the top rounds saved by ADG (k_round_aux)
  const bool use_list = list && st->top_n > 0;
  const int64_t cnt = use_list ? st->top_n : n;
  // kOrdItems vertices per thread per step, all loads before any use
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < cnt; i0 += stride * kOrdItems) {
    int vv[kOrdItems], np[kOrdItems], r[kOrdItems];
#pragma unroll
    for (int j = 0; j < kOrdItems; ++j) {
      const int64_t i = i0 + j * stride;
      vv[j] = i < cnt ? (use_list ? list[i] : (int)i) : 0;
    }
#pragma unroll
    for (int j = 0; j < kOrdItems; ++j) {
      const bool ok = i0 + j * stride < cnt;
      np[j] = ok ? (use_list ? npred[vv[j]] : __ldcs(npred + vv[j])) : -1;
      r[j] = ok ? (use_list ? round[vv[j]] : __ldcs(round + vv[j])) : 0;
    }
#pragma unroll
    for (int j = 0; j < kOrdItems; ++j)
      // part 0: the top keys only, 1: the rest, -1: all
      if (np[j] >= 0 && (part < 0 || ((rmax - r[j] <= ktop) == (part == 0))))
        atomicAdd(&bcnt[bucket_of(vv[j], r[j], seed, rmax, hist1, base1)], 1);
  }
}

// Places every ordered vertex's id at a slot of its bucket (4-byte stores into
// an n-int array that stays in L2; the 16-byte records are written by
// k_bucket_sort, bucket by bucket, after the sort).
__global__ void k_scatter(int64_t n, const int32_t* __restrict__ round, Key2 seed,
                          const State* st, const int32_t* __restrict__ hist1,
                          const int32_t* __restrict__ base1, int32_t* __restrict__ bcnt,
                          const int32_t* __restrict__ bstart, const int32_t* __restrict__ npred,
                          int32_t* __restrict__ ord, int part,
                          const int32_t* __restrict__ list) {
  const int rmax = st->rmax;
  const int ktop = st->ord_ktop;
  // the bottom part's buckets were counted and scanned on their own: its
  // positions start after the top part's
  const int base = part == 1 ? st->ord_ptop : 0;
  const bool use_list = list && st->top_n > 0;
  const int64_t cnt = use_list ? st->top_n : n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = use_list ? list[i] : i;
    if (!in_order(npred, v)) continue;  // isolated: not in the order
    const int r = round[v];
    // part 0: the top keys only, 1: the rest, -1: all
    if (part >= 0 && ((rmax - r <= ktop) != (part == 0))) continue;
    const int b = bucket_of((int)v, r, seed, rmax, hist1, base1);
    ord[base + bstart[b] + atomicSub(&bcnt[b], 1) - 1] = (int)v;
  }
}

// Sort every bucket by h descending (bucket = same round, same top hash
// bits) and write its JP work records {v, |pred|, P slot lo, hi} in that
// order.  One lane per bucket (insertion sort in registers, <= 12 entries, the
// common case at mean occupancy 4..8); larger buckets are ranked by a whole
// warp.  Every bucket is sorted: the bulk's workers hold one ticket AHEAD of
// the vertex they color (the prefetched record), so with an order that is
// exact only across buckets a worker could color v while its own prefetched
// ticket is a higher-priority same-bucket pred of v: a deadlock (seen once on
// JP-R at R-MAT 24).  In exact priority order a prefetched ticket always has a
// lower priority than the current one, and the highest-priority uncolored
// vertex is a current vertex (all preds colored) or the next ticket of a
// worker whose current vertex is colored.
constexpr int kLaneSortMax = 12;
__device__ __forceinline__ int4 work_rec(int v, const int32_t* __restrict__ npred,
                                         const int64_t* __restrict__ off) {
  const int64_t o = off[v];
  return make_int4(v, npred[v], (int)(uint32_t)o, (int)(o >> 32));
}
__global__ void k_bucket_sort(const State* st, const int32_t* __restrict__ bstart,
                              int32_t* __restrict__ ord, const int32_t* __restrict__ npred,
                              const int64_t* __restrict__ off, int4* __restrict__ rec,
                              Key2 seed, int part) {
  const int lane = lane_id();
  // part 0: buckets [0, ord_btop), 1: [ord_btop, nb), -1: all
  const int nb = part == 0 ? st->ord_btop : st->nbuckets;
  const int bfirst = part == 1 ? st->ord_btop : 0;
  const int base = part == 1 ? st->ord_ptop : 0;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = gridDim.x * blockDim.x;
  for (int b0 = bfirst + tid - lane; b0 < nb; b0 += nthreads) {
    const int b = b0 + lane;
    int s0 = 0, s = 0;
    if (b < nb) {
      s0 = bstart[b];
      s = bstart[b + 1] - s0;
      s0 += base;
    }
    if (s >= 1 && s <= kLaneSortMax) {
      int vv[kLaneSortMax];
      uint64_t hh[kLaneSortMax];
#pragma unroll
      for (int i = 0; i < kLaneSortMax; ++i)
        if (i < s) {
          vv[i] = ord[s0 + i];
          hh[i] = seed((uint32_t)vv[i]);
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
      int4 r[kLaneSortMax];
#pragma unroll
      for (int i = 0; i < kLaneSortMax; ++i)  // all gathers in flight
        if (i < s) r[i] = work_rec(vv[i], npred, off);
#pragma unroll
      for (int i = 0; i < kLaneSortMax; ++i)
        if (i < s) rec[s0 + i] = r[i];
    }
    // rare large buckets: the whole warp ranks them, one bucket at a time
    unsigned big = __ballot_sync(0xffffffffu, s > kLaneSortMax);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int bs0 = __shfl_sync(0xffffffffu, s0, src);
      const int bs = __shfl_sync(0xffffffffu, s, src);
      if (bs <= 32) {
        const int v = lane < bs ? ord[bs0 + lane] : 0;
        const uint64_t h = lane < bs ? seed((uint32_t)v) : 0;
        int rank = 0;
        for (int j = 0; j < bs; ++j) rank += __shfl_sync(0xffffffffu, h, j) > h;
        if (lane < bs) rec[bs0 + rank] = work_rec(v, npred, off);
      } else {
        if (lane == 0)  // very rare: insertion sort of the ids in place
          for (int i = 1; i < bs; ++i) {
            const int x = ord[bs0 + i];
            const uint64_t hx = seed((uint32_t)x);
            int j = i - 1;
            while (j >= 0 && seed((uint32_t)ord[bs0 + j]) < hx) {
              ord[bs0 + j + 1] = ord[bs0 + j];
              --j;
            }
            ord[bs0 + j + 1] = x;
          }
        __syncwarp();
        for (int i = lane; i < bs; i += 32) rec[bs0 + i] = work_rec(ord[bs0 + i], npred, off);
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
  st->sorted_bot = 0;
  st->n_order = 0;
}

// Split point of a deferred order: the smallest key index ktop whose keys
// 0..ktop (the top rounds) hold >= target ordered vertices (every key if
// none), and the first bucket past them.  One block, chunked scan of hist1.
__global__ void __launch_bounds__(1024) k_order_top(State* st, const int32_t* __restrict__ hist1,
                                                   const int32_t* __restrict__ base1, int L,
                                                   int target) {
  __shared__ int s_w[32];
  __shared__ int s_k;
  __shared__ long long s_p;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_k = L - 1;
    s_p = -1;
  }
  long long run = 0;
  for (int k0 = 0; k0 < L; k0 += blockDim.x) {
    const int k = k0 + threadIdx.x;
    const int x = k < L ? hist1[k] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    int wex = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) wex += s_w[w];
      tot += s_w[w];
    }
    if (k < L && run + wex + incl >= target && run + wex + incl - x < target) {
      s_k = k;
      s_p = run + wex + incl;
    }
    __syncthreads();
    run += tot;
    if (run >= target) break;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int k = s_k;
    st->ord_ktop = k;
    st->ord_btop = k + 1 < L ? base1[k + 1] : st->nbuckets;
    st->ord_ptop = s_p >= 0 ? (int)s_p : st->n_order;
  }
}

int jp_order_run(Ctx& c, const int32_t* round, uint64_t seed_, bool range_known, bool idkey,
                 bool defer) {
  NvtxRange nvtx_("pgc JP priority order");
  PGC_CHK_SIZES(c);
  int idshift = 0;
  if (idkey) {
    int bits = 1;
    while (bits < 63 && ((int64_t)1 << bits) < c.n) ++bits;  // bit length of n - 1
    idshift = 64 - bits;
  }
  const Key2 seed{seed_, idshift};
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
  if (range_known && L <= c.lay.range_cap) {
    // ADG rounds: the histogram was counted by the selection (k_adg_finalize)
    PGC_LAUNCH(c, kGOrder, "k_hist1_rounds",
               k_hist1_rounds<<<1, 1024, 0, c.st>>>(L, c.hist1 + c.lay.range_cap, c.hist1,
                                                    c.state));
  } else {
    PGC_LAUNCH(c, kGOrder, "k_zero_i32", k_zero_i32<<<G, 256, 0, c.st>>>(c.hist1, L));
    const size_t shb = L <= 8192 ? (size_t)L * sizeof(int) : 0;
    PGC_LAUNCH(c, kGOrder, "k_hist1",
               k_hist1<<<G, 256, shb, c.st>>>(c.n, round, c.npred, c.state, L, c.hist1));
  }
  PGC_LAUNCH(c, kGOrder, "k_bucket_sizes",
             k_bucket_sizes<<<G, 256, 0, c.st>>>(L, c.hist1, c.base1));
  if (int e = scan_ex(c, c.base1, c.base1, nullptr, L, L, &c.state->nbuckets)) return e;
  // deferred: the top rounds now (the core's prefix), the rest beside the core
  defer = defer && c.tune.jp_split_overlap && c.tune.core_max > 0;
  const int part = defer ? 0 : -1;
  // ADG's saved top-round list (superset of the top part) replaces the pass over n
  const int32_t* top_list = defer && range_known && c.top_list ? c.Rl : nullptr;
  if (defer)
    PGC_LAUNCH(c, kGOrder, "k_order_top",
               k_order_top<<<1, 1024, 0, c.st>>>(c.state, c.hist1, c.base1, L, core_reach(c.tune)));
  PGC_LAUNCH(c, kGOrder, "k_zero_i32_dev",
             k_zero_i32_dev<<<G, 256, 0, c.st>>>(c.bcnt, &c.state->nbuckets, 1));
  PGC_LAUNCH(c, kGOrder, "k_hist2",
             k_hist2<<<G, 256, 0, c.st>>>(c.n, round, seed, c.npred, c.state, c.hist1, c.base1,
                                          c.bcnt, part, top_list));
  if (int e = scan_ex(c, c.bcnt, c.bstart, &c.state->nbuckets, -1, c.lay.nb_cap,
                      &c.state->sorted))
    return e;
  PGC_LAUNCH(c, kGOrder, "k_scatter",
             k_scatter<<<G, 256, 0, c.st>>>(c.n, round, seed, c.state, c.hist1, c.base1, c.bcnt,
                                            c.bstart, c.npred, c.U[1], part, top_list));
  PGC_LAUNCH(c, kGOrder, "k_bucket_sort",
             k_bucket_sort<<<G, 256, 0, c.st>>>(c.state, c.bstart, c.U[1], c.npred, c.off, c.rec,
                                                seed, part));
  c.ord_pending = defer;
  c.ord_deferred = defer;
  c.ord_round = round;
  c.ord_seed = seed_;
  c.ord_idshift = idshift;
  return 0;
}

// The bottom part of a deferred order (on c.st, which may be a side stream).
static int jp_order_bottom(Ctx& c) {
  const Key2 seed{c.ord_seed, c.ord_idshift};
  const int G = c.nsm * 8;
  // the top part's bucket counts are spent (0): count and scan the rest alone
  PGC_LAUNCH(c, kGOrder, "k_hist2",
             k_hist2<<<G, 256, 0, c.st>>>(c.n, c.ord_round, seed, c.npred, c.state, c.hist1,
                                          c.base1, c.bcnt, 1, nullptr));
  if (int e = scan_ex(c, c.bcnt, c.bstart, &c.state->nbuckets, -1, c.lay.nb_cap,
                      &c.state->sorted_bot))
    return e;
  PGC_LAUNCH(c, kGOrder, "k_scatter",
             k_scatter<<<G, 256, 0, c.st>>>(c.n, c.ord_round, seed, c.state, c.hist1, c.base1,
                                            c.bcnt, c.bstart, c.npred, c.U[1], 1, nullptr));
  PGC_LAUNCH(c, kGOrder, "k_bucket_sort",
             k_bucket_sort<<<G, 256, 0, c.st>>>(c.state, c.bstart, c.U[1], c.npred, c.off, c.rec,
                                                seed, 1));
  c.ord_pending = false;
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

// ------------------------------------------------------------- byte maps ---
// GetColor's used-color set as a BYTE map per warp in shared memory: marking
// color c is a plain st.shared.u8 of 1 (idempotent, so lanes marking colors
// that share a word never lose an update and need no atomics -- a shared
// atomicOr costs 2 cycles per lane); the first zero byte is found 32 bytes per
// ballot.
__device__ __forceinline__ void bmap_clear(uint8_t* bm, int bytes) {
  uint4* w = reinterpret_cast<uint4*>(bm);
  for (int i = lane_id(); i < bytes / 16; i += 32) w[i] = make_uint4(0, 0, 0, 0);
}
__device__ __forceinline__ void bmap_mark(uint8_t* bm, int cc, int wbase, int bytes) {
  const int b = cc - wbase - 1;
  if (b >= 0 && b < bytes) bm[b] = 1;
}
// Index of the first zero byte at or after `from` in the warp's map (BYTES if
// none); warp-wide.  32 consecutive bytes per probe (conflict-free).
template <int BYTES>
__device__ __forceinline__ int bmap_next_zero(const uint8_t* bm, int from) {
  const int lane = lane_id();
  for (int b0 = from; b0 < BYTES; b0 += 32) {
    const int b = b0 + lane;
    const unsigned m = __ballot_sync(0xffffffffu, b < BYTES && bm[b] == 0);
    if (m) return b0 + __ffs(m) - 1;
  }
  return BYTES;
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
#ifndef PGC_CORE_BLOCK
#define PGC_CORE_BLOCK 1024
#endif
constexpr int kCoreBlock = PGC_CORE_BLOCK;
constexpr int kCoreWarps = kCoreBlock / 32;
constexpr int kCoreWin = 1024;   // colors per byte-map window
constexpr int kCorePend = 512;   // pending-pred list capacity per warp
constexpr int kCoreVertsPerCta = 1024;  // cluster sizing: core vertices per CTA
constexpr int kCoreRun = 32;     // consecutive core positions per CTA run
constexpr int kCoreFloor = 16384;  // core_div never caps the prefix below this
#ifndef PGC_CORE_TAIL
#define PGC_CORE_TAIL 4
#endif
constexpr int kCoreTail = PGC_CORE_TAIL;  // preds left for the collective-free tail
// dynamic shared memory ahead of the color replica: bitmaps + pending lists
constexpr int kCoreFixedSmem = kCoreWarps * kCoreWin + kCoreWarps * kCorePend * 2;

// One block: NC = the longest prefix p <= min(n, core_max) of the priority
// order with sum(npred) >= min_avg * p and sum(npred) <= arc_cap.
__global__ void __launch_bounds__(1024) k_core_select(const int4* __restrict__ rec,
                                                      State* st,
                                                      int core_max, int min_avg,
                                                      long long arc_cap, int tier2_max,
                                                      int core_div, int core_dmul) {
  // warp w scans the contiguous chunk [wb, we) of the prefix, lanes reading
  // consecutive records, kCsU strips in flight: pass 1 sums the chunk, a
  // block scan of the warp sums gives each chunk's base, pass 2 evaluates
  // every prefix length
  constexpr int kCsU = 8;
  __shared__ long long s_w[32];
  __shared__ unsigned long long s_best;
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int no = st->n_order;
  // the prefix is also capped at max(kCoreFloor, n_order / core_div): each
  // core vertex costs the one cluster ~6 ns, which only the chain's top
  // repays (R-MAT 20, 0.55 M ordered vertices: 65 535 core vertices 1.73 ms
  // per step, 32 768 1.71, 16 384 1.59, 8 192 1.65; R-MAT 24 and Chung-Lu,
  // 8 M ordered vertices, keep 65 535)
  // ... and, after ADG, at core_dmul x the largest mean degree of a G[U_l]
  // (ADG's peel is a 2-approximate densest-subgraph peel; that mean degree is
  // within 2x of the degeneracy): the best core sizes measured were 16 K / 24-32 K
  // / 49 K vertices at 808 / 1 603 / 2 287 (R-MAT 20 / Chung-Lu / R-MAT 24)
  long long capl = core_div > 0 ? (long long)(no / core_div) : (long long)core_max;
  if (core_dmul > 0 && st->avg_max > 0) capl = min(capl, (long long)core_dmul * st->avg_max);
  const int capn = (int)max((long long)kCoreFloor, min(capl, (long long)core_max));
  const int L = min(no, min(core_max, capn));
  const int cw = ((L + nw - 1) / nw + 31) & ~31;
  const int wb = min(L, warp * cw), we = min(L, wb + cw);
  if (threadIdx.x == 0) s_best = 0;
  long long loc = 0;
  for (int j0 = wb; j0 < we; j0 += 32 * kCsU) {
    int x[kCsU];
#pragma unroll
    for (int u = 0; u < kCsU; ++u) {
      const int p = j0 + 32 * u + lane;
      x[u] = p < we ? rec[p].y : 0;
    }
#pragma unroll
    for (int u = 0; u < kCsU; ++u) loc += x[u];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
  if (lane == 0) s_w[warp] = loc;
  __syncthreads();
  if (warp == 0) {
    const long long w = lane < nw ? s_w[lane] : 0;
    long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) s_w[lane] = wi - w;
  }
  __syncthreads();
  long long run = s_w[warp];  // sum over the positions before this chunk
  unsigned long long best = 0;
  for (int j0 = wb; j0 < we; j0 += 32 * kCsU) {
    int x[kCsU];
#pragma unroll
    for (int u = 0; u < kCsU; ++u) {
      const int p = j0 + 32 * u + lane;
      x[u] = p < we ? rec[p].y : 0;
    }
#pragma unroll
    for (int u = 0; u < kCsU; ++u) {
      long long incl = x[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int p = j0 + 32 * u + lane;
      const long long pre = run + incl;  // sum over the prefix of length p + 1
      if (p < we && pre >= (long long)min_avg * (p + 1) && pre <= arc_cap)
        best = ((unsigned long long)(p + 1) << 32) | (unsigned long long)pre;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  atomicMax(&s_best, best);
  __syncthreads();
  if (threadIdx.x == 0) {
    // tier 2: when the dense prefix runs into the cap, the next <= tier2_max
    // positions get a second cluster pass after the first (the priority
    // prefix of length NC1 + NC2 is closed under pred as well)
    const int nc1 = (int)(s_best >> 32);
    const int nc2 = (nc1 == core_max && tier2_max > 0) ? min(tier2_max, no - nc1) : 0;
    st->core_n1 = nc1;
    st->core_n = nc1 + nc2;
    st->core_arcs = (long long)(s_best & 0xffffffffull);
  }
}

// pos[v] = core position of v; also clears the per-vertex list states of the
// list rewrite beside the core (`ready`, when it runs there): one launch, no memset
__global__ void k_core_pos(const int4* __restrict__ rec, const State* st, int32_t* __restrict__ pos,
                           int32_t* __restrict__ ready) {
  const int NC = st->core_n;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < NC; p += gridDim.x * blockDim.x) {
    pos[rec[p].x] = p;
    if (ready && p < st->core_n1) ready[p] = 0;
  }
}

// One warp rewrites core vertex p's pred list in place (P slot, int32 ids ->
// u16 core positions at the start of the same slot): kListStrips strips of 32
// entries per step (loads, then gathers, in flight together); the u16 writes
// of a step land on int32 entries the step (or an earlier one) has read.
__device__ __forceinline__ void core_list_rewrite(const int4& r, const int32_t* __restrict__ pos,
                                                  int32_t* P) {
  const int lane = lane_id();
  const int np = r.y;
  const int64_t b = lo_hi(r.z, r.w);
  uint16_t* L = reinterpret_cast<uint16_t*>(P + b);
  constexpr int kListStrips = 8;
  for (int i0 = 0; i0 < np; i0 += 32 * kListStrips) {
    int x[kListStrips], y[kListStrips];
#pragma unroll
    for (int k = 0; k < kListStrips; ++k) {
      const int i = i0 + 32 * k + lane;
      x[k] = i < np ? __ldcg(P + b + i) : -1;
    }
#pragma unroll
    for (int k = 0; k < kListStrips; ++k) y[k] = x[k] >= 0 ? pos[x[k]] : 0;
    __syncwarp();  // every lane has read its int32 entries before any u16 lands
#pragma unroll
    for (int k = 0; k < kListStrips; ++k) {
      const int i = i0 + 32 * k + lane;
      if (i < np) L[i] = (uint16_t)y[k];
    }
    __syncwarp();
  }
}

// Per-vertex list states while the rewrite runs beside the core kernel:
// 0 = untouched, 1 = claimed (being rewritten), 2 = done.  Whoever claims a
// list (atomicCAS 0 -> 1) rewrites it and releases 2; the core claims the
// lists k_core_lists has not reached when it has waited too long -- so the
// core also finishes when the two kernels do not run concurrently (a
// profiler, CUDA_LAUNCH_BLOCKING).
constexpr int kListTodo = 0, kListBusy = 1, kListDone = 2;
__device__ __forceinline__ void list_release(int32_t* ready, int p) {
  // every lane's stores precede this (bar.warp.sync in core_list_rewrite)
  __threadfence();
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready + p), "r"(kListDone) : "memory");
}

// Warp per core vertex; with `ready`, each list is claimed first (see above).
__global__ void k_core_lists(const int4* __restrict__ rec, const int32_t* __restrict__ pos,
                             int32_t* P, const State* st, int32_t* ready) {
  const int lane = lane_id();
  const int NC = st->core_n1;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < NC; p += nw) {
    if (ready) {
      int claimed = 0;
      if (lane == 0) claimed = atomicCAS(ready + p, kListTodo, kListBusy) == kListTodo;
      if (!__shfl_sync(0xffffffffu, claimed, 0)) continue;  // the core took it
    }
    core_list_rewrite(rec[p], pos, P);
    if (ready && lane == 0) list_release(ready, p);
  }
}

// Tier 2's lists (positions [core_n1, core_n)), rewritten in place to int32
// codes: a pred in tier 2 -> its tier-2 position (>= 0), a pred in tier 1 ->
// -(id + 1) (its color is final when tier 2 runs: read from color[] once).
// Warp per vertex, strips of loads then pos gathers in flight.
__global__ void k_core2_lists(const int4* __restrict__ rec, const int32_t* __restrict__ pos,
                              int32_t* P, const State* st) {
  const int lane = lane_id();
  const int N1 = st->core_n1, NC = st->core_n;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  constexpr int kS = 8;
  for (int p = N1 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); p < NC; p += nw) {
    const int4 r = rec[p];
    const int np = r.y;
    int32_t* L = P + lo_hi(r.z, r.w);
    for (int i0 = 0; i0 < np; i0 += 32 * kS) {
      int x[kS], y[kS];
#pragma unroll
      for (int k = 0; k < kS; ++k) {
        const int i = i0 + 32 * k + lane;
        x[k] = i < np ? L[i] : -1;
      }
#pragma unroll
      for (int k = 0; k < kS; ++k) y[k] = x[k] >= 0 ? pos[x[k]] : 0;
#pragma unroll
      for (int k = 0; k < kS; ++k) {
        const int i = i0 + 32 * k + lane;
        PGC_DCHECK(i >= np || (y[k] >= 0 && y[k] < p), y[k], p);  // a pred precedes p
        if (i < np) L[i] = y[k] >= N1 ? y[k] - N1 : -(x[k] + 1);
      }
    }
  }
}

// 1 << d for 0 <= d < 32, else 0 (PTX clamps the shift amount)
__device__ __forceinline__ unsigned shl1(int d) {
  unsigned r;
  asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(d));
  return r;
}

__device__ __forceinline__ int ld_vol_u16(const uint16_t* p) {
  return *(volatile const uint16_t*)p;
}


// Examine core preds [from, np) (from even) in strips of 32 u16 pairs, 8 strips
// (512 preds) per step, the next step's pred words loaded before this step is
// processed (a hub's list is long: its scan must not pay one L2 latency per
// 256 preds): colored ones go into the window, uncolored ones into the warp's
// pending list; qmax tracks the largest pending core position (the
// lowest-priority pending pred, i.e. the one expected to be colored last).
// Returns where to resume when the list is full, np when every pred was examined.
#ifndef PGC_SCAN_STRIPS
#define PGC_SCAN_STRIPS 4
#endif
#ifndef PGC_SCAN_PREFETCH
#define PGC_SCAN_PREFETCH 1
#endif
constexpr int kScanStrips = PGC_SCAN_STRIPS;
__device__ __forceinline__ int core_scan(const uint16_t* __restrict__ L, int np, int from,
                                         const uint16_t* cc, uint8_t* bm, int wbase,
                                         uint16_t* plist, int& npend, int& qmax) {
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  const uint32_t* L2 = reinterpret_cast<const uint32_t*>(L);  // P slots are 4-byte aligned
  constexpr int kStep = 64 * kScanStrips;
  uint32_t w[kScanStrips];
#pragma unroll
  for (int k = 0; k < kScanStrips; ++k) {
    const int i = from + 64 * k + 2 * lane;
    w[k] = i < np ? __ldcg(L2 + (i >> 1)) : 0u;
  }
  for (int i0 = from; i0 < np; i0 += kStep) {
    uint32_t wn[kScanStrips];
    if (PGC_SCAN_PREFETCH) {
#pragma unroll
      for (int k = 0; k < kScanStrips; ++k) {
        const int i = i0 + kStep + 64 * k + 2 * lane;
        wn[k] = i < np ? __ldcg(L2 + (i >> 1)) : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < kScanStrips; ++k) {
      const int i = i0 + 64 * k + 2 * lane;
      const int qa = i < np ? (int)(w[k] & 0xffffu) : -1;
      const int qb = i + 1 < np ? (int)(w[k] >> 16) : -1;
      const int ca = qa >= 0 ? ld_vol_u16(cc + qa) : 1;
      const int cb = qb >= 0 ? ld_vol_u16(cc + qb) : 1;
      const unsigned ba = __ballot_sync(0xffffffffu, qa >= 0 && ca == 0);
      const unsigned bb = __ballot_sync(0xffffffffu, qb >= 0 && cb == 0);
      if (npend + __popc(ba) + __popc(bb) > kCorePend) return i0 + 64 * k;  // strips before k are complete
      if (qa >= 0 && ca) bmap_mark(bm, ca, wbase, kCoreWin);
      if (qb >= 0 && cb) bmap_mark(bm, cb, wbase, kCoreWin);
      if (qa >= 0 && ca == 0) {
        plist[npend + __popc(ba & lt)] = (uint16_t)qa;
        qmax = max(qmax, qa);
      }
      npend += __popc(ba);
      if (qb >= 0 && cb == 0) {
        plist[npend + __popc(bb & lt)] = (uint16_t)qb;
        qmax = max(qmax, qb);
      }
      npend += __popc(bb);
    }
    if (PGC_SCAN_PREFETCH) {
#pragma unroll
      for (int k = 0; k < kScanStrips; ++k) w[k] = wn[k];
    } else if (i0 + kStep < np) {
#pragma unroll
      for (int k = 0; k < kScanStrips; ++k) {
        const int i = i0 + kStep + 64 * k + 2 * lane;
        w[k] = i < np ? __ldcg(L2 + (i >> 1)) : 0u;
      }
    }
  }
  return np;
}

// Tier 2's scan: int32 codes (k_core2_lists), one per lane and strip; a
// tier-1 pred's color comes from color[] (final), a tier-2 pred's from the
// replica (pending while 0).  Same contract as core_scan.
__device__ __forceinline__ int core_scan2(const int32_t* __restrict__ L, int np, int from,
                                          const uint16_t* cc, const int32_t* color, uint8_t* bm,
                                          int wbase, uint16_t* plist, int& npend, int& qmax) {
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  constexpr int kStep = 32 * kScanStrips;
  constexpr int kNone = (int)0x80000000;
  int w[kScanStrips];
#pragma unroll
  for (int k = 0; k < kScanStrips; ++k) {
    const int i = from + 32 * k + lane;
    w[k] = i < np ? __ldcg(L + i) : kNone;
  }
  for (int i0 = from; i0 < np; i0 += kStep) {
    int wn[kScanStrips], cv[kScanStrips];
#pragma unroll
    for (int k = 0; k < kScanStrips; ++k) {
      const int i = i0 + kStep + 32 * k + lane;
      wn[k] = i < np ? __ldcg(L + i) : kNone;
    }
#pragma unroll
    for (int k = 0; k < kScanStrips; ++k)
      cv[k] = w[k] >= 0 ? ld_vol_u16(cc + w[k]) : (w[k] != kNone ? ld_relaxed(color + (-w[k] - 1)) : 1);
#pragma unroll
    for (int k = 0; k < kScanStrips; ++k) {
      const bool pend = w[k] >= 0 && cv[k] == 0;
      PGC_DCHECK(w[k] >= 0 || w[k] == kNone || cv[k] > 0, -w[k] - 1, cv[k]);  // tier 1 is final
      const unsigned b = __ballot_sync(0xffffffffu, pend);
      if (npend + __popc(b) > kCorePend) return i0 + 32 * k;  // strips before k are complete
      if (w[k] != kNone && cv[k]) bmap_mark(bm, cv[k], wbase, kCoreWin);
      if (pend) {
        plist[npend + __popc(b & lt)] = (uint16_t)w[k];
        qmax = max(qmax, w[k]);
      }
      npend += __popc(b);
    }
#pragma unroll
    for (int k = 0; k < kScanStrips; ++k) w[k] = wn[k];
  }
  return np;
}

template <bool T2>
__global__ void __launch_bounds__(kCoreBlock, 1) k_jp_core(const int4* __restrict__ rec,
                                                           int32_t* P,  // pred lists (u16 core positions; rewritten here if claimed)
                                                           int32_t* color, State* st,
                                                           unsigned long long* tr_grab,
                                                           unsigned long long* tr_done,
                                                           unsigned spin_ns, unsigned tail_ns,
                                                           unsigned pass_ns, int near_n,
                                                           unsigned long long watchdog_ns,
                                                           int32_t* ready,
                                                           const int32_t* __restrict__ pos,
                                                           int NC, int base) {
  // dynamic shared memory: bitmaps | pending lists | color replica [NC] (0 = uncolored)
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint8_t* s_bm = s_dyn;
  uint16_t* s_pend = reinterpret_cast<uint16_t*>(s_dyn + kCoreFixedSmem - kCoreWarps * kCorePend * 2);
  uint16_t* s_cc = reinterpret_cast<uint16_t*>(s_dyn + kCoreFixedSmem);
  __shared__ int s_ticket;
  __shared__ int s_selfserve;  // a list wait timed out: claim lists without waiting
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  for (int i = threadIdx.x; i < NC; i += blockDim.x) s_cc[i] = 0;
  if (threadIdx.x == 0) {
    s_ticket = 0;
    s_selfserve = 0;
  }
  cl.sync();  // every replica is zeroed before any color is published
  // lane r < C publishes into CTA r's replica: its shared::cluster address
  uint32_t remote = 0;
  if (lane < C)
    asm("mapa.shared::cluster.u32 %0, %1, %2;"
        : "=r"(remote)
        : "r"((uint32_t)__cvta_generic_to_shared(s_cc)), "r"(lane));
  const unsigned long long deadline = globaltimer() + watchdog_ns;
  uint8_t* bm = s_bm + warp * kCoreWin;
  uint16_t* plist = s_pend + warp * kCorePend;
  int kmax = 0;
  bool stall = false;
  while (!stall) {
    int k = 0;
    if (lane == 0) k = atomicAdd(&s_ticket, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    // runs of kCoreRun consecutive positions per CTA, runs dealt round-robin:
    // chain hops inside a run stay in local shared memory
    const int p = (rank + C * (k / kCoreRun)) * kCoreRun + (k % kCoreRun);
    if (p >= NC) break;
    const int4 r = rec[base + p];
    const int np = r.y;
    const uint16_t* L = reinterpret_cast<const uint16_t*>(P + lo_hi(r.z, r.w));
    const int32_t* L32 = P + lo_hi(r.z, r.w);  // tier 2: int32 codes
    const int vcore = r.x;
    if (!T2 && ready) {  // k_core_lists runs beside this kernel: p's list must be done
      int act = 0;  // 0: done, 1: rewrite it here, 2: watchdog
      if (lane == 0) {
        const unsigned long long t_give = globaltimer() + 20000;  // 20 us
        for (;;) {
          int f;
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(ready + p) : "memory");
          if (f == kListDone) break;
          if (f == kListTodo && (*(volatile int*)&s_selfserve || globaltimer() > t_give)) {
            if (atomicCAS(ready + p, kListTodo, kListBusy) == kListTodo) {
              *(volatile int*)&s_selfserve = 1;
              act = 1;
              break;
            }
          }
          if (stalled(st, deadline)) {
            st->err = 8;  // (diagnostic: the core waited for a list)
            act = 2;
            break;
          }
          __nanosleep(64);
        }
      }
      act = __shfl_sync(0xffffffffu, act, 0);
      if (act == 2) {
        stall = true;
        break;
      }
      if (act == 1) {
        core_list_rewrite(r, pos, P);
        if (lane == 0) list_release(ready, p);
      }
      __syncwarp();  // lane 0's acquire (or the warp's own rewrite) orders the list loads
    }
#ifdef PGC_PROBE
    const int vprobe = vcore;
    PROBE_STAMP(tr_grab, vprobe, 0);
#else
    if (tr_grab && lane == 0) tr_grab[vcore] = globaltimer();
#endif
    int found = 0;
    for (int wbase = 0; !found && !stall; wbase += kCoreWin) {
      bmap_clear(bm, kCoreWin);
      __syncwarp();
      int npend = 0, qmax = -1;
      int over = T2 ? core_scan2(L32, np, 0, s_cc, color, bm, wbase, plist, npend, qmax)
                    : core_scan(L, np, 0, s_cc, bm, wbase, plist, npend, qmax);
      __syncwarp();
      // zi = the GetColor candidate (first unused color of the window, 0-based),
      // kept current as pending colors arrive so that the last arrival costs
      // one compare
      int zi = bmap_next_zero<kCoreWin>(bm, 0);
      PROBE_STAMP(tr_grab, vprobe, 1);
      unsigned sleep_ns = 0, polls = 0;
      // Reduce the pending set with warp passes until at most kCoreTail preds
      // are left (backing off while nothing arrives, so far-away waiters leave
      // the shared-memory pipe to the warps near the front of the chain).
      for (;;) {
        if (npend == 0) {
          if (over >= np) break;
          over = T2 ? core_scan2(L32, np, over, s_cc, color, bm, wbase, plist, npend, qmax)
                    : core_scan(L, np, over, s_cc, bm, wbase, plist, npend, qmax);
          __syncwarp();
          zi = bmap_next_zero<kCoreWin>(bm, zi);
          continue;
        }
        if (npend <= kCoreTail && over >= np) break;  // the tail below takes them
        int keep = 0;
        for (int j0 = 0; j0 < npend; j0 += 128) {
          int q[4], cc[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int j = j0 + 32 * k + lane;
            q[k] = j < npend ? (int)plist[j] : -1;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) cc[k] = q[k] >= 0 ? ld_vol_u16(s_cc + q[k]) : 1;
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool still = q[k] >= 0 && cc[k] == 0;
            if (q[k] >= 0 && cc[k]) bmap_mark(bm, cc[k], wbase, kCoreWin);
            const unsigned bal = __ballot_sync(0xffffffffu, still);
            if (still) plist[keep + __popc(bal & lt)] = (uint16_t)q[k];
            keep += __popc(bal);
          }
        }
        const bool moved = keep < npend;
        npend = keep;
        __syncwarp();
        PROBE_STAMP(tr_grab, vprobe, 3);
        if (moved) {
          zi = bmap_next_zero<kCoreWin>(bm, zi);
          sleep_ns = 0;
          // rate-limit the passes of a warp still far from its tail: a pass
          // per arrival would take the issue slots of the warps on the chain
          if (pass_ns && npend > 4 * kCoreTail) __nanosleep(pass_ns);
        } else {
          if ((++polls & 63u) == 0 && __shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) {
            st->err = 9;
            stall = true;
            break;
          }
          if (npend <= near_n) {
            sleep_ns = 0;  // a few preds from the tail: poll without backing off
          } else {
            if (sleep_ns) __nanosleep(sleep_ns);
            sleep_ns = sleep_ns ? min(sleep_ns * 2, (unsigned)spin_ns) : (spin_ns ? 32u : 0u);
          }
        }
      }
      if (stall) break;
      if (npend > 0) {
        // Tail -- the critical path of a dependency chain, free of warp
        // collectives (each costs ~40-50 cycles on the chain).  With the used
        // set S of the colors already seen, GetColor after the last npend <=
        // kCoreTail colors c_k arrive is the first of the kCoreTail+1 smallest
        // colors missing from S that no c_k takes.  Those are found now (as a
        // bit mask); then the warp polls all pending preds at once and
        // finishes with a mask and a find-first-set.
        int z[kCoreTail + 1];
        z[0] = zi;
#pragma unroll
        for (int k = 1; k <= kCoreTail; ++k) z[k] = bmap_next_zero<kCoreWin>(bm, min(z[k - 1] + 1, kCoreWin));
        // candidate set as a 32-bit mask relative to z[0] (exact when every
        // candidate lies within 32 colors of z[0]; else the compare loop below)
        unsigned F = 0u;
#pragma unroll
        for (int k = 0; k <= kCoreTail; ++k)
          if (z[k] < kCoreWin && z[k] - z[0] < 32) F |= 1u << (z[k] - z[0]);
        int q[kCoreTail];
#pragma unroll
        for (int k = 0; k < kCoreTail; ++k) q[k] = (int)plist[k < npend ? k : 0];
        const int cbase = wbase + 1 + z[0];  // color -> bit index in F
        PROBE_STAMP(tr_grab, vprobe, 4);
        // all pending preds are polled together (independent loads, one latency
        // per poll; entries past npend repeat q[0]), the watchdog only every
        // 512 polls: the loop is short because every waiting warp of the SM
        // spins here and shares the issue slots with the warps on the chain
        int cc[kCoreTail];
        for (;;) {
          bool all = false;
          for (int it = 0; it < 512; ++it) {
            bool ok = true;
#pragma unroll
            for (int k = 0; k < kCoreTail; ++k) {
              cc[k] = ld_vol_u16(s_cc + q[k]);
              ok &= cc[k] != 0;
            }
            if (ok) {
              all = true;
              break;
            }
          }
          if (all) break;
          if (globaltimer() > deadline) {
            st->err = 9;
            stall = true;
            break;
          }
          if (tail_ns) __nanosleep(tail_ns);
        }
        PROBE_STAMP(tr_grab, vprobe, 5);
        unsigned M = 0u;
#pragma unroll
        for (int k = 0; k < kCoreTail; ++k) M |= shl1(cc[k] - cbase);
        const unsigned G = F & ~M;
        int res;
        if (G) {
          res = z[0] + __ffs(G) - 1;
        } else {  // candidates spread wider than 32 colors or past the window
          res = kCoreWin;
#pragma unroll
          for (int j = kCoreTail; j >= 0; --j) {
            bool taken = false;
#pragma unroll
            for (int k = 0; k < kCoreTail; ++k) taken |= cc[k] - wbase - 1 == z[j];
            if (!taken) res = z[j];
          }
        }
        zi = res;
        npend = 0;
      }
      if (stall) break;  // warp-uniform: every lane read the same timer in the same instruction
      if (zi < kCoreWin) found = wbase + zi + 1;  // GetColor (else: next window)
    }
    PROBE_STAMP(tr_grab, vprobe, 6);
    if (stall) break;
    // publish to every replica: DSMEM stores (relaxed, cluster scope) to the
    // peers, a plain shared store to the own replica (the chain's hops inside
    // a run of kCoreRun positions are local)
#ifndef PGC_LOCAL_PUBLISH
#define PGC_LOCAL_PUBLISH 1
#endif
    if (PGC_LOCAL_PUBLISH && lane == rank)
      *(volatile uint16_t*)(s_cc + p) = (uint16_t)found;
    else if (lane < C)
      asm volatile("st.relaxed.cluster.shared::cluster.u16 [%0], %1;" ::"r"(remote + 2u * (uint32_t)p),
                   "h"((unsigned short)found)
                   : "memory");
    PROBE_STAMP(tr_grab, vprobe, 7);
    PGC_DCHECK(found >= 1 && found <= np + 1, found, np);  // GetColor <= |pred| + 1
    PGC_DCHECK_V(vcore);
    if (lane == 0) {
      st_relaxed(color + vcore, found);
#ifndef PGC_PROBE
      if (tr_done) tr_done[vcore] = globaltimer();
#endif
    }
    kmax = max(kmax, found);
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&st->K, kmax);
  cl.sync();  // no CTA leaves while a peer may still store into its replica
}

// Pred-list and record reads of the bulk are read once: evict-first, so the
// randomly gathered color[] stays in L2 (PGC_JP_LDG keeps the default policy).
__device__ __forceinline__ int jp_stream(const int32_t* p) {
#ifdef PGC_JP_LDG
  return __ldg(p);
#else
  return __ldcs(p);
#endif
}

// ------------------------------------------------------------- bulk ---------
// JP on the rest of the priority order (positions >= core_n) as a sync-free
// dataflow.  The rest is split (stably, so each class stays in priority order)
// into heavy vertices (|pred| > kLightPredMax), colored warp-per-vertex with a
// 2048-color shared-memory bitmap window, and light ones, colored
// lane-per-vertex with a 64-bit used-color mask in registers.  Each class is
// handed out by its own atomic ticket in priority order; a vertex is colored
// by GetColor as soon as every pred's color is nonzero --
// the Join of line 1132 observed by polling.  Deadlock freedom: per class, the
// highest-priority uncolored vertex has all preds colored, and if it is not
// held then no later ticket of its class was handed out either, so a worker of
// its class is free to take it; no worker ever blocks.
constexpr int kLightPredMax = 62;  // light: colors 1..63 fit a u64 mask
constexpr int kJpBlock = 256;
constexpr int kMaxHeavyWarps = 4;  // heavy-path shared buffers exist for this many warps
constexpr int kHeavyWin = 2048;    // colors per heavy byte-map window
constexpr int kPendCap = 256;      // pending-pred list capacity per heavy warp (smem)
constexpr int kHeavyTail = 4;      // preds left for the collective-free heavy tail
#ifndef PGC_LIGHT_BATCH
#define PGC_LIGHT_BATCH 4
#endif
constexpr int kLightBatch = PGC_LIGHT_BATCH;  // pred loads in flight per light lane (re-exam)
#ifndef PGC_LIGHT_VEC
#define PGC_LIGHT_VEC 2
#endif
constexpr int kLV = PGC_LIGHT_VEC;  // 16-byte pred-id loads per first-pass step of a light lane
#ifndef PGC_LIGHT_STEPS
#define PGC_LIGHT_STEPS 2
#endif
#ifndef PGC_LIGHT_Q
#define PGC_LIGHT_Q 32
#endif
constexpr int kLightSteps = PGC_LIGHT_STEPS;  // first-pass steps per lane per loop iteration

// hflag = heavy work items of the vertex (1, or its pred chunks when it is a
// mega vertex), lflag = 1 for a light vertex
__device__ __forceinline__ int mega_chunks(int np, int mega_pred, int mega_chunk) {
  return mega_pred > 0 && np > mega_pred ? (np + mega_chunk - 1) / mega_chunk : 1;
}
__global__ void k_bulk_flags(int64_t n, const int4* __restrict__ rec, const State* st,
                             int32_t* __restrict__ hflag, int32_t* __restrict__ lflag,
                             int mega_pred, int mega_chunk) {
  const int NC = st->core_n;
  for (int64_t p = NC + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int np = rec[p].y;
    hflag[p - NC] = np > kLightPredMax ? mega_chunks(np, mega_pred, mega_chunk) : 0;
    lflag[p - NC] = np > 0 && np <= kLightPredMax ? 1 : 0;
  }
}

// Stable split of the bulk's records (priority order) into heavy and light
// work lists: streaming reads, monotone writes.  Roots of G_rho (no pred: JP
// Part 2's initial set) are colored 1 right here (GetColor
// of the empty set) and listed nowhere.  hpos / lpos are the exclusive prefix
// counts of the heavy / light flags.
__global__ void k_bulk_scatter(int64_t n, const int4* __restrict__ rec, State* st,
                               const int32_t* __restrict__ hpos, const int32_t* __restrict__ lpos,
                               int4* __restrict__ hrec, int4* __restrict__ lrec, int32_t* color,
                               int2* __restrict__ hmeta, uint32_t* __restrict__ mega,
                               int64_t mega_cap, int mega_pred, int mega_chunk) {
  const int NC = st->core_n;
  bool root = false;
  for (int64_t p = NC + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = rec[p];
    const int64_t i = p - NC;
    if (r.y > kLightPredMax) {
      const int nch = mega_chunks(r.y, mega_pred, mega_chunk);
      const int h = hpos[i];
      if (nch == 1) {
        hrec[h] = r;
        hmeta[h] = make_int2(-1, 1);
      } else {
        // a mega vertex: its own used-color set and counter (cleared here, the
        // bulk kernel runs after this one), then one item per pred chunk, in
        // place of the vertex in the priority order (equal priority: no chunk
        // waits on another chunk, so the ticket order stays deadlock-free)
        const int m = atomicAdd(&st->nmega, 1);
        PGC_DCHECK(m < mega_cap, m, mega_cap);
        for (int w = 0; w < kMegaWords; ++w) mega[(int64_t)m * kMegaWords + w] = 0u;
        mega[mega_cap * kMegaWords + m] = 0u;
        const uint64_t slot = ((uint64_t)(uint32_t)r.w << 32) | (uint32_t)r.z;
        for (int k = 0; k < nch; ++k) {
          const uint64_t sk = slot + (uint64_t)k * mega_chunk;
          hrec[h + k] = make_int4(r.x, min(mega_chunk, r.y - k * mega_chunk), (int)(uint32_t)sk,
                                  (int)(uint32_t)(sk >> 32));
          hmeta[h + k] = make_int2(m, nch);
        }
      }
    } else if (r.y > 0) lrec[lpos[i]] = r;
    else {
      st_relaxed(color + r.x, 1);
      root = true;
    }
  }
  if (__any_sync(0xffffffffu, root) && lane_id() == 0) atomicMax(&st->K, 1);
}

__device__ __forceinline__ int64_t rec_slot(const int4& r) {
  return (int64_t)(((uint64_t)(uint32_t)r.w << 32) | (uint32_t)r.z);
}

// Approximate priority key of u (a heuristic for WHICH pending pred to watch,
// never for a result): the first key's 32 bits, then the top 32 hash bits.
// Preds get colored roughly in priority order, so the pending pred of lowest
// key is the one expected to be colored last.
__device__ __forceinline__ unsigned long long watch_key_of(int ru, uint64_t seed, int u) {
  return ((unsigned long long)((uint32_t)ru ^ 0x80000000u) << 32) |
         (prio_hash(seed, (uint32_t)u) >> 32);
}

// Heavy path, one warp per vertex: examine preds [from, np) in strips of 4x32
// (4 independent loads in flight per lane), mark colored ones in the byte map,
// queue pending ones (id and watch key) in the warp's list.  Returns the index
// to resume from when the pending list is full, np when every pred was examined.
#ifndef PGC_HEAVY_STRIPS
#define PGC_HEAVY_STRIPS 4
#endif
constexpr int kHS = PGC_HEAVY_STRIPS;  // strips of 32 preds in flight per heavy-scan step
__device__ __forceinline__ int heavy_scan(const int32_t* __restrict__ P, int64_t pb, int np,
                                          int from, const int32_t* color,
                                          const int32_t* __restrict__ round, uint64_t seed,
                                          uint8_t* bm, int wbase, int* plist,
                                          unsigned long long* pkey, int& npend) {
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  int un[kHS];  // the next step's pred ids, loaded one step ahead
#pragma unroll
  for (int k = 0; k < kHS; ++k) {
    const int i = from + 32 * k + lane;
    un[k] = i < np ? jp_stream(P + pb + i) : -1;
    if (i < np) PGC_DCHECK_V(un[k]);
  }
  for (int i0 = from; i0 < np; i0 += 32 * kHS) {
    int u[kHS], cc[kHS];
#pragma unroll
    for (int k = 0; k < kHS; ++k) u[k] = un[k];
#pragma unroll
    for (int k = 0; k < kHS; ++k) {
      const int i = i0 + 32 * kHS + 32 * k + lane;
      un[k] = i < np ? jp_stream(P + pb + i) : -1;
    }
#pragma unroll
    for (int k = 0; k < kHS; ++k) cc[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 1;
    // first keys of the pending preds (only when some are pending: a ready
    // vertex pays no extra latency), all strips' loads in flight before any
    // is used (a load consumed in its own branch serialises)
    bool anyp = false;
#pragma unroll
    for (int k = 0; k < kHS; ++k) anyp |= u[k] >= 0 && cc[k] == 0;
    int rk[kHS];
#pragma unroll
    for (int k = 0; k < kHS; ++k) rk[k] = 0;
    if (round && __any_sync(0xffffffffu, anyp)) {
#pragma unroll
      for (int k = 0; k < kHS; ++k) rk[k] = __ldg(round + (u[k] >= 0 && cc[k] == 0 ? u[k] : 0));
    }
#pragma unroll
    for (int k = 0; k < kHS; ++k) {
      const bool pend = u[k] >= 0 && cc[k] == 0;
      if (u[k] >= 0 && cc[k]) bmap_mark(bm, cc[k], wbase, kHeavyWin);
      const unsigned bal = __ballot_sync(0xffffffffu, pend);
      const int cnt = __popc(bal);
      if (npend + cnt > kPendCap) return i0 + 32 * k;  // strips before k are complete
      if (pend) {
        const int at = npend + __popc(bal & lt);
        plist[at] = u[k];
        pkey[at] = watch_key_of(rk[k], seed, u[k]);
      }
      npend += cnt;
    }
  }
  return np;
}

// Warp-wide: the pending entries with the lowest and second-lowest watch key
// (their ids; -1 if absent).
__device__ __forceinline__ void lowest_two(const int* plist, const unsigned long long* pkey,
                                           int npend, int& u1, int& u2) {
  const int lane = lane_id();
  unsigned long long k1 = ~0ull, k2 = ~0ull;
  int a1 = -1, a2 = -1;
  for (int j = lane; j < npend; j += 32) {
    const unsigned long long k = pkey[j];
    const int u = plist[j];
    if (k < k1) {
      k2 = k1; a2 = a1; k1 = k; a1 = u;
    } else if (k < k2) {
      k2 = k; a2 = u;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ok1 = __shfl_xor_sync(0xffffffffu, k1, o);
    const unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, k2, o);
    const int oa1 = __shfl_xor_sync(0xffffffffu, a1, o);
    const int oa2 = __shfl_xor_sync(0xffffffffu, a2, o);
    if (ok1 < k1) {  // other's best wins; second = min(my best, other's second)
      if (k1 < ok2) { k2 = k1; a2 = a1; } else { k2 = ok2; a2 = oa2; }
      k1 = ok1; a1 = oa1;
    } else if (ok1 < k2) {
      k2 = ok1; a2 = oa1;
    }
  }
  u1 = a1;
  u2 = a2;
}

#ifndef PGC_BULK_MINB
#define PGC_BULK_MINB 5
#endif
// MEGA: the heavy warps also serve pred chunks of mega vertices.  Two
// instantiations, both launched: each returns at once unless the split found
// mega vertices (nmega > 0) iff it is the MEGA one -- the chunk bookkeeping
// (item meta loads, the set union, the live registers across the pending
// loop) cost the JP-ADG bulk 6 % (1.92 -> 2.04 ms on R-MAT 24) although its
// hubs are in the core and it has no mega vertex.
template <bool MEGA>
__global__ void __launch_bounds__(kJpBlock, PGC_BULK_MINB) k_jp_bulk(const int64_t* __restrict__ off,
                                                     const int32_t* __restrict__ P,
                                                     const int32_t* __restrict__ npred,
                                                     const int4* __restrict__ hrec,
                                                     const int4* __restrict__ lrec,
                                                     const int32_t* __restrict__ round,
                                                     uint64_t seed, int32_t* color,
                                                     State* st, int heavy_warps, int heavy_batch,
                                                     int heavy_stripes,
                                                     unsigned heavy_sleep_max,
                                                     unsigned light_sleep_max,
                                                     unsigned long long* tr_grab,
                                                     unsigned long long* tr_done,
                                                     unsigned long long watchdog_ns,
                                                     const int2* __restrict__ hmeta,
                                                     uint32_t* mega, int64_t mega_cap) {
  if ((st->nmega > 0) != MEGA) return;
  const unsigned long long deadline = globaltimer() + watchdog_ns;
  __shared__ __align__(16) uint8_t s_bm[kMaxHeavyWarps][kHeavyWin];
  __shared__ int s_pend[kMaxHeavyWarps][kPendCap];
  __shared__ unsigned long long s_pkey[kMaxHeavyWarps][kPendCap];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  const int nheavy = st->nheavy;
  int kmax = 0;
  if (warp < heavy_warps) {
    uint8_t* bm = s_bm[warp];
    int* plist = s_pend[warp];
    unsigned long long* pkey = s_pkey[warp];
    // the next ticket and its (vertex, |pred|, P slot) are fetched one vertex
    // ahead, so their dependent loads overlap the current vertex
    // tickets come `heavy_batch` at a time per warp (consecutive, so a held
    // ticket is always of lower priority than the current one: the
    // deadlock-freedom argument of the one-ahead prefetch holds for any batch)
    int q_next = 0, q_end = 0;
    // heavy_stripes > 1: item t belongs to stripe t mod S, each stripe has its
    // own ticket counter on its own line (one counter took ~1 atomic per heavy
    // item on one L2 slice) and its own warps; every stripe is handed out in
    // priority order, so the deadlock-freedom argument holds per stripe (the
    // highest-priority uncolored item, if not held, has no later item of its
    // stripe handed out, and the stripe's earlier items are colored: a warp of
    // its stripe is free)
    const int S = heavy_stripes;
    const int stripe = (blockIdx.x * heavy_warps + warp) % S;
    int* tick = stripe == 0 ? &st->ticket_heavy : &st->ticket_hs[32 * (stripe - 1)];
    auto fetch = [&](int& t, int& v, int& np, int64_t& pb, int2& mm) {
      if (q_next == q_end) {
        int b = 0;
        if (lane == 0) b = atomicAdd(tick, heavy_batch);
        q_next = __shfl_sync(0xffffffffu, b, 0);
        q_end = q_next + heavy_batch;
      }
      const int k = q_next++;
      t = k >= nheavy ? nheavy : stripe + S * k;
      if (t < nheavy) {
        const int4 r = __ldcs(hrec + t);
        v = r.x;
        np = r.y;
        pb = rec_slot(r);
        if (MEGA) mm = __ldcs(hmeta + t);
      }
    };
    int t_next, v_next = 0, np_next = 0;
    int64_t pb_next = 0;
    int2 mm_next = make_int2(-1, 1);
    fetch(t_next, v_next, np_next, pb_next, mm_next);
    for (;;) {
      const int t = t_next;
      if (t >= nheavy) break;
      const int v = v_next;
      int np = np_next;
      int64_t pb = pb_next;
      // a chunk of a mega vertex's preds (m >= 0): window 0 only, every pred
      // waited for, its colors ORed into the vertex's set; the last of the
      // vertex's nch chunks to finish takes GetColor from the union
      int m = MEGA ? mm_next.x : -1;
      const int nch = MEGA ? mm_next.y : 1;
      bool publish = true;
      fetch(t_next, v_next, np_next, pb_next, mm_next);
#ifndef PGC_PROBE
      if (tr_grab && lane == 0) tr_grab[v] = globaltimer();
#endif
      int found = 0;
      for (int wbase = 0; !found; wbase += kHeavyWin) {
        bmap_clear(bm, kHeavyWin);
        __syncwarp();
        int npend = 0;
        int over = heavy_scan(P, pb, np, 0, color, round, seed, bm, wbase, plist, pkey, npend);
        __syncwarp();
        // zi = GetColor candidate (first unused color of the window, 0-based),
        // kept current as pending colors arrive
        int zi = bmap_next_zero<kHeavyWin>(bm, 0);
        unsigned sleep_ns = 0;
        for (;;) {
          if (npend == 0) {
            if (over >= np) break;
            over = heavy_scan(P, pb, np, over, color, round, seed, bm, wbase, plist, pkey, npend);
            __syncwarp();
            zi = bmap_next_zero<kHeavyWin>(bm, zi);
            continue;
          }
          if (npend <= kHeavyTail && over >= np && (!MEGA || m < 0)) break;  // the tail below takes them
          // Several pending: watch the second-to-last expected (one load per
          // poll, exponential backoff), then one pass drops the colored entries.
          int u1, u2;
          lowest_two(plist, pkey, npend, u1, u2);
          const int w = u2 >= 0 ? u2 : u1;
          while (ld_relaxed(color + w) == 0) {
            if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) {
              found = -1;
              break;
            }
            __nanosleep(sleep_ns ? sleep_ns : 16u);
            sleep_ns = sleep_ns ? min(sleep_ns * 2, heavy_sleep_max) : 32u;
          }
          if (found < 0) break;
          sleep_ns = 0;
          int keep = 0;
          for (int j0 = 0; j0 < npend; j0 += 32) {
            const int j = j0 + lane;
            int u = 0, cc = 1;
            unsigned long long kk = 0;
            if (j < npend) {
              u = plist[j];
              kk = pkey[j];
              cc = ld_relaxed(color + u);
            }
            const bool still = j < npend && cc == 0;
            if (j < npend && cc) bmap_mark(bm, cc, wbase, kHeavyWin);
            const unsigned bal = __ballot_sync(0xffffffffu, still);
            __syncwarp();
            if (still) {
              plist[keep + __popc(bal & lt)] = u;
              pkey[keep + __popc(bal & lt)] = kk;
            }
            keep += __popc(bal);
          }
          npend = keep;
          __syncwarp();
          zi = bmap_next_zero<kHeavyWin>(bm, zi);
        }
        __syncwarp();
        if (found < 0) break;  // stalled (watchdog)
        if (npend > 0) {
          // Tail (the critical path of a chain), free of warp collectives: the
          // kHeavyTail+1 smallest colors missing so far are found now; every
          // lane then polls the <= kHeavyTail pending preds (one uniform load
          // per poll) from the highest priority down, and GetColor is the first
          // of those colors no arrival takes.
          int z[kHeavyTail + 1];
          z[0] = zi;
#pragma unroll
          for (int k = 1; k <= kHeavyTail; ++k)
            z[k] = bmap_next_zero<kHeavyWin>(bm, min(z[k - 1] + 1, kHeavyWin));
          int q[kHeavyTail];
          unsigned long long qk[kHeavyTail];
#pragma unroll
          for (int k = 0; k < kHeavyTail; ++k) {
            q[k] = k < npend ? plist[k] : -1;
            qk[k] = k < npend ? pkey[k] : 0ull;
          }
#pragma unroll
          for (int i = 1; i < kHeavyTail; ++i)  // descending priority key
#pragma unroll
            for (int k = kHeavyTail - 1; k > 0; --k)
              if (qk[k] > qk[k - 1]) {
                const unsigned long long tk = qk[k];
                qk[k] = qk[k - 1];
                qk[k - 1] = tk;
                const int t = q[k];
                q[k] = q[k - 1];
                q[k - 1] = t;
              }
          int cl[kHeavyTail];
          bool stl = false;
#pragma unroll
          for (int k = 0; k < kHeavyTail; ++k) {
            int c = 0;
            if (q[k] >= 0 && !stl) {
              unsigned spins = 0;
              while ((c = ld_relaxed(color + q[k])) == 0) {
                if ((++spins & 4095u) == 0 && globaltimer() > deadline) {
                  st->err = 5;
                  stl = true;
                  break;
                }
              }
            }
            cl[k] = q[k] >= 0 ? c - wbase - 1 : -1;
          }
          if (stl) {
            found = -1;
            break;
          }
          int res = kHeavyWin;
#pragma unroll
          for (int j = kHeavyTail; j >= 0; --j) {
            bool taken = false;
#pragma unroll
            for (int k = 0; k < kHeavyTail; ++k) taken |= cl[k] == z[j];
            if (!taken) res = z[j];
          }
          zi = res;
          npend = 0;
        }
        if (MEGA && m >= 0) {
          // (npend == 0 and every pred of the chunk examined: bm holds all of
          // the chunk's colors <= kMegaBits) byte map -> bits, OR into the set
          static_assert(kMegaBits == kHeavyWin, "one window per chunk");
          uint32_t* mbits = mega + (int64_t)m * kMegaWords;
#pragma unroll
          for (int h = 0; h < kMegaWords / 32; ++h) {
            const int w = lane + 32 * h;
            const uint4 b0 = *reinterpret_cast<const uint4*>(bm + 32 * w);
            const uint4 b1 = *reinterpret_cast<const uint4*>(bm + 32 * w + 16);
            const uint32_t by[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            uint32_t bits = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
              for (int y = 0; y < 4; ++y)
                if ((by[q] >> (8 * y)) & 0xffu) bits |= 1u << (4 * q + y);
            if (bits) atomicOr(mbits + w, bits);
          }
          __threadfence();
          __syncwarp();
          int last = 0;
          if (lane == 0)
            last = atomicAdd(mega + mega_cap * kMegaWords + m, 1) == nch - 1;
          last = __shfl_sync(0xffffffffu, last, 0);
          if (!last) {
            publish = false;
            break;
          }
          __threadfence();  // every other chunk's ORs precede its count
          int z = kMegaBits;
#pragma unroll
          for (int h = 0; h < kMegaWords / 32; ++h) {
            const uint32_t free_bits = ~__ldcg(mbits + lane + 32 * h);
            const unsigned any = __ballot_sync(0xffffffffu, free_bits != 0u);
            if (any && z == kMegaBits) {  // (warp-uniform)
              const int wl = __ffs(any) - 1;
              const uint32_t fb = __shfl_sync(0xffffffffu, free_bits, wl);
              z = 32 * (wl + 32 * h) + __ffs(fb) - 1;
            }
          }
          if (z < kMegaBits) {
            found = z + 1;  // GetColor over all of v's preds
            break;
          }
          // colors 1..kMegaBits all taken (every pred is colored by now): the
          // whole-vertex window loop over v's full list from the next window
          m = -1;
          pb = off[v];
          np = npred[v];
          __syncwarp();
          continue;
        }
        if (zi < kHeavyWin) found = wbase + zi + 1;  // GetColor (else: next window)
        __syncwarp();
      }
      if (found < 0) break;  // stalled: the host reports PGC_EINTERNAL
      if (MEGA && !publish) continue;  // a chunk of a mega vertex another warp finishes
#ifdef PGC_CHECKED
      if (nch > 1) np = npred[v];
#endif
      PGC_DCHECK(found >= 1 && found <= np + 1, found, np);  // GetColor <= |pred| + 1
      if (lane == 0) {
        st_relaxed(color + v, found);
        if (tr_done) tr_done[v] = globaltimer();
      }
      kmax = max(kmax, found);
    }
  } else {
    // Light vertices, one per lane; every lane refills independently (a lane
    // whose vertex waits never holds up the others).  A new vertex's preds are
    // scanned by its lane (kLightBatch loads in flight): colors go into a
    // 64-bit used-color mask, uncolored preds into a pending bit set; the lane
    // then watches ONE pending pred (the lowest pending index) with a single
    // load per poll and re-examines the rest only when it is colored.
    const int64_t nlight = st->nlight;
    int v = -1, np = 0, watch_j = -1, watch_u = -1;
    int64_t pb = 0, pe = 0, scan = 0;  // scan: next P slot of the first pass (pe: done)
    unsigned long long mask = 0, pend = 0;
    unsigned sleep_ns = 32;
    int4 nx = make_int4(0, 0, 0, 0);  // prefetched next record
    bool have_nx = false;
    // the warp's ticket queue [q_t, q_t + q_n): light tickets are taken 32 at a
    // time (one atomic on the shared counter per 32 vertices, not per refill)
    // and handed to the lanes in order, so every ticket the warp holds but has
    // not started is of lower priority than the ones it has started (the
    // deadlock-freedom argument of the prefetch, k_bucket_sort)
    constexpr int kLightQ = PGC_LIGHT_Q;  // tickets per refill of the queue (>= 32)
    int q_t = 0, q_n = 0;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(&st->ticket_light, 32);
      const int64_t t = (int64_t)__shfl_sync(0xffffffffu, t0, 0) + lane;
      if (t < nlight) {
        nx = __ldcs(lrec + t);
        have_nx = true;
      }
    }
    for (;;) {
      bool progress = false;
      // 1. free lanes take their prefetched record, then re-arm the prefetch
      //    with the next light tickets (one atomic per warp): the ticket and
      //    record loads of the NEXT vertex overlap the scan of this one
      const bool take = v < 0 && have_nx;
      if (take) {
        v = nx.x;
        np = nx.y;
        pb = rec_slot(nx);
        have_nx = false;
      }
      const unsigned want = __ballot_sync(0xffffffffu, take);
      if (want) {
        const int need = __popc(want);
        int fresh = 0;
        if (need > q_n) {  // the queue runs dry: a fresh block of 32 tickets
          const int leader = __ffs(want) - 1;
          if (lane == leader) fresh = atomicAdd(&st->ticket_light, kLightQ);
          fresh = __shfl_sync(0xffffffffu, fresh, leader);
        }
        if (take) {
          const int rank = __popc(want & lt);
          const int64_t t = rank < q_n ? (int64_t)q_t + rank : (int64_t)fresh + (rank - q_n);
          if (t < nlight) {
            nx = __ldcs(lrec + t);
            have_nx = true;
          }
        }
        if (need > q_n) {
          q_t = fresh + (need - q_n);
          q_n = kLightQ - (need - q_n);
        } else {
          q_t += need;
          q_n -= need;
        }
      }
      if (take) {
#ifndef PGC_PROBE
        if (tr_grab) tr_grab[v] = globaltimer();
#endif
        mask = 1ull;  // bit 0 reserved: colors start at 1
        pend = 0ull;
        watch_j = -1;
        watch_u = -1;
        pe = pb + np;
        scan = pb & ~3ll;
      }
      // first pass over the preds, at most kLightSteps steps per iteration (the
      // warp's lanes run in lockstep: one long list must not hold up the
      // lanes that could finish and refill).  Pred ids by aligned 16-byte loads,
      // 4 * kLV slots per step (slots outside [pb, pe) belong to neighbouring
      // lists: ignored), then their color gathers in flight.
      for (int step = 0; step < kLightSteps && v >= 0 && scan < pe; ++step) {
        const int64_t s0 = scan;
        int u[4 * kLV], cc[4 * kLV];
#pragma unroll
        for (int q = 0; q < kLV; ++q) {
          const int4 w = (q == 0 || s0 + 4 * q < pe)
                             ? __ldcs(reinterpret_cast<const int4*>(P + s0 + 4 * q))
                             : make_int4(-1, -1, -1, -1);
          u[4 * q] = w.x;
          u[4 * q + 1] = w.y;
          u[4 * q + 2] = w.z;
          u[4 * q + 3] = w.w;
        }
#pragma unroll
        for (int k = 0; k < 4 * kLV; ++k)
          if (s0 + k < pb || s0 + k >= pe) u[k] = -1;
#pragma unroll
        for (int k = 0; k < 4 * kLV; ++k) {
          if (u[k] >= 0) PGC_DCHECK_V(u[k]);
          cc[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 1;
        }
#pragma unroll
        for (int k = 0; k < 4 * kLV; ++k) {
          if (u[k] < 0) continue;
          const int j = (int)(s0 + k - pb);
          if (cc[k] == 0) {
            pend |= 1ull << j;
            if (watch_j < 0) {  // watch the first pending pred
              watch_j = j;
              watch_u = u[k];
            }
          } else if (cc[k] < 64) {
            mask |= 1ull << cc[k];
          }
        }
        scan = s0 + 4 * kLV;
        progress = true;
      }
      const bool scanned = v >= 0 && scan >= pe;
      if (__ballot_sync(0xffffffffu, v >= 0 || have_nx) == 0) break;  // all free, out of tickets
      // 2. poll the watched pred; when colored, re-examine the other pending preds
      if (scanned && watch_u >= 0) {
        const int cw = ld_relaxed(color + watch_u);
        if (cw) {
          if (cw < 64) mask |= 1ull << cw;
          pend &= ~(1ull << watch_j);
          progress = true;
          unsigned long long q = pend;
          watch_j = -1;
          watch_u = -1;
          while (q) {
            int js[kLightBatch], u[kLightBatch], cc[kLightBatch];
#pragma unroll
            for (int k = 0; k < kLightBatch; ++k) {
              js[k] = q ? __ffsll((long long)q) - 1 : -1;
              q &= q - 1;
            }
#pragma unroll
            for (int k = 0; k < kLightBatch; ++k) u[k] = js[k] >= 0 ? __ldg(P + pb + js[k]) : -1;
#pragma unroll
            for (int k = 0; k < kLightBatch; ++k) cc[k] = u[k] >= 0 ? ld_relaxed(color + u[k]) : 0;
#pragma unroll
            for (int k = 0; k < kLightBatch; ++k) {
              if (u[k] < 0) continue;
              if (cc[k]) {
                if (cc[k] < 64) mask |= 1ull << cc[k];
                pend &= ~(1ull << js[k]);
              } else if (watch_j < 0) {
                watch_j = js[k];
                watch_u = u[k];
              }
            }
          }
        }
      }
      // 3. GetColor once nothing is pending: the smallest color the preds do not use
      if (scanned && watch_u < 0) {
        const int cc = __ffsll((long long)~mask) - 1;
        PGC_DCHECK(cc >= 1 && cc <= (int)(pe - pb) + 1, cc, pe - pb);  // GetColor <= |pred| + 1
        st_relaxed(color + v, cc);
        if (tr_done) tr_done[v] = globaltimer();
        kmax = max(kmax, cc);
        v = -1;
        progress = true;
      }
      if (__ballot_sync(0xffffffffu, progress)) {
        sleep_ns = 32;
      } else {
        if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) break;
        __nanosleep(sleep_ns);
        sleep_ns = min(sleep_ns * 2, light_sleep_max);
      }
    }
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&st->K, kmax);
}

// J, the depth of JP (diagnostics; pgc_set_tuning("levels", 1)): level[v] =
// 1 + max level over pred(v) (roots: 1), J = max level = the number of
// vertices on a longest path of G_rho -- the quantity Alg. 3's depth is written
// in (Lemma 6, 1192-1294).  A dataflow over the priority
// order after JP has finished (every pred list is final): warp per vertex,
// tickets in priority order (deadlock-free: the highest-priority unfinished
// vertex is held by a warp whose preds are all finished, or not yet handed
// out, and then every warp is free), each lane polls its preds' levels (0 =
// not yet).  Core positions p < core_n1 hold u16 core positions in their P slot
// (k_core_lists), tier-2 positions int32 codes (k_core2_lists), both mapped
// back to ids through rec[].  lvl[] (n ints) starts at 0.
__global__ void k_jp_levels(const int4* __restrict__ rec, const int32_t* __restrict__ P,
                            int32_t* lvl, State* st, unsigned long long watchdog_ns) {
  const int lane = lane_id();
  const int no = st->n_order, NC = st->core_n, N1 = st->core_n1;
  const unsigned long long deadline = globaltimer() + watchdog_ns;
  int jmax = 0;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(&st->ticket_levels, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= no) break;
    const int4 r = rec[t];
    const int np = r.y;
    const int64_t pb = lo_hi(r.z, r.w);
    int mx = 0;
    bool stall = false;
    for (int i0 = 0; i0 < np && !stall; i0 += 32) {
      const int i = i0 + lane;
      int u = -1;
      if (i < np) {
        if (t < N1) {  // tier 1: u16 core positions
          u = rec[reinterpret_cast<const uint16_t*>(P + pb)[i]].x;
        } else if (t < NC) {  // tier 2: int32 codes
          const int code = P[pb + i];
          u = code >= 0 ? rec[N1 + code].x : -code - 1;
        } else {
          u = P[pb + i];
        }
      }
      int x = u >= 0 ? ld_relaxed(lvl + u) : 1;
      while (__any_sync(0xffffffffu, x == 0)) {
        if (__shfl_sync(0xffffffffu, (int)stalled(st, deadline), 0)) {
          stall = true;
          break;
        }
        __nanosleep(64);
        if (x == 0) x = ld_relaxed(lvl + u);
      }
      mx = max(mx, x);
    }
    if (stall) break;
    mx = warp_max(mx);
    if (lane == 0) st_relaxed(lvl + r.x, mx + 1);
    jmax = max(jmax, mx + 1);
  }
  if (lane == 0 && jmax) atomicMax(&st->jp_levels, jmax);
}

// K starts at 1 for a nonempty graph: the highest-priority vertex has no pred
// and gets color 1 (isolated vertices and roots are colored outside the JP kernels).
__global__ void k_jp_reset(State* st, int nonempty) {
  st->ticket_heavy = 0;
  for (int k = 0; k < kMaxHeavyStripes - 1; ++k) st->ticket_hs[32 * k] = 0;
  st->ticket_light = 0;
  st->ticket_levels = 0;
  st->jp_levels = nonempty;  // isolated vertices and roots are level 1
  st->nheavy = 0;
  st->nmega = 0;
  st->K = nonempty;
  st->core_n = 0;
  st->core_n1 = 0;
  st->core_arcs = 0;
}

// Largest cluster size (power of two <= want) that k_jp_core can launch with
// `smem` dynamic bytes; 0 if none.
// The attributes are set once per device (the dynamic shared memory opt-in at
// the largest core's size) and the answer is cached per (device, want, smem):
// the occupancy query sat on the critical path of every call (the host is
// between k_core_select's read-back and the core launch; 35 us gap in the
// kernel timeline, profiles/r2_b/timeline_rmat24.json).
static int core_cluster_size(int dev, int want, size_t smem) {
  bool& attr_done = once_flag(dev, 8);  // per device: attributes belong to one device
  if (!attr_done) {
    // both tiers' instantiations (attributes are per function)
    for (const void* f : {(const void*)k_jp_core<false>, (const void*)k_jp_core<true>}) {
      if (cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        cudaGetLastError();  // then only portable sizes (<= 8) are found below
      // the largest core's size (64 KB + 2 x 65 536 B): every later launch fits under it
      if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(kCoreFixedSmem + 2 * (size_t)kCoreCap)) != cudaSuccess) {
        cudaGetLastError();
        return 0;  // (retried on the next call)
      }
    }
    attr_done = true;
  }
  struct E { int dev, want; size_t smem; int C; };
  static thread_local E cache[16];
  static thread_local int ncache = 0;
  for (int i = 0; i < ncache; ++i)
    if (cache[i].dev == dev && cache[i].want == want && cache[i].smem == smem) return cache[i].C;
  int found = 0;
  for (int C = want; C >= 1 && !found; C >>= 1) {
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
    if (cudaOccupancyMaxActiveClusters(&nclusters, k_jp_core<false>, &cfg) == cudaSuccess &&
        nclusters >= 1)
      found = C;
    else
      cudaGetLastError();
  }
  cache[ncache < 16 ? ncache++ : 15] = {dev, want, smem, found};
  return found;
}

static int cuda_ok(cudaError_t e, const char* where) { return e == cudaSuccess ? 0 : cuda_fail(e, where); }

static int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

int jp_color_run(Ctx& c, int32_t* color) {
  NvtxRange nvtx_("pgc JP Part 2 (core + bulk)");
  PGC_CHK_SIZES(c);
  PGC_LAUNCH(c, kGJp, "k_jp_reset", k_jp_reset<<<1, 1, 0, c.st>>>(c.state, c.n > 0 ? 1 : 0));
  int64_t n_order = 0;
  if (c.n > 0) {
    // --- core selection and its pred-list rewrite ---
    int C = 0, C2 = 0, NC1 = 0, NC2 = 0;
    size_t core_smem = 0, core_smem2 = 0;
    if (c.tune.core_max > 0) {
      PGC_LAUNCH(c, kGCore, "k_core_select",
                 k_core_select<<<1, 1024, 0, c.st>>>(c.rec, c.state,
                                                      c.tune.core_max, c.tune.core_min_avg,
                                                      c.tune.core_arc_cap, c.tune.core_tier2,
                                                      c.tune.core_div, c.tune.core_dmul));
      if (int e = sync_state(c)) return e;
      const int NC = c.h_state->core_n1;
      NC2 = c.h_state->core_n - NC;
      const long long arcs = c.h_state->core_arcs;
      core_smem = kCoreFixedSmem + (((size_t)NC * 2 + 15) & ~(size_t)15);
      core_smem2 = kCoreFixedSmem + (((size_t)NC2 * 2 + 15) & ~(size_t)15);
      if (NC >= c.tune.core_min_n) {
        // CTAs for the arcs AND for the chain: each CTA keeps 32 vertices in
        // flight, and a long prefix needs many in flight even when its lists
        // are short (R-MAT 20: 65 535 core vertices, 22 M arcs -- 4 CTAs by
        // arcs, 1.86 ms; 16 CTAs, 1.00 ms)
        const long long by_arcs = (arcs + c.tune.core_arcs_per_cta - 1) / c.tune.core_arcs_per_cta;
        const long long by_verts = (NC + kCoreVertsPerCta - 1) / kCoreVertsPerCta;
        int want = c.tune.core_ctas > 0 ? c.tune.core_ctas
                                        : (int)(by_arcs > by_verts ? by_arcs : by_verts);
        want = pow2_floor(want < 1 ? 1 : (want > 16 ? 16 : want));
        C = core_cluster_size(c.dev, want, core_smem);
        if (C > 0 && NC2 > 0) C2 = core_cluster_size(c.dev, want, core_smem2);
      }
      if (C == 0) {
        static_assert(offsetof(State, core_n1) == offsetof(State, core_n) + sizeof(int),
                      "core_n, core_n1 adjacent");
        PGC_CUDA(cudaMemsetAsync(&c.state->core_n, 0, 2 * sizeof(int), c.st));
        NC1 = NC2 = 0;
      } else {
        if (C2 == 0 && NC2 > 0) {  // no cluster for tier 2: the bulk takes its positions
          PGC_CUDA(cudaMemcpyAsync(&c.state->core_n, &c.state->core_n1, sizeof(int),
                                   cudaMemcpyDeviceToDevice, c.st));
          NC2 = 0;
        }
        NC1 = NC;
        c.core_ctas = C;
        c.core_n = NC + NC2;
      }
    }
    // --- bulk split of positions [core_n, n_order) (needs only the records)
    //     and the core kernel: the core is one cluster of <= 16 SMs, so the
    //     split runs beside it on a second stream (it writes only the bulk's
    //     lists, the bulk's colors and its own counters; the core's pos[]
    //     in D is dead once k_core_lists has run) ---
    if (c.tune.core_max <= 0)
      if (int e = sync_state(c)) return e;
    n_order = c.h_state->n_order;
    const int NC = c.core_n;
    const int64_t nbulk = n_order - NC;
    int4* hrec = c.rec + c.n;
    int4* lrec = hrec + c.lay.rec_heavy_cap;
    const bool fork = C > 0 && nbulk > 0 && c.tune.jp_split_overlap;
    if (fork) {
      // CUDA loads kernels lazily at their first launch, and loading waits for
      // the running kernels: a side-stream kernel the core waits on (the list
      // rewrite) must be loaded before the core starts, or the first call
      // deadlocks until the watchdog.  Querying the attributes loads them.
      bool& loaded = once_flag(c.dev, 9);  // per device: modules are per context
      if (!loaded) {
        cudaFuncAttributes fa;
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_core_pos));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_core_lists));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_core2_lists));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_jp_core<true>));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_hist2));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_scatter));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_bucket_sort));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_bulk_flags));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_bulk_scatter));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_scan_reduce));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_scan_tmp));
        PGC_CUDA(cudaFuncGetAttributes(&fa, k_scan_down));
        loaded = true;
      }
    }
    // the core's list rewrite: before the core, or beside it with per-vertex
    // ready flags (the ADG filter buffers, free during JP, zeroed on the main
    // stream before the fork)
    int32_t* ready = fork ? reinterpret_cast<int32_t*>(c.filt) : nullptr;
    // pos[] before the fork (the core may rewrite lists itself), in the upper
    // half of the round-histogram space: the bulk split reuses D beside the core
    int32_t* pos = c.hist1 + c.lay.range_cap;
    if (C > 0)
      PGC_LAUNCH(c, kGCore, "k_core_pos",
                 k_core_pos<<<c.nsm * 4, 256, 0, c.st>>>(c.rec, c.state, pos, ready));
    auto lists = [&]() -> int {
      PGC_LAUNCH(c, kGCore, "k_core_lists",
                 k_core_lists<<<c.nsm * 8, 256, 0, c.st>>>(c.rec, pos, c.P, c.state, ready));
      return 0;
    };
    if (C > 0 && !fork)
      if (int e = lists()) return e;
    // tier 2's lists -> int32 codes (needs only pos[]: beside tier 1 when forked)
    auto lists2 = [&]() -> int {
      PGC_LAUNCH(c, kGCore, "k_core2_lists",
                 k_core2_lists<<<c.nsm * 8, 256, 0, c.st>>>(c.rec, pos, c.P, c.state));
      return 0;
    };
    auto split = [&]() -> int {
      if (c.ord_pending)  // the rest of the priority order first (same stream)
        if (int e = jp_order_bottom(c)) return e;
      if (nbulk <= 0) return 0;
      const int G = c.nsm * 8;
      // flags: heavy -> U0, light -> U1; prefix counts: heavy -> Rl, light -> D
      // (ADG's lists and degrees, and the core's pos[], are dead by now)
      int32_t* hflag = c.U[0];
      int32_t* lflag = c.U[1];
      int32_t* hpos = c.Rl;
      int32_t* lpos = c.D;
      PGC_LAUNCH(c, kGJp, "k_bulk_flags",
                 k_bulk_flags<<<G, 256, 0, c.st>>>(n_order, c.rec, c.state, hflag, lflag,
                                                   c.tune.jp_mega_pred, c.tune.jp_mega_chunk));
      if (int e = scan_ex(c, hflag, hpos, nullptr, nbulk, nbulk, &c.state->nheavy, kGJp)) return e;
      if (int e = scan_ex(c, lflag, lpos, nullptr, nbulk, nbulk, &c.state->nlight, kGJp)) return e;
      PGC_LAUNCH(c, kGJp, "k_bulk_scatter",
                 k_bulk_scatter<<<G, 256, 0, c.st>>>(n_order, c.rec, c.state, hpos, lpos, hrec, lrec,
                                                     color, c.hmeta, c.mega, c.lay.mega_cap,
                                                     c.tune.jp_mega_pred, c.tune.jp_mega_chunk));
      return 0;
    };
    // tier 1: positions [0, NC1) with u16 lists (rewritten beside it when
    // forked); tier 2: [NC1, NC1 + NC2) with int32 codes, after tier 1
    auto core = [&](bool t2) -> int {
      const int CC = t2 ? C2 : C;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CC);
      cfg.blockDim = dim3(kCoreBlock);
      cfg.dynamicSmemBytes = t2 ? core_smem2 : core_smem;
      cfg.stream = c.st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CC;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const unsigned long long wd = (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull;
      if (t2)
        PGC_LAUNCH(c, kGCore, "k_jp_core<tier2>",
                   PGC_CUDA(cudaLaunchKernelEx(&cfg, k_jp_core<true>, (const int4*)c.rec, c.P, color,
                                               c.state, c.trace_grab, c.trace_done,
                                               (unsigned)c.tune.core_spin_ns,
                                               (unsigned)c.tune.core_tail_ns,
                                               (unsigned)c.tune.core_pass_ns, c.tune.core_near, wd,
                                               (int32_t*)nullptr, (const int32_t*)pos, NC2, NC1)));
      else
        PGC_LAUNCH(c, kGCore, "k_jp_core",
                   PGC_CUDA(cudaLaunchKernelEx(&cfg, k_jp_core<false>, (const int4*)c.rec, c.P, color,
                                               c.state, c.trace_grab, c.trace_done,
                                               (unsigned)c.tune.core_spin_ns,
                                               (unsigned)c.tune.core_tail_ns,
                                               (unsigned)c.tune.core_pass_ns, c.tune.core_near, wd,
                                               ready, (const int32_t*)pos, NC1, 0)));
      return 0;
    };
    if (fork) {
      // fork: the core first (it is launched first and finds its SMs free);
      // the list rewrite, the rest of the order and the bulk split on the side
      // stream; join before the bulk
      // per thread and device (streams and events belong to one device)
      static thread_local cudaStream_t sides[kMaxDevices] = {};
      static thread_local cudaEvent_t evs[kMaxDevices][3] = {};
      cudaStream_t& side = sides[c.dev];
      cudaEvent_t* ev = evs[c.dev];
      if (!side) {
        PGC_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        for (int i = 0; i < 3; ++i) PGC_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
      }
      static_assert(65535 * 4 <= 2 * kFilterBytes, "list states fit the filter buffers");
      PGC_CUDA(cudaEventRecord(ev[0], c.st));  // (ready[] was cleared by k_core_pos)
      if (int e = core(false)) return e;
      PGC_CUDA(cudaStreamWaitEvent(side, ev[0], 0));
      const cudaStream_t main = c.st;
      c.st = side;
      int e = lists();
      if (!e && NC2 > 0) {  // tier 2's lists next on the side stream; tier 2 waits for them
        e = lists2();
        if (!e) e = cuda_ok(cudaEventRecord(ev[2], side), "cudaEventRecord(tier2 lists)");
      }
      if (!e) e = split();
      c.st = main;
      if (!e && NC2 > 0) {
        e = cuda_ok(cudaStreamWaitEvent(c.st, ev[2], 0), "cudaStreamWaitEvent(tier2 lists)");
        if (!e) e = core(true);
      }
      if (e) {
        cudaStreamSynchronize(side);  // nothing may stay in flight on the error path
        return e;
      }
      PGC_CUDA(cudaEventRecord(ev[1], side));
      PGC_CUDA(cudaStreamWaitEvent(c.st, ev[1], 0));
    } else {
      // (pos[] is read by the list rewrites: both before the split, which
      // may reuse its space)
      if (NC2 > 0)
        if (int e = lists2()) return e;
      if (int e = split()) return e;
      if (C > 0)
        if (int e = core(false)) return e;
      if (NC2 > 0)
        if (int e = core(true)) return e;
    }
    // --- bulk dataflow ---
    if (nbulk > 0) {
      const int GB = wave_grid(c, k_jp_bulk<false>, kJpBlock);
      PGC_LAUNCH(c, kGJp, "k_jp_bulk",
                 k_jp_bulk<false><<<GB, kJpBlock, 0, c.st>>>(
                     c.off, c.P, c.npred, hrec, lrec, c.round_key, c.seed, color, c.state,
                     c.tune.jp_heavy_warps, c.tune.jp_heavy_batch, c.tune.jp_heavy_stripes,
                     (unsigned)c.tune.jp_heavy_sleep_max,
                     (unsigned)c.tune.jp_light_sleep_max, c.trace_grab, c.trace_done,
                     (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull, c.hmeta, c.mega,
                     c.lay.mega_cap));
      if (c.tune.jp_mega_pred > 0) {  // (nmega > 0 needs the knob: else no launch at all)
        const int GM = wave_grid(c, k_jp_bulk<true>, kJpBlock);
        PGC_LAUNCH(c, kGJp, "k_jp_bulk_mega",
                   k_jp_bulk<true><<<GM, kJpBlock, 0, c.st>>>(
                       c.off, c.P, c.npred, hrec, lrec, c.round_key, c.seed, color, c.state,
                       c.tune.jp_heavy_warps, c.tune.jp_heavy_batch, c.tune.jp_heavy_stripes,
                       (unsigned)c.tune.jp_heavy_sleep_max,
                       (unsigned)c.tune.jp_light_sleep_max, c.trace_grab, c.trace_done,
                       (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull, c.hmeta, c.mega,
                       c.lay.mega_cap));
      }
    }
  }
  if (c.tune.levels && n_order > 0) {
    // lvl[] in D: free once the bulk (its split's prefix counts) has finished
    PGC_CUDA(cudaMemsetAsync(c.D, 0, 4 * (size_t)c.n, c.st));
    PGC_LAUNCH(c, kGJp, "k_jp_levels",
               k_jp_levels<<<c.nsm * 8, 256, 0, c.st>>>(
                   c.rec, c.P, c.D, c.state, (unsigned long long)c.tune.jp_watchdog_ms * 1000000ull));
  }
  if (int e = sync_state(c)) return e;
  c.jp_levels = c.tune.levels ? c.h_state->jp_levels : 0;
  if (c.h_state->err == 9)
    return fail(4, "JP core stalled: no progress within %d ms (watchdog)", c.tune.jp_watchdog_ms);
  if (c.h_state->err == 8)
    return fail(4, "JP core stalled waiting for a rewritten pred list (watchdog)");
  if (c.h_state->err == 5)
    return fail(4, "JP coloring stalled: no progress within %d ms (watchdog)", c.tune.jp_watchdog_ms);
  const long long placed =
      (long long)c.h_state->sorted + (c.ord_deferred ? c.h_state->sorted_bot : 0);
  if (c.n > 0 && placed != n_order)
    return fail(4, "priority order placed %lld of %lld vertices", placed, (long long)n_order);
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
  PGC_CHK_SIZES(c);
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
