// dec.cu -- DEC-ADG-ITR: ADG's partitions R(l) colored
// from the densest (l = T) down, each by SIM-COL with
// ITR's deterministic Part 1 -- the smallest color not used by an already
// colored neighbour -- and the conflict rule of reading Q23 (a vertex gives its
// tentative color up only to a same-colored active neighbour of larger
// h = splitmix64(seed ^ v)).
//
// One persistent cooperative kernel per partition (no launch per pass):
//   prep           B_v so far (the colors of v's neighbours in the colored
//                  partitions) summarised as base = mex(B_v) and a 64-bit mask
//                  of the free colors base..base+63; v's neighbours inside
//                  R(l) listed in its CSR slot of P (every pass reads only those)
//   loop over SIM-COL passes while the active list A is not empty:
//     Part 1       tent[v] = the smallest cached candidate not taken by an
//                  intra-partition neighbour colored in an earlier pass (all 64
//                  taken -- a dense partition -- : rescan, refresh the summary)
//     Part 2       won[v] = no active intra-partition neighbour u (color[u] ==
//                  0) has tent[u] == tent[v] and h(u) > h(v)
//     Part 3       color[v] = tent[v] for the winners (their colors reach the
//                  neighbours' B through the next Part 1), the others are
//                  compacted into the next list (U = U \ {colored})
//   with a grid barrier between the parts, so "active" in Part 2 is the state
//   at the start of the pass, as in the listing.  Data written by other blocks
//   is read with ld.cg (L1 is not coherent inside one kernel).
// The partitions are contiguous ranges of the priority order (jp_order_run
// sorts by round).
#include <cooperative_groups.h>

#include <cstdio>
#include <vector>

#include "pgc_internal.cuh"

namespace pgc {

namespace cg = cooperative_groups;

constexpr int kItrWin = 1024;  // colors per byte-map window
constexpr int kItrBlock = 256;
#ifndef PGC_ITR_STRIPS
#define PGC_ITR_STRIPS 4
#endif
constexpr int kItrStrips = PGC_ITR_STRIPS;  // strips of 32 neighbour loads in flight per pass step

__device__ __forceinline__ int ldcg(const int32_t* p) { return __ldcg(p); }

// mex over the colors of the colored vertices in two lists (a warp, byte-map
// windows); also the free mask of the 64 colors from the mex on (bits past the
// window: taken).  The lists are v's neighbours in R(l) and in the colored
// partitions: every neighbour that can be colored while R(l) is.
__device__ __forceinline__ int itr_full_mex(const int32_t* la, int na_, const int32_t* lb, int nb_,
                                            const int32_t* color, uint8_t* bm,
                                            unsigned long long& fm) {
  const int lane = lane_id();
  const int64_t b = 0, e = (int64_t)na_ + nb_;
  int found = 0;
  fm = 0;
  for (int wbase = 0; !found; wbase += kItrWin) {
    for (int j = lane; j < kItrWin / 16; j += 32) reinterpret_cast<uint4*>(bm)[j] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    // 8 strips of 32 arcs per step, all loads in flight (a hub's list is long)
    for (int64_t a0 = b; a0 < e; a0 += 256) {
      int u[8], c[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t x = a0 + 32 * k + lane;
        u[k] = x < e ? ldcg(x < na_ ? la + x : lb + (x - na_)) : -1;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = u[k] >= 0 ? ldcg(color + u[k]) : 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int q = c[k] - wbase - 1;
        if (c[k] > 0 && q >= 0 && q < kItrWin) bm[q] = 1;
      }
    }
    __syncwarp();
    int z = -1;
    for (int b0 = 0; b0 < kItrWin && z < 0; b0 += 32) {
      const unsigned m = __ballot_sync(0xffffffffu, bm[b0 + lane] == 0);
      if (m) z = b0 + __ffs(m) - 1;
    }
    if (z >= 0) {
      found = wbase + z + 1;
      const int k0 = z + lane, k1 = z + 32 + lane;
      const unsigned lo = __ballot_sync(0xffffffffu, k0 < kItrWin && bm[k0] == 0);
      const unsigned hi = __ballot_sync(0xffffffffu, k1 < kItrWin && bm[k1] == 0);
      fm = ((unsigned long long)hi << 32) | lo;
    }
    __syncwarp();
  }
  return found;
}

struct ItrArgs {
  int l;
  uint64_t seed;
  const int64_t* off;
  const int32_t* col;
  const int32_t* round;
  int32_t* color;
  const int4* rec;
  int pbase, cl;          // the partition: rec[pbase, pbase + cl)
  int32_t* A[2];          // active lists
  int* nA;                // their counters [2]
  int32_t* P;             // intra-partition neighbour lists (CSR slots)
  int32_t* icnt;          // intra-partition neighbours (first in the slot)
  int32_t* ucnt;          // neighbours in the colored partitions (at the back of the slot)
  int32_t* base;
  unsigned long long* freem;
  int32_t* tent;
  uint8_t* won;
  State* st;
  long long* passes;      // device counter
};

// Partition start (a plain launch over the whole GPU): the active list, the
// neighbour lists of the slots and the B_v summaries.
__global__ void __launch_bounds__(kItrBlock) k_itr_prep(ItrArgs a) {
  __shared__ __align__(16) uint8_t s_bm[kItrBlock / 32][kItrWin];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  uint8_t* bm = s_bm[warp];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  const int gw = tid >> 5, nwarps = nt >> 5;
  if (tid == 0) {
    a.nA[0] = a.cl;
    a.nA[1] = 0;
  }
  for (int i = gw; i < a.cl; i += nwarps) {
    const int v = a.rec[a.pbase + i].x;
    if (lane == 0) a.A[0][i] = v;
    const int64_t b = a.off[v], e = a.off[v + 1];
    // the slot: intra-partition neighbours from its front, those in colored
    // partitions from its back (8 strips of loads in flight: hubs are long);
    // then the latter are moved up behind the former
    int cnt = 0, upb = 0;
    for (int64_t a0 = b; a0 < e; a0 += 256) {
      int u[8], r[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t x = a0 + 32 * k + lane;
        u[k] = x < e ? __ldg(a.col + x) : -1;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = u[k] >= 0 ? __ldg(a.round + u[k]) : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool in = r[k] == a.l, hi = r[k] > a.l;
        const unsigned bi = __ballot_sync(0xffffffffu, in), bh = __ballot_sync(0xffffffffu, hi);
        if (in) a.P[b + cnt + __popc(bi & lt)] = u[k];
        if (hi) a.P[e - 1 - upb - __popc(bh & lt)] = u[k];
        cnt += __popc(bi);
        upb += __popc(bh);
      }
    }
    __syncwarp();
    unsigned long long fm;
    const int bs = itr_full_mex(a.P + b, cnt, a.P + e - upb, upb, a.color, bm, fm);
    if (lane == 0) {
      a.icnt[v] = cnt;
      a.ucnt[v] = upb;
      a.base[v] = bs;
      a.freem[v] = fm;
    }
  }
}

// The SIM-COL passes of one partition: a cooperative launch sized to the
// partition (a grid barrier among few blocks is cheap for the small, dense
// partitions that need many passes).
__global__ void __launch_bounds__(kItrBlock) k_itr_partition(ItrArgs a) {
  __shared__ __align__(16) uint8_t s_bm[kItrBlock / 32][kItrWin];
  __shared__ int sm[kItrBlock / 32 + 1];
  cg::grid_group grid = cg::this_grid();
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  uint8_t* bm = s_bm[warp];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  const int gw = tid >> 5, nwarps = nt >> 5;
  int cur = 0;
  int kmax = 0;
  for (;;) {
    const int na = ldcg(a.nA + cur);
    if (na == 0) break;
    const int32_t* A = a.A[cur];
    // Part 1
    for (int i = gw; i < na; i += nwarps) {
      const int v = ldcg(A + i);
      const int64_t b = a.off[v];
      const int ni = ldcg(a.icnt + v), bs = ldcg(a.base + v);
      unsigned long long taken = 0;
      // kItrStrips strips of 32 neighbours per step, all loads in flight (a
      // dense partition's lists are hundreds long: one L2 round trip per
      // strip would make every pass a chain of dependent loads)
      for (int j0 = 0; j0 < ni; j0 += 32 * kItrStrips) {
        int u[kItrStrips];
#pragma unroll
        for (int k = 0; k < kItrStrips; ++k) {
          const int j = j0 + 32 * k + lane;
          u[k] = j < ni ? ldcg(a.P + b + j) : -1;
        }
        int c[kItrStrips];
#pragma unroll
        for (int k = 0; k < kItrStrips; ++k) c[k] = u[k] >= 0 ? ldcg(a.color + u[k]) : 0;
#pragma unroll
        for (int k = 0; k < kItrStrips; ++k) {
          const int d = c[k] - bs;
          if (c[k] > 0 && d >= 0 && d < 64) taken |= 1ull << d;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) taken |= __shfl_xor_sync(0xffffffffu, taken, o);
      const unsigned long long g = __ldcg(a.freem + v) & ~taken;
      int found;
      if (g) {
        found = bs + __ffsll((long long)g) - 1;
      } else {  // the cached candidates are used up: rescan, refresh the summary
        unsigned long long fm;
        const int nup = ldcg(a.ucnt + v);
        found = itr_full_mex(a.P + b, ni, a.P + a.off[v + 1] - nup, nup, a.color, bm, fm);
        if (lane == 0) {
          a.base[v] = found;
          a.freem[v] = fm;
        }
      }
      if (lane == 0) a.tent[v] = found;
    }
    grid.sync();
    // Part 2
    for (int i = gw; i < na; i += nwarps) {
      const int v = ldcg(A + i);
      const int tv = ldcg(a.tent + v);
      const uint64_t hv = prio_hash(a.seed, (uint32_t)v);
      const int64_t b = a.off[v];
      const int ni = ldcg(a.icnt + v);
      bool lose = false;
      for (int j0 = 0; j0 < ni && !lose; j0 += 32 * kItrStrips) {
        int u[kItrStrips];
#pragma unroll
        for (int k = 0; k < kItrStrips; ++k) {
          const int j = j0 + 32 * k + lane;
          u[k] = j < ni ? ldcg(a.P + b + j) : -1;
        }
        int c[kItrStrips], t[kItrStrips];
#pragma unroll
        for (int k = 0; k < kItrStrips; ++k) {
          c[k] = u[k] >= 0 ? ldcg(a.color + u[k]) : 1;
          t[k] = u[k] >= 0 ? ldcg(a.tent + u[k]) : 0;
        }
        bool x = false;
#pragma unroll
        for (int k = 0; k < kItrStrips; ++k)
          if (c[k] == 0 && t[k] == tv) x |= prio_hash(a.seed, (uint32_t)u[k]) > hv;
        lose = __any_sync(0xffffffffu, x);
      }
      if (lane == 0) a.won[v] = lose ? 0 : 1;
    }
    grid.sync();
    // Part 3 and U = U \ {colored}
    int32_t* An = a.A[cur ^ 1];
    int* nn = a.nA + (cur ^ 1);
    for (int bb = blockIdx.x * blockDim.x; bb < na; bb += nt) {
      const int i = bb + threadIdx.x;
      int v = 0;
      bool stay = false;
      if (i < na) {
        v = ldcg(A + i);
        if (__ldcg(a.won + v)) {
          const int t = ldcg(a.tent + v);
          a.color[v] = t;
          kmax = max(kmax, t);
        } else {
          stay = true;
        }
      }
      block_append(stay, v, An, nn, sm);
    }
    if (tid == 0) ++*a.passes;
    grid.sync();
    if (tid == 0) a.nA[cur] = 0;  // the next pass's output counter (read two barriers later)
    cur ^= 1;
  }
  kmax = warp_max(kmax);
  if (lane == 0 && kmax) atomicMax(&a.st->K, kmax);
}

int dec_itr_run(Ctx& c, const int32_t* round, uint64_t seed, int32_t* color, long long* passes) {
  NvtxRange nvtx_("pgc DEC-ADG-ITR partitions");
  PGC_CHK_SIZES(c);
  *passes = 0;
  if (c.n == 0) return 0;
  // partition sizes: the order's per-key histogram (key = T - round)
  const int T = c.h_state->T;
  std::vector<int> cnt(T + 1, 0);
  PGC_CUDA(cudaMemcpyAsync(cnt.data(), c.hist1, sizeof(int) * (size_t)T, cudaMemcpyDeviceToHost, c.st));
  PGC_CUDA(cudaStreamSynchronize(c.st));
  // scratch: ADG's and the order's arrays are free now
  ItrArgs a = {};
  a.seed = seed;
  a.off = c.off;
  a.col = c.col;
  a.round = round;
  a.color = color;
  a.rec = c.rec;
  a.A[0] = c.U[0];
  a.A[1] = c.U[1];
  a.nA = c.hist1;  // two counters, then the pass counter (8-byte aligned)
  a.passes = reinterpret_cast<long long*>(c.hist1 + 2);
  a.P = c.P;
  a.icnt = c.npred;
  a.ucnt = reinterpret_cast<int32_t*>(c.rec + c.n);  // the bulk's record lists are unused here
  a.base = c.Rl;
  a.freem = reinterpret_cast<unsigned long long*>(c.bcnt);  // >= 2n + 2 ints
  a.tent = c.D;
  a.won = c.rs;
  a.st = c.state;
  PGC_CUDA(cudaMemsetAsync(a.passes, 0, sizeof(long long), c.st));
  // one wave: every block resident (a grid barrier needs them all)
  int occ = 0;
  PGC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_itr_partition, kItrBlock, 0));
  occ = occ < 1 ? 1 : occ;
  const int bps = c.tune.itr_blocks_per_sm > 0 && c.tune.itr_blocks_per_sm < occ ? c.tune.itr_blocks_per_sm : occ;
  const int G = c.nsm * bps;
  int pbase = 0;
  for (int l = T; l >= 1; --l) {
    const int cl = cnt[T - l];
    if (cl == 0) continue;
    a.l = l;
    a.pbase = pbase;
    a.cl = cl;
    pbase += cl;
    PGC_LAUNCH(c, kGJp, "k_itr_prep", k_itr_prep<<<G, kItrBlock, 0, c.st>>>(a));
    // passes: about one warp per itr_members_per_warp active vertices of the
    // partition's start
    const int mpw = c.tune.itr_members_per_warp;
    const int want = (cl + mpw * (kItrBlock / 32) - 1) / (mpw * (kItrBlock / 32));
    const int GP = want < G ? (want < 1 ? 1 : want) : G;
    void* args[] = {&a};
    PGC_LAUNCH(c, kGJp, "k_itr_partition",
               PGC_CUDA(cudaLaunchCooperativeKernel((const void*)k_itr_partition, dim3(GP),
                                                    dim3(kItrBlock), args, 0, c.st)));
  }
  if (int e = sync_state(c)) return e;
  PGC_CUDA(cudaMemcpy(passes, a.passes, sizeof(long long), cudaMemcpyDeviceToHost));
  return 0;
}

}  // namespace pgc
