// dec.cu -- DEC-ADG-ITR: ADG's partitions R(l) colored
// from the densest (l = T) down, each by SIM-COL with
// ITR's deterministic Part 1 -- the smallest color not used by an already
// colored neighbour -- and the conflict rule of reading Q23 (a vertex gives its
// tentative color up only to a same-colored active neighbour of larger
// h = splitmix64(seed ^ v)).
//
// One SIM-COL pass over the active list A of partition l = three kernels:
//   k_itr_tent     Part 1: tent[v] = mex of the colors of v's colored
//                  neighbours (warp per vertex, shared-memory byte map window)
//   k_itr_conflict Part 2: won[v] = no active neighbour u (round[u] == l,
//                  color[u] == 0) has tent[u] == tent[v] and h(u) > h(v)
//   k_itr_apply    Part 3 + U = U \ {colored}: color[v] = tent[v] for the
//                  winners (their colors reach the neighbours' B through the
//                  next Part 1), the others are compacted into the next list.
// The winners' colors are written only in k_itr_apply, so "active" in Part 2
// is the state at the start of the pass, as in the listing.  Passes run in
// batches between host synchronisations; a pass on an empty list exits at
// once.  The partitions are contiguous ranges of the priority order
// (jp_order_run sorts by round).
#include <cstdio>
#include <vector>

#include "pgc_internal.cuh"

namespace pgc {

constexpr int kItrWin = 1024;  // colors per byte-map window (Part 1)
constexpr int kItrBlock = 256;
constexpr int kItrBatch = 16;  // passes between host synchronisations

// Partition start (warp per vertex of R(l)): one scan of the full adjacency.
// B_v so far = the colors of v's neighbours in the colored partitions Q; it
// is summarised by base[v] = mex(B_v) and the 64-bit mask freem[v] of the
// colors base..base+63 NOT in B_v.  The neighbours inside R(l) are listed in
// v's own CSR slot of P (count icnt[v]): every pass only touches those.
__global__ void __launch_bounds__(kItrBlock) k_itr_prep(int l, const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ col,
                                                        const int32_t* __restrict__ round,
                                                        const int32_t* color,
                                                        const int32_t* __restrict__ A,
                                                        const int* __restrict__ nA,
                                                        int32_t* __restrict__ P,
                                                        int32_t* __restrict__ icnt,
                                                        int32_t* __restrict__ base,
                                                        unsigned long long* __restrict__ freem) {
  __shared__ __align__(16) uint8_t s_bm[kItrBlock / 32][kItrWin];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  uint8_t* bm = s_bm[warp];
  const int na = *nA;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nw) {
    const int v = A[i];
    const int64_t b = off[v], e = off[v + 1];
    int bs = 0;
    unsigned long long fm = 0;
    for (int wbase = 0;; wbase += kItrWin) {
      for (int j = lane; j < kItrWin / 16; j += 32) reinterpret_cast<uint4*>(bm)[j] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      int cnt = 0;
      for (int64_t a0 = b; a0 < e; a0 += 32) {
        const int64_t a = a0 + lane;
        const int u = a < e ? __ldg(col + a) : -1;
        const int c = u >= 0 ? color[u] : 0;
        const int k = c - wbase - 1;
        if (c > 0 && k >= 0 && k < kItrWin) bm[k] = 1;
        if (wbase == 0) {  // intra-partition neighbours, listed once
          const bool in = u >= 0 && round[u] == l;
          const unsigned bal = __ballot_sync(0xffffffffu, in);
          if (in) P[b + cnt + __popc(bal & lt)] = u;
          cnt += __popc(bal);
        }
      }
      if (wbase == 0 && lane == 0) icnt[v] = cnt;
      __syncwarp();
      int z = -1;
      for (int b0 = 0; b0 < kItrWin && z < 0; b0 += 32) {
        const unsigned m = __ballot_sync(0xffffffffu, bm[b0 + lane] == 0);
        if (m) z = b0 + __ffs(m) - 1;
      }
      if (z >= 0) {  // mex found in this window; the free mask of the next 64 colors
        bs = wbase + z + 1;
        const int k0 = z + lane, k1 = z + 32 + lane;
        // (colors past the window count as taken: a pass whose candidates run
        // out rescans and refreshes the summary)
        const unsigned lo = __ballot_sync(0xffffffffu, k0 < kItrWin && bm[k0] == 0);
        const unsigned hi = __ballot_sync(0xffffffffu, k1 < kItrWin && bm[k1] == 0);
        fm = ((unsigned long long)hi << 32) | lo;
        break;
      }
      __syncwarp();
    }
    if (lane == 0) {
      base[v] = bs;
      freem[v] = fm;
    }
  }
}

// Part 1: tent[v] = the smallest color free in B_v and not taken by an
// intra-partition neighbour colored in an earlier pass: from the cached 64
// candidates, else (all taken -- a dense partition) a rescan of the whole
// adjacency that also refreshes base/freem from every colored neighbour, so
// the next 64 passes of v are cheap again.
__global__ void __launch_bounds__(kItrBlock) k_itr_tent(const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ col,
                                                        const int32_t* color,
                                                        const int32_t* __restrict__ A,
                                                        const int* __restrict__ nA,
                                                        const int32_t* __restrict__ P,
                                                        const int32_t* __restrict__ icnt,
                                                        int32_t* __restrict__ base,
                                                        unsigned long long* __restrict__ freem,
                                                        int32_t* __restrict__ tent) {
  __shared__ __align__(16) uint8_t s_bm[kItrBlock / 32][kItrWin];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* bm = s_bm[warp];
  const int na = *nA;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nw) {
    const int v = A[i];
    const int64_t b = off[v];
    const int ni = icnt[v], bs = base[v];
    unsigned long long taken = 0;
    for (int j0 = 0; j0 < ni; j0 += 32) {
      const int j = j0 + lane;
      const int c = j < ni ? color[__ldg(P + b + j)] : 0;
      const int d = c - bs;
      if (c > 0 && d >= 0 && d < 64) taken |= 1ull << d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) taken |= __shfl_xor_sync(0xffffffffu, taken, o);
    const unsigned long long g = freem[v] & ~taken;
    int found = 0;
    if (g) {
      found = bs + __ffsll((long long)g) - 1;
    } else {  // rescan everything and refresh the summary
      const int64_t e = off[v + 1];
      unsigned long long fm = 0;
      for (int wbase = 0; !found; wbase += kItrWin) {
        for (int j = lane; j < kItrWin / 16; j += 32) reinterpret_cast<uint4*>(bm)[j] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        for (int64_t a0 = b; a0 < e; a0 += 32) {
          const int64_t a = a0 + lane;
          const int u = a < e ? __ldg(col + a) : -1;
          const int c = u >= 0 ? color[u] : 0;
          const int k = c - wbase - 1;
          if (c > 0 && k >= 0 && k < kItrWin) bm[k] = 1;
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
      if (lane == 0) {
        base[v] = found;
        freem[v] = fm;
      }
    }
    if (lane == 0) tent[v] = found;
  }
}

// Part 2: only the intra-partition neighbours can be active
__global__ void __launch_bounds__(kItrBlock) k_itr_conflict(uint64_t seed,
                                                            const int64_t* __restrict__ off,
                                                            const int32_t* color,
                                                            const int32_t* __restrict__ A,
                                                            const int* __restrict__ nA,
                                                            const int32_t* __restrict__ P,
                                                            const int32_t* __restrict__ icnt,
                                                            const int32_t* __restrict__ tent,
                                                            uint8_t* __restrict__ won) {
  const int lane = threadIdx.x & 31;
  const int na = *nA;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nw) {
    const int v = A[i];
    const int tv = tent[v];
    const uint64_t hv = prio_hash(seed, (uint32_t)v);
    const int64_t b = off[v];
    const int ni = icnt[v];
    bool lose = false;
    for (int j0 = 0; j0 < ni && !lose; j0 += 32) {
      const int j = j0 + lane;
      bool x = false;
      if (j < ni) {
        const int u = __ldg(P + b + j);
        if (color[u] == 0 && tent[u] == tv) x = prio_hash(seed, (uint32_t)u) > hv;
      }
      lose = __any_sync(0xffffffffu, x);
    }
    if (lane == 0) won[v] = lose ? 0 : 1;
  }
}

// Part 3 and U = U \ {colored}: block-level compaction of the losers
__global__ void __launch_bounds__(kItrBlock) k_itr_apply(const int32_t* __restrict__ A,
                                                         const int* __restrict__ nA,
                                                         const int32_t* __restrict__ tent,
                                                         const uint8_t* __restrict__ won,
                                                         int32_t* color, int32_t* __restrict__ Anext,
                                                         int* nAnext, State* st) {
  __shared__ int sm[kItrBlock / 32 + 1];
  const int na = *nA;
  int kmax = 0;
  for (int base = blockIdx.x * blockDim.x; base < na; base += gridDim.x * blockDim.x) {
    const int i = base + threadIdx.x;
    int v = 0;
    bool stay = false;
    if (i < na) {
      v = A[i];
      if (won[v]) {
        color[v] = tent[v];
        kmax = max(kmax, tent[v]);
      } else {
        stay = true;
      }
    }
    block_append(stay, v, Anext, nAnext, sm);
  }
  kmax = warp_max(kmax);
  if (lane_id() == 0 && kmax) atomicMax(&st->K, kmax);
}

// the partition's vertices (a range of the priority order) -> active list
__global__ void k_itr_init(const int4* __restrict__ rec, int base, int cnt, int32_t* __restrict__ A,
                           int* nA, int* nAnext) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    A[i] = rec[base + i].x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *nA = cnt;
    *nAnext = 0;
  }
}
// after a pass: the consumed list's counter becomes the next output counter;
// the remaining count is published for the host (State::sorted is free now)
__global__ void k_itr_swap(int* consumed, const int* remaining, State* st) {
  *consumed = 0;
  st->sorted = *remaining;
}

int dec_itr_run(Ctx& c, const int32_t* round, uint64_t seed, int32_t* color, long long* passes) {
  *passes = 0;
  if (c.n == 0) return 0;
  // partition sizes: the order's per-key histogram (key = T - round)
  const int T = c.h_state->T;
  std::vector<int> cnt(T + 1, 0);
  PGC_CUDA(cudaMemcpyAsync(cnt.data(), c.hist1, sizeof(int) * (size_t)T, cudaMemcpyDeviceToHost, c.st));
  PGC_CUDA(cudaStreamSynchronize(c.st));
  // scratch (ADG's and the order's arrays are free now)
  int32_t* A[2] = {c.U[0], c.U[1]};
  int* nA = c.hist1;                 // two list counters
  int32_t* tent = c.D;
  uint8_t* won = c.rs;
  int32_t* icnt = c.npred;
  int32_t* base = c.Rl;
  unsigned long long* freem = reinterpret_cast<unsigned long long*>(c.bcnt);  // >= 2n + 2 ints
  int32_t* intra = c.P;               // intra-partition neighbours, in each vertex's CSR slot
  const int G = c.nsm * 8;
  int pbase = 0;
  for (int l = T; l >= 1; --l) {
    const int cl = cnt[T - l];
    if (cl == 0) continue;
    int cur = 0;
    PGC_LAUNCH(c, kGJp, "k_itr_init",
               k_itr_init<<<G, 256, 0, c.st>>>(c.rec, pbase, cl, A[0], nA, nA + 1));
    pbase += cl;
    PGC_LAUNCH(c, kGJp, "k_itr_prep",
               k_itr_prep<<<G, kItrBlock, 0, c.st>>>(l, c.off, c.col, round, color, A[0], nA, intra,
                                                      icnt, base, freem));
    for (;;) {
      for (int j = 0; j < kItrBatch; ++j) {
        PGC_LAUNCH(c, kGJp, "k_itr_tent",
                   k_itr_tent<<<G, kItrBlock, 0, c.st>>>(c.off, c.col, color, A[cur], nA + cur,
                                                          intra, icnt, base, freem, tent));
        PGC_LAUNCH(c, kGJp, "k_itr_conflict",
                   k_itr_conflict<<<G, kItrBlock, 0, c.st>>>(seed, c.off, color, A[cur], nA + cur,
                                                              intra, icnt, tent, won));
        PGC_LAUNCH(c, kGJp, "k_itr_apply",
                   k_itr_apply<<<G, kItrBlock, 0, c.st>>>(A[cur], nA + cur, tent, won, color,
                                                           A[cur ^ 1], nA + (cur ^ 1), c.state));
        // A[cur^1] / nA[cur^1] hold the next active list
        PGC_LAUNCH(c, kGJp, "k_itr_swap",
                   k_itr_swap<<<1, 1, 0, c.st>>>(nA + cur, nA + (cur ^ 1), c.state));
        cur ^= 1;
        ++*passes;
      }
      if (int e = sync_state(c)) return e;
      if (c.h_state->sorted == 0) break;
    }
  }
  return sync_state(c);
}

}  // namespace pgc
