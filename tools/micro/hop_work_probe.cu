// hop_work_probe.cu -- cost of the core engine's per-hop work in isolation:
// a chain of hops between the 32 warps of one CTA where each hop does
//   mode 0: spin + publish only
//   mode 1: + one pending pass (31 entries: LDS list, LDS colour, ballot, compact)
//   mode 2: + byte-map next-zero search (LDS.U8 + ballot)
//   mode 3: mode 2 + a 64-bit __shfl warp_max (5 steps)
#include <cstdio>
#include <cstdint>

constexpr int kHops = 4096;
__device__ __forceinline__ int ldv(const volatile uint16_t* p) { return *p; }

__global__ void probe(int mode, unsigned long long* out) {
  __shared__ uint16_t cc[kHops + 64];
  __shared__ uint16_t plist[32][64];
  __shared__ uint8_t bm[32][1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < kHops + 64; i += blockDim.x) cc[i] = 0;
  for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) (&bm[0][0])[i] = (i & 1023) < 300;
  __syncthreads();
  const unsigned lt = (1u << lane) - 1;
  unsigned long long t0 = clock64();
  for (int h = warp; h < kHops; h += nw) {
    // pending list = the previous 31 hops (all but h-1 already coloured by now)
    int npend = 0;
    if (lane < 31 && h - 31 + lane >= 0) plist[warp][lane] = (uint16_t)(h - 31 + lane);
    npend = h >= 31 ? 31 : h;
    __syncwarp();
    if (h > 0)
      while (ldv(cc + h - 1) == 0) {
      }
    if (mode >= 1) {
      int keep = 0;
      const int q = lane < npend ? plist[warp][lane] : -1;
      const int c = q >= 0 ? ldv(cc + q) : 1;
      const bool still = q >= 0 && c == 0;
      if (q >= 0 && c) bm[warp][(c - 1) & 1023] = 1;
      const unsigned bal = __ballot_sync(0xffffffffu, still);
      __syncwarp();
      if (still) plist[warp][__popc(bal & lt)] = (uint16_t)q;
      keep = __popc(bal);
      npend = keep;
      __syncwarp();
    }
    int zi = 300;
    if (mode >= 2) {
      for (int b0 = 290; b0 < 1024; b0 += 32) {
        const unsigned m = __ballot_sync(0xffffffffu, bm[warp][b0 + lane] == 0);
        if (m) { zi = b0 + __ffs(m) - 1; break; }
      }
    }
    if (mode >= 3) {
      long long x = zi + lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
      zi = (int)x - 31;
    }
    if (lane == 0) *(volatile uint16_t*)(cc + h) = (uint16_t)(zi + 1);
    __syncwarp();
  }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  unsigned long long* o;
  cudaMalloc(&o, 8);
  const char* names[] = {"spin+publish", "+pending pass", "+next-zero search", "+warp_max"};
  for (int mode = 0; mode < 4; ++mode) {
    probe<<<1, 1024>>>(mode, o);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("mode %d %-20s: %7.1f cycles/hop (%s)\n", mode, names[mode], (double)h / kHops,
           cudaGetErrorString(e));
  }
  return 0;
}
