// atom_probe.cu -- UPDATE's per-arc random access pattern, three ways, on a
// 16.7M-vertex state (the R-MAT 24 size): (a) byte gather + RED on 42% of arcs
// (the current rs/D scheme), (b) one ATOM (fetch-sub, result used) per arc on a
// packed 32-bit word, (c) gather only, (d) RED only.  Random targets from a
// hash; each thread handles 8 arcs with all accesses in flight.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int K = 8;
__global__ void k_gather_red(const uint8_t* rs, int* D, int n, long long arcs, unsigned long long* sink) {
  unsigned acc = 0;
  for (long long a0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * K; a0 < arcs;
       a0 += (long long)gridDim.x * blockDim.x * K) {
    int u[K]; int s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) u[k] = hsh((uint32_t)(a0 + k)) % n;
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = __ldg(rs + u[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (s[k] < 107) atomicSub(D + u[k], 1);  // ~42% "alive"
      acc += s[k];
    }
  }
  if (acc == 0xffffffff) sink[0] = acc;
}
__global__ void k_atom(int* W, int n, long long arcs, unsigned long long* sink) {
  unsigned acc = 0;
  for (long long a0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * K; a0 < arcs;
       a0 += (long long)gridDim.x * blockDim.x * K) {
    int u[K]; int s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) u[k] = hsh((uint32_t)(a0 + k)) % n;
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = atomicSub(W + u[k], 1);
#pragma unroll
    for (int k = 0; k < K; ++k) acc += (unsigned)s[k] >> 24;
  }
  if (acc == 0xffffffff) sink[0] = acc;
}
__global__ void k_gather(const uint8_t* rs, int n, long long arcs, unsigned long long* sink) {
  unsigned acc = 0;
  for (long long a0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * K; a0 < arcs;
       a0 += (long long)gridDim.x * blockDim.x * K) {
    int u[K]; int s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) u[k] = hsh((uint32_t)(a0 + k)) % n;
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = __ldg(rs + u[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) acc += s[k];
  }
  if (acc == 0xffffffff) sink[0] = acc;
}
__global__ void k_red(int* D, int n, long long arcs) {
  for (long long a0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * K; a0 < arcs;
       a0 += (long long)gridDim.x * blockDim.x * K) {
#pragma unroll
    for (int k = 0; k < K; ++k) atomicSub(D + hsh((uint32_t)(a0 + k)) % n, 1);
  }
}
int main() {
  const int n = 1 << 24;
  const long long arcs = 100000000;
  uint8_t* rs; int* D; int* W; unsigned long long* sink;
  cudaMalloc(&rs, n); cudaMalloc(&D, 4ll * n); cudaMalloc(&W, 4ll * n); cudaMalloc(&sink, 8);
  cudaMemset(rs, 0x30, n); cudaMemset(D, 0, 4ll * n); cudaMemset(W, 0, 4ll * n);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bps : {4, 6, 8}) {
    const int G = nsm * bps;
    for (int rep = 0; rep < 2; ++rep) {
      float t[4];
      for (int w = 0; w < 4; ++w) {
        cudaEventRecord(a);
        if (w == 0) k_gather_red<<<G, 256>>>(rs, D, n, arcs, sink);
        if (w == 1) k_atom<<<G, 256>>>(W, n, arcs, sink);
        if (w == 2) k_gather<<<G, 256>>>(rs, n, arcs, sink);
        if (w == 3) k_red<<<G, 256>>>(D, n, arcs);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&t[w], a, b);
      }
      if (rep) printf("blocks/SM %d: 100M arcs: gather+RED(42%%) %.3f ms | ATOM %.3f ms | gather %.3f ms | RED(100%%) %.3f ms\n",
                      bps, t[0], t[1], t[2], t[3]);
    }
  }
  return 0;
}
