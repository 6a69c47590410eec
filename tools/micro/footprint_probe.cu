// footprint_probe.cu -- does the footprint of UPDATE's decrement targets bound
// round 1?  ATOM-with-return and RED on uniformly random targets, 100 M ops,
// (a) over a dense state of n words, n = 2^20 .. 2^25 (4 .. 134 MB), and
// (b) over S = 1.29 M "survivors" scattered in a 2^24-word array (R-MAT 24
// round 1: the decrements land on 1.29 M of the 16.7 M D entries, one per
// 32-byte sector: 41 MB of touched sectors), and the same survivors packed
// densely (5 MB).  Each thread keeps 8 ops in flight (as k_update_light).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int K = 8;
// target = map ? map[h % S] : h % S
template <bool RET>
__global__ void k_ops(int* W, const int* __restrict__ map, uint32_t S, long long ops, unsigned long long* sink) {
  unsigned acc = 0;
  for (long long a0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * K; a0 < ops;
       a0 += (long long)gridDim.x * blockDim.x * K) {
    int u[K], s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) u[k] = hsh((uint32_t)(a0 + k)) % S;
    if (map) {
#pragma unroll
      for (int k = 0; k < K; ++k) u[k] = __ldg(map + u[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (RET) s[k] = atomicSub(W + u[k], 1);
      else { atomicSub(W + u[k], 1); s[k] = 0; }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += (unsigned)s[k] >> 24;
  }
  if (acc == 0xffffffff) sink[0] = acc;
}
__global__ void k_map(int* map, uint32_t S, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
    map[i] = (int)(((uint64_t)i * n) / S) ^ (int)(hsh(i) & 7u);  // one per ~13 words, jittered
}
int main() {
  const long long ops = 100000000;
  int* W; int* map; unsigned long long* sink;
  cudaMalloc(&W, 4ll << 25); cudaMalloc(&map, 4ll << 21); cudaMalloc(&sink, 8);
  cudaMemset(W, 0, 4ll << 25);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int G = nsm * 6;
  auto run = [&](const char* name, const int* m, uint32_t S) {
    float t[2];
    for (int rep = 0; rep < 2; ++rep)
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(a);
        if (w == 0) k_ops<true><<<G, 256>>>(W, m, S, ops, sink);
        else k_ops<false><<<G, 256>>>(W, m, S, ops, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&t[w], a, b);
      }
    printf("%-34s ATOM %.3f ms (%.1f G/s) | RED %.3f ms (%.1f G/s)\n", name, t[0], ops / t[0] * 1e-6,
           t[1], ops / t[1] * 1e-6);
  };
  for (int lg = 20; lg <= 25; ++lg) {
    char nm[64]; snprintf(nm, sizeof nm, "dense 2^%d words (%d MB)", lg, 4 << (lg - 20));
    run(nm, nullptr, 1u << lg);
  }
  const uint32_t S = 1290000;
  k_map<<<nsm * 4, 256>>>(map, S, 1u << 24);
  run("1.29M survivors in 2^24 (41 MB)", map, S);
  run("1.29M survivors packed (5 MB)", nullptr, S);
  const uint32_t S2 = 190000;
  k_map<<<nsm * 4, 256>>>(map, S2, 1u << 24);
  run("190K survivors in 2^24 (6 MB)", map, S2);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
