// red_probe.cu -- throughput of global RED (atomicSub, result unused) when many
// threads hit ONE address (a hub's degree counter) vs spread addresses.
#include <cstdio>
__global__ void red_hot(int* p, int n_ops, int n_hot) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_ops) atomicSub(p + (i % n_hot) * 32, 1);
}
__global__ void red_warp_agg(int* p, int n_ops) {  // match_any aggregation within the warp
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_ops) {
    unsigned m = __match_any_sync(__activemask(), 0);
    if ((threadIdx.x & 31) == __ffs(m) - 1) atomicSub(p, __popc(m));
  }
}
int main() {
  int* p;
  cudaMalloc(&p, 1 << 26);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 1 << 22;
  for (int hot : {1, 8, 64, 1024, 1 << 16}) {
    red_hot<<<N / 256, 256>>>(p, N, hot);
    cudaEventRecord(a);
    red_hot<<<N / 256, 256>>>(p, N, hot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("RED %d ops over %6d addresses: %.3f ms = %.2f Gops/s\n", N, hot, ms, N / ms / 1e6);
  }
  red_warp_agg<<<N / 256, 256>>>(p, N);
  cudaEventRecord(a);
  red_warp_agg<<<N / 256, 256>>>(p, N);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("warp-aggregated RED %d ops on 1 address: %.3f ms\n", N, ms);
  return 0;
}
