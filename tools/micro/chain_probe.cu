// chain_probe.cu -- microbenchmark: latency of one dependency hop between warps
// (warp i waits for flag[i-1] != 0, then sets flag[i]) through
//   mode 0: local shared memory, volatile st/ld
//   mode 1: shared memory written through the cluster-mapped generic pointer (own CTA)
//   mode 2: st.relaxed.cluster.shared::cluster (mapa) to the next CTA of a 2-CTA cluster
//   mode 3: global memory, st.relaxed.gpu / ld.relaxed.gpu, warps on 2 CTAs
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_probe chain_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int kHops = 4096;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_vol(const int* p) { return *(volatile const int*)p; }

__global__ void __cluster_dims__(2, 1, 1) probe(int mode, int* gflag, unsigned long long* out) {
  __shared__ int sflag[kHops + 1];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i <= kHops; i += blockDim.x) sflag[i] = 0;
  cl.sync();
  int* peer = cl.map_shared_rank(sflag, rank ^ 1);
  int* self = cl.map_shared_rank(sflag, rank);
  unsigned long long t0 = clk();
  // hop h is done by CTA (mode>=2 ? h&1 : 0), warp (h / (mode>=2?2:1)) % nw
  for (int h = 0; h < kHops; ++h) {
    const int owner_cta = mode >= 2 ? (h & 1) : 0;
    const int owner_warp = (mode >= 2 ? h >> 1 : h) % nw;
    if (owner_cta != rank || owner_warp != warp) continue;
    if (h > 0) {
      if (mode == 3) {
        while (true) {
          int v;
          asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(gflag + h - 1) : "memory");
          if (v) break;
        }
      } else {
        while (ld_vol(sflag + h - 1) == 0) {
        }
      }
    }
    if (lane == 0) {
      if (mode == 0) *(volatile int*)(sflag + h) = 1;
      else if (mode == 1) *(volatile int*)(self + h) = 1;
      else if (mode == 2) {
        // own copy + peer copy
        *(volatile int*)(sflag + h) = 1;
        uint32_t a = (uint32_t)__cvta_generic_to_shared(sflag + h);
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank ^ 1));
        asm volatile("st.relaxed.cluster.shared::cluster.b32 [%0], %1;" ::"r"(ra), "r"(1) : "memory");
      } else {
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(gflag + h), "r"(1) : "memory");
      }
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) out[rank] = clk() - t0;
  cl.sync();
}

int main() {
  int* g;
  unsigned long long* o;
  cudaMalloc(&g, (kHops + 1) * sizeof(int));
  cudaMalloc(&o, 2 * sizeof(unsigned long long));
  const char* names[] = {"local volatile smem", "generic cluster ptr (own CTA)",
                         "DSMEM st.relaxed.cluster across 2 CTAs", "global relaxed.gpu across 2 CTAs"};
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {2, 8, 32}) {
      cudaMemset(g, 0, (kHops + 1) * sizeof(int));
      probe<<<2, 32 * warps>>>(mode, g, o);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[2];
      cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%-42s warps=%2d : %7.1f ns/hop  (%s)\n", names[mode], warps,
             (double)(h[0] > h[1] ? h[0] : h[1]) / kHops, cudaGetErrorString(e));
    }
  return 0;
}
