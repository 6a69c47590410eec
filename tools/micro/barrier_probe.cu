// Cost of one barrier as the one-kernel small path uses them: cluster.sync()
// on one 16-CTA cluster (1024 and 256 threads per CTA) and the cooperative
// grid.sync() (148 x 512 and 32 x 512), plus a cluster.sync with a DSMEM read
// of every peer's counter in between (the per-phase totals).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cl(int iters, unsigned long long* out, int dsmem) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int s_x;
  if (threadIdx.x == 0) s_x = 1;
  cl.sync();
  unsigned long long t0 = clock64();
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (dsmem && threadIdx.x < 16) acc += *cl.map_shared_rank(&s_x, threadIdx.x);
    cl.sync();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters + (acc == -1);
}
__global__ void k_grid(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  g.sync();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  unsigned long long h;
  cudaFuncSetAttribute(k_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int threads : {1024, 256}) for (int ds : {0, 1}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cl, 2000, d, ds);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster16 x %d threads, dsmem read %d: %llu cycles per cluster.sync (%s)\n", threads, ds, h,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int blocks : {148, 296, 32}) {
    int iters = 2000;
    void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)k_grid, dim3(blocks), dim3(512), args, 0, 0);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("grid %d x 512: %llu cycles per grid.sync (%s)\n", blocks, h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
