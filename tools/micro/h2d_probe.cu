// h2d_probe.cu -- pinned host -> device copy bandwidth of the 2.2 GB R-MAT 24
// CSR: one cudaMemcpyAsync vs the same bytes split over 2/4/8 streams, and
// chunked copies on one stream (the e2e path's H2D is link-bound).
#include <cstdio>
#include <vector>
int main() {
  const size_t bytes = 2217263952ull;
  char* h; char* d;
  cudaHostAlloc((void**)&h, bytes, cudaHostAllocDefault);
  cudaMalloc((void**)&d, bytes);
  for (size_t i = 0; i < bytes; i += 4096) h[i] = (char)i;
  std::vector<cudaStream_t> s(8);
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int ns : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s[0]);
      for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(s[k], a, 0);
      const size_t part = (bytes / ns + 4095) & ~(size_t)4095;
      for (int k = 0; k < ns; ++k) {
        const size_t o = k * part; if (o >= bytes) break;
        const size_t len = o + part > bytes ? bytes - o : part;
        cudaMemcpyAsync(d + o, h + o, len, cudaMemcpyHostToDevice, s[k]);
      }
      for (int k = 1; k < ns; ++k) { cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, s[k]); cudaStreamWaitEvent(s[0], e, 0); }
      cudaEventRecord(b, s[0]);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%d stream(s): %.2f ms = %.1f GB/s\n", ns, ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
