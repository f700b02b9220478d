// grid.sync() cost on this GPU (cooperative launch, full residency).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned v = 0;
  for (int i = 0; i < iters; ++i) { v += threadIdx.x ^ i; g.sync(); }
  if (v == 12345) *sink = v;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink; cudaMalloc(&sink, 4);
  for (int bps : {1, 2, 4, 6}) {
    int iters = 2000;
    void* args[] = {&iters, &sink};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)k, sms * bps, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, sms * bps, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("blocks=%d: %.2f us per grid.sync (%s)\n", sms * bps, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
