// Random 4 B lookups into shared memory: local smem vs distributed shared
// memory (DSMEM) across a thread-block cluster, against random global
// gathers. Sizes the per-SM / per-cluster hub caches of the heavy filter.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dsmem_bench.cu -o tools/dsmem_bench
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// kRemote: 0 local smem, 1 DSMEM (random rank in the cluster)
template <int kRemote, int kU>
__global__ void k_smem(uint32_t words_log2, uint64_t n, uint32_t seed, uint32_t* sink) {
  extern __shared__ uint32_t T[];
  const uint32_t W = 1u << words_log2;
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) T[i] = hash32(i ^ blockIdx.x);
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t C = cl.num_blocks();
  cl.sync();
  uint32_t acc = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU + threadIdx.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x * kU) {
    uint32_t v[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint32_t h = hash32((uint32_t)(base + k * blockDim.x) ^ seed);
      const uint32_t off = h & (W - 1);
      if (kRemote) {
        const uint32_t rank = (h >> 24) % C;
        const uint32_t* p = cl.map_shared_rank(T, rank);
        v[k] = p[off];
      } else {
        v[k] = T[off];
      }
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) acc += v[k];
  }
  cl.sync();
  if (acc == 0x12345678u) *sink = acc;
}

template <int kU>
__global__ void k_gather(const uint32_t* __restrict__ t, uint32_t mask, uint64_t n, uint32_t seed, uint32_t* sink) {
  uint32_t acc = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU + threadIdx.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x * kU) {
    uint32_t v[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) v[k] = __ldg(t + (hash32((uint32_t)(base + k * blockDim.x) ^ seed) & mask));
#pragma unroll
    for (int k = 0; k < kU; ++k) acc += v[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int kRemote>
int run_smem(int cluster, int words_log2, int threads, uint64_t n, uint32_t* sink) {
  auto k = k_smem<kRemote, 8>;
  const size_t smem = (size_t)4 << words_log2;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (cluster > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int sms = 148;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
  int nclusters = 0;
  cfg.gridDim = dim3(cluster);
  CK(cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg));
  cfg.gridDim = dim3(nclusters * cluster);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaLaunchKernelEx(&cfg, k, (uint32_t)words_log2, n, 1u, sink));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, k, (uint32_t)words_log2, n, 7u, sink));
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double rate = n / (ms * 1e-3);
  printf("%-6s cluster %2d table %4d KB/CTA thr %4d grid %4d : %8.3f ms %8.1f G/s  %.2f lookups/cyc/SM\n",
         kRemote ? "dsmem" : "local", cluster, (4 << words_log2) >> 10, threads, nclusters * cluster, ms, rate * 1e-9,
         rate / (sms * 1.965e9));
  (void)sms;
  return 0;
}

int main() {
  uint32_t* sink; cudaMalloc(&sink, 4);
  const uint64_t n = 1ull << 32;
  for (int cl : {1, 2, 4, 8, 16})
    for (int thr : {512, 1024}) {
      if (cl == 1) run_smem<0>(cl, 15, thr, n, sink);
      run_smem<1>(cl, 15, thr, n, sink);
    }
  run_smem<1>(8, 14, 1024, n, sink);
  run_smem<1>(16, 14, 1024, n, sink);
  run_smem<1>(16, 16, 1024, n, sink);  // 256 KB? (fails above the opt-in limit)
  uint32_t* t; cudaMalloc(&t, 64u << 20); cudaMemset(t, 1, 64u << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_gather<8><<<148 * 8, 256>>>(t, (16u << 20) - 1, n / 4, 1, sink);
  cudaEventRecord(e0);
  k_gather<8><<<148 * 8, 256>>>(t, (16u << 20) - 1, n / 4, 3, sink);
  cudaEventRecord(e1); cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("global gather 64 MB table: %.3f ms %.1f G/s\n", ms, n / 4 / (ms * 1e-3) * 1e-9);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
