// Microbenchmark: ordered stream compaction with the library's decoupled
// look-back (kernels.cuh), to find its tile-rate limit. Not part of the product.
#include <cstdio>
#include <vector>
#include "../include/mst_gpu.h"
#include "../paper_2005_06913_b200/csrc/kernels.cuh"
using namespace mstgpu;

// Look-back over a 32*kW-tile window per round trip (kW loads per lane).
template <int kW>
__device__ __forceinline__ uint32_t lookback_wide(unsigned long long* status, uint32_t tile, uint32_t aggregate,
                                                  uint32_t epoch) {
  const unsigned long long tag = (unsigned long long)epoch << 34;
  const uint32_t lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_relaxed(status, tag | (2ull << 32) | aggregate);
    return 0;
  }
  if (lane == 0) st_relaxed(status + tile, tag | (1ull << 32) | aggregate);
  uint32_t excl = 0;
  int64_t top = (int64_t)tile - 1;
  while (true) {
    unsigned long long sv[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int64_t idx = top - (int64_t)lane - 32 * j;
      sv[j] = idx >= 0 ? ld_relaxed(status + idx) : (tag | (2ull << 32));
    }
    bool done = false, retry = false;
    uint32_t add = 0;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      if (done || retry) break;
      const uint32_t flag = (uint32_t)(sv[j] >> 34) == epoch ? (uint32_t)(sv[j] >> 32) & 3u : 0u;
      const unsigned pm = __ballot_sync(0xffffffffu, flag == 2);
      const unsigned nr = __ballot_sync(0xffffffffu, flag == 0);
      const int first = pm ? __ffs(pm) - 1 : 31;
      const unsigned upto = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
      if (nr & upto) { retry = true; break; }
      add += warp_sum<uint32_t>((int)lane <= first ? (uint32_t)sv[j] : 0u);
      if (pm) done = true;
    }
    if (retry) { if (add == 0) {} }
    if (retry) {
      // keep what was confirmed before the not-ready window? simpler: redo from the same top
      continue;
    }
    excl += add;
    if (done) break;
    top -= 32 * kW;
  }
  if (lane == 0) st_relaxed(status + tile, tag | (2ull << 32) | (excl + aggregate));
  return excl;
}

template <int kIt, int kW>
__global__ void __launch_bounds__(kBlock) k_sel_wide(const uint4* __restrict__ in, uint64_t m, uint4* __restrict__ out,
                                                     unsigned int* tile_ctr, unsigned long long* status,
                                                     uint32_t epoch, unsigned int* kept_out) {
  __shared__ uint32_t s_scan[kIt * kWarps];
  __shared__ uint32_t s_misc[2];
  __shared__ uint32_t s_tile;
  constexpr int T = kBlock * kIt;
  const uint32_t ntiles = (uint32_t)((m + T - 1) / T);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    uint4 e[kIt];
    bool keep[kIt];
    unsigned bal[kIt];
#pragma unroll
    for (int k = 0; k < kIt; ++k) {
      const uint64_t i = (uint64_t)tile * T + k * kBlock + threadIdx.x;
      e[k] = i < m ? __ldcs(in + i) : make_uint4(0, 0, 0, 0);
      keep[k] = i < m && (e[k].z & 1u);
      bal[k] = __ballot_sync(0xffffffffu, keep[k]);
      if (lane == 0) s_scan[k * kWarps + warp] = __popc(bal[k]);
    }
    __syncthreads();
    if (warp == 0) {
      constexpr int kSlots = kIt * kWarps, kPer = (kSlots + 31) / 32;
      uint32_t v[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) { const int idx = lane * kPer + j; v[j] = idx < kSlots ? s_scan[idx] : 0u; sum += v[j]; }
      const uint32_t incl = warp_incl_scan(sum);
      uint32_t run = incl - sum;
#pragma unroll
      for (int j = 0; j < kPer; ++j) { const int idx = lane * kPer + j; if (idx < kSlots) s_scan[idx] = run; run += v[j]; }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t ex = lookback_wide<kW>(status, tile, tot, epoch);
      if (lane == 0) { s_misc[0] = ex; s_misc[1] = tot; }
    }
    __syncthreads();
    const uint32_t prefix = s_misc[0];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < kIt; ++k)
      if (keep[k]) __stcs(out + prefix + s_scan[k * kWarps + warp] + __popc(bal[k] & lt), e[k]);
    if (tile == ntiles - 1 && threadIdx.x == 0) *kept_out = prefix + s_misc[1];
    __syncthreads();
  }
}

template <int kIt, int kW>
void run_wide(const uint4* d_in, uint64_t m, uint4* d_out, unsigned int* d_ctr, unsigned long long* d_st, uint32_t& epoch,
              int sms) {
  auto kern = k_sel_wide<kIt, kW>;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kBlock, 0);
  const unsigned grid = sms * nb;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(d_ctr, 0, 8);
    cudaEventRecord(a);
    kern<<<grid, kBlock>>>(d_in, m, d_out, d_ctr, d_st, epoch++, d_ctr + 1);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  unsigned int kept; cudaMemcpy(&kept, d_ctr + 1, 4, cudaMemcpyDeviceToHost);
  printf("WIDE items=%2d window=%3d blocks/SM=%d: %.3f ms  %.0f GB/s  %.1f tiles/us kept=%u\n", kIt, 32 * kW, nb, best,
         (16.0 * m + 16.0 * kept) / best / 1e6, (m / (double)(kBlock * kIt)) / (best * 1e3), kept);
}

// two-pass: counts per tile (no dependencies), scan of counts, re-read + write
template <int kIt>
__global__ void __launch_bounds__(kBlock) k_count(const uint4* __restrict__ in, uint64_t m, unsigned int* counts) {
  __shared__ uint32_t s[kWarps];
  constexpr int T = kBlock * kIt;
  const uint64_t tile = blockIdx.x;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const uint64_t i = tile * T + k * kBlock + threadIdx.x;
    if (i < m) c += (__ldcs(in + i).z & 1u);
  }
  c = warp_sum<uint32_t>(c);
  if (lane_id() == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) { uint32_t t = 0; for (int w = 0; w < kWarps; ++w) t += s[w]; counts[tile] = t; }
}
__global__ void k_scan_counts(unsigned int* counts, uint32_t n) {  // one block, 1024 threads
  __shared__ uint32_t s[1024];
  uint32_t carry = 0;
  for (uint32_t base = 0; base < n; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < n ? counts[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) { const uint32_t t = threadIdx.x >= (unsigned)d ? s[threadIdx.x - d] : 0; __syncthreads(); s[threadIdx.x] += t; __syncthreads(); }
    if (i < n) counts[i] = carry + s[threadIdx.x] - v;
    const uint32_t tot = s[1023];
    __syncthreads();
    carry += tot;
  }
}
template <int kIt>
__global__ void __launch_bounds__(kBlock) k_write(const uint4* __restrict__ in, uint64_t m, const unsigned int* offs,
                                                  uint4* __restrict__ out) {
  __shared__ uint32_t s_scan[kIt * kWarps];
  constexpr int T = kBlock * kIt;
  const uint64_t tile = blockIdx.x;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint4 e[kIt]; bool keep[kIt]; unsigned bal[kIt];
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const uint64_t i = tile * T + k * kBlock + threadIdx.x;
    e[k] = i < m ? __ldcs(in + i) : make_uint4(0, 0, 0, 0);
    keep[k] = i < m && (e[k].z & 1u);
    bal[k] = __ballot_sync(0xffffffffu, keep[k]);
    if (lane == 0) s_scan[k * kWarps + warp] = __popc(bal[k]);
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int kSlots = kIt * kWarps, kPer = (kSlots + 31) / 32;
    uint32_t v[kPer], sum = 0;
    for (int j = 0; j < kPer; ++j) { const int idx = lane * kPer + j; v[j] = idx < kSlots ? s_scan[idx] : 0u; sum += v[j]; }
    const uint32_t incl = warp_incl_scan(sum);
    uint32_t run = incl - sum;
    for (int j = 0; j < kPer; ++j) { const int idx = lane * kPer + j; if (idx < kSlots) s_scan[idx] = run; run += v[j]; }
  }
  __syncthreads();
  const uint32_t prefix = offs[tile];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < kIt; ++k)
    if (keep[k]) __stcs(out + prefix + s_scan[k * kWarps + warp] + __popc(bal[k] & lt), e[k]);
}
template <int kIt>
void run_two_pass(const uint4* d_in, uint64_t m, uint4* d_out, unsigned int* d_counts) {
  constexpr int T = kBlock * kIt;
  const uint32_t nt = (uint32_t)((m + T - 1) / T);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_count<kIt><<<nt, kBlock>>>(d_in, m, d_counts);
    k_scan_counts<<<1, 1024>>>(d_counts, nt);
    k_write<kIt><<<nt, kBlock>>>(d_in, m, d_counts, d_out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
  }
  printf("TWO-PASS items=%2d tiles=%u: %.3f ms (%.0f GB/s of 1-pass bytes)\n", kIt, nt, best, (16.0 * m + 8.0 * m) / best / 1e6);
}

template <int kIt, bool kPrefetch>
__global__ void __launch_bounds__(kBlock) k_sel(const uint4* __restrict__ in, uint64_t m, uint4* __restrict__ out,
                                                unsigned int* tile_ctr, unsigned long long* status, uint32_t epoch,
                                                unsigned int* kept_out) {
  __shared__ uint32_t s_scan[kIt * kWarps];
  __shared__ uint32_t s_misc[2];
  __shared__ uint32_t s_tile[2];
  constexpr int T = kBlock * kIt;
  const uint32_t ntiles = (uint32_t)((m + T - 1) / T);
  int buf = 0;
  if (kPrefetch && threadIdx.x == 0) s_tile[0] = atomicAdd(tile_ctr, 1u);
  while (true) {
    if (!kPrefetch && threadIdx.x == 0) s_tile[0] = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile[kPrefetch ? buf : 0];
    if (tile >= ntiles) break;
    if (kPrefetch && threadIdx.x == 0) s_tile[buf ^ 1] = atomicAdd(tile_ctr, 1u);
    uint4 e[kIt];
    bool keep[kIt];
#pragma unroll
    for (int k = 0; k < kIt; ++k) {
      const uint64_t i = (uint64_t)tile * T + k * kBlock + threadIdx.x;
      e[k] = i < m ? __ldcs(in + i) : make_uint4(0, 0, 0, 0);
      keep[k] = i < m && (e[k].z & 1u);
    }
    uint32_t rank[kIt], prefix, total;
    tile_flag_scan<kIt>(keep, rank, s_scan, s_misc, status, tile, epoch, prefix, total);
#pragma unroll
    for (int k = 0; k < kIt; ++k)
      if (keep[k]) __stcs(out + prefix + rank[k], e[k]);
    if (tile == ntiles - 1 && threadIdx.x == 0) *kept_out = prefix + total;
    buf ^= 1;
  }
}

template <int kIt, bool kPrefetch>
void run(const uint4* d_in, uint64_t m, uint4* d_out, unsigned int* d_ctr, unsigned long long* d_st, uint32_t& epoch,
         int sms) {
  auto kern = k_sel<kIt, kPrefetch>;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kBlock, 0);
  const unsigned grid = sms * nb;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(d_ctr, 0, 8);
    cudaEventRecord(a);
    kern<<<grid, kBlock>>>(d_in, m, d_out, d_ctr, d_st, epoch++, d_ctr + 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  unsigned int kept;
  cudaMemcpy(&kept, d_ctr + 1, 4, cudaMemcpyDeviceToHost);
  const double bytes = 16.0 * m + 16.0 * kept;
  printf("items=%2d prefetch=%d blocks/SM=%d tiles=%llu: %.3f ms  %.0f GB/s  %.1f tiles/us kept=%u\n", kIt, (int)kPrefetch,
         nb, (unsigned long long)((m + kBlock * kIt - 1) / (kBlock * kIt)), best, bytes / best / 1e6,
         (m / (double)(kBlock * kIt)) / (best * 1e3), kept);
}

int main() {
  const uint64_t m = 256ull << 20;
  std::vector<uint4> h(m);
  uint64_t x = 88172645463325252ull;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = make_uint4((uint32_t)x, (uint32_t)(x >> 32), (uint32_t)(x >> 17), 7);
  }
  uint4 *d_in, *d_out;
  unsigned int* d_ctr;
  unsigned long long* d_st;
  cudaMalloc(&d_in, m * 16);
  cudaMalloc(&d_out, m * 16);
  cudaMalloc(&d_ctr, 16);
  cudaMalloc(&d_st, (m / 256 + 2) * 8);
  cudaMemset(d_st, 0, (m / 256 + 2) * 8);
  cudaMemcpy(d_in, h.data(), m * 16, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t epoch = 1;
  // copy roofline
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaMemcpy(d_out, d_in, m * 16, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("memcpy: %.3f ms %.0f GB/s\n", ms, 32.0 * m / ms / 1e6);
  run<4, false>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run<4, true>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run<8, false>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run<8, true>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run<16, false>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run<16, true>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run_wide<4, 1>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run_wide<4, 4>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run_wide<8, 4>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run_wide<8, 8>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  run_wide<16, 4>(d_in, m, d_out, d_ctr, d_st, epoch, sms);
  unsigned int* d_counts; cudaMalloc(&d_counts, (m / 256 + 2) * 4);
  run_two_pass<8>(d_in, m, d_out, d_counts);
  run_two_pass<16>(d_in, m, d_out, d_counts);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
