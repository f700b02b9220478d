// Structure experiment for the heavy filter's count pass (k_count<SoaView,
// kModeHeavy>): the same work (stream src/dst/w, weight test, 2 label
// gathers, ordered staging of the survivors, counts) as
//   A: the current block-tile shape (1024 edges per block iteration, three
//      __syncthreads, survivors compacted per tile, one count per tile);
//   B: warp-independent chunks (128 consecutive edges per warp iteration, no
//      block barrier, survivors compacted per chunk, one byte count per chunk);
//   C: B with the next chunk's stream loads issued before this chunk's gathers.
// Inputs: R-MAT-skewed endpoints (each of 26 bits set with p = 0.24), a
// 256 MB vertex map whose "giant" is the low-popcount vertices (~14 %
// survivors), uniform weights with a 9 % light quantile.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/filter_bench.cu -o tools/filter_bench
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

constexpr int kScale = 26;
__global__ void k_fill_rmat(uint32_t* x, uint64_t n, uint32_t seed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    uint32_t h = hash32(hash32((uint32_t)i + seed * 0x632be5abu) ^ seed);  // (i ^ seed alone makes dst[i] = src[i ^ 3])
    for (int b = 0; b < kScale; ++b) {
      if ((b & 3) == 0) h = hash32(h + 0x9e3779b9u * (b + 1) + (uint32_t)(i >> 32));
      if (((h >> ((b & 3) * 8)) & 255u) < 61u) v |= 1u << b;  // p = 0.238
    }
    x[i] = v;
  }
}
// the first `count` entries uniform random (the BASELINE generators' spanning-tree block)
__global__ void k_fill_uniform(uint32_t* x, uint64_t count, uint32_t seed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] = hash32(hash32((uint32_t)i ^ seed) + 12345u) & ((1u << kScale) - 1u);
}
__global__ void k_fill_w(uint32_t* x, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] = hash32((uint32_t)i * 2654435761u ^ 77u);
}
__global__ void k_fill_map(uint32_t* L, uint64_t nv) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x)
    L[v] = __popc((uint32_t)v) <= 9 ? 0u : (uint32_t)v;
}

constexpr int kBlock = 256, kWarps = 8, kItems = 4, kTile = kBlock * kItems;

// ---- A: the product kernel's shape
__global__ void __launch_bounds__(kBlock) k_filter_a(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                                     const uint32_t* __restrict__ w, const uint32_t* __restrict__ L,
                                                     uint64_t m, uint32_t pivot, uint4* __restrict__ stage,
                                                     uint32_t* __restrict__ counts) {
  __shared__ uint32_t s_cnt[kWarps];
  __shared__ uint32_t s_slot[kItems * kWarps];
  const uint32_t ntiles = (uint32_t)((m + kTile - 1) / kTile);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t a[kItems], b[kItems], ww[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      a[k] = b[k] = ww[k] = 0;
      if (i < m) {
        a[k] = __ldcs(src + i);
        b[k] = __ldcs(dst + i);
        ww[k] = __ldcs(w + i);
      }
    }
    uint32_t cnt = 0;
    bool keep[kItems];
    unsigned bal[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      keep[k] = false;
      if (i < m && ww[k] >= pivot) {
        a[k] = __ldg(L + a[k]);
        b[k] = __ldg(L + b[k]);
        keep[k] = a[k] != b[k];
      }
      bal[k] = __ballot_sync(0xffffffffu, keep[k]);
      if (lane == 0) s_slot[k * kWarps + warp] = __popc(bal[k]);
      cnt += __popc(bal[k]);
    }
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = s_slot[lane];
      const uint32_t incl = warp_incl_scan(v);
      s_slot[lane] = incl - v;
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (keep[k])
        __stcs(stage + (uint64_t)tile * kTile + s_slot[k * kWarps + warp] + __popc(bal[k] & lt),
               make_uint4(a[k], b[k], ww[k], (uint32_t)((uint64_t)tile * kTile + k * kBlock + threadIdx.x)));
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int q = 0; q < kWarps; ++q) t += s_cnt[q];
      counts[tile] = t;
    }
    __syncthreads();
  }
}

// ---- B / C: warp-independent chunks of 128 consecutive edges
constexpr int kChunk = 32 * kItems;
template <bool kPrefetch>
__global__ void __launch_bounds__(kBlock) k_filter_b(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                                     const uint32_t* __restrict__ w, const uint32_t* __restrict__ L,
                                                     uint64_t m, uint32_t pivot, uint4* __restrict__ stage,
                                                     uint8_t* __restrict__ counts) {
  const uint64_t nchunks = (m + kChunk - 1) / kChunk;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t stride = (uint64_t)gridDim.x * kWarps;
  const uint32_t lt = lanemask_lt();
  uint32_t a[kItems], b[kItems], ww[kItems];
  uint64_t chunk = (uint64_t)blockIdx.x * kWarps + warp;
  auto load = [&](uint64_t c, uint32_t (&x)[kItems], uint32_t (&y)[kItems], uint32_t (&z)[kItems]) {
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = c * kChunk + k * 32 + lane;
      x[k] = y[k] = z[k] = 0;
      if (i < m) {
        x[k] = __ldcs(src + i);
        y[k] = __ldcs(dst + i);
        z[k] = __ldcs(w + i);
      }
    }
  };
  if (kPrefetch && chunk < nchunks) load(chunk, a, b, ww);
  for (; chunk < nchunks; chunk += stride) {
    uint32_t na[kItems], nb[kItems], nw[kItems];
    if (kPrefetch) {
      if (chunk + stride < nchunks) load(chunk + stride, na, nb, nw);
    } else {
      load(chunk, a, b, ww);
    }
    bool keep[kItems];
    uint32_t la[kItems], lb[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = chunk * kChunk + k * 32 + lane;
      keep[k] = i < m && ww[k] >= pivot;
      la[k] = lb[k] = 0;
      if (keep[k]) {
        la[k] = __ldg(L + a[k]);
        lb[k] = __ldg(L + b[k]);
      }
    }
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const bool kp = keep[k] && la[k] != lb[k];
      const unsigned bal = __ballot_sync(0xffffffffu, kp);
      if (kp)
        __stcs(stage + chunk * kChunk + run + __popc(bal & lt),
               make_uint4(la[k], lb[k], ww[k], (uint32_t)(chunk * kChunk + k * 32 + lane)));
      run += __popc(bal);
    }
    if (lane == 0) counts[chunk] = (uint8_t)run;
    if (kPrefetch) {
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        a[k] = na[k];
        b[k] = nb[k];
        ww[k] = nw[k];
      }
    }
  }
}

int main(int argc, char** argv) {
  const bool tree = argc > 1;  // any argument: a uniform-random block of 2^26 edges first
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t m = 1ull << 30, nv = 1ull << kScale;
  uint32_t *s, *d, *w, *L, *counts;
  uint4* stage;
  cudaMalloc(&s, m * 4);
  cudaMalloc(&d, m * 4);
  cudaMalloc(&w, m * 4);
  cudaMalloc(&L, nv * 4);
  cudaMalloc(&stage, m * 16);
  cudaMalloc(&counts, (m / kChunk + 1) * 4);
  k_fill_rmat<<<sms * 8, 256>>>(s, m, 1);
  k_fill_rmat<<<sms * 8, 256>>>(d, m, 2);
  if (tree) {
    k_fill_uniform<<<sms * 8, 256>>>(s, 1ull << kScale, 5);
    k_fill_uniform<<<sms * 8, 256>>>(d, 1ull << kScale, 6);
    printf("first 2^26 edges: uniform random endpoints\n");
  }
  k_fill_w<<<sms * 8, 256>>>(w, m);
  k_fill_map<<<sms * 8, 256>>>(L, nv);
  const uint32_t pivot = (uint32_t)(0.09 * 4294967296.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](const char* name, auto&& launch) {
    launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.3f ms  %6.1f G edges/s\n", name, ms / 3, m / (ms / 3 / 1e3) / 1e9);
  };
  int ba = 0, bb = 0, bc = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ba, k_filter_a, kBlock, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bb, k_filter_b<false>, kBlock, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bc, k_filter_b<true>, kBlock, 0);
  printf("blocks/SM: A %d  B %d  C %d\n", ba, bb, bc);
  time("A block tiles (3 barriers)", [&] { k_filter_a<<<sms * ba, kBlock>>>(s, d, w, L, m, pivot, stage, counts); });
  time("B warp chunks (no barrier)", [&] { k_filter_b<false><<<sms * bb, kBlock>>>(s, d, w, L, m, pivot, stage, (uint8_t*)counts); });
  time("C warp chunks + prefetched stream", [&] { k_filter_b<true><<<sms * bc, kBlock>>>(s, d, w, L, m, pivot, stage, (uint8_t*)counts); });
  for (int bps : {4, 5, 6, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "B at %d blocks/SM", bps);
    time(nm, [&] { k_filter_b<false><<<sms * bps, kBlock>>>(s, d, w, L, m, pivot, stage, (uint8_t*)counts); });
    snprintf(nm, sizeof nm, "C at %d blocks/SM", bps);
    time(nm, [&] { k_filter_b<true><<<sms * bps, kBlock>>>(s, d, w, L, m, pivot, stage, (uint8_t*)counts); });
  }
  // survivors (sanity: both shapes keep the same edges)
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
