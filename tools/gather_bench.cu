// Random-access throughput on this GPU: what bounds the label gathers and
// the min-table offers of the edge passes (heavy filter, compactions).
//   gathers/s of random 4 B loads vs table size (L1 / L2 / DRAM resident)
//   and cache operator; random 8 B atomicMin (RED) and read-first offers;
//   a heavy-filter-shaped pass (stream src/dst + 2 gathers + compare).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_bench.cu -o tools/gather_bench
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int kOp, int kU>
__global__ void k_gather(const uint32_t* __restrict__ t, uint32_t mask, uint64_t n, uint32_t seed, uint32_t* sink) {
  uint32_t acc = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU + threadIdx.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x * kU) {
    uint32_t idx[kU], v[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) idx[k] = hash32((uint32_t)(base + k * blockDim.x) ^ seed) & mask;
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      if (kOp == 0) v[k] = t[idx[k]];
      else if (kOp == 1) v[k] = __ldcg(t + idx[k]);
      else if (kOp == 2) v[k] = __ldg(t + idx[k]);
      else v[k] = __ldcs(t + idx[k]);
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) acc += v[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <int kMode, int kU>
__global__ void k_offer(unsigned long long* __restrict__ t, uint32_t mask, uint64_t n, uint32_t seed) {
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU + threadIdx.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x * kU) {
    uint32_t idx[kU];
    unsigned long long key[kU], cur[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint32_t h = hash32((uint32_t)(base + k * blockDim.x) ^ seed);
      idx[k] = h & mask;
      key[k] = ((unsigned long long)hash32(h) << 32) | (uint32_t)(base + k * blockDim.x);
    }
    if (kMode == 0) {
#pragma unroll
      for (int k = 0; k < kU; ++k) atomicMin(t + idx[k], key[k]);
    } else {
#pragma unroll
      for (int k = 0; k < kU; ++k) cur[k] = __ldcg(t + idx[k]);
#pragma unroll
      for (int k = 0; k < kU; ++k)
        if (key[k] < cur[k]) atomicMin(t + idx[k], key[k]);
    }
  }
}

// heavy-filter shape: stream src,dst (8 B/edge), gather L[src], L[dst], count keeps
template <int kU>
__global__ void k_filter(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                         const uint32_t* __restrict__ L, uint64_t m, unsigned long long* cnt) {
  uint32_t c = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU + threadIdx.x; base < m;
       base += (uint64_t)gridDim.x * blockDim.x * kU) {
    uint32_t a[kU], b[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * blockDim.x;
      a[k] = i < m ? __ldcs(src + i) : 0u;
      b[k] = i < m ? __ldcs(dst + i) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      a[k] = __ldg(L + a[k]);
      b[k] = __ldg(L + b[k]);
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) c += a[k] != b[k];
  }
  atomicAdd(cnt, (unsigned long long)c);
}

__global__ void k_fill_rand(uint32_t* x, uint64_t n, uint32_t mask, uint32_t seed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] = hash32((uint32_t)i * 2654435761u ^ seed) & mask;
}

static float timeit(void (*f)(void*), void* arg, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f(arg);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f(arg);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

struct G { const uint32_t* t; uint32_t mask; uint64_t n; uint32_t* sink; int grid; int op; };
static void run_gather(void* p) {
  G& g = *(G*)p;
  switch (g.op) {
    case 0: k_gather<0, 8><<<g.grid, 256>>>(g.t, g.mask, g.n, 7, g.sink); break;
    case 1: k_gather<1, 8><<<g.grid, 256>>>(g.t, g.mask, g.n, 7, g.sink); break;
    case 2: k_gather<2, 8><<<g.grid, 256>>>(g.t, g.mask, g.n, 7, g.sink); break;
    default: k_gather<3, 8><<<g.grid, 256>>>(g.t, g.mask, g.n, 7, g.sink); break;
  }
}
struct O { unsigned long long* t; uint32_t mask; uint64_t n; int grid; int mode; };
static void run_offer(void* p) {
  O& o = *(O*)p;
  if (o.mode == 0) k_offer<0, 4><<<o.grid, 256>>>(o.t, o.mask, o.n, 9);
  else k_offer<1, 4><<<o.grid, 256>>>(o.t, o.mask, o.n, 9);
}
struct F { const uint32_t *s, *d, *L; uint64_t m; unsigned long long* c; int grid; };
static void run_filter(void* p) {
  F& f = *(F*)p;
  k_filter<4><<<f.grid, 256>>>(f.s, f.d, f.L, f.m, f.c);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ghz = clk / 1e6;
  printf("SMs %d, clock %.3f GHz (attribute)\n", sms, ghz);
  const uint64_t tbytes = 1ull << 31;  // 2 GiB table
  uint32_t* t;
  cudaMalloc(&t, tbytes);
  cudaMemset(t, 1, tbytes);
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  const uint64_t n = 1ull << 30;  // gathers per launch
  const int grid = sms * 8;
  const char* ops[] = {"ld (ca)", "ldcg", "ldg (nc)", "ldcs"};
  for (uint64_t sz : {16ull << 10, 1ull << 20, 16ull << 20, 64ull << 20, 256ull << 20, 2048ull << 20}) {
    for (int op = 0; op < 4; ++op) {
      G g{t, (uint32_t)(sz / 4 - 1), n, sink, grid, op};
      const float ms = timeit(run_gather, &g);
      const double gps = n / (ms / 1e3);
      printf("gather table %7llu KB %-9s: %7.3f ms  %6.1f G/s  %.2f cyc/gather/SM\n",
             (unsigned long long)(sz >> 10), ops[op], ms, gps / 1e9, sms * ghz * 1e9 / gps);
    }
  }
  unsigned long long* t64 = (unsigned long long*)t;
  const uint64_t no = 1ull << 28;
  for (uint64_t sz : {1ull << 20, 64ull << 20, 512ull << 20, 2048ull << 20}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(t, 0xFF, sz);
      O o{t64, (uint32_t)(sz / 8 - 1), no, grid, mode};
      const float ms = timeit(run_offer, &o, 3);
      const double ops_s = no / (ms / 1e3);
      printf("offer table %7llu KB %-10s: %7.3f ms  %6.1f G/s  %.2f cyc/offer/SM\n", (unsigned long long)(sz >> 10),
             mode ? "read-first" : "RED", ms, ops_s / 1e9, sms * ghz * 1e9 / ops_s);
    }
  }
  // heavy-filter shape: m edges, vertex map of nv entries
  const uint64_t m = 1ull << 30;
  uint32_t *s, *d;
  cudaMalloc(&s, m * 4);
  cudaMalloc(&d, m * 4);
  unsigned long long* c;
  cudaMalloc(&c, 8);
  for (uint64_t nv : {1ull << 20, 1ull << 24, 1ull << 26}) {
    k_fill_rand<<<sms * 8, 256>>>(s, m, (uint32_t)(nv - 1), 1);
    k_fill_rand<<<sms * 8, 256>>>(d, m, (uint32_t)(nv - 1), 2);
    F f{s, d, t, m, c, grid};
    const float ms = timeit(run_filter, &f, 3);
    printf("filter m=2^30 map %6llu MB: %7.3f ms  %.1f G edges/s  stream %.2f TB/s  %.2f cyc/gather/SM\n",
           (unsigned long long)(nv * 4 >> 20), ms, m / (ms / 1e3) / 1e9, m * 8 / (ms / 1e3) / 1e12,
           sms * ghz * 1e9 / (2.0 * m / (ms / 1e3)));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
