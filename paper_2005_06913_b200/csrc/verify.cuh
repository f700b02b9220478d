// GPU verifier of an MST result — the checks of the reference's verify_mst
// (/root/reference/proj/src/verify.cpp:15-57, VerifyReport in
// proj/include/mst/verify.hpp) without the CPU Kruskal in the loop:
//
//   range      every id < m, else out_of_range (verify.cpp:19-22)
//   count      |ids| == n - 1                  (verify.cpp:25)
//   acyclic /  a private union-find over the result edges (verify.cpp:27-37):
//   spanning   the reference counts failed unite() calls one by one; here
//              the edges are united concurrently (lock-free, hook larger root
//              under smaller by CAS) and the successful unions counted. Any
//              order of unions succeeds exactly n - components times, so
//              acyclic <=> unions == |ids| and spanning <=> unions == n - 1.
//   weight     sum of the result edges' weights (u64) vs the oracle total
//   edge set   the ids as a set (bitmap over m) vs the oracle's ids
//              (verify.cpp:41-43 sorts and compares; duplicates in the result
//              leave fewer bits than entries, so they never compare equal)
//
// The union-find is independent of the Boruvka engine (no shared kernels),
// so a bug there cannot hide itself here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mstgpu {

struct VerifyCounters {
  unsigned long long weight;
  unsigned long long unions;
  unsigned int range_err;
  unsigned int set_mismatch;
};

// Edge endpoint/weight access of the verifier: SoA u32 or the reference's
// AoS Edge {u32 src, u32 dest, u64 weight}.
struct VSoa {
  const uint32_t *src, *dst, *w;
  __device__ __forceinline__ uint32_t a(uint64_t e) const { return __ldg(src + e); }
  __device__ __forceinline__ uint32_t b(uint64_t e) const { return __ldg(dst + e); }
  __device__ __forceinline__ unsigned long long wt(uint64_t e) const { return __ldg(w + e); }
};
struct VAos {
  const uint4* e4;
  __device__ __forceinline__ uint32_t a(uint64_t e) const { return __ldg(&e4[e].x); }
  __device__ __forceinline__ uint32_t b(uint64_t e) const { return __ldg(&e4[e].y); }
  __device__ __forceinline__ unsigned long long wt(uint64_t e) const {
    const uint4 v = __ldg(e4 + e);
    return ((unsigned long long)v.w << 32) | v.z;
  }
};

__global__ void kv_iota(uint32_t* __restrict__ parent, uint32_t n) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    parent[v] = (uint32_t)v;
}

// Root with path halving. parent[x] <= x always (roots only ever hook under
// a smaller root), and every value written is an ancestor, so concurrent
// halving is benign.
__device__ __forceinline__ uint32_t v_find(uint32_t* parent, uint32_t x) {
  uint32_t p = __ldcg(parent + x);
  while (p != x) {
    const uint32_t gp = __ldcg(parent + p);
    if (gp != p) parent[x] = gp;
    x = p;
    p = gp;
  }
  return x;
}

// Range check, weight sum, union of the result edges and the result bitmap.
// range_err bit 0: an id >= m; bit 1: an endpoint >= n (a malformed graph:
// its union-find would index past parent[]).
template <class V>
__global__ void __launch_bounds__(256) kv_unite(V g, uint32_t n, uint64_t m, const uint32_t* __restrict__ ids,
                                                uint64_t count,
                                                uint32_t* __restrict__ parent, uint32_t* __restrict__ bits,
                                                VerifyCounters* ctr) {
  unsigned long long wsum = 0, unions = 0;
  unsigned int bad = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = __ldg(ids + i);
    if (e >= m) {
      bad = 1;
      continue;
    }
    const uint32_t ea = g.a(e), eb = g.b(e);
    if (ea >= n || eb >= n) {
      bad |= 2;
      continue;
    }
    wsum += g.wt(e);
    if (bits) atomicOr(bits + (e >> 5), 1u << (e & 31));
    uint32_t ra = v_find(parent, ea), rb = v_find(parent, eb);
    while (ra != rb) {
      const uint32_t hi = ra > rb ? ra : rb, lo = ra > rb ? rb : ra;
      const uint32_t old = atomicCAS(parent + hi, hi, lo);
      if (old == hi) {
        ++unions;
        break;
      }
      ra = v_find(parent, hi);
      rb = v_find(parent, lo);
    }
  }
  for (int o = 16; o; o >>= 1) {
    wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    unions += __shfl_xor_sync(0xffffffffu, unions, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (wsum) atomicAdd(&ctr->weight, wsum);
    if (unions) atomicAdd(&ctr->unions, unions);
    if (bad) atomicOr(&ctr->range_err, bad);
  }
}

__global__ void kv_mark(const uint32_t* __restrict__ ids, uint64_t count, uint64_t m, uint32_t* __restrict__ bits,
                        VerifyCounters* ctr) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = __ldg(ids + i);
    if (e >= m) {
      atomicOr(&ctr->set_mismatch, 1u);  // an oracle id outside the graph never matches
      continue;
    }
    atomicOr(bits + (e >> 5), 1u << (e & 31));
  }
}

__global__ void kv_compare(const uint4* __restrict__ a, const uint4* __restrict__ b, uint64_t n4,
                           VerifyCounters* ctr) {
  unsigned int diff = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 x = __ldcs(a + i), y = __ldcs(b + i);
    diff |= (x.x ^ y.x) | (x.y ^ y.y) | (x.z ^ y.z) | (x.w ^ y.w);
  }
  if (__any_sync(0xffffffffu, diff != 0) && (threadIdx.x & 31) == 0) atomicOr(&ctr->set_mismatch, 1u);
}

}  // namespace mstgpu
