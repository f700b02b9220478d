// Shared host/device helpers for the B200 Boruvka library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/mst_gpu.h"

#if defined(__CUDACC__)
#define MST_HD __host__ __device__ __forceinline__
#else
#define MST_HD inline
#endif

namespace mstgpu {

// ---------------------------------------------------------------------------
// Error plumbing: every C-ABI entry returns a status and leaves a
// thread-local message (mst_gpu_last_error).
// ---------------------------------------------------------------------------
void set_last_error(const std::string& msg);

struct MstError {
  int code;
  std::string msg;
};

#define MST_CUDA_CHECK(expr)                                                          \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      throw ::mstgpu::MstError{_e == cudaErrorMemoryAllocation ? MST_ERR_OOM          \
                                                               : MST_ERR_CUDA,        \
                               std::string(#expr " failed: ") + cudaGetErrorString(_e) + \
                                   " (" __FILE__ ":" + std::to_string(__LINE__) + ")"}; \
    }                                                                                 \
  } while (0)

// ---------------------------------------------------------------------------
// Counter-based randomness for the synthetic inputs. Every value is a pure
// function of (seed, stream, index), so host and device generators agree
// bit-for-bit and any slice of a graph can be produced independently.
// ---------------------------------------------------------------------------
MST_HD uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

MST_HD uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ mix64(stream * 0xd1b54a32d192ed03ull + 0x632be59bd9b4e019ull));
}

MST_HD uint64_t rand_at(uint64_t key, uint64_t i) { return mix64(key + i * 0x9e3779b97f4a7c15ull); }

// floor(r * bound / 2^64): Lemire's multiply-high bounded draw.
MST_HD uint64_t bounded(uint64_t r, uint64_t bound) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(r, bound);
#else
  return (uint64_t)(((unsigned __int128)r * (unsigned __int128)bound) >> 64);
#endif
}

// Keyed bijection on [0, N) (4-round balanced Feistel network on the
// smallest even bit-width >= log2 N, plus cycle walking).
struct Perm {
  uint64_t n;
  uint32_t half;   // bits per half
  uint64_t mask;   // (1<<half)-1
  uint64_t k[4];
};

inline Perm make_perm(uint64_t n, uint64_t seed, uint64_t stream) {
  Perm p;
  p.n = n;
  uint32_t bits = 2;
  while (bits < 64 && (1ull << bits) < n) ++bits;
  if (bits & 1) ++bits;
  p.half = bits / 2;
  p.mask = (1ull << p.half) - 1;
  for (int r = 0; r < 4; ++r) p.k[r] = stream_key(seed, stream * 8 + r);
  return p;
}

MST_HD uint64_t perm_apply(const Perm& p, uint64_t x) {
  do {
    uint64_t L = x >> p.half, R = x & p.mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t F = mix64(p.k[r] ^ R) & p.mask;
      const uint64_t nl = R;
      R = L ^ F;
      L = nl;
    }
    x = (L << p.half) | R;
  } while (x >= p.n);
  return x;
}

}  // namespace mstgpu
