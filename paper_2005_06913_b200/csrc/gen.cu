// Seeded synthetic graphs for the BASELINE.json configs (c0..c4), produced
// identically on the host (std::thread) and on the GPU.
//
// Shapes follow BASELINE.json "configs" and SURVEY.md §8(d):
//   uniform: random spanning tree over a random vertex relabelling (vertex
//            label[i] attaches to label[j], j uniform in [0,i) — the shape of
//            the reference's generate_graph, graph.cpp:158-174), then uniform
//            pairs u != v with NO dedup; weights a permutation of 0..m-1.
//   grid:    rows x cols 4-neighbour lattice, natural ids.
//   R-MAT:   edgefactor * 2^scale draws with (a,b,c,d), self-loops dropped,
//            duplicates kept, plus a random spanning tree (placed first).
// Edge order: tree edges first, then the rest (as graph.cpp:170-182).
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "common.cuh"

namespace mstgpu {

namespace {

struct GenPlan {
  int kind;
  uint32_t n;
  uint64_t m;         // total edges
  uint64_t n_tree;    // tree edges at the front
  // uniform
  uint64_t k_tree, k_u, k_v;
  Perm label, weight;
  // grid
  uint32_t rows, cols;
  uint64_t horiz;     // horizontal edge count
  // rmat
  uint32_t scale;
  uint64_t draws;
  uint64_t k_rmat;
  uint64_t tA, tAB, tABC;
};

uint64_t threshold(double p) {
  if (p <= 0) return 0;
  const double t = std::floor(p * 4294967296.0);
  return t >= 4294967296.0 ? 4294967296ull : (uint64_t)t;
}

// Fills everything except m / weight perm for R-MAT (needs the kept count).
void plan_base(const mst_gen_spec_t& s, GenPlan& g) {
  g = GenPlan{};
  g.kind = s.kind;
  if (s.kind == 0) {
    if (s.n < 2) throw MstError{MST_ERR_INVALID_ARG, "uniform generator: need n >= 2"};
    if (s.m < (uint64_t)s.n - 1)
      throw MstError{MST_ERR_INVALID_ARG, "uniform generator: m < n-1 cannot connect"};
    if (s.m >= 0xFFFFFFFFull) throw MstError{MST_ERR_INVALID_ARG, "generator: m must be < 2^32-1"};
    g.n = s.n;
    g.m = s.m;
    g.n_tree = s.n - 1;
  } else if (s.kind == 1) {
    if (s.rows < 1 || s.cols < 1 || (uint64_t)s.rows * s.cols < 2 ||
        (uint64_t)s.rows * s.cols > 0xFFFFFFFFull)
      throw MstError{MST_ERR_INVALID_ARG, "grid generator: bad rows/cols"};
    g.rows = s.rows;
    g.cols = s.cols;
    g.n = s.rows * s.cols;
    g.horiz = (uint64_t)s.rows * (s.cols - 1);
    g.m = g.horiz + (uint64_t)(s.rows - 1) * s.cols;
    g.n_tree = 0;
  } else if (s.kind == 2) {
    if (s.scale < 1 || s.scale > 31 || s.edgefactor < 1)
      throw MstError{MST_ERR_INVALID_ARG, "rmat generator: need 1 <= scale <= 31, edgefactor >= 1"};
    if (!(s.a >= 0 && s.b >= 0 && s.c >= 0 && s.a + s.b + s.c <= 1.0))
      throw MstError{MST_ERR_INVALID_ARG, "rmat generator: bad probabilities"};
    g.scale = s.scale;
    g.n = 1u << s.scale;
    g.n_tree = g.n - 1;
    g.draws = (uint64_t)s.edgefactor << s.scale;
    g.k_rmat = stream_key(s.seed, 6);
    g.tA = threshold(s.a);
    g.tAB = threshold(s.a + s.b);
    g.tABC = threshold(s.a + s.b + s.c);
  } else {
    throw MstError{MST_ERR_INVALID_ARG, "generator: unknown kind"};
  }
  g.k_tree = stream_key(s.seed, 2);
  g.k_u = stream_key(s.seed, 3);
  g.k_v = stream_key(s.seed, 4);
  if (g.n_tree) g.label = make_perm(g.n, s.seed, 1);
}

void plan_finish(const mst_gen_spec_t& s, GenPlan& g) {
  if (g.m >= 0xFFFFFFFFull) throw MstError{MST_ERR_INVALID_ARG, "generator: m must be < 2^32-1"};
  g.weight = make_perm(g.m, s.seed, 5);
}

MST_HD void tree_edge(const GenPlan& g, uint64_t e, uint32_t& a, uint32_t& b) {
  const uint64_t i = e + 1;
  const uint64_t j = bounded(rand_at(g.k_tree, i), i);
  a = (uint32_t)perm_apply(g.label, i);
  b = (uint32_t)perm_apply(g.label, j);
}

MST_HD void uniform_edge(const GenPlan& g, uint64_t e, uint32_t& a, uint32_t& b) {
  const uint64_t u = bounded(rand_at(g.k_u, e), g.n);
  const uint64_t v = (u + 1 + bounded(rand_at(g.k_v, e), g.n - 1)) % g.n;
  a = (uint32_t)u;
  b = (uint32_t)v;
}

MST_HD void grid_edge(const GenPlan& g, uint64_t e, uint32_t& a, uint32_t& b) {
  if (e < g.horiz) {
    const uint64_t r = e / (g.cols - 1), c = e % (g.cols - 1);
    a = (uint32_t)(r * g.cols + c);
    b = a + 1;
  } else {
    const uint64_t f = e - g.horiz;
    const uint64_t r = f / g.cols, c = f % g.cols;
    a = (uint32_t)(r * g.cols + c);
    b = a + g.cols;
  }
}

MST_HD void rmat_draw(const GenPlan& g, uint64_t k, uint32_t& a, uint32_t& b) {
  uint32_t s = 0, d = 0;
  uint64_t word = 0;
  for (uint32_t l = 0; l < g.scale; ++l) {
    if ((l & 1) == 0) word = rand_at(g.k_rmat, k * 16 + (l >> 1));
    const uint64_t u = (l & 1) ? (word >> 32) : (word & 0xFFFFFFFFull);
    const uint32_t bit = 1u << (g.scale - 1 - l);
    if (u < g.tA) {
    } else if (u < g.tAB) {
      d |= bit;
    } else if (u < g.tABC) {
      s |= bit;
    } else {
      s |= bit;
      d |= bit;
    }
  }
  a = s;
  b = d;
}

// ------------------------------- host --------------------------------------

int host_threads(int threads) {
  if (threads > 0) return threads;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? (int)hc : 1;
}

template <class F>
void parallel_for(uint64_t count, int threads, F&& f) {
  threads = (int)std::min<uint64_t>((uint64_t)threads, std::max<uint64_t>(1, count / 4096));
  if (threads <= 1) {
    f(0, 0, count);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const uint64_t lo = count * t / threads, hi = count * (t + 1) / threads;
    pool.emplace_back([&f, t, lo, hi] { f(t, lo, hi); });
  }
  for (auto& th : pool) th.join();
}

uint64_t rmat_count_host(const GenPlan& g, int threads, std::vector<uint64_t>* per_thread) {
  const int T = host_threads(threads);
  std::vector<uint64_t> counts(T, 0);
  parallel_for(g.draws, T, [&](int t, uint64_t lo, uint64_t hi) {
    uint64_t c = 0;
    for (uint64_t k = lo; k < hi; ++k) {
      uint32_t a, b;
      rmat_draw(g, k, a, b);
      c += (a != b);
    }
    counts[t] = c;
  });
  uint64_t total = 0;
  for (uint64_t c : counts) total += c;
  if (per_thread) *per_thread = counts;
  return total;
}

// ------------------------------- device ------------------------------------

__global__ void k_gen_simple(GenPlan g, uint32_t* src, uint32_t* dst, uint32_t* w) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < g.m; e += stride) {
    uint32_t a, b;
    if (e < g.n_tree) {
      tree_edge(g, e, a, b);
    } else if (g.kind == 0) {
      uniform_edge(g, e, a, b);
    } else {
      grid_edge(g, e, a, b);
    }
    src[e] = a;
    dst[e] = b;
    w[e] = (uint32_t)perm_apply(g.weight, e);
  }
}

constexpr int kGenBlock = 256;
constexpr uint64_t kGenChunk = 1ull << 16;  // draws per block in the R-MAT passes

__global__ void k_rmat_count(GenPlan g, uint32_t* counts) {
  __shared__ uint32_t s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * kGenChunk;
  const uint64_t hi = lo + kGenChunk < g.draws ? lo + kGenChunk : g.draws;
  uint32_t c = 0;
  for (uint64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    uint32_t a, b;
    rmat_draw(g, k, a, b);
    c += (a != b);
  }
  atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s_cnt;
}

// Ordered compaction of one chunk of draws to [offset[chunk], ...).
__global__ void k_rmat_write(GenPlan g, const uint64_t* offsets, uint32_t* src, uint32_t* dst) {
  __shared__ uint32_t s_warp[kGenBlock / 32];
  __shared__ uint64_t s_run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_run = g.n_tree + offsets[blockIdx.x];
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * kGenChunk;
  const uint64_t hi = lo + kGenChunk < g.draws ? lo + kGenChunk : g.draws;
  for (uint64_t base = lo; base < hi; base += blockDim.x) {
    const uint64_t k = base + threadIdx.x;
    uint32_t a = 0, b = 0;
    bool keep = false;
    if (k < hi) {
      rmat_draw(g, k, a, b);
      keep = a != b;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (int i = 0; i < kGenBlock / 32; ++i) {
      before += (i < warp) ? s_warp[i] : 0;
      total += s_warp[i];
    }
    const uint64_t run = s_run;
    if (keep) {
      const uint64_t pos = run + before + __popc(bal & ((1u << lane) - 1));
      src[pos] = a;
      dst[pos] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_run = run + total;
    __syncthreads();
  }
}

__global__ void k_gen_tree_and_weights(GenPlan g, uint32_t* src, uint32_t* dst, uint32_t* w) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < g.m; e += stride) {
    if (e < g.n_tree) {
      uint32_t a, b;
      tree_edge(g, e, a, b);
      src[e] = a;
      dst[e] = b;
    }
    w[e] = (uint32_t)perm_apply(g.weight, e);
  }
}

uint64_t rmat_count_device(const GenPlan& g, std::vector<uint64_t>* offsets_out) {
  const uint64_t chunks = (g.draws + kGenChunk - 1) / kGenChunk;
  uint32_t* d_counts = nullptr;
  MST_CUDA_CHECK(cudaMalloc(&d_counts, chunks * sizeof(uint32_t)));
  k_rmat_count<<<(unsigned)chunks, kGenBlock>>>(g, d_counts);
  std::vector<uint32_t> counts(chunks);
  cudaError_t e1 = cudaGetLastError();
  cudaError_t e2 = cudaMemcpy(counts.data(), d_counts, chunks * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(d_counts);
  MST_CUDA_CHECK(e1);
  MST_CUDA_CHECK(e2);
  uint64_t total = 0;
  if (offsets_out) offsets_out->resize(chunks);
  for (uint64_t i = 0; i < chunks; ++i) {
    if (offsets_out) (*offsets_out)[i] = total;
    total += counts[i];
  }
  return total;
}

}  // namespace

}  // namespace mstgpu

using namespace mstgpu;

extern "C" int mst_gen_count(const mst_gen_spec_t* spec, uint64_t* out_m) {
  try {
    if (!spec || !out_m) throw MstError{MST_ERR_INVALID_ARG, "mst_gen_count: null argument"};
    GenPlan g;
    plan_base(*spec, g);
    if (spec->kind == 2) {
      int dev_count = 0;
      const bool have_gpu = cudaGetDeviceCount(&dev_count) == cudaSuccess && dev_count > 0;
      cudaGetLastError();
      g.m = g.n_tree + (have_gpu ? rmat_count_device(g, nullptr) : rmat_count_host(g, 0, nullptr));
    }
    if (g.m >= 0xFFFFFFFFull) throw MstError{MST_ERR_INVALID_ARG, "generator: m must be < 2^32-1"};
    *out_m = g.m;
    return MST_OK;
  } catch (const MstError& e) {
    set_last_error(e.msg);
    return e.code;
  }
}

extern "C" int mst_gen_host(const mst_gen_spec_t* spec, uint32_t* src, uint32_t* dst, uint32_t* w,
                            int threads) {
  try {
    if (!spec || !src || !dst || !w) throw MstError{MST_ERR_INVALID_ARG, "mst_gen_host: null argument"};
    GenPlan g;
    plan_base(*spec, g);
    const int T = host_threads(threads);
    if (spec->kind == 2) {
      std::vector<uint64_t> per;
      const uint64_t kept = rmat_count_host(g, T, &per);
      g.m = g.n_tree + kept;
      plan_finish(*spec, g);
      // second pass: each thread writes its own ordered slice
      std::vector<uint64_t> off(per.size(), 0);
      for (size_t t = 1; t < per.size(); ++t) off[t] = off[t - 1] + per[t - 1];
      parallel_for(g.draws, T, [&](int t, uint64_t lo, uint64_t hi) {
        uint64_t pos = g.n_tree + off[t];
        for (uint64_t k = lo; k < hi; ++k) {
          uint32_t a, b;
          rmat_draw(g, k, a, b);
          if (a != b) {
            src[pos] = a;
            dst[pos] = b;
            ++pos;
          }
        }
      });
      parallel_for(g.m, T, [&](int, uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
          if (e < g.n_tree) tree_edge(g, e, src[e], dst[e]);
          w[e] = (uint32_t)perm_apply(g.weight, e);
        }
      });
    } else {
      plan_finish(*spec, g);
      parallel_for(g.m, T, [&](int, uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
          uint32_t a, b;
          if (e < g.n_tree)
            tree_edge(g, e, a, b);
          else if (g.kind == 0)
            uniform_edge(g, e, a, b);
          else
            grid_edge(g, e, a, b);
          src[e] = a;
          dst[e] = b;
          w[e] = (uint32_t)perm_apply(g.weight, e);
        }
      });
    }
    return MST_OK;
  } catch (const MstError& e) {
    set_last_error(e.msg);
    return e.code;
  }
}

extern "C" int mst_gen_device(const mst_gen_spec_t* spec, uint32_t* d_src, uint32_t* d_dst,
                              uint32_t* d_w) {
  try {
    if (!spec || !d_src || !d_dst || !d_w)
      throw MstError{MST_ERR_INVALID_ARG, "mst_gen_device: null argument"};
    GenPlan g;
    plan_base(*spec, g);
    int sms = 148;
    int dev = 0;
    MST_CUDA_CHECK(cudaGetDevice(&dev));
    MST_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = (unsigned)sms * 8;
    if (spec->kind == 2) {
      std::vector<uint64_t> offsets;
      const uint64_t kept = rmat_count_device(g, &offsets);
      g.m = g.n_tree + kept;
      plan_finish(*spec, g);
      uint64_t* d_off = nullptr;
      MST_CUDA_CHECK(cudaMalloc(&d_off, offsets.size() * sizeof(uint64_t)));
      cudaError_t e = cudaMemcpy(d_off, offsets.data(), offsets.size() * sizeof(uint64_t),
                                 cudaMemcpyHostToDevice);
      if (e == cudaSuccess) {
        k_rmat_write<<<(unsigned)offsets.size(), kGenBlock>>>(g, d_off, d_src, d_dst);
        k_gen_tree_and_weights<<<grid, kGenBlock>>>(g, d_src, d_dst, d_w);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
      }
      cudaFree(d_off);
      MST_CUDA_CHECK(e);
    } else {
      plan_finish(*spec, g);
      k_gen_simple<<<grid, kGenBlock>>>(g, d_src, d_dst, d_w);
      MST_CUDA_CHECK(cudaGetLastError());
      MST_CUDA_CHECK(cudaDeviceSynchronize());
    }
    return MST_OK;
  } catch (const MstError& e) {
    set_last_error(e.msg);
    return e.code;
  }
}
