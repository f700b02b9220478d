/*
 * oracle/gen_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the seeded synthetic-graph generator of the
 * BASELINE.json configs (c0..c4), so that the checkers (the golden-answer
 * script, bench.py's --impl reference and cpu_baseline legs) can build the
 * exact input bytes WITHOUT loading the product library
 * (paper_2005_06913_b200/libmstgpu.so). tests/test_generators.py checks it
 * byte for byte against the product's host and device generators.
 *
 * The generator itself is this repo's (the reference's generate_graph,
 * graph.cpp:143-194, makes simple graphs only, which the BASELINE configs
 * are not): counter-based randomness (a splitmix64 finaliser keyed by
 * (seed, stream, index)), a 4-round Feistel bijection for the vertex
 * relabelling and the weight permutation, then
 *   uniform : tree edge i links label[i+1] to label[j], j < i+1 uniform
 *             (the shape of graph.cpp:158-174), then uniform pairs u != v;
 *   grid    : rows x cols 4-neighbour lattice (horizontal edges first);
 *   R-MAT   : edgefactor * 2^scale quadrant draws (a, b, c, d), self-loops
 *             dropped, duplicates kept, after a random spanning tree.
 * Weights are a permutation of 0..m-1 applied to the edge position.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GEN_OK 0
#define GEN_ERR_ARG 1
#define GEN_ERR_OOM 8

static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ mix64(stream * 0xd1b54a32d192ed03ull + 0x632be59bd9b4e019ull));
}

static uint64_t rand_at(uint64_t key, uint64_t i) { return mix64(key + i * 0x9e3779b97f4a7c15ull); }

/* floor(r * bound / 2^64) */
static uint64_t bounded(uint64_t r, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)r * (unsigned __int128)bound) >> 64);
}

typedef struct {
  uint64_t n;
  uint32_t half;
  uint64_t mask;
  uint64_t k[4];
} perm_t;

static perm_t make_perm(uint64_t n, uint64_t seed, uint64_t stream) {
  perm_t p;
  uint32_t bits = 2;
  while (bits < 64 && (1ull << bits) < n) ++bits;
  if (bits & 1) ++bits;
  p.n = n;
  p.half = bits / 2;
  p.mask = (1ull << p.half) - 1;
  for (int r = 0; r < 4; ++r) p.k[r] = stream_key(seed, stream * 8 + (uint64_t)r);
  return p;
}

static uint64_t perm_apply(const perm_t* p, uint64_t x) {
  do {
    uint64_t L = x >> p->half, R = x & p->mask;
    for (int r = 0; r < 4; ++r) {
      const uint64_t F = mix64(p->k[r] ^ R) & p->mask;
      const uint64_t nl = R;
      R = L ^ F;
      L = nl;
    }
    x = (L << p->half) | R;
  } while (x >= p->n);
  return x;
}

typedef struct {
  int kind;
  uint32_t n;
  uint64_t m, n_tree;
  uint64_t k_tree, k_u, k_v, k_rmat;
  perm_t label, weight;
  uint32_t rows, cols;
  uint64_t horiz;
  uint32_t scale;
  uint64_t draws, tA, tAB, tABC;
} plan_t;

static uint64_t threshold(double p) {
  if (p <= 0) return 0;
  const double t = (double)(uint64_t)(p * 4294967296.0); /* floor for p >= 0 */
  return t >= 4294967296.0 ? 4294967296ull : (uint64_t)t;
}

static int plan_base(int kind, uint32_t n, uint64_t m, uint32_t rows, uint32_t cols, uint32_t scale,
                     uint32_t edgefactor, double a, double b, double c, uint64_t seed, plan_t* g) {
  memset(g, 0, sizeof(*g));
  g->kind = kind;
  if (kind == 0) {
    if (n < 2 || m < (uint64_t)n - 1 || m >= 0xFFFFFFFFull) return GEN_ERR_ARG;
    g->n = n;
    g->m = m;
    g->n_tree = n - 1;
  } else if (kind == 1) {
    if (rows < 1 || cols < 1 || (uint64_t)rows * cols < 2 || (uint64_t)rows * cols > 0xFFFFFFFFull) return GEN_ERR_ARG;
    g->rows = rows;
    g->cols = cols;
    g->n = rows * cols;
    g->horiz = (uint64_t)rows * (cols - 1);
    g->m = g->horiz + (uint64_t)(rows - 1) * cols;
  } else if (kind == 2) {
    if (scale < 1 || scale > 31 || edgefactor < 1 || !(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
      return GEN_ERR_ARG;
    g->scale = scale;
    g->n = 1u << scale;
    g->n_tree = g->n - 1;
    g->draws = (uint64_t)edgefactor << scale;
    g->k_rmat = stream_key(seed, 6);
    g->tA = threshold(a);
    g->tAB = threshold(a + b);
    g->tABC = threshold(a + b + c);
  } else {
    return GEN_ERR_ARG;
  }
  g->k_tree = stream_key(seed, 2);
  g->k_u = stream_key(seed, 3);
  g->k_v = stream_key(seed, 4);
  if (g->n_tree) g->label = make_perm(g->n, seed, 1);
  return GEN_OK;
}

static void tree_edge(const plan_t* g, uint64_t e, uint32_t* a, uint32_t* b) {
  const uint64_t i = e + 1;
  const uint64_t j = bounded(rand_at(g->k_tree, i), i);
  *a = (uint32_t)perm_apply(&g->label, i);
  *b = (uint32_t)perm_apply(&g->label, j);
}

static void uniform_edge(const plan_t* g, uint64_t e, uint32_t* a, uint32_t* b) {
  const uint64_t u = bounded(rand_at(g->k_u, e), g->n);
  const uint64_t v = (u + 1 + bounded(rand_at(g->k_v, e), g->n - 1)) % g->n;
  *a = (uint32_t)u;
  *b = (uint32_t)v;
}

static void grid_edge(const plan_t* g, uint64_t e, uint32_t* a, uint32_t* b) {
  if (e < g->horiz) {
    const uint64_t r = e / (g->cols - 1), c = e % (g->cols - 1);
    *a = (uint32_t)(r * g->cols + c);
    *b = *a + 1;
  } else {
    const uint64_t f = e - g->horiz;
    const uint64_t r = f / g->cols, c = f % g->cols;
    *a = (uint32_t)(r * g->cols + c);
    *b = *a + g->cols;
  }
}

/* quadrant descent: two 32-bit uniforms per 64-bit draw, one per level */
static void rmat_draw(const plan_t* g, uint64_t k, uint32_t* a, uint32_t* b) {
  uint32_t s = 0, d = 0;
  uint64_t word = 0;
  for (uint32_t l = 0; l < g->scale; ++l) {
    if ((l & 1) == 0) word = rand_at(g->k_rmat, k * 16 + (l >> 1));
    const uint64_t u = (l & 1) ? (word >> 32) : (word & 0xFFFFFFFFull);
    const uint32_t bit = 1u << (g->scale - 1 - l);
    if (u < g->tA) {
    } else if (u < g->tAB) {
      d |= bit;
    } else if (u < g->tABC) {
      s |= bit;
    } else {
      s |= bit;
      d |= bit;
    }
  }
  *a = s;
  *b = d;
}

static int nthreads(int threads) {
#ifdef _OPENMP
  return threads > 0 ? threads : omp_get_max_threads();
#else
  (void)threads;
  return 1;
#endif
}

/* Per-chunk kept-draw counts of the R-MAT stream (chunks of 2^16 draws). */
#define RMAT_CHUNK (1ull << 16)

static uint64_t* rmat_chunk_counts(const plan_t* g, int T, uint64_t* chunks_out) {
  const uint64_t chunks = (g->draws + RMAT_CHUNK - 1) / RMAT_CHUNK;
  uint64_t* cnt = (uint64_t*)malloc((chunks + 1) * sizeof(uint64_t));
  if (!cnt) return NULL;
#pragma omp parallel for schedule(dynamic, 16) num_threads(T)
  for (int64_t ch = 0; ch < (int64_t)chunks; ++ch) {
    const uint64_t lo = (uint64_t)ch * RMAT_CHUNK;
    const uint64_t hi = lo + RMAT_CHUNK < g->draws ? lo + RMAT_CHUNK : g->draws;
    uint64_t c = 0;
    for (uint64_t k = lo; k < hi; ++k) {
      uint32_t a, b;
      rmat_draw(g, k, &a, &b);
      c += (a != b);
    }
    cnt[ch] = c;
  }
  *chunks_out = chunks;
  return cnt;
}

int oracle_gen_count(int kind, uint32_t n, uint64_t m, uint32_t rows, uint32_t cols, uint32_t scale,
                     uint32_t edgefactor, double a, double b, double c, uint64_t seed, int threads,
                     uint64_t* out_m) {
  plan_t g;
  int rc = plan_base(kind, n, m, rows, cols, scale, edgefactor, a, b, c, seed, &g);
  if (rc) return rc;
  if (kind == 2) {
    uint64_t chunks = 0;
    uint64_t* cnt = rmat_chunk_counts(&g, nthreads(threads), &chunks);
    if (!cnt) return GEN_ERR_OOM;
    uint64_t kept = 0;
    for (uint64_t i = 0; i < chunks; ++i) kept += cnt[i];
    free(cnt);
    g.m = g.n_tree + kept;
  }
  if (g.m >= 0xFFFFFFFFull) return GEN_ERR_ARG;
  *out_m = g.m;
  return GEN_OK;
}

/* src/dst/w must hold oracle_gen_count's m entries. */
int oracle_gen(int kind, uint32_t n, uint64_t m, uint32_t rows, uint32_t cols, uint32_t scale,
               uint32_t edgefactor, double a, double b, double c, uint64_t seed, int threads, uint32_t* src,
               uint32_t* dst, uint32_t* w, uint64_t* out_m) {
  plan_t g;
  int rc = plan_base(kind, n, m, rows, cols, scale, edgefactor, a, b, c, seed, &g);
  if (rc) return rc;
  const int T = nthreads(threads);
  if (kind == 2) {
    uint64_t chunks = 0;
    uint64_t* off = rmat_chunk_counts(&g, T, &chunks);
    if (!off) return GEN_ERR_OOM;
    uint64_t run = 0;
    for (uint64_t i = 0; i < chunks; ++i) {
      const uint64_t x = off[i];
      off[i] = run;
      run += x;
    }
    g.m = g.n_tree + run;
    if (g.m >= 0xFFFFFFFFull) {
      free(off);
      return GEN_ERR_ARG;
    }
#pragma omp parallel for schedule(dynamic, 16) num_threads(T)
    for (int64_t ch = 0; ch < (int64_t)chunks; ++ch) {
      const uint64_t lo = (uint64_t)ch * RMAT_CHUNK;
      const uint64_t hi = lo + RMAT_CHUNK < g.draws ? lo + RMAT_CHUNK : g.draws;
      uint64_t pos = g.n_tree + off[ch];
      for (uint64_t k = lo; k < hi; ++k) {
        uint32_t x, y;
        rmat_draw(&g, k, &x, &y);
        if (x != y) {
          src[pos] = x;
          dst[pos] = y;
          ++pos;
        }
      }
    }
    free(off);
  }
  g.weight = make_perm(g.m, seed, 5);
#pragma omp parallel for schedule(static) num_threads(T)
  for (int64_t ee = 0; ee < (int64_t)g.m; ++ee) {
    const uint64_t e = (uint64_t)ee;
    uint32_t x, y;
    if (e < g.n_tree) {
      tree_edge(&g, e, &x, &y);
      src[e] = x;
      dst[e] = y;
    } else if (g.kind == 0) {
      uniform_edge(&g, e, &x, &y);
      src[e] = x;
      dst[e] = y;
    } else if (g.kind == 1) {
      grid_edge(&g, e, &x, &y);
      src[e] = x;
      dst[e] = y;
    }
    w[e] = (uint32_t)perm_apply(&g.weight, e);
  }
  *out_m = g.m;
  return GEN_OK;
}
