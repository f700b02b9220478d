/*
 * oracle/mst_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's MST algorithms, used as the
 * parity checker for the CUDA path. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * library (paper_2005_06913_b200/libmstgpu.so) never does.
 *
 * Pinned against the reference itself: tests/test_oracle.py checks these
 * functions against (a) the golden vectors produced by the unchanged
 * reference code (tests/golden/, made by tests/golden/make_golden.py through
 * oracle/_ref/libmstref.so), (b) the known-answer totals of SURVEY.md App. B,
 * and (c) the reference library directly when oracle/_ref is built.
 *
 * Tie rule: edges are ordered by (weight, id). With distinct weights — the
 * reference's input contract (graph.cpp:118-125) — this is the reference's
 * order exactly; with ties it is a stable Kruskal.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_RANGE 2
#define ORACLE_ERR_OOM 8

/* ---- union-find: reference proj/src/simple_dsu.hpp:13-39 ---------------- */
typedef struct {
  uint32_t* parent;
  uint32_t* size;
} dsu_t;

static int dsu_init(dsu_t* d, uint32_t n) {
  d->parent = (uint32_t*)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  d->size = (uint32_t*)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  if (!d->parent || !d->size) return ORACLE_ERR_OOM;
  for (uint32_t v = 0; v < n; ++v) {
    d->parent[v] = v;
    d->size[v] = 1;
  }
  return ORACLE_OK;
}

static void dsu_free(dsu_t* d) {
  free(d->parent);
  free(d->size);
}

/* find with path halving (simple_dsu.hpp:21-27) */
static uint32_t dsu_find(dsu_t* d, uint32_t v) {
  while (d->parent[v] != v) {
    d->parent[v] = d->parent[d->parent[v]];
    v = d->parent[v];
  }
  return v;
}

/* union by size, true iff a union happened (simple_dsu.hpp:29-38) */
static int dsu_unite(dsu_t* d, uint32_t a, uint32_t b) {
  a = dsu_find(d, a);
  b = dsu_find(d, b);
  if (a == b) return 0;
  if (d->size[a] < d->size[b]) {
    uint32_t t = a;
    a = b;
    b = t;
  }
  d->parent[b] = a;
  d->size[a] += d->size[b];
  return 1;
}

/* ---- LSD radix sort of 64-bit keys (16-bit digits) ----------------------- */
static int radix_sort_u64(uint64_t* keys, uint64_t count, int bits) {
  if (count < 2) return ORACLE_OK;
  uint64_t* tmp = (uint64_t*)malloc(count * sizeof(uint64_t));
  if (!tmp) return ORACLE_ERR_OOM;
  uint64_t* hist = (uint64_t*)malloc(65536 * sizeof(uint64_t));
  if (!hist) {
    free(tmp);
    return ORACLE_ERR_OOM;
  }
  uint64_t* a = keys;
  uint64_t* b = tmp;
  for (int shift = 0; shift < bits; shift += 16) {
    memset(hist, 0, 65536 * sizeof(uint64_t));
    for (uint64_t i = 0; i < count; ++i) hist[(a[i] >> shift) & 0xFFFF]++;
    uint64_t sum = 0;
    for (int d = 0; d < 65536; ++d) {
      const uint64_t c = hist[d];
      hist[d] = sum;
      sum += c;
    }
    for (uint64_t i = 0; i < count; ++i) b[hist[(a[i] >> shift) & 0xFFFF]++] = a[i];
    uint64_t* t = a;
    a = b;
    b = t;
  }
  if (a != keys) memcpy(keys, a, count * sizeof(uint64_t));
  free(hist);
  free(tmp);
  return ORACLE_OK;
}

static int check_range(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst) {
  for (uint64_t i = 0; i < m; ++i)
    if (src[i] >= n || dst[i] >= n) return ORACLE_ERR_RANGE;
  return ORACLE_OK;
}

/* Ascending ids, and the u64 sum of their weights (boruvka_seq.cpp:20-30). */
static int finish(uint32_t* ids, uint64_t count, const uint32_t* w, uint64_t* out_total) {
  uint64_t* tmp = (uint64_t*)malloc((count ? count : 1) * sizeof(uint64_t));
  if (!tmp) return ORACLE_ERR_OOM;
  for (uint64_t i = 0; i < count; ++i) tmp[i] = ids[i];
  int rc = radix_sort_u64(tmp, count, 32);
  uint64_t total = 0;
  for (uint64_t i = 0; i < count; ++i) {
    ids[i] = (uint32_t)tmp[i];
    total += w[ids[i]];
  }
  free(tmp);
  *out_total = total;
  return rc;
}

/*
 * Kruskal oracle — reference proj/src/boruvka_seq.cpp:121-143: order edge ids
 * by weight (:126-129), unite with a private DSU (:131-140), stop at n-1
 * edges (:138), return ids sorted with the total weight (:20-30).
 * out_ids must hold n-1 entries. For a disconnected input the minimum
 * spanning forest comes back (count < n-1).
 */
int oracle_kruskal(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                   const uint32_t* w, uint32_t* out_ids, uint64_t* out_count,
                   uint64_t* out_total) {
  if (n < 1 || m >= 0xFFFFFFFFull) return ORACLE_ERR_ARG;
  int rc = check_range(n, m, src, dst);
  if (rc) return rc;
  uint64_t* order = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
  if (!order) return ORACLE_ERR_OOM;
  for (uint64_t i = 0; i < m; ++i) order[i] = ((uint64_t)w[i] << 32) | i;
  rc = radix_sort_u64(order, m, 64);
  if (rc) {
    free(order);
    return rc;
  }
  dsu_t d;
  if (dsu_init(&d, n)) {
    free(order);
    return ORACLE_ERR_OOM;
  }
  uint64_t count = 0;
  for (uint64_t k = 0; k < m && count + 1 < n; ++k) {
    const uint32_t e = (uint32_t)order[k];
    if (dsu_unite(&d, src[e], dst[e])) out_ids[count++] = e;
  }
  dsu_free(&d);
  free(order);
  *out_count = count;
  return finish(out_ids, count, w, out_total);
}

/*
 * Sequential Boruvka — reference proj/src/boruvka_seq.cpp:34-71: per round
 * reset minimum[] (:47), scan all edges with find on both endpoints and keep
 * the lighter edge per component (:49-56), then union each component along
 * its minimum edge if still separate (:58-67). ComponentForest's
 * find_halving / union_by_size (union_find.cpp:37-64) are restated by the
 * DSU above. Returns the round count as well.
 */
int oracle_boruvka_seq(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                       const uint32_t* w, uint32_t* out_ids, uint64_t* out_count,
                       uint64_t* out_total, uint32_t* out_rounds) {
  if (n < 1 || m >= 0xFFFFFFFFull) return ORACLE_ERR_ARG;
  int rc = check_range(n, m, src, dst);
  if (rc) return rc;
  const uint64_t none = ~0ull;
  uint64_t* minimum = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  dsu_t d;
  if (!minimum || dsu_init(&d, n)) {
    free(minimum);
    return ORACLE_ERR_OOM;
  }
  uint64_t count = 0;
  uint32_t rounds = 0;
  uint32_t components = n;
  for (;;) {
    if (components <= 1) break;
    ++rounds;
    for (uint32_t v = 0; v < n; ++v) minimum[v] = none;
    for (uint64_t e = 0; e < m; ++e) {
      const uint32_t c1 = dsu_find(&d, src[e]);
      const uint32_t c2 = dsu_find(&d, dst[e]);
      if (c1 == c2) continue;
      const uint64_t key = ((uint64_t)w[e] << 32) | e;
      if (key < minimum[c1]) minimum[c1] = key;
      if (key < minimum[c2]) minimum[c2] = key;
    }
    uint32_t merged = 0;
    for (uint32_t v = 0; v < n; ++v) {
      if (minimum[v] == none) continue;
      const uint32_t e = (uint32_t)minimum[v];
      if (dsu_unite(&d, src[e], dst[e])) {
        out_ids[count++] = e;
        ++merged;
      }
    }
    if (merged == 0) break; /* disconnected: forest complete */
    components -= merged;
  }
  free(minimum);
  dsu_free(&d);
  *out_count = count;
  if (out_rounds) *out_rounds = rounds;
  return finish(out_ids, count, w, out_total);
}

/*
 * Round-1 minimum table — the first pass of boruvka_seq.cpp:47-56 with every
 * vertex its own component: for each vertex the key (w<<32 | id) of its
 * lightest incident non-loop edge, ~0 if none. The GPU's k_min_round1 must
 * reproduce it exactly.
 */
int oracle_min_edges(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint32_t* w, uint64_t* out_min) {
  if (n < 1) return ORACLE_ERR_ARG;
  int rc = check_range(n, m, src, dst);
  if (rc) return rc;
  for (uint32_t v = 0; v < n; ++v) out_min[v] = ~0ull;
  for (uint64_t e = 0; e < m; ++e) {
    if (src[e] == dst[e]) continue;
    const uint64_t key = ((uint64_t)w[e] << 32) | e;
    if (key < out_min[src[e]]) out_min[src[e]] = key;
    if (key < out_min[dst[e]]) out_min[dst[e]] = key;
  }
  return ORACLE_OK;
}

/*
 * Structural check of a result — reference proj/src/verify.cpp:15-57 minus
 * the oracle comparison: range, n-1 edges, acyclic, spanning, weight sum.
 * flags bit0 edge_count_ok, bit1 acyclic, bit2 spanning. Returns
 * ORACLE_ERR_RANGE on an id >= m (verify.cpp:19-22 throws out_of_range).
 */
int oracle_verify(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                  const uint32_t* w, const uint32_t* ids, uint64_t count, uint32_t* out_flags,
                  uint64_t* out_sum) {
  for (uint64_t i = 0; i < count; ++i)
    if (ids[i] >= m) return ORACLE_ERR_RANGE;
  dsu_t d;
  if (dsu_init(&d, n)) return ORACLE_ERR_OOM;
  uint32_t components = n;
  int acyclic = 1;
  uint64_t sum = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t e = ids[i];
    sum += w[e];
    if (dsu_unite(&d, src[e], dst[e]))
      --components;
    else
      acyclic = 0;
  }
  dsu_free(&d);
  *out_flags = (count == (uint64_t)n - 1 ? 1u : 0u) | (acyclic ? 2u : 0u) | (components == 1 ? 4u : 0u);
  *out_sum = sum;
  return ORACLE_OK;
}
