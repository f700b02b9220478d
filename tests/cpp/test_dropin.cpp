// tests/cpp/test_dropin.cpp — the drop-in proof: the reference's own Graph,
// generator, Kruskal oracle and verifier (compiled unchanged into
// oracle/_ref/libmstref.so) against mst::boruvka_gpu (include/mst/
// boruvka_gpu.hpp -> libmstgpu.so). Mirrors the shape of the reference's
// proj/tests/test_boruvka_parallel.cpp. Built by `make -C oracle dropin`.
//
//   test_dropin          full suite (needs a GPU)
//   test_dropin --cpu    argument / no-device behaviour only
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mst/boruvka_gpu.hpp"
#include "mst/boruvka_seq.hpp"
#include "mst/graph.hpp"
#include "mst/verify.hpp"

using namespace mst;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                               \
  do {                                                                            \
    if (cond) {                                                                   \
      ++g_pass;                                                                   \
    } else {                                                                      \
      ++g_fail;                                                                   \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                             \
  } while (0)

template <class Ex, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const Ex&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Graph triangle() {
  const Edge es[] = {{0, 1, 1}, {1, 2, 2}, {0, 2, 3}};
  return build_graph(3, es);
}

static void same_as_oracle(Graph& g, int gpus = 1) {
  const MstResult oracle = kruskal_oracle(g);
  GpuRunInfo info;
  const MstResult r = boruvka_gpu(g, gpus, &info);
  CHECK(r.mst_edges == oracle.mst_edges);
  CHECK(r.total_weight == oracle.total_weight);
  CHECK(info.final_components == 1);
  const VerifyReport rep = verify_mst(g, r, oracle);
  CHECK(rep.all_ok());
  if (!rep.all_ok()) std::fprintf(stderr, "  %s\n", rep.details.c_str());
  CHECK(verify_mst_gpu(g, r, oracle).all_ok());
}

// verify_mst_gpu must report exactly what the reference's verify_mst does
// (verify.cpp:15-57): the five flags and the details line.
static void same_report(const Graph& g, const MstResult& r, const MstResult& oracle) {
  const VerifyReport a = verify_mst(g, r, oracle);
  const VerifyReport b = verify_mst_gpu(g, r, oracle);
  CHECK(a.is_spanning == b.is_spanning);
  CHECK(a.is_acyclic == b.is_acyclic);
  CHECK(a.edge_count_ok == b.edge_count_ok);
  CHECK(a.weight_matches_oracle == b.weight_matches_oracle);
  CHECK(a.edge_set_matches_oracle == b.edge_set_matches_oracle);
  CHECK(a.details == b.details);
  if (a.details != b.details) std::fprintf(stderr, "  ref: %s\n  gpu: %s\n", a.details.c_str(), b.details.c_str());
}

static void verifier_cases() {
  Graph g = generate_graph(3000, 6, 2);
  const MstResult oracle = kruskal_oracle(g);
  same_report(g, oracle, oracle);
  MstResult r = oracle;
  r.mst_edges.pop_back();  // one edge short: not spanning
  same_report(g, r, oracle);
  r = oracle;
  r.mst_edges.back() = r.mst_edges.front();  // duplicate: a cycle, one short
  same_report(g, r, oracle);
  r = oracle;
  std::vector<bool> in(static_cast<std::size_t>(g.edge_count()), false);
  for (EdgeId e : oracle.mst_edges) in[static_cast<std::size_t>(e)] = true;
  EdgeId other = 0;
  while (in[static_cast<std::size_t>(other)]) ++other;
  r.mst_edges[r.mst_edges.size() / 2] = other;  // a non-MST edge swapped in
  same_report(g, r, oracle);
  r = oracle;
  std::reverse(r.mst_edges.begin(), r.mst_edges.end());  // order does not matter
  same_report(g, r, oracle);
  r = oracle;
  r.total_weight += 1;  // the result's own total disagrees with its edges
  same_report(g, r, oracle);
  r = oracle;
  r.mst_edges.push_back(g.edge_count());  // outside [0, m)
  CHECK(throws<std::out_of_range>([&] { verify_mst(g, r, oracle); }));
  CHECK(throws<std::out_of_range>([&] { verify_mst_gpu(g, r, oracle); }));
}

// binary SoA round trip through the reference's build_graph (host only)
static void io_cases() {
  Graph g = generate_graph(3000, 6, 5);
  const std::string path = "/tmp/test_dropin_soa.mstb";
  save_graph_soa(g, path);
  const Graph h = load_graph_soa(path);
  CHECK(h.vertex_count() == g.vertex_count() && h.edge_count() == g.edge_count());
  bool same = true;
  for (EdgeId i = 0; i < g.edge_count(); ++i)
    same = same && h.edge(i).src == g.edge(i).src && h.edge(i).dest == g.edge(i).dest &&
           h.edge(i).weight == g.edge(i).weight;
  CHECK(same);
  std::remove(path.c_str());
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  {
    Graph g = triangle();
    CHECK(throws<std::invalid_argument>([&] { boruvka_gpu(g, 0); }));   // boruvka_parallel.cpp:86
    CHECK(throws<std::invalid_argument>([&] { boruvka_gpu(g, -2); }));
  }
  io_cases();  // host-only: no device needed
  if (cpu_only) {
    Graph g = triangle();
    CHECK(throws<WorkerPanic>([&] { boruvka_gpu(g); }));  // no device: loud, no CPU fallback
    std::printf("cpu checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
  }
  // hand graphs of test_boruvka_seq.cpp:17-26,40-78,134-140
  {
    Graph g = triangle();
    const MstResult r = boruvka_gpu(g);
    CHECK((r.mst_edges == std::vector<EdgeId>{0, 1}) && r.total_weight == 3);
  }
  {
    const Edge es[] = {{0, 1, 4}, {1, 2, 9}};
    Graph g = build_graph(3, es);
    const MstResult r = boruvka_gpu(g);
    CHECK((r.mst_edges == std::vector<EdgeId>{0, 1}) && r.total_weight == 13);
  }
  {
    const Edge es[] = {{0, 1, 1}, {0, 2, 2}, {0, 3, 3}, {1, 2, 4}, {1, 3, 5}, {2, 3, 6}};
    Graph g = build_graph(4, es);
    CHECK(boruvka_gpu(g).total_weight == 6);
    same_as_oracle(g);
  }
  {
    const Edge es[] = {{0, 1, 1}, {0, 2, 2}, {0, 3, 3}, {0, 4, 4}};
    Graph g = build_graph(5, es);
    const MstResult r = boruvka_gpu(g);
    CHECK((r.mst_edges == std::vector<EdgeId>{0, 1, 2, 3}) && r.total_weight == 10);
  }
  {
    const Edge es[] = {{0, 1, 7}};
    Graph g = build_graph(2, es);
    CHECK((boruvka_gpu(g).mst_edges == std::vector<EdgeId>{0}));
  }
  // generated graphs of test_boruvka_parallel.cpp:49-137
  for (std::uint64_t seed : {2ull, 5ull}) {
    Graph g = generate_graph(3000, 6, seed);
    same_as_oracle(g);
  }
  {
    Graph g = generate_graph(10'000, 6, 2);
    same_as_oracle(g);
  }
  {
    Graph g = generate_graph(2000, 5, 21);
    const MstResult seq = boruvka_seq(g);
    CHECK(boruvka_gpu(g).mst_edges == seq.mst_edges);
  }
  {
    Graph g = generate_graph(1500, 4, 13);
    for (int rep = 0; rep < 10; ++rep) same_as_oracle(g);
  }
  {
    Graph g = generate_graph(100'000, 9, 7);
    const MstResult oracle = kruskal_oracle(g);
    for (int rep = 0; rep < 5; ++rep) {
      const MstResult r = boruvka_gpu(g);
      CHECK(r.total_weight == oracle.total_weight);
      CHECK(r.mst_edges == oracle.mst_edges);
      CHECK(r.mst_edges.size() == g.vertex_count() - 1);
    }
  }
  // App. B known answers, presets of bench.cpp:41-50
  {
    const struct { VertexId n; int d; std::uint64_t seed; Weight total; } kat[] = {
        {10'000, 3, 103, 54'539'809ull},        {10'000, 6, 106, 59'021'951ull},
        {10'000, 9, 109, 59'952'592ull},        {100'000, 3, 1003, 5'460'175'173ull},
        {100'000, 6, 1006, 5'911'779'114ull},   {100'000, 9, 1009, 5'981'724'212ull},
        {1'000'000, 8, 1, 596'658'426'921ull}};
    for (const auto& k : kat) {
      Graph g = generate_graph(k.n, k.d, k.seed);
      const MstResult r = boruvka_gpu(g);
      CHECK(r.total_weight == k.total);
      CHECK(r.mst_edges.size() == k.n - 1);
    }
  }
  verifier_cases();
  std::printf("drop-in checks: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
