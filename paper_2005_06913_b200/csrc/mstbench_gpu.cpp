// mstbench_gpu — the reference's benchmark CLI (proj/tools/mstbench.cpp) and
// run_bench loop (proj/src/bench.cpp:89-147) re-hosted for the GPU path
// (SURVEY §8(f)3). Same subcommands, CSV schema (bench.cpp:159-166:
// graph,algorithm,threads,trial,elapsed_ms,mst_weight,rounds,verified),
// progress lines and exit codes (0 ok, 1 usage, 2 graph error, 3
// verification failure); "threads" holds the GPU count. Only the C ABI of
// mst_gpu.h is used; a small argv parser replaces CLI11.
//
//   mstbench_gpu generate --config c0..c4 --out PATH [--binary]
//   mstbench_gpu run (--graph PATH | --config cN) --algo gpu[,gpu-device]
//                    [--gpus 1,2,..] [--reps 5] [--warmup 1] [--verify]
//                    [--oracle ANSWER] --csv OUT
//   mstbench_gpu summarize --csv PATH [--baseline REF.csv]
//   mstbench_gpu --list-presets
//
// Algorithms: "gpu" is mst_gpu_boruvka on host arrays (elapsed_ms = the
// whole call, copies included, like boruvka_cas's elapsed_ms); "gpu-device"
// keeps the edges resident in HBM and reports the device time of the MST.
// --verify checks every trial with the GPU verifier (mst_gpu_verify): the
// structural checks (n-1 edges, acyclic, spanning) and, with --oracle, the
// weight and the edge set against an answer file written by the pinned CPU
// oracle (oracle/answer.py: Kruskal of oracle/mst_oracle.c), computed once
// and reused for every trial like the reference's kruskal_oracle
// (bench.cpp:96-102, 119-126). Every row must also agree on the MST weight
// (bench.cpp:132-141). summarize prints per-(graph, algorithm, threads)
// medians and, when sequential / CAS rows of the reference's own mstbench
// are present (--baseline), the speedup table of bench.cpp:246-335 with the
// GPU rows as the parallel algorithms.
//
// Answer file: "MSTANS01", u32 n, u32 0, u64 count, u64 total weight, then
// count u32 edge ids in ascending order (little endian).
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <limits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mst_gpu.h"

namespace {

constexpr int kExitOk = 0, kExitUsage = 1, kExitGraph = 2, kExitVerify = 3;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct GraphError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct VerifyError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(int rc, const char* what) {
  if (rc == MST_OK || rc == MST_ERR_DISCONNECTED) return;
  const std::string msg = std::string(what) + ": " + mst_gpu_last_error();
  if (rc == MST_ERR_PARSE || rc == MST_ERR_RANGE || rc == MST_ERR_WEIGHT) throw GraphError(msg);
  if (rc == MST_ERR_INVALID_ARG) throw UsageError(msg);
  throw std::runtime_error(msg);
}

// The BASELINE.json workloads (paper_2005_06913_b200/configs.py).
struct Preset {
  const char* name;
  mst_gen_spec_t spec;
  const char* note;
};
const std::vector<Preset>& presets() {
  static const std::vector<Preset> p = {
      {"c0", {0, 1000000u, 4000000ull, 0, 0, 0, 0, 0.57, 0.19, 0.19, 0}, "uniform n=1M m=4M"},
      {"c1", {1, 2048u * 2048u, 0, 2048, 2048, 0, 0, 0.57, 0.19, 0.19, 1}, "grid 2048x2048"},
      {"c2", {2, 1u << 22, 0, 0, 0, 22, 16, 0.57, 0.19, 0.19, 2}, "R-MAT scale 22, edgefactor 16"},
      {"c3", {0, 16777216u, 268435456ull, 0, 0, 0, 0, 0.57, 0.19, 0.19, 3}, "uniform n=16.7M m=268M"},
      {"c4", {2, 1u << 26, 0, 0, 0, 26, 16, 0.57, 0.19, 0.19, 4}, "R-MAT scale 26, edgefactor 16"},
  };
  return p;
}
const Preset* find_preset(const std::string& name) {
  for (const Preset& p : presets())
    if (name == p.name) return &p;
  return nullptr;
}

struct HostGraph {
  std::string name;
  uint32_t n = 0;
  uint64_t m = 0;
  std::vector<uint32_t> src, dst, w;
};

HostGraph generate(const Preset& p) {
  HostGraph g;
  g.name = p.name;
  g.n = p.spec.n;
  check(mst_gen_count(&p.spec, &g.m), "generate");
  g.src.resize(g.m);
  g.dst.resize(g.m);
  g.w.resize(g.m);
  check(mst_gen_host(&p.spec, g.src.data(), g.dst.data(), g.w.data(), 0), "generate");
  return g;
}

std::string path_stem(const std::string& path) {
  const size_t slash = path.find_last_of("/\\");
  std::string name = slash == std::string::npos ? path : path.substr(slash + 1);
  const size_t dot = name.find_last_of('.');
  if (dot != std::string::npos && dot > 0) name.resize(dot);
  return name;
}

HostGraph load(const std::string& path) {
  HostGraph g;
  g.name = path_stem(path);
  const bool binary = mst_io_soa_header(path.c_str(), &g.n, &g.m) == MST_OK;
  if (!binary) check(mst_io_text_header(path.c_str(), &g.n, &g.m), "load");
  g.src.resize(g.m);
  g.dst.resize(g.m);
  g.w.resize(g.m);
  if (binary)
    check(mst_io_load_soa(path.c_str(), g.n, g.m, g.src.data(), g.dst.data(), g.w.data(), 0), "load");
  else
    check(mst_io_load_text(path.c_str(), g.n, g.m, g.src.data(), g.dst.data(), g.w.data()), "load");
  return g;
}

struct Row {
  std::string graph, algorithm;
  int threads = 1, trial = 1;
  double elapsed_ms = 0;
  uint64_t weight = 0;
  uint32_t rounds = 0;
  bool verified = false;
};

std::string format_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round-trip form, as bench.cpp
  return std::string(buf, r.ptr);
}

void write_csv(const std::vector<Row>& rows, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("write_csv: cannot open " + path);
  out << "graph,algorithm,threads,trial,elapsed_ms,mst_weight,rounds,verified\n";
  for (const Row& r : rows)
    out << r.graph << ',' << r.algorithm << ',' << r.threads << ',' << r.trial << ',' << format_double(r.elapsed_ms)
        << ',' << r.weight << ',' << r.rounds << ',' << (r.verified ? 1 : 0) << '\n';
  if (!out) throw std::runtime_error("write_csv: write failed for " + path);
}

std::vector<Row> read_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw UsageError("cannot open " + path);
  std::string line;
  std::getline(in, line);
  if (line != "graph,algorithm,threads,trial,elapsed_ms,mst_weight,rounds,verified")
    throw UsageError(path + ": not a benchmark CSV");
  std::vector<Row> rows;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::vector<std::string> f;
    std::stringstream ss(line);
    std::string x;
    while (std::getline(ss, x, ',')) f.push_back(x);
    if (f.size() != 8) throw UsageError(path + ": bad row '" + line + "'");
    Row r;
    r.graph = f[0];
    r.algorithm = f[1];
    r.threads = std::stoi(f[2]);
    r.trial = std::stoi(f[3]);
    r.elapsed_ms = std::stod(f[4]);
    r.weight = std::stoull(f[5]);
    r.rounds = (uint32_t)std::stoul(f[6]);
    r.verified = f[7] == "1";
    rows.push_back(r);
  }
  return rows;
}

struct Answer {
  uint32_t n = 0;
  uint64_t total = 0;
  std::vector<uint32_t> ids;
};

Answer read_answer(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw UsageError("cannot open oracle answer " + path);
  char magic[8];
  uint32_t hdr[2];
  uint64_t count = 0;
  Answer a;
  in.read(magic, 8);
  in.read(reinterpret_cast<char*>(hdr), 8);
  in.read(reinterpret_cast<char*>(&count), 8);
  in.read(reinterpret_cast<char*>(&a.total), 8);
  if (!in || std::memcmp(magic, "MSTANS01", 8) != 0) throw UsageError(path + ": not an MST answer file");
  a.n = hdr[0];
  if (count > (uint64_t)a.n) throw UsageError(path + ": corrupt answer (count > n)");
  a.ids.resize(count);
  in.read(reinterpret_cast<char*>(a.ids.data()), (std::streamsize)(count * 4));
  if (!in) throw UsageError(path + ": truncated answer file");
  return a;
}

struct Result {
  std::vector<uint32_t> ids;
  uint64_t total = 0;
  uint32_t rounds = 0;
  double ms = 0;
};

// One trial. Device-resident buffers are set up once per graph.
struct Runner {
  const HostGraph& g;
  uint32_t *d_src = nullptr, *d_dst = nullptr, *d_w = nullptr, *d_out = nullptr;
  explicit Runner(const HostGraph& hg) : g(hg) {}
  ~Runner() {
    cudaFree(d_src);
    cudaFree(d_dst);
    cudaFree(d_w);
    cudaFree(d_out);
  }
  Result run(const std::string& algo, int gpus) {
    Result r;
    r.ids.resize(g.n > 1 ? g.n - 1 : 1);
    uint64_t count = 0;
    mst_stats_t st{};
    if (algo == "gpu") {
      const mst_edges_soa_t e{g.n, g.m, g.src.data(), g.dst.data(), g.w.data(), 0};
      check(mst_gpu_boruvka(&e, gpus, r.ids.data(), &count, &r.total, &st), "gpu");
      r.ms = st.ms_total;
    } else if (algo == "gpu-device") {
      if (gpus != 1) throw UsageError("gpu-device runs on one GPU");
      if (!d_src) {
        const size_t bytes = std::max<uint64_t>(g.m, 1) * 4;
        if (cudaMalloc(&d_src, bytes) || cudaMalloc(&d_dst, bytes) || cudaMalloc(&d_w, bytes) ||
            cudaMalloc(&d_out, (size_t)std::max<uint32_t>(g.n, 1) * 4))
          throw std::runtime_error("gpu-device: device allocation failed");
        cudaMemcpy(d_src, g.src.data(), g.m * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(d_dst, g.dst.data(), g.m * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(d_w, g.w.data(), g.m * 4, cudaMemcpyHostToDevice);
      }
      const mst_edges_soa_t e{g.n, g.m, d_src, d_dst, d_w, 1};
      check(mst_gpu_boruvka_device(&e, d_out, nullptr, &count, &r.total, &st, nullptr, nullptr), "gpu-device");
      cudaMemcpy(r.ids.data(), d_out, count * 4, cudaMemcpyDeviceToHost);
      r.ms = st.ms_device;
    } else {
      throw UsageError("unknown algorithm '" + algo + "'");
    }
    r.ids.resize(count);
    r.rounds = st.rounds;
    return r;
  }
};

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, ','))
    if (!x.empty()) out.push_back(x);
  return out;
}

int to_int(const std::string& s, const char* opt) {
  int v = 0;
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc{} || p != s.data() + s.size()) throw UsageError(std::string(opt) + ": not an integer: " + s);
  return v;
}

// --opt value / --flag parser over argv[first..]
struct Args {
  std::map<std::string, std::string> opt;
  std::vector<std::string> flags;
  Args(int argc, char** argv, int first, const std::vector<std::string>& with_value,
       const std::vector<std::string>& flag_names) {
    for (int i = first; i < argc; ++i) {
      const std::string a = argv[i];
      if (std::find(with_value.begin(), with_value.end(), a) != with_value.end()) {
        if (i + 1 >= argc) throw UsageError(a + " needs a value");
        opt[a] = argv[++i];
      } else if (std::find(flag_names.begin(), flag_names.end(), a) != flag_names.end()) {
        flags.push_back(a);
      } else {
        throw UsageError("unknown argument '" + a + "'");
      }
    }
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  bool flag(const std::string& k) const { return std::find(flags.begin(), flags.end(), k) != flags.end(); }
};

void usage(std::ostream& o) {
  o << "Boruvka MST on B200: workload generator, benchmark runner, summary\n"
       "  mstbench_gpu generate --config c0..c4 --out PATH [--binary]\n"
       "  mstbench_gpu run (--graph PATH | --config cN) --algo gpu[,gpu-device] [--gpus 1,2,..]\n"
       "                   [--reps 5] [--warmup 1] [--verify] [--oracle ANSWER] --csv OUT\n"
       "  mstbench_gpu summarize --csv PATH [--baseline REF.csv]\n"
       "  mstbench_gpu --list-presets\n";
}

int cmd_generate(const Args& a) {
  if (!a.has("--config") || !a.has("--out")) throw UsageError("generate: --config and --out are required");
  const Preset* p = find_preset(a.opt.at("--config"));
  if (!p) throw UsageError("unknown preset '" + a.opt.at("--config") + "'");
  HostGraph g = generate(*p);
  const std::string& out = a.opt.at("--out");
  if (a.flag("--binary"))
    check(mst_io_save_soa(out.c_str(), g.n, g.m, g.src.data(), g.dst.data(), g.w.data()), "generate");
  else
    check(mst_io_save_text(out.c_str(), g.n, g.m, g.src.data(), g.dst.data(), g.w.data()), "generate");
  std::cout << "wrote " << out << ": n=" << g.n << " m=" << g.m << " seed=" << p->spec.seed << "\n";
  return kExitOk;
}

int cmd_run(const Args& a) {
  if (!a.has("--csv")) throw UsageError("run: --csv is required");
  if (!a.has("--algo")) throw UsageError("run: --algo is required");
  if (a.has("--graph") == a.has("--config")) throw UsageError("run: one of --graph or --config is required");
  const std::vector<std::string> algos = split(a.opt.at("--algo"));
  for (const std::string& s : algos)
    if (s != "gpu" && s != "gpu-device") throw UsageError("unknown algorithm '" + s + "'");
  std::vector<int> gpus{1};
  if (a.has("--gpus")) {
    gpus.clear();
    for (const std::string& s : split(a.opt.at("--gpus"))) gpus.push_back(to_int(s, "--gpus"));
  }
  const int reps = a.has("--reps") ? to_int(a.opt.at("--reps"), "--reps") : 5;
  const int warmup = a.has("--warmup") ? to_int(a.opt.at("--warmup"), "--warmup") : 1;
  if (reps < 1) throw UsageError("--reps must be >= 1");
  const bool verify = a.flag("--verify");
  if (a.has("--oracle") && !verify) throw UsageError("--oracle needs --verify");

  HostGraph g;
  if (a.has("--config")) {
    const Preset* p = find_preset(a.opt.at("--config"));
    if (!p) throw UsageError("unknown preset '" + a.opt.at("--config") + "'");
    g = generate(*p);
  } else {
    g = load(a.opt.at("--graph"));
  }
  std::cout << "# devices: " << mst_gpu_device_count() << ", hardware threads: " << std::thread::hardware_concurrency()
            << ", library " << mst_gpu_version() << "\n";
  Runner runner(g);
  const mst_edges_soa_t host{g.n, g.m, g.src.data(), g.dst.data(), g.w.data(), 0};
  Answer oracle;
  const bool have_oracle = a.has("--oracle");
  if (have_oracle) {
    oracle = read_answer(a.opt.at("--oracle"));
    if (oracle.n != g.n)
      throw UsageError("oracle answer is for n=" + std::to_string(oracle.n) + ", the graph has n=" + std::to_string(g.n));
    std::cout << "# oracle: " << a.opt.at("--oracle") << " (" << oracle.ids.size() << " edges, weight " << oracle.total
              << ")\n";
  } else if (verify) {
    std::cout << "# verify: structural checks only (no --oracle answer file)\n";
  }
  std::vector<Row> rows;
  for (const std::string& algo : algos) {
    const std::vector<int> ts = algo == "gpu" ? gpus : std::vector<int>{1};
    for (int t : ts) {
      for (int w = 0; w < warmup; ++w) runner.run(algo, t);
      for (int trial = 1; trial <= reps; ++trial) {
        Result res = runner.run(algo, t);
        Row row;
        row.graph = g.name;
        row.algorithm = algo;
        row.threads = t;
        row.trial = trial;
        row.elapsed_ms = res.ms;
        row.weight = res.total;
        row.rounds = res.rounds;
        if (verify) {
          mst_verify_t v{};
          check(mst_gpu_verify(&host, res.ids.data(), res.ids.size(), have_oracle ? oracle.ids.data() : nullptr,
                               have_oracle ? oracle.ids.size() : 0, have_oracle ? oracle.total : MST_VERIFY_NO_ORACLE,
                               &v),
                "verify");
          const bool oracle_ok = !have_oracle || (v.weight_matches_oracle == 1 && v.edge_set_matches_oracle == 1);
          if (!(v.is_spanning && v.is_acyclic && v.edge_count_ok && oracle_ok))
            throw VerifyError(g.name + "/" + algo + " T=" + std::to_string(t) + " trial " + std::to_string(trial) +
                              ": edges=" + std::to_string(res.ids.size()) + " (expected " + std::to_string(g.n - 1) +
                              "), weight=" + std::to_string(v.weight) + ", components=" +
                              std::to_string(v.components) + ", acyclic=" + (v.is_acyclic ? "yes" : "no") +
                              ", edge_set=" +
                              (!have_oracle ? "unchecked" : v.edge_set_matches_oracle == 1 ? "match" : "MISMATCH") +
                              (have_oracle ? ", oracle weight=" + std::to_string(oracle.total) : std::string()));
          row.verified = true;
        }
        std::cout << row.graph << "," << row.algorithm << ",T=" << t << ",trial=" << trial << ": " << row.elapsed_ms
                  << " ms, weight=" << row.weight << ", rounds=" << row.rounds << "\n";
        rows.push_back(row);
      }
    }
  }
  for (const Row& r : rows)
    if (r.weight != rows.front().weight)
      throw VerifyError("mst_weight mismatch: " + rows.front().algorithm + " got " +
                        std::to_string(rows.front().weight) + " but " + r.algorithm + " T=" +
                        std::to_string(r.threads) + " got " + std::to_string(r.weight));
  write_csv(rows, a.opt.at("--csv"));
  std::cout << "# wrote " << rows.size() << " rows to " << a.opt.at("--csv") << "\n";
  return kExitOk;
}

double median_of(std::vector<double> v) {
  if (v.empty()) return std::numeric_limits<double>::quiet_NaN();
  std::sort(v.begin(), v.end());
  const size_t h = v.size() / 2;
  return v.size() % 2 ? v[h] : (v[h - 1] + v[h]) / 2.0;
}

std::string cell(double v) {
  if (std::isnan(v)) return "-";
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.3f", v);
  return buf;
}

int cmd_summarize(const Args& a) {
  if (!a.has("--csv")) throw UsageError("summarize: --csv is required");
  std::vector<Row> rows = read_csv(a.opt.at("--csv"));
  if (a.has("--baseline")) {
    const std::vector<Row> base = read_csv(a.opt.at("--baseline"));
    rows.insert(rows.end(), base.begin(), base.end());
  }
  std::map<std::tuple<std::string, std::string, int>, std::vector<double>> by;
  std::vector<std::string> graph_order;
  for (const Row& r : rows) {
    if (std::find(graph_order.begin(), graph_order.end(), r.graph) == graph_order.end()) graph_order.push_back(r.graph);
    by[{r.graph, r.algorithm, r.threads}].push_back(r.elapsed_ms);
  }
  std::printf("%-16s %-12s %7s %7s %12s\n", "graph", "algorithm", "threads", "trials", "median_ms");
  for (auto& [k, v] : by)
    std::printf("%-16s %-12s %7d %7zu %12.4f\n", std::get<0>(k).c_str(), std::get<1>(k).c_str(), std::get<2>(k),
                v.size(), median_of(v));
  // speedups against the reference's sequential and CAS rows
  // (summarize_speedups / print_speedup_table, bench.cpp:246-335)
  bool any = false;
  for (const std::string& gname : graph_order) {
    std::vector<double> seq, seq_opt;
    double cas_best = std::numeric_limits<double>::quiet_NaN();
    for (auto& [k, v] : by) {
      if (std::get<0>(k) != gname) continue;
      const std::string& algo = std::get<1>(k);
      if (algo == "seq") seq.insert(seq.end(), v.begin(), v.end());
      if (algo == "seq-opt") seq_opt.insert(seq_opt.end(), v.begin(), v.end());
      if (algo == "cas") {
        const double m = median_of(v);
        if (std::isnan(cas_best) || m < cas_best) cas_best = m;
      }
    }
    if (seq.empty() && seq_opt.empty() && std::isnan(cas_best)) continue;
    if (!any) {
      std::printf("\n%-16s %-12s %7s %12s %14s %14s\n", "graph", "algo", "threads", "vs_seq", "vs_seq_opt",
                  "vs_best_cas");
      any = true;
    }
    const double ms = median_of(seq), mo = median_of(seq_opt);
    for (auto& [k, v] : by) {
      if (std::get<0>(k) != gname) continue;
      const std::string& algo = std::get<1>(k);
      if (algo == "seq" || algo == "seq-opt") continue;
      const double med = median_of(v);
      std::printf("%-16s %-12s %7d %12s %14s %14s\n", gname.c_str(), algo.c_str(), std::get<2>(k),
                  cell(ms / med).c_str(), cell(mo / med).c_str(), cell(cas_best / med).c_str());
    }
  }
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) {
      usage(std::cerr);
      return kExitUsage;
    }
    const std::string sub = argv[1];
    if (sub == "--list-presets") {
      for (const Preset& p : presets()) std::cout << p.name << ": " << p.note << " seed=" << p.spec.seed << "\n";
      return kExitOk;
    }
    if (sub == "-h" || sub == "--help") {
      usage(std::cout);
      return kExitOk;
    }
    if (sub == "generate") return cmd_generate(Args(argc, argv, 2, {"--config", "--out"}, {"--binary"}));
    if (sub == "run")
      return cmd_run(Args(argc, argv, 2,
                          {"--graph", "--config", "--algo", "--gpus", "--reps", "--warmup", "--csv", "--oracle"},
                          {"--verify"}));
    if (sub == "summarize") return cmd_summarize(Args(argc, argv, 2, {"--csv", "--baseline"}, {}));
    throw UsageError("unknown subcommand '" + sub + "'");
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    usage(std::cerr);
    return kExitUsage;
  } catch (const GraphError& e) {
    std::cerr << "graph error: " << e.what() << "\n";
    return kExitGraph;
  } catch (const VerifyError& e) {
    std::cerr << "verification failed: " << e.what() << "\n";
    return kExitVerify;
  } catch (const std::exception& e) {
    std::cerr << "worker panic: " << e.what() << "\n";  // device failures, as WorkerPanic
    return kExitVerify;
  }
}
