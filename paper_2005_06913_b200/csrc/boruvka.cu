// Host engine + C ABI of the B200 parallel Boruvka MST.
//
// Replaces mst::boruvka_cas (reference: proj/src/boruvka_parallel.cpp:85-291)
// with a device round loop. See kernels.cuh for the per-round kernels and
// DESIGN.md for layouts, the byte model and the multi-GPU protocol.
#include <dlfcn.h>
#include <nccl.h>
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "verify.cuh"

namespace mstgpu {

thread_local std::string t_last_error;
void set_last_error(const std::string& m) { t_last_error = m; }

namespace {

using Clock = std::chrono::steady_clock;

// ------------------------------- NCCL (dlopen) ------------------------------
// Loaded lazily so the library has no hard NCCL dependency and reuses the
// libnccl.so.2 torch already mapped, if any.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
#define MST_NCCL_SYM(field, name)                                         \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));      \
  if (!api.field) {                                                       \
    api.why = std::string("NCCL symbol missing: ") + name;                \
    return;                                                               \
  }
    MST_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    MST_NCCL_SYM(CommInitRank, "ncclCommInitRank");
    MST_NCCL_SYM(CommInitAll, "ncclCommInitAll");
    MST_NCCL_SYM(AllReduce, "ncclAllReduce");
    MST_NCCL_SYM(GroupStart, "ncclGroupStart");
    MST_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    MST_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    MST_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef MST_NCCL_SYM
    api.ok = true;
  });
  if (!api.ok) throw MstError{MST_ERR_NCCL, api.why};
  return api;
}

#define MST_NCCL_CHECK(expr)                                                                \
  do {                                                                                      \
    ncclResult_t _r = (expr);                                                               \
    if (_r != ncclSuccess)                                                                  \
      throw MstError{MST_ERR_NCCL, std::string(#expr " failed: ") + nccl().GetErrorString(_r)}; \
  } while (0)

// ------------------------------- tuning -------------------------------------
// Every tuning knob of the engine, in ONE table with its measured default.
// The product path never reads the environment: a process changes a knob
// only through mst_gpu_set_tuning (the A/B tools under tools/ and the
// parity matrix of tests/ do; tools map their MST_* environment onto it).
// Values are read per use with relaxed atomics, so a knob set before a call
// holds for the whole call.
enum Knob {
  kKnobFilter,            // -1 auto (filter_mode: m >= 5n, or m >= 2.5n once m >= 24 M), 0 plain loop, 1 Filter-Boruvka
  kKnobFilterBeta,        // light edges ~ beta * n
  kKnobPivotSamples,      // sampled weights for the pivot
  kKnobFilterTableMB,     // read-first filter off for min tables above this size
  kKnobOfferMin1,         // offer modes per site (-1 default, 0/1/2, see filt_for)
  kKnobOfferSplit,
  kKnobOfferCount,
  kKnobOfferHeavy,
  kKnobPdl,               // programmatic dependent launch
  kKnobTail,              // tail megakernel
  kKnobTailEdges,         // tail entry edge bound (0: 12 M plain / 3 M light)
  kKnobTailComps,         // tail entry component bound
  kKnobTailSmallN,        // the tail also takes over below this many components
  kKnobTailBps,           // tail CTAs per SM (capped by residency)
  kKnobTailTiny,          // one-sync tiny rounds
  kKnobTailTrace,         // globaltimer stamps of the tail phases (stderr)
  kKnobTailStartC,        // round 1 handed to the tail at its phase C
  kKnobTailStartCD,       // phase D's first round handed to the tail at phase C
  kKnobTailStartCDEdges,
  kKnobTailDedup,         // tagged pair dedup inside the tail
  kKnobTailDedupRatio,
  kKnobTailDedupMin,
  kKnobDedup,             // pair dedup in the round kernels
  kKnobDedupMinEdges,
  kKnobDedupActive,
  kKnobDedupTableDiv,
  kKnobDedupRetry,
  kKnobDedupMinRatio,     // dedup a round only when m_r >= ratio * active components
  kKnobDedupCapLog2,      // pair table slots <= 2^this
  kKnobLazyRound1,
  kKnobPipelineH2D,       // chunked host copy overlapping round 1's min pass
  kKnobPipelineChunks,
  kKnobDebugRounds,       // per-round counters on stderr
  kKnobL2Fetch,           // cudaLimitMaxL2FetchGranularity in bytes (0: leave the device default)
  kKnobOfferCached,       // offer filter reads through L1 (bit kFiltCached) at these sites (bitmask of OfferSite)
  kKnobRetire,            // light phase: retire isolated components (tables sized by components with edges)
  kKnobGiantBits,         // relabel rounds with more components than this: giant bits (0 off)
  kKnobRangeOffers,       // split / heavy filter offers in range passes over L2-sized table slices
  kKnobRangeMB,           // ... slice size
  kKnobBytesMax,          // MST output as bytes up to this many edges, a bitmap above
  kKnobTimeline,          // tools only: an event after every launch, per-launch stream times on stderr
  kKnobEmitSparse,        // warp-per-32-tiles copy for the split's / heavy filter's staged survivors
  kKnobInterleave,        // count passes walk the list in this many interleaved segments (<= 1 off)
  kKnobDedupGuarantee,    // dedup a round only when the next round's components can form <= m_r / this pairs (0: off)
  kKnobCount
};
struct KnobDef {
  const char* name;
  double dflt;
};
constexpr KnobDef kKnobDefs[kKnobCount] = {
    {"MST_FILTER", -1},          {"MST_FILTER_BETA", 1.25},       {"MST_PIVOT_SAMPLES", 262144},
    {"MST_FILTER_TABLE_MB", 1e7}, {"MST_OFFER_MIN1", -1},         {"MST_OFFER_SPLIT", -1},
    {"MST_OFFER_COUNT", -1},     {"MST_OFFER_HEAVY", -1},        {"MST_PDL", 1},
    {"MST_TAIL", 1},             {"MST_TAIL_EDGES", 0},          {"MST_TAIL_COMPS", 8e6},
    {"MST_TAIL_SMALL_N", 65536}, {"MST_TAIL_BPS", MST_TAIL_MINB}, {"MST_TAIL_TINY", 1},
    {"MST_TAIL_TRACE", 0},       {"MST_TAIL_START_C", 1},        {"MST_TAIL_START_C_D", 1},
    {"MST_TAIL_START_C_D_EDGES", 3.2e7}, {"MST_TAIL_DEDUP", 0},   {"MST_TAIL_DEDUP_RATIO", 4},
    {"MST_TAIL_DEDUP_MIN", 16384}, {"MST_DEDUP", 1},             {"MST_DEDUP_MIN_EDGES", 2e6},
    {"MST_DEDUP_ACTIVE", 262144}, {"MST_DEDUP_TABLE_DIV", 4},    {"MST_DEDUP_RETRY", 0},
    {"MST_DEDUP_MIN_RATIO", 8},  {"MST_DEDUP_CAP_LOG2", 25},
    {"MST_LAZY_ROUND1", 1},      {"MST_PIPELINE_H2D", 0},        {"MST_PIPELINE_CHUNKS", 16},
    {"MST_DEBUG_ROUNDS", 0},     {"MST_L2_FETCH", 0},         {"MST_OFFER_CACHED", 15},
    {"MST_RETIRE", 1},           {"MST_GIANT_BITS", 16e6},   {"MST_RANGE_OFFERS", 1},
    {"MST_RANGE_MB", 128},       {"MST_BYTES_MAX", 67108864},    {"MST_TIMELINE", 0},
    {"MST_EMIT_SPARSE", 1},      {"MST_INTERLEAVE", 128},
    {"MST_DEDUP_GUARANTEE", 4}};

std::atomic<double>* knob_table() {
  static std::atomic<double> t[kKnobCount];
  static std::once_flag once;
  std::call_once(once, [] {
    for (int k = 0; k < kKnobCount; ++k) t[k].store(kKnobDefs[k].dflt, std::memory_order_relaxed);
  });
  return t;
}
double knob(Knob k) { return knob_table()[k].load(std::memory_order_relaxed); }
int knob_i(Knob k) { return (int)knob(k); }

// ------------------------------- workspace ----------------------------------
// One per (device, slot): named grow-only device buffers, a stream, pinned
// counter snapshots and the look-back epoch. Reused across calls like a
// library handle; guarded by its mutex (one call at a time per workspace).
struct Workspace {
  int device = 0;
  std::mutex mu;
  cudaStream_t stream = nullptr;
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs;
  unsigned long long* status = nullptr;
  size_t status_words = 0;
  uint32_t epoch = 1;
  // tail pair-dedup table: slots tagged (call epoch, round); cleared only
  // when it grows or the 10-bit epoch wraps
  uint32_t pair_epoch = 0;
  size_t pair_slots = 0;
  DevCounters* h_snap = nullptr;  // pinned, kMaxR + 1 snapshots
  unsigned int* h_u32 = nullptr;  // pinned, 16 words (single counters read mid-run)
  // pinned staging for pageable host buffers (two chunks, ping-pong)
  static constexpr size_t kStageBytes = 32u << 20;
  void* hstage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  bool stage_busy[2] = {false, false};
  cudaStream_t copy_stream = nullptr;  // pipelined host -> device copies
  cudaEvent_t chunk_ev[16] = {};
  std::vector<cudaEvent_t> ev;    // per-round events
  std::vector<cudaEvent_t> tev;   // timing events (hot kernels)
  cudaEvent_t join_in = nullptr, join_out = nullptr;  // ordering with the caller's legacy stream 0

  void init(int dev) {
    device = dev;
    MST_CUDA_CHECK(cudaSetDevice(dev));
    MST_CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    MST_CUDA_CHECK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    for (auto& e : chunk_ev) MST_CUDA_CHECK(cudaEventCreate(&e));
    MST_CUDA_CHECK(cudaMallocHost(&h_snap, sizeof(DevCounters) * (kMaxR + 1)));
    MST_CUDA_CHECK(cudaMallocHost(&h_u32, 16 * sizeof(unsigned int)));
    ev.resize(kMaxR + 1);
    for (auto& e : ev) MST_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    tev.resize(4 * kMaxR + 8);
    for (auto& e : tev) MST_CUDA_CHECK(cudaEventCreate(&e));
    for (auto& e : stage_ev) MST_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MST_CUDA_CHECK(cudaEventCreateWithFlags(&join_in, cudaEventDisableTiming));
    MST_CUDA_CHECK(cudaEventCreateWithFlags(&join_out, cudaEventDisableTiming));
  }

  void* staging(int b) {
    if (!hstage[b]) MST_CUDA_CHECK(cudaMallocHost(&hstage[b], kStageBytes));
    return hstage[b];
  }

  void release() {
    cudaSetDevice(device);
    cudaStreamSynchronize(stream);
    for (auto& kv : bufs) cudaFree(kv.second.p);
    bufs.clear();
    pair_slots = 0;
    if (status) cudaFree(status);
    status = nullptr;
    status_words = 0;
  }

  template <class T>
  T* get(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    Buf& b = bufs[name];
    if (b.bytes < bytes) {
      if (b.p) {
        MST_CUDA_CHECK(cudaStreamSynchronize(stream));
        MST_CUDA_CHECK(cudaFree(b.p));
        b.p = nullptr;
        b.bytes = 0;
      }
      MST_CUDA_CHECK(cudaMalloc(&b.p, bytes));
      b.bytes = bytes;
    }
    return static_cast<T*>(b.p);
  }

  unsigned long long* status_array(size_t tiles) {
    if (status_words < tiles + 1) {
      MST_CUDA_CHECK(cudaStreamSynchronize(stream));
      if (status) MST_CUDA_CHECK(cudaFree(status));
      status_words = tiles + 1;
      MST_CUDA_CHECK(cudaMalloc(&status, status_words * sizeof(unsigned long long)));
      MST_CUDA_CHECK(cudaMemsetAsync(status, 0, status_words * sizeof(unsigned long long), stream));
      epoch = 1;
    }
    return status;
  }

  uint32_t next_epoch() {
    if (epoch >= (1u << 30) - 1) {
      MST_CUDA_CHECK(cudaMemsetAsync(status, 0, status_words * sizeof(unsigned long long), stream));
      epoch = 1;
    }
    return epoch++;
  }
};

std::mutex g_ws_mu;
std::map<std::pair<int, int>, std::unique_ptr<Workspace>> g_ws;

Workspace& workspace(int device, int slot = 0) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  auto& p = g_ws[{device, slot}];
  if (!p) {
    p = std::make_unique<Workspace>();
    p->init(device);
  }
  return *p;
}

// ------------------------------- host <-> device ----------------------------
// Pinned host memory is copied directly. Pageable memory goes through two
// pinned 32 MB chunks: host threads (OpenMP) fill one chunk while the copy
// engine moves the other. Measured on the B200 host (tools/xfer_bench.cu):
// 100 MB H2D pageable 9.5 ms vs pinned 2.4 ms; 16 MB D2H 1.1 vs 0.3 ms.
bool host_is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const int T = bytes >= (4u << 20) ? std::max(1, std::min(omp_get_max_threads(), 16)) : 1;
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; ++t) {
    const size_t lo = bytes * t / T, hi = bytes * (t + 1) / T;
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  }
}

void copy_h2d(Workspace& ws, void* d, const void* h, size_t bytes) {
  if (!bytes) return;
  if (bytes < (2u << 20) || host_is_pinned(h)) {
    MST_CUDA_CHECK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ws.stream));
    return;
  }
  for (size_t off = 0, k = 0; off < bytes; off += Workspace::kStageBytes, ++k) {
    const int b = (int)(k & 1);
    const size_t len = std::min(Workspace::kStageBytes, bytes - off);
    if (ws.stage_busy[b]) MST_CUDA_CHECK(cudaEventSynchronize(ws.stage_ev[b]));
    par_memcpy(ws.staging(b), static_cast<const char*>(h) + off, len);
    MST_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(d) + off, ws.staging(b), len, cudaMemcpyHostToDevice,
                                   ws.stream));
    MST_CUDA_CHECK(cudaEventRecord(ws.stage_ev[b], ws.stream));
    ws.stage_busy[b] = true;
  }
}

// Synchronous with respect to the host (the data is needed on return).
void copy_d2h(Workspace& ws, void* h, const void* d, size_t bytes) {
  if (!bytes) return;
  if (bytes < (2u << 20) || host_is_pinned(h)) {
    MST_CUDA_CHECK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ws.stream));
    return;
  }
  const size_t chunk = Workspace::kStageBytes;
  const size_t nchunks = (bytes + chunk - 1) / chunk;
  auto issue = [&](size_t k) {
    const int b = (int)(k & 1);
    const size_t off = k * chunk, len = std::min(chunk, bytes - off);
    if (ws.stage_busy[b]) MST_CUDA_CHECK(cudaEventSynchronize(ws.stage_ev[b]));
    MST_CUDA_CHECK(cudaMemcpyAsync(ws.staging(b), static_cast<const char*>(d) + off, len, cudaMemcpyDeviceToHost,
                                   ws.stream));
    MST_CUDA_CHECK(cudaEventRecord(ws.stage_ev[b], ws.stream));
    ws.stage_busy[b] = true;
  };
  issue(0);
  for (size_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    const size_t off = k * chunk, len = std::min(chunk, bytes - off);
    MST_CUDA_CHECK(cudaEventSynchronize(ws.stage_ev[b]));
    ws.stage_busy[b] = false;
    if (k + 1 < nchunks) issue(k + 1);  // the engine fills the other chunk meanwhile
    par_memcpy(static_cast<char*>(h) + off, ws.staging(b), len);
  }
}

// ------------------------------- launch helpers -----------------------------

int sm_count(int device) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int sms = 0;
  MST_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cache[device] = sms;
  return sms;
}

template <class K>
int blocks_per_sm(K kernel, size_t dyn_smem = 0) {
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const std::pair<const void*, size_t> key{reinterpret_cast<const void*>(kernel), dyn_smem};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int nb = 0;
  MST_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kBlock, dyn_smem));
  cache[key] = std::max(nb, 1);
  return cache[key];
}

// Persistent grid: min(resident capacity, work tiles), at least 1.
template <class K>
unsigned persistent_grid(K kernel, int device, uint64_t tiles) {
  const uint64_t cap = (uint64_t)sm_count(device) * blocks_per_sm(kernel);
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cap, tiles));
}

uint64_t tiles_of(uint64_t count) { return (count + kTile - 1) / kTile; }
uint64_t tiles_c(uint64_t count) { return (count + kCTile - 1) / kCTile; }
unsigned long long next_pow2(unsigned long long x) {
  unsigned long long p = 1024;
  while (p < x) p <<= 1;
  return p;
}

// Read-before-atomic: always on by default. Even for DRAM-sized tables it
// wins, because hub / giant-component entries are hot — unfiltered REDs to
// one address serialise at its L2 slice (c4: 172 -> 53 ms with the filter).
// The MST_FILTER_TABLE_MB knob turns it off for tables above that size.
// Offer mode per call site (kernels.cuh offer_both): 0 plain REDs, 1
// read-first one offer at a time, 2 read-first with a thread's reads batched
// (more memory-level parallelism; but a batch's reads all miss its own
// atomics, which costs on hub-heavy tables). MST_OFFER_<SITE>=0|1|2
// overrides. Defaults from tools/sweep_offer.sh and tools/ab2.sh (one
// B200, c0-c4): batched for round 1 and for the round compactions of the
// plain loop (sparse graphs: c1 -11 % with both); one at a time for the
// light split, the heavy filter and the compactions of Filter-Boruvka's
// phases, whose survivors concentrate on hubs (batched: c2 +3 %, c3 +1.5 %,
// c4 +1.7 %).
enum OfferSite { kSiteMin1 = 0, kSiteSplit = 1, kSiteCount = 2, kSiteHeavy = 3, kSiteCount_ = 4 };
int filt_mode(uint64_t table_entries, int site, bool dense) {
  const double limit_mb = knob(kKnobFilterTableMB);
  const int mode[kSiteCount_] = {knob_i(kKnobOfferMin1), knob_i(kKnobOfferSplit), knob_i(kKnobOfferCount),
                                 knob_i(kKnobOfferHeavy)};
  if ((double)table_entries * 8.0 > limit_mb * 1048576.0) return 0;
  if (mode[site] >= 0) return mode[site];
  switch (site) {
    case kSiteMin1:
      return 2;
    case kSiteCount:
      return dense ? 1 : 2;
    default:
      return 1;
  }
}
int filt_for(uint64_t table_entries, int site = kSiteCount, bool dense = true) {
  const int f = filt_mode(table_entries, site, dense);
  return (f != 0 && ((knob_i(kKnobOfferCached) >> site) & 1)) ? (f | kFiltCached) : f;
}

double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  MST_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

// ------------------------------- run state ----------------------------------

struct RunOut {
  uint64_t count = 0;
  uint64_t total_weight = 0;
  uint32_t rounds = 0;
  uint32_t final_components = 0;
  uint32_t err = 0;
  uint32_t launches = 0;
  double ms_hot = 0;
  uint32_t hot_launches = 0;
  uint64_t hot_bytes = 0;
  uint32_t phase_end = 0;  // Filter-Boruvka: the first round past the light phase (0: the plain loop)
  DevCounters ctr{};
};

void init_counters(Workspace& ws, DevCounters* d_ctr, uint32_t n, uint64_t m) {
  DevCounters& h = ws.h_snap[kMaxR];
  std::memset(&h, 0, sizeof(h));
  h.n[1] = n;
  h.m[0] = m;
  h.m[1] = m;
  h.stop_round = kNoStop;
  h.phase_end = kNoStop;
  h.pivot = 0xFFFFFFFFu;
  MST_CUDA_CHECK(cudaMemcpyAsync(d_ctr, &h, sizeof(DevCounters), cudaMemcpyHostToDevice, ws.stream));
}


// Kernel launch with programmatic dependent launch (kernels.cuh pdl_prologue):
// the next kernel's launch overlaps this one's tail. The MST_PDL knob = 0 disables it.
bool pdl_enabled() { return knob_i(kKnobPdl) != 0; }

// MST_TIMELINE (tools only): an event after every launch on the calling
// thread, printed as stream-time offsets by run_single once the call is done.
struct TimelineMark {
  const void* fn;
  cudaEvent_t ev;
};
thread_local std::vector<TimelineMark> t_timeline;
thread_local std::vector<cudaEvent_t> t_timeline_pool;
void timeline_mark(const void* fn, cudaStream_t s) {
  if (!knob_i(kKnobTimeline)) return;
  const size_t i = t_timeline.size();
  if (i >= t_timeline_pool.size()) {
    cudaEvent_t e;
    MST_CUDA_CHECK(cudaEventCreate(&e));
    t_timeline_pool.push_back(e);
  }
  MST_CUDA_CHECK(cudaEventRecord(t_timeline_pool[i], s));
  t_timeline.push_back(TimelineMark{fn, t_timeline_pool[i]});
}
void timeline_print(cudaEvent_t start) {
  if (t_timeline.empty()) return;
  float prev = 0;
  for (const TimelineMark& m : t_timeline) {
    float ms = 0;
    cudaEventElapsedTime(&ms, start, m.ev);
    const char* name = "(mark)";
    if (m.fn) cudaFuncGetName(&name, m.fn);
    fprintf(stderr, "timeline %9.1f us  +%8.1f  %s\n", ms * 1e3, (ms - prev) * 1e3, name);
    prev = ms;
  }
  t_timeline.clear();
}

// Kernels launched by the calling thread (GpuRunInfo::kernel_launches is
// the difference over a call).
thread_local uint64_t t_launches = 0;

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
  ++t_launches;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  MST_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
  timeline_mark(reinterpret_cast<const void*>(kernel), s);
}

// Sorted id list (ascending) from the MST bitmap the hook kernels set.
// words = (m + 31) / 32; the bitmap buffer is allocated with mst_bits_words(m).
uint64_t mst_bits_words(uint64_t m) { return ((m + 31) / 32 + 3) & ~3ull; }  // whole uint4 vectors
// The single-GPU output's words: one byte per edge up to MST_BYTES_MAX edges
// (kernels.cuh mst_mark), else the bitmap.
bool mst_out_bytes(uint64_t m) { return (double)m <= knob(kKnobBytesMax); }
uint64_t mst_out_words(uint64_t m) { return mst_out_bytes(m) ? ((m + 16 + 15) / 16) * 4 : mst_bits_words(m); }

// Sorted id list from one flag byte per edge (small lists, see mst_mark).
uint32_t sort_from_bytes(Workspace& ws, const uint8_t* flags, uint64_t m, uint32_t* d_sorted, DevCounters* d_ctr) {
  const uint64_t tiles = (m + kFlagTile - 1) / kFlagTile;
  uint32_t* counts = ws.get<uint32_t>("sort_counts", std::max<uint64_t>(tiles, 1));
  const int fused = tiles <= kFusedScanMaxTiles ? 1 : 0;
  // done[0][kSlotSort] is zero: cleared at the run's start, re-armed by every fused scan
  const unsigned g = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(tiles, (uint64_t)sm_count(ws.device) * blocks_per_sm(k_flags_count)));
  launch_k(k_flags_count, g, kBlock, ws.stream, flags, m, counts, d_ctr, fused);
  uint32_t launches = 2;
  if (!fused) {
    unsigned long long* st = ws.status_array(tiles);
    launch_k(k_scan_counts<kScanPlain>,
             (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((tiles + kScanTile - 1) / kScanTile, (uint64_t)sm_count(ws.device))),
             kScanBlock, ws.stream, counts, tiles, d_ctr, 0, st, ws.next_epoch(), 0, 0);
    ++launches;
  }
  const unsigned ge = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(tiles, (uint64_t)sm_count(ws.device) * blocks_per_sm(k_flags_emit)));
  launch_k(k_flags_emit, ge, kBlock, ws.stream, flags, m, counts, d_sorted);
  MST_CUDA_CHECK(cudaGetLastError());
  return launches;
}
uint32_t sort_from_bits(Workspace& ws, const uint32_t* bits, uint64_t m, uint32_t* d_sorted, DevCounters* d_ctr) {
  const uint64_t words = (m + 31) / 32;
  const uint64_t tiles = tiles_of(words);
  uint32_t* counts = ws.get<uint32_t>("sort_counts", std::max<uint64_t>(tiles, 1));
  const int fused = tiles <= kFusedScanMaxTiles ? 1 : 0;
  // done[0][kSlotSort] is zero: cleared at the run's start, re-armed by every fused scan
  const unsigned g = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(tiles, (uint64_t)sm_count(ws.device) * blocks_per_sm(k_bitmap_count)));
  launch_k(k_bitmap_count, g, kBlock, ws.stream, bits, words, counts, d_ctr, fused);
  uint32_t launches = 2;
  if (!fused) {
    unsigned long long* st = ws.status_array(tiles);
    launch_k(k_scan_counts<kScanPlain>,
             (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((tiles + kScanTile - 1) / kScanTile, (uint64_t)sm_count(ws.device))),
             kScanBlock, ws.stream, counts, tiles, d_ctr, 0, st, ws.next_epoch(), 0, 0);
    ++launches;
  }
  // the emit's own residency (32 KB of staging per block)
  const unsigned ge = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(tiles, (uint64_t)sm_count(ws.device) * blocks_per_sm(k_bitmap_emit)));
  launch_k(k_bitmap_emit, ge, kBlock, ws.stream, bits, words, counts, d_sorted);
  MST_CUDA_CHECK(cudaGetLastError());
  return launches;
}

// ------------------------------- single GPU ---------------------------------
// Literal keys (w<<32 | index into this round's edge array): the hook reads
// the winning edge directly. The host runs one round ahead of the device;
// kernels of rounds past a stop early-exit on the device counters.
//
// Filter-Boruvka (default for dense or large lists, filter_mode): a sampled weight pivot splits the
// edges; the round loop first runs on the light edges alone (phase B), then
// one pass drops every heavy edge inside a light component (cycle property,
// exact) and the loop continues on the survivors (phase D). Uniform and
// R-MAT graphs keep most edges alive for many rounds otherwise
// (sum m_r = 4.5-8.3 m).

enum { kHotMin1 = 0, kHotCompact = 1, kHotSplit = 2, kHotHeavy = 3, kHotTail = 4 };
struct HotLaunch {
  int ev;
  int kind;
  int r;
  bool light;
};

bool filter_mode(uint32_t n, uint64_t m) {
  const int f = knob_i(kKnobFilter);
  if (f >= 0) return f > 0 && m > 0;
  // m >= 5n: measured crossover (tools/filter_rule.py, one B200): uniform
  // m/n = 4 plain 0.65 vs filter 0.97 ms (c0), m/n = 6 0.92 vs 1.01, m/n = 8
  // 4.25 vs 1.05; R-MAT m/n = 5 1.41 vs 1.23. (The light phase of a sparse
  // graph stalls on the parallel light edges of a few active components.)
  // Large lists gain from the filter at lower densities too (round 2,
  // tools/knob_ab_sizes.py --plain, profiles/r2s4/filter_rule_sparse.log):
  // from m >= 2.5 n once m >= 24 M (uniform n = 16 M, m = 64 M: 12.3 -> 5.6
  // ms; R-MAT 24 ef 2: 6.0 -> 4.4; a 256^3 grid: 3.1 -> 2.8; an 8-neighbour
  // 4096^2 grid: 3.06 -> 2.83), while 4-neighbour grids (m = 2 n: +46-83 %
  // with the filter) and lists under ~17 M edges (8-neighbour 2048^2 grid,
  // 128^3 grid: +40 %; c0: +11 %) stay on the plain loop.
  if (m >= (uint64_t)5 * n) return m >= (1u << 16);
  return 2 * m >= (uint64_t)5 * n && m >= (24ull << 20);
}


struct CompactBufs {
  uint32_t* counts;
  uint32_t* masks;
  unsigned long long* st;
  uint4* stage;  // survivors of the sparse modes, compacted per tile
};

// Ordered compaction as count + emit (kernels.cuh, "two-pass ordered compaction").
// min_next receives the offers for round r+1: keyed by the position in the
// input list for every mode but the heavy filter (see k_count).
template <class View, int kMode>
void launch_two_pass(Workspace& ws, const CompactBufs& cb, View in, uint4* relabeled, const uint32_t* L, uint4* out,
                     unsigned long long* min_next, DevCounters* d_ctr, int r, uint64_t m_bound, uint32_t n_orig,
                     int slot, int light, int filt, PairTable pt = PairTable{nullptr, 0},
                     bool emit = true, const uint32_t* gbits = nullptr, uint64_t range_table = 0) {
  const int dev = ws.device;
  const uint64_t tiles = tiles_c(m_bound);
  const int fused = tiles <= kFusedScanMaxTiles ? 1 : 0;  // small: the last count block scans
  const bool armed = kMode == kModeRelabel && !View::kOriginal && pt.pairs != nullptr;
  auto kcnt = (filt & 3) == 2 ? k_count<View, kMode, true> : k_count<View, kMode, false>;
  const unsigned gc = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(tiles, (uint64_t)sm_count(dev) * blocks_per_sm(kcnt)));
  // armed: this launch relabels + inserts pairs if the device chose dedup
  // (decided and table cleared by k_label2), the kModeDedup pass counts
  launch_k(kcnt, gc, kBlock, ws.stream, in, kMode == kModeRelabel ? relabeled : cb.stage, L, cb.masks, cb.counts, n_orig,
           d_ctr, r, fused, slot, light, pt, min_next, filt, gbits, (uint32_t)std::max(0, knob_i(kKnobInterleave)));
  if constexpr (!View::kOriginal) {
    if (armed) {
      auto kdc = k_count<PackedView, kModeDedup>;
      launch_k(kdc, gc, kBlock, ws.stream, PackedView{relabeled}, cb.stage, L, cb.masks, cb.counts, n_orig, d_ctr, r,
               fused, slot, light, pt, min_next, filt, (const uint32_t*)nullptr,
               (uint32_t)std::max(0, knob_i(kKnobInterleave)));
    }
  }
  if (!fused) {
    auto ksc = k_scan_counts<kScanEdges>;
    const unsigned gs = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((tiles + kScanTile - 1) / kScanTile,
                                                                            (uint64_t)sm_count(dev)));
    launch_k(ksc, gs, kScanBlock, ws.stream, cb.counts, tiles, d_ctr, r, cb.st, ws.next_epoch(), light,
             View::kOriginal ? 1 : 0);
  }
  if (!emit) {  // count + scan only (round 1 of the lazy plain loop)
    MST_CUDA_CHECK(cudaGetLastError());
    return;
  }
  const unsigned ge = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)sm_count(dev) * 8));
  if (armed) {
    auto kde = k_emit_staged<kModeDedup>;
    launch_k(kde, ge, kBlock, ws.stream, cb.stage, cb.counts, out, min_next, d_ctr, r, filt);
  }
  if (kMode == kModeRelabel) {
    auto kem = k_emit<View, kMode>;
    launch_k(kem, ge, kBlock, ws.stream, in, relabeled, L, cb.masks, cb.counts, out, d_ctr, r, armed ? 1 : 0, n_orig);
  } else {
    auto kes = (filt & 3) == 2 ? k_emit_staged<kMode, true> : k_emit_staged<kMode, false>;
    // range passes (kernels.cuh k_range_offers) for a table of range_table
    // entries larger than the slice: the emit only copies
    const uint64_t slice = (uint64_t)(knob(kKnobRangeMB) * 1048576.0 / 8.0);
    const bool ranged = (kMode == kModeHeavy || kMode == kModeLight) && knob_i(kKnobRangeOffers) && slice > 0 &&
                        range_table > slice;
    if (ranged && knob_i(kKnobEmitSparse)) {
      const uint64_t groups = (tiles + 31) / 32;
      const unsigned gw = (unsigned)std::max<uint64_t>(
          1, std::min<uint64_t>((groups + kWarps - 1) / kWarps, (uint64_t)sm_count(dev) * blocks_per_sm(k_emit_sparse)));
      launch_k(k_emit_sparse, gw, kBlock, ws.stream, (const uint4*)cb.stage, (const uint32_t*)cb.counts, out, d_ctr, r);
    } else {
      launch_k(kes, ge, kBlock, ws.stream, cb.stage, cb.counts, out, ranged ? nullptr : min_next, d_ctr, r, filt);
    }
    if (ranged) {
      const unsigned gr = (unsigned)(sm_count(dev) * blocks_per_sm(k_range_offers));
      for (uint64_t lo = 0; lo < range_table; lo += slice)
        launch_k(k_range_offers, gr, kBlock, ws.stream, (const uint4*)out, (const DevCounters*)d_ctr, r, min_next,
                 (uint32_t)lo, (uint32_t)std::min<uint64_t>(range_table, lo + slice), filt);
    }
  }
  MST_CUDA_CHECK(cudaGetLastError());
}

enum { kSrcIn = 0, kSrcPairs = 1, kSrcPacked = 2 };
struct HookSrc {
  int kind;
  const uint4* packed;  // kSrcPacked: the list; kSrcPairs: the uint2 pair list
};

// Pipelined host copy of the caller's list: chunk j = edges [bound[j],
// bound[j+1]) is on the device once ev[j] has completed.
struct CopyChunks {
  static constexpr int kMax = 16;
  int count = 0;
  uint64_t bound[kMax + 1];
  cudaEvent_t ev[kMax];
};

// ---- retirement bookkeeping (kernels.cuh "retirement"), shared by the
// single-device and the sharded loops: one bitmap region per retiring light
// round (sized by the host's bound on n_r), the last region kept for the
// final one; at the light phase's end the regions are ranked and the level
// maps composed top-down into final labels.
struct RetireState {
  static constexpr uint64_t kRegions = 5;
  uint32_t* bits = nullptr;
  uint64_t region = 0;  // words of one region (bound)
  uint64_t used = 0;
  std::vector<std::pair<int, uint64_t>> woff;  // (round, first word) of each retiring round

  void init(Workspace& ws, uint32_t n, bool on) {
    woff.clear();
    used = 0;
    region = ((uint64_t)n + 31) / 32 + 1;
    bits = on ? ws.get<uint32_t>("ret_bits", kRegions * region) : nullptr;
  }
  bool active() const { return !woff.empty(); }
  // round r's region (cleared), or nullptr when retirement is off or full
  uint32_t* take(cudaStream_t s, int r, uint64_t n_bound) {
    const uint64_t need = (n_bound + 31) / 32;
    if (!bits || used + need + region > kRegions * region) return nullptr;
    uint32_t* rb = bits + used;
    MST_CUDA_CHECK(cudaMemsetAsync(rb, 0, need * 4, s));
    woff.push_back({r, used});
    used += need;
    return rb;
  }
  void drop_from(int P) {
    while (!woff.empty() && woff.back().first >= P) woff.pop_back();
  }
  // Final labels of the light phase ending at round P: every level map of
  // `levels` (buffer, round; level 1 first) becomes vertex/component -> final
  // label, n[P] the number of final components, and `heavy_min` (the heavy
  // filter's table) is cleared for them. Returns the launches.
  uint32_t finalize(Workspace& ws, cudaStream_t s, DevCounters* d_ctr, int P,
                    const std::vector<std::pair<uint32_t*, int>>& levels, const DevCounters& snap,
                    unsigned long long* heavy_min) {
    const int dev = ws.device;
    const uint64_t woff_final = used;  // after every region handed out (dropped rounds' are zero)
    MST_CUDA_CHECK(cudaMemsetAsync(bits + woff_final, 0, region * 4, s));
    launch_k(k_ret_fill_final, (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(region / 256 + 1, 4096)), 256, s,
             bits + woff_final, (const DevCounters*)d_ctr, P);
    const uint64_t W = woff_final + region;
    uint32_t* prefix = ws.get<uint32_t>("ret_prefix", W);
    launch_k(k_ret_popc, (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(W / 256 + 1, (uint64_t)sm_count(dev) * 8)),
             256, s, (const uint32_t*)bits, W, prefix);
    unsigned long long* st = ws.status_array((W + kScanTile - 1) / kScanTile + 1);
    launch_k(k_scan_counts<kScanDense>,
             (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((W + kScanTile - 1) / kScanTile, (uint64_t)sm_count(dev))),
             kScanBlock, s, prefix, W, d_ctr, P, st, ws.next_epoch(), 0, 0);
    for (int k = (int)levels.size() - 1; k >= 0; --k) {
      uint64_t wo = 0;
      for (const auto& rw : woff)
        if (rw.first == levels[k].second) wo = rw.second;
      const uint32_t* Lnext = k + 1 < (int)levels.size() ? levels[k + 1].first : nullptr;
      const unsigned g = (unsigned)std::max<uint64_t>(
          1, std::min<uint64_t>((snap.n[levels[k].second] + 1023) / 1024, (uint64_t)sm_count(dev) * 8));
      launch_k(k_compose_ret, g, 256, s, levels[k].first, Lnext, (const uint32_t*)bits, (const uint32_t*)prefix, wo,
               woff_final, (const DevCounters*)d_ctr, levels[k].second);
    }
    launch_k(k_fill_keys, (unsigned)(sm_count(dev) * 8), 256, s, heavy_min, (const DevCounters*)d_ctr, P);
    return 5 + (uint32_t)levels.size();
  }
};

// n[P] on the host (one sync): the component count after a retiring light
// phase exists on the device only.
uint32_t read_count(Workspace& ws, cudaStream_t s, const DevCounters* d_ctr, int P) {
  MST_CUDA_CHECK(cudaMemcpyAsync(ws.h_u32, &d_ctr->n[P], sizeof(unsigned int), cudaMemcpyDeviceToHost, s));
  MST_CUDA_CHECK(cudaStreamSynchronize(s));
  return ws.h_u32[0];
}

// `enqueue_after` (optional) is enqueued on the stream right behind the last
// round, before the one host sync that reads the verdict: the sorted output
// and its copy-back need no host decision, so they follow the MST without a
// host round trip (the verdict is checked after the sync; an error discards
// them).
template <class InView>
void run_single_impl(Workspace& ws, InView in, const uint32_t* wbase, uint32_t wstride, uint32_t n,
                     uint64_t m, RunOut& out, bool time_hot, bool filter, const CopyChunks* chunks = nullptr,
                     const std::function<void()>* enqueue_after = nullptr) {
  cudaStream_t s = ws.stream;
  auto* d_ctr = ws.get<DevCounters>("ctr", 1);
  unsigned long long* minb[2] = {ws.get<unsigned long long>("minA", n),
                                 ws.get<unsigned long long>("minB", n)};
  uint32_t* parent = ws.get<uint32_t>("parent", n);
  uint32_t* L = ws.get<uint32_t>("label", n);
  // the sorted output comes from the per-edge flags (the sharded loop too:
  // every rank sets the flags of every hooked component), no MST slot array
  uint4* E[2] = {ws.get<uint4>("E0", m), ws.get<uint4>("E1", m)};
  unsigned long long* st = ws.status_array(std::max(tiles_of(m), tiles_of(n)));
  const int dev = ws.device;
  const CompactBufs cb{ws.get<uint32_t>("tile_counts", tiles_c(m)),
                       ws.get<uint32_t>("tile_masks", tiles_c(m) * kCItems * kWarps), st,
                       ws.get<uint4>("stage", tiles_c(m) * kCTile)};
  uint32_t* hcounts = ws.get<uint32_t>("hook_counts", tiles_of(n));
  uint32_t* hmasks = ws.get<uint32_t>("hook_masks", tiles_of(n) * kItems * kWarps);
  uint32_t* hslot = ws.get<uint32_t>("hook_slotpref", tiles_of(n) * kItems * kWarps);

  // counters, the first min table and the MST flags in one launch (three
  // stream operations cost c1 ~20 us before its first kernel)
  uint32_t* flags = ws.get<uint32_t>("mst_bits", mst_out_words(m));
  const int mst_bytes = mst_out_bytes(m) ? 1 : 0;
  launch_k(k_init_run, (unsigned)(sm_count(dev) * 8), 256, s, d_ctr, n, m, minb[0], (uint4*)flags, mst_out_words(m) / 4);
  timeline_mark(nullptr, s);
  uint32_t launches = 0;
  int tix = 0;
  std::vector<HotLaunch> hot;
  auto tmark = [&]() {
    if (time_hot) MST_CUDA_CHECK(cudaEventRecord(ws.tev[tix++], s));
  };
  auto hot_begin = [&](int kind, int r, bool light) {
    if (time_hot) hot.push_back(HotLaunch{tix, kind, r, light});
    tmark();
  };

  double light_target = (double)m;  // expected light edges (Filter-Borůvka)
  if (filter) {
    uint32_t* hist = ws.get<uint32_t>("hist", 65536);
    MST_CUDA_CHECK(cudaMemsetAsync(hist, 0, 65536 * sizeof(uint32_t), s));
    // 256 K sampled weights place a pivot at the ~beta*n/m quantile within
    // ~1 % (the light set's size is a tuning target, not a correctness one)
    const uint32_t samples = (uint32_t)std::min<uint64_t>(m, (uint64_t)knob(kKnobPivotSamples));
    const uint64_t step = std::max<uint64_t>(1, m / samples);
    launch_k(k_weight_hist, std::max(1u, samples / 1024), 256, s, wbase, wstride, m, step, samples, hist);
    const double beta = knob(kKnobFilterBeta);
    const double frac = std::min(1.0, beta * (double)n / (double)m);
    light_target = frac * (double)m;
    launch_k(k_pick_pivot, 1, 1024, s, hist, frac, d_ctr);
    launches += 2;
    hot_begin(kHotSplit, 0, true);
    launch_two_pass<InView, kModeLight>(ws, cb, in, nullptr, nullptr, E[1], minb[0], d_ctr, 0, m, n,
                                        kSlotCompact, 0, filt_for(n, kSiteSplit), PairTable{nullptr, 0}, true,
                                        nullptr, n);
    tmark();
    launches += 2;
  } else {
    auto kmin = k_min_round1<InView>;
    hot_begin(kHotMin1, 0, false);
    // one launch per host-copy chunk when the caller's list is still
    // arriving (run_single's pipelined H2D), else one over the whole list
    const int nch = chunks ? chunks->count : 1;
    for (int j = 0; j < nch; ++j) {
      const uint64_t lo = chunks ? chunks->bound[j] : 0, hi = chunks ? chunks->bound[j + 1] : m;
      if (chunks) MST_CUDA_CHECK(cudaStreamWaitEvent(s, chunks->ev[j], 0));
      const unsigned g = (unsigned)std::max<uint64_t>(
          1, std::min<uint64_t>((hi - lo + 4 * kBlock - 1) / (4 * kBlock), (uint64_t)sm_count(dev) * blocks_per_sm(kmin)));
      launch_k(kmin, g, kBlock, s, in, n, lo, hi, minb[0], d_ctr, filt_for(n, kSiteMin1));
      ++launches;
    }
    tmark();
  }

  bool light = filter;
  std::vector<std::pair<uint32_t*, int>> levels;  // light-phase relabel maps (buffer, round)
  // Retirement (kernels.cuh, k_ret_*): the light rounds run by the round
  // kernels retire their isolated components into bitmap regions, one per
  // round (sized by the host's bound on n_r), then the final region. R-MAT's
  // light phase: 44 M of c4's 67 M vertices have no light edge, so from round
  // 2 on the per-component tables cover ~5 M instead of ~49 M components.
  RetireState ret;
  ret.init(ws, n, filter && knob_i(kKnobRetire) != 0 && n < (1u << 31));
  uint64_t n_bound = n, m_bound = m;
  int r = 1, loop_start = 1;
  int phase_end = 0;
  DevCounters snap_b{};  // counters at the end of the light phase
  const bool tail_on = knob_i(kKnobTail) != 0;
  const bool dedup_on = knob_i(kKnobDedup) != 0;
  // off by default: the tail's inserts are latency-bound at 2 CTAs/SM (c1
  // round 3: 106 us for 3.0 M edges), slower than what they save
  const bool tail_dedup_on = dedup_on && knob_i(kKnobTailDedup) != 0;
  const uint64_t dedup_min_edges = (uint64_t)knob(kKnobDedupMinEdges);
  const unsigned int dedup_active = (unsigned int)knob(kKnobDedupActive);
  // low byte: table slots >= m_r / div; bit 8: retry after an overflowed
  // attempt without waiting for the K(K-1)/2 <= m_r/8 guarantee; bits
  // 16-23: the minimum edges-per-active-component ratio of a dedup round
  const unsigned int pair_div = (unsigned int)std::max(1, std::min(255, knob_i(kKnobDedupTableDiv))) |
                                (knob_i(kKnobDedupRetry) ? 0x100u : 0u) |
                                ((unsigned int)std::max(1, std::min(255, knob_i(kKnobDedupMinRatio))) << 16) |
                                ((unsigned int)std::max(0, std::min(255, knob_i(kKnobDedupGuarantee))) << 24);
  // Tail entry (m_bound is the host's one-round-stale edge bound). Measured
  // (tools/sweep_tail.sh, tools/sweep_tail2.sh): the plain loop and phase D
  // gain from entering early (12 M: c1's round 2 with 5.1 M edges runs in
  // the segmented tail, 0.631 -> 0.602 ms), the light phase from keeping the round kernels,
  // whose pair dedup the tail lacks, a little longer (c2: 3.02 ms at 3 M vs
  // 3.19 ms at 6 M).
  const double tail_env = knob(kKnobTailEdges);
  const uint64_t tail_comps = (uint64_t)knob(kKnobTailComps);
  // Few components but many edges (uniform graphs collapse their components
  // long before their edges): every offer of a round kernel then hits one of
  // a few thousand table entries and the atomics serialise (uniform m/n = 8:
  // ~0.7 ms per such round); the tail aggregates those offers per block in
  // shared memory (4.1 -> 1.2 ms). So the tail also takes over once
  // n_r <= tail_small_n, whatever the edge count.
  const uint64_t tail_small_n = (uint64_t)knob(kKnobTailSmallN);
  auto tail_edges = [&]() -> uint64_t { return (uint64_t)(tail_env > 0 ? tail_env : (light ? 3.0e6 : 12.0e6)); };

  // Lazy round 1 (plain loop): round 1 stops after its count pass, whose
  // relabelled label pairs (one per caller edge) are round 2's edge list;
  // round 2 compacts them. Saves round 1's emit pass (c1: 32 us). Not when
  // round 2 enters the tail, which needs a compacted list.
  // Round 1 handed to the tail at its phase C (plain loop, SoA input): the
  // round kernels do round 1's min / hook / label at full occupancy, the
  // tail's first pass relabels + compacts + offers straight from the caller's
  // list, replacing round 1's count + emit passes.
  const bool start_c_ok = tail_on && !filter && std::is_same<InView, SoaView>::value &&
                          knob_i(kKnobTailStartC) != 0 && m <= (32ull << 20) && n <= (16u << 20);
  bool tail_c_pending = false;
  auto tail_grid = [&]() -> unsigned {
    const int bps = std::max(1, std::min(blocks_per_sm(k_tail, 0), knob_i(kKnobTailBps)));
    return std::min<unsigned>(kTailMaxBlocks, (unsigned)(sm_count(dev) * bps));
  };
  const bool lazy1 = !start_c_ok && !filter && knob_i(kKnobLazyRound1) != 0 &&
                     !(tail_on && (m <= tail_edges() || (uint64_t)n <= tail_small_n) && (uint64_t)n <= tail_comps);
  const uint4* P1 = lazy1 ? reinterpret_cast<const uint4*>(ws.get<uint2>("pairs1", m)) : E[1];

  // Light phase over: compose its relabel maps into a vertex -> component map,
  // run the heavy filter pass, continue with the plain loop (phase D).
  // Returns false when the run was restarted in plain mode.
  auto end_light_phase = [&](const DevCounters& snap) -> bool {
    phase_end = (int)snap.phase_end;
    snap_b = snap;
    if (phase_end == 1) {
      // not a single light non-loop edge: run the plain loop instead
      MST_CUDA_CHECK(cudaStreamSynchronize(s));
      RunOut plain;
      run_single_impl<InView>(ws, in, wbase, wstride, n, m, plain, time_hot, false, nullptr, enqueue_after);
      plain.launches += launches;
      out = plain;
      return false;
    }
    while (!levels.empty() && levels.back().second >= phase_end) levels.pop_back();
    ret.drop_from(phase_end);
    const bool retired = ret.active() && !levels.empty();
    if (retired) {
      launches += ret.finalize(ws, s, d_ctr, phase_end, levels, snap, minb[(phase_end - 1) & 1]);
    } else {
      for (int k = (int)levels.size() - 2; k >= 0; --k) {
        const unsigned g = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>((snap.n[levels[k].second] + 255) / 256, (uint64_t)sm_count(dev) * 8));
        launch_k(k_compose, g, 256, s, levels[k].first, levels[k + 1].first, d_ctr, levels[k].second);
        ++launches;
      }
    }
    const uint32_t* vlabel = levels.empty() ? nullptr : levels[0].first;
    MST_CUDA_CHECK(cudaMemsetAsync(&d_ctr->phase_end, 0xFF, sizeof(unsigned int), s));
    const int R1 = phase_end;
    // retirement: n[R1] (all final components) was counted on the device
    const uint64_t n_heavy = retired ? read_count(ws, s, d_ctr, R1) : snap.n[R1];
    hot_begin(kHotHeavy, R1, false);
    // launched as round R1-1's producer: it writes m[R1] and E/min of round R1
    launch_two_pass<InView, kModeHeavy>(ws, cb, in, nullptr, vlabel, E[R1 & 1], minb[(R1 - 1) & 1], d_ctr,
                                        R1 - 1, m, n, kSlotFilter, 0, filt_for(snap.n[R1], kSiteHeavy),
                                        PairTable{nullptr, 0}, true, nullptr, n_heavy);
    tmark();
    launches += 2;
    light = false;
    r = R1;
    loop_start = R1;
    n_bound = n_heavy;
    m_bound = m;
    return true;
  };

  // The list round r's min-table keys index (see k_count): the caller's list
  // in round 1 of the plain loop, the light split's / heavy filter's output
  // in the first round after them, round 1's label pairs in round 2 of the
  // plain loop, else round r-1's list (relabelled in place by its count pass).
  auto hook_src = [&](int rr) -> HookSrc {
    if (rr == 1) return filter ? HookSrc{kSrcPacked, E[1]} : HookSrc{kSrcIn, nullptr};
    if (phase_end && rr == phase_end) return HookSrc{kSrcPacked, E[rr & 1]};
    if (rr == 2 && !filter) return HookSrc{kSrcPairs, P1};
    if (rr == 3 && lazy1) return HookSrc{kSrcPairs, P1};  // round 2 relabelled the pairs in place
    return HookSrc{kSrcPacked, E[(rr - 1) & 1]};
  };

  while (true) {
    if (r > MST_MAX_ROUNDS) throw MstError{MST_ERR_STALL, "no convergence within MST_MAX_ROUNDS rounds"};
    const bool original_in = (r == 1 && !filter);
    // after retirement n_bound counts the light components with edges only:
    // few of them can still carry millions of edges, which the round
    // kernels' pair dedup collapses and the tail would not (c3: 4 tail
    // rounds over ~9 M edges, +0.8 ms), so the small-n rule stays off there
    const bool retiring = light && ret.active();
    // round 1 of the light phase: the split keeps ~beta*n edges (the pivot's
    // target), a better bound than m before its count is known
    const uint64_t m_est = (light && r == 1) ? std::min<uint64_t>(m_bound, (uint64_t)(1.1 * light_target)) : m_bound;
    // the tail runs at 2 CTAs/SM: its component phases are latency-bound when
    // n_r is huge (c4's light phase ends with 47 M components and 406 edges:
    // 1.2 ms in the tail vs 0.3 ms of round kernels)
    if (tail_c_pending ||
        (tail_on && !original_in && (m_est <= tail_edges() || (n_bound <= tail_small_n && !retiring)) &&
         n_bound <= tail_comps)) {
      // ---- all remaining rounds in one cooperative launch
      uint32_t* M = nullptr;
      if (light) {
        M = ws.get<uint32_t>("Ltail", n_bound);
        launch_k(k_iota, (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_bound + 255) / 256, 4096)), 256, s, 
            M, n_bound);
        ++launches;
      }
      auto kt = k_tail;
      const size_t tail_smem = 0;  // all static (< 48 KB)
      const unsigned G = tail_grid();
      uint32_t* broots = ws.get<uint32_t>("tail_broots", G);
      uint32_t* tmasks = ws.get<uint32_t>("tail_masks", n_bound / 32 + 64);
      uint32_t* twpref = ws.get<uint32_t>("tail_wpref", n_bound / 32 + 64);
      unsigned long long* trace = nullptr;
      if (knob_i(kKnobTailTrace)) {
        trace = ws.get<unsigned long long>("tail_trace", 512);
        MST_CUDA_CHECK(cudaMemsetAsync(trace, 0, 512 * 8, s));
      }
      const HookSrc src = hook_src(r);
      TailArgs ta{{E[0], E[1]}, {minb[0], minb[1]}, parent, L, broots, tmasks, twpref, M, flags,
                  trace, 0, nullptr, nullptr, nullptr, 0, d_ctr, n, r, (int)light};
      ta.start_c = tail_c_pending ? 1 : 0;
      ta.mst_bytes = mst_bytes;
      ta.retired = (light && ret.active()) ? 1 : 0;
      ta.c_soa = (tail_c_pending && r == 1) ? 1 : 0;
      if (knob_i(kKnobTailTiny)) {
        // three rotating min tables for the one-sync rounds (k_tail "tiny")
        unsigned long long* tiny = ws.get<unsigned long long>("tail_tiny", 3 * kTailSmemMin);
        MST_CUDA_CHECK(cudaMemsetAsync(tiny, 0xFF, 3 * kTailSmemMin * sizeof(unsigned long long), s));
        for (int k = 0; k < 3; ++k) ta.tiny[k] = tiny + k * kTailSmemMin;
      }
      if (tail_dedup_on) {
        // per-round table mask <= next_pow2(m_r / 2) <= this
        const size_t slots = (size_t)std::max<unsigned long long>(1024, next_pow2(std::max<uint64_t>(m_bound / 2, 1)));
        ulonglong2* pairs = ws.get<ulonglong2>("tail_pairs", slots);
        if (slots > ws.pair_slots || ws.pair_epoch >= 1022) {
          ws.pair_slots = std::max(ws.pair_slots, slots);
          MST_CUDA_CHECK(cudaMemsetAsync(pairs, 0xFF, ws.pair_slots * sizeof(ulonglong2), s));
          ws.pair_epoch = 0;
        }
        ta.pairs = pairs;
        ta.pair_cap = slots;
        ta.pair_epoch = ++ws.pair_epoch;
        ta.dedup_ratio = (uint32_t)knob_i(kKnobTailDedupRatio);
        ta.dedup_min = (uint32_t)knob(kKnobTailDedupMin);
      }
      if (src.kind == kSrcPacked) {
        ta.src_kind = kTailSrcPacked;
        ta.src0 = src.packed;
      } else if (src.kind == kSrcPairs) {
        ta.src_kind = kTailSrcPairs;
        ta.src0 = src.packed;
        ta.src_w = wbase;
        ta.src_wstride = wstride;
      } else if constexpr (std::is_same_v<InView, SoaView>) {
        ta.src_kind = kTailSrcSoa;
        ta.src0 = in.src;
        ta.src1 = in.dst;
        ta.src_w = in.w;
      } else {
        ta.src_kind = kTailSrcAos;
        ta.src0 = in.e;
      }
      void* args[] = {&ta};
      hot_begin(kHotTail, r, light);
      MST_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)kt, G, kBlock, args, tail_smem, s));
      ++t_launches;
      timeline_mark((const void*)kt, s);
      ++launches;
      tmark();
      // outside the light phase the tail runs the loop to its verdict (stop,
      // error or stall), which the epilogue reads after its one sync
      if (!light && !trace) break;
      MST_CUDA_CHECK(cudaMemcpyAsync(&ws.h_snap[kMaxR - 1], d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
      MST_CUDA_CHECK(cudaStreamSynchronize(s));
      const DevCounters& snap = ws.h_snap[kMaxR - 1];
      if (trace) {
        std::vector<unsigned long long> tt(512);
        MST_CUDA_CHECK(cudaMemcpy(tt.data(), trace, 512 * 8, cudaMemcpyDeviceToHost));
        fprintf(stderr, "tail r0=%d G=%u:", r, G);
        for (int i = 1; i < 512 && tt[i]; ++i) fprintf(stderr, " %.1f", (tt[i] - tt[i - 1]) * 1e-3);
        fprintf(stderr, " (us per phase: A B C per round)\n");
      }
      if (snap.err || snap.stop_round != kNoStop) break;
      if (light && snap.phase_end != kNoStop) {
        if (M) levels.push_back({M, r});
        if (!end_light_phase(snap)) return;
        continue;
      }
      throw MstError{MST_ERR_STALL, "tail kernel ended without a verdict"};
    }
    unsigned long long* mcur = minb[(r - 1) & 1];
    unsigned long long* mnext = minb[r & 1];
    uint4* Eout = E[(r + 1) & 1];
    uint32_t* rb = nullptr;  // this round's retirement region (light phase)
    {
      const uint64_t ht = tiles_of(n_bound);
      const int hfused = ht <= kFusedScanMaxTiles ? 1 : 0;
      const HookSrc src = hook_src(r);
      // a light round retires its isolated components into its own region
      // (the last region is kept for the final one)
      rb = light ? ret.take(s, r, n_bound) : nullptr;
      const int hphase = (light && ret.active()) ? (int)kPhaseLightRetire : (int)light;
      auto launch_hook = [&](auto view) {
        auto kd = k_hook_decide<decltype(view)>;
        launch_k(kd, (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ht, (uint64_t)sm_count(dev) * blocks_per_sm(kd))),
                 kBlock, s, view, mcur, parent, hmasks, hcounts, d_ctr, r, hfused, hphase, hslot, flags, mst_bytes, rb);
      };
      if (src.kind == kSrcIn)
        launch_hook(in);
      else if (src.kind == kSrcPairs)
        launch_hook(PairsView<InView>{reinterpret_cast<const uint2*>(src.packed), in});
      else
        launch_hook(PackedView{src.packed});
      if (!hfused)
        launch_k(k_scan_counts<kScanRoots>,
                 (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ht + kScanTile - 1) / kScanTile, (uint64_t)sm_count(dev))),
                 kScanBlock, s, hcounts, ht, d_ctr, r, st, ws.next_epoch(), hphase, 0);
      launches += 1;
    }
    uint32_t* Lr = L;
    if (light) {
      Lr = ws.get<uint32_t>("Llvl" + std::to_string(r), n_bound);
      levels.push_back({Lr, r});
    }
    // pair dedup is armed for big rounds; k_label2 decides on the device
    PairTable pt{nullptr, 0};
    const bool lazy2 = lazy1 && r == 2;  // round 2 over round 1's uncompacted pairs
    // phase D's first round (Filter-Boruvka): hook + label here, then the
    // tail starts at its phase C over the heavy survivors in place (the host
    // knows only m here, not the survivor count: bounded by components and
    // by m <= 32 M: measured across sizes (tools/knob_ab_sizes.py) the
    // hand-off gains 2 % on lists of <= 18 M edges and loses 1-3 % from 64 M
    // on, where the round kernels' full-occupancy compaction wins; c4's 47 M
    // components are excluded either way)
    const bool d_start_c = tail_on && !light && phase_end && r == phase_end && knob_i(kKnobTailStartCD) != 0 &&
                           m_bound <= (uint64_t)knob(kKnobTailStartCDEdges) &&
                           n_bound <= (16u << 20);
    if (!original_in && !lazy2 && !d_start_c && dedup_on && m_bound >= dedup_min_edges) {
      const unsigned long long cap = std::min<unsigned long long>(1ull << std::max(10, std::min(30, knob_i(kKnobDedupCapLog2))),
                                                                   next_pow2(m_bound / 2));
      unsigned long long* tab = ws.get<unsigned long long>("pair_table", 2 * cap);
      pt = PairTable{tab, cap};
      launches += 2;
    }
    {
      const unsigned g = (unsigned)std::max<uint64_t>(
          1, std::min<uint64_t>(tiles_of(n_bound), (uint64_t)sm_count(dev) * blocks_per_sm(k_label2)));
      launch_k(k_label2, g, kBlock, s, parent, hmasks, hslot, hcounts, Lr, mnext, d_ctr, r, pt.pairs, pt.cap,
               dedup_active, pair_div, (const uint32_t*)rb);
    }
    if ((original_in && start_c_ok) || d_start_c) {  // this round's compaction: the tail's first phase C
      tail_c_pending = true;
      continue;
    }
    hot_begin(kHotCompact, r, light);
    if (original_in) {
      // plain round 1: label pairs of the caller's list in P1 (lazy: that is
      // round 2's list), else compacted into E[0]
      launch_two_pass<InView, kModeRelabel>(ws, cb, in, const_cast<uint4*>(P1), Lr, Eout, mnext, d_ctr, r, m_bound, n,
                                            kSlotCompact, (int)light, filt_for(n_bound, kSiteCount, filter),
                                            PairTable{nullptr, 0}, !lazy1);
    } else if (lazy2) {
      using PV = PairsInView<InView>;
      launch_two_pass<PV, kModeRelabel>(ws, cb, PV{reinterpret_cast<const uint2*>(P1), in, in.base},
                                        const_cast<uint4*>(P1), Lr, Eout, mnext, d_ctr, r, m, n, kSlotCompact,
                                        (int)light, filt_for(n_bound, kSiteCount, filter));
    } else {
      // a round with a huge component count (phase D's first on R-MAT):
      // most endpoints join one giant, whose label the compaction takes from
      // a bitmap (kernels.cuh k_giant_bits)
      const uint32_t* gb = nullptr;
      const double giant_min = knob(kKnobGiantBits);
      if (giant_min > 0 && !light && (double)n_bound >= giant_min) {
        uint32_t* bits = ws.get<uint32_t>("giant_bits", (n_bound + 31) / 32 + 1);
        launch_k(k_pick_giant, 1, 1024, s, (const uint4*)E[r & 1], (const uint32_t*)Lr, d_ctr, r);
        launch_k(k_giant_bits, (unsigned)(sm_count(dev) * 8), 256, s, (const uint32_t*)Lr, (const DevCounters*)d_ctr, r,
                 bits);
        gb = bits;
        launches += 2;
      }
      launch_two_pass<PackedView, kModeRelabel>(ws, cb, PackedView{E[r & 1]}, E[r & 1], Lr, Eout, mnext, d_ctr,
                                                r, m_bound, n, kSlotCompact, (int)light, filt_for(n_bound, kSiteCount, filter), pt,
                                                true, gb);
    }
    tmark();
    launches += 5;
    MST_CUDA_CHECK(cudaGetLastError());
    MST_CUDA_CHECK(cudaMemcpyAsync(&ws.h_snap[r], d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    MST_CUDA_CHECK(cudaEventRecord(ws.ev[r], s));
    if (r > loop_start) {
      MST_CUDA_CHECK(cudaEventSynchronize(ws.ev[r - 1]));
      const DevCounters& snap = ws.h_snap[r - 1];
      if (snap.err) break;
      if (snap.stop_round != kNoStop && (int)snap.stop_round <= r) break;
      if (light && snap.phase_end != kNoStop && (int)snap.phase_end <= r) {
        if (!end_light_phase(snap)) return;
        continue;
      }
      n_bound = snap.n[r];
      m_bound = snap.m[r];
    }
    ++r;
  }
  // the sort first: the counter read-back is a copy-engine operation in
  // the stream that the sort kernels would otherwise queue behind
  if (enqueue_after) (*enqueue_after)();
  MST_CUDA_CHECK(cudaMemcpyAsync(&out.ctr, d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
  MST_CUDA_CHECK(cudaStreamSynchronize(s));
  const DevCounters& c = out.ctr;
  out.err = c.err;
  out.launches = launches;
  if (c.err) return;
  const int stop = (int)c.stop_round;
  if (c.stop_round == kNoStop) throw MstError{MST_ERR_STALL, "round loop ended without a stop verdict"};
  out.rounds = (uint32_t)stop - 1;
  out.phase_end = (uint32_t)phase_end;
  out.final_components = c.n[stop];
  out.count = (uint64_t)n - out.final_components;
  out.total_weight = c.total_weight;
  if (knob_i(kKnobDebugRounds)) {
    for (int rr = 1; rr < stop && rr < kMaxR; ++rr)
      fprintf(stderr, "round %2d: n=%u m=%llu active=%u dedup=%u%s\n", rr, c.n[rr], (unsigned long long)c.m[rr],
              c.active[rr], c.dedup[rr], (phase_end && rr == phase_end) ? "  <- heavy survivors" : "");
  }
  if (time_hot) {
    for (const HotLaunch& h : hot) {
      uint64_t bytes = 0;
      if (h.kind == kHotMin1) {
        bytes = 12ull * m;
      } else if (h.kind == kHotSplit) {
        bytes = 12ull * m + 16ull * c.m[1];
      } else if (h.kind == kHotHeavy) {
        bytes = 12ull * m + 16ull * c.m[h.r];
      } else if (h.kind == kHotTail) {
        // algorithmic: one 16 B read per live edge, one 16 B write per kept edge
        const int last = (h.light && phase_end) ? phase_end : stop;
        const DevCounters& cc = (h.light && phase_end) ? snap_b : c;
        for (int rr = h.r; rr + 1 < last && rr < kMaxR - 1; ++rr)
          bytes += ((rr == 1 && !filter) ? 12ull : 16ull) * cc.m[rr] + 16ull * cc.m[rr + 1];
      } else {
        const bool ran = h.r + 1 < stop && (!h.light || phase_end == 0 || h.r < phase_end);
        if (!ran) continue;
        const DevCounters& cc = (h.light && phase_end) ? snap_b : c;
        const uint64_t in_bytes = (h.r == 1 && !filter) ? 12ull : 16ull;
        bytes = in_bytes * cc.m[h.r] + 16ull * cc.m[h.r + 1];
      }
      out.ms_hot += ms_between(ws.tev[h.ev], ws.tev[h.ev + 1]);
      out.hot_launches += 1;
      out.hot_bytes += bytes;
    }
  }
}

uint64_t alg_bytes_from(const DevCounters& c, uint32_t rounds, uint32_t phase_end) {
  // SURVEY.md §8(d)'s units: 12 B per caller edge read, 16 B per packed edge
  // read, 16 B per kept edge written, 32 B per live component.
  // Plain loop: 12 m + 32 sum k_r + 32 sum n_r (its formula).
  // Filter-Boruvka: the caller's list is streamed twice (split, heavy
  // filter: 2 x 12 m[0]) and every round list m[r] -- the split's output,
  // each emit's, the heavy survivors' -- is written once and read once.
  uint64_t b = 0;
  for (uint32_t r = 1; r <= rounds; ++r) b += 32ull * c.n[r];
  if (phase_end == 0) {
    b += 12ull * c.m[1];
    for (uint32_t r = 2; r <= rounds; ++r) b += 32ull * c.m[r];
  } else {
    b += 24ull * c.m[0];
    for (uint32_t r = 1; r <= rounds; ++r) b += 32ull * c.m[r];
  }
  return b;
}

void fill_stats(mst_stats_t* st, const RunOut& o) {
  if (!st) return;
  st->rounds = o.rounds;
  st->final_components = o.final_components;
  st->alg_bytes = alg_bytes_from(o.ctr, o.rounds, o.phase_end);
  for (int r = 0; r < MST_MAX_ROUNDS; ++r) {
    const bool live = (uint32_t)(r + 1) <= o.rounds;
    st->live_edges[r] = live ? o.ctr.m[r + 1] : 0;
    st->live_comps[r] = live ? o.ctr.n[r + 1] : 0;
  }
  st->kernel_launches = o.launches;
}

void check_err_bits(uint32_t err) {
  if (err & kErrRange)
    throw MstError{MST_ERR_RANGE, "endpoint out of range: an edge touches a vertex outside [0,n)"};
  if (err & kErrWeight) throw MstError{MST_ERR_WEIGHT, "edge weight does not fit in 32 bits"};
}

void validate_common(uint32_t n, uint64_t m) {
  if (n < 1) throw MstError{MST_ERR_INVALID_ARG, "vertex count must be >= 1"};
  if (m >= 0xFFFFFFFFull) throw MstError{MST_ERR_INVALID_ARG, "edge count must be < 2^32-1"};
}

int current_device_checked() {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw MstError{MST_ERR_NO_DEVICE, std::string("no CUDA device available: ") +
                                          (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e))};
  }
  int dev = 0;
  MST_CUDA_CHECK(cudaGetDevice(&dev));
  return dev;
}

// Common tail: sort the emitted ids, copy back, timing, stats.
struct SingleArgs {
  uint32_t n;
  uint64_t m;
  int kind;  // 0 SoA, 1 AoS
  const uint32_t *src, *dst, *w;
  const mst_edge_t* aos;
  int on_device;
  uint32_t* out_ids;       // host (or device when device_out)
  bool device_out;
  cudaStream_t user_stream;
  bool time_hot;
};

// The L2 fetch granularity knob (a device-wide limit): applied when it
// changes, per device.
void apply_l2_fetch(int dev) {
  static std::mutex mu;
  static std::map<int, int> applied;
  static std::map<int, size_t> dflt;
  const int want = knob_i(kKnobL2Fetch);
  std::lock_guard<std::mutex> g(mu);
  auto it = applied.find(dev);
  if (want <= 0 && it == applied.end()) return;
  if (it != applied.end() && it->second == want) return;
  if (!dflt.count(dev)) {
    size_t d = 0;
    MST_CUDA_CHECK(cudaDeviceGetLimit(&d, cudaLimitMaxL2FetchGranularity));
    dflt[dev] = d;
  }
  MST_CUDA_CHECK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, want > 0 ? (size_t)want : dflt[dev]));
  applied[dev] = want;
}

RunOut run_single(const SingleArgs& a, mst_stats_t* stats) {
  const auto t_start = Clock::now();
  const uint64_t launches0 = t_launches;
  const int dev = current_device_checked();
  apply_l2_fetch(dev);
  Workspace& ws = workspace(dev, 0);
  std::lock_guard<std::mutex> lock(ws.mu);
  MST_CUDA_CHECK(cudaSetDevice(dev));
  cudaStream_t saved = ws.stream;
  if (a.user_stream) ws.stream = a.user_stream;
  struct Restore {
    Workspace& w;
    cudaStream_t s;
    ~Restore() { w.stream = s; }
  } restore{ws, saved};
  cudaStream_t s = ws.stream;
  // Device input (or a device result) with no caller stream: the caller's
  // work is on the legacy default stream 0, which the private non-blocking
  // stream does not wait for. Join it both ways: the MST starts after the
  // caller's earlier work (input writes, an L2 flush, a timing event) and
  // stream 0's later work (timing events, consumers of the ids) waits for it.
  const bool join_legacy = !a.user_stream && (a.on_device || a.device_out);
  if (join_legacy) {
    MST_CUDA_CHECK(cudaEventRecord(ws.join_in, cudaStreamLegacy));
    MST_CUDA_CHECK(cudaStreamWaitEvent(s, ws.join_in, 0));
  }

  cudaEvent_t e0, e1, e2, e3;
  e0 = ws.tev[ws.tev.size() - 4];
  e1 = ws.tev[ws.tev.size() - 3];
  e2 = ws.tev[ws.tev.size() - 2];
  e3 = ws.tev[ws.tev.size() - 1];
  MST_CUDA_CHECK(cudaEventRecord(e0, s));
  const uint32_t* src = a.src;
  const uint32_t* dst = a.dst;
  const uint32_t* w = a.w;
  const mst_edge_t* aos = a.aos;
  // Pinned SoA input on the plain loop: copy in chunks on the copy stream
  // while round 1's min pass consumes the chunks that have landed (and the
  // table clears run), so the H2D hides that work. Off by default: measured
  // on c1 (tools/exp_pipeline_h2d.sh), 24 chunk copies move the 100 MB in 1.94 ms vs
  // 1.83 ms for three whole-array copies, more than the ~45 us they hide.
  CopyChunks chunks;
  const bool pipelined = !a.on_device && a.kind == 0 && a.m >= (4u << 20) && !filter_mode(a.n, a.m) &&
                         knob_i(kKnobPipelineH2D) != 0 && host_is_pinned(a.src) && host_is_pinned(a.dst) &&
                         host_is_pinned(a.w);
  if (!a.on_device && a.m > 0) {
    if (a.kind == 0) {
      uint32_t* d_src = ws.get<uint32_t>("in_src", a.m);
      uint32_t* d_dst = ws.get<uint32_t>("in_dst", a.m);
      uint32_t* d_w = ws.get<uint32_t>("in_w", a.m);
      if (pipelined) {
        // the copies may not overwrite the buffers before earlier work on
        // the compute stream is done with them
        MST_CUDA_CHECK(cudaStreamWaitEvent(ws.copy_stream, e0, 0));
        const int want = std::max(1, std::min(CopyChunks::kMax, knob_i(kKnobPipelineChunks)));
        const uint64_t per = std::max<uint64_t>(1u << 20, (a.m + want - 1) / want);
        chunks.count = (int)((a.m + per - 1) / per);
        for (int j = 0; j <= chunks.count; ++j) chunks.bound[j] = std::min<uint64_t>(a.m, (uint64_t)j * per);
        for (int j = 0; j < chunks.count; ++j) {
          const uint64_t lo = chunks.bound[j], len = (chunks.bound[j + 1] - lo) * 4;
          MST_CUDA_CHECK(cudaMemcpyAsync(d_src + lo, a.src + lo, len, cudaMemcpyHostToDevice, ws.copy_stream));
          MST_CUDA_CHECK(cudaMemcpyAsync(d_dst + lo, a.dst + lo, len, cudaMemcpyHostToDevice, ws.copy_stream));
          MST_CUDA_CHECK(cudaMemcpyAsync(d_w + lo, a.w + lo, len, cudaMemcpyHostToDevice, ws.copy_stream));
          chunks.ev[j] = ws.chunk_ev[j];
          MST_CUDA_CHECK(cudaEventRecord(chunks.ev[j], ws.copy_stream));
        }
      } else {
        copy_h2d(ws, d_src, a.src, a.m * 4);
        copy_h2d(ws, d_dst, a.dst, a.m * 4);
        copy_h2d(ws, d_w, a.w, a.m * 4);
      }
      src = d_src;
      dst = d_dst;
      w = d_w;
    } else {
      mst_edge_t* d_e = ws.get<mst_edge_t>("in_aos", a.m);
      copy_h2d(ws, d_e, a.aos, a.m * sizeof(mst_edge_t));
      aos = d_e;
    }
  }
  MST_CUDA_CHECK(cudaEventRecord(e1, s));

  RunOut o;
  uint32_t* d_sorted = a.device_out ? a.out_ids : ws.get<uint32_t>("sorted", std::max<uint32_t>(a.n, 1));
  auto* d_ctr = ws.get<DevCounters>("ctr", 1);
  uint32_t* d_flags = ws.get<uint32_t>("mst_bits", mst_out_words(a.m));
  // the sorted ids and their copy-back, enqueued behind the last round: a
  // spanning tree has n - 1 edges, so n - 1 ids are copied (a forest's
  // shorter list is followed by stale slots, which the caller's n - 1
  // capacity holds and the returned count excludes)
  uint32_t sort_launches = 0;
  const std::function<void()> after = [&]() {
    sort_launches = mst_out_bytes(a.m)
                        ? sort_from_bytes(ws, reinterpret_cast<const uint8_t*>(d_flags), std::max<uint64_t>(a.m, 1),
                                          d_sorted, d_ctr)
                        : sort_from_bits(ws, d_flags, std::max<uint64_t>(a.m, 1), d_sorted, d_ctr);
    MST_CUDA_CHECK(cudaEventRecord(e2, s));
    if (!a.device_out && a.n > 1) copy_d2h(ws, a.out_ids, d_sorted, (uint64_t)(a.n - 1) * 4);
    MST_CUDA_CHECK(cudaEventRecord(e3, s));
  };
  if (a.kind == 0) {
    SoaView v{src, dst, w, 0};
    run_single_impl<SoaView>(ws, v, w, 1, a.n, a.m, o, a.time_hot, filter_mode(a.n, a.m),
                             chunks.count ? &chunks : nullptr, &after);
  } else {
    AosView v{reinterpret_cast<const uint4*>(aos), 0};
    const uint32_t* wb = reinterpret_cast<const uint32_t*>(aos) + 2;
    run_single_impl<AosView>(ws, v, wb, 4, a.n, a.m, o, a.time_hot, filter_mode(a.n, a.m), nullptr, &after);
  }
  check_err_bits(o.err);
  o.launches = (uint32_t)(t_launches - launches0);  // every kernel of the call, counted at launch
  (void)sort_launches;
  if (join_legacy) {
    MST_CUDA_CHECK(cudaEventRecord(ws.join_out, s));
    MST_CUDA_CHECK(cudaStreamWaitEvent(cudaStreamLegacy, ws.join_out, 0));
  }
  MST_CUDA_CHECK(cudaStreamSynchronize(s));
  timeline_print(e0);
  if (stats) {
    fill_stats(stats, o);
    if (chunks.count) {
      // pipelined: h2d = until the last chunk landed, device = what remained
      const cudaEvent_t last = chunks.ev[chunks.count - 1];
      stats->ms_h2d = ms_between(e0, last);
      stats->ms_device = ms_between(last, e2);
    } else {
      stats->ms_h2d = ms_between(e0, e1);
      stats->ms_device = ms_between(e1, e2);
    }
    stats->ms_d2h = ms_between(e2, e3);
    stats->ms_total = std::chrono::duration<double, std::milli>(Clock::now() - t_start).count();
  }
  return o;
}

// ------------------------------- sharded (multi-GPU) ------------------------
// Edge-sharded, component state replicated (kernels.cuh, "sharded exchange"):
// every shard runs the same hook/label on the all-reduced (w, global id) keys
// and partner labels, so the MST ids, labels and verdicts agree everywhere and
// only the local edge lists differ.

struct Shard {
  Workspace* ws = nullptr;
  uint64_t m = 0;        // local edges
  uint32_t base = 0;     // global id of local edge 0
  SoaView in{};
  unsigned long long* minb[2]{};
  unsigned long long *xch = nullptr, *own = nullptr;
  uint32_t *parent = nullptr, *L = nullptr, *partner = nullptr;
  uint32_t* flags = nullptr;  // MST bitmap over global edge ids (replicated: every rank sets every bit)
  RetireState ret;           // light-phase retirement (replicated decisions)
  uint32_t* hist = nullptr;  // Filter-Borůvka: weight histogram (summed across shards)
  uint32_t* errw = nullptr;  // error bits as counts (summed across shards)
  uint4* E[2]{};
  DevCounters* d_ctr = nullptr;
  unsigned long long* st = nullptr;
};

struct Exchanger {
  virtual ~Exchanger() = default;
  virtual void min_u64(std::vector<Shard>& sh, unsigned long long* Shard::*buf, uint64_t count) = 0;
  virtual void min_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) = 0;
  virtual void sum_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) = 0;
};

// All shards on one device, one stream: an element-wise min kernel.
struct EmulatedExchanger : Exchanger {
  template <class T, bool kSum = false>
  static void run(std::vector<Shard>& sh, T* Shard::*buf, uint64_t count) {
    if (sh.size() == 1 || count == 0) return;
    ShardPtrs<T, 8> p{};
    for (size_t i = 0; i < sh.size(); ++i) p.p[i] = sh[i].*buf;
    ++t_launches;
    k_shard_min<T, kSum><<<(unsigned)std::min<uint64_t>((count + 255) / 256, 4096), 256, 0, sh[0].ws->stream>>>(
        p, (int)sh.size(), count);
    MST_CUDA_CHECK(cudaGetLastError());
  }
  void min_u64(std::vector<Shard>& sh, unsigned long long* Shard::*buf, uint64_t count) override {
    run(sh, buf, count);
  }
  void min_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) override { run(sh, buf, count); }
  void sum_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) override {
    run<uint32_t, true>(sh, buf, count);
  }
};

// NCCL: one communicator per shard (single process driving several GPUs via
// ncclCommInitAll, or one rank per process via ncclCommInitRank).
struct NcclExchanger : Exchanger {
  std::vector<ncclComm_t> comms;
  template <class T>
  void run(std::vector<Shard>& sh, T* Shard::*buf, uint64_t count, ncclDataType_t type, ncclRedOp_t op = ncclMin) {
    if (count == 0) return;
    MST_NCCL_CHECK(nccl().GroupStart());
    for (size_t i = 0; i < sh.size(); ++i) {
      MST_CUDA_CHECK(cudaSetDevice(sh[i].ws->device));
      T* p = sh[i].*buf;
      MST_NCCL_CHECK(nccl().AllReduce(p, p, count, type, op, comms[i], sh[i].ws->stream));
    }
    MST_NCCL_CHECK(nccl().GroupEnd());
  }
  void min_u64(std::vector<Shard>& sh, unsigned long long* Shard::*buf, uint64_t count) override {
    run(sh, buf, count, ncclUint64);
  }
  void min_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) override {
    run(sh, buf, count, ncclUint32);
  }
  void sum_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) override {
    run(sh, buf, count, ncclUint32, ncclSum);
  }
};

// A caller-supplied collective (mst_collective_t: MPI, gloo, a test
// harness): each exchange is staged through pinned host memory, reduced by
// the callback in place across the ranks, and copied back. One local shard.
struct CallbackExchanger : Exchanger {
  mst_collective_t coll{};
  void* host = nullptr;
  size_t host_bytes = 0;
  ~CallbackExchanger() override {
    if (host) cudaFreeHost(host);
  }
  template <class T>
  void run(std::vector<Shard>& sh, T* Shard::*buf, uint64_t count, int dtype, int op) {
    if (count == 0) return;
    Shard& s = sh.at(0);
    const size_t bytes = count * sizeof(T);
    if (bytes > host_bytes) {
      MST_CUDA_CHECK(cudaStreamSynchronize(s.ws->stream));
      if (host) MST_CUDA_CHECK(cudaFreeHost(host));
      host = nullptr;
      host_bytes = 0;
      MST_CUDA_CHECK(cudaMallocHost(&host, bytes));
      host_bytes = bytes;
    }
    MST_CUDA_CHECK(cudaMemcpyAsync(host, s.*buf, bytes, cudaMemcpyDeviceToHost, s.ws->stream));
    MST_CUDA_CHECK(cudaStreamSynchronize(s.ws->stream));
    const int rc = coll.allreduce(coll.ctx, host, count, dtype, op);
    if (rc != 0)
      throw MstError{MST_ERR_NCCL, "collective callback failed with status " + std::to_string(rc)};
    MST_CUDA_CHECK(cudaMemcpyAsync(s.*buf, host, bytes, cudaMemcpyHostToDevice, s.ws->stream));
  }
  void min_u64(std::vector<Shard>& sh, unsigned long long* Shard::*buf, uint64_t count) override {
    run(sh, buf, count, MST_DTYPE_U64, MST_OP_MIN);
  }
  void min_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) override {
    run(sh, buf, count, MST_DTYPE_U32, MST_OP_MIN);
  }
  void sum_u32(std::vector<Shard>& sh, uint32_t* Shard::*buf, uint64_t count) override {
    run(sh, buf, count, MST_DTYPE_U32, MST_OP_SUM);
  }
};

// NCCL communicators of the single-process multi-GPU entry, created once per
// GPU count and kept for the life of the process (ncclCommInitAll costs
// hundreds of milliseconds).
std::vector<ncclComm_t>& cached_comms(int num_gpus) {
  static std::mutex mu;
  static std::map<int, std::vector<ncclComm_t>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto& c = cache[num_gpus];
  if (c.empty()) {
    std::vector<ncclComm_t> comms(num_gpus);
    std::vector<int> devs(num_gpus);
    for (int i = 0; i < num_gpus; ++i) devs[i] = i;
    MST_NCCL_CHECK(nccl().CommInitAll(comms.data(), num_gpus, devs.data()));
    c = comms;
  }
  return c;
}

// The sharded loop (kernels.cuh "sharded exchange"). With filter, the
// Filter-Borůvka phases run sharded too: the weight histograms are summed
// across shards so every shard picks the same pivot, each shard splits and
// later filters its own edges, and the light-phase relabel maps are
// replicated like every other piece of component state.
void run_sharded_rounds(std::vector<Shard>& sh, Exchanger& ex, uint32_t n, uint64_t m_total, bool filter,
                        RunOut& out) {
  const int G = (int)sh.size();
  uint32_t launches = 0;
  for (auto& s : sh) {
    MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
    init_counters(*s.ws, s.d_ctr, n, s.m);
    MST_CUDA_CHECK(cudaMemsetAsync(s.minb[0], 0xFF, (size_t)n * 8, s.ws->stream));
    MST_CUDA_CHECK(cudaMemsetAsync(s.flags, 0, mst_bits_words(m_total) * 4, s.ws->stream));
    s.ret.init(*s.ws, n, filter && knob_i(kKnobRetire) != 0 && n < (1u << 31));
  }
  if (filter) {
    // pivot from the summed histogram of every shard's weight sample
    const uint64_t total_samples_target = std::min<uint64_t>(m_total, 1u << 20);
    for (auto& s : sh) {
      MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
      s.hist = s.ws->get<uint32_t>("hist", 65536);
      MST_CUDA_CHECK(cudaMemsetAsync(s.hist, 0, 65536 * sizeof(uint32_t), s.ws->stream));
      const uint32_t samples = (uint32_t)std::min<uint64_t>(
          s.m, std::max<uint64_t>(1, total_samples_target * s.m / std::max<uint64_t>(m_total, 1)));
      if (s.m) {
        const uint64_t step = std::max<uint64_t>(1, s.m / samples);
        launch_k(k_weight_hist, std::max(1u, samples / 1024), 256, s.ws->stream, s.in.w, 1u, s.m, step, samples, s.hist);
      }
    }
    ex.sum_u32(sh, &Shard::hist, 65536);
    const double beta = knob(kKnobFilterBeta);
    const double frac = std::min(1.0, beta * (double)n / (double)std::max<uint64_t>(m_total, 1));
    for (auto& s : sh) {
      MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
      Workspace& ws = *s.ws;
      // the target comes from the summed histogram's total (k_pick_pivot),
      // identical on every rank
      launch_k(k_pick_pivot, 1, 1024, ws.stream, s.hist, frac, s.d_ctr);
      const CompactBufs cb{ws.get<uint32_t>("tile_counts", tiles_c(s.m)),
                           ws.get<uint32_t>("tile_masks", tiles_c(s.m) * kCItems * kWarps), s.st,
                           ws.get<uint4>("stage", tiles_c(s.m) * kCTile)};
      launch_two_pass<SoaView, kModeLight>(ws, cb, s.in, nullptr, nullptr, s.E[1], s.minb[0], s.d_ctr, 0, s.m, n,
                                           kSlotCompact, (int)kPhaseSharded, filt_for(n, kSiteSplit),
                                           PairTable{nullptr, 0}, true, nullptr, n);
      launches += 4;
    }
  } else {
    for (auto& s : sh) {
      MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
      auto kmin = k_min_round1<SoaView>;
      launch_k(kmin, persistent_grid(kmin, s.ws->device, (s.m + kBlock - 1) / kBlock), kBlock, s.ws->stream, s.in, n, (uint64_t)0,
               s.m, s.minb[0], s.d_ctr, filt_for(n, kSiteMin1));
      ++launches;
    }
  }
  // errors (range / weight) are checked before the first key exchange, and
  // summed across ranks first: a rank whose own slice is bad must not leave
  // while the others wait in the collective
  for (auto& s : sh) {
    MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
    s.errw = s.ws->get<uint32_t>("errw", 2);
    launch_k(k_err_words, 1, 32, s.ws->stream, (const DevCounters*)s.d_ctr, s.errw);
  }
  ex.sum_u32(sh, &Shard::errw, 2);
  for (auto& s : sh) {
    MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
    uint32_t* h = reinterpret_cast<uint32_t*>(&s.ws->h_snap[0]);
    MST_CUDA_CHECK(cudaMemcpyAsync(h, s.errw, 8, cudaMemcpyDeviceToHost, s.ws->stream));
    MST_CUDA_CHECK(cudaStreamSynchronize(s.ws->stream));
    const uint32_t err = (h[0] ? kErrRange : 0u) | (h[1] ? kErrWeight : 0u);
    if (err) out.err = err;
  }
  if (out.err) return;
  bool light = filter;
  int R1 = 0;                  // first round after the heavy filter
  int loop_start = 1;
  std::vector<int> levels;     // light rounds whose relabel map ("Llvl<r>") is kept
  // The host runs one round ahead of the devices, as in the single-device
  // loop: round r is enqueued with bounds from round r-2's counters (n and
  // each shard's m only shrink), then round r-1's counters are read. The
  // verdicts are replicated (same hook on the same all-reduced keys), so every
  // rank takes the same branch and enqueues the same collectives; kernels of
  // rounds past a stop or a light-phase end exit on the device counters, and
  // an exchange whose count exceeds n_r only reduces entries nobody reads.
  uint64_t n_bound = n;
  std::vector<uint64_t> m_bound(G);
  for (int g = 0; g < G; ++g) m_bound[g] = sh[g].m;
  int r = 1;
  while (true) {
    if (r >= MST_MAX_ROUNDS) throw MstError{MST_ERR_STALL, "no convergence within MST_MAX_ROUNDS rounds"};
    // 1. local literal keys -> (w, global id) keys + owned partners; exchange.
    // The keys index the list named by the single-device rule (run_single_impl
    // hook_src).
    for (auto& s : sh) {
      MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
      const uint64_t t = (n_bound + kBlock - 1) / kBlock;
      unsigned long long* mcur = s.minb[(r - 1) & 1];
      auto keys = [&](auto view) {
        auto kk = k_shard_keys<decltype(view)>;
        launch_k(kk, persistent_grid(kk, s.ws->device, t), kBlock, s.ws->stream, view, mcur, s.xch, s.own, s.d_ctr, r);
      };
      if (r == 1 && !filter)
        keys(s.in);
      else if (r == 1)
        keys(PackedView{s.E[1]});
      else if (r == R1)
        keys(PackedView{s.E[r & 1]});
      else if (r == 2 && !filter)
        keys(PairsView<SoaView>{reinterpret_cast<const uint2*>(s.E[1]), s.in});
      else
        keys(PackedView{s.E[(r - 1) & 1]});
    }
    ex.min_u64(sh, &Shard::xch, n_bound);
    for (auto& s : sh) {
      MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
      launch_k(k_shard_partner, persistent_grid(k_shard_partner, s.ws->device, (n_bound + kBlock - 1) / kBlock), kBlock,
               s.ws->stream, s.xch, s.own, s.partner, s.d_ctr, r);
    }
    ex.min_u32(sh, &Shard::partner, n_bound);
    launches += 2;
    // 2. replicated hook + label, local compaction (as the single-device loop)
    for (int g = 0; g < G; ++g) {
      Shard& s = sh[g];
      MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
      Workspace& ws = *s.ws;
      const int dev = ws.device;
      cudaStream_t st = ws.stream;
      const uint64_t ht = tiles_of(n_bound);
      const int hfused = ht <= kFusedScanMaxTiles ? 1 : 0;
      uint32_t* rb = light ? s.ret.take(st, r, n_bound) : nullptr;  // same decision on every shard
      const int phase = light ? (s.ret.active() ? (int)kPhaseLightRetire : (int)kPhaseLight) : (int)kPhasePlain;
      uint32_t* hcounts = ws.get<uint32_t>("hook_counts", tiles_of(n));
      uint32_t* hmasks = ws.get<uint32_t>("hook_masks", tiles_of(n) * kItems * kWarps);
      uint32_t* hslot = ws.get<uint32_t>("hook_slotpref", tiles_of(n) * kItems * kWarps);
      auto kd = k_hook_decide<PartnerView, true>;
      launch_k(kd, persistent_grid(kd, dev, ht), kBlock, st, PartnerView{s.partner}, s.xch, s.parent, hmasks,
               hcounts, s.d_ctr, r, hfused, phase, hslot, s.flags, 0, rb);
      if (!hfused)
        launch_k(k_scan_counts<kScanRoots>,
                 (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ht + kScanTile - 1) / kScanTile, (uint64_t)sm_count(dev))),
                 kScanBlock, st, hcounts, ht, s.d_ctr, r, s.st, ws.next_epoch(), phase, 0);
      unsigned long long* mnext = s.minb[r & 1];
      uint32_t* Lr = light ? ws.get<uint32_t>("Llvl" + std::to_string(r), n_bound) : s.L;
      launch_k(k_label2, persistent_grid(k_label2, dev, ht), kBlock, st, s.parent, hmasks, hslot, hcounts, Lr, mnext,
               s.d_ctr, r, (unsigned long long*)nullptr, 0ull, 0u, 4u | (8u << 16), (const uint32_t*)rb);
      const CompactBufs cb{ws.get<uint32_t>("tile_counts", tiles_c(s.m)),
                           ws.get<uint32_t>("tile_masks", tiles_c(s.m) * kCItems * kWarps), s.st,
                           ws.get<uint4>("stage", tiles_c(s.m) * kCTile)};
      uint4* Eout = s.E[(r + 1) & 1];
      if (r == 1 && !filter)
        launch_two_pass<SoaView, kModeRelabel>(ws, cb, s.in, s.E[1], Lr, Eout, mnext, s.d_ctr, r, m_bound[g], n,
                                               kSlotCompact, (int)kPhaseSharded, filt_for(n_bound, kSiteCount, filter));
      else
      {
        // giant bits for huge rounds (phase D's first): each shard picks its
        // own giant from its own list; any choice is exact
        const uint32_t* gb = nullptr;
        const double giant_min = knob(kKnobGiantBits);
        if (giant_min > 0 && !light && (double)n_bound >= giant_min && s.m) {
          uint32_t* bits = ws.get<uint32_t>("giant_bits", (n_bound + 31) / 32 + 1);
          launch_k(k_pick_giant, 1, 1024, st, (const uint4*)s.E[r & 1], (const uint32_t*)Lr, s.d_ctr, r);
          launch_k(k_giant_bits, (unsigned)(sm_count(dev) * 8), 256, st, (const uint32_t*)Lr,
                   (const DevCounters*)s.d_ctr, r, bits);
          gb = bits;
          launches += 2;
        }
        launch_two_pass<PackedView, kModeRelabel>(ws, cb, PackedView{s.E[r & 1]}, s.E[r & 1], Lr, Eout, mnext,
                                                  s.d_ctr, r, m_bound[g], n, kSlotCompact, (int)kPhaseSharded,
                                                  filt_for(n_bound, kSiteCount, filter), PairTable{nullptr, 0}, true,
                                                  gb);
      }
      launches += 5;
      MST_CUDA_CHECK(cudaGetLastError());
      MST_CUDA_CHECK(cudaMemcpyAsync(&ws.h_snap[r], s.d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
      MST_CUDA_CHECK(cudaEventRecord(ws.ev[r], st));
    }
    if (light) levels.push_back(r);
    if (r > loop_start) {
      // round r-1's verdict (identical on every shard: replicated hook)
      for (int g = 0; g < G; ++g) {
        MST_CUDA_CHECK(cudaEventSynchronize(sh[g].ws->ev[r - 1]));
        const DevCounters& a = sh[0].ws->h_snap[r - 1];
        const DevCounters& b = sh[g].ws->h_snap[r - 1];
        if (b.err) out.err |= b.err;
        if (b.stop_round != a.stop_round || b.phase_end != a.phase_end || b.n[r] != a.n[r])
          throw MstError{MST_ERR_STALL, "replicated hook diverged between shards"};
      }
      const DevCounters& snap = sh[0].ws->h_snap[r - 1];
      if (knob_i(kKnobDebugRounds))
        fprintf(stderr, "shard round %2d: n=%u light=%d stop=%d phase_end=%d m0=%llu\n", r - 1, snap.n[r - 1],
                (int)light, (int)snap.stop_round, (int)snap.phase_end, (unsigned long long)snap.m[r - 1]);
      if (out.err) break;
      if (snap.stop_round != kNoStop && (int)snap.stop_round <= r) break;
      if (light && snap.phase_end != kNoStop && (int)snap.phase_end <= r) {
        // light phase over (no light edge left between components)
        const int pe = (int)snap.phase_end;
        if (pe == 1) {
          // not a single light hook: the plain sharded loop instead
          for (auto& s : sh) {
            MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
            MST_CUDA_CHECK(cudaStreamSynchronize(s.ws->stream));
          }
          run_sharded_rounds(sh, ex, n, m_total, false, out);
          out.launches += launches;
          return;
        }
        while (!levels.empty() && levels.back() >= pe) levels.pop_back();
        R1 = pe;
        bool retired = false;
        for (auto& s : sh) {
          MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
          Workspace& ws = *s.ws;
          s.ret.drop_from(pe);
          retired = s.ret.active() && !levels.empty();
          if (retired) {
            std::vector<std::pair<uint32_t*, int>> lv;
            for (int lr : levels) lv.push_back({ws.get<uint32_t>("Llvl" + std::to_string(lr), 1), lr});
            launches += s.ret.finalize(ws, ws.stream, s.d_ctr, pe, lv, snap, s.minb[(pe - 1) & 1]);
          } else {
            for (int k = (int)levels.size() - 2; k >= 0; --k) {
              const unsigned gk = (unsigned)std::max<uint64_t>(
                  1, std::min<uint64_t>((snap.n[levels[k]] + 255) / 256, (uint64_t)sm_count(ws.device) * 8));
              launch_k(k_compose, gk, 256, ws.stream, ws.get<uint32_t>("Llvl" + std::to_string(levels[k]), 1),
                       (const uint32_t*)ws.get<uint32_t>("Llvl" + std::to_string(levels[k + 1]), 1), s.d_ctr, levels[k]);
              ++launches;
            }
          }
          MST_CUDA_CHECK(cudaMemsetAsync(&s.d_ctr->phase_end, 0xFF, sizeof(unsigned int), ws.stream));
        }
        // after retirement n[R1] exists on the devices only (identical on every shard)
        const uint64_t n_heavy = retired ? read_count(*sh[0].ws, sh[0].ws->stream, sh[0].d_ctr, R1) : snap.n[R1];
        for (auto& s : sh) {
          MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
          Workspace& ws = *s.ws;
          const uint32_t* vlabel = levels.empty() ? nullptr : ws.get<uint32_t>("Llvl" + std::to_string(levels[0]), 1);
          const CompactBufs cb{ws.get<uint32_t>("tile_counts", tiles_c(s.m)),
                               ws.get<uint32_t>("tile_masks", tiles_c(s.m) * kCItems * kWarps), s.st,
                               ws.get<uint4>("stage", tiles_c(s.m) * kCTile)};
          // launched as round R1-1's producer: m[R1], E and the min table of round R1
          launch_two_pass<SoaView, kModeHeavy>(ws, cb, s.in, nullptr, vlabel, s.E[R1 & 1], s.minb[(R1 - 1) & 1],
                                               s.d_ctr, R1 - 1, s.m, n, kSlotFilter, (int)kPhaseSharded,
                                               filt_for(snap.n[R1], kSiteHeavy), PairTable{nullptr, 0}, true,
                                               nullptr, n_heavy);
          launches += 2;
        }
        light = false;
        n_bound = n_heavy;
        for (int g = 0; g < G; ++g) m_bound[g] = sh[g].m;
        r = R1;
        loop_start = R1;
        continue;
      }
      n_bound = snap.n[r];
      for (int g = 0; g < G; ++g) m_bound[g] = sh[g].ws->h_snap[r - 1].m[r];
    }
    ++r;
  }
  for (auto& s : sh) {
    MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
    MST_CUDA_CHECK(cudaStreamSynchronize(s.ws->stream));
  }
  DevCounters c;
  MST_CUDA_CHECK(cudaSetDevice(sh[0].ws->device));
  MST_CUDA_CHECK(cudaMemcpy(&c, sh[0].d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost));
  out.ctr = c;
  // per-shard kept counts differ; report the sum over shards as m_r
  for (int g = 1; g < G; ++g) {
    DevCounters cg;
    MST_CUDA_CHECK(cudaSetDevice(sh[g].ws->device));
    MST_CUDA_CHECK(cudaMemcpy(&cg, sh[g].d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost));
    for (int r2 = 1; r2 < kMaxR; ++r2) out.ctr.m[r2] += cg.m[r2];
    out.err |= cg.err;
  }
  out.err |= c.err;
  out.launches = launches;
  if (out.err) return;
  if (c.stop_round == kNoStop) throw MstError{MST_ERR_STALL, "sharded loop ended without a stop verdict"};
  const int stop = (int)c.stop_round;
  out.rounds = (uint32_t)stop - 1;
  out.phase_end = (uint32_t)R1;
  out.final_components = c.n[stop];
  out.count = (uint64_t)n - out.final_components;
  out.total_weight = c.total_weight;
}

// Shared driver for emulated / single-process multi-GPU / one-rank-per-process.
// `parts` gives each local shard's (device, slot, src, dst, w, m, base).
struct PartSpec {
  int device, slot;
  const uint32_t *src, *dst, *w;
  uint64_t m;
  uint32_t base;
  int on_device;
};

// device_out: the sorted ids stay in HBM (out_ids is a device pointer on the
// first shard's device). user_stream (one local shard only): run on the
// caller's stream; nullptr with device input or output joins the legacy
// stream 0 both ways (see run_single).
RunOut run_sharded(const std::vector<PartSpec>& parts, Exchanger& ex, uint32_t n, uint64_t m_total,
                   uint32_t* out_ids, mst_stats_t* stats, bool device_out = false,
                   cudaStream_t user_stream = nullptr) {
  const auto t_start = Clock::now();
  const uint64_t launches0 = t_launches;
  std::vector<Shard> sh(parts.size());
  std::vector<std::unique_lock<std::mutex>> locks;
  struct Restore {
    Workspace* w = nullptr;
    cudaStream_t s = nullptr;
    ~Restore() {
      if (w) w->stream = s;
    }
  } restore;
  bool join_legacy = false;
  for (size_t i = 0; i < parts.size(); ++i) {
    Workspace& ws = workspace(parts[i].device, parts[i].slot);
    locks.emplace_back(ws.mu);
    MST_CUDA_CHECK(cudaSetDevice(ws.device));
    if (i == 0 && parts.size() == 1) {
      if (user_stream) {
        restore.w = &ws;
        restore.s = ws.stream;
        ws.stream = user_stream;
      } else if (parts[0].on_device || device_out) {
        join_legacy = true;
        MST_CUDA_CHECK(cudaEventRecord(ws.join_in, cudaStreamLegacy));
        MST_CUDA_CHECK(cudaStreamWaitEvent(ws.stream, ws.join_in, 0));
      }
    }
    Shard& s = sh[i];
    s.ws = &ws;
    s.m = parts[i].m;
    s.base = parts[i].base;
    const uint32_t* src = parts[i].src;
    const uint32_t* dst = parts[i].dst;
    const uint32_t* w = parts[i].w;
    if (!parts[i].on_device && s.m) {
      uint32_t* d_src = ws.get<uint32_t>("in_src", s.m);
      uint32_t* d_dst = ws.get<uint32_t>("in_dst", s.m);
      uint32_t* d_w = ws.get<uint32_t>("in_w", s.m);
      copy_h2d(ws, d_src, src, s.m * 4);
      copy_h2d(ws, d_dst, dst, s.m * 4);
      copy_h2d(ws, d_w, w, s.m * 4);
      src = d_src;
      dst = d_dst;
      w = d_w;
    }
    s.in = SoaView{src, dst, w, s.base};
    s.minb[0] = ws.get<unsigned long long>("minA", n);
    s.minb[1] = ws.get<unsigned long long>("minB", n);
    s.xch = ws.get<unsigned long long>("xch", n);
    s.own = ws.get<unsigned long long>("own", n);
    s.parent = ws.get<uint32_t>("parent", n);
    s.L = ws.get<uint32_t>("label", n);
    s.partner = ws.get<uint32_t>("partner", n);
    s.flags = ws.get<uint32_t>("mst_bits", mst_bits_words(m_total));
    s.E[0] = ws.get<uint4>("E0", s.m);
    s.E[1] = ws.get<uint4>("E1", s.m);
    s.d_ctr = ws.get<DevCounters>("ctr", 1);
    s.st = ws.status_array(std::max(tiles_of(s.m), tiles_of(n)));
  }
  MST_CUDA_CHECK(cudaSetDevice(sh[0].ws->device));
  cudaEvent_t e1 = sh[0].ws->tev[sh[0].ws->tev.size() - 3];
  cudaEvent_t e2 = sh[0].ws->tev[sh[0].ws->tev.size() - 2];
  MST_CUDA_CHECK(cudaEventRecord(e1, sh[0].ws->stream));
  RunOut o;
  run_sharded_rounds(sh, ex, n, m_total, filter_mode(n, m_total), o);
  check_err_bits(o.err);
  Workspace& ws0 = *sh[0].ws;
  MST_CUDA_CHECK(cudaSetDevice(ws0.device));
  uint32_t* d_sorted = device_out ? out_ids : ws0.get<uint32_t>("sorted", n);
  sort_from_bits(ws0, sh[0].flags, std::max<uint64_t>(m_total, 1), d_sorted, sh[0].d_ctr);
  o.launches = (uint32_t)(t_launches - launches0);  // every kernel of the call (all shards), counted at launch
  MST_CUDA_CHECK(cudaEventRecord(e2, ws0.stream));
  if (o.count && out_ids && !device_out)
    copy_d2h(ws0, out_ids, d_sorted, o.count * 4);
  if (join_legacy) {
    MST_CUDA_CHECK(cudaEventRecord(ws0.join_out, ws0.stream));
    MST_CUDA_CHECK(cudaStreamWaitEvent(cudaStreamLegacy, ws0.join_out, 0));
  }
  for (auto& s : sh) {
    MST_CUDA_CHECK(cudaSetDevice(s.ws->device));
    MST_CUDA_CHECK(cudaStreamSynchronize(s.ws->stream));
  }
  if (stats) {
    fill_stats(stats, o);
    stats->ms_device = ms_between(e1, e2);
    stats->ms_h2d = 0;
    stats->ms_d2h = 0;
    stats->ms_total = std::chrono::duration<double, std::milli>(Clock::now() - t_start).count();
  }
  return o;
}

int finish_status(const RunOut& o, uint64_t* out_count, uint64_t* out_total) {
  if (out_count) *out_count = o.count;
  if (out_total) *out_total = o.total_weight;
  if (o.final_components > 1) {
    set_last_error("disconnected: " + std::to_string(o.final_components) +
                   " components (a minimum spanning forest was returned)");
    return MST_ERR_DISCONNECTED;
  }
  set_last_error("");
  return MST_OK;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const MstError& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(std::string("internal error: ") + e.what());
    return MST_ERR_CUDA;
  }
}

}  // namespace

struct CommImpl {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

}  // namespace mstgpu

using namespace mstgpu;

struct mst_comm {
  CommImpl impl;
};

namespace mstgpu {
namespace {

// verify.cuh: range, count, acyclic/spanning by a private concurrent
// union-find, weight sum, and (with an oracle) weight + edge-set equality.
// make_view(ws) stages host edges into verifier-private buffers (under the
// same workspace lock as everything below) and returns the device view.
template <class MakeView>
void run_verify(MakeView make_view, uint32_t n, uint64_t m, int on_device, const uint32_t* ids, uint64_t count,
                const uint32_t* oracle_ids, uint64_t oracle_count, uint64_t oracle_total, mst_verify_t* out) {
  const int dev = current_device_checked();
  Workspace& ws = workspace(dev, 0);
  std::lock_guard<std::mutex> lock(ws.mu);
  MST_CUDA_CHECK(cudaSetDevice(dev));
  cudaStream_t s = ws.stream;
  const auto g = make_view(ws);
  if (!on_device) {
    if (count) {
      uint32_t* d = ws.get<uint32_t>("v_ids", count);
      copy_h2d(ws, d, ids, count * 4);
      ids = d;
    }
    if (oracle_ids && oracle_count) {
      uint32_t* d = ws.get<uint32_t>("v_oracle", oracle_count);
      copy_h2d(ws, d, oracle_ids, oracle_count * 4);
      oracle_ids = d;
    }
  }
  const bool with_oracle = oracle_total != MST_VERIFY_NO_ORACLE;
  const uint64_t words4 = (m + 127) / 128;
  uint32_t* parent = ws.get<uint32_t>("v_parent", n);
  auto* ctr = ws.get<VerifyCounters>("v_ctr", 1);
  uint32_t* bits_got = with_oracle ? reinterpret_cast<uint32_t*>(ws.get<uint4>("v_bits_got", std::max<uint64_t>(words4, 1))) : nullptr;
  uint32_t* bits_ora = with_oracle ? reinterpret_cast<uint32_t*>(ws.get<uint4>("v_bits_ora", std::max<uint64_t>(words4, 1))) : nullptr;
  MST_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(VerifyCounters), s));
  if (with_oracle) {
    MST_CUDA_CHECK(cudaMemsetAsync(bits_got, 0, std::max<uint64_t>(words4, 1) * 16, s));
    MST_CUDA_CHECK(cudaMemsetAsync(bits_ora, 0, std::max<uint64_t>(words4, 1) * 16, s));
  }
  const unsigned grid = (unsigned)sm_count(dev) * 8;
  kv_iota<<<grid, 256, 0, s>>>(parent, n);
  if (count) kv_unite<<<grid, 256, 0, s>>>(g, n, m, ids, count, parent, bits_got, ctr);
  if (with_oracle) {
    if (oracle_count) kv_mark<<<grid, 256, 0, s>>>(oracle_ids, oracle_count, m, bits_ora, ctr);
    if (words4)
      kv_compare<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(bits_got), reinterpret_cast<const uint4*>(bits_ora),
                                      words4, ctr);
  }
  MST_CUDA_CHECK(cudaGetLastError());
  VerifyCounters h{};
  MST_CUDA_CHECK(cudaMemcpyAsync(&h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  MST_CUDA_CHECK(cudaStreamSynchronize(s));
  if (h.range_err & 1u) throw MstError{MST_ERR_RANGE, "verify: an edge id lies outside [0, m)"};
  if (h.range_err & 2u) throw MstError{MST_ERR_RANGE, "verify: an edge endpoint lies outside [0, n)"};
  out->edge_count_ok = count == (uint64_t)n - 1;
  out->components = (uint64_t)n - h.unions;
  out->is_acyclic = h.unions == count;
  out->is_spanning = out->components == 1;
  out->weight = h.weight;
  out->weight_matches_oracle = with_oracle ? (h.weight == oracle_total) : -1;
  out->edge_set_matches_oracle = with_oracle ? (!h.set_mismatch && count == oracle_count) : -1;
}

}  // namespace
}  // namespace mstgpu

extern "C" {

const char* mst_gpu_last_error(void) { return t_last_error.c_str(); }

const char* mst_gpu_version(void) { return "paper_2005_06913_b200 0.1 (sm_100a)"; }

int mst_gpu_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

int mst_gpu_boruvka(const mst_edges_soa_t* edges, int num_gpus, uint32_t* out_ids,
                    uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats) {
  return guarded([&]() -> int {
    if (!edges) throw MstError{MST_ERR_INVALID_ARG, "edges is NULL"};
    validate_common(edges->n, edges->m);
    if (num_gpus < 1 || num_gpus > 8) throw MstError{MST_ERR_INVALID_ARG, "num_gpus must be in [1,8]"};
    if (edges->m && (!edges->src || !edges->dst || !edges->w))
      throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    if (edges->n > 1 && !out_ids) throw MstError{MST_ERR_INVALID_ARG, "out_ids is NULL"};
    if (num_gpus > 1 && edges->on_device)
      throw MstError{MST_ERR_INVALID_ARG, "device input requires num_gpus == 1"};
    const int dev = current_device_checked();
    if (num_gpus == 1) {
      SingleArgs a{edges->n, edges->m, 0, edges->src, edges->dst, edges->w, nullptr,
                   edges->on_device, out_ids, false, nullptr, false};
      RunOut o = run_single(a, stats);
      return finish_status(o, out_count, out_total_weight);
    }
    int count = 0;
    MST_CUDA_CHECK(cudaGetDeviceCount(&count));
    if (count < num_gpus)
      throw MstError{MST_ERR_INVALID_ARG, "num_gpus=" + std::to_string(num_gpus) + " but only " +
                                              std::to_string(count) + " devices are visible"};
    (void)dev;
    NcclExchanger ex;
    ex.comms = cached_comms(num_gpus);
    std::vector<PartSpec> parts;
    for (int g = 0; g < num_gpus; ++g) {
      const uint64_t lo = edges->m * g / num_gpus, hi = edges->m * (g + 1) / num_gpus;
      parts.push_back(PartSpec{g, 0, edges->src + lo, edges->dst + lo, edges->w + lo, hi - lo, (uint32_t)lo, 0});
    }
    RunOut o = run_sharded(parts, ex, edges->n, edges->m, out_ids, stats);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_boruvka_aos(uint32_t n, uint64_t m, const mst_edge_t* edges, int on_device,
                        uint32_t* out_ids, uint64_t* out_count, uint64_t* out_total_weight,
                        mst_stats_t* stats) {
  return guarded([&]() -> int {
    validate_common(n, m);
    if (m && !edges) throw MstError{MST_ERR_INVALID_ARG, "edges is NULL"};
    if (n > 1 && !out_ids) throw MstError{MST_ERR_INVALID_ARG, "out_ids is NULL"};
    current_device_checked();
    SingleArgs a{n, m, 1, nullptr, nullptr, nullptr, edges, on_device, out_ids, false, nullptr, false};
    RunOut o = run_single(a, stats);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_boruvka_emulated(const mst_edges_soa_t* edges, int num_shards, uint32_t* out_ids,
                             uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats) {
  return guarded([&]() -> int {
    if (!edges) throw MstError{MST_ERR_INVALID_ARG, "edges is NULL"};
    validate_common(edges->n, edges->m);
    if (num_shards < 1 || num_shards > 8) throw MstError{MST_ERR_INVALID_ARG, "num_shards must be in [1,8]"};
    if (edges->m && (!edges->src || !edges->dst || !edges->w))
      throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    if (edges->n > 1 && !out_ids) throw MstError{MST_ERR_INVALID_ARG, "out_ids is NULL"};
    const int dev = current_device_checked();
    // every emulated shard shares the first shard's stream (serial, one device)
    Workspace& ws0 = workspace(dev, 1);
    std::vector<PartSpec> parts;
    for (int g = 0; g < num_shards; ++g) {
      const uint64_t lo = edges->m * g / num_shards, hi = edges->m * (g + 1) / num_shards;
      parts.push_back(PartSpec{dev, 1 + g, edges->src + lo, edges->dst + lo, edges->w + lo, hi - lo,
                               (uint32_t)lo, edges->on_device});
      Workspace& wsg = workspace(dev, 1 + g);
      if (g > 0) {
        std::lock_guard<std::mutex> lk(wsg.mu);
        wsg.stream = ws0.stream;
      }
    }
    EmulatedExchanger ex;
    RunOut o = run_sharded(parts, ex, edges->n, edges->m, out_ids, stats);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_verify(const mst_edges_soa_t* edges, const uint32_t* ids, uint64_t count, const uint32_t* oracle_ids,
                   uint64_t oracle_count, uint64_t oracle_total, mst_verify_t* report) {
  return guarded([&]() -> int {
    if (!edges || !report) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    validate_common(edges->n, edges->m);
    if (edges->m && (!edges->src || !edges->dst || !edges->w))
      throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    if (count && !ids) throw MstError{MST_ERR_INVALID_ARG, "ids is NULL"};
    if (oracle_count && !oracle_ids) throw MstError{MST_ERR_INVALID_ARG, "oracle_ids is NULL"};
    current_device_checked();
    auto make_view = [&](Workspace& ws) {
      const uint32_t *src = edges->src, *dst = edges->dst, *w = edges->w;
      if (!edges->on_device && edges->m) {
        uint32_t* d_src = ws.get<uint32_t>("v_src", edges->m);
        uint32_t* d_dst = ws.get<uint32_t>("v_dst", edges->m);
        uint32_t* d_w = ws.get<uint32_t>("v_w", edges->m);
        copy_h2d(ws, d_src, src, edges->m * 4);
        copy_h2d(ws, d_dst, dst, edges->m * 4);
        copy_h2d(ws, d_w, w, edges->m * 4);
        src = d_src;
        dst = d_dst;
        w = d_w;
      }
      return VSoa{src, dst, w};
    };
    run_verify(make_view, edges->n, edges->m, edges->on_device, ids, count, oracle_ids, oracle_count,
               oracle_total, report);
    set_last_error("");
    return MST_OK;
  });
}

int mst_gpu_verify_aos(uint32_t n, uint64_t m, const mst_edge_t* edges, int on_device, const uint32_t* ids,
                       uint64_t count, const uint32_t* oracle_ids, uint64_t oracle_count, uint64_t oracle_total,
                       mst_verify_t* report) {
  return guarded([&]() -> int {
    if (!report) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    validate_common(n, m);
    if (m && !edges) throw MstError{MST_ERR_INVALID_ARG, "edges is NULL"};
    if (count && !ids) throw MstError{MST_ERR_INVALID_ARG, "ids is NULL"};
    if (oracle_count && !oracle_ids) throw MstError{MST_ERR_INVALID_ARG, "oracle_ids is NULL"};
    current_device_checked();
    auto make_view = [&](Workspace& ws) {
      const uint4* e4 = reinterpret_cast<const uint4*>(edges);
      if (!on_device && m) {
        uint4* d = ws.get<uint4>("v_aos", m);
        copy_h2d(ws, d, e4, m * 16);
        e4 = d;
      }
      return VAos{e4};
    };
    run_verify(make_view, n, m, on_device, ids, count, oracle_ids, oracle_count, oracle_total, report);
    set_last_error("");
    return MST_OK;
  });
}

int mst_comm_unique_id(uint8_t out_id[MST_UNIQUE_ID_BYTES]) {
  return guarded([&]() -> int {
    if (!out_id) throw MstError{MST_ERR_INVALID_ARG, "out_id is NULL"};
    ncclUniqueId id;
    MST_NCCL_CHECK(nccl().GetUniqueId(&id));
    std::memcpy(out_id, id.internal, MST_UNIQUE_ID_BYTES);
    return MST_OK;
  });
}

int mst_comm_init(const uint8_t id[MST_UNIQUE_ID_BYTES], int nranks, int rank, int device,
                  mst_comm_t* out_comm) {
  return guarded([&]() -> int {
    if (!id || !out_comm) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    if (nranks < 1 || rank < 0 || rank >= nranks) throw MstError{MST_ERR_INVALID_ARG, "bad rank/nranks"};
    current_device_checked();
    MST_CUDA_CHECK(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, MST_UNIQUE_ID_BYTES);
    auto* c = new mst_comm;
    c->impl.nranks = nranks;
    c->impl.rank = rank;
    c->impl.device = device;
    ncclResult_t r = nccl().CommInitRank(&c->impl.comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      throw MstError{MST_ERR_NCCL, std::string("ncclCommInitRank failed: ") + nccl().GetErrorString(r)};
    }
    *out_comm = c;
    return MST_OK;
  });
}

int mst_comm_destroy(mst_comm_t comm) {
  return guarded([&]() -> int {
    if (!comm) return MST_OK;
    if (comm->impl.comm) nccl().CommDestroy(comm->impl.comm);
    delete comm;
    return MST_OK;
  });
}

int mst_gpu_boruvka_rank(mst_comm_t comm, uint32_t n, uint64_t m_total, uint64_t shard_base,
                         uint64_t shard_m, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                         int on_device, uint32_t* out_ids, uint64_t* out_count,
                         uint64_t* out_total_weight, mst_stats_t* stats) {
  return guarded([&]() -> int {
    if (!comm) throw MstError{MST_ERR_INVALID_ARG, "comm is NULL"};
    validate_common(n, m_total);
    if (shard_base + shard_m > m_total) throw MstError{MST_ERR_INVALID_ARG, "shard outside [0, m_total)"};
    if (shard_m && (!src || !dst || !w)) throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    if (n > 1 && !out_ids) throw MstError{MST_ERR_INVALID_ARG, "out_ids is NULL"};
    current_device_checked();
    MST_CUDA_CHECK(cudaSetDevice(comm->impl.device));
    NcclExchanger ex;
    ex.comms = {comm->impl.comm};
    std::vector<PartSpec> parts{
        PartSpec{comm->impl.device, 0, src, dst, w, shard_m, (uint32_t)shard_base, on_device}};
    RunOut o = run_sharded(parts, ex, n, m_total, out_ids, stats);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_boruvka_rank_device(mst_comm_t comm, uint32_t n, uint64_t m_total, uint64_t shard_base,
                                uint64_t shard_m, const uint32_t* d_src, const uint32_t* d_dst, const uint32_t* d_w,
                                uint32_t* d_out_ids, void* stream, uint64_t* out_count, uint64_t* out_total_weight,
                                mst_stats_t* stats) {
  return guarded([&]() -> int {
    if (!comm || !d_out_ids) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    validate_common(n, m_total);
    if (shard_base + shard_m > m_total) throw MstError{MST_ERR_INVALID_ARG, "shard outside [0, m_total)"};
    if (shard_m && (!d_src || !d_dst || !d_w)) throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    current_device_checked();
    MST_CUDA_CHECK(cudaSetDevice(comm->impl.device));
    NcclExchanger ex;
    ex.comms = {comm->impl.comm};
    std::vector<PartSpec> parts{
        PartSpec{comm->impl.device, 0, d_src, d_dst, d_w, shard_m, (uint32_t)shard_base, 1}};
    RunOut o = run_sharded(parts, ex, n, m_total, d_out_ids, stats, true, (cudaStream_t)stream);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_boruvka_rank_cb(const mst_collective_t* coll, uint32_t n, uint64_t m_total, uint64_t shard_base,
                            uint64_t shard_m, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                            int on_device, uint32_t* out_ids, uint64_t* out_count, uint64_t* out_total_weight,
                            mst_stats_t* stats) {
  return guarded([&]() -> int {
    if (!coll || !coll->allreduce) throw MstError{MST_ERR_INVALID_ARG, "collective is NULL"};
    if (coll->nranks < 1 || coll->rank < 0 || coll->rank >= coll->nranks)
      throw MstError{MST_ERR_INVALID_ARG, "bad rank/nranks"};
    validate_common(n, m_total);
    if (shard_base + shard_m > m_total) throw MstError{MST_ERR_INVALID_ARG, "shard outside [0, m_total)"};
    if (shard_m && (!src || !dst || !w)) throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    if (n > 1 && !out_ids) throw MstError{MST_ERR_INVALID_ARG, "out_ids is NULL"};
    current_device_checked();
    MST_CUDA_CHECK(cudaSetDevice(coll->device));
    CallbackExchanger ex;
    ex.coll = *coll;
    std::vector<PartSpec> parts{
        PartSpec{coll->device, 0, src, dst, w, shard_m, (uint32_t)shard_base, on_device}};
    RunOut o = run_sharded(parts, ex, n, m_total, out_ids, stats);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_boruvka_device(const mst_edges_soa_t* edges, uint32_t* d_out_ids, void* stream,
                           uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats,
                           double* ms_hot, uint32_t* hot_launches) {
  return guarded([&]() -> int {
    if (!edges || !d_out_ids) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    validate_common(edges->n, edges->m);
    if (!edges->on_device) throw MstError{MST_ERR_INVALID_ARG, "mst_gpu_boruvka_device needs device input"};
    current_device_checked();
    SingleArgs a{edges->n, edges->m, 0, edges->src, edges->dst, edges->w, nullptr, 1, d_out_ids, true,
                 (cudaStream_t)stream, ms_hot != nullptr};
    RunOut o = run_single(a, stats);
    if (ms_hot) *ms_hot = o.ms_hot;
    if (hot_launches) *hot_launches = o.hot_launches;
    if (stats) stats->hot_bytes = o.hot_bytes;
    if (stats) stats->alg_bytes = alg_bytes_from(o.ctr, o.rounds, o.phase_end);
    return finish_status(o, out_count, out_total_weight);
  });
}

int mst_gpu_round1_min(const mst_edges_soa_t* edges, uint64_t* out_min) {
  return guarded([&]() -> int {
    if (!edges || !out_min) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    validate_common(edges->n, edges->m);
    if (edges->m && (!edges->src || !edges->dst || !edges->w))
      throw MstError{MST_ERR_INVALID_ARG, "edge arrays are NULL"};
    const int dev = current_device_checked();
    Workspace& ws = workspace(dev, 0);
    std::lock_guard<std::mutex> lock(ws.mu);
    MST_CUDA_CHECK(cudaSetDevice(dev));
    const uint32_t n = edges->n;
    const uint64_t m = edges->m;
    const uint32_t *src = edges->src, *dst = edges->dst, *w = edges->w;
    if (!edges->on_device && m) {
      uint32_t* d_src = ws.get<uint32_t>("in_src", m);
      uint32_t* d_dst = ws.get<uint32_t>("in_dst", m);
      uint32_t* d_w = ws.get<uint32_t>("in_w", m);
      MST_CUDA_CHECK(cudaMemcpyAsync(d_src, src, m * 4, cudaMemcpyHostToDevice, ws.stream));
      MST_CUDA_CHECK(cudaMemcpyAsync(d_dst, dst, m * 4, cudaMemcpyHostToDevice, ws.stream));
      MST_CUDA_CHECK(cudaMemcpyAsync(d_w, w, m * 4, cudaMemcpyHostToDevice, ws.stream));
      src = d_src;
      dst = d_dst;
      w = d_w;
    }
    auto* d_ctr = ws.get<DevCounters>("ctr", 1);
    auto* mn = ws.get<unsigned long long>("minA", n);
    init_counters(ws, d_ctr, n, m);
    MST_CUDA_CHECK(cudaMemsetAsync(mn, 0xFF, (size_t)n * 8, ws.stream));
    auto kmin = k_min_round1<SoaView>;
    const unsigned g = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((m + 4 * kBlock - 1) / (4 * kBlock), (uint64_t)sm_count(dev) * blocks_per_sm(kmin)));
    kmin<<<g, kBlock, 0, ws.stream>>>(SoaView{src, dst, w, 0}, n, (uint64_t)0, m, mn, d_ctr, filt_for(n, kSiteMin1));
    MST_CUDA_CHECK(cudaGetLastError());
    MST_CUDA_CHECK(cudaMemcpyAsync(out_min, mn, (size_t)n * 8, cudaMemcpyDeviceToHost, ws.stream));
    MST_CUDA_CHECK(cudaMemcpyAsync(&ws.h_snap[0], d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost,
                                   ws.stream));
    MST_CUDA_CHECK(cudaStreamSynchronize(ws.stream));
    check_err_bits(ws.h_snap[0].err);
    return MST_OK;
  });
}

int mst_gpu_set_tuning(const char* name, double value) {
  return guarded([&]() -> int {
    if (!name) throw MstError{MST_ERR_INVALID_ARG, "tuning knob name is NULL"};
    for (int k = 0; k < kKnobCount; ++k) {
      if (std::strcmp(name, kKnobDefs[k].name) == 0) {
        knob_table()[k].store(value, std::memory_order_relaxed);
        return MST_OK;
      }
    }
    throw MstError{MST_ERR_INVALID_ARG, std::string("unknown tuning knob: ") + name};
  });
}

int mst_gpu_get_tuning(const char* name, double* out_value) {
  return guarded([&]() -> int {
    if (!name || !out_value) throw MstError{MST_ERR_INVALID_ARG, "NULL argument"};
    for (int k = 0; k < kKnobCount; ++k) {
      if (std::strcmp(name, kKnobDefs[k].name) == 0) {
        *out_value = knob((Knob)k);
        return MST_OK;
      }
    }
    throw MstError{MST_ERR_INVALID_ARG, std::string("unknown tuning knob: ") + name};
  });
}

int mst_gpu_reset_tuning(void) {
  for (int k = 0; k < kKnobCount; ++k) knob_table()[k].store(kKnobDefs[k].dflt, std::memory_order_relaxed);
  return MST_OK;
}

const char* mst_gpu_tuning_name(int index) {
  return (index >= 0 && index < kKnobCount) ? kKnobDefs[index].name : nullptr;
}

int mst_gpu_release_workspace(void) {
  return guarded([&]() -> int {
    std::lock_guard<std::mutex> g(g_ws_mu);
    for (auto& kv : g_ws) {
      std::lock_guard<std::mutex> lk(kv.second->mu);
      kv.second->release();
    }
    return MST_OK;
  });
}

}  // extern "C"
