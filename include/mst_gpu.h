/*
 * mst_gpu.h — C ABI of the B200-native parallel Boruvka MST (arXiv 2005.06913).
 *
 * This is the drop-in boundary for the reference's hot path
 *   mst::boruvka_cas(Graph&, int, ParallelRunInfo*)
 *     /root/reference/proj/include/mst/boruvka_parallel.hpp:70
 *     /root/reference/proj/src/boruvka_parallel.cpp:85-291
 * Plain pointers and sizes only; no C++ or torch types cross it. The C++
 * wrapper with the reference's shape (Graph& in, MstResult out, exceptions)
 * is include/mst/boruvka_gpu.hpp; the Python mirror is
 * paper_2005_06913_b200/api.py. See INTEGRATION.md for the bindings.
 *
 * Types follow the reference: VertexId = uint32 (graph.hpp:12), EdgeId is
 * int64 there (graph.hpp:13) and uint32 here (m < 2^32 - 1 is checked),
 * Weight is uint64 there (graph.hpp:14) and uint32 here (checked at the AoS
 * entry, which accepts the reference's 16-byte Edge directly).
 *
 * Result contract = mst::MstResult (mst_result.hpp:10-20): the MST edge ids
 * sorted ascending, their total weight as uint64, the round count. Weights
 * are expected to be distinct (the reference's build_graph contract,
 * graph.cpp:118-125); on a single GPU ties are broken by lower edge id, which
 * equals a stable Kruskal over (weight, id).
 *
 * Threading: calls are synchronous w.r.t. the host (like boruvka_cas) and
 * may be made from several host threads on different devices. The last
 * error string is thread-local.
 */
#ifndef MST_GPU_H_
#define MST_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. 0 = success. Mirrors the reference's error behaviour:
 *   MST_ERR_INVALID_ARG  ~ std::invalid_argument (boruvka_parallel.cpp:86,
 *                          graph.cpp:93)
 *   MST_ERR_RANGE        ~ GraphError{EndpointOutOfRange} (graph.cpp:98-100)
 *   MST_ERR_WEIGHT       weight does not fit the 32-bit device key
 *   MST_ERR_DISCONNECTED ~ GraphError{Disconnected} (graph.cpp:127-134); the
 *                          minimum spanning FOREST is still returned
 *   MST_ERR_CUDA / _NCCL ~ WorkerPanic (boruvka_parallel.hpp:44-47)
 */
enum {
  MST_OK = 0,
  MST_ERR_INVALID_ARG = 1,
  MST_ERR_RANGE = 2,
  MST_ERR_WEIGHT = 3,
  MST_ERR_DISCONNECTED = 4,
  MST_ERR_CUDA = 5,
  MST_ERR_NCCL = 6,
  MST_ERR_NO_DEVICE = 7,
  MST_ERR_OOM = 8,
  MST_ERR_STALL = 9,
  MST_ERR_PARSE = 10, /* ~ GraphError{ParseError} (graph.cpp:229-281) */
  MST_ERR_IO = 11
};

#define MST_MAX_ROUNDS 48

/* The reference's Edge, bit-for-bit (graph.hpp:41-45): 16 bytes. */
typedef struct mst_edge {
  uint32_t src;
  uint32_t dest;
  uint64_t weight;
} mst_edge_t;

/* SoA edge list: the device-native layout (12 bytes/edge). */
typedef struct mst_edges_soa {
  uint32_t n;            /* vertex count, >= 1 */
  uint64_t m;            /* edge count, < 2^32 - 1 */
  const uint32_t* src;   /* [m] */
  const uint32_t* dst;   /* [m] */
  const uint32_t* w;     /* [m] */
  int on_device;         /* 1: pointers are device pointers on the run's GPU */
} mst_edges_soa_t;

/* Per-run statistics (ParallelRunInfo analogue, boruvka_parallel.hpp:52-56,
 * plus the per-round counters the byte model of DESIGN.md needs). */
typedef struct mst_stats {
  uint32_t rounds;            /* Boruvka rounds (min-edge passes) */
  uint32_t final_components;  /* 1 for a connected input */
  double ms_total;            /* host wall time of the whole call */
  double ms_device;           /* device time, first kernel .. result ready */
  double ms_h2d;              /* host->device edge copy (0 for device input) */
  double ms_d2h;              /* device->host result copy */
  uint64_t alg_bytes;         /* algorithmic bytes over all rounds */
  uint64_t live_edges[MST_MAX_ROUNDS]; /* m_r: live edges entering round r */
  uint64_t live_comps[MST_MAX_ROUNDS]; /* n_r: live components in round r */
  uint32_t kernel_launches;   /* kernels launched by this call */
  uint64_t hot_bytes;         /* algorithmic bytes of the timed edge passes
                                 (mst_gpu_boruvka_device with ms_hot only) */
} mst_stats_t;

/* Single-GPU (num_gpus == 1) or single-process multi-GPU (num_gpus in 2..8,
 * devices 0..num_gpus-1 of the calling process, edge list sharded, one
 * NCCL allreduce(min, uint64) per round). Device input requires
 * num_gpus == 1 and pointers on the current CUDA device.
 * out_ids must hold n-1 entries; they come back sorted ascending.
 * out_count/out_total_weight/stats may be NULL. */
int mst_gpu_boruvka(const mst_edges_soa_t* edges, int num_gpus, uint32_t* out_ids,
                    uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats);

/* Same, taking the reference's AoS Edge array unchanged (16 B/edge). Weights
 * >= 2^32 give MST_ERR_WEIGHT. Single GPU. */
int mst_gpu_boruvka_aos(uint32_t n, uint64_t m, const mst_edge_t* edges, int on_device,
                        uint32_t* out_ids, uint64_t* out_count, uint64_t* out_total_weight,
                        mst_stats_t* stats);

/* Test hook: runs the sharded (multi-GPU) algorithm with `num_shards` edge
 * shards emulated on the current device; the per-round allreduce becomes an
 * on-device min over the shard buffers. Same result contract. */
int mst_gpu_boruvka_emulated(const mst_edges_soa_t* edges, int num_shards, uint32_t* out_ids,
                             uint64_t* out_count, uint64_t* out_total_weight,
                             mst_stats_t* stats);

/* Test hook: the round-1 minimum table alone (k_min_round1): for every
 * vertex the key (w<<32 | edge id) of its lightest incident non-loop edge, ~0
 * if none — the first pass of boruvka_seq.cpp:47-56. out_min: n entries
 * (host memory). */
int mst_gpu_round1_min(const mst_edges_soa_t* edges, uint64_t* out_min);

/* ---- one process per GPU (torchrun) ----
 * Rank r owns the contiguous edge slice [shard_base, shard_base + shard_m) of
 * the global list (global ids are shard_base + local index). Every rank gets
 * the full sorted result. The NCCL unique id is created on one rank and
 * broadcast by the caller (paper_2005_06913_b200/dist.py uses torch.distributed). */
typedef struct mst_comm* mst_comm_t;
#define MST_UNIQUE_ID_BYTES 128
int mst_comm_unique_id(uint8_t out_id[MST_UNIQUE_ID_BYTES]);
int mst_comm_init(const uint8_t id[MST_UNIQUE_ID_BYTES], int nranks, int rank, int device,
                  mst_comm_t* out_comm);
int mst_comm_destroy(mst_comm_t comm);
int mst_gpu_boruvka_rank(mst_comm_t comm, uint32_t n, uint64_t m_total, uint64_t shard_base,
                         uint64_t shard_m, const uint32_t* src, const uint32_t* dst,
                         const uint32_t* w, int on_device, uint32_t* out_ids,
                         uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats);

/* The same with this rank's shard already in HBM (device pointers on the
 * communicator's device) and the sorted ids left in HBM (d_out_ids, n-1
 * entries): the multi-GPU counterpart of mst_gpu_boruvka_device. Runs on
 * `stream` (NULL: ordered after / before the legacy default stream 0). */
int mst_gpu_boruvka_rank_device(mst_comm_t comm, uint32_t n, uint64_t m_total, uint64_t shard_base,
                                uint64_t shard_m, const uint32_t* d_src, const uint32_t* d_dst,
                                const uint32_t* d_w, uint32_t* d_out_ids, void* stream,
                                uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats);

/* Bring-your-own collective (MPI, gloo, a test harness): the sharded loop of
 * mst_gpu_boruvka_rank with every exchange handed to `allreduce`, which must
 * reduce `count` elements of `host_buf` (pinned host memory, in place)
 * across all ranks and return 0. dtype MST_DTYPE_U32 / MST_DTYPE_U64
 * (unsigned), op MST_OP_MIN / MST_OP_SUM. Every rank makes the same calls
 * in the same order. */
#define MST_DTYPE_U32 0
#define MST_DTYPE_U64 1
#define MST_OP_MIN 0
#define MST_OP_SUM 1
typedef struct mst_collective {
  int (*allreduce)(void* ctx, void* host_buf, uint64_t count, int dtype, int op);
  void* ctx;
  int nranks, rank, device;
} mst_collective_t;
int mst_gpu_boruvka_rank_cb(const mst_collective_t* coll, uint32_t n, uint64_t m_total,
                            uint64_t shard_base, uint64_t shard_m, const uint32_t* src,
                            const uint32_t* dst, const uint32_t* w, int on_device, uint32_t* out_ids,
                            uint64_t* out_count, uint64_t* out_total_weight, mst_stats_t* stats);

/* Device-resident timing entry (bench): edges already in HBM, result left in
 * HBM (sorted ids in d_out_ids, count/total in host outputs). Runs `reps`
 * back-to-back MSTs on `stream` (0 = legacy default stream) and returns the
 * summed device time of the min-edge/compaction kernel family in
 * *ms_hot and its launch count in *hot_launches (for the roofline). */
int mst_gpu_boruvka_device(const mst_edges_soa_t* edges, uint32_t* d_out_ids, void* stream,
                           uint64_t* out_count, uint64_t* out_total_weight,
                           mst_stats_t* stats, double* ms_hot, uint32_t* hot_launches);

/* ---- GPU verifier ----
 * The checks of the reference's verify_mst (proj/src/verify.cpp:15-57,
 * VerifyReport in proj/include/mst/verify.hpp:11-24) on the device, with the
 * oracle's result supplied by the caller (the reference's second overload,
 * verify.hpp:31, "computed once and reused"): ids in range (else
 * MST_ERR_RANGE ~ std::out_of_range, verify.cpp:19-22), |ids| == n-1,
 * acyclic and spanning through a private union-find over the result edges,
 * weight sum, and weight / edge-set equality with the oracle. `ids` (and
 * `oracle_ids`) live where the edges live (edges->on_device). Pass
 * oracle_total = MST_VERIFY_NO_ORACLE to run the structural checks only;
 * the two oracle flags are then -1. */
#define MST_VERIFY_NO_ORACLE (~(uint64_t)0)
typedef struct mst_verify {
  int is_spanning;
  int is_acyclic;
  int edge_count_ok;
  int weight_matches_oracle;   /* -1: no oracle given */
  int edge_set_matches_oracle; /* -1: no oracle given */
  uint64_t components;         /* after uniting the result edges */
  uint64_t weight;             /* sum of the result edges' weights */
} mst_verify_t;
int mst_gpu_verify(const mst_edges_soa_t* edges, const uint32_t* ids, uint64_t count,
                   const uint32_t* oracle_ids, uint64_t oracle_count, uint64_t oracle_total,
                   mst_verify_t* report);
/* Same over the reference's 16-byte Edge array (full 64-bit weights). */
int mst_gpu_verify_aos(uint32_t n, uint64_t m, const mst_edge_t* edges, int on_device,
                       const uint32_t* ids, uint64_t count, const uint32_t* oracle_ids,
                       uint64_t oracle_count, uint64_t oracle_total, mst_verify_t* report);

/* ---- edge-list files ----
 * Text: the reference's format, "<n> <m>\n" + m lines "<src> <dest> <weight>\n"
 * (load_graph / save_graph, graph.cpp:228-295), parsed and formatted in
 * parallel with load_graph's strict rules and messages (MST_ERR_PARSE);
 * weights must fit 32 bits (MST_ERR_WEIGHT). build_graph's structural
 * checks are not applied (see the widenings above).
 * Binary SoA ("MSTSOA01"): 4 KiB header, then u32 src / dst / w arrays on
 * 4 KiB boundaries; mst_io_load_soa(on_device = 1) streams the file into
 * device arrays through pinned chunks (read of chunk k+1 overlaps the copy
 * of chunk k). The *_header calls give n and m for sizing the arrays. */
int mst_io_text_header(const char* path, uint32_t* out_n, uint64_t* out_m);
int mst_io_load_text(const char* path, uint32_t n, uint64_t m, uint32_t* src, uint32_t* dst,
                     uint32_t* w);
int mst_io_save_text(const char* path, uint32_t n, uint64_t m, const uint32_t* src,
                     const uint32_t* dst, const uint32_t* w);
int mst_io_soa_header(const char* path, uint32_t* out_n, uint64_t* out_m);
int mst_io_load_soa(const char* path, uint32_t n, uint64_t m, uint32_t* src, uint32_t* dst,
                    uint32_t* w, int on_device);
int mst_io_save_soa(const char* path, uint32_t n, uint64_t m, const uint32_t* src,
                    const uint32_t* dst, const uint32_t* w);

/* ---- tuning knobs ----
 * Every engine knob sits in one process-wide table with its measured
 * default (DESIGN.md §2 gives the measurements); the library never reads the
 * environment. Knobs are named like the A/B tools' MST_* variables
 * ("MST_FILTER", "MST_FILTER_BETA", "MST_TAIL", ...; mst_gpu_tuning_name(i)
 * enumerates them, NULL past the last). Unknown names -> MST_ERR_INVALID_ARG.
 * Changing a knob while another thread runs an MST is not supported. */
int mst_gpu_set_tuning(const char* name, double value);
int mst_gpu_get_tuning(const char* name, double* out_value);
int mst_gpu_reset_tuning(void);
const char* mst_gpu_tuning_name(int index);

/* Frees the cached device workspaces of the calling thread's devices. */
int mst_gpu_release_workspace(void);

/* Thread-local description of the last failure ("" if none). */
const char* mst_gpu_last_error(void);

/* Library version string and the number of visible CUDA devices (no GPU
 * work; safe on a GPU-less host). */
const char* mst_gpu_version(void);
int mst_gpu_device_count(void);

/* ---- seeded synthetic inputs for the BASELINE.json configs ----
 * Counter-based (hash of seed and index), so the CPU and GPU generators
 * produce identical bytes and any slice can be produced independently.
 * kind: 0 uniform (spanning tree + uniform pairs, configs 0/3),
 *       1 grid (rows x cols 4-neighbour, config 1; n = rows*cols),
 *       2 R-MAT (scale, edgefactor; self-loops dropped, spanning tree added,
 *         configs 2/4).
 * mst_gen_count returns the edge count the generator will produce. */
typedef struct mst_gen_spec {
  int kind;
  uint32_t n;            /* uniform: vertices; grid: rows*cols; rmat: 2^scale */
  uint64_t m;            /* uniform: total edges (tree included) */
  uint32_t rows, cols;   /* grid */
  uint32_t scale;        /* rmat */
  uint32_t edgefactor;   /* rmat */
  double a, b, c;        /* rmat quadrant probabilities (d = 1-a-b-c) */
  uint64_t seed;
} mst_gen_spec_t;
int mst_gen_count(const mst_gen_spec_t* spec, uint64_t* out_m);
/* CPU generator (threads <= 0: all hardware threads). */
int mst_gen_host(const mst_gen_spec_t* spec, uint32_t* src, uint32_t* dst, uint32_t* w,
                 int threads);
/* GPU generator into device arrays of mst_gen_count() entries. */
int mst_gen_device(const mst_gen_spec_t* spec, uint32_t* d_src, uint32_t* d_dst, uint32_t* d_w);

#ifdef __cplusplus
}
#endif

#endif /* MST_GPU_H_ */
