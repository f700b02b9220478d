// Device kernels of the B200 parallel Boruvka (arXiv 2005.06913, CAS variant
// re-designed for the GPU). One round r with n_r live components (dense
// labels 0..n_r-1) and m_r live edges:
//
//   k_hook_decide (n_r)  every component reads its lightest edge key, picks
//                        the partner, breaks mutual 2-cycles by lower label,
//                        flags roots and counts them per tile. Replaces the
//                        merge phase + try_union_cas (boruvka_parallel.cpp:
//                        176-227, union_find.cpp:75-92).
//   k_label2      (n_r)  MST slot n - n_r + c - roots_before(c) for every
//                        hooked component, root finding with concurrent path
//                        halving over the hook forest (the reference's find
//                        walk, union_find.cpp:28-35), dense relabel, clears
//                        the next min table.
//   k_count       (m_r)  relabels both endpoints in place, drops
//                        intra-component edges (the covered flags,
//                        graph.hpp:62-67), counts the kept edges per tile and
//                        offers each kept edge to both endpoint components of
//                        round r+1 with a filtered 64-bit atomicMin keyed by
//                        its position in this list (the edge scan + offer,
//                        boruvka_parallel.cpp:150-167). The caller's list is
//                        walked in interleaved segments (MST_INTERLEAVE).
//   k_emit        (m_r)  writes the kept edges in order (a pure copy). The
//                        light split and the heavy filter stage their sparse
//                        survivors per tile instead (k_emit_sparse copies
//                        them) and make their offers in range passes over
//                        L2-sized table slices (k_range_offers).
//
// Round 1 reads the caller's edge list directly (k_min_round1 + the count
// pass over the original view; in the plain loop its label pairs are round
// 2's list, PairsInView). Offers are read-first 64-bit atomicMins, batched
// per thread where that pays (offer_both). Filter-Boruvka, pair dedup, the
// tail megakernel (segmented in-place compaction, one-sync tiny rounds),
// the sorted output and the sharded exchange are described at their
// kernels below.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mstgpu {

// Minimum resident blocks per SM for the round kernels (register caps):
// these kernels are memory-latency bound, so more resident warps = more
// loads in flight. 0 = ptxas's own choice. Overridable at build time (A/B).
#define MST_LB_(n) MST_LB_SEL_(n)
#define MST_LB_SEL_(n) MST_LB_##n
#define MST_LB_0 __launch_bounds__(256)
#define MST_LB_5 __launch_bounds__(256, 5)
#define MST_LB_6 __launch_bounds__(256, 6)
#define MST_LB_8 __launch_bounds__(256, 8)
#ifndef MST_MINB_MIN1
#define MST_MINB_MIN1 0
#endif
#ifndef MST_MINB_HOOK
#define MST_MINB_HOOK 0
#endif
#ifndef MST_MINB_LABEL
#define MST_MINB_LABEL 0
#endif
#ifndef MST_MINB_COUNT
#define MST_MINB_COUNT 0
#endif
#ifndef MST_MINB_EMIT
#define MST_MINB_EMIT 0
#endif
constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 4;                // per thread, component tiles (hook)
constexpr int kTile = kBlock * kItems;   // elements per tile (striped)
constexpr int kCItems = 4;               // per thread, edge tiles (compaction)
constexpr int kCTile = kBlock * kCItems;

constexpr int kMaxR = MST_MAX_ROUNDS + 2;
constexpr uint64_t kNoKey = ~0ull;
constexpr int kFiltCached = 8;  // offer filter reads through L1 (see offer)
constexpr uint32_t kRetFlag = 0x80000000u;  // level-map entry of a retired component: kRetFlag | own index
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kErrRange = 1u;
constexpr uint32_t kErrWeight = 2u;
constexpr uint32_t kNoStop = 0xFFFFFFFFu;

// Tile-counter slots per round.
enum { kSlotHook = 0, kSlotCompact = 1, kSlotSort = 2, kSlotFilter = 3 };

// Per-call device counters. Round r (1-based) reads n[r], m[r] and writes
// n[r+1], m[r+1]; nothing is reset between rounds, so the whole round
// sequence can be enqueued without host round trips.
struct DevCounters {
  unsigned long long m[kMaxR];
  unsigned int n[kMaxR];
  unsigned int tile[kMaxR][4];
  unsigned int done[kMaxR][4];  // last-block-done check-ins (fused scans)
  unsigned int err;
  unsigned int stop_round;  // first round whose hook must not run
  unsigned int phase_end;   // first round past the light phase (Filter-Boruvka)
  unsigned int pivot;       // light edges: w < pivot
  unsigned long long total_weight;
  unsigned int active[kMaxR];     // components with a live edge at round r (hook)
  unsigned int dedup[kMaxR];      // round r's compaction keeps one edge per component pair
  unsigned long long pair_mask[kMaxR];
  unsigned int pair_count[kMaxR];  // distinct pairs inserted
  unsigned int pair_abort[kMaxR];  // table overflowed: keep every edge this round
  unsigned int dedup_fail;         // some dedup attempt overflowed (sticky, see k_label2)
  unsigned int giant;              // k_pick_giant: the most frequent next-round label of a round's endpoints
};


// Programmatic dependent launch: every kernel first waits for its stream
// predecessor to complete (and its memory to be visible), then lets its own
// successor start launching, so launch latency and block ramp-up overlap the
// predecessor's tail. Without a PDL launch both are no-ops.
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------ edge views ---------------------------------

struct EdgeRec {
  uint32_t a, b, w, eid;
  bool ok;  // false: weight did not fit 32 bits (AoS input)
};

// Caller's SoA list (12 B/edge), global id = base + i.
struct SoaView {
  const uint32_t* __restrict__ src;
  const uint32_t* __restrict__ dst;
  const uint32_t* __restrict__ w;
  uint32_t base;
  static constexpr bool kOriginal = true;
  static constexpr bool kMayBeDead = false;
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    return EdgeRec{__ldcs(src + i), __ldcs(dst + i), __ldcs(w + i), base + (uint32_t)i, true};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    return EdgeRec{__ldg(src + i), __ldg(dst + i), __ldg(w + i), base + (uint32_t)i, true};
  }
  // endpoints and id only (the hook has the weight in its key)
  __device__ __forceinline__ EdgeRec gather_ends(uint64_t i) const {
    return EdgeRec{__ldg(src + i), __ldg(dst + i), 0u, base + (uint32_t)i, true};
  }
  __device__ __forceinline__ uint32_t weight(uint64_t i) const { return __ldcs(w + i); }
};

// The reference's AoS Edge {u32 src, u32 dest, u64 weight} (graph.hpp:41-45).
struct AosView {
  const uint4* __restrict__ e;
  uint32_t base;
  static constexpr bool kOriginal = true;
  static constexpr bool kMayBeDead = false;
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    const uint4 v = __ldcs(e + i);
    return EdgeRec{v.x, v.y, v.z, base + (uint32_t)i, v.w == 0};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    const uint4 v = __ldg(e + i);
    return EdgeRec{v.x, v.y, v.z, base + (uint32_t)i, v.w == 0};
  }
  __device__ __forceinline__ EdgeRec gather_ends(uint64_t i) const { return gather(i); }
  __device__ __forceinline__ uint32_t weight(uint64_t i) const {
    return __ldcs(reinterpret_cast<const uint32_t*>(e + i) + 2);
  }
};

// Compacted edges of round >= 2: {a, b, w, eid} (16 B/edge, one LDG.128).
struct PackedView {
  const uint4* __restrict__ e;
  static constexpr bool kOriginal = false;
  static constexpr bool kMayBeDead = false;
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    const uint4 v = __ldcs(e + i);
    return EdgeRec{v.x, v.y, v.z, v.w, true};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    const uint4 v = __ldg(e + i);
    return EdgeRec{v.x, v.y, v.z, v.w, true};
  }
  __device__ __forceinline__ EdgeRec gather_ends(uint64_t i) const { return gather(i); }
  __device__ __forceinline__ uint32_t weight(uint64_t i) const {
    return __ldcs(reinterpret_cast<const uint32_t*>(e + i) + 2);
  }
  static constexpr uint32_t base = 0;
};

// Round 1's relabelled list when the input was the caller's list: the count
// pass leaves 8 B label pairs at each input position; weight and id come
// from the caller's list. Round 2's hook gathers through this view.
template <class In>
struct PairsView {
  const uint2* __restrict__ xy;
  In in;
  static constexpr bool kOriginal = false;
  static constexpr bool kMayBeDead = false;
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    const uint2 p = __ldcg(xy + i);
    return EdgeRec{p.x, p.y, in.weight(i), in.base + (uint32_t)i, true};
  }
  __device__ __forceinline__ EdgeRec gather_ends(uint64_t i) const {
    const uint2 p = __ldcg(xy + i);
    return EdgeRec{p.x, p.y, 0u, in.base + (uint32_t)i, true};
  }
};

// Round 2 of the plain loop over round 1's label pairs, uncompacted (round
// 1 skips its emit pass): the pair list IS round 2's edge list, indexed like
// the caller's list (positions = edge ids), with the weights read from the
// caller's list. Round 1's dead edges are the pairs with a == b; round 2's
// count pass skips them and relabels the live pairs in place, so round 3's
// hook gathers from the same list (PairsView).
template <class In>
struct PairsInView {
  const uint2* __restrict__ xy;
  In in;
  uint32_t base;
  static constexpr bool kOriginal = true;
  static constexpr bool kMayBeDead = true;
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    const uint2 p = __ldcg(xy + i);
    return EdgeRec{p.x, p.y, in.weight(i), base + (uint32_t)i, true};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const { return stream(i); }
  __device__ __forceinline__ uint32_t weight(uint64_t i) const { return in.weight(i); }
};

// ------------------------------ primitives ---------------------------------

// The MST output: one bit per edge id (c4: 143 MB, mostly L2-resident, where
// a byte per edge was 1.14 GB of partial-sector writes), set by a
// fire-and-forget RED.OR from the hook of the edge's component.
__device__ __forceinline__ void mst_set(uint32_t* bits, uint32_t eid) {
  atomicOr(bits + (eid >> 5), 1u << (eid & 31));
}
// The output for a caller's list small enough that one byte per edge stays
// in L2 (<= MST_BYTES_MAX edges, 64 Mi): plain byte stores. Grids hook neighbouring
// components along neighbouring edges, ~16 MST edges per bitmap word, whose
// REDs queue on the same word (c1 round-1 hook: 57 us with the bitmap, 39 us
// with bytes).
__device__ __forceinline__ void mst_mark(uint32_t* out, int bytes, uint32_t eid) {
  if (bytes)
    reinterpret_cast<uint8_t*>(out)[eid] = 1;
  else
    mst_set(out, eid);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
    if ((int)lane_id() >= d) v += t;
  }
  return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Decoupled look-back (single pass prefix over tiles taken in order from a
// dynamic tile counter). Status word: epoch(30) | flag(2) | value(32);
// flag 1 = tile aggregate, 2 = inclusive prefix. Stale words from earlier
// scans carry an older epoch and read as "not ready". Called by a full warp;
// returns the exclusive prefix of `tile` on every lane.
__device__ __forceinline__ uint32_t lookback(unsigned long long* status, uint32_t tile,
                                             uint32_t aggregate, uint32_t epoch) {
  const unsigned long long tag = (unsigned long long)epoch << 34;
  const uint32_t lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_relaxed(status, tag | (2ull << 32) | aggregate);
    return 0;
  }
  if (lane == 0) st_relaxed(status + tile, tag | (1ull << 32) | aggregate);
  uint32_t excl = 0;
  int64_t top = (int64_t)tile - 1;
  uint32_t backoff = 32;
  while (true) {
    // One read of a 32-tile window per attempt; predecessors that have not
    // published yet make the warp back off instead of spinning on L2 (the
    // window's lines are the hottest in the machine while a scan runs).
    const int64_t idx = top - (int64_t)lane;
    uint32_t flag = 2, val = 0;
    if (idx >= 0) {
      const unsigned long long s = ld_relaxed(status + idx);
      flag = (uint32_t)(s >> 34) == epoch ? (uint32_t)(s >> 32) & 3u : 0u;
      val = (uint32_t)s;
    }
    const unsigned pm = __ballot_sync(0xffffffffu, flag == 2);
    const unsigned nr = __ballot_sync(0xffffffffu, flag == 0);
    const int first = pm ? __ffs(pm) - 1 : 31;
    const unsigned upto = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
    if (nr & upto) {
      __nanosleep(backoff);
      backoff = backoff < 1024 ? backoff * 2 : 1024;
      continue;
    }
    excl += warp_sum<uint32_t>((int)lane <= first ? val : 0u);
    if (pm) break;
    top -= 32;
  }
  if (lane == 0) st_relaxed(status + tile, tag | (2ull << 32) | (excl + aggregate));
  return excl;
}

// Filtered 64-bit min: read first (a stale read is never below the true
// value, so skipping is always safe), atomic only when it can win. (A
// warp-level pre-reduction with __match_any_sync + redux.sync measured
// slower on every config and was removed.)
__device__ __forceinline__ void offer(unsigned long long* table, uint32_t c, uint64_t key,
                                      bool valid, int filt = 1) {
  if (!valid) return;
  // filt & 3 == 0: a fire-and-forget RED (no dependent read on the path).
  // filt & kFiltCached: the filter read goes through L1 (a stale copy is
  // never below the truth either), so hot hub entries are not re-read from
  // their one L2 slice by every offer.
  if (filt & 3) {
    const unsigned long long cur = (filt & kFiltCached) ? __ldca(table + c) : __ldcg(table + c);
    if (key < cur) atomicMin(table + c, (unsigned long long)key);
  } else {
    atomicMin(table + c, (unsigned long long)key);
  }
}

// K edges' offers to both endpoints with all filter reads in flight together,
// then the atomics. (Offer by offer, each read waits behind the previous
// item's atomic on the same table: 2K serial L2 round trips per thread.)
// filt & 3: 0 = plain REDs, 1 = read-first one offer at a time (each read sees
// the previous atomics: best for hot hub entries), 2 = read-first batched;
// | kFiltCached: filter reads through L1.
template <int K>
__device__ __forceinline__ void offer_both(unsigned long long* table, const uint32_t (&x)[K], const uint32_t (&y)[K],
                                           const unsigned long long (&key)[K], const bool (&valid)[K], int filt) {
  if ((filt & 3) == 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      offer(table, x[k], key[k], valid[k], filt);
      offer(table, y[k], key[k], valid[k], filt);
    }
  } else if ((filt & 3) == 2) {
    const bool cached = (filt & kFiltCached) != 0;
    unsigned long long cx[K], cy[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      cx[k] = valid[k] ? (cached ? __ldca(table + x[k]) : __ldcg(table + x[k])) : 0ull;
      cy[k] = valid[k] ? (cached ? __ldca(table + y[k]) : __ldcg(table + y[k])) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!valid[k]) continue;
      if (key[k] < cx[k]) atomicMin(table + x[k], key[k]);
      if (key[k] < cy[k]) atomicMin(table + y[k], key[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!valid[k]) continue;
      atomicMin(table + x[k], key[k]);
      atomicMin(table + y[k], key[k]);
    }
  }
}

// kU independent root walks interleaved step by step (path halving), so each
// thread keeps kU dependent-load chains in flight instead of one.
template <int kU>
__device__ __forceinline__ void find_roots(uint32_t* parent, const uint32_t (&c)[kU], const bool (&valid)[kU],
                                           uint32_t (&root)[kU]) {
  uint32_t x[kU], px[kU];
  bool live[kU];
#pragma unroll
  for (int k = 0; k < kU; ++k) {
    x[k] = c[k];
    live[k] = valid[k];
    root[k] = c[k];
    px[k] = live[k] ? __ldcg(parent + x[k]) : x[k];
  }
  while (true) {
    uint32_t gp[kU];
#pragma unroll
    // through L1: the roots' entries are read by every walk that ends there
    // (the giant's root: millions of reads of one line, which serialise on
    // its L2 slice with ld.cg). A stale line only shows an older ancestor.
    for (int k = 0; k < kU; ++k) gp[k] = (live[k] && px[k] != x[k]) ? __ldca(parent + px[k]) : px[k];
    bool any = false;
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      if (!live[k]) continue;
      if (px[k] == x[k]) {
        root[k] = x[k];
        live[k] = false;
      } else if (gp[k] == px[k]) {
        root[k] = px[k];
        live[k] = false;
      } else {
        parent[x[k]] = gp[k];  // path halving: every value ever stored is an ancestor
        x[k] = gp[k];
        any = true;
      }
    }
    if (!any) break;
#pragma unroll
    for (int k = 0; k < kU; ++k)
      if (live[k]) px[k] = __ldca(parent + x[k]);
  }
}

__device__ __forceinline__ uint32_t find_root(uint32_t* parent, uint32_t c) {
  uint32_t p = __ldcg(parent + c);
  while (p != c) {
    const uint32_t gp = __ldcg(parent + p);
    if (gp == p) return p;
    parent[c] = gp;  // path halving: every value ever stored is an ancestor
    c = gp;
    p = __ldcg(parent + c);
  }
  return c;
}

// ------------------------------ round 1 ------------------------------------

// Lightest incident edge per vertex over the caller's list, literal keys
// (w<<32 | index in the list).
// Edges [lo, m) of the list (lo > 0: a later chunk of a pipelined host copy).
template <class View>
__global__ void MST_LB_(MST_MINB_MIN1) k_min_round1(View v, uint32_t n, uint64_t lo, uint64_t m,
                                                       unsigned long long* __restrict__ minimum,
                                                       DevCounters* ctr, int filt) {
  pdl_prologue();
  constexpr int kU = 4;
  const uint64_t stride = (uint64_t)gridDim.x * kBlock * kU;
  uint32_t err = 0;
  for (uint64_t base = lo + (uint64_t)blockIdx.x * kBlock * kU; base < m; base += stride) {
    EdgeRec e[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * kBlock + threadIdx.x;
      e[k] = EdgeRec{0, 0, 0, 0, false};
      if (i < m) e[k] = v.stream(i);
    }
    uint32_t xa[kU], xb[kU];
    unsigned long long key[kU];
    bool valid[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * kBlock + threadIdx.x;
      valid[k] = i < m;
      if (valid[k]) {
        if (e[k].a >= n || e[k].b >= n) {
          err |= kErrRange;
          valid[k] = false;
        } else if (!e[k].ok) {
          err |= kErrWeight;
          valid[k] = false;
        } else if (e[k].a == e[k].b) {
          valid[k] = false;  // self-loop: never in an MST
        }
      }
      xa[k] = e[k].a;
      xb[k] = e[k].b;
      key[k] = ((unsigned long long)e[k].w << 32) | (uint32_t)i;
    }
    offer_both<kU>(minimum, xa, xb, key, valid, filt);
  }
  if (err) atomicOr(&ctr->err, err);
}

// ------------------------------ Filter-Boruvka helpers --------------------

// Pivot of the split: histogram of the top 16 weight bits over a strided
// sample, then the smallest bin boundary with >= target sampled weights
// below it (kept in ctr->pivot; 0xFFFFFFFF means "everything light").
__global__ void k_weight_hist(const uint32_t* __restrict__ w, uint32_t wstride, uint64_t m,
                              uint64_t step, uint32_t samples, uint32_t* __restrict__ hist) {
  pdl_prologue();
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < samples; k += gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)k * step;
    if (i < m) atomicAdd(hist + (__ldg(w + i * wstride) >> 16), 1u);
  }
}

// target = max(1, frac * (sampled weights)), computed here from the
// histogram's own total: in the sharded loop the histograms are summed
// across ranks first, so every rank derives the same target and pivot.
__global__ void __launch_bounds__(1024) k_pick_pivot(const uint32_t* __restrict__ hist, double frac, DevCounters* ctr) {
  pdl_prologue();
  // one block of 1024 threads: 64 bins per thread (16 independent 16 B loads
  // in flight, not 64 dependent ones), block scan of the sums, then the 64
  // bins of the thread whose range holds the target are searched by 64
  // threads at once
  __shared__ uint32_t s_sum[1024];
  __shared__ uint32_t s_tstar, s_before, s_w0;
  const uint32_t t = threadIdx.x;
  const uint4* h4 = reinterpret_cast<const uint4*>(hist) + t * 16;
  uint32_t sum = 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(h4 + half * 8 + i);
#pragma unroll
    for (int i = 0; i < 8; ++i) sum += v[i].x + v[i].y + v[i].z + v[i].w;
  }
  if (t == 0) s_tstar = 0xFFFFFFFFu;
  s_sum[t] = sum;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const uint32_t v = t >= (uint32_t)d ? s_sum[t - d] : 0u;
    __syncthreads();
    s_sum[t] += v;
    __syncthreads();
  }
  const uint32_t target = (uint32_t)fmax(1.0, frac * (double)s_sum[1023]);
  const uint32_t before = t ? s_sum[t - 1] : 0u;
  if (before < target && s_sum[t] >= target) {  // at most one thread
    s_tstar = t;
    s_before = before;
  }
  __syncthreads();
  if (s_tstar == 0xFFFFFFFFu || t >= 64) return;  // target above the total: everything light
  const uint32_t bin = s_tstar * 64 + t;
  const uint32_t c = __ldg(hist + bin);
  const uint32_t incl = warp_incl_scan(c);
  if (t == 31) s_w0 = incl;
  __syncwarp();
  asm volatile("bar.sync 1, 64;" ::: "memory");  // the two searching warps only
  const uint32_t run = s_before + incl + (t >= 32 ? s_w0 : 0u);
  const unsigned hit = __ballot_sync(0xffffffffu, run >= target);
  // the first bin reaching the target: the lowest hit lane of warp 0, else of warp 1
  if (hit && (uint32_t)(__ffs(hit) - 1) == (t & 31)) {
    const bool first = t < 32 || (s_before + s_w0 < target);
    if (first) ctr->pivot = bin == 0xFFFFu ? 0xFFFFFFFFu : (bin + 1) << 16;
  }
}

// Top-down composition of the light phase's relabel maps:
// L_r[c] = L_{r+1}[L_r[c]] for c < n[r] (in place on level r).
__global__ void k_compose(uint32_t* __restrict__ Lr, const uint32_t* __restrict__ Lnext,
                          const DevCounters* ctr, int r) {
  pdl_prologue();
  const uint32_t n_r = ctr->n[r];
  // 4 items per thread: the 4 gathers of Lnext are in flight together
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; base < n_r; base += stride) {
    uint32_t x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = base + (uint64_t)k * blockDim.x;
      x[k] = c < n_r ? Lr[c] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = base + (uint64_t)k * blockDim.x;
      if (c < n_r) x[k] = __ldg(Lnext + x[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = base + (uint64_t)k * blockDim.x;
      if (c < n_r) Lr[c] = x[k];
    }
  }
}

// ---- retirement (light phase): the final dense labels
// A light round's hook may retire its isolated components (no edge left):
// they get no label in the next round's dense space (so the tables of later
// rounds cover only components that still have edges), their level-map
// entry is kRetFlag | own index, and the hook records them in a bitmap
// region of that round. At the end of the light phase the bitmap regions
// (round 1, 2, ..., then the final region: one bit per component still
// labelled at the phase end) enumerate every final component exactly once;
// a component's final label is its rank in that bitmap (word prefix +
// popcount), which the top-down composition applies.
__global__ void k_ret_fill_final(uint32_t* __restrict__ words, const DevCounters* ctr, int P) {
  pdl_prologue();
  const uint32_t cnt = ctr->n[P];
  const uint32_t nw = (cnt + 31) / 32;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x)
    words[i] = (i + 1) * 32 <= cnt ? 0xFFFFFFFFu : ((1u << (cnt & 31)) - 1u);
}

__global__ void k_ret_popc(const uint32_t* __restrict__ words, uint64_t nw, uint32_t* __restrict__ counts) {
  pdl_prologue();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x)
    counts[i] = __popc(__ldg(words + i));
}

__device__ __forceinline__ uint32_t ret_rank(const uint32_t* __restrict__ words, const uint32_t* __restrict__ prefix,
                                             uint64_t s) {
  const uint64_t w = s >> 5;
  return __ldg(prefix + w) + __popc(__ldg(words + w) & ((1u << (s & 31)) - 1u));
}

// Level r of the light phase's maps to final labels, top-down: a retired
// entry -> its rank in region r; otherwise the top level -> the rank in the
// final region, a lower level -> the (already final) entry of level r+1.
__global__ void k_compose_ret(uint32_t* __restrict__ Lr, const uint32_t* __restrict__ Lnext,
                              const uint32_t* __restrict__ words, const uint32_t* __restrict__ prefix,
                              uint64_t woff_r, uint64_t woff_final, const DevCounters* ctr, int r) {
  pdl_prologue();
  const uint32_t n_r = ctr->n[r];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; base < n_r; base += stride) {
    uint32_t x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = base + (uint64_t)k * blockDim.x;
      x[k] = c < n_r ? Lr[c] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = base + (uint64_t)k * blockDim.x;
      if (c >= n_r) continue;
      if (x[k] & kRetFlag)
        x[k] = ret_rank(words, prefix, woff_r * 32 + (x[k] & ~kRetFlag));
      else if (Lnext == nullptr)
        x[k] = ret_rank(words, prefix, woff_final * 32 + x[k]);
      else
        x[k] = __ldg(Lnext + x[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = base + (uint64_t)k * blockDim.x;
      if (c < n_r) Lr[c] = x[k];
    }
  }
}

__global__ void k_fill_keys(unsigned long long* __restrict__ t, const DevCounters* ctr, int r) {
  pdl_prologue();
  const uint32_t cnt = ctr->n[r];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    t[i] = kNoKey;
}

// Giant bits for a relabel round with a huge component count (phase D's
// first round on R-MAT: 47 M components, most of which its hooks join into
// one giant). The most frequent next-round label among the endpoints of
// kGiantSamples evenly spaced list edges becomes ctr->giant, and
// gbits[c / 32] marks the components c with L[c] == giant: the round's
// compaction then relabels those endpoints from an L2-resident bitmap (6 MB)
// instead of gathering from the DRAM-sized map. Any choice is exact; ties
// go to the smaller label (deterministic).
constexpr int kGiantSamples = 2048;  // 4096 endpoint labels: the giant holds tens of per cent of them (8192: 70 us per launch, 2048: ~20)
constexpr int kGiantSlots = 4096;
__global__ void __launch_bounds__(1024) k_pick_giant(const uint4* __restrict__ E, const uint32_t* __restrict__ L,
                                                     DevCounters* ctr, int r) {
  pdl_prologue();
  __shared__ uint32_t s_key[kGiantSlots];
  __shared__ uint32_t s_cnt[kGiantSlots];
  __shared__ unsigned long long s_best[32];
  if ((uint32_t)r + 1 >= ctr->stop_round) return;
  const uint64_t m_r = ctr->m[r];
  for (int i = threadIdx.x; i < kGiantSlots; i += blockDim.x) {
    s_key[i] = kNone;
    s_cnt[i] = 0;
  }
  __syncthreads();
  const uint64_t step = m_r / kGiantSamples > 0 ? m_r / kGiantSamples : 1;
  for (int k = threadIdx.x; k < 2 * kGiantSamples; k += blockDim.x) {
    const uint64_t i = (uint64_t)(k >> 1) * step;
    if (i >= m_r) continue;
    const uint4 e = __ldg(E + i);
    const uint32_t lab = __ldg(L + ((k & 1) ? e.y : e.x));
    uint32_t h = (lab * 2654435761u) & (kGiantSlots - 1);
    for (int probe = 0; probe < 64; ++probe) {
      const uint32_t cur = atomicCAS(s_key + h, kNone, lab);
      if (cur == kNone || cur == lab) {
        atomicAdd(s_cnt + h, 1u);
        break;
      }
      h = (h + 1) & (kGiantSlots - 1);
    }
  }
  __syncthreads();
  unsigned long long best = 0;  // (count, ~label): max count, then min label
  for (int i = threadIdx.x; i < kGiantSlots; i += blockDim.x)
    if (s_cnt[i]) best = max(best, ((unsigned long long)s_cnt[i] << 32) | (uint32_t)~s_key[i]);
  for (int d = 16; d > 0; d >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, d));
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < blockDim.x / 32 ? s_best[threadIdx.x] : 0ull;
    for (int d = 16; d > 0; d >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, d));
    if (threadIdx.x == 0) ctr->giant = best ? ~(uint32_t)best : kNone;
  }
}

__global__ void k_giant_bits(const uint32_t* __restrict__ L, const DevCounters* ctr, int r,
                             uint32_t* __restrict__ gbits) {
  pdl_prologue();
  if ((uint32_t)r + 1 >= ctr->stop_round) return;
  const uint32_t n_r = ctr->n[r], g = ctr->giant;
  const uint32_t words = (n_r + 31) / 32;
  const uint32_t lane = lane_id();
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words; w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t c = w * 32 + lane;
    const unsigned gb = __ballot_sync(0xffffffffu, c < n_r && __ldcs(L + c) == g);
    if (lane == 0) gbits[w] = gb;
  }
}

// ------------------------------ scan helpers -------------------------------
//   kScanEdges : m[r+1] = kept; none kept -> stop (or light-phase end)
//   kScanRoots : n[r+1] = roots; <= 1 -> stop; == n[r] -> stop (or light end)
enum { kScanEdges = 0, kScanRoots = 1, kScanPlain = 2, kScanDense = 3 };
// the `light_phase` argument of the scans: which loop the round belongs to
// kPhaseLightRetire: a light-phase round whose hook retires isolated
// components (see "retirement" at k_hook_decide): its root count covers the
// components that still have edges only, so <= 1 of them ends the light
// phase, not the MST
enum { kPhasePlain = 0, kPhaseLight = 1, kPhaseSharded = 2, kPhaseLightRetire = 3 };
constexpr uint32_t kFusedScanMaxTiles = 16384;  // one block scans <= this many counts

template <int kKind>
__device__ __forceinline__ void scan_verdict(DevCounters* ctr, int r, uint32_t total, int light_phase) {
  if (kKind == kScanEdges) {
    ctr->m[r + 1] = total;
    // a shard holding no edge says nothing about the others: the sharded
    // loop stops on the replicated hook verdict only
    if (total == 0) {
      if (light_phase == kPhaseLight)
        ctr->phase_end = (uint32_t)r + 1;
      else if (light_phase == kPhasePlain && ctr->stop_round == kNoStop)
        ctr->stop_round = (uint32_t)r + 1;
    }
  } else if (kKind == kScanRoots) {
    ctr->n[r + 1] = total;
    if (light_phase == kPhaseLightRetire) {
      // retired components are final: nothing left with an edge ends the
      // light phase at round r + 1 (round 1: no light edge at all, which the
      // host answers with the plain loop); one component with edges left ends
      // it once its last (internal) edges are dropped by the compaction
      if (total == 0)
        ctr->phase_end = r == 1 ? 1u : (uint32_t)r + 1;
      else if (total == ctr->n[r])
        ctr->phase_end = (uint32_t)r;  // no progress (a round without retirement after retiring ones)
    } else if (total <= 1) {
      ctr->stop_round = (uint32_t)r + 1;
    } else if (total == ctr->n[r]) {
      // no live edge anywhere: done (a forest if total > 1), unless this is
      // the light phase of Filter-Boruvka, which then simply ends
      if (light_phase == kPhaseLight)
        ctr->phase_end = (uint32_t)r;
      else
        ctr->stop_round = (uint32_t)r + 1;
    }
  } else if (kKind == kScanDense) {
    ctr->n[r] = total;  // the light phase's final component count (retirement)
  } else {
    ctr->m[kMaxR - 1] = total;
  }
}

// Exclusive in-place scan of counts[0..T) by ONE block of kBlock threads
// (chunks of kBlock*8 with a running offset). Returns the total.
__device__ __forceinline__ uint32_t block_scan_counts(uint32_t* counts, uint32_t T, uint32_t* s_warp) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t running = 0;
  for (uint32_t base = 0; base < T; base += kBlock * 8) {
    const uint32_t i0 = base + threadIdx.x * 8;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = i0 + k < T ? __ldcg(counts + i0 + k) : 0u;
      sum += v[k];
    }
    const uint32_t incl = warp_incl_scan(sum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t wv = lane < kWarps ? s_warp[lane] : 0u;
      const uint32_t wi = warp_incl_scan(wv);
      if (lane < kWarps) s_warp[lane] = wi - wv;
      if (lane == 31) s_warp[kWarps] = wi;
    }
    __syncthreads();
    uint32_t run = running + s_warp[warp] + incl - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (i0 + k < T) counts[i0 + k] = run;
      run += v[k];
    }
    running += s_warp[kWarps];
    __syncthreads();
  }
  return running;
}

// Last-block-done: every block fences its count writes and checks in; the
// block that checks in last scans all T counts and publishes the verdict.
template <int kKind>
__device__ __forceinline__ void fused_scan_if_last(uint32_t* counts, uint32_t T, DevCounters* ctr, int r, int slot,
                                                   int light_phase, uint32_t* s_warp, uint32_t* s_flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *s_flag = atomicAdd(&ctr->done[r][slot], 1u) == gridDim.x - 1 ? 1u : 0u;
  __syncthreads();
  if (*s_flag) {
    __threadfence();
    const uint32_t total = block_scan_counts(counts, T, s_warp);
    if (threadIdx.x == 0) {
      scan_verdict<kKind>(ctr, r, total, light_phase);
      // every block has checked in: re-arm the counter, so a round index
      // that runs twice (the light phase's last round is phase D's first)
      // finds it at zero
      ctr->done[r][slot] = 0;
    }
  }
}

// ------------------------------ two-pass ordered compaction ----------------
// The single-pass look-back above leaves each tile ~10 us in flight (its
// aggregate needs the tile's loads + gathers first), which caps a pass at
// ~1/3 of HBM bandwidth (tools/lookback_bench.cu). Here the work is split:
//   k_count : per-tile keep counts, no inter-tile dependency (streams at
//             near copy speed); round compactions relabel in place, the
//             filter passes record the keep flags as a bitmask (one ballot
//             word per 32 consecutive edges);
//   k_emit  : ordered write + fused offers; a tile's aggregate is just
//             counts[tile], so it is published the moment the tile is taken
//             and the look-back overlaps the tile's own loads.
enum { kModeRelabel = 0, kModeLight = 1, kModeHeavy = 2, kModeDedup = 3 };

// ------------------------------ pair dedup ---------------------------------
// When few components carry many edges (a "dense core": R-MAT hubs, the
// giant component of a light phase), Boruvka keeps every parallel edge
// between the same two components alive for several rounds. Only the
// lightest edge of a component pair can be in the MST (cycle property), so a
// round may keep just that one: relabel + insert (pair -> lightest key) into
// an open-addressing table, then keep an edge iff it is its pair's minimum.
// Decided on the device per round from the active-component count:
// components with a live edge at round r+1 <= active[r]/2, so pairs <=
// (active[r]/2)^2/2; dedup when that is < m_r/4.
struct PairTable {
  unsigned long long* pairs;  // slot i = {pair, min key} at pairs[2i], pairs[2i+1]: one sector
  unsigned long long cap;     // power of two, allocated slots
};
constexpr unsigned long long kNoPair = ~0ull;
constexpr int kPairProbes = 64;
constexpr unsigned long long kDedupActive = 262144;

__device__ __forceinline__ unsigned long long pair_hash(unsigned long long p) {
  p ^= p >> 33;
  p *= 0xff51afd7ed558ccdull;
  p ^= p >> 33;
  return p;
}

// Relabel in place and record each pair's lightest (w<<32 | index) key
// (the first pass of a dedup round, run by k_count<kModeRelabel>).
__device__ __forceinline__ void dedup_insert(uint4* __restrict__ E, const uint32_t* __restrict__ L, PairTable t,
                                             DevCounters* ctr, int r) {
  const uint64_t m_r = ctr->m[r];
  const unsigned long long mask = ctr->pair_mask[r];
  const unsigned int limit = (unsigned int)((mask + 1) / 2);  // half load
  volatile unsigned int* abort_flag = &ctr->pair_abort[r];
  constexpr int kU = 4;
  for (uint64_t base = (uint64_t)blockIdx.x * kBlock * kU; base < m_r; base += (uint64_t)gridDim.x * kBlock * kU) {
    uint4 e[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * kBlock + threadIdx.x;
      e[k] = i < m_r ? __ldcs(E + i) : make_uint4(0, 0, 0, 0);
    }
    const bool aborted = *abort_flag != 0;
    uint32_t fresh = 0;
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * kBlock + threadIdx.x;
      if (i >= m_r) continue;
      const uint32_t x = __ldg(L + e[k].x), y = __ldg(L + e[k].y);
      E[i] = make_uint4(x, y, e[k].z, e[k].w);  // whole entry (see k_count)
      if (x == y || aborted) continue;
      const unsigned long long pair = ((unsigned long long)min(x, y) << 32) | max(x, y);
      const unsigned long long key = ((unsigned long long)e[k].z << 32) | (uint32_t)i;
      unsigned long long h = pair_hash(pair) & mask;
      for (int probe = 0; probe < kPairProbes; ++probe) {
        // through L1 (hot pairs: the giant's): a claimed slot never changes, a
        // stale empty one is settled by the CAS, a stale key only costs an atomic
        const unsigned long long cur = __ldca(t.pairs + 2 * h);
        const unsigned long long got = cur == pair ? pair : atomicCAS(t.pairs + 2 * h, kNoPair, pair);
        if (got == kNoPair || got == pair) {
          fresh += got == kNoPair;
          if (key < __ldca(t.pairs + 2 * h + 1)) atomicMin(t.pairs + 2 * h + 1, key);
          break;
        }
        h = (h + 1) & mask;  // a failed insert keeps the edge (see pair_keep)
      }
    }
    fresh = warp_sum<uint32_t>(fresh);
    if (lane_id() == 0 && fresh && atomicAdd(&ctr->pair_count[r], fresh) + fresh > limit) {
      *abort_flag = 1;
      ctr->dedup_fail = 1;
    }
  }
}

__device__ __forceinline__ bool pair_keep(const PairTable& t, unsigned long long mask, uint32_t x, uint32_t y,
                                          unsigned long long key) {
  const unsigned long long pair = ((unsigned long long)min(x, y) << 32) | max(x, y);
  unsigned long long h = pair_hash(pair) & mask;
  for (int probe = 0; probe < kPairProbes; ++probe) {
    const ulonglong2 slot = __ldca(reinterpret_cast<const ulonglong2*>(t.pairs) + h);  // read-only in this pass
    const unsigned long long cur = slot.x;
    if (cur == pair) return key <= slot.y;
    if (cur == kNoPair) return true;
    h = (h + 1) & mask;
  }
  return true;
}

template <class View, int kMode, bool kBatch = false>
__global__ void MST_LB_(MST_MINB_COUNT) k_count(View in, uint4* __restrict__ relabeled,
                                                  const uint32_t* __restrict__ L,
                                                  uint32_t* __restrict__ masks, uint32_t* __restrict__ counts,
                                                  uint32_t n_orig, DevCounters* ctr, int r, int fused, int slot,
                                                  int light_phase, PairTable pt,
                                                  unsigned long long* __restrict__ min_next, int filt,
                                                  const uint32_t* __restrict__ gbits, uint32_t ileave) {
  pdl_prologue();
  __shared__ uint32_t s_cnt[kWarps];
  __shared__ uint32_t s_slot[kCItems * kWarps];
  const uint32_t stop = ctr->stop_round;
  if ((uint32_t)r >= ctr->phase_end || (uint32_t)r + 1 >= stop) return;
  // A dedup round: this pass relabels + inserts pairs, the kModeDedup pass
  // counts (and stages survivors unless the attempt aborted).
  if (kMode == kModeRelabel && !View::kOriginal && pt.pairs && ctr->dedup[r]) {
    dedup_insert(reinterpret_cast<uint4*>(relabeled), L, pt, ctr, r);
    return;
  }
  if (kMode == kModeDedup && !ctr->dedup[r]) return;
  const uint64_t m_r = (kMode == kModeRelabel || kMode == kModeDedup) && !View::kOriginal ? ctr->m[r] : ctr->m[0];
  const unsigned long long pmask = kMode == kModeDedup ? ctr->pair_mask[r] : 0ull;
  const bool pabort = kMode == kModeDedup && ctr->pair_abort[r] != 0;
  const uint32_t pivot = ctr->pivot;
  // giant bits (relabel rounds of huge component counts, see k_giant_bits):
  // an endpoint whose bit is set takes the giant's label without a gather
  constexpr bool kGiant = kMode == kModeRelabel && !View::kOriginal;
  const uint32_t giant = (kGiant && gbits) ? ctr->giant : 0u;
  const uint32_t ntiles = (uint32_t)((m_r + kCTile - 1) / kCTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  // Interleaved tile order: the list is cut into S equal segments and the
  // grid walks them round-robin, so regions of a different character are in
  // flight together instead of one after the other (the BASELINE generators
  // put the uniform-random spanning tree first: its label gathers are
  // DRAM-random-bound, the R-MAT block's are L1-request-bound). Per-tile
  // outputs are indexed by the tile itself, so nothing else changes.
  const uint32_t S = (View::kOriginal && ileave > 1 && ntiles >= 4 * ileave) ? ileave : 1u;
  const uint32_t seg = (ntiles + S - 1) / S;
  const uint32_t nvt = seg * S;
  for (uint32_t vt = blockIdx.x; vt < nvt; vt += gridDim.x) {
    const uint32_t tile = S > 1 ? (vt % S) * seg + vt / S : vt;
    if (tile >= ntiles) continue;
    EdgeRec e[kCItems];
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
      e[k] = EdgeRec{0, 0, 0, 0, false};
      if (i < m_r) e[k] = in.stream(i);
    }
    uint32_t gwa[kCItems], gwb[kCItems];  // giant words of the endpoints, all in flight first
    if (kGiant && gbits) {
#pragma unroll
      for (int k = 0; k < kCItems; ++k) {
        const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
        gwa[k] = i < m_r ? __ldg(gbits + (e[k].a >> 5)) : 0u;
        gwb[k] = i < m_r ? __ldg(gbits + (e[k].b >> 5)) : 0u;
      }
    }
    uint32_t err = 0, cnt = 0;
    bool keep[kCItems];
    unsigned bal[kCItems];
    uint32_t ofx[kCItems], ofy[kCItems];
    unsigned long long okey[kCItems];
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
      keep[k] = false;
      uint32_t ox = e[k].a, oy = e[k].b;  // the endpoint labels of round r+1
      if (i < m_r) {
        bool ok = true;
        if (View::kOriginal) {
          // every input edge is range/weight checked in the first pass over
          // the caller's list (the light pass may be the only one)
          ok = e[k].a < n_orig && e[k].b < n_orig && e[k].ok;
          if (!ok) err |= (e[k].a < n_orig && e[k].b < n_orig) ? kErrWeight : kErrRange;
        }
        if (kMode == kModeLight) {
          keep[k] = ok && e[k].w < pivot && e[k].a != e[k].b;
        } else if (kMode == kModeDedup) {
          keep[k] = e[k].a != e[k].b &&
                    (pabort || pair_keep(pt, pmask, e[k].a, e[k].b, ((unsigned long long)e[k].w << 32) | (uint32_t)i));
        } else if (kMode == kModeHeavy) {
          if (ok && e[k].w >= pivot) {
            if (L) {
              e[k].a = __ldg(L + e[k].a);
              e[k].b = __ldg(L + e[k].b);
            }
            keep[k] = e[k].a != e[k].b;
          }
        } else if (View::kMayBeDead && e[k].a == e[k].b) {
          // dead since an earlier round: no gather, no write (stays a == b)
        } else if (ok) {
          if (kGiant && gbits) {
            ox = ((gwa[k] >> (e[k].a & 31)) & 1u) ? giant : __ldg(L + e[k].a);
            oy = ((gwb[k] >> (e[k].b & 31)) & 1u) ? giant : __ldg(L + e[k].b);
          } else {
            ox = __ldg(L + e[k].a);
            oy = __ldg(L + e[k].b);
          }
          keep[k] = ox != oy;
          if (View::kOriginal)
            __stcs(reinterpret_cast<uint2*>(relabeled) + i, make_uint2(ox, oy));
          else
            // the whole 16 B entry: an 8 B store into it is a partial-sector
            // write, merged in L2 (or read back from DRAM once evicted)
            __stcs(relabeled + i, make_uint4(ox, oy, e[k].w, e[k].eid));
        } else if (View::kOriginal && kMode == kModeRelabel) {
          __stcs(reinterpret_cast<uint2*>(relabeled) + i, make_uint2(0, 0));  // rejected edge: a self-loop
        }
      }
      // Offers for round r+1, keyed by the position in THIS list (the
      // relabelled input, which round r+1's hook gathers from), so they
      // need no output position and leave the emit pass a pure copy. The
      // light split and the heavy filter keep few, scattered survivors of a
      // DRAM-sized stream: their offers are made by output position in
      // k_emit_staged, where they do not stall the stream (c3 split: 1.8 ms
      // there vs 3.1 ms here).
      ofx[k] = ox;
      ofy[k] = oy;
      okey[k] = ((unsigned long long)e[k].w << 32) | (uint32_t)i;
      if ((kMode == kModeRelabel || kMode == kModeDedup) && !kBatch && keep[k]) {
        // one offer at a time, as each edge is decided (hub-heavy tables)
        offer(min_next, ox, okey[k], true, filt);
        offer(min_next, oy, okey[k], true, filt);
      }
      bal[k] = __ballot_sync(0xffffffffu, keep[k]);
      if (lane == 0) s_slot[k * kWarps + warp] = __popc(bal[k]);
      cnt += __popc(bal[k]);
    }
    if ((kMode == kModeRelabel || kMode == kModeDedup) && kBatch)
      offer_both<kCItems>(min_next, ofx, ofy, okey, keep, 2 | (filt & kFiltCached));
    if (err) atomicOr(&ctr->err, err);
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    if (kMode != kModeRelabel && !pabort) {
      // sparse survivors: stage them compacted inside the tile's own slice,
      // so the emit pass touches survivors only
      if (warp == 0) {
        constexpr int kSlots = kCItems * kWarps, kPer = (kSlots + 31) / 32;
        uint32_t v[kPer], sum = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int idx = lane * kPer + j;
          v[j] = idx < kSlots ? s_slot[idx] : 0u;
          sum += v[j];
        }
        const uint32_t incl = warp_incl_scan(sum);
        uint32_t run = incl - sum;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int idx = lane * kPer + j;
          if (idx < kSlots) s_slot[idx] = run;
          run += v[j];
        }
      }
      __syncthreads();
      const uint32_t lt = lanemask_lt();
#pragma unroll
      for (int k = 0; k < kCItems; ++k)
        if (keep[k])
          __stcs(relabeled + (uint64_t)tile * kCTile + s_slot[k * kWarps + warp] + __popc(bal[k] & lt),
                 make_uint4(e[k].a, e[k].b, e[k].w, e[k].eid));
    }
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) t += s_cnt[w];
      counts[tile] = t;
    }
    __syncthreads();
  }
  if (fused) {
    __shared__ uint32_t s_warp[kWarps + 1], s_flag;
    fused_scan_if_last<kScanEdges>(counts, ntiles, ctr, r, slot, light_phase, s_warp, &s_flag);
  }
}

template <class View, int kMode>
__global__ void MST_LB_(MST_MINB_EMIT) k_emit(View in, const uint4* __restrict__ relabeled,
                                                 const uint32_t* __restrict__ L,
                                                 const uint32_t* __restrict__ masks,
                                                 const uint32_t* __restrict__ offsets, uint4* __restrict__ out,
                                                 DevCounters* ctr, int r, int dedup_armed, uint32_t n_orig) {
  pdl_prologue();
  __shared__ uint32_t s_scan[kCItems * kWarps];
  const uint32_t stop = ctr->stop_round;
  if ((uint32_t)r >= ctr->phase_end || (uint32_t)r + 1 >= stop) return;
  if (kMode == kModeRelabel && !View::kOriginal && dedup_armed && ctr->dedup[r] && !ctr->pair_abort[r]) return;
  if (kMode == kModeDedup && !ctr->dedup[r]) return;
  const uint64_t m_r = (kMode == kModeRelabel || kMode == kModeDedup) && !View::kOriginal ? ctr->m[r] : ctr->m[0];
  const uint32_t ntiles = (uint32_t)((m_r + kCTile - 1) / kCTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint4 e[kCItems];
    unsigned bal[kCItems];
    bool keep[kCItems];
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
      e[k] = make_uint4(0, 0, 0, 0);
      if (kMode == kModeRelabel && View::kOriginal) {
        // plain round 1: the count pass left the new endpoint labels as an
        // 8 B pair per edge; weight from the caller's list, id = position
        if (i < m_r) {
          const uint2 xy = __ldcs(reinterpret_cast<const uint2*>(relabeled) + i);
          e[k] = make_uint4(xy.x, xy.y, in.weight(i), in.base + (uint32_t)i);
        }
      } else if (kMode == kModeRelabel) {
        if (i < m_r) e[k] = __ldcs(relabeled + i);
      } else {
        bal[k] = __ldg(masks + (uint64_t)tile * (kCItems * kWarps) + k * kWarps + warp);
        if ((bal[k] >> lane) & 1u) {
          const EdgeRec x = in.gather(i);
          e[k] = make_uint4(x.a, x.b, x.w, x.eid);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      if (kMode == kModeRelabel) {
        const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
        keep[k] = i < m_r && e[k].x != e[k].y;
        bal[k] = __ballot_sync(0xffffffffu, keep[k]);
      } else {
        keep[k] = (bal[k] >> lane) & 1u;
        if (kMode == kModeHeavy && keep[k] && L) {
          e[k].x = __ldg(L + e[k].x);
          e[k].y = __ldg(L + e[k].y);
        }
      }
      if (lane == 0) s_scan[k * kWarps + warp] = __popc(bal[k]);
    }
    __syncthreads();
    if (warp == 0) {
      constexpr int kSlots = kCItems * kWarps, kPer = (kSlots + 31) / 32;
      uint32_t v[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int idx = lane * kPer + j;
        v[j] = idx < kSlots ? s_scan[idx] : 0u;
        sum += v[j];
      }
      const uint32_t incl = warp_incl_scan(sum);
      uint32_t run = incl - sum;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int idx = lane * kPer + j;
        if (idx < kSlots) s_scan[idx] = run;
        run += v[j];
      }
    }
    __syncthreads();
    const uint32_t prefix = __ldg(offsets + tile);
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint32_t j = prefix + s_scan[k * kWarps + warp] + __popc(bal[k] & lt);
      if (keep[k]) __stcs(out + j, e[k]);
    }
    __syncthreads();
  }
}

// Emit of the staged modes: tile t's survivors sit at stage[t*kCTile ..
// t*kCTile + count); copy them to their final slots (and, for the light
// split and the heavy filter, make the offers by output position).
template <int kMode, bool kBatch = false>
__global__ void __launch_bounds__(kBlock) k_emit_staged(const uint4* __restrict__ stage,
                                                        const uint32_t* __restrict__ offsets, uint4* __restrict__ out,
                                                        unsigned long long* __restrict__ min_next, DevCounters* ctr,
                                                        int r, int filt) {
  pdl_prologue();
  const uint32_t stop = ctr->stop_round;
  if ((uint32_t)r >= ctr->phase_end || (uint32_t)r + 1 >= stop) return;
  if (kMode == kModeDedup && (!ctr->dedup[r] || ctr->pair_abort[r])) return;
  const uint64_t m_src = kMode == kModeDedup ? ctr->m[r] : ctr->m[0];
  const uint32_t total = (uint32_t)ctr->m[r + 1];
  const uint32_t ntiles = (uint32_t)((m_src + kCTile - 1) / kCTile);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t off = __ldg(offsets + tile);
    const uint32_t end = tile + 1 < ntiles ? __ldg(offsets + tile + 1) : total;
    const uint32_t cnt = end - off;
    if constexpr (!kBatch) {
      for (uint32_t base = 0; base < cnt; base += kBlock) {
        const uint32_t j = base + threadIdx.x;
        const bool v = j < cnt;
        const uint4 e = v ? __ldcs(stage + (uint64_t)tile * kCTile + j) : make_uint4(0, 0, 0, 0);
        if (v) __stcs(out + off + j, e);
        if ((kMode == kModeHeavy || kMode == kModeLight) && min_next) {  // null: k_range_offers does them
          const unsigned long long key = ((unsigned long long)e.z << 32) | (off + j);
          offer(min_next, e.x, key, v, filt);
          offer(min_next, e.y, key, v, filt);
        }
      }
    } else {
      for (uint32_t base = 0; base < cnt; base += kBlock * kCItems) {
        uint4 e[kCItems];
        bool v[kCItems];
        uint32_t x[kCItems], y[kCItems];
        unsigned long long key[kCItems];
#pragma unroll
        for (int k = 0; k < kCItems; ++k) {
          const uint32_t j = base + k * kBlock + threadIdx.x;
          v[k] = j < cnt;
          e[k] = v[k] ? __ldcs(stage + (uint64_t)tile * kCTile + j) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < kCItems; ++k) {
          const uint32_t j = base + k * kBlock + threadIdx.x;
          if (v[k]) __stcs(out + off + j, e[k]);
          x[k] = e[k].x;
          y[k] = e[k].y;
          key[k] = ((unsigned long long)e[k].z << 32) | (off + j);
        }
        if ((kMode == kModeHeavy || kMode == kModeLight) && min_next)
          offer_both<kCItems>(min_next, x, y, key, v, 2 | (filt & kFiltCached));
      }
    }
  }
}

// Pure copy of the staged survivors (the split / heavy filter with range
// offers): tile t's ~10 % survivors sit at stage[t*kCTile ..), so a block
// per tile leaves most lanes idle and the pass latency-bound on the per-tile
// offsets (c4 split: 3.4 TB/s). Here a warp takes 32 consecutive tiles,
// reads their 33 offsets in one load and copies each tile with up to
// 4 x 32 loads in flight.
__global__ void __launch_bounds__(kBlock) k_emit_sparse(const uint4* __restrict__ stage,
                                                        const uint32_t* __restrict__ offsets, uint4* __restrict__ out,
                                                        DevCounters* ctr, int r) {
  pdl_prologue();
  const uint32_t stop = ctr->stop_round;
  if ((uint32_t)r >= ctr->phase_end || (uint32_t)r + 1 >= stop) return;
  const uint64_t m_src = ctr->m[0];
  const uint32_t total = (uint32_t)ctr->m[r + 1];
  const uint32_t ntiles = (uint32_t)((m_src + kCTile - 1) / kCTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t groups = (ntiles + 31) / 32;
  for (uint32_t g = blockIdx.x * kWarps + warp; g < groups; g += gridDim.x * kWarps) {
    const uint32_t t0 = g * 32;
    const uint32_t my = t0 + lane;
    const uint32_t off_l = my < ntiles ? __ldg(offsets + my) : total;
    const uint32_t nxt = __shfl_down_sync(0xffffffffu, off_l, 1);
    const uint32_t end_l = lane < 31 ? nxt : (my + 1 < ntiles ? __ldg(offsets + my + 1) : total);
    const uint32_t tiles = min(32u, ntiles - t0);
    for (uint32_t t = 0; t < tiles; ++t) {
      const uint32_t off = __shfl_sync(0xffffffffu, off_l, t);
      const uint32_t cnt = __shfl_sync(0xffffffffu, end_l, t) - off;
      const uint4* src = stage + (uint64_t)(t0 + t) * kCTile;
      for (uint32_t base = 0; base < cnt; base += 128) {
        uint4 e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t j = base + k * 32 + lane;
          if (j < cnt) e[k] = __ldcs(src + j);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t j = base + k * 32 + lane;
          if (j < cnt) __stcs(out + off + j, e[k]);
        }
      }
    }
  }
}

// Range passes (the split's and the heavy filter's offers): their min tables
// are DRAM-sized (c4: 537 / 376 MB), so an offer straight from the emit
// costs a 64 B DRAM fetch. Instead the emit only copies, and the output list
// is streamed once per slice [lo, hi) of the table (128 MB by default):
// each pass offers the endpoints whose label falls in its slice, keyed by
// list position exactly like the emit would. The list itself is read with
// evict-first loads, so the slice stays in L2. The minimum does not depend
// on the order of the offers.
__global__ void __launch_bounds__(kBlock) k_range_offers(const uint4* __restrict__ E, const DevCounters* ctr, int r,
                                                         unsigned long long* __restrict__ table, uint32_t lo,
                                                         uint32_t hi, int filt) {
  pdl_prologue();
  if ((uint32_t)r >= ctr->phase_end || (uint32_t)r + 1 >= ctr->stop_round) return;  // as the emit
  const uint64_t m = ctr->m[r + 1];
  const uint32_t span = hi - lo;
  constexpr int kU = 4;
  for (uint64_t base = (uint64_t)blockIdx.x * kBlock * kU; base < m; base += (uint64_t)gridDim.x * kBlock * kU) {
    uint4 e[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * kBlock + threadIdx.x;
      e[k] = i < m ? __ldcs(E + i) : make_uint4(0, 0, 0, 0);
    }
    uint32_t x[kU], y[kU];
    unsigned long long key[kU];
    bool vx[kU], vy[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t i = base + k * kBlock + threadIdx.x;
      x[k] = e[k].x;
      y[k] = e[k].y;
      key[k] = ((unsigned long long)e[k].z << 32) | (uint32_t)i;
      vx[k] = i < m && (x[k] - lo) < span;
      vy[k] = i < m && (y[k] - lo) < span;
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      offer(table, x[k], key[k], vx[k], filt);
      offer(table, y[k], key[k], vy[k], filt);
    }
  }
}

// ------------------------------ tile-count scan ----------------------------
// Exclusive scan of per-tile counts in place (8192 counts per block, chained
// with the look-back across <= a few hundred blocks), so the emit passes need
// no inter-tile communication at all. The last block also publishes the
// total and the round verdict (scan_verdict). Small scans are instead fused
// into the counting kernel (fused_scan_if_last) and cost no launch.
constexpr int kScanItems = 8;
constexpr int kScanBlock = 1024;
constexpr int kScanTile = kScanBlock * kScanItems;

template <int kKind>
__global__ void __launch_bounds__(kScanBlock) k_scan_counts(uint32_t* __restrict__ counts, uint64_t ntiles_max,
                                                             DevCounters* ctr, int r, unsigned long long* status,
                                                             uint32_t epoch, int light_phase, int count_src) {
  pdl_prologue();
  __shared__ uint32_t s_warp[kScanBlock / 32];
  __shared__ uint32_t s_misc[2];
  if (kKind == kScanEdges || kKind == kScanRoots) {
    if ((uint32_t)r >= ctr->phase_end) return;
    if (kKind == kScanEdges && (uint32_t)r + 1 >= ctr->stop_round) return;
    if (kKind == kScanRoots && (uint32_t)r >= ctr->stop_round) return;
  }
  // number of tiles actually in use this round
  uint64_t n_items;
  if (kKind == kScanRoots)
    n_items = (ctr->n[r] + (uint64_t)kTile - 1) / kTile;
  else if (kKind == kScanEdges)
    n_items = ((count_src ? ctr->m[0] : ctr->m[r]) + (uint64_t)kCTile - 1) / kCTile;
  else
    n_items = ntiles_max;  // kScanPlain, kScanDense
  const uint32_t nblocks = (uint32_t)((n_items + kScanTile - 1) / kScanTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t blk = blockIdx.x; blk < max(nblocks, 1u); blk += gridDim.x) {
    const uint64_t base = (uint64_t)blk * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      v[k] = base + k < n_items ? counts[base + k] : 0u;
      sum += v[k];
    }
    const uint32_t incl = warp_incl_scan(sum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t wv = s_warp[lane];
      const uint32_t wi = warp_incl_scan(wv);
      s_warp[lane] = wi - wv;
      const uint32_t tot = __shfl_sync(0xffffffffu, wi, 31);
      const uint32_t ex = lookback(status, blk, tot, epoch);
      if (lane == 0) {
        s_misc[0] = ex;
        s_misc[1] = tot;
      }
    }
    __syncthreads();
    uint32_t run = s_misc[0] + s_warp[warp] + incl - sum;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (base + k < n_items) counts[base + k] = run;
      run += v[k];
    }
    if (blk == max(nblocks, 1u) - 1 && threadIdx.x == 0) scan_verdict<kKind>(ctr, r, s_misc[0] + s_misc[1], light_phase);
    __syncthreads();
  }
}

// ------------------------------ sharded exchange ---------------------------
// Each shard holds a contiguous slice of the caller's edge list (global id =
// base + local index) and runs the same rounds with replicated component
// state. A shard's local table has literal keys (w << 32 | position in the
// shard's current list); since compaction keeps list order, the position
// order is the global id order, so the local minimum is also the minimum of
// (w, global id). Per round:
//   k_shard_keys    : xch[c] = (w << 32 | global id), own[c] = (id, partner)
//   allreduce(min, u64) of xch        -> the global lightest edge per component
//   k_shard_partner : partner[c] = own partner if this shard owns xch[c], else ~0
//   allreduce(min, u32) of partner    -> the other endpoint's label
// and k_hook_decide<_, kExchanged> then hooks exactly like the single-device
// loop (same keys, same tie order, MST ids straight from the keys).
struct PartnerView {
  static constexpr bool kOriginal = false;
  static constexpr bool kMayBeDead = false;
  const uint32_t* partner;
};

template <class View>
__global__ void __launch_bounds__(kBlock) k_shard_keys(View E, const unsigned long long* __restrict__ minimum,
                                                       unsigned long long* __restrict__ xch,
                                                       unsigned long long* __restrict__ own, DevCounters* ctr, int r) {
  pdl_prologue();
  if ((uint32_t)r >= ctr->stop_round || (uint32_t)r >= ctr->phase_end) return;
  const uint32_t n_r = ctr->n[r];
  for (uint64_t c = (uint64_t)blockIdx.x * kBlock + threadIdx.x; c < n_r; c += (uint64_t)gridDim.x * kBlock) {
    const unsigned long long key = __ldcs(minimum + c);
    unsigned long long x = kNoKey, o = kNoKey;
    if (key != kNoKey) {
      const EdgeRec e = E.gather((uint32_t)key);
      const uint32_t partner = e.a == (uint32_t)c ? e.b : e.a;
      x = (key & 0xFFFFFFFF00000000ull) | e.eid;
      o = ((unsigned long long)e.eid << 32) | partner;
    }
    xch[c] = x;
    own[c] = o;
  }
}

__global__ void __launch_bounds__(kBlock) k_shard_partner(const unsigned long long* __restrict__ xch,
                                                          const unsigned long long* __restrict__ own,
                                                          uint32_t* __restrict__ partner, DevCounters* ctr, int r) {
  pdl_prologue();
  if ((uint32_t)r >= ctr->stop_round || (uint32_t)r >= ctr->phase_end) return;
  const uint32_t n_r = ctr->n[r];
  for (uint64_t c = (uint64_t)blockIdx.x * kBlock + threadIdx.x; c < n_r; c += (uint64_t)gridDim.x * kBlock) {
    const unsigned long long x = __ldcs(xch + c), o = __ldcs(own + c);
    // ids are unique across shards: exactly one shard owns the winner
    partner[c] = (x != kNoKey && o != kNoKey && (uint32_t)x == (uint32_t)(o >> 32)) ? (uint32_t)o : kNone;
  }
}

// ------------------------------ hook ---------------------------------------
// k_hook_decide: per component, the partner along its lightest edge, the
// mutual-pair root rule, parent[], the MST flag of the edge, a root bitmask,
// in-tile root prefixes and per-tile root counts; k_label2 turns the scanned
// counts into dense root labels.
// kExchanged: the sharded loop. minimum[c] holds the all-reduced global
// key (w << 32 | global edge id) and E.partner[c] the other endpoint's label
// of that edge (all-reduced too), so nothing is gathered from an edge list.
template <class View, bool kExchanged = false>
__global__ void MST_LB_(MST_MINB_HOOK) k_hook_decide(View E, const unsigned long long* __restrict__ minimum,
                                                        uint32_t* __restrict__ parent,
                                                        uint32_t* __restrict__ masks, uint32_t* __restrict__ counts,
                                                        DevCounters* ctr, int r, int fused, int light_phase,
                                                        uint32_t* __restrict__ slotpref,
                                                        uint32_t* __restrict__ mst_bits, int mst_bytes,
                                                        uint32_t* __restrict__ rbits) {
  pdl_prologue();
  __shared__ uint32_t s_cnt[kWarps];
  __shared__ uint32_t s_slot[kItems * kWarps];
  __shared__ unsigned long long s_wsum[kWarps];
  if ((uint32_t)r >= ctr->stop_round || (uint32_t)r >= ctr->phase_end) return;
  const uint32_t n_r = ctr->n[r];
  const uint32_t ntiles = (uint32_t)(((uint64_t)n_r + kTile - 1) / kTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned long long wsum = 0;
  uint32_t active = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    unsigned long long key[kItems], okey[kItems];
    EdgeRec e[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t c = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      key[k] = c < n_r ? __ldcs(minimum + c) : kNoKey;
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      e[k] = EdgeRec{0, 0, 0, 0, true};
      if constexpr (kExchanged) {
        const uint32_t c = (uint32_t)((uint64_t)tile * kTile + k * kBlock + threadIdx.x);
        if (key[k] != kNoKey) e[k] = EdgeRec{c, __ldg(E.partner + c), (uint32_t)(key[k] >> 32), (uint32_t)key[k], true};
      } else {
        if (key[k] != kNoKey) e[k] = E.gather_ends((uint32_t)key[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint32_t c = (uint32_t)((uint64_t)tile * kTile + k * kBlock + threadIdx.x);
      const uint32_t o = (e[k].a == c) ? e[k].b : e[k].a;
      okey[k] = key[k] != kNoKey ? __ldg(minimum + o) : kNoKey;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t c = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      bool isroot = false, iso = false;
      if (c < n_r) {
        if (key[k] == kNoKey) {
          // no edge: a root; with rbits it is retired instead (final, no
          // label in round r+1's dense space)
          iso = rbits != nullptr;
          isroot = !iso;
          parent[c] = (uint32_t)c;
        } else {
          const uint32_t o = (e[k].a == (uint32_t)c) ? e[k].b : e[k].a;
          isroot = okey[k] == key[k] && (uint32_t)c < o;
          parent[c] = isroot ? (uint32_t)c : o;
          ++active;
          if (!isroot) {
            mst_mark(mst_bits, mst_bytes, e[k].eid);  // the MST edge (global id in the sharded loop)
            wsum += (uint32_t)(key[k] >> 32);
          }
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, isroot);
      if (rbits) {
        const unsigned rb = __ballot_sync(0xffffffffu, iso);
        const uint64_t c0 = (uint64_t)tile * kTile + k * kBlock + warp * 32;
        if (lane == 0 && c0 < n_r) rbits[c0 >> 5] = rb;
      }
      if (lane == 0) {
        masks[(uint64_t)tile * (kItems * kWarps) + k * kWarps + warp] = bal;
        s_slot[k * kWarps + warp] = __popc(bal);
      }
      cnt += __popc(bal);
    }
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    if (slotpref && warp == 0) {
      // in-tile exclusive root prefix per (item, warp) slot, for k_label2
      const uint32_t v = s_slot[lane];
      const uint32_t incl = warp_incl_scan(v);
      slotpref[(uint64_t)tile * 32 + lane] = incl - v;
    }
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) t += s_cnt[w];
      counts[tile] = t;
    }
    __syncthreads();
  }
  wsum = warp_sum<unsigned long long>(wsum);
  active = warp_sum<uint32_t>(active);
  if (lane == 0) {
    s_wsum[warp] = wsum;
    s_cnt[warp] = active;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    uint32_t a = 0;
    for (int i = 0; i < kWarps; ++i) {
      t += s_wsum[i];
      a += s_cnt[i];
    }
    if (t) atomicAdd(&ctr->total_weight, t);
    if (a) atomicAdd(&ctr->active[r], a);
  }
  if (fused) {
    __shared__ uint32_t s_warp[kWarps + 1], s_flag;
    fused_scan_if_last<kScanRoots>(counts, ntiles, ctr, r, 0, light_phase, s_warp, &s_flag);
  }
}

// ------------------------------ label --------------------------------------
// The dense label of a root is the number of roots before it; with the
// hook's root masks, per-tile offsets (scanned counts) and in-tile slot
// prefixes it is three small loads, so k_label2 finds every component's
// root and writes its next-round label in one pass.
__device__ __forceinline__ uint32_t roots_before(uint32_t x, const uint32_t* __restrict__ masks,
                                                 const uint32_t* __restrict__ slotpref,
                                                 const uint32_t* __restrict__ offsets) {
  const uint32_t t = x / kTile, rem = x % kTile;
  const uint32_t k = rem / kBlock, within = rem % kBlock;
  const uint32_t slot = k * kWarps + (within >> 5), lane = within & 31;
  const uint32_t m = __ldg(masks + (uint64_t)t * 32 + slot);
  return __ldg(offsets + t) + __ldg(slotpref + (uint64_t)t * 32 + slot) + __popc(m & ((1u << lane) - 1u));
}

__global__ void MST_LB_(MST_MINB_LABEL) k_label2(uint32_t* __restrict__ parent,
                                                   const uint32_t* __restrict__ masks,
                                                   const uint32_t* __restrict__ slotpref,
                                                   const uint32_t* __restrict__ offsets, uint32_t* __restrict__ L,
                                                   unsigned long long* __restrict__ min_next, DevCounters* ctr, int r,
                                                   unsigned long long* pair_keys, unsigned long long pair_cap,
                                                   unsigned int dedup_active, unsigned int pair_div,
                                                   const uint32_t* __restrict__ rbits = nullptr) {
  pdl_prologue();
  if ((uint32_t)r >= ctr->stop_round || (uint32_t)r >= ctr->phase_end) return;
  if ((uint32_t)r + 1 >= ctr->stop_round) return;  // the last hook round: its MST flags are all set
  const uint32_t n_r = ctr->n[r];
  const uint32_t n_next = ctr->n[r + 1];
  if (pair_keys) {
    // pair dedup decision for this round's compaction + table clear (see
    // "pair dedup"); tried when few active components carry many edges each
    const unsigned long long K = ctr->active[r];
    const unsigned long long m_r = ctr->m[r];
    // after an overflowed attempt (pairs mostly distinct: uniform graphs),
    // try again only once K(K-1)/2 pairs guarantee an 8x reduction;
    // R-MAT's repeated hub pairs keep succeeding and are not held back
    const bool doubtful = ctr->dedup_fail && K * (K - 1) / 2 > m_r / 8 && !(pair_div & 0x100u);
    // bits 24-31 of pair_div: only when the n_next components of the next
    // round can form at most m_r / g distinct pairs, i.e. the dedup is
    // guaranteed to shrink the list g-fold. (Uniform graphs: c3's light round
    // 4 has 148 K active components, 9.4 M edges and almost as many distinct
    // pairs; the attempt overflowed its table and cost 0.4 ms.)
    const unsigned long long gfac = (pair_div >> 24) & 0xFFu;
    const unsigned long long pairs_next = (unsigned long long)n_next * (n_next > 0 ? n_next - 1 : 0) / 2;
    const bool guaranteed = gfac == 0 || pairs_next <= m_r / gfac;
    const bool use = K <= dedup_active && m_r >= ((pair_div >> 16) & 0xFFu) * K && m_r >= 4096 && !doubtful &&
                     guaranteed;
    // table >= m_r / div slots, but no more than twice the pairs the next
    // round's n_next components can form (after retirement they are few: c4
    // round 3, 825 components, 1 M slots in L2 instead of 32 M in DRAM:
    // 3.3 -> 1.05 ms) and no fewer than 256 K (a few hundred hot pairs
    // packed into a few KB serialise their inserts: c3 round 7, 0.15 vs
    // 0.65 ms with 2 K slots)
    const unsigned long long pairs_max = (unsigned long long)n_next * (n_next > 0 ? n_next - 1 : 0) / 2;
    const unsigned long long want = min(m_r / (pair_div & 0xFFu), max(2 * pairs_max, 1ull << 18));
    unsigned long long P = 1024;
    while (P < want && P < pair_cap) P <<= 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctr->dedup[r] = use ? 1u : 0u;
      ctr->pair_mask[r] = P - 1;
      ctr->pair_count[r] = 0;
      ctr->pair_abort[r] = 0;
    }
    if (use)
      for (unsigned long long i = (unsigned long long)blockIdx.x * kBlock + threadIdx.x; i < P;
           i += (unsigned long long)gridDim.x * kBlock)
        reinterpret_cast<ulonglong2*>(pair_keys)[i] = make_ulonglong2(~0ull, ~0ull);
  }
  const uint32_t ntiles = (uint32_t)(((uint64_t)n_r + kTile - 1) / kTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t toff = __ldg(offsets + tile);
    uint32_t c[kItems], root[kItems], own[kItems];
    bool v[kItems], isroot[kItems], iso[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      c[k] = tile * kTile + k * kBlock + threadIdx.x;
      v[k] = c[k] < n_r;
      const uint32_t slot = k * kWarps + warp;
      const uint32_t m = __ldg(masks + (uint64_t)tile * 32 + slot);
      isroot[k] = (m >> lane) & 1u;
      own[k] = toff + __ldg(slotpref + (uint64_t)tile * 32 + slot) + __popc(m & lt);
      iso[k] = rbits != nullptr && v[k] && ((__ldg(rbits + (c[k] >> 5)) >> lane) & 1u);
    }
    bool walk[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) walk[k] = v[k] && !isroot[k] && !iso[k];
    find_roots<kItems>(parent, c, walk, root);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      if (!v[k]) continue;
      L[c[k]] = iso[k] ? (kRetFlag | c[k]) : isroot[k] ? own[k] : roots_before(root[k], masks, slotpref, offsets);
      if (c[k] < n_next) min_next[c[k]] = kNoKey;
    }
  }
}

// ------------------------------ tail megakernel ----------------------------

// Once a round has few live edges, per-round kernel launches, ramp-up/tail
// effects and look-back latency dominate. k_tail runs all remaining rounds
// in ONE cooperative launch (all blocks co-resident), three grid-wide steps
// per round, same hook rule, counters, keys and verdicts as the round
// kernels:
//   A: round r's hook decisions over the block's component chunk; each block
//      records its chunk's root bitmask and per-word root prefixes.
//   B: dense labels: roots_before(x) = block prefix + word prefix + popc,
//      root finding (path halving), MST slots of the hooked components,
//      clear of the next min table.
//   C: relabel + compact the block's own SEGMENT of the edge list in place
//      and make the offers (w << 32 | new position) for round r+1
//      (aggregated in a block-local shared-memory table when <=
//      kTailSmemMin components remain).
// The list is segmented: block b owns positions [b*es, b*es + len_b) of
// the entry list for the whole launch and compacts its segment in place, so
// no cross-block prefix and no second pass over the edges is needed.
// Segments keep list order, so position order is still edge-id order (the
// tie rule of the keys).
//
// Pair dedup (C0, optional per round): when the live edges outnumber the
// next round's components (m_r >= ratio * n_{r+1}), many edges join the
// same two components (grids and other low-genus graphs: <= 3 n_{r+1}
// distinct pairs; R-MAT cores). C0 relabels in place and records each
// pair's lightest key in a hash table; C then keeps only that edge (cycle
// property: exact). Slots carry a 16-bit tag (call epoch, round) in the
// pair word, so the table is never cleared between rounds; a slot is claimed
// with a 128-bit CAS of {pair, key}. A round whose dedup removed < half the
// edges turns it off until K(K-1)/2 <= m_r/4 guarantees the gain.
struct TailArgs {
  uint4* E[2];
  unsigned long long* minb[2];
  uint32_t* parent;
  uint32_t* L;
  uint32_t* broots;     // [gridDim.x] roots per block chunk (A -> B)
  uint32_t* masks;      // root bitmask, one word per 32 components
  uint32_t* wpref;      // roots of the block's chunk before each word
  uint32_t* M;          // light phase: entry-label -> current-label map (n[r0] entries)
  uint32_t* mst_bits;   // MST output: bitmap, or one byte per edge (mst_bytes)
  unsigned long long* trace;  // optional: globaltimer stamps at phase boundaries (block 0)
  // the list the entry round's keys index (kTailSrc*): a packed list, round
  // 1's label pairs with the caller's weights, or the caller's SoA / AoS list
  int src_kind;
  const void* src0;         // packed / pairs / SoA src / AoS records
  const uint32_t* src1;     // SoA dst
  const uint32_t* src_w;    // weights (pairs, SoA)
  uint32_t src_wstride;
  DevCounters* ctr;
  uint32_t n_orig;
  int r0;
  int light;
  // pair dedup (pairs == nullptr: off)
  ulonglong2* pairs;
  unsigned long long pair_cap;  // slots, power of two
  uint32_t pair_epoch;          // 1..1022, tag = epoch << 6 | round
  uint32_t dedup_ratio;
  uint32_t dedup_min;
  // tiny rounds (n_r <= kTailSmemMin, plain loop): three rotating min tables,
  // cleared by the host before the launch (nullptr: off)
  unsigned long long* tiny[3];
  // start_c: round r0 = 1 of the plain loop had its min / hook / label done by
  // the round kernels; the launch starts at its phase C, reading the caller's
  // SoA list (src0 / src1 / src_w) in place of round 1's count + emit passes
  int start_c;
  int c_soa;  // start_c's phase C reads the caller's SoA list (plain round 1), else the list E[r0 & 1]
  // light phase after retiring round kernels: components outside the tail's
  // label space exist, so one component left ends the light phase, not the MST
  int retired;
  int mst_bytes;
};

constexpr uint32_t kTailSmemMin = 2048;  // block-local min table entries (16 KB); tiny rounds up to this
constexpr uint32_t kTailMaxBlocks = 1024;
constexpr uint32_t kTailPairLabelBits = 24;
constexpr int kTailPairProbes = 64;

// Ordered ranks of kItems striped flags per thread; returns the total.
__device__ __forceinline__ uint32_t block_ranks(const bool (&f)[kItems], uint32_t (&rank)[kItems],
                                                uint32_t* s_cnt) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned bal[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    bal[k] = __ballot_sync(0xffffffffu, f[k]);
    if (lane == 0) s_cnt[k * kWarps + warp] = __popc(bal[k]);
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = s_cnt[lane];
    const uint32_t incl = warp_incl_scan(v);
    s_cnt[lane] = incl - v;
    if (lane == 31) s_cnt[32] = incl;
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < kItems; ++k) rank[k] = s_cnt[k * kWarps + warp] + __popc(bal[k] & lt);
  const uint32_t total = s_cnt[32];
  __syncthreads();
  return total;
}

// Exclusive prefix of cnt[0..G) into s_pre[0..G] (s_pre[G] = total), by the
// whole block.
__device__ __forceinline__ void block_scan_array(const uint32_t* cnt, uint32_t G, uint32_t* s_pre,
                                                 uint32_t* s_warp) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < G; base += kBlock) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < G ? __ldcg(cnt + i) : 0u;
    const uint32_t incl = warp_incl_scan(v);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t t = lane < kWarps ? s_warp[lane] : 0u;
      const uint32_t ti = warp_incl_scan(t);
      if (lane < kWarps) s_warp[lane] = ti - t;
      if (lane == kWarps - 1) s_warp[kWarps] = ti;
    }
    __syncthreads();
    if (i < G) s_pre[i] = carry + s_warp[warp] + incl - v;
    carry += s_warp[kWarps];
    __syncthreads();
  }
  if (threadIdx.x == 0) s_pre[G] = carry;
  __syncthreads();
}

__device__ __forceinline__ void tail_stamp(const TailArgs& a, int& slot) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && slot < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[slot] = t;
  }
  ++slot;
}

enum { kTailSrcPacked = 0, kTailSrcPairs = 1, kTailSrcSoa = 2, kTailSrcAos = 3 };

// Edge i of the list the entry round's keys index, as {a, b, -, id} (the
// hook has the weight in its key).
__device__ __forceinline__ uint4 tail_entry_edge(const TailArgs& a, uint32_t i) {
  switch (a.src_kind) {
    case kTailSrcPacked:
      return __ldcg(static_cast<const uint4*>(a.src0) + i);
    case kTailSrcPairs: {
      const uint2 p = __ldcg(static_cast<const uint2*>(a.src0) + i);
      return make_uint4(p.x, p.y, 0u, i);
    }
    case kTailSrcSoa:
      return make_uint4(__ldg(static_cast<const uint32_t*>(a.src0) + i), __ldg(a.src1 + i), 0u, i);
    default: {
      const uint4 v = __ldg(static_cast<const uint4*>(a.src0) + i);
      return make_uint4(v.x, v.y, v.z, i);
    }
  }
}

// Tagged pair word: tag(16) | min label(24) | max label(24).
__device__ __forceinline__ unsigned long long tail_pair_word(uint32_t tag, uint32_t x, uint32_t y) {
  const uint32_t lo = min(x, y), hi = max(x, y);
  return ((unsigned long long)tag << 48) | ((unsigned long long)lo << kTailPairLabelBits) | hi;
}

// Record key as a candidate minimum of its pair. A failed insert (64 probes
// over slots owned by other pairs this round) leaves the pair absent, so
// every edge of it is kept by tail_pair_keep: always safe.
__device__ __forceinline__ void tail_pair_insert(ulonglong2* t, unsigned long long mask, unsigned long long pw,
                                                 unsigned long long key) {
  const unsigned long long tag = pw >> 48;
  unsigned long long h = pair_hash(pw) & mask;
  ulonglong2 s = __ldcg(t + h);
  for (int probe = 0; probe < kTailPairProbes;) {
    if (s.x == pw) {
      if (key < s.y) atomicMin(&t[h].y, key);
      return;
    }
    if ((s.x >> 48) == tag) {  // another pair of this round
      h = (h + 1) & mask;
      ++probe;
      s = __ldcg(t + h);
      continue;
    }
    // empty for this round (stale tag): claim it with {pair, key}
    const ulonglong2 want = make_ulonglong2(pw, key);
    const ulonglong2 got = atomicCAS(t + h, s, want);
    if (got.x == s.x && got.y == s.y) return;
    s = got;  // lost the race: look at the winner's slot again
  }
}

__device__ __forceinline__ bool tail_pair_keep(const ulonglong2* t, unsigned long long mask, unsigned long long pw,
                                               unsigned long long key) {
  const unsigned long long tag = pw >> 48;
  unsigned long long h = pair_hash(pw) & mask;
  for (int probe = 0; probe < kTailPairProbes; ++probe) {
    const ulonglong2 s = __ldcg(t + h);
    if (s.x == pw) return key <= s.y;
    if ((s.x >> 48) != tag) return true;
    h = (h + 1) & mask;
  }
  return true;
}

// kItems inserts with their first probes in flight together (slot loads,
// then the CASes); the rare unresolved ones finish one by one.
__device__ __forceinline__ void tail_pair_insert_batch(ulonglong2* t, unsigned long long mask,
                                                       const unsigned long long (&pw)[kItems],
                                                       const unsigned long long (&key)[kItems],
                                                       const bool (&v)[kItems]) {
  unsigned long long h[kItems];
  ulonglong2 s[kItems], got[kItems];
  bool todo[kItems], cas[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    todo[k] = v[k];
    h[k] = pair_hash(pw[k]) & mask;
    s[k] = todo[k] ? __ldcg(t + h[k]) : make_ulonglong2(0, 0);
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    cas[k] = false;
    if (!todo[k]) continue;
    if (s[k].x == pw[k]) {
      if (key[k] < s[k].y) atomicMin(&t[h[k]].y, key[k]);
      todo[k] = false;
    } else if ((s[k].x >> 48) != (pw[k] >> 48)) {
      got[k] = atomicCAS(t + h[k], s[k], make_ulonglong2(pw[k], key[k]));
      cas[k] = true;
    }
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    if (cas[k] && got[k].x == s[k].x && got[k].y == s[k].y) todo[k] = false;
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    if (todo[k]) tail_pair_insert(t, mask, pw[k], key[k]);
}

__device__ __forceinline__ void tail_pair_keep_batch(const ulonglong2* t, unsigned long long mask,
                                                     const unsigned long long (&pw)[kItems],
                                                     const unsigned long long (&key)[kItems], bool (&f)[kItems]) {
  unsigned long long h[kItems];
  ulonglong2 s[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    h[k] = pair_hash(pw[k]) & mask;
    s[k] = f[k] ? __ldcg(t + h[k]) : make_ulonglong2(0, 0);
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    if (!f[k]) continue;
    if (s[k].x == pw[k])
      f[k] = key[k] <= s[k].y;
    else if ((s[k].x >> 48) == (pw[k] >> 48))
      f[k] = tail_pair_keep(t, mask, pw[k], key[k]);  // probe on (rare)
  }
}

// 2*kItems filtered offers with their reads in flight together.
__device__ __forceinline__ void offer_batch(unsigned long long* table, const uint4 (&e)[kItems],
                                            const unsigned long long (&key)[kItems], const bool (&f)[kItems]) {
  unsigned long long cx[kItems], cy[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    cx[k] = f[k] ? __ldca(table + e[k].x) : 0ull;
    cy[k] = f[k] ? __ldca(table + e[k].y) : 0ull;
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    if (!f[k]) continue;
    if (key[k] < cx[k]) atomicMin(table + e[k].x, key[k]);
    if (key[k] < cy[k]) atomicMin(table + e[k].y, key[k]);
  }
}

// 3 CTAs/SM (<= 80 registers): since the tail also streams round 1's edges
// (start at phase C) the extra warps pay: c1 -1.5 %, c2 -1 %, c3 -1 %, c4
// neutral, c0 +2 % (tools/ab: tail3 vs 2)
#ifndef MST_TAIL_MINB
#define MST_TAIL_MINB 3
#endif
__global__ void __launch_bounds__(kBlock, MST_TAIL_MINB) k_tail(TailArgs a) {
  pdl_prologue();
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  int slot = 0;
  tail_stamp(a, slot);
  __shared__ uint32_t s_cnt[kItems * kWarps + 1];
  __shared__ uint32_t s_warp[kWarps + 1];
  __shared__ uint32_t s_bpre[kTailMaxBlocks + 1];
  __shared__ unsigned long long s_wsum[kWarps];
  __shared__ uint32_t s_par[kTailSmemMin];             // tiny rounds: parent / root per component
  __shared__ uint32_t s_mask[kTailSmemMin / 32];       // tiny rounds: root bitmask
  __shared__ uint32_t s_wpre[kTailSmemMin / 32 + 1];   // tiny rounds: roots before each mask word
  __shared__ unsigned long long s_min[kTailSmemMin];
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  volatile DevCounters* vc = a.ctr;
  const uint32_t n_entry = vc->n[a.r0];
  // this WARP's segment of the (single, in place) edge list: a share of its
  // block's chunk, compacted with ballot ranks (no block barrier)
  uint4* const E = (a.r0 & 1) ? a.E[1] : a.E[0];
  const uint64_t m_entry = (a.start_c && a.c_soa) ? vc->m[0] : vc->m[a.r0];
  const uint64_t es = (m_entry + G - 1) / G;
  const uint64_t blo = min((uint64_t)b * es, m_entry), bhi = min(blo + es, m_entry);
  const uint64_t wes = (bhi - blo + kWarps - 1) / kWarps;
  const uint64_t seg_lo = min(blo + warp * wes, bhi);
  uint64_t seg_len = min(seg_lo + wes, bhi) - seg_lo;
  bool dedup_off = false;  // identical on every block (from global counters)
  int last_dedup = -1;
  // Round state kept in registers: every block derives n_{r+1} and the
  // verdicts from the same data, and only this kernel changes them while it
  // runs, so no counter is re-read at the top of a round (each read is a
  // dependent L2 round trip on the critical path of a tiny round).
  if ((uint32_t)a.r0 >= vc->stop_round || (uint32_t)a.r0 >= vc->phase_end) return;
  if (a.start_c && (uint32_t)a.r0 + 1 >= vc->stop_round) return;  // round r0's hook finished the MST
  uint32_t n_r = n_entry;
  int tiny_rounds = 0;
  uint64_t m_prev = m_entry;  // live edges entering round r-1 (dedup statistics)
  for (int r = a.r0; r < kMaxR - 1; ++r) {
    // edges kept by round r-1 (C's atomics, complete at the last grid.sync);
    // issued here, first used after A
    const uint64_t m_r = r > a.r0 ? __ldcg(reinterpret_cast<const unsigned long long*>(&a.ctr->m[r])) : m_entry;
    // ternaries, not a dynamic index: keeps TailArgs out of local memory
    const unsigned long long* mcur = (r & 1) ? a.minb[0] : a.minb[1];
    unsigned long long* mnext = (r & 1) ? a.minb[1] : a.minb[0];
    // ---- tiny round (n_r <= kTailSmemMin, plain loop): every block makes
    // the hook decisions and finds the roots of ALL components itself, in
    // shared memory (the same rule, the same dense labels as A + B), then
    // relabels its segment from shared memory: ONE grid sync per round
    // instead of three. Min tables rotate through three small buffers: round
    // r reads T[r%3] (the first tiny round: the normal table), offers into
    // T[(r+1)%3] and clears T[(r+2)%3], which every block finished reading
    // before the previous round's sync.
    if (a.tiny[0] != nullptr && !a.light && r > a.r0 && n_r <= kTailSmemMin) {
      const int rr = r % 3;
      const unsigned long long* tcur =
          (tiny_rounds == 0) ? mcur : (rr == 0 ? a.tiny[0] : rr == 1 ? a.tiny[1] : a.tiny[2]);
      unsigned long long* tnext = rr == 0 ? a.tiny[1] : rr == 1 ? a.tiny[2] : a.tiny[0];
      unsigned long long* tclear = rr == 0 ? a.tiny[2] : rr == 1 ? a.tiny[0] : a.tiny[1];
      // the list ping-pongs between E and the other list (same segment
      // bounds): every block gathers the min edges of ALL components from the
      // list this round reads while other blocks already compact theirs, so a
      // round may not overwrite the list it gathers from (the other list is
      // free past round r0; ternaries on the kernel parameters keep this out
      // of the register budget)
      const bool flip = ((a.r0 ^ tiny_rounds) & 1) != 0;
      const uint4* const Et = flip ? a.E[1] : a.E[0];
      uint4* const Eo = flip ? a.E[0] : a.E[1];
      ++tiny_rounds;
      if (m_r == 0) {  // round r-1 kept no edge (scan_verdict)
        if (b == 0 && threadIdx.x == 0) a.ctr->stop_round = (uint32_t)r;
        break;
      }
      for (uint32_t c = threadIdx.x; c < n_r; c += kBlock) s_min[c] = __ldcg(tcur + c);
      for (uint32_t c = b * kBlock + threadIdx.x; c < n_r; c += G * kBlock) tclear[c] = kNoKey;
      __syncthreads();
      // hook (same rule as A): partner, mutual pair -> lower label is root
      unsigned long long wsum = 0;
      for (uint32_t base = 0; base < n_r; base += kBlock * kItems) {
        unsigned long long key[kItems];
        uint4 e[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {  // the gathers of kItems components in flight together
          const uint32_t c = base + k * kBlock + threadIdx.x;
          key[k] = c < n_r ? s_min[c] : kNoKey;
          e[k] = key[k] != kNoKey ? __ldcg(Et + (uint32_t)key[k]) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint32_t c = base + k * kBlock + threadIdx.x;
          bool isroot = false;
          if (c < n_r) {
            if (key[k] == kNoKey) {
              isroot = true;
              s_par[c] = c;
            } else {
              const uint32_t o = (e[k].x == c) ? e[k].y : e[k].x;
              isroot = s_min[o] == key[k] && c < o;
              s_par[c] = isroot ? c : o;
              if (!isroot && b == 0) {  // block 0 records the MST edge (flags, weight)
                mst_mark(a.mst_bits, a.mst_bytes, e[k].w);
                wsum += (uint32_t)(key[k] >> 32);
              }
            }
          }
          const unsigned bal = __ballot_sync(0xffffffffu, isroot);
          const uint32_t c0 = base + k * kBlock + warp * 32;
          if (lane == 0 && c0 < n_r) s_mask[c0 >> 5] = bal;
        }
      }
      __syncthreads();
      if (warp == 0) {  // roots before each mask word (<= 64 words)
        constexpr int kW = (kTailSmemMin / 32 + 31) / 32;
        const uint32_t words = (n_r + 31) / 32;
        uint32_t v[kW], sum = 0;
#pragma unroll
        for (int j = 0; j < kW; ++j) {
          const uint32_t wi = lane * kW + j;
          v[j] = wi < words ? __popc(s_mask[wi]) : 0u;
          sum += v[j];
        }
        const uint32_t incl = warp_incl_scan(sum);
        uint32_t run = incl - sum;
#pragma unroll
        for (int j = 0; j < kW; ++j) {
          const uint32_t wi = lane * kW + j;
          if (wi < words) s_wpre[wi] = run;
          run += v[j];
        }
        if (lane == 31) s_wpre[kTailSmemMin / 32] = incl;
      }
      // root finding in shared memory (path halving: every value ever
      // stored is an ancestor, so the races are benign)
      for (uint32_t c = threadIdx.x; c < n_r; c += kBlock) {
        uint32_t x = c, p = s_par[x];
        while (p != x) {
          const uint32_t gp = s_par[p];
          if (gp == p) {
            x = p;
            break;
          }
          s_par[x] = gp;
          x = gp;
          p = s_par[x];
        }
        s_par[c] = x;  // the root
      }
      __syncthreads();
      const uint32_t n_next = s_wpre[kTailSmemMin / 32];
      const bool stop_now = n_next <= 1 || n_next == n_r;
      if (b == 0) {
        wsum = warp_sum<unsigned long long>(wsum);
        if (lane == 0 && wsum) atomicAdd(&a.ctr->total_weight, wsum);
        if (threadIdx.x == 0) {
          a.ctr->n[r + 1] = n_next;
          a.ctr->m[r + 2] = 0;  // the next round's kept counter (used after the sync)
          if (stop_now) a.ctr->stop_round = (uint32_t)r + 1;
        }
      }
      tail_stamp(a, slot);
      if (stop_now) break;
      // relabel + compact the warp's segment in place, offers aggregated in
      // shared memory and flushed into T[(r+1)%3]
      for (uint32_t c = threadIdx.x; c < n_next; c += kBlock) s_min[c] = kNoKey;
      __syncthreads();
      const uint64_t seg_hi = seg_lo + seg_len;
      uint64_t out = seg_lo;
      const uint32_t lt = lanemask_lt();
      for (uint64_t base = seg_lo; base < seg_hi; base += 32 * kItems) {
        uint4 e[kItems];
        bool f[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t i = base + k * 32 + lane;
          e[k] = i < seg_hi ? __ldcg(Et + i) : make_uint4(0, 0, 0, 0);
          if (i < seg_hi) {
            const uint32_t ra = s_par[e[k].x], rb = s_par[e[k].y];
            e[k].x = s_wpre[ra >> 5] + __popc(s_mask[ra >> 5] & ((1u << (ra & 31)) - 1u));
            e[k].y = s_wpre[rb >> 5] + __popc(s_mask[rb >> 5] & ((1u << (rb & 31)) - 1u));
          }
          f[k] = i < seg_hi && e[k].x != e[k].y;
        }
        uint32_t rank[kItems], tot = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const unsigned bal = __ballot_sync(0xffffffffu, f[k]);
          rank[k] = tot + __popc(bal & lt);
          tot += __popc(bal);
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          if (!f[k]) continue;
          const uint64_t j = out + rank[k];
          Eo[j] = e[k];
          const unsigned long long key = ((unsigned long long)e[k].z << 32) | (uint32_t)j;
          if (key < s_min[e[k].x]) atomicMin(s_min + e[k].x, key);
          if (key < s_min[e[k].y]) atomicMin(s_min + e[k].y, key);
        }
        out += tot;
      }
      seg_len = out - seg_lo;
      if (lane == 0 && seg_len) atomicAdd(const_cast<unsigned long long*>(&a.ctr->m[r + 1]), seg_len);
      __syncthreads();
      for (uint32_t c = threadIdx.x; c < n_next; c += kBlock) {
        const unsigned long long v = s_min[c];
        if (v != kNoKey && v < __ldcg(tnext + c)) atomicMin(tnext + c, v);
      }
      grid.sync();
      tail_stamp(a, slot);
      n_r = n_next;
      m_prev = m_r;
      continue;
    }
    uint32_t n_next = 0;
    bool stop_now = false, phase_now = false, light_final = false;
    const bool first_c = a.start_c && r == a.r0;
    if (first_c) n_next = vc->n[r + 1];  // the round kernels' hook + label ran round r0
    if (!first_c) {
    // ---- A: hook decisions over this block's chunk (a multiple of 32
    // components, so root-mask words never straddle chunks)
    const uint32_t cs = (((n_r + G - 1) / G) + 31u) & ~31u;
    {
      const uint32_t clo = min(b * cs, n_r), chi = min(clo + cs, n_r);
      uint32_t running = 0;
      unsigned long long wsum = 0;
      for (uint32_t base = clo; base < chi; base += kBlock * kItems) {
        unsigned long long key[kItems];
        uint4 e[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint32_t c = base + k * kBlock + threadIdx.x;
          key[k] = c < chi ? __ldcg(mcur + c) : kNoKey;
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          e[k] = make_uint4(0, 0, 0, 0);
          if (key[k] != kNoKey) e[k] = r == a.r0 ? tail_entry_edge(a, (uint32_t)key[k]) : __ldcg(E + (uint32_t)key[k]);
        }
        unsigned long long okey[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint32_t c = base + k * kBlock + threadIdx.x;
          const uint32_t o = (e[k].x == c) ? e[k].y : e[k].x;
          okey[k] = key[k] != kNoKey ? __ldca(mcur + o) : kNoKey;
        }
        unsigned bal[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint32_t c = base + k * kBlock + threadIdx.x;
          bool isroot = false;
          if (c < chi) {
            if (key[k] == kNoKey) {
              isroot = true;
              a.parent[c] = c;
            } else {
              const uint32_t o = (e[k].x == c) ? e[k].y : e[k].x;
              isroot = okey[k] == key[k] && c < o;
              a.parent[c] = isroot ? c : o;
              if (!isroot) {
                mst_mark(a.mst_bits, a.mst_bytes, e[k].w);  // the MST edge
                wsum += (uint32_t)(key[k] >> 32);
              }
            }
          }
          bal[k] = __ballot_sync(0xffffffffu, isroot);
          if (lane == 0) s_cnt[k * kWarps + warp] = __popc(bal[k]);
        }
        __syncthreads();
        if (warp == 0) {
          const uint32_t v = s_cnt[lane];
          const uint32_t incl = warp_incl_scan(v);
          s_cnt[lane] = incl - v;
          if (lane == 31) s_cnt[32] = incl;
        }
        __syncthreads();
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < kItems; ++k) {
            const uint32_t c0 = base + k * kBlock + warp * 32;
            if (c0 < chi) {
              a.masks[c0 >> 5] = bal[k];
              a.wpref[c0 >> 5] = running + s_cnt[k * kWarps + warp];
            }
          }
        }
        running += s_cnt[32];
        __syncthreads();
      }
      wsum = warp_sum<unsigned long long>(wsum);
      if (lane == 0) s_wsum[warp] = wsum;
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < kWarps; ++i) t += s_wsum[i];
        if (t) atomicAdd(&a.ctr->total_weight, t);
        a.broots[b] = running;
      }
    }
    grid.sync();
    tail_stamp(a, slot);
    // ---- B: dense labels, MST slots, next min table
    if (r > a.r0 && m_r == 0) {
      // round r-1 kept no edge: the same verdict the round kernels' edge
      // scan gives (scan_verdict)
      if (b == 0 && threadIdx.x == 0) {
        if (a.light)
          a.ctr->phase_end = (uint32_t)r;
        else
          a.ctr->stop_round = (uint32_t)r;
      }
      break;
    }
    if (last_dedup == r - 1 && 2 * m_r > m_prev) dedup_off = true;
    block_scan_array(a.broots, G, s_bpre, s_warp);
    n_next = s_bpre[G];
    light_final = a.light && a.retired && n_next <= 1 && n_next < n_r;
    if (n_next <= 1 && !(a.light && a.retired)) {
      stop_now = true;
    } else if (n_next == n_r) {
      // no live edge anywhere: done (a forest), or the light phase ends
      if (a.light)
        phase_now = true;
      else
        stop_now = true;
    }
    if (b == 0 && threadIdx.x == 0) {
      a.ctr->n[r + 1] = n_next;
      a.ctr->m[r + 1] = 0;  // C adds every block's kept count
      a.ctr->m[r + 2] = 0;  // (a tiny round r+1 adds into m[r+2] without a prior sync)
      if (stop_now) a.ctr->stop_round = (uint32_t)r + 1;
      if (phase_now) a.ctr->phase_end = (uint32_t)r;
      // round r's merges are kept (their MST flags are set): its labels and
      // the map update below still run, then the phase ends at round r + 1
      if (light_final) a.ctr->phase_end = (uint32_t)r + 1;
    }
    if (phase_now) break;  // the host composes the maps; nothing of round r is kept
    for (uint32_t base = b * kBlock * kItems; base < n_r; base += G * kBlock * kItems) {
      uint32_t c[kItems], root[kItems];
      bool v[kItems], walk[kItems], isroot[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        c[k] = base + k * kBlock + threadIdx.x;
        v[k] = c[k] < n_r;
        isroot[k] = v[k] && ((__ldcg(a.masks + (c[k] >> 5)) >> (c[k] & 31)) & 1u);
        walk[k] = v[k] && !isroot[k] && !stop_now;
      }
      if (stop_now) continue;
      find_roots<kItems>(a.parent, c, walk, root);
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        if (!v[k]) continue;
        const uint32_t x = isroot[k] ? c[k] : root[k], w = x >> 5;
        a.L[c[k]] = s_bpre[x / cs] + __ldca(a.wpref + w) + __popc(__ldca(a.masks + w) & ((1u << (x & 31)) - 1u));
        if (c[k] < n_next) mnext[c[k]] = kNoKey;
      }
    }
    grid.sync();
    tail_stamp(a, slot);
    if (stop_now) break;
    }  // !first_c
    if (a.light) {
      // entry label -> current label, 4 gathers in flight per thread
      for (uint32_t base = b * kBlock * 4 + threadIdx.x; base < n_entry; base += G * kBlock * 4) {
        uint32_t x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = base + k * kBlock < n_entry ? __ldcg(a.M + base + k * kBlock) : 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (base + k * kBlock < n_entry) x[k] = __ldca(a.L + x[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (base + k * kBlock < n_entry) a.M[base + k * kBlock] = x[k];
      }
      if (light_final) break;  // the host composes the maps (phase_end = r + 1)
    }
    // ---- C0 (optional): relabel in place + each pair's lightest key
    const bool dedup = a.pairs != nullptr && !first_c && n_next < (1u << kTailPairLabelBits) && m_r >= a.dedup_min &&
                       m_r >= (uint64_t)a.dedup_ratio * n_next &&
                       (!dedup_off || (uint64_t)n_next * (n_next - 1) / 2 <= m_r / 4);
    const uint32_t tag = (a.pair_epoch << 6) | ((uint32_t)r & 63u);
    unsigned long long pmask = 0;
    if (dedup) {
      unsigned long long cap = 1024;
      while (cap < m_r / 2 && cap < a.pair_cap) cap <<= 1;
      pmask = min(cap, a.pair_cap) - 1;
      last_dedup = r;
      for (uint64_t base = seg_lo; base < seg_lo + seg_len; base += 32 * kItems) {
        uint4 e[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t i = base + k * 32 + lane;
          e[k] = i < seg_lo + seg_len ? __ldcg(E + i) : make_uint4(0, 0, 0, 0);
        }
        uint32_t x[kItems], y[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t i = base + k * 32 + lane;
          x[k] = i < seg_lo + seg_len ? __ldca(a.L + e[k].x) : 0u;
          y[k] = i < seg_lo + seg_len ? __ldca(a.L + e[k].y) : 0u;
        }
        unsigned long long pw[kItems], key[kItems];
        bool v[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t i = base + k * 32 + lane;
          v[k] = i < seg_lo + seg_len && x[k] != y[k];
          pw[k] = tail_pair_word(tag, x[k], y[k]);
          key[k] = ((unsigned long long)e[k].z << 32) | (uint32_t)i;
        }
        tail_pair_insert_batch(a.pairs, pmask, pw, key, v);
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t i = base + k * 32 + lane;
          if (i < seg_lo + seg_len) *reinterpret_cast<uint2*>(E + i) = make_uint2(x[k], y[k]);
        }
      }
      grid.sync();
      tail_stamp(a, slot);
    }
    // ---- C: relabel + compact the segment in place, offers for round r+1
    {
      // Few components left: offers hammer a handful of lines. Aggregate them
      // in a block-local shared-memory table and flush once per block.
      const bool local = n_next <= kTailSmemMin;
      if (local) {
        for (uint32_t c = threadIdx.x; c < n_next; c += kBlock) s_min[c] = kNoKey;
        __syncthreads();
      }
      uint64_t out = seg_lo;
      const uint32_t lt = lanemask_lt();
      const uint64_t seg_hi = seg_lo + seg_len;
      for (uint64_t base = seg_lo; base < seg_hi; base += 32 * kItems) {
        uint4 e[kItems];
        bool live[kItems];
        if (first_c && a.c_soa) {
          // round 1 straight from the caller's SoA list (k_min_round1 has
          // flagged any out-of-range endpoint; such edges are dropped here)
#pragma unroll
          for (int k = 0; k < kItems; ++k) {
            const uint64_t i = base + k * 32 + lane;
            e[k] = i < seg_hi ? make_uint4(__ldcs(static_cast<const uint32_t*>(a.src0) + i), __ldcs(a.src1 + i),
                                           __ldcs(a.src_w + i), (uint32_t)i)
                              : make_uint4(0, 0, 0, 0);
            live[k] = i < seg_hi && e[k].x < a.n_orig && e[k].y < a.n_orig;
          }
        } else {
#pragma unroll
          for (int k = 0; k < kItems; ++k) {
            const uint64_t i = base + k * 32 + lane;
            e[k] = i < seg_hi ? __ldcg(E + i) : make_uint4(0, 0, 0, 0);
            live[k] = i < seg_hi;
          }
        }
        bool f[kItems];
        if (!dedup) {
#pragma unroll
          for (int k = 0; k < kItems; ++k) {
            if (live[k]) {
              e[k].x = __ldca(a.L + e[k].x);
              e[k].y = __ldca(a.L + e[k].y);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) f[k] = live[k] && e[k].x != e[k].y;
        if (dedup) {
          unsigned long long pw[kItems], key[kItems];
#pragma unroll
          for (int k = 0; k < kItems; ++k) {
            pw[k] = tail_pair_word(tag, e[k].x, e[k].y);
            key[k] = ((unsigned long long)e[k].z << 32) | (uint32_t)(base + k * 32 + lane);
          }
          tail_pair_keep_batch(a.pairs, pmask, pw, key, f);
        }
        // ordered ranks within the warp's tile (positions are k-major); the
        // ballots need every lane's loads, so the in-place stores below never
        // overwrite an unread edge
        uint32_t rank[kItems], tot = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const unsigned bal = __ballot_sync(0xffffffffu, f[k]);
          rank[k] = tot + __popc(bal & lt);
          tot += __popc(bal);
        }
        unsigned long long key[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t j = out + rank[k];
          key[k] = ((unsigned long long)e[k].z << 32) | (uint32_t)j;
          if (f[k]) E[j] = e[k];
        }
        if (local) {
#pragma unroll
          for (int k = 0; k < kItems; ++k) {
            if (!f[k]) continue;
            if (key[k] < s_min[e[k].x]) atomicMin(s_min + e[k].x, key[k]);
            if (key[k] < s_min[e[k].y]) atomicMin(s_min + e[k].y, key[k]);
          }
        } else {
          offer_batch(mnext, e, key, f);
        }
        out += tot;
      }
      seg_len = out - seg_lo;
      if (lane == 0 && seg_len) atomicAdd(const_cast<unsigned long long*>(&a.ctr->m[r + 1]), seg_len);
      if (local) {
        __syncthreads();
        for (uint32_t c = threadIdx.x; c < n_next; c += kBlock) {
          const unsigned long long v = s_min[c];
          if (v != kNoKey && v < __ldcg(mnext + c)) atomicMin(mnext + c, v);
        }
      }
    }
    grid.sync();
    tail_stamp(a, slot);
    n_r = n_next;
    m_prev = m_r;
  }
}

// The error bits of a shard as one count per bit, so a sum-allreduce gives
// every rank the union of all ranks' errors (they then stop together).
__global__ void k_err_words(const DevCounters* ctr, uint32_t* __restrict__ out) {
  pdl_prologue();
  if (blockIdx.x == 0 && threadIdx.x < 2) out[threadIdx.x] = (ctr->err >> threadIdx.x) & 1u;
}

// A run's start: zeroed counters with n[1] = n, m[0] = m[1] = m and no
// verdict (block 0), the first min table all "no key", the MST bitmap clear.
__global__ void k_init_run(DevCounters* ctr, uint32_t n, uint64_t m, unsigned long long* __restrict__ minb0,
                           uint4* __restrict__ bits16, uint64_t bit_vecs) {
  pdl_prologue();
  if (blockIdx.x == 0) {
    static_assert(sizeof(DevCounters) % 4 == 0, "DevCounters is word-sized");
    uint32_t* cw = reinterpret_cast<uint32_t*>(ctr);
    for (uint32_t i = threadIdx.x; i < sizeof(DevCounters) / 4; i += blockDim.x) cw[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
      ctr->n[1] = n;
      ctr->m[0] = m;
      ctr->m[1] = m;
      ctr->stop_round = kNoStop;
      ctr->phase_end = kNoStop;
      ctr->pivot = 0xFFFFFFFFu;
    }
  }
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  // 16 B stores (the table comes from cudaMalloc: 256 B aligned)
  ulonglong2* m2 = reinterpret_cast<ulonglong2*>(minb0);
  for (uint64_t i = tid; i < n / 2; i += stride) m2[i] = make_ulonglong2(kNoKey, kNoKey);
  if (tid == 0 && (n & 1u)) minb0[n - 1] = kNoKey;
  for (uint64_t i = tid; i < bit_vecs; i += stride) bits16[i] = make_uint4(0, 0, 0, 0);
}

__global__ void k_iota(uint32_t* __restrict__ x, uint64_t count) {
  pdl_prologue();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] = (uint32_t)i;
}

// ------------------------------ result -------------------------------------

// Sharded mode: element-wise min of G shard buffers, written back to all
// (the on-device stand-in for ncclAllReduce(min) when shards are emulated).
template <class T, int kMaxShards>
struct ShardPtrs {
  T* p[kMaxShards];
};

// Emulated allreduce over the shard buffers (min, or sum for histograms).
template <class T, bool kSum = false>
__global__ void k_shard_min(ShardPtrs<T, 8> bufs, int shards, uint64_t count) {
  pdl_prologue();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    T v = bufs.p[0][i];
    for (int s = 1; s < shards; ++s) {
      const T x = bufs.p[s][i];
      v = kSum ? v + x : (x < v ? x : v);
    }
    for (int s = 0; s < shards; ++s) bufs.p[s][i] = v;
  }
}


// Sorted id list from the bitmap: popc per word, ordered scan with look-back,
// then each word writes its set bits in ascending order.
// Sorted output, two passes like the compactions: popcount per tile of
// bitmap words (+ fused or separate scan), then each word writes its set
// bits at their final positions in ascending order.
// Sorted output from per-edge flags set by the hook kernels (no atomics):
// count set flags per tile of kTile x 16 bytes, scan, emit ids ascending.
constexpr int kFlagTile = kTile * 16;

__global__ void __launch_bounds__(kBlock) k_flags_count(const uint8_t* __restrict__ flags, uint64_t m,
                                                        uint32_t* __restrict__ counts, DevCounters* ctr, int fused) {
  pdl_prologue();
  __shared__ uint32_t s_cnt[kWarps];
  const uint32_t ntiles = (uint32_t)((m + kFlagTile - 1) / kFlagTile);
  const uint64_t nvec = (m + 15) / 16;
  const uint4* v4 = reinterpret_cast<const uint4*>(flags);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      if (i < nvec) {
        const uint4 v = __ldcs(v4 + i);
        c += ((v.x * 0x01010101u) >> 24) + ((v.y * 0x01010101u) >> 24) + ((v.z * 0x01010101u) >> 24) +
             ((v.w * 0x01010101u) >> 24);
      }
    }
    c = warp_sum<uint32_t>(c);
    if (lane_id() == 0) s_cnt[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < kWarps; ++w) t += s_cnt[w];
      counts[tile] = t;
    }
    __syncthreads();
  }
  if (fused) {
    __shared__ uint32_t s_warp[kWarps + 1], s_flag;
    fused_scan_if_last<kScanPlain>(counts, ntiles, ctr, 0, kSlotSort, 0, s_warp, &s_flag);
  }
}

__global__ void __launch_bounds__(kBlock) k_flags_emit(const uint8_t* __restrict__ flags, uint64_t m,
                                                       const uint32_t* __restrict__ offsets,
                                                       uint32_t* __restrict__ out) {
  pdl_prologue();
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_stage[kWarps][32 * 16];
  const uint32_t ntiles = (uint32_t)((m + kFlagTile - 1) / kFlagTile);
  const uint64_t nvec = (m + 15) / 16;
  const uint4* v4 = reinterpret_cast<const uint4*>(flags);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint4 v[kItems];
    uint32_t cnt[kItems], incl[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      v[k] = i < nvec ? __ldcs(v4 + i) : make_uint4(0, 0, 0, 0);
      cnt[k] = ((v[k].x * 0x01010101u) >> 24) + ((v[k].y * 0x01010101u) >> 24) + ((v[k].z * 0x01010101u) >> 24) +
               ((v[k].w * 0x01010101u) >> 24);
      incl[k] = warp_incl_scan(cnt[k]);
      if (lane == 31) s_scan[k * kWarps + warp] = incl[k];
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = s_scan[lane];
      const uint32_t in = warp_incl_scan(x);
      s_scan[lane] = in - x;
    }
    __syncthreads();
    const uint32_t prefix = __ldg(offsets + tile);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      // a warp's ids for item k are one contiguous run of <= 512: stage them
      // in shared memory, then store the run coalesced (lane-by-lane stores
      // from the bit loop hit one sector per lane per store)
      const uint32_t wtot = __shfl_sync(0xffffffffu, incl[k], 31);
      if (!wtot) continue;
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      uint32_t pos = incl[k] - cnt[k];
      const uint32_t words[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t wd = words[q];
        while (wd) {
          const int byte = (__ffs(wd) - 1) >> 3;
          wd &= ~(0xFFu << (byte * 8));
          s_stage[warp][pos++] = (uint32_t)(i * 16 + q * 4 + byte);
        }
      }
      __syncwarp();
      uint32_t* dst = out + prefix + s_scan[k * kWarps + warp];
      for (uint32_t j = lane; j < wtot; j += 32) __stcs(dst + j, s_stage[warp][j]);
      __syncwarp();
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBlock) k_bitmap_count(const uint32_t* __restrict__ bits, uint64_t words,
                                                         uint32_t* __restrict__ counts, DevCounters* ctr,
                                                         int fused) {
  pdl_prologue();
  __shared__ uint32_t s_cnt[kWarps];
  const uint32_t ntiles = (uint32_t)((words + kTile - 1) / kTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      c += i < words ? __popc(__ldcs(bits + i)) : 0u;
    }
    c = warp_sum<uint32_t>(c);
    if (lane == 0) s_cnt[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < kWarps; ++w) t += s_cnt[w];
      counts[tile] = t;
    }
    __syncthreads();
  }
  if (fused) {
    __shared__ uint32_t s_warp[kWarps + 1], s_flag;
    fused_scan_if_last<kScanPlain>(counts, ntiles, ctr, 0, kSlotSort, 0, s_warp, &s_flag);
  }
}

// Ascending MST ids from the bitmap: a warp's ids for item k come from 32
// consecutive words, one contiguous run of <= 1024, staged in shared memory
// and stored coalesced (lane-by-lane stores from the bit loops would touch
// one sector per lane).
__global__ void __launch_bounds__(kBlock) k_bitmap_emit(const uint32_t* __restrict__ bits, uint64_t words,
                                                        const uint32_t* __restrict__ offsets,
                                                        uint32_t* __restrict__ out) {
  pdl_prologue();
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_stage[kWarps][32 * 32];
  const uint32_t ntiles = (uint32_t)((words + kTile - 1) / kTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t wv[kItems], cnt[kItems], incl[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      wv[k] = i < words ? __ldcs(bits + i) : 0u;
      cnt[k] = __popc(wv[k]);
      incl[k] = warp_incl_scan(cnt[k]);
      if (lane == 31) s_scan[k * kWarps + warp] = incl[k];
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = s_scan[lane];
      const uint32_t in = warp_incl_scan(v);
      s_scan[lane] = in - v;
    }
    __syncthreads();
    const uint32_t prefix = __ldg(offsets + tile);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint32_t wtot = __shfl_sync(0xffffffffu, incl[k], 31);
      if (!wtot) continue;
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      uint32_t pos = incl[k] - cnt[k];
      uint32_t x = wv[k];
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1;
        s_stage[warp][pos++] = (uint32_t)(i * 32 + bit);
      }
      __syncwarp();
      uint32_t* dst = out + prefix + s_scan[k * kWarps + warp];
      for (uint32_t j = lane; j < wtot; j += 32) __stcs(dst + j, s_stage[warp][j]);
      __syncwarp();
    }
    __syncthreads();
  }
}


}  // namespace mstgpu
