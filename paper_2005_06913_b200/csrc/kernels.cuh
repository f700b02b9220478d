// Device kernels of the B200 parallel Boruvka (arXiv 2005.06913, CAS variant
// re-designed for the GPU). One round r with n_r live components (dense
// labels 0..n_r-1) and m_r live edges runs three kernels:
//
//   k_hook    (n_r)  every component reads its lightest edge key, picks the
//                    partner, breaks mutual 2-cycles by lower label, emits its
//                    MST edge and flags roots; a decoupled look-back scan over
//                    the root flags assigns the next round's dense labels.
//                    Replaces the merge phase + try_union_cas
//                    (boruvka_parallel.cpp:176-227, union_find.cpp:75-92).
//   k_label  (n_r)   root finding with concurrent path halving over the hook
//                    forest (the reference's find walk, union_find.cpp:28-35)
//                    and the dense relabel; clears the next min table.
//   k_compact (m_r)  relabels both endpoints, drops intra-component edges
//                    (the covered flags, graph.hpp:62-67), writes the kept
//                    edges in order (ballot + block scan + decoupled
//                    look-back) and, fused, offers every kept edge to both
//                    endpoint components of round r+1 with a filtered 64-bit
//                    atomicMin (the edge scan + offer,
//                    boruvka_parallel.cpp:150-167).
//
// Round 1 reads the caller's edge list directly (k_min_round1 + k_compact).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mstgpu {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 4;                // per thread, component tiles (hook)
constexpr int kTile = kBlock * kItems;   // elements per tile (striped)
constexpr int kCItems = 8;               // per thread, edge tiles (compaction)
constexpr int kCTile = kBlock * kCItems;

constexpr int kMaxR = MST_MAX_ROUNDS + 2;
constexpr uint64_t kNoKey = ~0ull;
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
  unsigned int err;
  unsigned int stop_round;  // first round whose hook must not run
  unsigned int phase_end;   // first round past the light phase (Filter-Boruvka)
  unsigned int pivot;       // light edges: w < pivot
  unsigned long long total_weight;
};

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
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    return EdgeRec{__ldcs(src + i), __ldcs(dst + i), __ldcs(w + i), base + (uint32_t)i, true};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    return EdgeRec{__ldg(src + i), __ldg(dst + i), __ldg(w + i), base + (uint32_t)i, true};
  }
};

// The reference's AoS Edge {u32 src, u32 dest, u64 weight} (graph.hpp:41-45).
struct AosView {
  const uint4* __restrict__ e;
  uint32_t base;
  static constexpr bool kOriginal = true;
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    const uint4 v = __ldcs(e + i);
    return EdgeRec{v.x, v.y, v.z, base + (uint32_t)i, v.w == 0};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    const uint4 v = __ldg(e + i);
    return EdgeRec{v.x, v.y, v.z, base + (uint32_t)i, v.w == 0};
  }
};

// Compacted edges of round >= 2: {a, b, w, eid} (16 B/edge, one LDG.128).
struct PackedView {
  const uint4* __restrict__ e;
  static constexpr bool kOriginal = false;
  __device__ __forceinline__ EdgeRec stream(uint64_t i) const {
    const uint4 v = __ldcs(e + i);
    return EdgeRec{v.x, v.y, v.z, v.w, true};
  }
  __device__ __forceinline__ EdgeRec gather(uint64_t i) const {
    const uint4 v = __ldg(e + i);
    return EdgeRec{v.x, v.y, v.z, v.w, true};
  }
};

// ------------------------------ primitives ---------------------------------

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

// Ordered ranks of per-item flags over a striped tile (item k of thread t
// is tile element k*kBlock + t), with the tile's global exclusive prefix
// from the look-back. s_scan: kIt*kWarps words of smem; s_misc: 2 words.
template <int kIt>
__device__ __forceinline__ void tile_flag_scan(const bool (&flag)[kIt], uint32_t (&rank)[kIt],
                                               uint32_t* s_scan, uint32_t* s_misc,
                                               unsigned long long* status, uint32_t tile,
                                               uint32_t epoch, uint32_t& prefix, uint32_t& total) {
  constexpr int kSlots = kIt * kWarps;
  constexpr int kPer = (kSlots + 31) / 32;  // slots per lane in the warp-0 scan
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned bal[kIt];
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    bal[k] = __ballot_sync(0xffffffffu, flag[k]);
    if (lane == 0) s_scan[k * kWarps + warp] = __popc(bal[k]);
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t v[kPer];
    uint32_t sum = 0;
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
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t ex = lookback(status, tile, tot, epoch);
    if (lane == 0) {
      s_misc[0] = ex;
      s_misc[1] = tot;
    }
  }
  __syncthreads();
  prefix = s_misc[0];
  total = s_misc[1];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < kIt; ++k) rank[k] = s_scan[k * kWarps + warp] + __popc(bal[k] & lt);
}

// Filtered 64-bit min: read first (a stale read is never below the true
// value, so skipping is always safe), atomic only when it can win. With
// kWarpPre, lanes of a warp that target the same component first reduce
// to one candidate (__match_any_sync + redux.sync), so hub components see
// one atomic per warp instead of up to 32.
template <bool kWarpPre>
__device__ __forceinline__ void offer(unsigned long long* table, uint32_t c, uint64_t key,
                                      bool valid, bool filt = true) {
  if (kWarpPre) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const unsigned grp = __match_any_sync(act, c);
    if (__popc(grp) > 1) {
      const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
      const uint32_t mhi = __reduce_min_sync(grp, hi);
      const uint32_t mlo = __reduce_min_sync(grp, hi == mhi ? lo : 0xFFFFFFFFu);
      if (hi != mhi || lo != mlo) return;
    }
  }
  if (!valid) return;
  // Large (DRAM-resident) tables: a fire-and-forget RED; the read-first
  // filter would put a dependent DRAM round trip on the critical path.
  if (filt) {
    const unsigned long long cur = __ldcg(table + c);
    if (key < cur) atomicMin(table + c, (unsigned long long)key);
  } else {
    atomicMin(table + c, (unsigned long long)key);
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

// Lightest incident edge per vertex over the caller's list. kKeyPartner
// selects the sharded key (w<<32 | partner vertex) instead of the literal
// (w<<32 | local index); both are decided by the weight (distinct weights).
template <class View, bool kKeyPartner, bool kWarpPre>
__global__ void __launch_bounds__(kBlock) k_min_round1(View v, uint32_t n, uint64_t m,
                                                       unsigned long long* __restrict__ minimum,
                                                       DevCounters* ctr, int filt) {
  const uint64_t stride = (uint64_t)gridDim.x * kBlock;
  uint32_t err = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kBlock; base < m; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool valid = i < m;
    EdgeRec e{0, 0, 0, 0, true};
    if (valid) {
      e = v.stream(i);
      if (e.a >= n || e.b >= n) {
        err |= kErrRange;
        valid = false;
      } else if (!e.ok) {
        err |= kErrWeight;
        valid = false;
      } else if (e.a == e.b) {
        valid = false;  // self-loop: never in an MST
      }
    }
    const uint64_t hi = (uint64_t)e.w << 32;
    const uint64_t ka = kKeyPartner ? (hi | e.b) : (hi | (uint32_t)i);
    const uint64_t kb = kKeyPartner ? (hi | e.a) : (hi | (uint32_t)i);
    offer<kWarpPre>(minimum, e.a, ka, valid, filt);
    offer<kWarpPre>(minimum, e.b, kb, valid, filt);
  }
  if (err) atomicOr(&ctr->err, err);
}

// ------------------------------ hook ---------------------------------------

// kKeyPartner = false: key low word indexes the round's edge array (E).
// kKeyPartner = true:  key low word is the partner label (sharded mode).
template <class View, bool kKeyPartner>
__global__ void __launch_bounds__(kBlock) k_hook(View E, const unsigned long long* __restrict__ minimum,
                                                 uint32_t* __restrict__ parent,
                                                 uint32_t* __restrict__ rootlabel,
                                                 uint32_t* __restrict__ mst_or_pos, uint32_t n_orig,
                                                 DevCounters* ctr, int r,
                                                 unsigned long long* status, uint32_t epoch,
                                                 int light_phase) {
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_misc[2];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wsum[kWarps];
  if ((uint32_t)r >= ctr->stop_round || (uint32_t)r >= ctr->phase_end) return;
  const uint32_t n_r = ctr->n[r];
  const uint32_t mst_base = n_orig - n_r;
  const uint32_t ntiles = (uint32_t)(((uint64_t)n_r + kTile - 1) / kTile);
  unsigned long long wsum = 0;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile[r][kSlotHook], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    bool isroot[kItems];
    uint32_t part[kItems], eidv[kItems], wv[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t c = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      isroot[k] = false;
      part[k] = kNone;
      eidv[k] = 0;
      wv[k] = 0;
      if (c < n_r) {
        const unsigned long long key = minimum[c];
        if (key == kNoKey) {
          isroot[k] = true;  // no live edge: isolated component
        } else {
          const uint32_t w = (uint32_t)(key >> 32);
          uint32_t o;
          unsigned long long mutual_key;
          if (kKeyPartner) {
            o = (uint32_t)key;
            mutual_key = ((unsigned long long)w << 32) | (uint32_t)c;
          } else {
            const EdgeRec e = E.gather((uint32_t)key);
            o = (e.a == (uint32_t)c) ? e.b : e.a;
            mutual_key = key;
            eidv[k] = e.eid;
          }
          const bool mutual = __ldg(minimum + o) == mutual_key;
          isroot[k] = mutual && (uint32_t)c < o;
          part[k] = o;
          wv[k] = w;
        }
      }
    }
    uint32_t rank[kItems], prefix, total;
    tile_flag_scan<kItems>(isroot, rank, s_scan, s_misc, status, tile, epoch, prefix, total);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t c = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      if (c < n_r) {
        const uint32_t roots_before = prefix + rank[k];
        if (isroot[k]) {
          parent[c] = (uint32_t)c;
          rootlabel[c] = roots_before;
          if (kKeyPartner) mst_or_pos[c] = kNone;
        } else {
          parent[c] = part[k];
          const uint32_t pos = mst_base + ((uint32_t)c - roots_before);
          if (kKeyPartner)
            mst_or_pos[c] = pos;
          else
            mst_or_pos[pos] = eidv[k];
          wsum += wv[k];
        }
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      const uint32_t roots = prefix + total;
      ctr->n[r + 1] = roots;
      if (roots <= 1) {
        ctr->stop_round = (uint32_t)r + 1;
      } else if (roots == n_r) {
        // no live edge anywhere: done (a forest if roots > 1), unless this is
        // the light phase of Filter-Boruvka, which then simply ends
        if (light_phase)
          ctr->phase_end = (uint32_t)r;
        else
          ctr->stop_round = (uint32_t)r + 1;
      }
    }
    __syncthreads();
  }
  wsum = warp_sum<unsigned long long>(wsum);
  if (lane_id() == 0) s_wsum[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < kWarps; ++i) t += s_wsum[i];
    if (t) atomicAdd(&ctr->total_weight, t);
  }
}

// ------------------------------ label --------------------------------------

__global__ void __launch_bounds__(kBlock) k_label(uint32_t* __restrict__ parent,
                                                  const uint32_t* __restrict__ rootlabel,
                                                  uint32_t* __restrict__ L,
                                                  unsigned long long* __restrict__ min_next,
                                                  DevCounters* ctr, int r) {
  if ((uint32_t)r + 1 >= ctr->stop_round || (uint32_t)r >= ctr->phase_end) return;
  const uint32_t n_r = ctr->n[r];
  const uint32_t n_next = ctr->n[r + 1];
  const uint64_t stride = (uint64_t)gridDim.x * kBlock;
  for (uint64_t c = (uint64_t)blockIdx.x * kBlock + threadIdx.x; c < n_r; c += stride) {
    const uint32_t root = find_root(parent, (uint32_t)c);
    L[c] = __ldcg(rootlabel + root);
    if (c < n_next) min_next[c] = kNoKey;
  }
}

// ------------------------------ compact + next-round min -------------------

// Sharded-mode extra work (kKeyPartner): recover the global id of every edge
// some component hooked along in round r, into its MST slot.
struct Recover {
  const unsigned long long* __restrict__ min_cur;
  const uint32_t* __restrict__ mstpos;
  uint32_t* __restrict__ slots;
};

// kFilter selects the edge predicate of the pass:
//   kFilterNone  : round r of the plain loop: keep a != b after relabelling
//   kFilterLight : the split pass of Filter-Boruvka (over the caller's list,
//                  labels = vertex ids): keep the light edges w < pivot
//   kFilterHeavy : the filter pass (caller's list, labels = the light-phase
//                  components): keep heavy edges w >= pivot whose endpoints
//                  lie in different light components. Heavier edges closing
//                  a cycle of lighter ones are never in the MST (cycle
//                  property), so dropping them is exact.
enum { kFilterNone = 0, kFilterLight = 1, kFilterHeavy = 2 };

template <class View, bool kKeyPartner, bool kWarpPre, int kFilter>
__global__ void __launch_bounds__(kBlock) k_compact(View Ein, uint4* __restrict__ Eout,
                                                    const uint32_t* __restrict__ L,
                                                    unsigned long long* __restrict__ min_next,
                                                    Recover rec, uint32_t n_orig, DevCounters* ctr,
                                                    int r, unsigned long long* status,
                                                    uint32_t epoch, int slot, int light_phase, int filt) {
  __shared__ uint32_t s_scan[kCItems * kWarps];
  __shared__ uint32_t s_misc[2];
  __shared__ uint32_t s_tile;
  const uint32_t stop = ctr->stop_round;
  if ((uint32_t)r >= ctr->phase_end) return;
  const bool full = (uint32_t)r + 1 < stop;
  if (!full && !(kKeyPartner && (uint32_t)r < stop)) return;
  const uint64_t m_r = kFilter == kFilterHeavy ? ctr->m[0] : ctr->m[r];
  const uint32_t pivot = ctr->pivot;
  const uint32_t ntiles = (uint32_t)((m_r + kCTile - 1) / kCTile);
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile[r][slot], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    EdgeRec e[kCItems];
    bool keep[kCItems];
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
      keep[k] = false;
      e[k] = EdgeRec{0, 0, 0, 0, false};
      if (i < m_r) e[k] = Ein.stream(i);
    }
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint64_t i = (uint64_t)tile * kCTile + k * kBlock + threadIdx.x;
      if (i < m_r) {
        bool ok = true;
        if (View::kOriginal) {
          ok = e[k].a < n_orig && e[k].b < n_orig && e[k].ok;
          if (!ok) atomicOr(&ctr->err, (e[k].a < n_orig && e[k].b < n_orig) ? kErrWeight : kErrRange);
        }
        if (kFilter == kFilterLight) ok = ok && e[k].w < pivot;
        if (kFilter == kFilterHeavy) ok = ok && e[k].w >= pivot;
        if (ok) {
          if (kKeyPartner) {
            const unsigned long long hi = (unsigned long long)e[k].w << 32;
            if (__ldcg(rec.min_cur + e[k].a) == (hi | e[k].b)) {
              const uint32_t p = __ldg(rec.mstpos + e[k].a);
              if (p != kNone) rec.slots[p] = e[k].eid;
            }
            if (__ldcg(rec.min_cur + e[k].b) == (hi | e[k].a)) {
              const uint32_t p = __ldg(rec.mstpos + e[k].b);
              if (p != kNone) rec.slots[p] = e[k].eid;
            }
          }
          if (full) {
            if (kFilter == kFilterNone || (kFilter == kFilterHeavy && L != nullptr)) {
              e[k].a = __ldg(L + e[k].a);
              e[k].b = __ldg(L + e[k].b);
            }
            keep[k] = e[k].a != e[k].b;
          }
        }
      }
    }
    if (!full) {
      __syncthreads();
      continue;  // sharded final round: recovery only
    }
    uint32_t rank[kCItems], prefix, total;
    tile_flag_scan<kCItems>(keep, rank, s_scan, s_misc, status, tile, epoch, prefix, total);
#pragma unroll
    for (int k = 0; k < kCItems; ++k) {
      const uint32_t j = prefix + rank[k];
      if (keep[k]) __stcs(Eout + j, make_uint4(e[k].a, e[k].b, e[k].w, e[k].eid));
      const unsigned long long hi = (unsigned long long)e[k].w << 32;
      const unsigned long long ka = kKeyPartner ? (hi | e[k].b) : (hi | j);
      const unsigned long long kb = kKeyPartner ? (hi | e[k].a) : (hi | j);
      offer<kWarpPre>(min_next, e[k].a, ka, keep[k], filt);
      offer<kWarpPre>(min_next, e[k].b, kb, keep[k], filt);
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      const uint32_t kept = prefix + total;
      ctr->m[r + 1] = kept;
      // A light phase running dry ends the phase (the filter pass follows);
      // a sharded shard running dry says nothing about the others (the
      // replicated hook decides there); otherwise no edges left = done.
      if (kept == 0 && kFilter == kFilterNone) {
        if (light_phase)
          ctr->phase_end = (uint32_t)r + 1;
        else if (!kKeyPartner && ctr->stop_round == kNoStop)
          ctr->stop_round = (uint32_t)r + 1;
      }
    }
    __syncthreads();
  }
}

// Pivot of the split: histogram of the top 16 weight bits over a strided
// sample, then the smallest bin boundary with >= target sampled weights
// below it (kept in ctr->pivot; 0xFFFFFFFF means "everything light").
__global__ void k_weight_hist(const uint32_t* __restrict__ w, uint32_t wstride, uint64_t m,
                              uint64_t step, uint32_t samples, uint32_t* __restrict__ hist) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < samples; k += gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)k * step;
    if (i < m) atomicAdd(hist + (__ldg(w + i * wstride) >> 16), 1u);
  }
}

__global__ void __launch_bounds__(1024) k_pick_pivot(const uint32_t* __restrict__ hist, uint32_t target, DevCounters* ctr) {
  // one block of 1024 threads: 64 bins per thread, block scan of sums
  __shared__ uint32_t s_sum[1024];
  const uint32_t t = threadIdx.x;
  uint32_t sum = 0;
  for (int i = 0; i < 64; ++i) sum += hist[t * 64 + i];
  s_sum[t] = sum;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const uint32_t v = t >= (uint32_t)d ? s_sum[t - d] : 0u;
    __syncthreads();
    s_sum[t] += v;
    __syncthreads();
  }
  const uint32_t before = t ? s_sum[t - 1] : 0u;
  if (before < target && s_sum[t] >= target) {
    uint32_t run = before;
    for (int i = 0; i < 64; ++i) {
      run += hist[t * 64 + i];
      if (run >= target) {
        const uint32_t bin = t * 64 + i;
        ctr->pivot = bin == 0xFFFFu ? 0xFFFFFFFFu : (bin + 1) << 16;
        break;
      }
    }
  }
}

// Top-down composition of the light phase's relabel maps:
// L_r[c] = L_{r+1}[L_r[c]] for c < n[r] (in place on level r).
__global__ void k_compose(uint32_t* __restrict__ Lr, const uint32_t* __restrict__ Lnext,
                          const DevCounters* ctr, int r) {
  const uint32_t n_r = ctr->n[r];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_r; c += stride)
    Lr[c] = __ldg(Lnext + Lr[c]);
}

// ------------------------------ result -------------------------------------

// Sharded mode: element-wise min of G shard buffers, written back to all
// (the on-device stand-in for ncclAllReduce(min) when shards are emulated).
template <class T, int kMaxShards>
struct ShardPtrs {
  T* p[kMaxShards];
};

template <class T>
__global__ void k_shard_min(ShardPtrs<T, 8> bufs, int shards, uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    T v = bufs.p[0][i];
    for (int s = 1; s < shards; ++s) {
      const T x = bufs.p[s][i];
      v = x < v ? x : v;
    }
    for (int s = 0; s < shards; ++s) bufs.p[s][i] = v;
  }
}

__global__ void k_mark(const uint32_t* __restrict__ ids, uint32_t count, uint32_t* __restrict__ bits,
                       uint64_t m) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint32_t e = ids[i];
    if (e < m) atomicOr(bits + (e >> 5), 1u << (e & 31));
  }
}

// Sorted id list from the bitmap: popc per word, ordered scan with look-back,
// then each word writes its set bits in ascending order.
__global__ void __launch_bounds__(kBlock) k_bitmap_emit(const uint32_t* __restrict__ bits,
                                                        uint64_t words, uint32_t* __restrict__ out,
                                                        unsigned int* tile_ctr,
                                                        unsigned long long* status, uint32_t epoch) {
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_misc[2];
  __shared__ uint32_t s_tile;
  const uint32_t ntiles = (uint32_t)((words + kTile - 1) / kTile);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
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
      const uint32_t tot = __shfl_sync(0xffffffffu, in, 31);
      const uint32_t ex = lookback(status, tile, tot, epoch);
      if (lane == 0) s_misc[0] = ex;
    }
    __syncthreads();
    const uint32_t prefix = s_misc[0];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t i = (uint64_t)tile * kTile + k * kBlock + threadIdx.x;
      uint32_t pos = prefix + s_scan[k * kWarps + warp] + incl[k] - cnt[k];
      uint32_t x = wv[k];
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        out[pos++] = (uint32_t)(i * 32 + b);
      }
    }
    __syncthreads();
  }
}

}  // namespace mstgpu
