// K2/K7 event generation, K3 fused group+reduce+classify+incremental update,
// K5 dirty compaction metadata.
//
// Reference mapping (proj/src/core/engine.cpp):
//   seed_edge_events            101-112  -> k_seed_events
//   next-layer Del/Add events   271-283  -> k_expand_events (one record per
//                                           out-list entry: PAIR for edges live
//                                           before and after, DEL for tombstones,
//                                           ADD for NEW entries)
//   user_propagate / stash      199-203, 285-288 -> k_self_events (SELF records)
//   group_and_reduce            27-43    -> sort on the target bits + k_classify
//   classify                    45-78    -> k_classify (warp ballots)
//   incremental_update          80-87    -> k_classify
//   first-neighbour rule        234-238  -> k_classify
//   rows_equal + prune          135-138, 254-258 -> k_classify / k_recompute
// Message rows are never copied into event payloads: a record names where its
// source's previous (pre-image slab) and/or current (table) message of this
// layer lives.
#pragma once

#include <cub/cub.cuh>

#include "dev_common.cuh"
#include "graph_kernels.cuh"

namespace sgb {

// Table/row addressing for one layer's messages.
struct MsgView {
  const float4* cur;      // m_l table, pitch V float4
  const float4* old;      // pre-image slab (rows indexed by dirty slot), or null at layer 1
  const uint32_t* stamp;  // round stamp per node (msg_l rewritten this round), or null
  const uint32_t* slot;
  const uint64_t* net;    // this round's net delta (seed records)
  const uint32_t* dprev;  // previous layer's dirty list (expansion records)
  uint32_t round;
  uint32_t V;
  __device__ __forceinline__ const float4* cur_row(uint32_t u) const { return cur + static_cast<size_t>(u) * V; }
  __device__ __forceinline__ const float4* prev_row(uint32_t u) const {
    if (stamp && stamp[u] == round) return old + static_cast<size_t>(slot[u]) * V;
    return cur_row(u);
  }
};

__global__ void k_seed_events(const uint64_t* net, uint32_t num_net, uint32_t mult, uint64_t* rec) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= num_net) return;
  const uint64_t k = net[j];
  const uint32_t s = static_cast<uint32_t>(k >> 32) & kNodeMask, d = static_cast<uint32_t>(k) & kNodeMask;
  (void)s;
  const uint64_t r = make_record(d, j, (k >> 63) ? EV_SEED_DEL : EV_SEED_ADD);
  for (uint32_t m = 0; m < mult; ++m) rec[static_cast<size_t>(j) * mult + m] = r;
}

// Thread per output record (load-balanced across hub and leaf sources): the
// owning dirty source is found by binary search over the exclusive scan of the
// sources' out-list lengths.
__global__ void k_expand_events(const uint32_t* dirty, const uint64_t* offsets, uint32_t n_dirty, uint64_t total,
                                AdjView out, uint32_t mult, uint64_t* rec, unsigned long long* events_ctr) {
  unsigned long long events = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t lo = 0, hi = n_dirty;  // first index with offsets > i
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offsets[mid] <= i) lo = mid + 1; else hi = mid;
    }
    const uint32_t j = lo - 1;
    const uint32_t v = dirty[j];
    const uint32_t x = out.ent[out.off[v] + (i - offsets[j])];
    const uint32_t type = (x & kFlagDel) ? EV_EXP_DEL : ((x & kFlagNew) ? EV_EXP_ADD : EV_EXP_PAIR);
    events += type == EV_EXP_PAIR ? 2 : 1;
    const uint64_t r = make_record(x & kNodeMask, j, type);
    for (uint32_t m = 0; m < mult; ++m) rec[i * mult + m] = r;
  }
  warp_add(events_ctr, events * mult);
}

__global__ void k_self_events(const uint32_t* dirty, const uint8_t* changed, uint32_t n_dirty, uint64_t* rec,
                              unsigned long long* cursor) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_dirty || !changed[j]) return;
  const uint32_t v = dirty[j];
  rec[atomicAdd(cursor, 1ull)] = make_record(v, 0, EV_SELF);
}

__global__ void k_fill_sentinel(uint64_t* rec, const unsigned long long* from, uint32_t to) {
  for (uint32_t i = static_cast<uint32_t>(*from) + blockIdx.x * blockDim.x + threadIdx.x; i < to;
       i += gridDim.x * blockDim.x)
    rec[i] = kSentinelRecord;
}

__global__ void k_mark_heads(const uint64_t* rec, uint32_t n, uint8_t* head, unsigned long long* n_valid) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t t = static_cast<uint32_t>(rec[i] >> 32);
  const bool valid = t != 0xFFFFFFFFu;
  head[i] = valid && (i == 0 || static_cast<uint32_t>(rec[i - 1] >> 32) != t);
  if (valid && (i + 1 == n || static_cast<uint32_t>(rec[i + 1] >> 32) == 0xFFFFFFFFu)) *n_valid = i + 1;
}

__global__ void k_finish_runs(uint32_t* run_start, const unsigned long long* num_runs,
                              const unsigned long long* n_valid) {
  run_start[*num_runs] = static_cast<uint32_t>(*n_valid);
}

constexpr uint32_t kSeg = 32;  // records per classify work item (one per lane)

struct ClassifyArgs {
  const uint64_t* rec;
  const uint32_t* run_start;
  const unsigned long long* num_runs;
  MsgView msg;
  float4* agg;              // a_l table (pitch V float4)
  uint32_t d;               // logical dim of layer l
  const uint32_t* in_len;   // in-adjacency entry counts (incl. flagged)
  const uint32_t* in_new;
  uint8_t* run_flags;
  // segments (run << 32 | k) of <= kSeg records; multi-segment runs merge
  // their partial reductions through scratch rows (2 x P ints: del, add)
  uint64_t* seg;
  unsigned long long* n_seg;
  int* cls_scratch;
  uint32_t* cls_slot;
  uint32_t* cls_remaining;
  uint32_t* cls_flags;      // bit0 del, bit1 add, bit2 self
  uint32_t* run_target;     // target node of each run (written by the planner)
  unsigned long long* n_cls_scratch;
  // exposed-reset work list for k_aggregate (K4)
  uint64_t* work;
  unsigned long long* n_work;
  uint32_t chunk;
  int* scratch;             // multi-chunk recompute reductions, P ints per row
  uint32_t* scratch_idx;
  uint32_t* remaining;
  uint32_t* any_live;
  unsigned long long* n_scratch;
  unsigned long long* ctr;  // C_NUM counters of this layer
};

// Thread per run: cut it into kSeg-record segments (block-aggregated
// allocation, one global atomic per CTA); multi-segment runs get a merge slot
// (identity-initialised scratch rows and a completion counter).
template <bool IsMax>
__global__ void __launch_bounds__(256) k_plan_segments(ClassifyArgs A) {
  using BlockScan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ unsigned long long base;
  const uint32_t num_runs = static_cast<uint32_t>(*A.num_runs);
  const uint32_t P = A.msg.V * 4;
  for (uint32_t r0 = blockIdx.x * blockDim.x; r0 < num_runs; r0 += gridDim.x * blockDim.x) {
    const uint32_t r = r0 + threadIdx.x;
    uint32_t nseg = 0, rb = 0;
    if (r < num_runs) {
      rb = A.run_start[r];
      nseg = (A.run_start[r + 1] - rb + kSeg - 1) / kSeg;
      A.run_target[r] = static_cast<uint32_t>(A.rec[rb] >> 32);
    }
    uint32_t off = 0, total = 0;
    BlockScan(tmp).ExclusiveSum(nseg, off, total);
    if (threadIdx.x == 0) base = atomicAdd(A.n_seg, static_cast<unsigned long long>(total));
    __syncthreads();
    for (uint32_t k = 0; k < nseg; ++k) A.seg[base + off + k] = (static_cast<uint64_t>(r) << 32) | k;
    if (nseg > 1) {
      const uint32_t slot = static_cast<uint32_t>(atomicAdd(A.n_cls_scratch, 1ull));
      A.cls_slot[r] = slot;
      A.cls_remaining[r] = nseg;
      A.cls_flags[r] = 0;
      int* row = A.cls_scratch + static_cast<size_t>(slot) * 2 * P;
      for (uint32_t i = 0; i < 2 * P; ++i) row[i] = IsMax ? INT_MIN : INT_MAX;
    }
    __syncthreads();
  }
}

// Classify one grouped target from its reduced Del/Add rows (engine.cpp:45-87,
// 229-258): first-neighbour rule, reset positions, covered test, incremental
// update or exposed-reset hand-off to K4, bitwise change test, alpha write.
template <bool IsMax, int CPL>
__device__ __forceinline__ void classify_target(const ClassifyArgs& A, uint32_t r, uint32_t w, float4 (&del)[CPL],
                                                float4 (&add)[CPL], const float4 (&a)[CPL], bool has_del,
                                                bool has_add, bool has_self, unsigned long long* sc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t V = A.msg.V;
  const bool grp = has_del || has_add;
  uint8_t flags = (grp ? RUN_GRP : 0) | (has_self ? RUN_SELF : 0);
  int kind = -1;  // 0 NoDeletion 1 DeletionNoEffect 2 Covered 3 Exposed
  if (grp) {
    float4* arow = A.agg + static_cast<size_t>(w) * V;
    float4 anew[CPL];
    const uint32_t prev_indeg = A.in_len[w] - A.in_new[w];
    if (!has_del && prev_indeg == 0) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) anew[c] = add[c];
      kind = 0;
    } else if (!has_del) {
      kind = 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) anew[c] = sel4<IsMax>(a[c], add[c]);
    } else {
      bool reset = false, covered = true;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t idx = lane + 32u * c;
        const float av[4] = {a[c].x, a[c].y, a[c].z, a[c].w};
        const float dv[4] = {del[c].x, del[c].y, del[c].z, del[c].w};
        const float pv[4] = {add[c].x, add[c].y, add[c].z, add[c].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (idx < V && 4 * idx + q < A.d && av[q] == dv[q]) {
            reset = true;
            if (!has_add || !(IsMax ? pv[q] >= dv[q] : pv[q] <= dv[q])) covered = false;
          }
        }
      }
      reset = __any_sync(0xffffffffu, reset);
      covered = __all_sync(0xffffffffu, covered);
      kind = !reset ? 1 : (covered ? 2 : 3);
      if (kind != 3) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) anew[c] = has_add ? sel4<IsMax>(a[c], add[c]) : a[c];
      }
    }
    if (kind == 3) {
      flags |= RUN_EXPOSED;
      uint32_t nch = 0, si = 0;
      if (lane == 0) {
        const uint32_t raw = A.in_len[w];
        nch = raw == 0 ? 1u : (raw + A.chunk - 1) / A.chunk;
        const unsigned long long base = atomicAdd(A.n_work, static_cast<unsigned long long>(nch));
        for (uint32_t c = 0; c < nch; ++c) A.work[base + c] = (static_cast<uint64_t>(r) << 32) | c;
        if (nch > 1) {
          si = static_cast<uint32_t>(atomicAdd(A.n_scratch, 1ull));
          A.scratch_idx[r] = si;
          A.remaining[r] = nch;
          A.any_live[r] = 0;
        }
      }
      nch = __shfl_sync(0xffffffffu, nch, 0);
      si = __shfl_sync(0xffffffffu, si, 0);
      if (nch > 1) {
        int* srow = A.scratch + static_cast<size_t>(si) * V * 4;
        for (uint32_t i = lane; i < V * 4; i += 32) srow[i] = IsMax ? INT_MIN : INT_MAX;
      }
    } else {
      bool changed = false;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t idx = lane + 32u * c;
        if (idx < V && neq4(anew[c], a[c])) changed = true;
      }
      changed = __any_sync(0xffffffffu, changed);
      if (changed) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t idx = lane + 32u * c;
          if (idx < V) arow[idx] = anew[c];
        }
      }
      if (changed || has_self) flags |= RUN_DIRTY;
      if (changed && lane == 0) atomicAdd(&sc[C_AWRITES], 1ull);
    }
  } else if (has_self) {
    flags |= RUN_DIRTY;  // user-only target (engine.cpp:222-227)
  }
  if (lane == 0) {
    A.run_flags[r] = flags;
    if (grp) {
      atomicAdd(&sc[C_TARGETS], 1ull);
      atomicAdd(&sc[C_NO_DEL + kind], 1ull);
      atomicAdd(&sc[C_FETCH_OTHER], 1ull);  // read_prev(l, v, Aggregated), engine.cpp:233
      if (kind == 3) atomicAdd(&sc[C_RECOMPUTES], 1ull);
    }
    if (has_self) atomicAdd(&sc[C_USER_TARGETS], 1ull);
  }
}

// K3: warp per segment of <= 32 records. Each lane resolves one record's row
// addresses, then the warp gathers the rows (coalesced float4, UNR rows in
// flight) and reduces Del and Add messages (group_and_reduce, engine.cpp:27-43).
// Single-segment runs classify immediately; segments of longer runs merge
// through order-preserving integer atomics and the last one classifies.
template <bool IsMax, int CPL>
__global__ void __launch_bounds__(256, CPL <= 2 ? 3 : 1) k_classify(ClassifyArgs A) {
  __shared__ unsigned long long sc[C_NUM];
  for (int i = threadIdx.x; i < C_NUM; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t V = A.msg.V;
  const uint64_t n_seg = *A.n_seg;
  const float ident = IsMax ? -INFINITY : INFINITY;
  for (uint64_t sidx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sidx < n_seg; sidx += warps) {
    const uint64_t sg = A.seg[sidx];
    const uint32_t r = static_cast<uint32_t>(sg >> 32), k = static_cast<uint32_t>(sg);
    const uint32_t rb = A.run_start[r], re = A.run_start[r + 1];
    const uint32_t w = A.run_target[r];
    const uint32_t b = rb + k * kSeg, e = min(re, b + kSeg);
    const uint32_t nseg = (re - rb + kSeg - 1) / kSeg;
    // alpha_prev of the target: independent of the records, issue it first
    float4 a[CPL];
    {
      const float4* arow = A.agg + static_cast<size_t>(w) * V;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t idx = lane + 32u * c;
        a[c] = (idx < V && nseg == 1) ? arow[idx] : make_float4(0, 0, 0, 0);
      }
    }
    float4 del[CPL], add[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) del[c] = add[c] = make_float4(ident, ident, ident, ident);
    // each lane resolves one record's row addresses (parallel, not a chain)
    const uint32_t n_here = e - b;
    const float4* p_add = nullptr;
    const float4* p_del = nullptr;
    bool self = false;
    if (lane < n_here) {
      const uint64_t rr = A.rec[b + lane];
      const uint32_t type = static_cast<uint32_t>(rr) & 7u, ix = static_cast<uint32_t>(rr >> 3) & 0x1FFFFFFFu;
      if (type == EV_SELF) {
        self = true;
      } else if (type <= EV_SEED_DEL) {
        const uint32_t s = static_cast<uint32_t>(A.msg.net[ix] >> 32) & kNodeMask;
        if (type == EV_SEED_ADD) p_add = A.msg.cur_row(s); else p_del = A.msg.prev_row(s);
      } else {
        if (type != EV_EXP_DEL) p_add = A.msg.cur_row(A.msg.dprev[ix]);
        if (type != EV_EXP_ADD) p_del = A.msg.old + static_cast<size_t>(ix) * V;
      }
    }
    const bool has_self = __any_sync(0xffffffffu, self);
    const unsigned m_add = __ballot_sync(0xffffffffu, p_add != nullptr);
    const unsigned m_del = __ballot_sync(0xffffffffu, p_del != nullptr);
    const bool has_add = m_add != 0, has_del = m_del != 0;
    const uint32_t rows_read = __popc(m_add) + __popc(m_del);
    constexpr int UNR = CPL <= 2 ? 4 : (CPL <= 4 ? 2 : 1);
    unsigned ma = m_add, md = m_del;
    while (ma | md) {
      const float4* rows[UNR];
      bool is_del[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        rows[q] = nullptr;
        is_del[q] = false;
        if (ma) {
          const int src = __ffs(ma) - 1;
          ma &= ma - 1;
          rows[q] = reinterpret_cast<const float4*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(p_add), src));
        } else if (md) {
          const int src = __ffs(md) - 1;
          md &= md - 1;
          rows[q] = reinterpret_cast<const float4*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(p_del), src));
          is_del[q] = true;
        }
      }
      float4 v[UNR][CPL];
#pragma unroll
      for (int q = 0; q < UNR; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t idx = lane + 32u * c;
          v[q][c] = (rows[q] && idx < V) ? __ldg(rows[q] + idx) : make_float4(ident, ident, ident, ident);
        }
#pragma unroll
      for (int q = 0; q < UNR; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          if (is_del[q]) del[c] = sel4<IsMax>(del[c], v[q][c]);
          else add[c] = sel4<IsMax>(add[c], v[q][c]);
        }
    }
    if (lane == 0 && rows_read) atomicAdd(&sc[C_EVROWS], static_cast<unsigned long long>(rows_read));
    if (nseg == 1) {
      classify_target<IsMax, CPL>(A, r, w, del, add, a, has_del, has_add, has_self, sc);
      continue;
    }
    // multi-segment run: merge, the last segment classifies
    int* srow = A.cls_scratch + static_cast<size_t>(A.cls_slot[r]) * 2 * V * 4;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t idx = lane + 32u * c;
      if (idx >= V) continue;
      const float4 dv = del[c], av = add[c];
      int* pd = srow + 4 * idx;
      int* pa = srow + 4 * V + 4 * idx;
      if (has_del) {
        if (IsMax) {
          atomicMax(pd + 0, f2o(dv.x)); atomicMax(pd + 1, f2o(dv.y)); atomicMax(pd + 2, f2o(dv.z)); atomicMax(pd + 3, f2o(dv.w));
        } else {
          atomicMin(pd + 0, f2o(dv.x)); atomicMin(pd + 1, f2o(dv.y)); atomicMin(pd + 2, f2o(dv.z)); atomicMin(pd + 3, f2o(dv.w));
        }
      }
      if (has_add) {
        if (IsMax) {
          atomicMax(pa + 0, f2o(av.x)); atomicMax(pa + 1, f2o(av.y)); atomicMax(pa + 2, f2o(av.z)); atomicMax(pa + 3, f2o(av.w));
        } else {
          atomicMin(pa + 0, f2o(av.x)); atomicMin(pa + 1, f2o(av.y)); atomicMin(pa + 2, f2o(av.z)); atomicMin(pa + 3, f2o(av.w));
        }
      }
    }
    if (lane == 0) atomicOr(&A.cls_flags[r], (has_del ? 1u : 0u) | (has_add ? 2u : 0u) | (has_self ? 4u : 0u));
    __threadfence();
    __syncwarp();
    uint32_t prev = 0;
    if (lane == 0) prev = atomicSub(&A.cls_remaining[r], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != 1) continue;
    __threadfence();
    const uint32_t f = __ldcg(&A.cls_flags[r]);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t idx = lane + 32u * c;
      if (idx < V) {
        const int4 od = __ldcg(reinterpret_cast<const int4*>(srow) + idx);
        const int4 oa = __ldcg(reinterpret_cast<const int4*>(srow + 4 * V) + idx);
        del[c] = make_float4(o2f(od.x), o2f(od.y), o2f(od.z), o2f(od.w));
        add[c] = make_float4(o2f(oa.x), o2f(oa.y), o2f(oa.z), o2f(oa.w));
      }
    }
    {
      const float4* arow = A.agg + static_cast<size_t>(w) * V;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t idx = lane + 32u * c;
        a[c] = idx < V ? arow[idx] : make_float4(0, 0, 0, 0);
      }
    }
    classify_target<IsMax, CPL>(A, r, w, del, add, a, f & 1u, f & 2u, f & 4u, sc);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C_NUM; i += blockDim.x)
    if (sc[i]) atomicAdd(&A.ctr[i], sc[i]);
}

__global__ void k_dirty_flags(const uint8_t* run_flags, uint32_t n, uint8_t* out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (run_flags[i] & RUN_DIRTY) ? 1 : 0;
}

// Dirty list of this layer (ascending: runs are in target order), out-list
// lengths for the next layer's expansion, and the dirty-dependent row reads:
// user-only alpha read (engine.cpp:262-265), self-message reads
// (EngineApplyContext, 125-128), read_prev(l+1) (272).
__global__ void k_dirty_meta(const uint32_t* dirty_runs, const unsigned long long* n_dirty, const uint64_t* rec,
                             const uint32_t* run_start, const uint8_t* run_flags, const uint32_t* out_len,
                             uint32_t* dirty_nodes, uint64_t* lens, unsigned long long* sum_len,
                             unsigned long long* ctr, uint32_t user_ops, bool has_next, bool layer1) {
  const uint32_t n = static_cast<uint32_t>(*n_dirty);
  unsigned long long sl = 0, l1 = 0, other = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t r = dirty_runs[j];
    const uint32_t v = static_cast<uint32_t>(rec[run_start[r]] >> 32);
    const uint8_t f = run_flags[r];
    dirty_nodes[j] = v;
    const uint32_t L = out_len[v];
    lens[j] = L;
    sl += L;
    if (!(f & RUN_GRP)) other += 1;
    if (!(f & RUN_SELF)) (layer1 ? l1 : other) += user_ops;
    if (has_next) other += 1;
  }
  // block-level reduction through warp shuffles then atomics
  for (int o = 16; o; o >>= 1) {
    sl += __shfl_xor_sync(0xffffffffu, sl, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    other += __shfl_xor_sync(0xffffffffu, other, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (sl) atomicAdd(sum_len, sl);
    if (l1) atomicAdd(&ctr[C_FETCH_L1MSG], l1);
    if (other) atomicAdd(&ctr[C_FETCH_OTHER], other);
  }
}

}  // namespace sgb
