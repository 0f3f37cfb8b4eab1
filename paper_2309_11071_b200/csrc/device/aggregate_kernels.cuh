// K4 — neighbourhood re-aggregation.
//
// Replaces recompute (proj/src/core/engine.cpp:89-99) for exposed resets and the
// whole-graph aggregation of init_full_inference / full_inference
// (checkpoint.cpp:123-134, baseline.cpp:41-55): alpha = A over the current
// in-neighbours' current messages, zero vector when there are none.
//
// Work is split into (target, chunk of `chunk` in-list entries) items so a hub
// with 10^5 in-neighbours is spread over many warps. A single-chunk target is
// finalised by its warp; multi-chunk targets reduce into a scratch row with
// atomicMax/atomicMin on order-preserving integer images of the floats (exact
// and order-invariant, since NaN is rejected and -0 flushed), and the last chunk
// to finish finalises. Rows are gathered as coalesced float4 vectors; each warp
// keeps UNROLL rows in flight.
#pragma once

#include "dev_common.cuh"
#include "event_kernels.cuh"

namespace sgb {

struct AggArgs {
  // work items: (target index << 32 | chunk)
  const uint64_t* work;
  const unsigned long long* n_work;  // device count (update) ...
  uint64_t n_work_host;              // ... or host count (init) when n_work == null
  // update mode: target index = run index; init mode: target index = node id
  bool update;
  const uint32_t* runs;         // update mode: run -> target node
  const unsigned long long* abort;
  uint8_t* run_flags;
  const uint32_t* scratch_idx;  // per target index (multi-chunk only)
  uint32_t* remaining;
  uint32_t* any_live;
  int* scratch;
  // adjacency (in) and messages
  const uint64_t* in_off;
  const uint32_t* in_len;
  const uint32_t* in_ent;
  RowTable msg;       // m_l current table (rows of every shard, dev_common.cuh)
  float4* agg;        // destination a_l table
  uint32_t V, d, chunk;
  unsigned long long* fetch_ctr;  // live rows read
  unsigned long long* ctr;        // layer counters (update mode), for C_RECOMP_ROWS / C_AWRITES
  unsigned long long* next;       // dynamic work cursor (update mode), null = static
};

template <bool IsMax, int CPL>
__device__ __forceinline__ void finalize_alpha(const AggArgs& A, uint32_t t, uint32_t w, float4 (&acc)[CPL], bool any) {
  const uint32_t lane = threadIdx.x & 31;
  float4* arow = A.agg + static_cast<size_t>(w) * A.V;
  float4 anew[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const uint32_t idx = lane + 32u * c;
    float4 v = any ? acc[c] : make_float4(0, 0, 0, 0);
    // keep pitch padding at zero
    if (4 * idx + 0 >= A.d) v.x = 0;
    if (4 * idx + 1 >= A.d) v.y = 0;
    if (4 * idx + 2 >= A.d) v.z = 0;
    if (4 * idx + 3 >= A.d) v.w = 0;
    anew[c] = v;
  }
  if (!A.update) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t idx = lane + 32u * c;
      if (idx < A.V) arow[idx] = anew[c];
    }
    return;
  }
  bool changed = false;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const uint32_t idx = lane + 32u * c;
    if (idx < A.V && neq4(anew[c], arow[idx])) changed = true;
  }
  changed = __any_sync(0xffffffffu, changed);
  if (changed) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t idx = lane + 32u * c;
      if (idx < A.V) arow[idx] = anew[c];
    }
  }
  if (lane == 0) {
    const uint8_t f = A.run_flags[t];
    if (changed || (f & RUN_SELF)) A.run_flags[t] = f | RUN_DIRTY;
    if (changed) atomicAdd(&A.ctr[C_AWRITES], 1ull);
  }
}

// After a warp reduced `covered` consecutive chunks of a target: a target
// whose chunks were all covered by this warp finalises in place; otherwise the
// partial result merges into the target's scratch row with order-preserving
// integer atomics and the warp that brings the last chunks finalises.
template <bool IsMax, int CPL>
__device__ __forceinline__ void finish_chunks(const AggArgs& A, uint32_t t, uint32_t w, uint32_t nch,
                                              uint32_t covered, float4 (&acc)[CPL], uint32_t live) {
  const uint32_t lane = threadIdx.x & 31;
  if (covered == nch) {
    finalize_alpha<IsMax, CPL>(A, t, w, acc, live > 0);
    return;
  }
  const uint32_t si = A.scratch_idx[t];
  int* srow = A.scratch + static_cast<size_t>(si) * A.V * 4;
  if (live) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t idx = lane + 32u * c;
      if (idx < A.V) {
        int* p = srow + 4 * idx;
        if (IsMax) {
          atomicMax(p + 0, f2o(acc[c].x));
          atomicMax(p + 1, f2o(acc[c].y));
          atomicMax(p + 2, f2o(acc[c].z));
          atomicMax(p + 3, f2o(acc[c].w));
        } else {
          atomicMin(p + 0, f2o(acc[c].x));
          atomicMin(p + 1, f2o(acc[c].y));
          atomicMin(p + 2, f2o(acc[c].z));
          atomicMin(p + 3, f2o(acc[c].w));
        }
      }
    }
    if (lane == 0) atomicOr(&A.any_live[t], 1u);
  }
  __threadfence();
  __syncwarp();
  uint32_t prev = 0;
  if (lane == 0) prev = atomicSub(&A.remaining[t], covered);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != covered) return;
  __threadfence();
  const bool any = __ldcg(&A.any_live[t]) != 0;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const uint32_t idx = lane + 32u * c;
    if (idx < A.V) {
      const int4 o = __ldcg(reinterpret_cast<const int4*>(srow) + idx);
      acc[c] = make_float4(o2f(o.x), o2f(o.y), o2f(o.z), o2f(o.w));
    }
  }
  finalize_alpha<IsMax, CPL>(A, t, w, acc, any);
}

// One chunk [b, e) of a target's in-list folded into acc; returns the live
// entries (warp-uniform).
template <bool IsMax, int CPL, int UNROLL>
__device__ __forceinline__ uint32_t reduce_chunk(const AggArgs& A, const uint32_t* ent, uint32_t b, uint32_t e,
                                                 float4 (&acc)[CPL]) {
  const uint32_t lane = threadIdx.x & 31;
  const float ident = IsMax ? -INFINITY : INFINITY;
  uint32_t live = 0;
  if (CPL == 1 && A.V <= 16) {
    // Narrow rows (<= 64 floats): the warp splits into 32 / LPR groups of
    // LPR lanes, each group gathering its own rows (2-4x the rows in flight
    // of one row per warp step), then the groups merge by shuffles.
    const uint32_t LPR = A.V <= 8 ? 8u : 16u, grp = lane / LPR, idx = lane % LPR, G = 32u / LPR;
    for (uint32_t i = b; i < e; i += 32) {
      const uint32_t x = (i + lane < e) ? ent[i + lane] : kFlagDel;
      live += __popc(__ballot_sync(0xffffffffu, !(x & kFlagDel)));
      const uint32_t n = min(32u, e - i);
      // entry q0 + q*G + grp goes to group grp (UNROLL * G divides 32)
      for (uint32_t q0 = 0; q0 < n; q0 += UNROLL * G) {
        float4 rows[UNROLL];
#pragma unroll
        for (int q = 0; q < UNROLL; ++q) {
          const uint32_t id = __shfl_sync(0xffffffffu, x, (q0 + q * G + grp) & 31u);
          rows[q] = (!(id & kFlagDel) && idx < A.V) ? __ldg(A.msg.row4(id & kNodeMask, A.V) + idx)
                                                    : make_float4(ident, ident, ident, ident);
        }
#pragma unroll
        for (int q = 0; q < UNROLL; ++q) acc[0] = sel4<IsMax>(acc[0], rows[q]);
      }
    }
    for (uint32_t o = LPR; o < 32; o <<= 1) {
      float4 v;
      v.x = __shfl_xor_sync(0xffffffffu, acc[0].x, o);
      v.y = __shfl_xor_sync(0xffffffffu, acc[0].y, o);
      v.z = __shfl_xor_sync(0xffffffffu, acc[0].z, o);
      v.w = __shfl_xor_sync(0xffffffffu, acc[0].w, o);
      acc[0] = sel4<IsMax>(acc[0], v);
    }
    return live;
  }
  // Entry q of the 32 loaded is broadcast by one shuffle (no compaction of
  // the live ones: tombstones are rare, and a warp-uniform skip costs less
  // than the per-row find-first-set chain it replaces).
  for (uint32_t i = b; i < e; i += 32) {
    const uint32_t x = (i + lane < e) ? ent[i + lane] : kFlagDel;
    live += __popc(__ballot_sync(0xffffffffu, !(x & kFlagDel)));
    const uint32_t n = min(32u, e - i);
    for (uint32_t q0 = 0; q0 < n; q0 += UNROLL) {
      float4 rows[UNROLL][CPL];
#pragma unroll
      for (int q = 0; q < UNROLL; ++q) {
        const uint32_t id = __shfl_sync(0xffffffffu, x, (q0 + q) & 31u);
        const float4* rp = (id & kFlagDel) ? nullptr : A.msg.row4(id & kNodeMask, A.V);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t idx = lane + 32u * c;
          if (rp && idx < A.V)
            rows[q][c] = __ldg(rp + idx);
          else
            rows[q][c] = make_float4(ident, ident, ident, ident);
        }
      }
#pragma unroll
      for (int q = 0; q < UNROLL; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = sel4<IsMax>(acc[c], rows[q][c]);
    }
  }
  return live;
}

// Work distribution: a round with a few thousand items gives every item its
// own warp visit (latency: a hub's chunks spread over many warps). A round
// with far more items than warps (a hub reset exposing 10^5 targets, or the
// whole-graph pass) hands each warp a block of consecutive items: a target's
// chunks are adjacent in the list, so the warp folds them in registers and
// merges once per target (or finalises in place when it covered all of them)
// instead of once per chunk — fewer scratch atomics and fences.
template <bool IsMax, int CPL>
__global__ void __launch_bounds__(256) k_aggregate(AggArgs A) {
  pdl_prologue();
  constexpr int UNROLL = CPL <= 2 ? 8 : (CPL <= 4 ? 4 : (CPL <= 8 ? 2 : 1));  // rows in flight per warp
  const uint32_t lane = threadIdx.x & 31;
  if (A.abort && *A.abort) return;
  const uint64_t n_work = A.n_work ? *A.n_work : A.n_work_host;
  const float ident = IsMax ? -INFINITY : INFINITY;
  const uint64_t W = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t per_warp = n_work / (2 * W);
  const uint64_t G = per_warp < 1 ? 1 : (per_warp < kAggBlockMax ? per_warp : kAggBlockMax);
  unsigned long long fetched = 0;
  for (uint64_t s0 = gw * G; s0 < n_work; s0 += W * G) {
    const uint64_t s_end = min(s0 + G, n_work);
    uint64_t s = s0, item = A.work[s0];
    uint32_t t = static_cast<uint32_t>(item >> 32);
    while (true) {
      // the run of this block's items that belong to target t
      const uint32_t w = t;  // work items carry the target node
      const uint32_t len = A.in_len[w];
      const uint32_t nch = len == 0 ? 1u : (len + A.chunk - 1) / A.chunk;
      const uint32_t* ent = A.in_ent + A.in_off[w];
      float4 acc[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = make_float4(ident, ident, ident, ident);
      uint32_t live = 0, covered = 0, nt = t;
      for (; s < s_end; ++s) {
        if (covered) {
          item = A.work[s];
          nt = static_cast<uint32_t>(item >> 32);
          if (nt != t) break;
        }
        const uint32_t b = static_cast<uint32_t>(item) * A.chunk, e = min(len, b + A.chunk);
        live += reduce_chunk<IsMax, CPL, UNROLL>(A, ent, b, e, acc);
        ++covered;
      }
      if (lane == 0) fetched += live;  // live is warp-uniform
      finish_chunks<IsMax, CPL>(A, t, w, nch, covered, acc, live);
      if (s >= s_end) break;
      t = nt;
    }
  }
  warp_add(A.fetch_ctr, fetched);
  if (A.ctr) warp_add(&A.ctr[C_RECOMP_ROWS], fetched);
}


// K4 with rows staged through the bulk-copy engine: each warp owns a ring of
// `ring` row slots in shared memory (one mbarrier per slot). Lane 0 issues
// cp.async.bulk for the next rows while the warp reduces the ones that landed,
// so ring * row bytes per warp are in flight regardless of register pressure.
// Smem per warp: ring * V * 16 (rows) + ring * 8 (barriers) + chunk * 4 (ids).
template <bool IsMax, int CPL>
__global__ void __launch_bounds__(128) k_aggregate_bulk(AggArgs A, uint32_t ring) {
  pdl_prologue();
  extern __shared__ __align__(128) unsigned char smem[];
  if (A.abort && *A.abort) return;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t rowbytes = A.V * 16;
  const uint32_t per_warp = ((ring * rowbytes + ring * 8 + A.chunk * 4) + 127) & ~127u;
  unsigned char* base = smem + static_cast<size_t>(wib) * per_warp;
  float4* rows = reinterpret_cast<float4*>(base);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + ring * rowbytes);
  uint32_t* ids = reinterpret_cast<uint32_t*>(base + ring * rowbytes + ring * 8);
  if (lane == 0) {
    for (uint32_t q = 0; q < ring; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  __syncwarp();
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t n_work = A.n_work ? *A.n_work : A.n_work_host;
  const float ident = IsMax ? -INFINITY : INFINITY;
  unsigned long long fetched = 0;
  uint32_t g = 0;  // rows issued by this warp so far (slot = g % ring, parity = (g / ring) & 1)
  WarpQueue wq;
  wq.init(A.next, n_work, 2);
  (void)warps;
  for (uint64_t it; wq.next(it);) {
    const uint64_t item = A.work[it];
    const uint32_t t = static_cast<uint32_t>(item >> 32), c0 = static_cast<uint32_t>(item);
    const uint32_t w = t;  // work items carry the target node
    const uint32_t len = A.in_len[w];
    const uint32_t nch = len == 0 ? 1u : (len + A.chunk - 1) / A.chunk;
    const uint32_t b = c0 * A.chunk, e = min(len, b + A.chunk);
    const uint32_t* ent = A.in_ent + A.in_off[w];
    // live ids of this chunk into shared memory
    uint32_t n = 0;
    for (uint32_t i = b; i < e; i += 32) {
      const uint32_t x = (i + lane < e) ? ent[i + lane] : kFlagDel;
      const bool live = !(x & kFlagDel);
      const uint32_t mask = __ballot_sync(0xffffffffu, live);
      if (live) ids[n + __popc(mask & ((1u << lane) - 1u))] = x & kNodeMask;
      n += __popc(mask);
    }
    __syncwarp();
    float4 acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = make_float4(ident, ident, ident, ident);
    const uint32_t g0 = g;
    // Slot reuse needs no proxy fence: every generic read of a slot has been
    // consumed (its value folded into acc) before the __syncwarp that precedes
    // the next bulk copy into it.
    if (lane == 0) {
      for (uint32_t q = 0; q < min(ring, n); ++q) {
        const uint32_t slot = (g0 + q) % ring;
        bulk_row_load(rows + static_cast<size_t>(slot) * A.V, A.msg.row4(ids[q], A.V), rowbytes,
                      &bar[slot]);
      }
    }
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t gi = g0 + i, slot = gi % ring;
      mbar_wait(&bar[slot], (gi / ring) & 1u);
      const float4* r = rows + static_cast<size_t>(slot) * A.V;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t idx = lane + 32u * c;
        if (idx < A.V) acc[c] = sel4<IsMax>(acc[c], r[idx]);
      }
      __syncwarp();
      if (lane == 0 && i + ring < n) {
        bulk_row_load(rows + static_cast<size_t>(slot) * A.V, A.msg.row4(ids[i + ring], A.V),
                      rowbytes, &bar[slot]);
      }
    }
    g = g0 + n;
    __syncwarp();
    if (lane == 0) fetched += n;
    finish_chunks<IsMax, CPL>(A, t, w, nch, 1u, acc, n);
  }
  warp_add(A.fetch_ctr, fetched);
  if (A.ctr) warp_add(&A.ctr[C_RECOMP_ROWS], fetched);
}

// Sparse exposed-reset recompute (see classify_target): warp per (slot, chunk
// of kSparseChunk in-list entries); each lane takes live in-neighbours and
// reads only the slot's <= kSparseDims uncovered positions of their current
// messages (4-byte gathers instead of whole rows), the warp reduces, and lane 0
// merges with order-preserving integer atomics. Counters match the dense path:
// every live in-neighbour is one fetched row (recompute, engine.cpp:89-99).
struct SparseArgs {
  const uint64_t* swork;
  const unsigned long long* n_swork;
  const unsigned long long* abort;
  const uint32_t* sp_target;
  const uint32_t* sp_n;
  const uint32_t* sp_dims;
  const float* sp_aold;
  int* sp_acc;
  uint32_t* sp_live;
  const uint32_t* sp_changed;
  const unsigned long long* n_sparse;
  uint32_t* sp_remaining;
  const uint64_t* in_off;
  const uint32_t* in_len;
  const uint32_t* in_ent;
  RowTable msg;        // m_l, pitch P floats (rows of every shard)
  float* agg;          // a_l, pitch P floats
  uint32_t P;
  uint8_t* run_flags;
  unsigned long long* fetch_ctr;
  unsigned long long* ctr;
};

// Finalise one sparse slot (called by the slot's last merging chunk): write
// the recomputed positions (zero when no live in-neighbour remains,
// engine.cpp:89-99), bitwise change test, dirty flag. Returns 1 when alpha
// changed.
template <bool IsMax>
__device__ __forceinline__ unsigned long long sparse_finalize_slot(const SparseArgs& S, uint32_t sp) {
  const uint32_t w = S.sp_target[sp], nd = S.sp_n[sp];
  const bool any = __ldcg(&S.sp_live[sp]) != 0;
  bool changed = S.sp_changed[sp] != 0;
  float* arow = S.agg + static_cast<size_t>(w) * S.P;
  // all loads before the stores (one round trip instead of one per position)
  float v[kSparseDims], old[kSparseDims];
  uint32_t dim[kSparseDims];
#pragma unroll
  for (uint32_t k = 0; k < kSparseDims; ++k) {
    if (k < nd) {
      v[k] = any ? o2f(__ldcg(&S.sp_acc[sp * kSparseDims + k])) : 0.0f;
      dim[k] = S.sp_dims[sp * kSparseDims + k];
      old[k] = S.sp_aold[sp * kSparseDims + k];
    }
  }
#pragma unroll
  for (uint32_t k = 0; k < kSparseDims; ++k) {
    if (k < nd) {
      arow[dim[k]] = v[k];
      if (__float_as_uint(v[k]) != __float_as_uint(old[k])) changed = true;
    }
  }
  const uint8_t f = S.run_flags[w];
  if (changed || (f & RUN_SELF)) S.run_flags[w] = f | RUN_DIRTY;
  return changed ? 1ull : 0ull;
}

template <bool IsMax>
__global__ void __launch_bounds__(256) k_recompute_sparse(SparseArgs S) {
  pdl_prologue();
  if (*S.abort) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t n_work = *S.n_swork;
  const float ident = IsMax ? -INFINITY : INFINITY;
  unsigned long long fetched = 0, loads = 0, writes = 0;
  for (uint64_t it = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; it < n_work;
       it += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    const uint64_t item = S.swork[it];
    const uint32_t sp = static_cast<uint32_t>(item >> 32), c = static_cast<uint32_t>(item);
    const uint32_t w = S.sp_target[sp], n = S.sp_n[sp];
    uint32_t dims[kSparseDims];
#pragma unroll
    for (uint32_t k = 0; k < kSparseDims; ++k) dims[k] = k < n ? S.sp_dims[sp * kSparseDims + k] : 0u;
    const uint32_t len = S.in_len[w];
    const uint32_t b = c * kSparseChunk, e = min(len, b + kSparseChunk);
    const uint32_t* ent = S.in_ent + S.in_off[w];
    float acc[kSparseDims];
#pragma unroll
    for (uint32_t k = 0; k < kSparseDims; ++k) acc[k] = ident;
    uint32_t live = 0;
    // 4 entries per lane per step: all 4 * n gathers are issued (predicated
    // loads, no per-entry branch) before the first compare, so a step costs
    // one memory round trip instead of one per entry
    for (uint32_t i0 = b; i0 < e; i0 += 128) {
      uint32_t x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + 32u * u + lane;
        x[u] = i < e ? ent[i] : kFlagDel;
      }
      float v[4][kSparseDims];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = !(x[u] & kFlagDel);
        live += ok ? 1u : 0u;
        const float* row = S.msg.row(x[u] & kNodeMask, S.P);
#pragma unroll
        for (uint32_t k = 0; k < kSparseDims; ++k) v[u][k] = (ok && k < n) ? __ldg(row + dims[k]) : ident;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (uint32_t k = 0; k < kSparseDims; ++k) acc[k] = sel<IsMax>(acc[k], v[u][k]);
    }
#pragma unroll
    for (uint32_t k = 0; k < kSparseDims; ++k) {
      if (k >= n) break;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float v = __shfl_xor_sync(0xffffffffu, acc[k], o);
        acc[k] = IsMax ? fmaxf(acc[k], v) : fminf(acc[k], v);
      }
    }
    for (int o = 16; o; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
    if (lane == 0) {
      if (live) {
        for (uint32_t k = 0; k < n; ++k) {
          if (IsMax) atomicMax(&S.sp_acc[sp * kSparseDims + k], f2o(acc[k]));
          else atomicMin(&S.sp_acc[sp * kSparseDims + k], f2o(acc[k]));
        }
        atomicAdd(&S.sp_live[sp], live);
      }
      fetched += live;
      loads += static_cast<unsigned long long>(live) * n;
      __threadfence();
      if (atomicSub(&S.sp_remaining[sp], 1u) == 1u) {  // last chunk of the slot: finalise it
        __threadfence();
        writes += sparse_finalize_slot<IsMax>(S, sp);
      }
    }
  }
  if (writes) atomicAdd(&S.ctr[C_AWRITES], writes);
  warp_add(S.fetch_ctr, fetched);
  warp_add(&S.ctr[C_SPARSE_LOADS], loads);
  warp_add(&S.ctr[C_SPARSE_ROWS], fetched);
}

// Init/verify work list over all nodes: items (v, c) for c < max(1, ceil(len/chunk)).
// Whole-graph pass over the nodes [v0, v0 + n) (a shard's own range): chunk
// counts and work items indexed by local position, items name node ids.
__global__ void k_node_chunks(const uint32_t* in_len, uint32_t v0, uint32_t n, uint32_t chunk, uint64_t* nch) {
  pdl_prologue();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t len = in_len[v0 + i];
  nch[i] = len == 0 ? 1u : (len + chunk - 1) / chunk;
}

__global__ void k_node_work(const uint64_t* nch_scan, const uint64_t* nch, uint32_t v0, uint32_t n, uint64_t* work,
                            uint32_t* scratch_idx, uint32_t* remaining, uint32_t* any_live,
                            unsigned long long* n_scratch) {
  pdl_prologue();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t v = v0 + i;
  const uint64_t base = nch_scan[i], c = nch[i];
  for (uint64_t q = 0; q < c; ++q) work[base + q] = (static_cast<uint64_t>(v) << 32) | q;
  if (c > 1) {
    scratch_idx[v] = static_cast<uint32_t>(atomicAdd(n_scratch, 1ull));
    remaining[v] = static_cast<uint32_t>(c);
    any_live[v] = 0;
  }
}

// Node-list variants (k-hop recompute comparator): chunk counts and work items
// for the targets list[0..n), indexed by node id like the whole-graph pass.
__global__ void k_list_chunks(const uint32_t* list, uint32_t n, const uint32_t* in_len, uint32_t chunk,
                              uint64_t* nch) {
  pdl_prologue();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t len = in_len[list[i]];
  nch[i] = len == 0 ? 1u : (len + chunk - 1) / chunk;
}

__global__ void k_list_work(const uint32_t* list, const uint64_t* nch_scan, const uint64_t* nch, uint32_t n,
                            uint64_t* work, uint32_t* scratch_idx, uint32_t* remaining, uint32_t* any_live,
                            unsigned long long* n_scratch) {
  pdl_prologue();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t v = list[i];
  const uint64_t base = nch_scan[i], c = nch[i];
  for (uint64_t j = 0; j < c; ++j) work[base + j] = (static_cast<uint64_t>(v) << 32) | j;
  if (c > 1) {
    scratch_idx[v] = static_cast<uint32_t>(atomicAdd(n_scratch, 1ull));
    remaining[v] = static_cast<uint32_t>(c);
    any_live[v] = 0;
  }
}

__global__ void k_fill_int(int* p, uint64_t n, int value) {
  pdl_prologue();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = value;
}

}  // namespace sgb
