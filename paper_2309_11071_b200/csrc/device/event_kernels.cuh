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

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "dev_common.cuh"
#include "graph_kernels.cuh"

namespace sgb {

// Table/row addressing for one layer's messages.
struct MsgView {
  RowTable cur;           // m_l table, pitch V float4 (rows of every shard)
  const float4* old;      // pre-image slab (rows indexed by dirty slot), or null at layer 1
  const uint32_t* stamp;  // round stamp per node (msg_l rewritten this round), or null
  const uint32_t* slot;
  const uint64_t* net;    // this round's net delta (seed records)
  const uint32_t* dprev;  // previous layer's dirty list (expansion records)
  const uint32_t* round;   // device-resident round id (graph-replay safe)
  uint32_t V;
  __device__ __forceinline__ const float4* cur_row(uint32_t u) const { return cur.row4(u, V); }
  __device__ __forceinline__ const float4* prev_row(uint32_t u) const {
    if (stamp && stamp[u] == *round) return old + static_cast<size_t>(slot[u]) * V;
    return cur_row(u);
  }
};

// Grouping by target is a counting sort: every generator bumps cnt[target]
// (the returned ordinal is the record's slot inside its group) and the first
// record of a target appends it to the run list; an exclusive scan of cnt over
// the node range gives each group's offset and k_scatter places the records.
struct RecSink {
  uint64_t* rec;              // unsorted records
  uint32_t* ord;              // their slot within the target's group
  uint32_t* cnt;              // [N] records per target (zeroed per layer)
  uint32_t* runs;             // targets with >= 1 record (unordered)
  unsigned long long* num_runs;
  unsigned long long* cursor; // next free record slot
  uint8_t* exact;             // run flags: RUN_EXACT marks put() targets (pre-filtered layers), else null
  uint32_t lo, hi;            // owned target range [lo, hi) (the whole graph unless sharded)
  // Pre-filtered layers: targets are registered as runs through this 2-bit
  // per target map (touch), since a target may have events but no records
  // (hit-free PAIRs write none): bit 0 = touched, bit 1 = has a PAIR (hence a
  // Del event). null = a target's first record registers it.
  uint32_t* touched;
  __device__ __forceinline__ bool owns(uint32_t t) const { return t >= lo && t < hi; }
  __device__ __forceinline__ void touch(uint32_t t, bool pair = false) const {
    const uint32_t sh = 2u * (t & 15u);
    if (!(atomicOr(&touched[t >> 4], (pair ? 3u : 1u) << sh) & (1u << sh))) runs[atomicAdd(num_runs, 1ull)] = t;
  }
  __device__ __forceinline__ void put(uint64_t i, uint64_t r) const {
    const uint32_t t = static_cast<uint32_t>(r >> 32);
    if (!owns(t)) {  // another shard's target: leave an empty slot
      rec[i] = kNoRecord;
      return;
    }
    const uint32_t o = atomicAdd(&cnt[t], 1u);
    if (touched) touch(t);
    else if (o == 0) runs[atomicAdd(num_runs, 1ull)] = t;
    rec[i] = r;
    ord[i] = o;
    if (exact) exact[t] = RUN_EXACT;
  }
};

// One next-layer expansion work item: kExpandChunk entries of a dirty source's
// out-list, with the list already resolved by its producer (K5 or the shard
// import's plan), so an expansion task starts from one 32-byte load instead of
// the chain item -> dirty node -> list offset / length.
struct ExpItem {
  uint64_t off;   // out-list start in the slab pool
  uint32_t j;     // the source's position in the previous layer's dirty list
  uint32_t v;     // the source node
  uint32_t len;   // out-list length (this round's DEL/NEW entries included)
  uint32_t c;     // chunk index
  uint32_t pad[2];
};
__device__ __forceinline__ void put_exp_items(ExpItem* work, unsigned long long* exp_n, uint32_t j, uint32_t v,
                                              uint32_t len, uint64_t off) {
  const uint32_t nch = (len + kExpandChunk - 1) / kExpandChunk;
  if (!nch) return;
  const unsigned long long w0 = atomicAdd(exp_n, static_cast<unsigned long long>(nch));
  for (uint32_t c = 0; c < nch; ++c) work[w0 + c] = ExpItem{off, j, v, len, c, {0, 0}};
}

// Seeds (seed_edge_events, engine.cpp:101-112): one record per net edge per
// layer; Del carries the source's previous message, Add its current one.
struct SeedArgs {
  const uint64_t* net;  // null: no seeds in this launch
  const unsigned long long* num_net;
  uint32_t mult;
  RecSink S;
  unsigned long long* ctr;
};
__device__ __forceinline__ void put_seeds(const SeedArgs& A) {
  if (!A.net) return;
  const uint64_t num_net = *A.num_net;
  unsigned long long owned = 0;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < num_net;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = A.net[j];
    const uint32_t d = static_cast<uint32_t>(k) & kNodeMask;
    const uint64_t r = make_record(d, static_cast<uint32_t>(j), (k >> 63) ? EV_SEED_DEL : EV_SEED_ADD);
    owned += A.S.owns(d);
    for (uint32_t m = 0; m < A.mult; ++m) A.S.put(j * A.mult + m, r);
  }
  warp_add(A.ctr, owned);
}

__global__ void k_seed_records(const uint64_t* net, const unsigned long long* num_net_p, uint32_t mult, RecSink S,
                               unsigned long long* seeds_ctr, const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  const uint64_t num_net = *num_net_p;
  unsigned long long owned = 0;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < num_net;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = net[j];
    const uint32_t d = static_cast<uint32_t>(k) & kNodeMask;
    const uint64_t r = make_record(d, static_cast<uint32_t>(j), (k >> 63) ? EV_SEED_DEL : EV_SEED_ADD);
    owned += S.owns(d);
    for (uint32_t m = 0; m < mult; ++m) S.put(j * mult + m, r);
  }
  warp_add(seeds_ctr, owned);
}

// K1 for batches of <= kGroupCap updates (graph_kernels.cuh): grouping,
// validation, relocation election and the gate, then (round not aborted) the
// slab relocations, the net ops and layer 1's seed records, in one CTA.
__global__ void __launch_bounds__(1024, 1) k_batch_group(const char* ops, const uint32_t* src, const uint32_t* dst,
                                                      uint32_t B, uint32_t n, uint32_t cap, EdgeHash h, AdjView out,
                                                      AdjView in, uint64_t* keys, uint64_t* net,
                                                      unsigned long long* err, uint32_t* badop,
                                                      unsigned long long* counts, unsigned long long* num_net,
                                                      const uint32_t* round_p, uint32_t* reloc_list,
                                                      const unsigned long long* pool_top,
                                                      unsigned long long pool_cap, unsigned long long* abort,
                                                      uint32_t mult, unsigned long long* cursors, uint32_t stride,
                                                      uint32_t layers, unsigned long long* pool_top_rw,
                                                      uint32_t* touched_out, uint32_t* touched_in, DelLists dl,
                                                      bool seed, RecSink S, unsigned long long* seeds_ctr,
                                                      unsigned long long* scal, uint32_t n_scal,
                                                      unsigned long long* ctr, uint32_t n_ctr) {
  pdl_prologue();
  extern __shared__ __align__(16) unsigned char gsm_[];
  // the round's scalars and counters start here (no memset nodes in the
  // round graph): all zero but the first-failure slot (min-reduced)
  for (uint32_t q = threadIdx.x; q < n_scal; q += blockDim.x) scal[q] = scal + q == err ? ~0ull : 0ull;
  for (uint32_t q = threadIdx.x; q < n_ctr; q += blockDim.x) ctr[q] = 0ull;
  const uint32_t tsz = 2 * cap, tmask = tsz - 1;
  unsigned long long* tkey = reinterpret_cast<unsigned long long*>(gsm_);
  uint64_t* bkey = reinterpret_cast<uint64_t*>(gsm_ + 8ull * tsz);
  uint32_t* tfirst = reinterpret_cast<uint32_t*>(gsm_ + 8ull * tsz + 8ull * cap);
  uint32_t* tcount = tfirst + tsz;
  uint32_t* slot_of = tcount + tsz;
  for (uint32_t q = threadIdx.x; q < tsz; q += blockDim.x) {
    tkey[q] = kHashEmpty;
    tfirst[q] = 0xFFFFFFFFu;
    tcount[q] = 0;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
    const char o = ops[i];
    if (o != '+' && o != '-') atomicOr(badop, 1u);
    const uint32_t s = src[i], d = dst[i];
    const uint64_t key = (static_cast<uint64_t>(s) << 32) | d;
    keys[i] = key;
    if (s >= n || d >= n) {
      atomicMin(err, (static_cast<unsigned long long>(i) << 8) | ERR_RANGE);
      bkey[i] = kHashEmpty;  // never grouped
      continue;
    }
    bkey[i] = key;
    uint32_t slot = static_cast<uint32_t>(hash_home(key, tmask));
    for (;; slot = (slot + 1) & tmask) {
      const unsigned long long prev = atomicCAS(&tkey[slot], kHashEmpty, static_cast<unsigned long long>(key));
      if (prev == kHashEmpty || prev == key) break;
    }
    slot_of[i] = slot;
    atomicMin(&tfirst[slot], i);
    atomicAdd(&tcount[slot], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
    const uint64_t key = bkey[i];
    if (key == kHashEmpty) continue;
    const uint32_t slot = slot_of[i];
    if (tfirst[slot] != i) continue;  // not the key's first op
    const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
    uint64_t hslot;
    const bool present = hash_find(h, key, &hslot);
    bool p = present, ok = true;
    uint32_t left = tcount[slot];
    for (uint32_t j = i; j < B && left; ++j) {
      if (bkey[j] != key) continue;
      --left;
      const bool ins = ops[j] == '+';
      if (ins && p) {
        atomicMin(err, (static_cast<unsigned long long>(j) << 8) | ERR_DUP);
        ok = false;
        break;
      }
      if (!ins && !p) {
        atomicMin(err, (static_cast<unsigned long long>(j) << 8) | ERR_MISSING);
        ok = false;
        break;
      }
      p = ins;
    }
    if (!ok || p == present) continue;
    net[atomicAdd(num_net, 1ull)] = p ? key : (key | (1ull << 63));
    if (p) {
      atomicAdd(&counts[0], 1ull);
      atomicAdd(&out.n_new[s], 1u);
      atomicAdd(&in.n_new[d], 1u);
    } else {
      atomicAdd(&counts[1], 1ull);
    }
  }
  // k_reloc_plan and k_round_gate, fused: the CTA's own writes are visible
  // after the barrier
  __syncthreads();
  const uint32_t round = *round_p;
  const uint64_t nn = *num_net;
  for (uint64_t j = threadIdx.x; j < nn; j += blockDim.x) reloc_plan_one(net[j], out, in, round, reloc_list, counts);
  __syncthreads();
  if (threadIdx.x == 0)
    round_gate(err, reinterpret_cast<const unsigned long long*>(badop), counts + 3, pool_top, pool_cap, abort,
               num_net, mult, cursors, stride, layers);
  // k_relocate, k_apply_net and layer 1's k_seed_records, fused: a warp per
  // elected slab, then a thread per net op (the CTA's global writes are
  // visible to it after each barrier)
  __syncthreads();
  if (*abort) return;
  const uint32_t n_reloc = static_cast<uint32_t>(counts[2]);
  for (uint32_t w = threadIdx.x >> 5; w < n_reloc; w += blockDim.x >> 5)
    relocate_one(reloc_list[w], out, in, pool_top_rw);
  __syncthreads();
  unsigned long long owned = 0;
  for (uint64_t j = threadIdx.x; j < nn; j += blockDim.x) {
    const uint64_t k = net[j];
    apply_net_one(k, out, in, h, round, touched_out, touched_in, dl, counts);
    if (seed) {  // seed_edge_events (engine.cpp:101-112) of layer 1
      const uint32_t d = static_cast<uint32_t>(k) & kNodeMask;
      const uint64_t r = make_record(d, static_cast<uint32_t>(j), (k >> 63) ? EV_SEED_DEL : EV_SEED_ADD);
      owned += S.owns(d);
      for (uint32_t m = 0; m < mult; ++m) S.put(j * mult + m, r);
    }
  }
  if (seed) warp_add(seeds_ctr, owned);
}

// K1 for batches of <= kGroupCapPre updates: k_batch_group with the round's
// dependent global round trips cut from about a dozen to four. Everything a
// later phase needs from the committed graph is loaded in the grouping phase,
// where every op's loads are independent and overlap: the edge-index probe
// (found slot and its out/in positions, or the first free slot on the probe
// path for an insert), and the length, capacity and list offset of both
// endpoints. The CTA's own counters (net ops, first failure, relocation
// demand, touched lists, deletion records) live in shared memory and are
// written out once at the end, and the gate reads nothing from global memory.
// A slab relocation is elected by the insert whose returned NEW ordinal is
// the first that does not fit (len + ordinal == cap; n_new starts at 0 and
// len <= cap), so the common round reads no counter back; the demand of the
// (rare) elected lists is summed after the grouping phase.
constexpr uint32_t kGroupCapPre = 2048;
__host__ __device__ constexpr size_t batch_group_pre_smem(uint32_t cap) {
  return batch_group_smem(cap) + static_cast<size_t>(cap) * (8 + 8 + 16 + 16 + 4);
}
constexpr unsigned long long kProbePresent = 1ull << 63, kProbeTomb = 1ull << 62;

__global__ void __launch_bounds__(1024, 1) k_batch_group_pre(const char* ops, const uint32_t* src, const uint32_t* dst,
                                                          uint32_t B, uint32_t n, uint32_t cap, EdgeHash h,
                                                          AdjView out, AdjView in, uint64_t* keys, uint64_t* net,
                                                          unsigned long long* err, uint32_t* badop,
                                                          unsigned long long* counts, unsigned long long* num_net,
                                                          const uint32_t* round_p, uint32_t* reloc_list,
                                                          const unsigned long long* pool_top,
                                                          unsigned long long pool_cap, unsigned long long* abort,
                                                          uint32_t mult, unsigned long long* cursors, uint32_t stride,
                                                          uint32_t layers, unsigned long long* pool_top_rw,
                                                          uint32_t* touched_out, uint32_t* touched_in, DelLists dl,
                                                          bool seed, RecSink S, unsigned long long* seeds_ctr,
                                                          unsigned long long* scal, uint32_t n_scal,
                                                          unsigned long long* ctr, uint32_t n_ctr) {
  pdl_prologue();
  extern __shared__ __align__(16) unsigned char gsm_[];
  __shared__ unsigned long long sh_err, sh_cnt[6], sh_num_net, sh_delrec, sh_pool_top;
  __shared__ uint32_t sh_badop, sh_round, sh_abort;
  for (uint32_t q = threadIdx.x; q < n_scal; q += blockDim.x) scal[q] = scal + q == err ? ~0ull : 0ull;
  for (uint32_t q = threadIdx.x; q < n_ctr; q += blockDim.x) ctr[q] = 0ull;
  const uint32_t tsz = 2 * cap, tmask = tsz - 1;
  unsigned long long* tkey = reinterpret_cast<unsigned long long*>(gsm_);
  uint64_t* bkey = reinterpret_cast<uint64_t*>(gsm_ + 8ull * tsz);
  uint32_t* tfirst = reinterpret_cast<uint32_t*>(gsm_ + 8ull * tsz + 8ull * cap);
  uint32_t* tcount = tfirst + tsz;
  uint32_t* slot_of = tcount + tsz;
  // prefetched per op: probe result, out/in positions, len/cap of both ends,
  // list offsets of both ends, and (per net op) the op it came from
  uint64_t* p_slot = reinterpret_cast<uint64_t*>(gsm_ + batch_group_smem(cap));
  uint64_t* p_off = p_slot + cap;       // [2 cap]
  uint32_t* p_pos = reinterpret_cast<uint32_t*>(p_off + 2ull * cap);  // [2 cap]
  uint32_t* p_lc = p_pos + 2ull * cap;  // [4 cap]: len_s, cap_s, len_d, cap_d
  uint32_t* p_net_op = p_lc + 4ull * cap;
  for (uint32_t q = threadIdx.x; q < tsz; q += blockDim.x) {
    tkey[q] = kHashEmpty;
    tfirst[q] = 0xFFFFFFFFu;
    tcount[q] = 0;
  }
  if (threadIdx.x == 0) {
    sh_err = ~0ull;
    for (int q = 0; q < 6; ++q) sh_cnt[q] = 0;
    sh_num_net = 0;
    sh_delrec = 0;
    sh_badop = 0;
    sh_round = *round_p;
    sh_pool_top = *pool_top;
  }
  __syncthreads();
  // ---- grouping + every committed-state load of the round
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
    const char o = ops[i];
    const uint32_t s = src[i], d = dst[i];
    if (o != '+' && o != '-') atomicOr(&sh_badop, 1u);
    const uint64_t key = (static_cast<uint64_t>(s) << 32) | d;
    keys[i] = key;
    if (s >= n || d >= n) {
      atomicMin(&sh_err, (static_cast<unsigned long long>(i) << 8) | ERR_RANGE);
      bkey[i] = kHashEmpty;  // never grouped
      continue;
    }
    // independent loads first: endpoint lengths, capacities, offsets, probe head
    const uint32_t ls = out.len[s], cs = out.cap[s], ld = in.len[d], cd = in.cap[d];
    const uint64_t os = out.off[s], od = in.off[d];
    uint64_t hi = hash_home(key, h.mask);
    HashSlot hsl = load_slot(h.s + hi);
    unsigned long long hk = hsl.key;
    bkey[i] = key;
    uint32_t slot = static_cast<uint32_t>(hash_home(key, tmask));
    for (;; slot = (slot + 1) & tmask) {
      const unsigned long long prev = atomicCAS(&tkey[slot], kHashEmpty, static_cast<unsigned long long>(key));
      if (prev == kHashEmpty || prev == key) break;
    }
    slot_of[i] = slot;
    atomicMin(&tfirst[slot], i);
    atomicAdd(&tcount[slot], 1u);
    // probe: the key's slot, or the first free (empty / tombstone) slot on its
    // path (where hash_insert would put it)
    uint64_t free_slot = ~0ull;
    bool free_tomb = false;
    for (;;) {
      if (hk == key) break;
      if (hk == kHashTomb && free_slot == ~0ull) {
        free_slot = hi;
        free_tomb = true;
      }
      if (hk == kHashEmpty) {
        if (free_slot == ~0ull) free_slot = hi;
        break;
      }
      hi = (hi + 1) & h.mask;
      hsl = load_slot(h.s + hi);
      hk = hsl.key;
    }
    if (hk == key) {
      p_slot[i] = hi | kProbePresent;
      p_pos[2 * i] = hsl.pos_out;
      p_pos[2 * i + 1] = hsl.pos_in;
    } else {
      p_slot[i] = free_slot | (free_tomb ? kProbeTomb : 0ull);
    }
    p_lc[4 * i] = ls;
    p_lc[4 * i + 1] = cs;
    p_lc[4 * i + 2] = ld;
    p_lc[4 * i + 3] = cd;
    p_off[2 * i] = os;
    p_off[2 * i + 1] = od;
  }
  __syncthreads();
  // ---- validation walk (k_validate), net ops, relocation election
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
    const uint64_t key = bkey[i];
    if (key == kHashEmpty) continue;
    const uint32_t slot = slot_of[i];
    if (tfirst[slot] != i) continue;  // not the key's first op
    const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
    const bool present = (p_slot[i] & kProbePresent) != 0;
    bool p = present, ok = true;
    uint32_t left = tcount[slot];
    for (uint32_t j = i; j < B && left; ++j) {
      if (bkey[j] != key) continue;
      --left;
      const bool ins = ops[j] == '+';
      if (ins && p) {
        atomicMin(&sh_err, (static_cast<unsigned long long>(j) << 8) | ERR_DUP);
        ok = false;
        break;
      }
      if (!ins && !p) {
        atomicMin(&sh_err, (static_cast<unsigned long long>(j) << 8) | ERR_MISSING);
        ok = false;
        break;
      }
      p = ins;
    }
    if (!ok || p == present) continue;
    const uint32_t j = static_cast<uint32_t>(atomicAdd(&sh_num_net, 1ull));
    net[j] = p ? key : (key | (1ull << 63));
    p_net_op[j] = i;
    if (p) {
      atomicAdd(&sh_cnt[0], 1ull);
      const uint32_t os_new = atomicAdd(&out.n_new[s], 1u), od_new = atomicAdd(&in.n_new[d], 1u);
      if (p_lc[4 * i] + os_new == p_lc[4 * i + 1]) reloc_list[atomicAdd(&sh_cnt[2], 1ull)] = s;
      if (p_lc[4 * i + 2] + od_new == p_lc[4 * i + 3]) reloc_list[atomicAdd(&sh_cnt[2], 1ull)] = (1u << 31) | d;
    } else {
      atomicAdd(&sh_cnt[1], 1ull);
    }
  }
  __syncthreads();
  const uint32_t n_reloc = static_cast<uint32_t>(sh_cnt[2]);
  for (uint32_t w = threadIdx.x; w < n_reloc; w += blockDim.x) {  // demand of the elected lists (rare)
    const uint32_t code = reloc_list[w], v = code & 0x7FFFFFFFu;
    const AdjView& a = (code >> 31) ? in : out;
    atomicAdd(&sh_cnt[3], static_cast<unsigned long long>(grow_cap(a.len[v] + a.n_new[v])));
  }
  __syncthreads();
  const uint64_t nn = sh_num_net;
  if (threadIdx.x == 0) {  // the gate (round_gate), from shared memory
    unsigned long long a = 0;
    if (sh_badop) a = 1;
    else if (sh_err != ~0ull) a = 2;
    else if (sh_pool_top + sh_cnt[3] > pool_cap) a = 3;
    sh_abort = static_cast<uint32_t>(a);
    *abort = a;
    for (uint32_t l = 0; l < layers; ++l) cursors[l * stride] = nn * mult;
  }
  __syncthreads();
  if (!sh_abort) {
    for (uint32_t w = threadIdx.x >> 5; w < n_reloc; w += blockDim.x >> 5)
      relocate_one(reloc_list[w], out, in, pool_top_rw);
    if (n_reloc) __syncthreads();
    const uint32_t round = sh_round;
    unsigned long long owned = 0;
    for (uint32_t j = threadIdx.x; j < nn; j += blockDim.x) {
      const uint32_t i = p_net_op[j];
      const uint64_t key = bkey[i], ps = p_slot[i];
      const bool del = (ps & kProbePresent) != 0;  // a net op flips the committed presence
      const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
      const uint32_t ts = atomicExch(&out.touch[s], round), td = atomicExch(&in.touch[d], round);
      const uint64_t os = n_reloc ? out.off[s] : p_off[2 * i], od = n_reloc ? in.off[d] : p_off[2 * i + 1];
      if (!del) {
        const uint32_t po = atomicAdd(&out.len[s], 1u);
        const uint32_t pi = atomicAdd(&in.len[d], 1u);
        const uint64_t fs = ps & ~(kProbePresent | kProbeTomb);
        const unsigned long long expect = (ps & kProbeTomb) ? kHashTomb : kHashEmpty;
        uint64_t slot = fs;
        if (atomicCAS(&h.s[fs].key, expect, static_cast<unsigned long long>(key)) != expect)
          slot = hash_insert(h, key);  // another insert of this round took the slot
        out.ent[os + po] = d | kFlagNew;
        in.ent[od + pi] = s | kFlagNew;
        h.s[slot].pos_out = po;
        h.s[slot].pos_in = pi;
      } else {
        const uint32_t r = static_cast<uint32_t>(atomicAdd(&sh_delrec, 2ull));
        const uint32_t ho = atomicExch(&dl.head_out[s], r), hi = atomicExch(&dl.head_in[d], r + 1);
        atomicAdd(&out.n_del[s], 1u);
        atomicAdd(&in.n_del[d], 1u);
        const uint32_t po = p_pos[2 * i], pi = p_pos[2 * i + 1];
        atomicOr(&out.ent[os + po], kFlagDel);
        atomicOr(&in.ent[od + pi], kFlagDel);
        dl.pos[r] = po;
        dl.next[r] = ho;
        dl.pos[r + 1] = pi;
        dl.next[r + 1] = hi;
      }
      if (ts != round) touched_out[atomicAdd(&sh_cnt[4], 1ull)] = s;
      if (td != round) touched_in[atomicAdd(&sh_cnt[5], 1ull)] = d;
      if (seed) {  // seed_edge_events (engine.cpp:101-112) of layer 1
        const uint64_t r = make_record(d, j, del ? EV_SEED_DEL : EV_SEED_ADD);
        owned += S.owns(d);
        for (uint32_t m = 0; m < mult; ++m) S.put(j * mult + m, r);
      }
    }
    if (seed) warp_add(seeds_ctr, owned);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the CTA's counters, once
    *err = sh_err;
    *badop = sh_badop;
    for (int q = 0; q < 6; ++q) counts[q] = sh_cnt[q];
    *num_net = sh_num_net;
    *dl.cursor = sh_delrec;
  }
}



// K1 as one 8-CTA thread-block cluster (batches <= kGroupCapCluster): the
// same phases as k_batch_group_pre, spread over eight SMs. A batch's K1 is a
// few random accesses per op into the committed graph (edge-index probe,
// endpoint lengths/capacities/offsets, then the appends, tombstones and index
// inserts), about 20K scattered memory operations per 1K-op batch; from one
// SM their rate, not their dependency chain, bounds the kernel (the
// single-CTA kernel stayed at ~35 us at C2 after its chain was cut from a
// dozen round trips to four). Here each SM issues an eighth of them. The
// grouping table and the round's counters live in rank 0's shared memory and
// are reached through distributed shared memory (atomics included); each CTA
// keeps a copy of the batch keys for the in-order validation walk and the
// prefetched state of its own ops, and applies its own ops' net effects.
// Cluster barriers order every phase (release/acquire at cluster scope, with a
// fence for the global writes other CTAs read).
constexpr uint32_t kClusterK1 = 8, kClusterK1Threads = 128;
constexpr uint32_t kGroupCapCluster = 2048;
constexpr uint32_t kOpsPerCtaMax = kGroupCapCluster / kClusterK1;  // 256 ops per CTA
__host__ __device__ constexpr size_t batch_cluster_smem(uint32_t cap) {
  // rank 0's grouping table (2 cap slots: key, first op, op count), every
  // CTA's copy of the keys (cap) and ops (cap bytes), per-op prefetch of the
  // CTA's own ops: probe (8), offsets (16), positions (8), len/cap (16),
  // table slot (4), net index (4)
  return static_cast<size_t>(2 * cap) * (8 + 4 + 4) + static_cast<size_t>(cap) * (8 + 1) +
         static_cast<size_t>(kOpsPerCtaMax) * (8 + 16 + 8 + 16 + 4 + 4) + 64;
}

struct ClusterK1Shared {
  unsigned long long err, cnt[6], num_net, delrec, pool_top;
  uint32_t badop, round, abort;
};

__global__ void __cluster_dims__(kClusterK1, 1, 1) __launch_bounds__(kClusterK1Threads, 1)
    k_batch_cluster(const char* ops, const uint32_t* src, const uint32_t* dst, uint32_t B, uint32_t n, uint32_t cap,
                    EdgeHash h, AdjView out, AdjView in, uint64_t* keys, uint64_t* net, unsigned long long* err,
                    uint32_t* badop, unsigned long long* counts, unsigned long long* num_net,
                    const uint32_t* round_p, uint32_t* reloc_list, const unsigned long long* pool_top,
                    unsigned long long pool_cap, unsigned long long* abort, uint32_t mult,
                    unsigned long long* cursors, uint32_t stride, uint32_t layers,
                    unsigned long long* pool_top_rw, uint32_t* touched_out, uint32_t* touched_in, DelLists dl,
                    bool seed, RecSink S, unsigned long long* seeds_ctr, unsigned long long* scal, uint32_t n_scal,
                    unsigned long long* ctr, uint32_t n_ctr) {
  namespace cg = cooperative_groups;
  pdl_prologue();
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t rank = cluster.block_rank();
  extern __shared__ __align__(16) unsigned char gsm_[];
  __shared__ ClusterK1Shared sh;
  const uint32_t tsz = 2 * cap, tmask = tsz - 1;
  // local layout (identical in every CTA)
  unsigned long long* tkey_l = reinterpret_cast<unsigned long long*>(gsm_);
  uint32_t* tfirst_l = reinterpret_cast<uint32_t*>(gsm_ + 8ull * tsz);
  uint32_t* tcount_l = tfirst_l + tsz;
  uint64_t* bkey = reinterpret_cast<uint64_t*>(gsm_ + 16ull * tsz);
  uint64_t* p_slot = bkey + cap;
  uint64_t* p_off = p_slot + kOpsPerCtaMax;        // [2 x]
  uint32_t* p_pos = reinterpret_cast<uint32_t*>(p_off + 2 * kOpsPerCtaMax);  // [2 x]
  uint32_t* p_lc = p_pos + 2 * kOpsPerCtaMax;      // [4 x]
  uint32_t* slot_of = p_lc + 4 * kOpsPerCtaMax;
  uint32_t* netj = slot_of + kOpsPerCtaMax;
  uint8_t* bop = reinterpret_cast<uint8_t*>(netj + kOpsPerCtaMax);
  // rank 0's table and counters, as seen from this CTA
  unsigned long long* tkey = cluster.map_shared_rank(tkey_l, 0);
  uint32_t* tfirst = cluster.map_shared_rank(tfirst_l, 0);
  uint32_t* tcount = cluster.map_shared_rank(tcount_l, 0);
  ClusterK1Shared* s0 = cluster.map_shared_rank(&sh, 0);
  const uint32_t T = kClusterK1 * kClusterK1Threads;  // 1024 threads
  const uint32_t g = rank * kClusterK1Threads + threadIdx.x;
  if (rank == 0) {
    for (uint32_t q = threadIdx.x; q < n_scal; q += blockDim.x) scal[q] = scal + q == err ? ~0ull : 0ull;
    for (uint32_t q = threadIdx.x; q < n_ctr; q += blockDim.x) ctr[q] = 0ull;
    for (uint32_t q = threadIdx.x; q < tsz; q += blockDim.x) {
      tkey_l[q] = kHashEmpty;
      tfirst_l[q] = 0xFFFFFFFFu;
      tcount_l[q] = 0;
    }
    if (threadIdx.x == 0) {
      sh.err = ~0ull;
      for (int q = 0; q < 6; ++q) sh.cnt[q] = 0;
      sh.num_net = 0;
      sh.delrec = 0;
      sh.badop = 0;
      sh.pool_top = *pool_top;
    }
  }
  if (threadIdx.x == 0) sh.round = *round_p;
  cluster.sync();
  // ---- grouping + every committed-state load of this CTA's ops (op i = g + q T)
  for (uint32_t q = 0, i = g; i < B; ++q, i += T) {
    const uint32_t ls = q * kClusterK1Threads + threadIdx.x;
    netj[ls] = 0xFFFFFFFFu;
    const char o = ops[i];
    const uint32_t s = src[i], d = dst[i];
    if (o != '+' && o != '-') atomicOr(&s0->badop, 1u);
    const uint64_t key = (static_cast<uint64_t>(s) << 32) | d;
    keys[i] = key;
    if (s >= n || d >= n) {
      atomicMin(&s0->err, (static_cast<unsigned long long>(i) << 8) | ERR_RANGE);
      continue;
    }
    const uint32_t ls_ = out.len[s], cs = out.cap[s], ld = in.len[d], cd = in.cap[d];
    const uint64_t os = out.off[s], od = in.off[d];
    uint64_t hi = hash_home(key, h.mask);
    HashSlot hsl = load_slot(h.s + hi);
    unsigned long long hk = hsl.key;
    uint32_t slot = static_cast<uint32_t>(hash_home(key, tmask));
    for (;; slot = (slot + 1) & tmask) {
      const unsigned long long prev = atomicCAS(&tkey[slot], kHashEmpty, static_cast<unsigned long long>(key));
      if (prev == kHashEmpty || prev == key) break;
    }
    slot_of[ls] = slot;
    atomicMin(&tfirst[slot], i);
    atomicAdd(&tcount[slot], 1u);
    uint64_t free_slot = ~0ull;
    bool free_tomb = false;
    for (;;) {
      if (hk == key) break;
      if (hk == kHashTomb && free_slot == ~0ull) {
        free_slot = hi;
        free_tomb = true;
      }
      if (hk == kHashEmpty) {
        if (free_slot == ~0ull) free_slot = hi;
        break;
      }
      hi = (hi + 1) & h.mask;
      hsl = load_slot(h.s + hi);
      hk = hsl.key;
    }
    if (hk == key) {
      p_slot[ls] = hi | kProbePresent;
      p_pos[2 * ls] = hsl.pos_out;
      p_pos[2 * ls + 1] = hsl.pos_in;
    } else {
      p_slot[ls] = free_slot | (free_tomb ? kProbeTomb : 0ull);
    }
    p_lc[4 * ls] = ls_;
    p_lc[4 * ls + 1] = cs;
    p_lc[4 * ls + 2] = ld;
    p_lc[4 * ls + 3] = cd;
    p_off[2 * ls] = os;
    p_off[2 * ls + 1] = od;
  }
  __threadfence();
  cluster.sync();
  // every CTA's copy of the batch (keys, ops) for the in-order validation walk
  for (uint32_t j = threadIdx.x; j < B; j += blockDim.x) {
    const uint64_t key = __ldcg(keys + j);
    const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
    bkey[j] = (s >= n || d >= n) ? kHashEmpty : key;
    bop[j] = static_cast<uint8_t>(ops[j]);
  }
  __syncthreads();
  // ---- validation walk, net ops, relocation election (own ops)
  for (uint32_t q = 0, i = g; i < B; ++q, i += T) {
    const uint32_t ls = q * kClusterK1Threads + threadIdx.x;
    const uint64_t key = bkey[i];
    if (key == kHashEmpty) continue;
    const uint32_t slot = slot_of[ls];
    if (tfirst[slot] != i) continue;  // not the key's first op
    const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
    const bool present = (p_slot[ls] & kProbePresent) != 0;
    bool p = present, ok = true;
    uint32_t left = tcount[slot];
    for (uint32_t j = i; j < B && left; ++j) {
      if (bkey[j] != key) continue;
      --left;
      const bool ins = bop[j] == '+';
      if (ins && p) {
        atomicMin(&s0->err, (static_cast<unsigned long long>(j) << 8) | ERR_DUP);
        ok = false;
        break;
      }
      if (!ins && !p) {
        atomicMin(&s0->err, (static_cast<unsigned long long>(j) << 8) | ERR_MISSING);
        ok = false;
        break;
      }
      p = ins;
    }
    if (!ok || p == present) continue;
    const uint32_t j = static_cast<uint32_t>(atomicAdd(&s0->num_net, 1ull));
    net[j] = p ? key : (key | (1ull << 63));
    netj[ls] = j;
    if (p) {
      atomicAdd(&s0->cnt[0], 1ull);
      const uint32_t os_new = atomicAdd(&out.n_new[s], 1u), od_new = atomicAdd(&in.n_new[d], 1u);
      if (p_lc[4 * ls] + os_new == p_lc[4 * ls + 1]) reloc_list[atomicAdd(&s0->cnt[2], 1ull)] = s;
      if (p_lc[4 * ls + 2] + od_new == p_lc[4 * ls + 3]) reloc_list[atomicAdd(&s0->cnt[2], 1ull)] = (1u << 31) | d;
    } else {
      atomicAdd(&s0->cnt[1], 1ull);
    }
  }
  __threadfence();
  cluster.sync();
  if (rank == 0) {
    const uint32_t n_reloc0 = static_cast<uint32_t>(sh.cnt[2]);
    for (uint32_t w = threadIdx.x; w < n_reloc0; w += blockDim.x) {  // demand of the elected lists (rare)
      const uint32_t code = reloc_list[w], v = code & 0x7FFFFFFFu;
      const AdjView& a = (code >> 31) ? in : out;
      atomicAdd(&sh.cnt[3], static_cast<unsigned long long>(grow_cap(a.len[v] + a.n_new[v])));
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // the gate (round_gate)
      unsigned long long a = 0;
      if (sh.badop) a = 1;
      else if (sh.err != ~0ull) a = 2;
      else if (sh.pool_top + sh.cnt[3] > pool_cap) a = 3;
      sh.abort = static_cast<uint32_t>(a);
      *abort = a;
      for (uint32_t l = 0; l < layers; ++l) cursors[l * stride] = sh.num_net * mult;
    }
  }
  cluster.sync();
  const uint32_t ab = s0->abort;
  const uint32_t n_reloc = static_cast<uint32_t>(s0->cnt[2]);
  if (!ab) {
    const uint32_t wg = g >> 5, nw = T >> 5;
    for (uint32_t w = wg; w < n_reloc; w += nw) relocate_one(reloc_list[w], out, in, pool_top_rw);
    if (n_reloc) {
      __threadfence();
      cluster.sync();
    }
    const uint32_t round = sh.round;
    unsigned long long owned = 0;
    for (uint32_t q = 0, i = g; i < B; ++q, i += T) {
      const uint32_t ls = q * kClusterK1Threads + threadIdx.x;
      const uint32_t j = netj[ls];
      if (j == 0xFFFFFFFFu) continue;
      const uint64_t key = bkey[i], ps = p_slot[ls];
      const bool del = (ps & kProbePresent) != 0;  // a net op flips the committed presence
      const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
      const uint32_t ts = atomicExch(&out.touch[s], round), td = atomicExch(&in.touch[d], round);
      const uint64_t os = n_reloc ? out.off[s] : p_off[2 * ls], od = n_reloc ? in.off[d] : p_off[2 * ls + 1];
      if (!del) {
        const uint32_t po = atomicAdd(&out.len[s], 1u);
        const uint32_t pi = atomicAdd(&in.len[d], 1u);
        const uint64_t fs = ps & ~(kProbePresent | kProbeTomb);
        const unsigned long long expect = (ps & kProbeTomb) ? kHashTomb : kHashEmpty;
        uint64_t slot = fs;
        if (atomicCAS(&h.s[fs].key, expect, static_cast<unsigned long long>(key)) != expect)
          slot = hash_insert(h, key);  // another insert of this round took the slot
        out.ent[os + po] = d | kFlagNew;
        in.ent[od + pi] = s | kFlagNew;
        h.s[slot].pos_out = po;
        h.s[slot].pos_in = pi;
      } else {
        const uint32_t r = static_cast<uint32_t>(atomicAdd(&s0->delrec, 2ull));
        const uint32_t ho = atomicExch(&dl.head_out[s], r), hi = atomicExch(&dl.head_in[d], r + 1);
        atomicAdd(&out.n_del[s], 1u);
        atomicAdd(&in.n_del[d], 1u);
        const uint32_t po = p_pos[2 * ls], pi = p_pos[2 * ls + 1];
        atomicOr(&out.ent[os + po], kFlagDel);
        atomicOr(&in.ent[od + pi], kFlagDel);
        dl.pos[r] = po;
        dl.next[r] = ho;
        dl.pos[r + 1] = pi;
        dl.next[r + 1] = hi;
      }
      if (ts != round) touched_out[atomicAdd(&s0->cnt[4], 1ull)] = s;
      if (td != round) touched_in[atomicAdd(&s0->cnt[5], 1ull)] = d;
      if (seed) {  // seed_edge_events (engine.cpp:101-112) of layer 1
        const uint64_t r = make_record(d, j, del ? EV_SEED_DEL : EV_SEED_ADD);
        owned += S.owns(d);
        for (uint32_t m = 0; m < mult; ++m) S.put(j * mult + m, r);
      }
    }
    if (seed) warp_add(seeds_ctr, owned);
  }
  __threadfence();
  cluster.sync();  // (also keeps rank 0's shared memory alive until every remote access is done)
  if (rank == 0 && threadIdx.x == 0) {  // the round's counters, once
    *err = sh.err;
    *badop = sh.badop;
    for (int q = 0; q < 6; ++q) counts[q] = sh.cnt[q];
    *num_net = sh.num_net;
    *dl.cursor = sh.delrec;
  }
}

// Next-layer Del/Add events (engine.cpp:271-283): warp per (dirty source,
// 256-entry chunk of its out-list) work item; the source reserved its record
// range when it was found dirty (k_collect_dirty), so hubs spread over many warps.
// PAIR = Del(old)+Add(new) of an edge live before and after the round.
// gate (emit_changed_only, else null): the previous layer's change flags; an
// unchanged source's reserved slots are left empty.
__global__ void k_expand_records(const ExpItem* work, const unsigned long long* n_work_p, const uint32_t* dirty,
                                 const uint64_t* exp_base, AdjView out, uint32_t mult, RecSink S,
                                 unsigned long long* events_ctr, const uint32_t* gate, SeedArgs seeds,
                                 const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  put_seeds(seeds);  // this layer's seed records (their own slots ahead of the expansion ranges)
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t n_work = *n_work_p;
  unsigned long long events = 0;
  for (uint64_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n_work; it += warps) {
    const ExpItem item = work[it];
    const uint32_t j = item.j, c = item.c, len = item.len;
    const uint32_t* e = out.ent + item.off;
    const uint64_t base = exp_base[j];
    const bool skip = gate && !gate[j];
    for (uint32_t i = c * kExpandChunk + lane; i < min(len, (c + 1) * kExpandChunk); i += 32) {
      if (skip) {
        for (uint32_t m = 0; m < mult; ++m) S.rec[base + static_cast<uint64_t>(i) * mult + m] = kNoRecord;
        continue;
      }
      const uint32_t x = e[i];
      const uint32_t type = (x & kFlagDel) ? EV_EXP_DEL : ((x & kFlagNew) ? EV_EXP_ADD : EV_EXP_PAIR);
      if (S.owns(x & kNodeMask)) events += type == EV_EXP_PAIR ? 2 : 1;
      const uint64_t r = make_record(x & kNodeMask, j, type);
      for (uint32_t m = 0; m < mult; ++m) S.put(base + static_cast<uint64_t>(i) * mult + m, r);
    }
  }
  warp_add(events_ctr, events * mult);
}

// Layers >= 2: expansion fused with a per-edge pre-classification. For a PAIR
// (edge live before and after the round) from source s to target w, with
// alpha = alpha_prev(w) (the max/min over w's previous in-neighbour messages):
//   * the Del half can reset a position only where old_s[j] == alpha[j] (j < d);
//   * the Add half changes alpha only where new_s[j] beats alpha[j].
// The reduced Del/Add rows of group_and_reduce are elementwise max/min over the
// target's events and select one of their inputs, so a target ALL of whose
// events are PAIRs with neither condition classifies as DeletionNoEffect with
// alpha bitwise unchanged (engine.cpp:45-87) and is not dirty. Only targets with
// a hit, or with any non-PAIR event (seed, tombstone, new entry, SELF), are
// marked RUN_EXACT and go through the grouped classify; the others are counted
// by k_scatter_plan; only relevant PAIRs append a record. One warp per 32
// entries of a dirty source. Rows of > 128 floats first test the target's
// 16-bit alpha bound codes (dev_common.cuh abound_code: half the bytes, twice
// the rows in flight) against per-position thresholds of the source's rows;
// only PAIRs the codes cannot settle read the exact alpha row.
template <bool IsMax, int CPL, int UNR_ = 0, int MINB = 1, bool Codes = true>
__global__ void __launch_bounds__(256, MINB) k_expand_filter(const ExpItem* work, const unsigned long long* n_work_p,
                                                       const uint32_t* dirty, const uint64_t* exp_base, AdjView out,
                                                       RecSink S, const float4* old_slab, RowTable cur,
                                                       const float4* agg, const uint2* abound,
                                                       const uint2* thr_tab, uint32_t V,
                                                       uint32_t d, const float* cmin, const float* astat,
                                                       uint8_t* run_flags, unsigned long long* ctr,
                                                       const uint32_t* gate, SeedArgs seeds,
                                                       const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  put_seeds(seeds);  // this layer's seed records (their own slots ahead of the appended records)
  constexpr uint32_t kNone = 0xFFFFFFFFu;
  // Rows of <= 128 floats (CPL 1) compare alpha directly: at C3 (64-d) the
  // bound stage cost more (threshold setup per task, 35.6 -> 40.2 us/round)
  // than the 128 B per PAIR it saves.
  // (Codes = false: the variant for the scalar-summary path, which reads no
  // code rows; without the code stage's registers it fits 4 CTAs per SM)
  constexpr bool kBounds = Codes && CPL >= 2;
  // PAIR rows in flight per warp (bound codes: 8 B per lane per column)
  constexpr int UNR = UNR_ ? UNR_ : (CPL <= 1 ? 8 : (CPL <= 2 ? 8 : (CPL <= 4 ? 4 : 2)));
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t n_work = *n_work_p;
  unsigned long long events = 0, rows = 0, ents = 0, brows = 0;
  // warp task = 32 entries of a 256-entry work item (short dependent chains)
  constexpr uint32_t kSub = kExpandChunk / 32;
  for (uint64_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_work * kSub; t += warps) {
    const ExpItem item = work[t / kSub];
    const uint32_t sub = static_cast<uint32_t>(t % kSub);
    const uint32_t j = item.j, c = item.c, v = item.v, len = item.len;
    if (gate && !gate[j]) continue;  // emit_changed_only: unchanged source
    const uint32_t i0 = c * kExpandChunk + sub * 32;
    if (i0 >= len) continue;
    const uint32_t* e = out.ent + item.off;
    (void)exp_base;  // records are appended (no reserved range)
    // the lane's out-list entry, issued before the source rows: it depends on
    // the work item only, and loaded after them it added a round trip per task
    const uint32_t end = min(len, i0 + 32);
    const uint32_t xe = i0 + lane < end ? e[i0 + lane] : 0u;
    // thresholds of u = orient(max/min(old, new)) on the alpha bound grid,
    // precomputed per dirty source by K8 (k_write_messages): a PAIR is settled
    // irrelevant when every position's bound code reaches its threshold
    // (positions >= d never block: threshold 0)
    uint32_t thr[CPL][4];
    float4 o[CPL], nw[CPL];  // the source's rows (direct test; the summary's umax)
    if (kBounds && abound) {
      const uint2* trow = thr_tab + static_cast<size_t>(j) * V;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const uint32_t idx = lane + 32u * q;
        const uint2 tv = idx < V ? __ldg(trow + idx) : make_uint2(0, 0);
        thr[q][0] = tv.x & 0xFFFFu;
        thr[q][1] = tv.x >> 16;
        thr[q][2] = tv.y & 0xFFFFu;
        thr[q][3] = tv.y >> 16;
      }
    }
    if (!kBounds || cmin) {
      const float4* orow = old_slab + static_cast<size_t>(j) * V;
      const float4* nrow = cur.row4(v, V);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const uint32_t idx = lane + 32u * q;
        o[q] = idx < V ? __ldg(orow + idx) : make_float4(0, 0, 0, 0);
        nw[q] = idx < V ? __ldg(nrow + idx) : make_float4(0, 0, 0, 0);
      }
    }
    // The source's largest normalised value (combine_kernels.cuh
    // summarise_row): a PAIR whose target's row minimum exceeds it is settled
    // from the target's 4-byte summary.
    float umax = -INFINITY;
    if (cmin) {
      const uint32_t P4 = 4 * V;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const uint32_t idx = lane + 32u * q;
        const float ov[4] = {o[q].x, o[q].y, o[q].z, o[q].w};
        const float nv[4] = {nw[q].x, nw[q].y, nw[q].z, nw[q].w};
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const uint32_t c = 4 * idx + tt;
          if (idx < V && c < d) {
            const float u = IsMax ? fmaxf(ov[tt], nv[tt]) : -fminf(ov[tt], nv[tt]);
            umax = fmaxf(umax, norm_up(u, astat[c], astat[2 * P4 + c]));
          }
        }
      }
      for (int off = 16; off; off >>= 1) umax = fmaxf(umax, __shfl_xor_sync(0xffffffffu, umax, off));
    }
    rows += lane == 0 ? 2 : 0;
    ents += lane == 0 ? end - i0 : 0;
    {
      const uint32_t i = i0 + lane;
      uint32_t w = kNone;
      bool pair = false;
      // Records are appended compactly (no reserved slots): a non-PAIR entry
      // always writes one; a PAIR writes one only if it is relevant to its
      // target's classification (below) — a PAIR whose old and new rows stay
      // strictly below alpha everywhere (max; above for min) changes neither
      // the reset set, nor the coverage test, nor alpha (engine.cpp:45-87).
      bool nonpair = false;
      uint32_t type = EV_EXP_PAIR;
      float cw = 0.0f;  // the target's summary, loaded ahead of the run-map atomics
      if (i < end) {
        const uint32_t x = xe;
        type = (x & kFlagDel) ? EV_EXP_DEL : ((x & kFlagNew) ? EV_EXP_ADD : EV_EXP_PAIR);
        w = x & kNodeMask;
        if (S.owns(w)) {
          pair = type == EV_EXP_PAIR;
          nonpair = !pair;
          if (pair && cmin) cw = __ldg(cmin + w);  // written by an earlier round's K8
          events += pair ? 2 : 1;
          S.touch(w, pair);
          if (nonpair) run_flags[w] = RUN_EXACT;
        }
      }
      {
        const unsigned npm = __ballot_sync(0xffffffffu, nonpair);
        unsigned long long b0 = 0;
        if (lane == 0 && npm) b0 = atomicAdd(S.cursor, static_cast<unsigned long long>(__popc(npm)));
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (nonpair) {
          const uint64_t slot = b0 + __popc(npm & ((1u << lane) - 1u));
          const uint32_t o = atomicAdd(&S.cnt[w], 1u);
          S.rec[slot] = make_record(w, j, type);
          S.ord[slot] = o;
        }
      }
      // settled by the target's summary: no code or alpha row, no record
      if (pair && cmin && umax < cw) pair = false;
      unsigned pm = __ballot_sync(0xffffffffu, pair);
      brows += lane == 0 ? __popc(pm) : 0;
      while (pm) {
        uint32_t tw[UNR];
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          tw[q] = kNone;
          if (pm) {
            const int src = __ffs(pm) - 1;
            pm &= pm - 1;
            tw[q] = __shfl_sync(0xffffffffu, w, src);
          }
        }
        // stage 1: the 16-bit alpha bound codes (half the bytes of an alpha
        // row, so twice the rows in flight); a PAIR whose thresholds are all
        // reached is settled irrelevant without reading alpha
        uint32_t maybe = 0;  // bit q: pair q needs the exact alpha row
        if (!kBounds || !abound) {  // (no code table when the summary settles the PAIRs)
#pragma unroll
          for (int q = 0; q < UNR; ++q)
            if (tw[q] != kNone) maybe |= 1u << q;
        } else {
          uint2 b[UNR][CPL];
#pragma unroll
          for (int q = 0; q < UNR; ++q) {
            const uint2* brow = abound + static_cast<size_t>(tw[q]) * V;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const uint32_t idx = lane + 32u * k;
              b[q][k] = (tw[q] != kNone && idx < V) ? brow[idx] : make_uint2(0, 0);
            }
          }
#pragma unroll
          for (int q = 0; q < UNR; ++q) {
            bool m = false;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const uint32_t cv[4] = {b[q][k].x & 0xFFFFu, b[q][k].x >> 16, b[q][k].y & 0xFFFFu, b[q][k].y >> 16};
#pragma unroll
              for (int t = 0; t < 4; ++t)
                if (cv[t] < thr[k][t]) m = true;  // thr = 0 past d and past V
            }
            if (tw[q] != kNone && __any_sync(0xffffffffu, m)) maybe |= 1u << q;
          }
        }
        rows += lane == 0 ? __popc(maybe) : 0;
        uint32_t mytw = kNone;
#pragma unroll
        for (int q = 0; q < UNR; ++q)
          if (lane == static_cast<uint32_t>(q)) mytw = tw[q];
        // stage 2: exact test (old/new rows re-read, L1-resident) on the
        // undecided PAIRs, G alpha rows at a time
        // (the summary variant, Codes = false, reaches this stage for a few % of
        // the PAIRs: 2 alpha rows at a time keep it within 64 registers)
        constexpr int G = kBounds ? (CPL >= 4 ? 1 : 2) : (Codes ? UNR : 2);
        uint32_t hits = 0, ties = 0;  // bit q: pair q hit / tied alpha
        for (uint32_t mb = maybe; mb;) {  // warp-uniform
          int qs[G];
#pragma unroll
          for (int h = 0; h < G; ++h) {
            qs[h] = -1;
            if (mb) {
              qs[h] = __ffs(mb) - 1;
              mb &= mb - 1;
            }
          }
          const float4* orow = old_slab + static_cast<size_t>(j) * V;
          const float4* nrow = cur.row4(v, V);
          float4 oo[CPL], nn[CPL], a[G][CPL];
          uint32_t tt[G];
#pragma unroll
          for (int h = 0; h < G; ++h) {
            const uint32_t tq = __shfl_sync(0xffffffffu, mytw, qs[h] < 0 ? 0 : qs[h]);
            tt[h] = qs[h] < 0 ? kNone : tq;
          }
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const uint32_t idx = lane + 32u * k;
            if (kBounds && !cmin) {
              oo[k] = idx < V ? __ldg(orow + idx) : make_float4(0, 0, 0, 0);
              nn[k] = idx < V ? __ldg(nrow + idx) : make_float4(0, 0, 0, 0);
            } else {
              oo[k] = o[k];
              nn[k] = nw[k];
            }
#pragma unroll
            for (int h = 0; h < G; ++h)
              a[h][k] = (tt[h] != kNone && idx < V) ? agg[static_cast<size_t>(tt[h]) * V + idx]
                                                     : make_float4(0, 0, 0, 0);
          }
#pragma unroll
          for (int h = 0; h < G; ++h) {
            if (tt[h] == kNone) continue;  // warp-uniform
            bool hit = false, tie = false;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const uint32_t idx = lane + 32u * k;
              if (idx < V) {
                const float av[4] = {a[h][k].x, a[h][k].y, a[h][k].z, a[h][k].w};
                const float ov[4] = {oo[k].x, oo[k].y, oo[k].z, oo[k].w};
                const float nv[4] = {nn[k].x, nn[k].y, nn[k].z, nn[k].w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  if (4 * idx + t < d && ov[t] == av[t]) hit = true;
                  if (IsMax ? nv[t] > av[t] : nv[t] < av[t]) hit = true;
                  if (4 * idx + t < d && nv[t] == av[t]) tie = true;  // may cover another source's reset
                }
              }
            }
            if (__any_sync(0xffffffffu, hit)) hits |= 1u << qs[h];
            if (__any_sync(0xffffffffu, tie)) ties |= 1u << qs[h];
          }
        }
        // lane q settles pair q: flags, and the records of relevant PAIRs
        // (hit or tie) appended with one cursor atomic per warp
        const bool myhit = lane < UNR && ((hits >> lane) & 1u), myrel = lane < UNR && (((hits | ties) >> lane) & 1u);
        if (mytw != kNone && lane < UNR && myhit) run_flags[mytw] = RUN_EXACT;
        const unsigned relm = __ballot_sync(0xffffffffu, mytw != kNone && myrel);
        if (relm) {
          unsigned long long b1 = 0;
          if (lane == 0) b1 = atomicAdd(S.cursor, static_cast<unsigned long long>(__popc(relm)));
          b1 = __shfl_sync(0xffffffffu, b1, 0);
          if ((relm >> lane) & 1u) {
            const uint64_t slot = b1 + __popc(relm & ((1u << lane) - 1u));
            const uint32_t o2 = atomicAdd(&S.cnt[mytw], 1u);
            S.rec[slot] = make_record(mytw, j, EV_EXP_PAIR);
            S.ord[slot] = o2;
          }
        }
      }
    }
  }
  warp_add(&ctr[C_EVENTS], events);
  warp_add(&ctr[C_FILTER_ROWS], rows);
  warp_add(&ctr[C_FILTER_ENTS], ents);
  warp_add(&ctr[C_FILTER_BROWS], brows);
}

// user_propagate (engine.cpp:285-288): the node's own refreshed message as a
// SELF record, when the model has user ops and m_{l+1} changed bitwise.
__global__ void k_self_records(const uint32_t* dirty, const uint32_t* changed, const unsigned long long* n_dirty_p,
                               RecSink S, const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  const uint64_t n = *n_dirty_p;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (!changed[j]) continue;
    S.put(atomicAdd(S.cursor, 1ull), make_record(dirty[j], 0, EV_SELF));
  }
}

constexpr uint32_t kSeg = 32;  // records per classify work item (one per lane)

struct ClassifyArgs {
  const uint32_t* tmap;     // pre-filtered layers: RecSink::touched (bit 1 = the target had a PAIR), else null
  const uint64_t* rec;      // records grouped by target
  const uint32_t* runs;     // run r -> target node
  const uint32_t* off;      // [N] first record of each target's group
  const uint32_t* cnt;      // [N] group sizes
  const unsigned long long* num_runs;
  const unsigned long long* abort;
  MsgView msg;
  float4* agg;              // a_l table (pitch V float4)
  uint32_t d;               // logical dim of layer l
  const uint32_t* in_len;   // in-adjacency entry counts (incl. flagged)
  const uint32_t* in_new;
  uint8_t* run_flags;
  // segments {target, first record, end record, run | multi << 31} of <= kSeg
  // records; multi-segment runs merge their partial reductions through
  // scratch rows (2 x P ints: del, add)
  uint4* seg;
  unsigned long long* n_seg;
  int* cls_scratch;
  uint32_t* cls_slot;
  uint32_t* cls_remaining;
  uint32_t* cls_flags;      // bit0 del, bit1 add, bit2 self
  unsigned long long* n_cls_scratch;
  unsigned long long* seg_next;  // dynamic segment cursor
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
  // sparse exposed-reset recompute (null sp_target = always dense)
  uint32_t* sp_target;      // [slot] target node
  uint32_t* sp_n;           // [slot] uncovered reset positions (<= kSparseDims)
  uint32_t* sp_dims;        // [slot][kSparseDims] positions
  float* sp_aold;           // [slot][kSparseDims] alpha_prev at those positions
  int* sp_acc;              // [slot][kSparseDims] order-preserving max/min accumulators
  uint32_t* sp_live;        // [slot] live in-neighbours seen
  uint32_t* sp_changed;     // [slot] alpha changed outside the recomputed positions
  unsigned long long* n_sparse;
  uint64_t* swork;          // (slot << 32 | chunk) items of kSparseChunk in-list entries
  unsigned long long* n_swork;
  uint32_t* sp_remaining;  // sparse chunks still to merge (the last one finalises)
};

// Counting-sort scatter fused with the segment planner: the thread holding a
// group's first record (ordinal 0) cuts that group into kSeg-record segments
// (block-aggregated allocation: one global atomic per CTA) and, for groups
// longer than one segment, prepares the merge slot (identity scratch rows,
// completion counter). Per-target state is indexed by node id.
// Group offsets of the counting sort: each target that will be scattered gets
// a contiguous slice of the sorted record array, allocated with one
// block-aggregated atomic per block over the run list (any order of the
// groups is as good as ascending: classification is order-invariant and the
// slices only need to be disjoint). Replaces an exclusive scan over all N
// counters. Filtered layers allocate RUN_EXACT targets only.
__global__ void __launch_bounds__(256) k_alloc_runs(const uint32_t* runs, const unsigned long long* num_runs_p,
                                                    const uint32_t* cnt, const uint8_t* run_flags, bool filtered,
                                                    uint32_t* off, unsigned long long* cursor,
                                                    unsigned long long* ctr, const unsigned long long* abort) {
  pdl_prologue();
  using BlockScan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ unsigned long long base;
  if (*abort) return;
  const uint64_t n = *num_runs_p;
  unsigned long long skipped = 0;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x); i0 < n;
       i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t w = 0, c = 0;
    if (i < n) {
      w = runs[i];
      const uint32_t cw = cnt[w];  // issued beside the flag load (not after it)
      if (!filtered || (run_flags[w] & RUN_EXACT)) c = cw;
      else ++skipped;  // a pre-filtered target: grouped, DeletionNoEffect, alpha read
    }
    uint32_t o = 0, total = 0;
    BlockScan(tmp).ExclusiveSum(c, o, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(cursor, static_cast<unsigned long long>(total)) : 0;
    __syncthreads();
    if (c) off[w] = static_cast<uint32_t>(base) + o;
    __syncthreads();
  }
  if (filtered) {
    for (int o2 = 16; o2; o2 >>= 1) skipped += __shfl_xor_sync(0xffffffffu, skipped, o2);
    if ((threadIdx.x & 31) == 0 && skipped) {
      atomicAdd(&ctr[C_TARGETS], skipped);
      atomicAdd(&ctr[C_DEL_NO_EFFECT], skipped);
      atomicAdd(&ctr[C_FETCH_OTHER], skipped);  // read_prev(l, v, Aggregated), engine.cpp:233
    }
  }
}

// With `filtered` (layers >= 2 of a pre-filtered round, k_expand_filter) the
// records of targets without RUN_EXACT are dropped here and each such target is
// counted once as a grouped DeletionNoEffect target with its alpha read.
template <bool IsMax>
__global__ void __launch_bounds__(256) k_scatter_plan(const uint64_t* rec_u, const uint32_t* ord,
                                                      const unsigned long long* n_p, ClassifyArgs A,
                                                      uint64_t* rec_sorted, bool filtered) {
  pdl_prologue();
  using BlockScan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ unsigned long long base;
  if (*A.abort) return;
  const uint64_t n = *n_p;
  const uint32_t P = A.msg.V * 4;
  unsigned long long skipped = 0;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x); i0 < n;
       i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t nseg = 0, w = 0, rb = 0, re = 0;
    const uint64_t r = i < n ? rec_u[i] : kNoRecord;
    if (r != kNoRecord) {
      w = static_cast<uint32_t>(r >> 32);
      const uint32_t o = ord[i];
      // the group's offset and size are loaded beside the flag (one round trip)
      const uint32_t ow = A.off[w], cw = o == 0 ? A.cnt[w] : 0u;
      if (filtered && !(A.run_flags[w] & RUN_EXACT)) {
        // counted by k_alloc_runs (a filtered target may have no records)
      } else {
        rb = ow;
        rec_sorted[rb + o] = r;
        if (o == 0) {
          re = rb + cw;
          nseg = (re - rb + kSeg - 1) / kSeg;
        }
      }
    }
    uint32_t off = 0, total = 0;
    BlockScan(tmp).ExclusiveSum(nseg, off, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(A.n_seg, static_cast<unsigned long long>(total)) : 0;
    __syncthreads();
    for (uint32_t k = 0; k < nseg; ++k)
      A.seg[base + off + k] = make_uint4(w, rb + k * kSeg, min(re, rb + (k + 1) * kSeg), nseg > 1 ? 0x80000000u : 0u);
    if (nseg > 1) {
      const uint32_t slot = static_cast<uint32_t>(atomicAdd(A.n_cls_scratch, 1ull));
      A.cls_slot[w] = slot;
      A.cls_remaining[w] = nseg;
      A.cls_flags[w] = 0;
      int* row = A.cls_scratch + static_cast<size_t>(slot) * 2 * P;
      for (uint32_t q = 0; q < 2 * P; ++q) row[q] = IsMax ? INT_MIN : INT_MAX;
    }
    __syncthreads();
  }
  (void)skipped;
}

// Classify one grouped target from its reduced Del/Add rows (engine.cpp:45-87,
// 229-258): first-neighbour rule, reset positions, covered test, incremental
// update or exposed-reset hand-off to K4, bitwise change test, alpha write.
template <bool IsMax, int CPL>
__device__ __forceinline__ void classify_target(const ClassifyArgs& A, uint32_t r, uint32_t w, float4 (&del)[CPL],
                                                float4 (&add)[CPL], const float4 (&a)[CPL], bool has_del,
                                                bool has_add, bool has_self, uint32_t in_len, uint32_t in_new,
                                                unsigned long long* sc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t V = A.msg.V;
  const bool grp = has_del || has_add;
  uint8_t flags = (grp ? RUN_GRP : 0) | (has_self ? RUN_SELF : 0);
  int kind = -1;  // 0 NoDeletion 1 DeletionNoEffect 2 Covered 3 Exposed
  if (grp) {
    float4* arow = A.agg + static_cast<size_t>(w) * V;
    float4 anew[CPL];
    const uint32_t prev_indeg = in_len - in_new;
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
      // Exposed reset. Only the uncovered reset positions (alpha_prev == Del
      // and no Add reaching it) need the full neighbourhood: every other
      // position's new value is sel(alpha_prev, Add) — the removed
      // contributions were strictly below alpha there and max/min selects an
      // input exactly — so when there are few, recompute just those positions.
      uint32_t n_r = 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t idx = lane + 32u * c;
        const float av[4] = {a[c].x, a[c].y, a[c].z, a[c].w};
        const float dv[4] = {del[c].x, del[c].y, del[c].z, del[c].w};
        const float pv[4] = {add[c].x, add[c].y, add[c].z, add[c].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool bit = idx < V && 4 * idx + q < A.d && av[q] == dv[q] &&
                           !(has_add && (IsMax ? pv[q] >= dv[q] : pv[q] <= dv[q]));
          n_r += __popc(__ballot_sync(0xffffffffu, bit));
        }
      }
      if (A.sp_target && n_r <= kSparseDims) {
        bool changed_base = false;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t idx = lane + 32u * c;
          const float4 an = has_add ? sel4<IsMax>(a[c], add[c]) : a[c];
          anew[c] = an;
          const float av[4] = {a[c].x, a[c].y, a[c].z, a[c].w};
          const float dv[4] = {del[c].x, del[c].y, del[c].z, del[c].w};
          const float pv[4] = {add[c].x, add[c].y, add[c].z, add[c].w};
          const float nv[4] = {an.x, an.y, an.z, an.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool bit = idx < V && 4 * idx + q < A.d && av[q] == dv[q] &&
                             !(has_add && (IsMax ? pv[q] >= dv[q] : pv[q] <= dv[q]));
            if (idx < V && !bit && __float_as_uint(nv[q]) != __float_as_uint(av[q])) changed_base = true;
          }
        }
        changed_base = __any_sync(0xffffffffu, changed_base);
        uint32_t sp = 0;
        if (lane == 0) {
          sp = static_cast<uint32_t>(atomicAdd(A.n_sparse, 1ull));
          A.sp_target[sp] = r;
          A.sp_n[sp] = n_r;
          A.sp_live[sp] = 0;
          A.sp_remaining[sp] = in_len == 0 ? 1u : (in_len + kSparseChunk - 1) / kSparseChunk;
          A.sp_changed[sp] = changed_base;
          const uint32_t nch = in_len == 0 ? 1u : (in_len + kSparseChunk - 1) / kSparseChunk;
          const unsigned long long base = atomicAdd(A.n_swork, static_cast<unsigned long long>(nch));
          for (uint32_t c = 0; c < nch; ++c) A.swork[base + c] = (static_cast<uint64_t>(sp) << 32) | c;
        }
        sp = __shfl_sync(0xffffffffu, sp, 0);
        uint32_t pos = 0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t idx = lane + 32u * c;
          const float av[4] = {a[c].x, a[c].y, a[c].z, a[c].w};
          const float dv[4] = {del[c].x, del[c].y, del[c].z, del[c].w};
          const float pv[4] = {add[c].x, add[c].y, add[c].z, add[c].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool bit = idx < V && 4 * idx + q < A.d && av[q] == dv[q] &&
                             !(has_add && (IsMax ? pv[q] >= dv[q] : pv[q] <= dv[q]));
            const unsigned m = __ballot_sync(0xffffffffu, bit);
            if (bit) {
              const uint32_t k = pos + __popc(m & ((1u << lane) - 1u));
              A.sp_dims[sp * kSparseDims + k] = 4 * idx + q;
              A.sp_aold[sp * kSparseDims + k] = av[q];
              A.sp_acc[sp * kSparseDims + k] = IsMax ? INT_MIN : INT_MAX;
            }
            pos += __popc(m);
          }
        }
        if (changed_base) {
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const uint32_t idx = lane + 32u * c;
            if (idx < V) arow[idx] = anew[c];
          }
        }
      } else {
        uint32_t nch = 0, si = 0;
        if (lane == 0) {
          const uint32_t raw = in_len;
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
  pdl_prologue();
  __shared__ unsigned long long sc[C_NUM];
  if (*A.abort) return;
  for (int i = threadIdx.x; i < C_NUM; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t V = A.msg.V;
  const uint64_t n_seg = *A.n_seg;
  const float ident = IsMax ? -INFINITY : INFINITY;
  WarpQueue q;
  q.init(A.seg_next, n_seg, 4);
  (void)warps;
  for (uint64_t sidx; q.next(sidx);) {
    const uint4 sg = A.seg[sidx];
    const uint32_t w = sg.x, b = sg.y, e = sg.z, r = w;  // per-target state is indexed by node id
    const uint32_t nseg = (sg.w >> 31) ? 2u : 1u;  // 1 = the whole run
    const uint32_t in_len = A.in_len[w], in_new = A.in_new[w];  // issued early, used by classify_target
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
    // each lane resolves one record's rows (parallel, not a chain) as 32-bit
    // row ids: bit 31 set = pre-image slab row, clear = current-table row
    const uint32_t n_here = e - b;
    constexpr uint32_t kNone = 0xFFFFFFFFu, kOld = 0x80000000u;
    uint32_t id_add = kNone, id_del = kNone;
    bool self = false;
    if (lane < n_here) {
      const uint64_t rr = A.rec[b + lane];
      const uint32_t type = static_cast<uint32_t>(rr) & 7u, ix = static_cast<uint32_t>(rr >> 3) & 0x1FFFFFFFu;
      if (type == EV_SELF) {
        self = true;
      } else if (type <= EV_SEED_DEL) {
        const uint32_t s = static_cast<uint32_t>(A.msg.net[ix] >> 32) & kNodeMask;
        if (type == EV_SEED_ADD) {
          id_add = s;
        } else {
          const bool stamped = A.msg.stamp && A.msg.stamp[s] == *A.msg.round;
          id_del = stamped ? (kOld | A.msg.slot[s]) : s;
        }
      } else {
        if (type != EV_EXP_DEL) id_add = A.msg.dprev[ix];
        if (type != EV_EXP_ADD) id_del = kOld | ix;
      }
    }
    const bool has_self = __any_sync(0xffffffffu, self);
    const unsigned m_add = __ballot_sync(0xffffffffu, id_add != kNone);
    const unsigned m_del = __ballot_sync(0xffffffffu, id_del != kNone);
    const bool has_add = m_add != 0;
    // a dropped (hit- and tie-free) PAIR still contributes a Del event whose row
    // lies strictly inside alpha: it only makes the target grouped
    const bool has_del = m_del != 0 || (A.tmap && ((A.tmap[w >> 4] >> (2u * (w & 15u) + 1u)) & 1u));
    const uint32_t rows_read = __popc(m_add) + __popc(m_del);
    constexpr int UNR = CPL <= 1 ? 4 : (CPL <= 4 ? 2 : 1);
    unsigned ma = m_add, md = m_del;
    while (ma | md) {
      uint32_t rid[UNR];
      bool is_del[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        rid[q] = kNone;
        is_del[q] = false;
        if (ma) {
          const int src = __ffs(ma) - 1;
          ma &= ma - 1;
          rid[q] = __shfl_sync(0xffffffffu, id_add, src);
        } else if (md) {
          const int src = __ffs(md) - 1;
          md &= md - 1;
          rid[q] = __shfl_sync(0xffffffffu, id_del, src);
          is_del[q] = true;
        }
      }
      float4 v[UNR][CPL];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const float4* row = (rid[q] & kOld) ? A.msg.old + static_cast<size_t>(rid[q] & ~kOld) * V
                                            : A.msg.cur.row4(rid[q], V);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t idx = lane + 32u * c;
          v[q][c] = (rid[q] != kNone && idx < V) ? __ldg(row + idx) : make_float4(ident, ident, ident, ident);
        }
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
      classify_target<IsMax, CPL>(A, r, w, del, add, a, has_del, has_add, has_self, in_len, in_new, sc);
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
    classify_target<IsMax, CPL>(A, r, w, del, add, a, f & 1u, f & 2u, f & 4u, in_len, in_new, sc);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C_NUM; i += blockDim.x)
    if (sc[i]) atomicAdd(&A.ctr[i], sc[i]);
}

// K5: dirty list of this layer (unordered; readout sorts), with the
// dirty-dependent counted reads (user-only alpha read, engine.cpp:262-265;
// self-message reads, 125-128; read_prev(l+1), 272), and — when a next layer
// exists — the record range and expansion work items each dirty source needs.
__global__ void k_collect_dirty(const uint32_t* runs, const unsigned long long* num_runs_p, uint8_t* run_flags,
                                uint32_t* cnt, uint32_t* touched, bool reserve_next,
                                uint32_t* dirty, unsigned long long* n_dirty, AdjView out, bool has_next,
                                uint32_t mult, uint64_t* exp_base, ExpItem* exp_work, unsigned long long* exp_n,
                                unsigned long long* next_cursor, unsigned long long* ctr, uint32_t user_ops,
                                bool layer1, bool plan, uint32_t* changed, const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  const uint64_t num_runs = *num_runs_p;
  unsigned long long l1 = 0, other = 0;
  const uint32_t lane = threadIdx.x & 31;
  const bool planning = has_next && plan;
  // Warp-aligned grid stride (the whole warp iterates together), so the
  // dirty slots, record ranges and expansion items are allocated with one
  // atomic per warp and counter (a warp-wide scan gives each lane its
  // offset); the next layer's list length and offset are loaded beside the
  // run flags instead of after the slot allocation.
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t r0 = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) & ~31ull; r0 < num_runs;
       r0 += stride) {
    const uint64_t r = r0 + lane;
    const bool in = r < num_runs;
    uint32_t v = 0, len = 0;
    uint64_t off = 0;
    uint8_t f = 0;
    if (in) {
      v = runs[r];
      if (planning) {
        len = out.len[v];
        off = out.off[v];
      }
      f = run_flags[v];
      if (f) run_flags[v] = 0;  // per-node flags and group counters are cleared here for the next layer
      cnt[v] = 0;
      if (touched) atomicAnd(&touched[v >> 4], ~(3u << (2u * (v & 15u))));
    }
    const bool dirty_v = in && (f & RUN_DIRTY);
    const uint32_t dmask = __ballot_sync(0xffffffffu, dirty_v);
    if (!dmask) continue;
    const uint32_t nch = dirty_v && planning ? (len + kExpandChunk - 1) / kExpandChunk : 0u;
    const unsigned long long span = dirty_v && planning && reserve_next ? static_cast<unsigned long long>(len) * mult : 0ull;
    // inclusive warp scans of the expansion items and record ranges
    uint32_t nch_inc = nch;
    unsigned long long span_inc = span;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, nch_inc, o);
      const unsigned long long b = __shfl_up_sync(0xffffffffu, span_inc, o);
      if (lane >= static_cast<uint32_t>(o)) {
        nch_inc += a;
        span_inc += b;
      }
    }
    const uint32_t nch_tot = __shfl_sync(0xffffffffu, nch_inc, 31);
    const unsigned long long span_tot = __shfl_sync(0xffffffffu, span_inc, 31);
    unsigned long long jb = 0, wb = 0, eb = 0;
    if (lane == 0) {  // independent atomics: issued back to back
      jb = atomicAdd(n_dirty, static_cast<unsigned long long>(__popc(dmask)));
      if (nch_tot) wb = atomicAdd(exp_n, static_cast<unsigned long long>(nch_tot));
      if (span_tot) eb = atomicAdd(next_cursor, span_tot);
    }
    jb = __shfl_sync(0xffffffffu, jb, 0);
    wb = __shfl_sync(0xffffffffu, wb, 0);
    eb = __shfl_sync(0xffffffffu, eb, 0);
    if (!dirty_v) continue;
    const uint32_t j = static_cast<uint32_t>(jb) + __popc(dmask & ((1u << lane) - 1u));
    dirty[j] = v;
    if (changed) changed[j] = 0;  // ORed by the fused combination write-back
    if (!(f & RUN_GRP)) other += 1;
    if (!(f & RUN_SELF)) (layer1 ? l1 : other) += user_ops;
    if (has_next) other += 1;
    if (planning) {
      // record range of the next layer's expansion (a pre-filtered next layer
      // appends its records compactly instead)
      if (reserve_next) exp_base[j] = eb + span_inc - span;
      const unsigned long long w0 = wb + nch_inc - nch;
      for (uint32_t c = 0; c < nch; ++c) exp_work[w0 + c] = ExpItem{off, j, v, len, c, {0, 0}};
    }
  }
  for (int o = 16; o; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    other += __shfl_xor_sync(0xffffffffu, other, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (l1) atomicAdd(&ctr[C_FETCH_L1MSG], l1);
    if (other) atomicAdd(&ctr[C_FETCH_OTHER], other);
  }
}

}  // namespace sgb

namespace sgb {

// Expansion planning for a dirty list assembled from every shard (sharded
// rounds; the unsharded path plans inside k_collect_dirty): record range and
// work items of each dirty source's next-layer expansion (engine.cpp:271-283).
__global__ void k_plan_expand(const uint32_t* dirty, const unsigned long long* n_dirty_p, AdjView out, uint32_t mult,
                              uint64_t* exp_base, ExpItem* exp_work, unsigned long long* exp_n,
                              unsigned long long* next_cursor, bool reserve_next) {
  pdl_prologue();
  const uint64_t n = *n_dirty_p;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = dirty[j];
    const uint32_t len = out.len[v];
    if (reserve_next) exp_base[j] = atomicAdd(next_cursor, static_cast<unsigned long long>(len) * mult);
    put_exp_items(exp_work, exp_n, static_cast<uint32_t>(j), v, len, out.off[v]);
  }
}

// ---- per-layer shard exchange (owner-computes, partitioned tables) ----------
// A shard's boundary record for one dirty node v of layer l: {v, changed} and
// the node's PREVIOUS m_{l+1} row (its pre-image, pitch P floats), 16 + 4P
// bytes. The new row needs no copy: the owner wrote it into its own partition
// of m_{l+1}, which every shard reads through peer memory (RowTable). Every
// shard imports every record, so the pre-image slab, the stamps/slots (the
// reference's read_prev, checkpoint.cpp:52-57) and the dirty list of layer l
// are identical on all shards before layer l+1 expands its events.
__host__ __device__ inline size_t shard_row_bytes(uint32_t P) { return 16 + 4ull * P; }

// Warp copy of one V-float4 row, 4 columns of loads per lane issued before the
// stores (one L2 / peer round trip per 128 float4 instead of one per 32).
__device__ __forceinline__ void warp_copy_row(float4* d0, const float4* s0, uint32_t V, uint32_t lane) {
  constexpr int U = 4;
  for (uint32_t c0 = lane; c0 < V; c0 += 32 * U) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t c = c0 + 32u * u;
      if (c < V) a[u] = s0[c];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t c = c0 + 32u * u;
      if (c < V) d0[c] = a[u];
    }
  }
}

__global__ void k_pack_rows(const uint32_t* dirty, const unsigned long long* n_p, const float4* old_slab,
                            const uint32_t* changed, uint32_t P, uint8_t* out) {
  pdl_prologue();
  const uint32_t lane = threadIdx.x & 31, V = P / 4;
  const uint64_t n = *n_p;
  const size_t rb = shard_row_bytes(P);
  for (uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; w < n;
       w += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    uint8_t* rec = out + w * rb;
    if (lane == 0) *reinterpret_cast<uint4*>(rec) = make_uint4(dirty[w], changed[w], 0, 0);
    warp_copy_row(reinterpret_cast<float4*>(rec + 16), old_slab + w * V, V, lane);
  }
}

// Every shard's records in one launch, read in place from the peers' pack
// buffers through a device table the host fills after the count exchange:
// tab[3r] = records of shard r (device address, peer memory), tab[3r+1] = their
// count, tab[3r+2] = first global dirty position; tab[3w] = total, stored as
// the layer's dirty count. Graph-capturable (no per-round kernel arguments).
constexpr int kMaxShards = kMaxPeers;
__global__ void k_import_table(const unsigned long long* tab, uint32_t world, uint32_t P, uint32_t* dirty,
                               uint32_t* changed, float4* old_slab, uint32_t* stamp, uint32_t* slot,
                               const uint32_t* round_p, unsigned long long* n_dirty) {
  pdl_prologue();
  const uint32_t lane = threadIdx.x & 31, V = P / 4;
  const size_t rb = shard_row_bytes(P);
  const uint64_t total = tab[3 * world];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_dirty = total;
  for (uint64_t g = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; g < total;
       g += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    uint32_t r = 0;
    while (r + 1 < world && g >= tab[3 * (r + 1) + 2]) ++r;
    const uint64_t i = g - tab[3 * r + 2];
    const uint8_t* rec = reinterpret_cast<const uint8_t*>(tab[3 * r]) + i * rb;
    const uint4 h = *reinterpret_cast<const uint4*>(rec);
    warp_copy_row(old_slab + g * V, reinterpret_cast<const float4*>(rec + 16), V, lane);
    if (lane == 0) {
      dirty[g] = h.x;
      changed[g] = h.y;
      stamp[h.x] = *round_p;
      slot[h.x] = static_cast<uint32_t>(g);
    }
  }
}

}  // namespace sgb
