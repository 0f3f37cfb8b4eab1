// K1 — batched edge update on the device-resident dynamic graph.
//
// Replaces DynamicGraph::apply_delta / net_edge_delta / commit
// (proj/src/core/graph.cpp:52-131): the batch is sorted by (src,dst) with its
// sequence index (stable), each key segment is walked in batch order against
// the committed presence of the edge to find the first failing op (the
// reference's overlay validation), the net effect per key is extracted, and
// only net changes touch the adjacency: NEW entries appended into per-vertex
// slabs (relocated into the slab pool when full), DEL tombstones set in place.
// commit compacts the touched lists.
#pragma once

#include "dev_common.cuh"

namespace sgb {

enum : unsigned long long { ERR_RANGE = 1, ERR_DUP = 2, ERR_MISSING = 3 };
enum : uint8_t { NET_NONE = 0, NET_INSERT = 1, NET_DELETE = 2 };

// One direction of the adjacency. `ent` is the slab pool base.
struct AdjView {
  uint64_t* off;
  uint32_t* len;        // entries in use, including this round's DEL/NEW ones
  uint32_t* cap;
  uint32_t* ent;
  uint32_t* n_new;      // NEW entries this round
  uint32_t* n_del;      // DEL entries this round
  uint32_t* touch;      // round stamp of the last modification (commit list)
  uint32_t* reloc;      // round stamp of the last relocation election
};

__device__ __forceinline__ uint32_t grow_cap(uint32_t need) {
  uint32_t c = need + (need >> 1) + 8;
  return (c + 7u) & ~7u;
}

__global__ void k_batch_keys(const char* ops, const uint32_t* src, const uint32_t* dst, uint32_t B, uint32_t n,
                             uint64_t* keys, uint32_t* vals, unsigned long long* err, uint32_t* badop) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  char o = ops[i];
  if (o != '+' && o != '-') atomicOr(badop, 1u);
  uint32_t s = src[i], d = dst[i];
  keys[i] = (static_cast<uint64_t>(s) << 32) | d;
  vals[i] = i;
  if (s >= n || d >= n) atomicMin(err, (static_cast<unsigned long long>(i) << 8) | ERR_RANGE);
}

// Warp-cooperative membership test of `target` in the committed list of v.
__device__ bool warp_list_has(const AdjView& a, uint32_t v, uint32_t target) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t* e = a.ent + a.off[v];
  const uint32_t len = a.len[v];
  for (uint32_t i = 0; i < len; i += 32) {
    bool hit = false;
    if (i + lane < len) {
      uint32_t x = e[i + lane];
      hit = (x & kNodeMask) == target && !(x & (kFlagDel | kFlagNew));
    }
    if (__any_sync(0xffffffffu, hit)) return true;
  }
  return false;
}

// Warp per sorted position; segment heads walk their ops in batch order.
__global__ void k_validate(const uint64_t* skeys, const uint32_t* svals, const char* ops, uint32_t B, uint32_t n,
                           AdjView out, AdjView in, uint8_t* seg_op, uint64_t* net_cand,
                           unsigned long long* err, unsigned long long* counts) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= B) return;
  const uint64_t key = skeys[w];
  const bool head = (w == 0) || skeys[w - 1] != key;
  const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
  if (!head || s >= n || d >= n) {
    if (lane == 0) seg_op[w] = NET_NONE;
    return;
  }
  // presence in the committed graph: scan the shorter of out(s) / in(d)
  const bool present =
      out.len[s] <= in.len[d] ? warp_list_has(out, s, d) : warp_list_has(in, d, s);
  if (lane == 0) {
    bool p = present, ok = true;
    for (uint32_t j = w; j < B && skeys[j] == key; ++j) {
      const uint32_t seq = svals[j];
      const bool ins = ops[seq] == '+';
      if (ins && p) {
        atomicMin(err, (static_cast<unsigned long long>(seq) << 8) | ERR_DUP);
        ok = false;
        break;
      }
      if (!ins && !p) {
        atomicMin(err, (static_cast<unsigned long long>(seq) << 8) | ERR_MISSING);
        ok = false;
        break;
      }
      p = ins;
    }
    uint8_t net = NET_NONE;
    if (ok && p != present) net = p ? NET_INSERT : NET_DELETE;
    seg_op[w] = net;
    net_cand[w] = net == NET_DELETE ? (key | (1ull << 63)) : key;
    if (net == NET_INSERT) {
      atomicAdd(&counts[0], 1ull);
      atomicAdd(&out.n_new[s], 1u);
      atomicAdd(&in.n_new[d], 1u);
    } else if (net == NET_DELETE) {
      atomicAdd(&counts[1], 1ull);
    }
  }
}

// Elects vertices whose slab cannot take this round's appends; sums the pool
// demand so the host can grow the pool before anything is mutated.
__global__ void k_reloc_plan(const uint64_t* net, const unsigned long long* num_net, AdjView out, AdjView in,
                             uint32_t round, uint32_t* reloc_list, unsigned long long* counts) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *num_net) return;
  const uint64_t k = net[j];
  if (k >> 63) return;  // deletions never grow a list
  const uint32_t s = static_cast<uint32_t>(k >> 32) & kNodeMask, d = static_cast<uint32_t>(k) & kNodeMask;
  for (int dir = 0; dir < 2; ++dir) {
    const AdjView& a = dir == 0 ? out : in;
    const uint32_t v = dir == 0 ? s : d;
    const uint32_t need = a.len[v] + a.n_new[v];
    if (need <= a.cap[v]) continue;
    if (atomicExch(&a.reloc[v], round) == round) continue;
    const unsigned long long slot = atomicAdd(&counts[2], 1ull);
    reloc_list[slot] = (static_cast<uint32_t>(dir) << 31) | v;
    atomicAdd(&counts[3], static_cast<unsigned long long>(grow_cap(need)));
  }
}

// Undo of the per-vertex planning counters after a rejected batch.
__global__ void k_reset_plan(const uint64_t* skeys, uint32_t B, uint32_t n, AdjView out, AdjView in) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const uint32_t s = static_cast<uint32_t>(skeys[i] >> 32), d = static_cast<uint32_t>(skeys[i]);
  if (s < n) {
    out.n_new[s] = 0;
    out.reloc[s] = 0;
  }
  if (d < n) {
    in.n_new[d] = 0;
    in.reloc[d] = 0;
  }
}

// Warp per elected vertex: move its slab to a larger region of the pool.
__global__ void k_relocate(const uint32_t* reloc_list, uint32_t count, AdjView out, AdjView in,
                           unsigned long long* pool_top) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= count) return;
  const uint32_t code = reloc_list[w];
  const AdjView& a = (code >> 31) ? in : out;
  const uint32_t v = code & 0x7FFFFFFFu;
  const uint32_t len = a.len[v];
  const uint32_t ncap = grow_cap(len + a.n_new[v]);
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(pool_top, static_cast<unsigned long long>(ncap));
  base = __shfl_sync(0xffffffffu, base, 0);
  const uint32_t* src = a.ent + a.off[v];
  uint32_t* dst = a.ent + base;
  for (uint32_t i = lane; i < len; i += 32) dst[i] = src[i];
  __syncwarp();
  if (lane == 0) {
    a.off[v] = base;
    a.cap[v] = ncap;
  }
}

__device__ __forceinline__ void mark_touched(const AdjView& a, uint32_t v, uint32_t round, uint32_t* list,
                                             unsigned long long* cursor) {
  if (atomicExch(&a.touch[v], round) != round) list[atomicAdd(cursor, 1ull)] = v;
}

// Warp per net op: append NEW entries / set DEL tombstones in both directions.
__global__ void k_apply_net(const uint64_t* net, uint32_t num_net, AdjView out, AdjView in, uint32_t round,
                            uint32_t* touched_out, uint32_t* touched_in, unsigned long long* counts) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= num_net) return;
  const uint64_t k = net[w];
  const bool del = k >> 63;
  const uint32_t s = static_cast<uint32_t>(k >> 32) & kNodeMask, d = static_cast<uint32_t>(k) & kNodeMask;
  for (int dir = 0; dir < 2; ++dir) {
    const AdjView& a = dir == 0 ? out : in;
    const uint32_t v = dir == 0 ? s : d, other = dir == 0 ? d : s;
    if (!del) {
      if (lane == 0) {
        const uint32_t slot = atomicAdd(&a.len[v], 1u);
        a.ent[a.off[v] + slot] = other | kFlagNew;
      }
    } else {
      uint32_t* e = a.ent + a.off[v];
      const uint32_t len = a.len[v];
      for (uint32_t i = 0; i < len; i += 32) {
        bool hit = false;
        if (i + lane < len) {
          const uint32_t x = e[i + lane];
          hit = x == other;  // committed entry, no flags
          if (hit) e[i + lane] = x | kFlagDel;
        }
        if (__any_sync(0xffffffffu, hit)) break;
      }
      if (lane == 0) atomicAdd(&a.n_del[v], 1u);
    }
    if (lane == 0) mark_touched(a, v, round, dir == 0 ? touched_out : touched_in, &counts[4 + dir]);
  }
}

// Warp per touched vertex: drop tombstones, clear NEW bits (DynamicGraph::commit).
__global__ void k_commit(const uint32_t* touched, uint32_t count, AdjView a) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= count) return;
  const uint32_t v = touched[w];
  uint32_t* e = a.ent + a.off[v];
  const uint32_t len = a.len[v];
  uint32_t cursor = 0;
  for (uint32_t i = 0; i < len; i += 32) {
    uint32_t x = 0;
    bool keep = false;
    if (i + lane < len) {
      x = e[i + lane];
      keep = !(x & kFlagDel);
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) e[cursor + __popc(mask & ((1u << lane) - 1u))] = x & ~kFlagNew;
    cursor += __popc(mask);
    __syncwarp();
  }
  if (lane == 0) {
    a.len[v] = cursor;
    a.n_new[v] = 0;
    a.n_del[v] = 0;
  }
}

}  // namespace sgb
