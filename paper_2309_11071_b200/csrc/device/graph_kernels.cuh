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

// Edge index: open-addressing hash (src<<32|dst) -> position of the edge in
// out(src) and in(dst). Gives O(1) presence tests for validation and O(1)
// tombstoning / swap-removal, so hub lists (10^5 entries) are never scanned.
constexpr unsigned long long kHashEmpty = ~0ull, kHashTomb = ~0ull - 1;

struct EdgeHash {
  unsigned long long* keys;
  uint32_t* pos_out;
  uint32_t* pos_in;
  uint64_t mask;
};

__device__ __forceinline__ uint64_t hash_home(uint64_t key, uint64_t mask) {
  uint64_t x = key * 0x9E3779B97F4A7C15ull;
  x ^= x >> 29;
  return x & mask;
}

__device__ __forceinline__ bool hash_find(const EdgeHash& h, uint64_t key, uint64_t* slot) {
  for (uint64_t i = hash_home(key, h.mask);; i = (i + 1) & h.mask) {
    const unsigned long long k = h.keys[i];
    if (k == key) {
      *slot = i;
      return true;
    }
    if (k == kHashEmpty) return false;
  }
}

__device__ __forceinline__ uint64_t hash_insert(const EdgeHash& h, uint64_t key) {
  for (uint64_t i = hash_home(key, h.mask);; i = (i + 1) & h.mask) {
    unsigned long long k = h.keys[i];
    while (k == kHashEmpty || k == kHashTomb) {
      const unsigned long long prev = atomicCAS(&h.keys[i], k, key);
      if (prev == k) return i;
      k = prev;
    }
  }
}

// Warp per vertex: index every committed out-list entry (position in out(u)).
__global__ void k_hash_build_out(AdjView out, uint32_t n, EdgeHash h) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint32_t* e = out.ent + out.off[u];
    const uint32_t len = out.len[u];
    for (uint32_t i = lane; i < len; i += 32) {
      const uint64_t slot = hash_insert(h, (static_cast<uint64_t>(u) << 32) | (e[i] & kNodeMask));
      h.pos_out[slot] = i;
    }
  }
}

// Warp per vertex: record each edge's position in in(v).
__global__ void k_hash_build_in(AdjView in, uint32_t n, EdgeHash h) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const uint32_t* e = in.ent + in.off[v];
    const uint32_t len = in.len[v];
    for (uint32_t i = lane; i < len; i += 32) {
      uint64_t slot;
      if (hash_find(h, (static_cast<uint64_t>(e[i] & kNodeMask) << 32) | v, &slot)) h.pos_in[slot] = i;
    }
  }
}

// Thread per sorted position; segment heads walk their ops in batch order
// against the committed presence of the edge.
__global__ void k_validate(const uint64_t* skeys, const uint32_t* svals, const char* ops, uint32_t B, uint32_t n,
                           EdgeHash h, AdjView out, AdjView in, uint8_t* seg_op, uint64_t* net_cand,
                           unsigned long long* err, unsigned long long* counts) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= B) return;
  const uint64_t key = skeys[w];
  const bool head = (w == 0) || skeys[w - 1] != key;
  const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
  if (!head || s >= n || d >= n) {
    seg_op[w] = NET_NONE;
    return;
  }
  uint64_t slot;
  const bool present = hash_find(h, key, &slot);
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

// Thread per net op: append NEW entries / set DEL tombstones in both
// directions through the edge index; deletions leave (dir, v, ~pos) records
// for the commit's swap-removal.
__global__ void k_apply_net(const uint64_t* net, uint32_t num_net, AdjView out, AdjView in, EdgeHash h,
                            uint32_t round, uint32_t* touched_out, uint32_t* touched_in, uint64_t* del_rec,
                            unsigned long long* counts, unsigned long long* del_cursor) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= num_net) return;
  const uint64_t k = net[j];
  const bool del = k >> 63;
  const uint64_t key = k & ~(1ull << 63);
  const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
  if (!del) {
    const uint32_t po = atomicAdd(&out.len[s], 1u);
    out.ent[out.off[s] + po] = d | kFlagNew;
    const uint32_t pi = atomicAdd(&in.len[d], 1u);
    in.ent[in.off[d] + pi] = s | kFlagNew;
    const uint64_t slot = hash_insert(h, key);
    h.pos_out[slot] = po;
    h.pos_in[slot] = pi;
  } else {
    uint64_t slot = 0;
    hash_find(h, key, &slot);  // validated present
    const uint32_t po = h.pos_out[slot], pi = h.pos_in[slot];
    out.ent[out.off[s] + po] |= kFlagDel;
    in.ent[in.off[d] + pi] |= kFlagDel;
    atomicAdd(&out.n_del[s], 1u);
    atomicAdd(&in.n_del[d], 1u);
    const unsigned long long r = atomicAdd(del_cursor, 2ull);
    del_rec[r] = (static_cast<uint64_t>(s) << 32) | static_cast<uint32_t>(~po);
    del_rec[r + 1] = (1ull << 63) | (static_cast<uint64_t>(d) << 32) | static_cast<uint32_t>(~pi);
  }
  mark_touched(out, s, round, touched_out, &counts[4]);
  mark_touched(in, d, round, touched_in, &counts[5]);
}

// Commit step 1 (DynamicGraph::commit, graph.cpp:108-111), warp per touched
// list: clear the NEW bits, which sit exactly in [len - n_new, len).
__global__ void k_clear_new(const uint32_t* touched, uint32_t count, AdjView a) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= count) return;
  const uint32_t v = touched[w];
  uint32_t* e = a.ent + a.off[v];
  const uint32_t len = a.len[v], nn = a.n_new[v];
  for (uint32_t i = len - nn + lane; i < len; i += 32) e[i] &= ~kFlagNew;
  __syncwarp();
  if (lane == 0) a.n_new[v] = 0;
}

// Commit step 2: thread per (dir, v) run of deletion records sorted by
// descending position; each tombstone is swap-removed with the list's last
// entry and the moved edge's index position is updated. O(changes), not O(deg).
__global__ void k_swap_remove(const uint64_t* rec, uint32_t n, AdjView out, AdjView in, EdgeHash h) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i > 0 && (rec[i] >> 32) == (rec[i - 1] >> 32)) return;
  const bool dir_in = rec[i] >> 63;
  const uint32_t v = static_cast<uint32_t>(rec[i] >> 32) & 0x7FFFFFFFu;
  const AdjView& a = dir_in ? in : out;
  uint32_t* e = a.ent + a.off[v];
  uint32_t len = a.len[v];
  for (uint32_t j = i; j < n && (rec[j] >> 32) == (rec[i] >> 32); ++j) {
    const uint32_t pos = ~static_cast<uint32_t>(rec[j]);
    const uint32_t last = len - 1;
    if (pos != last) {
      const uint32_t moved = e[last];
      e[pos] = moved;
      const uint32_t other = moved & kNodeMask;
      const uint64_t key = dir_in ? ((static_cast<uint64_t>(other) << 32) | v) : ((static_cast<uint64_t>(v) << 32) | other);
      uint64_t slot;
      if (hash_find(h, key, &slot)) (dir_in ? h.pos_in : h.pos_out)[slot] = pos;
    }
    len = last;
  }
  a.len[v] = len;
  a.n_del[v] = 0;
}

// Commit step 3: drop deleted edges from the index.
__global__ void k_hash_erase(const uint64_t* net, uint32_t num_net, EdgeHash h) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= num_net) return;
  const uint64_t k = net[j];
  if (!(k >> 63)) return;
  uint64_t slot;
  if (hash_find(h, k & ~(1ull << 63), &slot)) h.keys[slot] = kHashTomb;
}

}  // namespace sgb
