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

// Sort keys are packed to 2b bits, b = bits of the node count: (s << b) | d
// for in-range ids (exact, decoded by batch_key_src/dst); an out-of-range id is
// clamped to 2^b - 1 (>= n, still invalid) so it can never merge with a valid
// key's segment. Fewer key bits = fewer radix passes for the batch sort.
__host__ __device__ __forceinline__ uint64_t batch_key(uint32_t s, uint32_t d, uint32_t b) {
  const uint32_t top = b >= 32 ? 0xFFFFFFFFu : (1u << b) - 1u;
  return (static_cast<uint64_t>(min(s, top)) << b) | min(d, top);
}
__device__ __forceinline__ uint32_t batch_key_src(uint64_t k, uint32_t b) { return static_cast<uint32_t>(k >> b); }
__device__ __forceinline__ uint32_t batch_key_dst(uint64_t k, uint32_t b) {
  return static_cast<uint32_t>(k & ((1ull << b) - 1ull));
}

__global__ void k_batch_keys(const char* ops, const uint32_t* src, const uint32_t* dst, uint32_t B, uint32_t n,
                             uint32_t b, uint64_t* keys, uint32_t* vals, unsigned long long* err, uint32_t* badop) {
  pdl_prologue();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  char o = ops[i];
  if (o != '+' && o != '-') atomicOr(badop, 1u);
  uint32_t s = src[i], d = dst[i];
  keys[i] = batch_key(s, d, b);
  vals[i] = i;
  if (s >= n || d >= n) atomicMin(err, (static_cast<unsigned long long>(i) << 8) | ERR_RANGE);
}

// Edge index: open-addressing hash (src<<32|dst) -> position of the edge in
// out(src) and in(dst). Gives O(1) presence tests for validation and O(1)
// tombstoning / swap-removal, so hub lists (10^5 entries) are never scanned.
constexpr unsigned long long kHashEmpty = ~0ull, kHashTomb = ~0ull - 1;

// One 16-byte slot per key: the key and the edge's positions in out(src) and
// in(dst) share a sector, so a probe that finds the key has its positions
// too (three separate arrays cost three scattered DRAM accesses per lookup in
// K1 and the commit, whose first touches bound them).
struct __align__(16) HashSlot {
  unsigned long long key;
  uint32_t pos_out;
  uint32_t pos_in;
};

struct EdgeHash {
  HashSlot* s;
  uint64_t mask;
};

// The whole slot in one 16-byte load.
__device__ __forceinline__ HashSlot load_slot(const HashSlot* p) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
  HashSlot r;
  r.key = v.x;
  r.pos_out = static_cast<uint32_t>(v.y);
  r.pos_in = static_cast<uint32_t>(v.y >> 32);
  return r;
}

__device__ __forceinline__ uint64_t hash_home(uint64_t key, uint64_t mask) {
  uint64_t x = key * 0x9E3779B97F4A7C15ull;
  x ^= x >> 29;
  return x & mask;
}

__device__ __forceinline__ bool hash_find(const EdgeHash& h, uint64_t key, uint64_t* slot) {
  for (uint64_t i = hash_home(key, h.mask);; i = (i + 1) & h.mask) {
    const unsigned long long k = h.s[i].key;
    if (k == key) {
      *slot = i;
      return true;
    }
    if (k == kHashEmpty) return false;
  }
}

__device__ __forceinline__ uint64_t hash_insert(const EdgeHash& h, uint64_t key) {
  for (uint64_t i = hash_home(key, h.mask);; i = (i + 1) & h.mask) {
    unsigned long long k = h.s[i].key;
    while (k == kHashEmpty || k == kHashTomb) {
      const unsigned long long prev = atomicCAS(&h.s[i].key, k, key);
      if (prev == k) return i;
      k = prev;
    }
  }
}

// Warp per vertex: index every committed out-list entry (position in out(u)).
__global__ void k_hash_build_out(AdjView out, uint32_t n, EdgeHash h) {
  pdl_prologue();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint32_t* e = out.ent + out.off[u];
    const uint32_t len = out.len[u];
    for (uint32_t i = lane; i < len; i += 32) {
      const uint64_t slot = hash_insert(h, (static_cast<uint64_t>(u) << 32) | (e[i] & kNodeMask));
      h.s[slot].pos_out = i;
    }
  }
}

// Warp per vertex: record each edge's position in in(v).
__global__ void k_hash_build_in(AdjView in, uint32_t n, EdgeHash h) {
  pdl_prologue();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const uint32_t* e = in.ent + in.off[v];
    const uint32_t len = in.len[v];
    for (uint32_t i = lane; i < len; i += 32) {
      uint64_t slot;
      if (hash_find(h, (static_cast<uint64_t>(e[i] & kNodeMask) << 32) | v, &slot)) h.s[slot].pos_in = i;
    }
  }
}

// Thread per sorted position; segment heads walk their ops in batch order
// against the committed presence of the edge. Net changes are appended (order
// irrelevant downstream) to `net` as key | delete << 63.
__global__ void k_validate(const uint64_t* skeys, const uint32_t* svals, const char* ops, uint32_t B, uint32_t n,
                           uint32_t b, EdgeHash h, AdjView out, AdjView in, uint64_t* net, unsigned long long* err,
                           unsigned long long* counts, unsigned long long* num_net) {
  pdl_prologue();
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= B) return;
  const uint64_t bkey = skeys[w];
  const bool head = (w == 0) || skeys[w - 1] != bkey;
  const uint32_t s = batch_key_src(bkey, b), d = batch_key_dst(bkey, b);
  if (!head || s >= n || d >= n) return;
  const uint64_t key = (static_cast<uint64_t>(s) << 32) | d;
  uint64_t slot;
  const bool present = hash_find(h, key, &slot);
  bool p = present, ok = true;
  for (uint32_t j = w; j < B && skeys[j] == bkey; ++j) {
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
  if (!ok || p == present) return;
  net[atomicAdd(num_net, 1ull)] = p ? key : (key | (1ull << 63));
  if (p) {
    atomicAdd(&counts[0], 1ull);
    atomicAdd(&out.n_new[s], 1u);
    atomicAdd(&in.n_new[d], 1u);
  } else {
    atomicAdd(&counts[1], 1ull);
  }
}

// Elects vertices whose slab cannot take this round's appends; sums the pool
// demand so the host can grow the pool before anything is mutated.
__device__ __forceinline__ void reloc_plan_one(uint64_t k, AdjView out, AdjView in, uint32_t round,
                                               uint32_t* reloc_list, unsigned long long* counts);

__global__ void k_reloc_plan(const uint64_t* net, const unsigned long long* num_net, AdjView out, AdjView in,
                             const uint32_t* round_p, uint32_t* reloc_list, unsigned long long* counts) {
  pdl_prologue();
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *num_net) return;
  reloc_plan_one(net[j], out, in, *round_p, reloc_list, counts);
}

// Slab relocation election for one net edge: a list that will not fit its
// NEW entries is elected once per round and its grown capacity added to the
// pool demand.
__device__ __forceinline__ void reloc_plan_one(uint64_t k, AdjView out, AdjView in, uint32_t round,
                                               uint32_t* reloc_list, unsigned long long* counts) {
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

// Decides, on the device, whether this round may mutate anything: no invalid
// op, no failing edge op, and enough slab-pool headroom for the relocations.
// Also starts every layer's record cursor after its seed block.
__device__ __forceinline__ void round_gate(const unsigned long long* err, const unsigned long long* badop,
                                           const unsigned long long* demand, const unsigned long long* pool_top,
                                           unsigned long long pool_cap, unsigned long long* abort,
                                           const unsigned long long* num_net, uint32_t mult,
                                           unsigned long long* cursors, uint32_t stride, uint32_t layers) {
  unsigned long long a = 0;
  if (*badop) a = 1;
  else if (*err != ~0ull) a = 2;
  else if (*pool_top + *demand > pool_cap) a = 3;
  *abort = a;
  for (uint32_t l = 0; l < layers; ++l) cursors[l * stride] = *num_net * mult;
}

__global__ void k_round_gate(const unsigned long long* err, const unsigned long long* badop,
                             const unsigned long long* demand, const unsigned long long* pool_top,
                             unsigned long long pool_cap, unsigned long long* abort,
                             const unsigned long long* num_net, uint32_t mult, unsigned long long* cursors,
                             uint32_t stride, uint32_t layers) {
  pdl_prologue();
  round_gate(err, badop, demand, pool_top, pool_cap, abort, num_net, mult, cursors, stride, layers);
}


// Batches of <= cap updates (cap = 4096): k_batch_keys + sort + k_validate in
// one CTA without sorting. Every in-range op inserts its key into a
// shared-memory hash table (2 cap slots) that records the key's first batch
// index and op count; the head op of each key then walks that key's ops in
// batch order (a single op needs no walk — the common case) against the
// committed presence, exactly like k_validate walks a sorted segment. The
// first failing op overall is the minimum index over the keys' first failures
// (keys are independent), as in the reference's in-order overlay validation.
constexpr uint32_t kGroupCap = 4096;
__host__ __device__ constexpr size_t batch_group_smem(uint32_t cap) {
  return static_cast<size_t>(2 * cap) * (8 + 4 + 4) + static_cast<size_t>(cap) * (8 + 4);
}

// Undo of the per-vertex planning counters after a rejected batch.
__global__ void k_reset_plan(const uint64_t* skeys, uint32_t B, uint32_t n, uint32_t b, AdjView out, AdjView in) {
  pdl_prologue();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const uint32_t s = batch_key_src(skeys[i], b), d = batch_key_dst(skeys[i], b);
  if (s < n) {
    out.n_new[s] = 0;
    out.reloc[s] = 0;
  }
  if (d < n) {
    in.n_new[d] = 0;
    in.reloc[d] = 0;
  }
}

// One elected vertex's slab moved to a larger region of the pool (warp-wide).
__device__ __forceinline__ void relocate_one(uint32_t code, const AdjView& out, const AdjView& in,
                                             unsigned long long* pool_top) {
  const uint32_t lane = threadIdx.x & 31;
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

// Warp per elected vertex.
__global__ void k_relocate(const uint32_t* reloc_list, const unsigned long long* count_p, AdjView out, AdjView in,
                           unsigned long long* pool_top, const unsigned long long* abort) {
  pdl_prologue();
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (*abort || w >= *count_p) return;
  relocate_one(reloc_list[w], out, in, pool_top);
}

// Per-round deletion lists: each tombstone pushes its list position onto a
// per-(direction, vertex) linked list, consumed by the commit.
struct DelLists {
  uint32_t* head_out;  // [n] index of the last record, ~0 = empty
  uint32_t* head_in;
  uint32_t* pos;       // record -> list position
  uint32_t* next;      // record -> next record of the same list
  unsigned long long* cursor;
};

// One net op: append the NEW entries / set the DEL tombstones in both
// directions through the edge index.
__device__ __forceinline__ void apply_net_one(uint64_t k, const AdjView& out, const AdjView& in, const EdgeHash& h,
                                              uint32_t round, uint32_t* touched_out, uint32_t* touched_in,
                                              const DelLists& dl, unsigned long long* counts) {
  const bool del = k >> 63;
  const uint64_t key = k & ~(1ull << 63);
  const uint32_t s = static_cast<uint32_t>(key >> 32), d = static_cast<uint32_t>(key);
  // independent memory operations first, so one update's chain of dependent
  // round trips stays short (results-free atomics compile to reductions)
  const uint32_t ts = atomicExch(&out.touch[s], round), td = atomicExch(&in.touch[d], round);
  const uint64_t os = out.off[s], od = in.off[d];
  if (!del) {
    const uint32_t po = atomicAdd(&out.len[s], 1u);
    const uint32_t pi = atomicAdd(&in.len[d], 1u);
    const uint64_t slot = hash_insert(h, key);
    out.ent[os + po] = d | kFlagNew;
    in.ent[od + pi] = s | kFlagNew;
    h.s[slot].pos_out = po;
    h.s[slot].pos_in = pi;
  } else {
    const uint32_t r = static_cast<uint32_t>(atomicAdd(dl.cursor, 2ull));
    const uint32_t ho = atomicExch(&dl.head_out[s], r), hi = atomicExch(&dl.head_in[d], r + 1);
    atomicAdd(&out.n_del[s], 1u);
    atomicAdd(&in.n_del[d], 1u);
    uint64_t slot = 0;
    hash_find(h, key, &slot);  // validated present
    const uint32_t po = h.s[slot].pos_out, pi = h.s[slot].pos_in;
    atomicOr(&out.ent[os + po], kFlagDel);
    atomicOr(&in.ent[od + pi], kFlagDel);
    dl.pos[r] = po;
    dl.next[r] = ho;
    dl.pos[r + 1] = pi;
    dl.next[r + 1] = hi;
  }
  if (ts != round) touched_out[atomicAdd(&counts[4], 1ull)] = s;
  if (td != round) touched_in[atomicAdd(&counts[5], 1ull)] = d;
}

// Thread per net op (large batches; small ones are applied inside k_batch_group).
__global__ void k_apply_net(const uint64_t* net, const unsigned long long* num_net_p, AdjView out, AdjView in,
                            EdgeHash h, const uint32_t* round_p, uint32_t* touched_out, uint32_t* touched_in,
                            DelLists dl, unsigned long long* counts, const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  const uint32_t round = *round_p;
  const uint64_t num_net = *num_net_p;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < num_net;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    apply_net_one(net[j], out, in, h, round, touched_out, touched_in, dl, counts);
}

// DynamicGraph::commit (graph.cpp:108-111), warp per touched list, O(changes):
// clear the NEW bits (they sit exactly in [len - n_new, len)), then shrink the
// list by n_del: every tombstone below the new length L' is filled with one of
// the live entries of the tail [L', len) and that edge's index position is
// updated. Lists with more than kCommitSmall deletions in one round are
// compacted whole (every moved edge re-indexed).
constexpr uint32_t kCommitSmall = 128;

// One touched list of one direction (warp-wide).
__device__ __forceinline__ void commit_list(uint32_t v, const AdjView& a, bool dir_in, const EdgeHash& h,
                                            uint32_t* head, const uint32_t* dpos, const uint32_t* dnext,
                                            uint32_t* holes, uint32_t* movers) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* e = a.ent + a.off[v];
  const uint32_t len = a.len[v], nn = a.n_new[v], nd = a.n_del[v];
  for (uint32_t i = len - nn + lane; i < len; i += 32) e[i] &= ~kFlagNew;
  __syncwarp();
  auto reindex = [&](uint32_t pos, uint32_t x) {
    const uint32_t other = x & kNodeMask;
    const uint64_t key = dir_in ? ((static_cast<uint64_t>(other) << 32) | v) : ((static_cast<uint64_t>(v) << 32) | other);
    uint64_t slot;
    if (hash_find(h, key, &slot)) (dir_in ? h.s[slot].pos_in : h.s[slot].pos_out) = pos;
  };
  if (nd > 0 && nd <= kCommitSmall) {
    const uint32_t L = len - nd;
    // holes below L' from the deletion list (walked by lane 0)
    uint32_t nh = 0;
    if (lane == 0) {
      for (uint32_t r = head[v]; r != 0xFFFFFFFFu; r = dnext[r])
        if (dpos[r] < L) holes[nh++] = dpos[r];
    }
    nh = __shfl_sync(0xffffffffu, nh, 0);
    // live movers in the tail [L', len)
    uint32_t nm = 0;
    for (uint32_t i = L; i < len; i += 32) {
      const bool live = (i + lane < len) && !(e[i + lane] & kFlagDel);
      const uint32_t mask = __ballot_sync(0xffffffffu, live);
      if (live) movers[nm + __popc(mask & ((1u << lane) - 1u))] = i + lane;
      nm += __popc(mask);
    }
    __syncwarp();
    for (uint32_t q = lane; q < nh; q += 32) {
      const uint32_t dst = holes[q], src = movers[q];
      const uint32_t x = e[src];
      e[dst] = x;
      reindex(dst, x);
    }
    __syncwarp();
    if (lane == 0) a.len[v] = L;
  } else if (nd > kCommitSmall) {
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
      const uint32_t dst = cursor + __popc(mask & ((1u << lane) - 1u));
      if (keep) {
        e[dst] = x;
        if (dst != i + lane) reindex(dst, x);
      }
      cursor += __popc(mask);
      __syncwarp();
    }
    if (lane == 0) a.len[v] = cursor;
  }
  if (lane == 0) {
    a.n_new[v] = 0;
    a.n_del[v] = 0;
    head[v] = 0xFFFFFFFFu;
  }
}

// The whole commit in one launch: every touched out-list and in-list (warp
// each; the two directions touch disjoint lists and index fields), and the
// erase of deleted keys from the index (thread per net op; it only tombstones
// deleted keys, which no list fix-up looks up: probes pass tombstones).
__global__ void __launch_bounds__(256) k_commit(const uint32_t* touched_out, const uint32_t* touched_in,
                                                const unsigned long long* counts, AdjView out, AdjView in,
                                                EdgeHash h, uint32_t* head_out, uint32_t* head_in,
                                                const uint32_t* dpos, const uint32_t* dnext, const uint64_t* net,
                                                const unsigned long long* num_net_p, const unsigned long long* abort) {
  pdl_prologue();
  __shared__ uint32_t holes[8][kCommitSmall];
  __shared__ uint32_t movers[8][kCommitSmall];
  if (*abort) return;
  const uint32_t wib = threadIdx.x >> 5;
  const uint64_t n_out = counts[4], n_in = counts[5], num_net = *num_net_p;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < num_net;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = net[j];
    if (!(k >> 63)) continue;
    uint64_t slot;
    if (hash_find(h, k & ~(1ull << 63), &slot)) h.s[slot].key = kHashTomb;
  }
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_out + n_in; w += warps) {
    if (w < n_out) commit_list(touched_out[w], out, false, h, head_out, dpos, dnext, holes[wib], movers[wib]);
    else commit_list(touched_in[w - n_out], in, true, h, head_in, dpos, dnext, holes[wib], movers[wib]);
  }
}

}  // namespace sgb
