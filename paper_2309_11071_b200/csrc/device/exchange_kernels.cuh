// Device-side shard exchange over peer memory.
//
// Every shard owns a small "mailbox" in its own HBM that the other shards
// read through peer memory (same device, NVLink P2P, or a CUDA IPC mapping).
// A round's collectives — the per-layer dirty-count all-gather and the
// round-end counter all-reduce — become publish / wait kernel pairs inside the
// round's one CUDA graph, so a sharded round needs no host synchronisation
// until its result copy:
//   publish: store the value(s) into the own mailbox, fence at system scope,
//            then release-store the shard's event sequence number;
//   wait:    one lane per peer acquire-spins on the peer's sequence number
//            until it reaches this shard's own (every shard runs the same
//            event sequence), then reads the peer's value(s).
// The sequence counter lives on the device (bumped by the publishing thread),
// so the captured graph replays correctly round after round. A wait that
// exceeds kSpinLimitNs (a peer died or stopped) sets the round's error flag
// and returns instead of hanging the GPU.
#pragma once

#include "dev_common.cuh"

namespace sgb {

// Mailbox layout (u64 words).
enum : uint32_t {
  MB_SEQ = 0,          // last published event sequence number
  MB_COUNT = 8,        // [l] dirty count of layer l (l < 8)
  MB_CTR = 16,         // round counters, two alternating copies of MB_CTR_N words
  MB_CTR_N = 512,
  MB_WORDS = MB_CTR + 2 * MB_CTR_N
};
constexpr unsigned long long kSpinLimitNs = 30ull * 1000 * 1000 * 1000;

struct PeerBoxes {
  const uint64_t* box[kMaxPeers];  // every shard's mailbox (this shard's included)
  uint32_t world;
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Peer data after an acquire (by this thread or, behind a CTA barrier, by the
// polling thread): relaxed system-scope loads, never a stale L1 line.
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spins until box[MB_SEQ] >= seq; false on timeout.
__device__ __forceinline__ bool wait_seq(const uint64_t* box, uint64_t seq) {
  const unsigned long long t0 = globaltimer_ns();
  for (uint32_t i = 0; ld_acquire_sys(box + MB_SEQ) < seq; ++i) {
    if ((i & 255u) == 255u && globaltimer_ns() - t0 > kSpinLimitNs) return false;
    __nanosleep(64);
  }
  return true;
}

// Publishes this shard's layer-l dirty count (everything earlier on the stream
// — the pack buffer, the owner's table rows — is visible to peers first).
__global__ void k_publish_count(uint64_t* mybox, uint64_t* seq_ctr, const unsigned long long* count, uint32_t l) {
  pdl_prologue();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  mybox[MB_COUNT + l] = *count;
  __threadfence_system();
  const uint64_t s = ++*seq_ctr;
  st_release_sys(mybox + MB_SEQ, s);
}

// The import table of layer l from every peer's published count: tab[3r] =
// shard r's pack buffer (peer address), tab[3r+1] = count, tab[3r+2] = first
// global dirty position, tab[3w] = total (k_import_table's input).
__global__ void k_wait_counts(PeerBoxes P, const uint64_t* seq_ctr, uint32_t l, const unsigned long long* packs,
                              unsigned long long* tab, unsigned long long* err) {
  pdl_prologue();
  __shared__ unsigned long long cnt[kMaxPeers];
  const uint32_t q = threadIdx.x;
  const uint64_t s = *seq_ctr;
  if (q < P.world) {
    if (!wait_seq(P.box[q], s)) {
      atomicExch(err, 1ull);
      cnt[q] = 0;
    } else {
      cnt[q] = ld_relaxed_sys(P.box[q] + MB_COUNT + l);
    }
  }
  __syncthreads();
  if (q == 0) {
    unsigned long long g0 = 0;
    for (uint32_t r = 0; r < P.world; ++r) {
      tab[3 * r] = packs[r];
      tab[3 * r + 1] = cnt[r];
      tab[3 * r + 2] = g0;
      g0 += cnt[r];
    }
    tab[3 * P.world] = g0;
  }
}

// Round-end counter all-reduce: publish a copy of the local counters (slot by
// round parity), wait for every peer's, sum them into the local counters.
__global__ void k_publish_counters(uint64_t* mybox, uint64_t* seq_ctr, const unsigned long long* ctr, uint32_t n) {
  pdl_prologue();
  __shared__ uint64_t s;
  if (threadIdx.x == 0) s = *seq_ctr + 1;
  __syncthreads();
  uint64_t* dst = mybox + MB_CTR + (s & 1) * MB_CTR_N;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = ctr[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    *seq_ctr = s;
    st_release_sys(mybox + MB_SEQ, s);
  }
}

__global__ void k_reduce_counters(PeerBoxes P, const uint64_t* seq_ctr, unsigned long long* ctr, uint32_t n,
                                  unsigned long long* err) {
  pdl_prologue();
  __shared__ int ok;
  const uint64_t s = *seq_ctr;
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  if (threadIdx.x < P.world && !wait_seq(P.box[threadIdx.x], s)) {
    atomicExch(err, 1ull);
    ok = 0;
  }
  __syncthreads();
  if (!ok) return;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long sum = 0;
    for (uint32_t r = 0; r < P.world; ++r) sum += ld_relaxed_sys(P.box[r] + MB_CTR + (s & 1) * MB_CTR_N + i);
    ctr[i] = sum;
  }
}

}  // namespace sgb
