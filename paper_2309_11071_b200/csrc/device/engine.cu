// DeviceEngine: host orchestration of one update round on a B200.
//
// Round = Engine::process_update_round (proj/src/core/engine.cpp:171-319), issued
// as one asynchronous kernel sequence on the engine's stream with NO host
// synchronisation until the round is complete. Every data-dependent size lives
// in device memory (round scalars) and every kernel after the batch sort is
// grid-stride over those counts; buffers are provisioned from host-side bounds
// (edge count, batch size, node count) before the round starts.
//   K1  sort batch, validate (first failing op decides), net delta, gate
//       (k_round_gate: abort flag when invalid or the slab pool is short),
//       slab relocation, NEW appends / DEL tombstones through the edge index
//   per layer l = 1..k:
//     K2/K7 records: seeds, expansion of layer l-1's dirty sources (reserved
//           ranges, 256-entry work items), SELF records; counting sort by target
//     K3  segment plan + group-reduce + classify + incremental update
//     K4  exposed-reset recompute (chunked work items, hub-safe)
//     K5  dirty collection + next-layer record reservations
//     K6  combination over the dirty rows (exact serial-k GEMM chain)
//     K8  message write-back with pre-image capture and change flags
//   commit: O(changes) list fixes, index erase; one D2H of scalars + counters.
// A round rejected by the gate mutated nothing; the host decodes the error (or
// grows the slab pool and replays the round).
#include "engine.hpp"

#include <cub/cub.cuh>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include "../tensor_io.hpp"
#include "aggregate_kernels.cuh"
#include "combine_kernels.cuh"
#include "combine_tc.cuh"
#include "dev_common.cuh"
#include "event_kernels.cuh"
#include "exchange_kernels.cuh"
#include "graph_kernels.cuh"

namespace sgb {

namespace {

// Kernel launch with a programmatic dependency on the preceding kernel in the
// stream (PDL; every kernel opens with pdl_prologue(), dev_common.cuh), so a
// round's chain of small kernels overlaps each launch with the previous tail.
// Off by default (SGNN_B200_PDL=1 enables): it gained ~1 % at C3 and nothing at
// C2, and a sharded parity case failed once in a run with it on (under study).
// Sharded rounds never use it (host-driven exchanges, import-table uploads and
// two-stream segments are outside the pdl_prologue argument): apply() clears
// it for the calling thread while a sharded engine's round is enqueued.
thread_local bool tl_pdl_allowed = true;
inline bool use_pdl() {
  static const bool on = [] {
    const char* e = std::getenv("SGNN_B200_PDL");
    return e && std::atoi(e) != 0;
  }();
  return on && tl_pdl_allowed;
}
struct PdlScope {
  bool saved;
  explicit PdlScope(bool allow) : saved(tl_pdl_allowed) { tl_pdl_allowed = allow && saved; }
  ~PdlScope() { tl_pdl_allowed = saved; }
};
template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  SGB_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

constexpr uint32_t kChunk = 512;        // in-list entries per aggregation work item (full inference)
constexpr uint32_t kChunkUpdate = 32;   // ... per exposed-reset recompute work item (more, smaller items)

// Bumped on every device allocation: a captured round graph bakes pointers in,
// so any reallocation invalidates it.
inline std::atomic<uint64_t>& alloc_epoch() {
  static std::atomic<uint64_t> e{0};
  return e;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) {
    o.p = nullptr;
    o.cap = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(cap, o.cap);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) SGB_CUDA(cudaFree(p));
    p = nullptr;
    size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    SGB_CUDA(cudaMalloc(&p, want));
    cap = want;
    ++alloc_epoch();
  }
  void alloc_exact(size_t bytes) {
    if (p) SGB_CUDA(cudaFree(p));
    p = nullptr;
    cap = 0;
    if (bytes) {
      SGB_CUDA(cudaMalloc(&p, bytes));
      cap = bytes;
    }
    ++alloc_epoch();
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) SGB_CUDA(cudaFreeHost(p));
    p = nullptr;
    size_t want = std::max<size_t>(bytes + bytes / 4, 4096);
    SGB_CUDA(cudaMallocHost(&p, want));
    cap = want;
    ++alloc_epoch();
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Round-scoped device scalars: a global block, then one block per layer.
enum : int {
  S_ERR = 0, S_BADOP, S_NET_INS, S_NET_DEL, S_RELOC_N, S_RELOC_DEMAND, S_TOUCH_OUT, S_TOUCH_IN, S_NUM_NET, S_ABORT,
  S_DELREC, S_FRONT_A, S_FRONT_B, S_COUNT, S_COUNT2, S_XERR, S_GLOBAL = 16
};
enum : int {
  L_RUNS = 0, L_NSEG, L_NCLS, L_NWORK, L_NSCRATCH, L_NDIRTY, L_CURSOR, L_EXPWORK, L_NCHANGED, L_NSPARSE, L_NSWORK,
  L_ALLOC, L_STRIDE = 12
};

// Every transfer goes through the engine's (non-blocking) stream and is waited
// for: legacy-stream cudaMemcpy from pageable memory may return before its DMA
// lands and does not order against a non-blocking stream.
inline cudaError_t copy_sync(cudaStream_t st, void* dst, const void* src, size_t n, cudaMemcpyKind k) {
  cudaError_t e = cudaMemcpyAsync(dst, src, n, k, st);
  return e != cudaSuccess ? e : cudaStreamSynchronize(st);
}
inline cudaError_t copy2d_sync(cudaStream_t st, void* dst, size_t dp, const void* src, size_t sp, size_t w, size_t h,
                               cudaMemcpyKind k) {
  cudaError_t e = cudaMemcpy2DAsync(dst, dp, src, sp, w, h, k, st);
  return e != cudaSuccess ? e : cudaStreamSynchronize(st);
}
inline cudaError_t memset_sync(cudaStream_t st, void* dst, int v, size_t n) {
  cudaError_t e = cudaMemsetAsync(dst, v, n, st);
  return e != cudaSuccess ? e : cudaStreamSynchronize(st);
}

inline unsigned grid_for(uint64_t threads, unsigned block = 256) {
  uint64_t g = (threads + block - 1) / block;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(g, 1u << 30)));
}

int num_bits(uint32_t n) {  // smallest b with 2^b > n
  int b = 0;
  while (b < 32 && (uint64_t(1) << b) <= n) ++b;
  return b;
}

int cpl_for(uint32_t V) {
  if (V <= 32) return 1;
  if (V <= 64) return 2;
  if (V <= 128) return 4;
  if (V <= 256) return 8;
  if (V <= 512) return 16;
  fail(Errc::unsupported_model, "message dimension " + std::to_string(V * 4) +
                                    " exceeds the device engine limit of 2048 floats");
}

struct Adj {
  DevBuf off, len, cap, n_new, n_del, touch, reloc;
  AdjView view(uint32_t* pool) const {
    return AdjView{off.as<uint64_t>(), len.as<uint32_t>(), cap.as<uint32_t>(), pool, n_new.as<uint32_t>(),
                   n_del.as<uint32_t>(), touch.as<uint32_t>(), reloc.as<uint32_t>()};
  }
};

// ---- BFS helpers for the baseline counters (baseline.cpp:101-232) --------

__global__ void k_seed_area(const uint64_t* net, const unsigned long long* num_net_p, uint8_t* reached,
                            uint32_t* front, unsigned long long* front_n) {
  pdl_prologue();
  const uint64_t num_net = *num_net_p;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < num_net;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = net[j];
    const uint32_t us[2] = {static_cast<uint32_t>(k >> 32) & kNodeMask, static_cast<uint32_t>(k) & kNodeMask};
    for (int q = 0; q < 2; ++q) {
      uint32_t* word = reinterpret_cast<uint32_t*>(reached + (us[q] & ~3u));
      const uint32_t bit = 1u << (8 * (us[q] & 3u));
      if (!(atomicOr(word, bit) & bit)) front[atomicAdd(front_n, 1ull)] = us[q];
    }
  }
}

// Warp per frontier node: expand live entries of its list (out or in view).
__global__ void k_bfs_expand(const uint32_t* front, const unsigned long long* front_n, AdjView a, uint8_t* reached,
                             uint32_t* next, unsigned long long* next_n) {
  pdl_prologue();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t n = *front_n;
  for (uint64_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
    const uint32_t v = front[w];
    const uint32_t* e = a.ent + a.off[v];
    const uint32_t len = a.len[v];
    for (uint32_t i = lane; i < len; i += 32) {
      const uint32_t x = e[i];
      if (x & kFlagDel) continue;
      const uint32_t u = x & kNodeMask;
      uint32_t* word = reinterpret_cast<uint32_t*>(reached + (u & ~3u));
      const uint32_t bit = 1u << (8 * (u & 3u));
      if (!(atomicOr(word, bit) & bit)) next[atomicAdd(next_n, 1ull)] = u;
    }
  }
}

// Sum over members of (live in-degree + self), and the member list.
__global__ void k_need_count(const uint8_t* member, uint32_t n, const uint32_t* in_len, const uint32_t* in_del,
                             uint32_t self, unsigned long long* out, unsigned long long* members, uint32_t* list) {
  pdl_prologue();
  unsigned long long s = 0, c = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (member[v]) {
      s += in_len[v] - in_del[v] + self;
      ++c;
      if (list) list[atomicAdd(members + 1, 1ull)] = v;
    }
  warp_add(out, s);
  warp_add(members, c);
}

__global__ void k_first_mismatch(const float* a, const float* b, uint32_t n, uint32_t pitch, uint32_t d,
                                 unsigned long long* out) {
  pdl_prologue();
  const uint64_t total = static_cast<uint64_t>(n) * d;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = static_cast<uint32_t>(i / d), c = static_cast<uint32_t>(i % d);
    const size_t o = static_cast<size_t>(v) * pitch + c;
    if (__float_as_uint(a[o]) != __float_as_uint(b[o]))
      atomicMin(out, (static_cast<unsigned long long>(v) << 32) | c);
  }
}

__global__ void k_add_u64(unsigned long long* p, unsigned long long v) {
  pdl_prologue(); *p += v; }

__global__ void k_l2_flush(uint4* p, size_t n, uint32_t salt) {
  pdl_prologue();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = make_uint4(salt, salt, salt, salt);
}


}  // namespace

bool cuda_device_available(std::string* why) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    if (why) *why = e != cudaSuccess ? cudaGetErrorString(e) : "no CUDA device";
    cudaGetLastError();
    return false;
  }
  return true;
}

struct DeviceEngine::Impl {
  std::shared_ptr<const BoundModel> model;
  EngineOptions opts;
  cudaStream_t st = nullptr;
  // Side stream for independent kernels of a round (fork/join through events,
  // captured as parallel graph branches): the sparse recompute beside the
  // dense one, the in-list commit beside the out-list commit.
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_producer = nullptr, ev_result = nullptr;
  void fork() {
    SGB_CUDA(cudaEventRecord(ev_fork, st));
    SGB_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
  }
  void join() {
    SGB_CUDA(cudaEventRecord(ev_join, st2));
    SGB_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  }
  int device = 0;
  int sms = 148;
  int smem_per_sm = 228 << 10;  // shared memory per SM (bytes), for one-wave grids of smem-heavy kernels
  uint32_t N = 0;
  uint64_t E = 0;
  int k = 0;
  bool is_max = false;
  std::vector<uint32_t> d, P;  // [l] for l = 1..k+1 (index 0 unused)
  uint32_t maxP = 0;
  std::vector<float> features;  // host copy, for prefix models and verify
  uint32_t F = 0;
  uint32_t round = 1;

  // tables
  std::vector<DevBuf> msg, agg;              // msg[1..k+1], agg[1..k]
  std::vector<DevBuf> stamp, slot, oldslab;  // [l] for l = 2..k
  // [l] for filtered layers l = 2..k: 16-bit alpha bound codes (N x P[l] u16,
  // dev_common.cuh abound_code) and their column grid (base[P], step[P], 1/step[P]);
  // codes refreshed by K8 for dirty rows, grid and codes by refresh_abound()
  // after any whole-table rewrite of a_l
  std::vector<DevBuf> abound, abstat;
  // [l] for every filtered layer: per-target summary = the row minimum of the
  // alpha codes over c < d (combine_kernels.cuh summarise_row); abstat is kept
  // for these layers too (their filter computes thresholds on the fly)
  std::vector<DevBuf> cmin;
  // [l] for filtered layers with bound codes: 16-bit per-position thresholds
  // of layer l-1's dirty sources (row = dirty position), written by K8 of
  // layer l-1 (k_source_thresholds after a shard exchange), read by the filter
  std::vector<DevBuf> thrtab;
  DevBuf abcolr;  // 2 * maxP ints: column range scratch of refresh_abound()

  // graph
  Adj out, in;
  DevBuf pool;
  uint64_t pool_cap = 0;     // entries
  DevBuf pool_top;           // u64 device scalar
  uint64_t in_entries = 0;   // host bound of sum in_len (live + this round's NEW)
  uint64_t out_entries = 0;  // host bound of sum out_len
  DevBuf h_slots;  // edge index, 16-byte HashSlot per slot (graph_kernels.cuh)
  uint64_t hcap = 0, h_tombs = 0;
  DevBuf del_head_out, del_head_in, del_pos, del_next;

  // weights
  std::map<const void*, DevBuf> wdev;  // matrix / bias host ptr -> device copy
  std::map<const void*, uint32_t> wld;

  // round buffers (provisioned by ensure_capacity)
  DevBuf b_src, b_keys, b_vals, b_keys_s, b_vals_s, b_net, b_reloc, b_touch_out, b_touch_in;
  DevBuf scal;                   // S_NUM u64
  int S_NUM = 0;
  PinnedBuf h_scal, h_batch, h_ctr;
  DevBuf ctr;                    // (k+1) * C_NUM u64
  DevBuf rec, rec_s, ord, cnt, off, runs, run_flags, seg, cls_scratch, cls_slot, cls_remaining, cls_flags;
  DevBuf work, scratch, scratch_idx, remaining, any_live;
  DevBuf sp_target, sp_n, sp_dims, sp_aold, sp_acc, sp_live, sp_changed, sp_remaining, swork;  // sparse recompute
  std::vector<DevBuf> dirty, changed, exp_base, exp_work;  // per layer [l]
  std::vector<uint32_t> n_dirty_host;
  DevBuf xbuf[2];
  DevBuf cub_tmp;
  DevBuf l2buf;
  uint64_t rec_cap = 0;

  KernelTimes kt;
  cudaEvent_t ev[64];
  bool ev_ready = false;
  DevBuf d_round;     // u32: the round id kernels read (graph-replay safe)
  PinnedBuf h_round;

  // One captured CUDA graph per (batch size, duplicate factor, profiling) and
  // allocation epoch: a round is then a single graph launch.
  struct RoundGraph {
    uint32_t B = 0, mult = 0;
    bool profile = false, emit_gate = false;
    uint64_t epoch = ~0ull;
    cudaGraphExec_t exec = nullptr;
    size_t kernel_nodes = 0;  // kernel launches per round (for gpu_launches)
  } graph;
  bool use_graphs = true;
  bool use_bulk = true;
  bool use_filter = true;  // k_expand_filter on layers >= 2 (SGNN_B200_FILTER=0 disables)
  bool use_sparse = true;  // sparse exposed-reset recompute (SGNN_B200_SPARSE=0 disables)
  bool use_fused_k8 = true;  // K8 fused into the last combination GEMM (SGNN_B200_FUSED_K8=0 disables)
  bool use_k1_pre = true;    // K1 with prefetched committed state and CTA counters (SGNN_B200_K1PRE=0 disables)
  uint32_t gemm_m_ab = 0;     // rows below which the exact GEMM takes 16x32 tiles (0: from the SM count; SGNN_B200_GEMM_MAB)
  bool use_k1_cluster = true;  // K1 as one 8-CTA cluster (SGNN_B200_K1CLUSTER=0: the one-CTA kernel)
  bool filter_minb4 = true;  // filter at 4 CTAs/SM when its code stage is off (SGNN_B200_FILTER_MINB4=0: 3)
  bool use_summary = true;   // filter's per-target scalar pre-test (SGNN_B200_SUMMARY=0 disables)
  bool use_tma = true;       // tensor-core mode operands by TMA (SGNN_B200_TMA=0: per-thread cp.async kernel)
  int tma_stages = 2;        // TF32 TMA ring depth (SGNN_B200_TMA_STAGES=3: one CTA per SM)
  // layers >= 2 run the pre-filtered expansion (k_expand_filter) unless seeds
  // are duplicated or rows exceed 1024 floats
  bool filtered_layer(int l, uint32_t mult) const {
    return l > 1 && l <= k && mult == 1 && use_filter && cpl_for(P[l] / 4) <= 8;
  }
  DevBuf touched;  // [N / 16] 2-bit run map of pre-filtered layers (RecSink::touch; cleared by k_collect_dirty)
  int bulk_grid = 4;       // most CTAs per SM of the bulk-copy recompute (SGNN_B200_BULK_GRID)
  int grid_mult = 4;       // blocks per SM of the grid-stride round kernels (SGNN_B200_GRID; 4 beat 8 and 2 at C2)
  // in-list entries per exposed-reset recompute work item (rows <= 1 KB / wider):
  // short items spread the few exposed targets of a round over more warps
  // (C2 p50 0.397 -> 0.363 ms against 128 / 64); rows > 256 floats (the
  // bulk-copy path) take 16-entry items (C2 recompute 45.6 -> 43.4 us/round
  // against 32; 64 cost 51 us; narrow rows: 16 / 64 entries 48.2 / 44.8 us vs
  // 45.5 at C3, kept at 32)
  uint32_t chunk_narrow = kChunkUpdate, chunk_wide = kChunkUpdate / 2;
  bool trace = false;

  // Sharding (owner-computes): this engine classifies, recomputes and combines
  // only targets in [shard_lo, shard_hi); graph and message tables m_1..m_k are
  // replicated and kept identical by the per-layer exchange; a_l and m_{k+1}
  // rows are valid on their owner only.
  bool sharded = false;
  int shard_rank = 0, shard_world = 1;
  uint32_t shard_lo = 0, shard_hi = 0;
  // Boundary-record pack buffers, alternating by layer: in a graph-launched
  // round segment l imports the peers' layer-l packs and then packs layer
  // l + 1, so that pack must not overwrite a buffer a slower peer is still
  // importing; the layer-l buffer is next written after the following
  // exchange's count all-gather, which every shard enters with its stream
  // (hence its imports) complete. Sized for every owned node being dirty and
  // shared with the peers once (they read them in place).
  DevBuf pack2[2];
  DevBuf& pack_for(int l) { return pack2[l & 1]; }
  std::vector<const void*> pack_peers[2];
  DevBuf pack_tab;  // [2][kMaxPeers] the peers' pack buffers (device-side exchange tables)
  // device-side exchange (exchange_kernels.cuh): this shard's mailbox, its
  // event sequence counter, every shard's mailbox
  DevBuf mbox, xseq;
  PeerBoxes boxes{};
  bool use_device_exchange = true;  // SGNN_B200_DEVICE_EXCHANGE=0: host collectives per layer
  std::shared_ptr<ShardTransport> transport;
  std::vector<uint32_t> bounds;  // shard r owns [bounds[r], bounds[r + 1]) (sharded engines)
  // every shard's allocation of m_l (l = 1..k): the rows other shards read
  std::vector<std::vector<const void*>> msg_peers;

  // Rows this engine holds of every table: its own range when sharded.
  uint32_t rows_owned() const { return shard_hi - shard_lo; }
  // Virtual base of an owned-rows allocation: row v (owned) at vb + v * pitch.
  template <typename T>
  T* vb(const DevBuf& b, uint32_t pitch) const {
    return b.as<T>() - static_cast<ptrdiff_t>(static_cast<size_t>(shard_lo) * pitch);
  }
  // Rows of every shard of a message table (dev_common.cuh RowTable).
  RowTable rows_of(const std::vector<const void*>& peers, const DevBuf& own, uint32_t pitch) const {
    RowTable t{};
    for (int r = 0; r < kMaxPeers; ++r) t.lo[r] = 0xFFFFFFFFu;
    t.lo[0] = 0;
    t.parts = 1;
    if (!sharded || peers.empty()) {
      t.base[0] = own.as<float>();
      return t;
    }
    t.parts = static_cast<uint32_t>(shard_world);
    for (int r = 0; r < shard_world; ++r) {
      t.lo[r] = bounds[r];
      t.base[r] = static_cast<const float*>(peers[r]) - static_cast<ptrdiff_t>(static_cast<size_t>(bounds[r]) * pitch);
    }
    return t;
  }
  RowTable msg_rows(int l) const {
    return rows_of(l < static_cast<int>(msg_peers.size()) ? msg_peers[l] : std::vector<const void*>{}, msg[l], P[l]);
  }
  // Every shard's device work queued so far is complete, then the host barrier.
  void shard_sync() {
    SGB_CUDA(cudaStreamSynchronize(st));
    transport->barrier();
  }
  int tc_mode = 0;  // K6 on tcgen05 (kind::tf32): 1 = 3xTF32 split, 2 = TF32; 0 = exact serial-k GEMM

  // Layers of a sharded round, after K1 passed the gate (no abort): per layer
  // the owned targets' event path, then (l < k) the boundary exchange — pack
  // this shard's dirty rows, import every shard's at global dirty positions,
  // plan the next layer's expansion over the global dirty list — and finally
  // the counter all-reduce and the commit (whose D2H then carries global
  // counters). Not graph-captured: the exchange needs host-known counts.
  // ---- graph-launched sharded round: the work between two exchanges is one
  // captured segment (segment 0 = K1 + layer 1 + pack; segment l = import +
  // plan + layer l+1 (+ pack); then the commit), so only the exchanges, the
  // import table upload and the counter all-reduce are issued per round from
  // the host.
  struct ShardGraphs {
    uint32_t B = ~0u, mult = 0;
    bool emit_gate = false;
    uint64_t epoch = ~0ull;
    std::vector<cudaGraphExec_t> seg;
    cudaGraphExec_t commit = nullptr;
    size_t kernel_nodes = 0;
    void reset() {
      for (auto g : seg)
        if (g) cudaGraphExecDestroy(g);
      seg.clear();
      if (commit) cudaGraphExecDestroy(commit);
      commit = nullptr;
      kernel_nodes = 0;
    }
  } shard_graphs;
  DevBuf d_imp;
  PinnedBuf h_imp;

  template <typename Fn>
  cudaGraphExec_t capture(Fn&& fn, size_t* kernel_nodes) {
    cudaGraph_t g = nullptr;
    SGB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    fn();
    SGB_CUDA(cudaStreamEndCapture(st, &g));
    size_t nn = 0;
    SGB_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) SGB_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      SGB_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t == cudaGraphNodeTypeKernel) ++*kernel_nodes;
    }
    cudaGraphExec_t exec = nullptr;
    SGB_CUDA(cudaGraphInstantiate(&exec, g, 0));
    SGB_CUDA(cudaGraphDestroy(g));
    return exec;
  }

  void enqueue_pack(int l) {
    pdl_launch(k_pack_rows, sms * 4, 256, 0, st, dirty[l].as<uint32_t>(), ds(L(l, L_NDIRTY)),
               oldslab[l + 1].as<float4>(), changed[l].as<uint32_t>(), P[l + 1], pack_for(l).as<uint8_t>());
    SGB_CUDA(cudaGetLastError());
  }

  // Import of every shard's layer-l records (read in place from the peers'
  // pack buffers through the device table d_imp) and the next layer's
  // expansion plan over the global dirty list.
  void enqueue_import(int l, uint32_t mult) {
    AdjView ov = out.view(pool.as<uint32_t>());
    pdl_launch(k_import_table, sms * 4, 256, 0, st, d_imp.as<unsigned long long>(), static_cast<uint32_t>(shard_world),
               P[l + 1], dirty[l].as<uint32_t>(), changed[l].as<uint32_t>(), oldslab[l + 1].as<float4>(),
               stamp[l + 1].as<uint32_t>(), slot[l + 1].as<uint32_t>(), d_round.as<uint32_t>(),
               ds(L(l, L_NDIRTY)));
    pdl_launch(k_plan_expand, sms * 2, 256, 0, st, dirty[l].as<uint32_t>(), ds(L(l, L_NDIRTY)), ov, mult,
                                           exp_base[l].as<uint64_t>(), exp_work[l + 1].as<ExpItem>(),
                                           ds(L(l + 1, L_EXPWORK)), ds(L(l + 1, L_CURSOR)),
                                           !filtered_layer(l + 1, mult));
    enqueue_source_thresholds(l, mult);
    SGB_CUDA(cudaGetLastError());
  }

  // The host side of the layer-l exchange: this shard's dirty count (its pack
  // is complete once the stream is), every shard's count, and the import table
  // naming the peers' pack buffers and global dirty offsets.
  void exchange_counts(int l) {
    unsigned long long n_local = 0;
    SGB_CUDA(cudaMemcpyAsync(h_imp.p, ds(L(l, L_NDIRTY)), 8, cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaStreamSynchronize(st));
    n_local = *h_imp.as<unsigned long long>();
    const std::vector<uint64_t> counts = transport->all_gather(n_local);
    unsigned long long* t = h_imp.as<unsigned long long>();
    uint64_t g0 = 0;
    for (int r = 0; r < shard_world; ++r) {
      t[3 * r] = reinterpret_cast<unsigned long long>(pack_peers[l & 1][r]);
      t[3 * r + 1] = counts[r];
      t[3 * r + 2] = g0;
      g0 += counts[r];
    }
    t[3 * shard_world] = g0;
    SGB_CUDA(cudaMemcpyAsync(d_imp.p, h_imp.p, 8ull * (3 * shard_world + 1), cudaMemcpyHostToDevice, st));
  }

  // Round counters summed over the shards (every shard reports the global line).
  void allreduce_counters() {
    const size_t n = static_cast<size_t>(k + 1) * C_NUM;
    SGB_CUDA(cudaMemcpyAsync(h_ctr.p, ctr.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaStreamSynchronize(st));
    transport->allreduce_sum(h_ctr.as<unsigned long long>(), n);
    SGB_CUDA(cudaMemcpyAsync(ctr.p, h_ctr.p, n * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
  }

  // Sharded rounds: the next layer's filter thresholds for every imported
  // dirty source of layer l (unsharded rounds write them in K8).
  void enqueue_source_thresholds(int l, uint32_t mult) {
    if (!(filtered_layer(l + 1, mult) && thrtab[l + 1].p)) return;
    auto* kt = is_max ? k_source_thresholds<true> : k_source_thresholds<false>;
    pdl_launch(kt, sms * 4, 256, 0, st, dirty[l].as<uint32_t>(), ds(L(l, L_NDIRTY)), oldslab[l + 1].as<float>(),
               msg_rows(l + 1), P[l + 1], d[l + 1], thrtab[l + 1].as<uint16_t>(), abstat[l + 1].as<float>());
  }

  void sharded_round_graphs(const char* d_ops, const uint32_t* d_src, const uint32_t* d_dst, uint32_t B,
                            uint32_t mult, RoundStats& stats) {
    ShardGraphs& G = shard_graphs;
    if (G.B != B || G.mult != mult || G.emit_gate != opts.emit_changed_only || G.epoch != alloc_epoch().load() ||
        G.seg.empty()) {
      G.reset();
      G.seg.push_back(capture([&] {
        enqueue_round(d_ops, d_src, d_dst, B, mult, false, false);
        enqueue_layer(1, mult);
        if (k > 1) enqueue_pack(1);
      }, &G.kernel_nodes));
      for (int l = 1; l < k; ++l)
        G.seg.push_back(capture([&] {
          enqueue_import(l, mult);
          enqueue_layer(l + 1, mult);
          if (l + 1 < k) enqueue_pack(l + 1);
        }, &G.kernel_nodes));
      G.commit = capture([&] { enqueue_commit(); }, &G.kernel_nodes);
      G.B = B;
      G.mult = mult;
      G.emit_gate = opts.emit_changed_only;
      G.epoch = alloc_epoch().load();
    }
    SGB_CUDA(cudaGraphLaunch(G.seg[0], st));
    for (int l = 1; l < k; ++l) {
      exchange_counts(l);
      SGB_CUDA(cudaGraphLaunch(G.seg[l], st));
    }
    allreduce_counters();
    if (opts.baseline_counters) {
      SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      SGB_CUDA(cudaStreamSynchronize(st));
      if (!hs(S_ABORT)) baseline_counters(stats);
    }
    SGB_CUDA(cudaGraphLaunch(G.commit, st));
    graph.kernel_nodes = G.kernel_nodes;
  }

  // The whole sharded round as ONE captured graph: the layer exchanges and
  // the counter all-reduce are publish / wait kernels over the peers'
  // mailboxes (exchange_kernels.cuh), so the host only launches the graph and
  // waits for the round's result copy.
  struct DeviceRoundGraph {
    uint32_t B = ~0u, mult = 0;
    bool emit_gate = false;
    uint64_t epoch = ~0ull;
    cudaGraphExec_t exec = nullptr;
    size_t kernel_nodes = 0;
  } dev_round;

  void enqueue_device_exchange(int l, uint32_t mult) {
    pdl_launch(k_publish_count, 1, 32, 0, st, mbox.as<uint64_t>(), xseq.as<uint64_t>(),
               static_cast<const unsigned long long*>(ds(L(l, L_NDIRTY))), static_cast<uint32_t>(l));
    pdl_launch(k_wait_counts, 1, 32, 0, st, boxes, static_cast<const uint64_t*>(xseq.as<uint64_t>()),
               static_cast<uint32_t>(l), static_cast<const unsigned long long*>(pack_tab.as<unsigned long long>() + (l & 1) * kMaxPeers),
               d_imp.as<unsigned long long>(), ds(S_XERR));
    SGB_CUDA(cudaGetLastError());
    enqueue_import(l, mult);
  }

  void sharded_round_device(const char* d_ops, const uint32_t* d_src, const uint32_t* d_dst, uint32_t B,
                            uint32_t mult) {
    DeviceRoundGraph& G = dev_round;
    if (!G.exec || G.B != B || G.mult != mult || G.emit_gate != opts.emit_changed_only ||
        G.epoch != alloc_epoch().load()) {
      if (G.exec) SGB_CUDA(cudaGraphExecDestroy(G.exec));
      G = {};
      const uint32_t n_ctr = static_cast<uint32_t>((k + 1) * C_NUM);
      G.exec = capture([&] {
        enqueue_round(d_ops, d_src, d_dst, B, mult, false, false);
        enqueue_layer(1, mult);
        for (int l = 1; l < k; ++l) {
          enqueue_pack(l);
          enqueue_device_exchange(l, mult);
          enqueue_layer(l + 1, mult);
        }
        pdl_launch(k_publish_counters, 1, 256, 0, st, mbox.as<uint64_t>(), xseq.as<uint64_t>(),
                   static_cast<const unsigned long long*>(ctr.as<unsigned long long>()), n_ctr);
        pdl_launch(k_reduce_counters, 1, 256, 0, st, boxes, static_cast<const uint64_t*>(xseq.as<uint64_t>()),
                   ctr.as<unsigned long long>(), n_ctr, ds(S_XERR));
        SGB_CUDA(cudaGetLastError());
        enqueue_commit();
      }, &G.kernel_nodes);
      G.B = B;
      G.mult = mult;
      G.emit_gate = opts.emit_changed_only;
      G.epoch = alloc_epoch().load();
    }
    // Every shard has finished its host-side preparation (allocations,
    // captures) before any shard's round can spin on a peer: in one process
    // the shards share a CUDA context, and an implicitly synchronising call
    // (cudaFree) of one shard would otherwise wait on another's spinning wait.
    transport->barrier();
    SGB_CUDA(cudaGraphLaunch(G.exec, st));
    graph.kernel_nodes = G.kernel_nodes;
  }

  // The same round enqueued kernel by kernel (profiling; SGNN_B200_GRAPHS=0).
  void sharded_layers(uint32_t mult, RoundStats& stats) {
    for (int l = 1; l <= k; ++l) {
      if (l > 1) {
        exchange_counts(l - 1);
        enqueue_import(l - 1, mult);
      }
      enqueue_layer(l, mult);
      if (l < k) enqueue_pack(l);
    }
    allreduce_counters();
    if (opts.baseline_counters) {
      SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      SGB_CUDA(cudaStreamSynchronize(st));
      if (!hs(S_ABORT)) baseline_counters(stats);
    }
    enqueue_commit();
  }

  ~Impl() {
    if (graph.exec) cudaGraphExecDestroy(graph.exec);
    if (dev_round.exec) cudaGraphExecDestroy(dev_round.exec);
    shard_graphs.reset();
    if (ev_ready)
      for (auto& e : ev) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_producer) cudaEventDestroy(ev_producer);
    if (ev_result) cudaEventDestroy(ev_result);
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }

  int L(int l, int f) const { return S_GLOBAL + (l - 1) * L_STRIDE + f; }
  // Batch sort keys are (src << b) | dst packed to 2b bits (graph_kernels.cuh
  // batch_key), b = bits(N).
  int key_bits() const { return std::min(32, num_bits(N)); }
  unsigned long long hs(int i) const { return h_scal.as<unsigned long long>()[i]; }
  unsigned long long* ds(int i) const { return scal.as<unsigned long long>() + i; }
  const unsigned long long* abort_flag() const { return ds(S_ABORT); }

  EdgeHash hash() const {
    return EdgeHash{h_slots.as<HashSlot>(), hcap - 1};
  }

  // (Re)builds the edge index from the committed adjacency, sized for the
  // live edges plus `headroom` future inserts at load factor <= 1/2.
  void build_hash(uint64_t headroom) {
    uint64_t want = 1024;
    while (want < 2 * (E + headroom)) want <<= 1;
    if (want != hcap) {
      hcap = want;
      h_slots.alloc_exact(hcap * sizeof(HashSlot));
    }
    SGB_CUDA(cudaMemsetAsync(h_slots.p, 0xFF, hcap * sizeof(HashSlot), st));  // every key empty
    AdjView ov = out.view(pool.as<uint32_t>()), iv = in.view(pool.as<uint32_t>());
    pdl_launch(k_hash_build_out, sms * 16, 256, 0, st, ov, N, hash());
    pdl_launch(k_hash_build_in, sms * 16, 256, 0, st, iv, N, hash());
    SGB_CUDA(cudaGetLastError());
    SGB_CUDA(cudaStreamSynchronize(st));
    h_tombs = 0;
  }

  // ---------------------------------------------------------------- setup

  void* cub_temp(size_t bytes) {
    cub_tmp.ensure(bytes);
    return cub_tmp.p;
  }

  const float* dev_weight(const std::vector<float>& host, uint32_t rows, uint32_t cols, uint32_t* ld) {
    auto it = wdev.find(host.data());
    if (it != wdev.end()) {
      *ld = wld[host.data()];
      return it->second.as<float>();
    }
    const uint32_t pitch = pitch_of(cols);
    std::vector<float> padded(static_cast<size_t>(rows) * pitch, 0.0f);
    for (uint32_t r = 0; r < rows; ++r)
      std::memcpy(&padded[static_cast<size_t>(r) * pitch], &host[static_cast<size_t>(r) * cols], cols * sizeof(float));
    DevBuf& b = wdev[host.data()];
    b.alloc_exact(padded.size() * sizeof(float));
    SGB_CUDA(copy_sync(st, b.p, padded.data(), padded.size() * sizeof(float), cudaMemcpyHostToDevice));
    wld[host.data()] = pitch;
    *ld = pitch;
    return b.as<float>();
  }

  // Weight matrix (rows = outputs N, cols = K) in the GEMM's panel layout:
  // Wp[ceil(N/32)][K][32] (zero-padded columns), one contiguous K-chunk per
  // 32-column panel (k_gemm_bulk).
  const float* dev_weight_t(const std::vector<float>& host, uint32_t rows, uint32_t cols, uint32_t* ld) {
    const void* key = reinterpret_cast<const char*>(host.data()) + 1;  // distinct from the row-major key
    auto it = wdev.find(key);
    if (it != wdev.end()) {
      *ld = wld[key];
      return it->second.as<float>();
    }
    const uint32_t panels = (rows + 31) / 32;
    std::vector<float> t(static_cast<size_t>(panels) * cols * 32, 0.0f);
    for (uint32_t r = 0; r < rows; ++r)
      for (uint32_t c = 0; c < cols; ++c)
        t[(static_cast<size_t>(r / 32) * cols + c) * 32 + (r % 32)] = host[static_cast<size_t>(r) * cols + c];
    DevBuf& b = wdev[key];
    b.alloc_exact(std::max<size_t>(t.size(), 4) * sizeof(float));
    if (!t.empty()) SGB_CUDA(copy_sync(st, b.p, t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice));
    wld[key] = cols;
    *ld = cols;
    return b.as<float>();
  }

  // Uploads every weight of every program once, so no transfer happens inside
  // a round.
  void upload_weights() {
    auto up = [&](const std::vector<ProgramOp>& prog) {
      for (const ProgramOp& op : prog) {
        uint32_t ld;
        if (op.w) dev_weight_t(op.w->data, op.w->rows, op.w->cols, &ld);
        if (op.bias) dev_weight(*op.bias, 1, static_cast<uint32_t>(op.bias->size()), &ld);
      }
    };
    up(model->prefix());
    for (int p = 0; p < k; ++p) up(model->program(p));
  }

  void upload_graph(const HostGraph& g) {
    const uint32_t n = N;
    for (int dir = 0; dir < 2; ++dir) {
      Adj& a = dir == 0 ? out : in;
      a.off.alloc_exact(sizeof(uint64_t) * n);
      for (DevBuf* b : {&a.len, &a.cap, &a.n_new, &a.n_del, &a.touch, &a.reloc}) {
        b->alloc_exact(sizeof(uint32_t) * n);
        SGB_CUDA(memset_sync(st, b->p, 0, sizeof(uint32_t) * n));
      }
    }
    // slab layout: per vertex capacity = deg + deg/8 + 4, both directions in one pool
    std::vector<uint64_t> off_o(n), off_i(n);
    std::vector<uint32_t> len_o(n), len_i(n), cap_o(n), cap_i(n);
    uint64_t cursor = 0;
    auto cap_of = [](uint64_t deg) { return static_cast<uint32_t>(((deg + deg / 8 + 4) + 7) & ~7ull); };
    for (uint32_t v = 0; v < n; ++v) {
      len_o[v] = static_cast<uint32_t>(g.out(v).size());
      cap_o[v] = cap_of(len_o[v]);
      off_o[v] = cursor;
      cursor += cap_o[v];
      out_entries += len_o[v];
    }
    for (uint32_t v = 0; v < n; ++v) {
      len_i[v] = static_cast<uint32_t>(g.in(v).size());
      cap_i[v] = cap_of(len_i[v]);
      off_i[v] = cursor;
      cursor += cap_i[v];
      in_entries += len_i[v];
    }
    const uint64_t used = cursor;
    pool_cap = used + used / 4 + (1u << 20);
    pool.alloc_exact(pool_cap * sizeof(uint32_t));
    {
      std::vector<uint32_t> host(used, 0);
      for (uint32_t v = 0; v < n; ++v) {
        std::copy(g.out(v).begin(), g.out(v).end(), host.begin() + static_cast<long>(off_o[v]));
        std::copy(g.in(v).begin(), g.in(v).end(), host.begin() + static_cast<long>(off_i[v]));
      }
      SGB_CUDA(copy_sync(st, pool.p, host.data(), used * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    SGB_CUDA(copy_sync(st, out.off.p, off_o.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
    SGB_CUDA(copy_sync(st, in.off.p, off_i.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
    SGB_CUDA(copy_sync(st, out.len.p, len_o.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SGB_CUDA(copy_sync(st, in.len.p, len_i.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SGB_CUDA(copy_sync(st, out.cap.p, cap_o.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SGB_CUDA(copy_sync(st, in.cap.p, cap_i.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    pool_top.alloc_exact(sizeof(uint64_t));
    SGB_CUDA(copy_sync(st, pool_top.p, &used, sizeof(uint64_t), cudaMemcpyHostToDevice));
    E = g.num_edges();
    build_hash(E / 4 + (1u << 16));
    for (DevBuf* b : {&del_head_out, &del_head_in}) {
      b->alloc_exact(sizeof(uint32_t) * n);
      SGB_CUDA(memset_sync(st, b->p, 0xFF, sizeof(uint32_t) * n));
    }
  }

  void grow_pool(uint64_t need_entries, uint64_t top) {
    uint64_t ncap = std::max<uint64_t>(pool_cap * 2, top + need_entries + (1u << 20));
    DevBuf np;
    np.alloc_exact(ncap * sizeof(uint32_t));
    SGB_CUDA(cudaMemcpyAsync(np.p, pool.p, top * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    SGB_CUDA(cudaStreamSynchronize(st));
    std::swap(pool.p, np.p);
    std::swap(pool.cap, np.cap);
    pool_cap = ncap;
  }

  // Provisions every round buffer from host-side bounds so the round itself
  // needs no host knowledge of data-dependent sizes.
  void ensure_capacity(uint32_t B, uint32_t mult) {
    const uint64_t Bq = std::max<uint32_t>(B, 1);
    b_src.ensure(Bq * 9);
    b_keys.ensure(Bq * 8);
    b_vals.ensure(Bq * 4);
    b_keys_s.ensure(Bq * 8);
    b_vals_s.ensure(Bq * 4);
    b_net.ensure(Bq * 8);
    b_reloc.ensure(Bq * 8);
    b_touch_out.ensure(Bq * 4);
    b_touch_in.ensure(Bq * 4);
    del_pos.ensure(Bq * 8);
    del_next.ensure(Bq * 8);
    // records of one layer: seeds + every out-list entry (+ this round's NEW) + SELF
    const uint64_t rc = (out_entries + 2 * Bq) * mult + N + 16;
    if (rc > rec_cap) {
      rec_cap = rc + rc / 4;
      rec.ensure(rec_cap * 8);
      rec_s.ensure(rec_cap * 8);
      ord.ensure(rec_cap * 4);
      seg.ensure((N + rec_cap / kSeg + 2) * 16);
      const uint64_t multi = std::min<uint64_t>(N, rec_cap / (kSeg + 1) + 1);
      cls_scratch.ensure(multi * 2 * maxP * sizeof(int));
    }
    const uint64_t in_b = in_entries + Bq;
    const uint32_t min_chunk = std::min(chunk_narrow, chunk_wide);
    work.ensure((N + in_b / min_chunk + 16) * 8);
    swork.ensure((N + in_b / kSparseChunk + 16) * 8);
    scratch.ensure(std::min<uint64_t>(N, in_b / min_chunk + 1) * maxP * sizeof(int));
    const uint64_t out_b = out_entries + Bq;
    for (int l = 1; l <= k; ++l) exp_work[l].ensure((N + out_b / kExpandChunk + 16) * sizeof(ExpItem));
  }

  // Every allocation a round needs, done before it is enqueued or captured.
  void prepare_round(uint32_t B, uint32_t mult) {
    ensure_capacity(B, mult);
    if (B) {
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, b_keys.as<uint64_t>(), b_keys_s.as<uint64_t>(),
                                      b_vals.as<uint32_t>(), b_vals_s.as<uint32_t>(), static_cast<int>(B), 0,
                                      2 * key_bits(), st);
      cub_tmp.ensure(tb);
    }
    for (int l = 1; l <= k; ++l) {
      uint32_t maxd = d[l];
      for (const ProgramOp& op : model->program(l - 1)) maxd = std::max(maxd, op.out_dim);
      for (auto& b : xbuf) b.ensure(static_cast<size_t>(N) * pitch_of(maxd) * sizeof(float));
    }
  }

  // ------------------------------------------------------- combination

  // Row pitch of the staging buffers of `prog` run on d_in-wide rows.
  static uint32_t program_pitch(const std::vector<ProgramOp>& prog, uint32_t d_in) {
    uint32_t maxd = d_in;
    for (const ProgramOp& op : prog) maxd = std::max(maxd, op.out_dim);
    return pitch_of(maxd);
  }

  // A 2-D fp32 tensor map (rows x cols, row pitch in bytes), 128-byte swizzle,
  // zero fill out of bounds (cuTensorMapEncodeTiled through the runtime's
  // driver entry point: no link-time libcuda dependency).
  static CUtensorMap tensor_map(const float* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                                uint32_t box_cols, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q{};
      SGB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess) fail(Errc::unknown, "cuTensorMapEncodeTiled is unavailable");
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    CUtensorMap m{};
    const cuuint64_t dims[2] = {cols, std::max<uint64_t>(rows, 1)};
    const cuuint64_t strides[1] = {pitch_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(Errc::unknown, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
  }

  // K6 tensor-core mode (combine_tc.cuh): W row-major, rows padded to pitch.
  // x_rows: rows of the table x addresses (the tensor map's extent).
  void launch_gemm_tc(RowSrc x, const float* w, uint32_t ld, const float* b, RowSrc r, bool res, RowDst y,
                      const unsigned long long* M_dev, uint32_t M_host, uint32_t M_cap, uint32_t Nout, uint32_t K,
                      bool relu, const unsigned long long* abort, uint32_t x_rows) {
    if (x.pitch % 4 || (res && r.pitch % 4) || ld % 4) fail(Errc::unknown, "gemm_tc: bad operand layout");
    const uint32_t nt = tc_ntile(Nout);
    dim3 grid((std::max<uint32_t>(M_dev ? M_cap : M_host, 1) + kTcM - 1) / kTcM, (Nout + nt - 1) / nt);
    if (use_tma && shard_lo == 0) {
      // operands by TMA: W tiles (32 x nt), activation rows by gather4 (or tiles when contiguous)
      const CUtensorMap ma = tensor_map(x.base, x.pitch, x_rows, x.pitch * 4ull, kTcK, x.ids ? 1u : kTcM);
      const CUtensorMap mb = tensor_map(w, ld, Nout, ld * 4ull, kTcK, nt);
      if (tc_mode == 1)
        pdl_launch(k_gemm_tma<true, 2>, grid, kTcThreads, tma_smem_bytes(nt, true, 2), st, ma, mb, x, b, r, res, y,
                   M_dev, M_host, Nout, K, relu, abort);
      else if (tma_stages == 3)
        pdl_launch(k_gemm_tma<false, 3>, grid, kTcThreads, tma_smem_bytes(nt, false, 3), st, ma, mb, x, b, r, res, y,
                   M_dev, M_host, Nout, K, relu, abort);
      else
        pdl_launch(k_gemm_tma<false, 2>, grid, kTcThreads, tma_smem_bytes(nt, false, 2), st, ma, mb, x, b, r, res, y,
                   M_dev, M_host, Nout, K, relu, abort);
      SGB_CUDA(cudaGetLastError());
      return;
    }
    if (tc_mode == 1)
      pdl_launch(k_gemm_tc<true>, grid, kTcThreads, tc_smem_bytes(nt, true), st, x, w, ld, b, r, res, y, M_dev, M_host, Nout,
                                                                         K, relu, abort);
    else
      pdl_launch(k_gemm_tc<false>, grid, kTcThreads, tc_smem_bytes(nt, false), st, x, w, ld, b, r, res, y, M_dev, M_host,
                                                                           Nout, K, relu, abort);
    SGB_CUDA(cudaGetLastError());
  }

  void launch_gemm(RowSrc x, const float* w, uint32_t ld, const float* b, RowSrc r, bool res, RowDst y,
                   const unsigned long long* M_dev, uint32_t M_host, uint32_t Nout, uint32_t K, bool relu,
                   const unsigned long long* abort, const WriteBack& wb = WriteBack{}) {
    // Tile shape by row count (picked on the device, one launch): every output
    // is a serial K-long dot product (no split-K), so small dirty sets need
    // small tiles to cover the SMs.
    //   M <  m_ab : 16x32 tiles     M < m_bc : 32x32     otherwise : 64x64
    if (x.pitch % 4 || (res && r.pitch % 4) || y.pitch % 4 || ld != K) fail(Errc::unknown, "gemm: bad operand layout");
    const uint32_t nt32 = (Nout + 31) / 32, nt64 = (Nout + 63) / 64, s = static_cast<uint32_t>(sms);
    // (forcing any single shape measured slower at C2: combine 56 us/round vs 67 / 67 / 99)
    const uint32_t m_ab = gemm_m_ab ? gemm_m_ab : 32u * ((s + nt32 - 1) / nt32);
    const uint32_t m_bc = 64u * ((2 * s + nt64 - 1) / nt64);
    pdl_launch(k_gemm_bulk, static_cast<unsigned>(2 * sms), kGemmThreads, gemm_bulk_smem(), st,  // 2 CTAs/SM fit
        x, w, b, r, res, y, M_dev, M_host, m_ab, m_bc, Nout, K, relu, wb, abort);
    SGB_CUDA(cudaGetLastError());
  }

  // Runs `prog` on the rows of x0 (aggregates) with self = the nodes' own layer
  // messages; M rows from the device (M_dev) or the host. Returns the result
  // rows (a dense buffer, pitch *out_pitch, width *out_dim).
  // With `wb`, the program's last op, when it is an exact GEMM (Linear or
  // SageSelf, ReLU fused), writes its rows through the fused write-back
  // (combine_kernels.cuh WriteBack) instead of a staging buffer; *fused says
  // whether it did (otherwise the caller runs K8 on the returned rows).
  const float* run_program(const std::vector<ProgramOp>& prog, RowSrc x0, RowSrc self,
                           const unsigned long long* M_dev, uint32_t M_host, uint32_t M_cap, uint32_t d_in,
                           uint32_t* out_pitch, uint32_t* out_dim, const unsigned long long* abort,
                           const WriteBack* wb = nullptr, bool* fused = nullptr) {
    if (fused) *fused = false;
    const uint32_t x_rows = rows_owned();  // rows of the tables x0 / self address (this engine's own)
    const uint32_t bp = program_pitch(prog, d_in);
    for (auto& b : xbuf) b.ensure(static_cast<size_t>(M_cap) * bp * sizeof(float));
    RowSrc cur = x0;
    uint32_t cd = d_in;
    int which = 0;
    bool in_buf = false;

    auto dst_of = [&](int w) { return RowDst{xbuf[w].as<float>(), nullptr, 0, bp}; };
    auto src_of = [&](int w) { return RowSrc{xbuf[w].as<float>(), nullptr, 0, bp}; };
    const unsigned ew_grid = static_cast<unsigned>(sms * 8);
    for (size_t i = 0; i < prog.size(); ++i) {
      const ProgramOp& op = prog[i];
      const bool fuse_relu = i + 1 < prog.size() && prog[i + 1].kind == ProgramOp::Relu &&
                             (op.kind == ProgramOp::Linear || op.kind == ProgramOp::SageSelf);
      const bool last = i + (fuse_relu ? 1 : 0) + 1 == prog.size();
      const bool wb_here = wb && fused && last && !tc_mode &&
                           (op.kind == ProgramOp::Linear || op.kind == ProgramOp::SageSelf);
      const WriteBack wbv = wb_here ? *wb : WriteBack{};
      if (wb_here) *fused = true;
      switch (op.kind) {
        case ProgramOp::Linear: {
          uint32_t ld = 0, bld = 0;
          const float* b = op.bias ? dev_weight(*op.bias, 1, static_cast<uint32_t>(op.bias->size()), &bld) : nullptr;
          if (tc_mode) {
            const float* w = dev_weight(op.w->data, op.w->rows, op.w->cols, &ld);
            launch_gemm_tc(cur, w, ld, b, RowSrc{}, false, dst_of(which), M_dev, M_host, M_cap, op.out_dim, cd,
                           fuse_relu, abort, in_buf ? M_cap : x_rows);
          } else {
            const float* w = dev_weight_t(op.w->data, op.w->rows, op.w->cols, &ld);
            launch_gemm(cur, w, ld, b, RowSrc{}, false, dst_of(which), M_dev, M_host, op.out_dim, cd, fuse_relu,
                        abort, wbv);
          }
          break;
        }
        case ProgramOp::SageSelf: {
          uint32_t ld = 0;
          if (tc_mode) {
            const float* w = dev_weight(op.w->data, op.w->rows, op.w->cols, &ld);
            launch_gemm_tc(self, w, ld, nullptr, cur, true, dst_of(which), M_dev, M_host, M_cap, op.out_dim,
                           op.w->cols, fuse_relu, abort, x_rows);
          } else {
            const float* w = dev_weight_t(op.w->data, op.w->rows, op.w->cols, &ld);
            launch_gemm(self, w, ld, nullptr, cur, true, dst_of(which), M_dev, M_host, op.out_dim, op.w->cols,
                        fuse_relu, abort, wbv);
          }
          break;
        }
        case ProgramOp::GinSelf:
          pdl_launch(k_gin_self, ew_grid, 256, 0, st, cur, self, op.gin_scale, dst_of(which), M_dev, M_host, cd, abort);
          break;
        case ProgramOp::Relu:
          pdl_launch(k_relu_rows, ew_grid, 256, 0, st, cur, dst_of(which), M_dev, M_host, cd, abort);
          break;
      }
      SGB_CUDA(cudaGetLastError());
      cd = op.out_dim;
      cur = src_of(which);
      which ^= 1;
      in_buf = true;
      if (fuse_relu) ++i;
    }
    if (!in_buf) {
      pdl_launch(k_copy_rows, ew_grid, 256, 0, st, cur, dst_of(which), M_dev, M_host, cd, abort);
      SGB_CUDA(cudaGetLastError());
      cur = src_of(which);
    }
    *out_pitch = bp;
    *out_dim = cd;
    return cur.base;
  }

  // ------------------------------------------------------ full inference

  template <bool IsMax, int CPL>
  void launch_bulk(const AggArgs& A, uint32_t V) {
    const uint32_t rowbytes = V * 16;
    const uint32_t ring = std::max<uint32_t>(2, std::min<uint32_t>(32, (24u << 10) / rowbytes));
    const uint32_t per_warp = ((ring * rowbytes + ring * 8 + A.chunk * 4) + 127) & ~127u;
    const size_t smem = 4ull * per_warp;
    // one wave: the CTAs that fit beside each other (1 KB reserved per CTA);
    // a second wave of ~98 KB CTAs only added launch latency to rounds with a
    // few dozen items
    const int per_sm = std::max(1, smem_per_sm / static_cast<int>(smem + 1024));
    pdl_launch(k_aggregate_bulk<IsMax, CPL>, sms * std::min(per_sm, bulk_grid), 128, smem, st, A, ring);
  }

  // Opt-in shared memory for the bulk-copy kernels (set outside any capture).
  template <bool IsMax, int... C>
  void bulk_attrs(std::integer_sequence<int, C...>, int smem) {
    const cudaError_t errs[] = {
        cudaFuncSetAttribute(k_aggregate_bulk<IsMax, C + 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)...};
    for (cudaError_t e : errs) SGB_CUDA(e);
  }
  void set_kernel_attributes() {
    SGB_CUDA(cudaFuncSetAttribute(k_gemm_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(gemm_bulk_smem())));
    SGB_CUDA(cudaFuncSetAttribute(k_batch_group, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(batch_group_smem(kGroupCap))));
    SGB_CUDA(cudaFuncSetAttribute(k_batch_group_pre, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(batch_group_pre_smem(kGroupCapPre))));
    SGB_CUDA(cudaFuncSetAttribute(k_batch_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(batch_cluster_smem(kGroupCapCluster))));
    SGB_CUDA(cudaFuncSetAttribute(k_gemm_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tc_smem_bytes(256, true))));
    SGB_CUDA(cudaFuncSetAttribute(k_gemm_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tc_smem_bytes(256, false))));
    SGB_CUDA(cudaFuncSetAttribute(k_gemm_tma<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tma_smem_bytes(256, true, 2))));
    SGB_CUDA(cudaFuncSetAttribute(k_gemm_tma<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tma_smem_bytes(256, false, 2))));
    SGB_CUDA(cudaFuncSetAttribute(k_gemm_tma<false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tma_smem_bytes(256, false, 3))));
    const int smem = 200 * 1024;
    bulk_attrs<true>(std::make_integer_sequence<int, 13>{}, smem);
    bulk_attrs<false>(std::make_integer_sequence<int, 13>{}, smem);
  }

  template <bool IsMax>
  void launch_aggregate(const AggArgs& A, uint32_t V) {
    const unsigned grid = static_cast<unsigned>(sms * grid_mult);
    if (V * 16 >= 2048 && use_bulk) {  // wide rows (>= 2 KB): stage through the bulk-copy engine
      // exact float4 columns per lane (ceil(V/32), 4..16): no dead predicated columns
      switch ((V + 31) / 32) {
        case 4: launch_bulk<IsMax, 4>(A, V); break;
        case 5: launch_bulk<IsMax, 5>(A, V); break;
        case 6: launch_bulk<IsMax, 6>(A, V); break;
        case 7: launch_bulk<IsMax, 7>(A, V); break;
        case 8: launch_bulk<IsMax, 8>(A, V); break;
        case 9: launch_bulk<IsMax, 9>(A, V); break;
        case 10: launch_bulk<IsMax, 10>(A, V); break;
        case 11: launch_bulk<IsMax, 11>(A, V); break;
        case 12: launch_bulk<IsMax, 12>(A, V); break;
        case 13: launch_bulk<IsMax, 13>(A, V); break;
        case 14: launch_bulk<IsMax, 14>(A, V); break;
        case 15: launch_bulk<IsMax, 15>(A, V); break;
        default: launch_bulk<IsMax, 16>(A, V); break;
      }
      SGB_CUDA(cudaGetLastError());
      return;
    }
    switch (cpl_for(V)) {
      case 1: pdl_launch(k_aggregate<IsMax, 1>, grid, 256, 0, st, A); break;
      case 2: pdl_launch(k_aggregate<IsMax, 2>, grid, 256, 0, st, A); break;
      case 4: pdl_launch(k_aggregate<IsMax, 4>, grid, 256, 0, st, A); break;
      case 8: pdl_launch(k_aggregate<IsMax, 8>, grid, 256, 0, st, A); break;
      default: pdl_launch(k_aggregate<IsMax, 16>, grid, 256, 0, st, A); break;
    }
    SGB_CUDA(cudaGetLastError());
  }

  // Whole-graph inference into the given tables (init_full_inference,
  // checkpoint.cpp:105-145 / baseline::full_inference, baseline.cpp:67-99).
  // Whole-graph inference into the given tables (init_full_inference,
  // checkpoint.cpp:105-145 / baseline::full_inference, baseline.cpp:67-99).
  // A sharded engine computes its own rows of every layer, reading the other
  // shards' rows of m_l through m_peers[l]; every shard runs it together (a
  // barrier after each layer's rows are written).
  void full_inference(std::vector<DevBuf>& m_out, std::vector<DevBuf>& a_out,
                      const std::vector<std::vector<const void*>>& m_peers) {
    layer1_messages(m_out[1]);
    if (sharded) transport->barrier();  // every shard's m_1 rows are in place
    InferPlan plan = infer_plan();
    for (int l = 1; l <= k; ++l) {
      infer_layer(plan, l, rows_of(l < static_cast<int>(m_peers.size()) ? m_peers[l] : std::vector<const void*>{},
                                   m_out[l], P[l]),
                  vb<float>(m_out[l], P[l]), vb<float>(a_out[l], P[l]), vb<float>(m_out[l + 1], P[l + 1]));
      SGB_CUDA(cudaStreamSynchronize(st));
      if (sharded) transport->barrier();  // layer l + 1 reads every shard's m_{l+1} rows
    }
  }

  // m_1 of the owned rows: the features, or the prefix program run on them
  // (run_prefix, model.cpp:271-284).
  void layer1_messages(DevBuf& m1) {
    const uint32_t lo = shard_lo, n = rows_owned();
    const uint32_t rows_chunk = std::max<uint32_t>(1, std::min<uint32_t>(n, 1u << 16));
    const uint32_t fp = pitch_of(F);
    // without a prefix the features go straight into m_1 (no staging copy)
    DevBuf fdev;
    float* dst = model->has_prefix() ? nullptr : m1.as<float>();
    if (!dst) {
      fdev.alloc_exact(std::max<size_t>(static_cast<size_t>(n) * fp * sizeof(float), 256));
      dst = fdev.as<float>();
    }
    std::vector<float> padded;
    const size_t rows_per = std::max<size_t>(1, (64u << 20) / (fp * sizeof(float)));
    for (size_t r0 = 0; r0 < n; r0 += rows_per) {
      const size_t r1 = std::min<size_t>(n, r0 + rows_per);
      padded.assign((r1 - r0) * fp, 0.0f);
      for (size_t r = r0; r < r1; ++r) std::memcpy(&padded[(r - r0) * fp], &features[(lo + r) * F], F * sizeof(float));
      SGB_CUDA(copy_sync(st, dst + r0 * fp, padded.data(), padded.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    if (model->has_prefix()) {
      for (uint32_t r0 = 0; r0 < n; r0 += rows_chunk) {
        const uint32_t M = std::min(rows_chunk, n - r0);
        uint32_t op_pitch = 0, od = 0;
        RowSrc x0{fdev.as<float>(), nullptr, r0, fp};
        const float* res = run_program(model->prefix(), x0, x0, nullptr, M, rows_chunk, F, &op_pitch, &od, nullptr);
        pdl_launch(k_copy_rows, sms * 8, 256, 0, st, RowSrc{res, nullptr, 0, op_pitch},
                                             RowDst{vb<float>(m1, P[1]), nullptr, lo + r0, P[1]}, nullptr,
                                             M, od, nullptr);
        SGB_CUDA(cudaGetLastError());
      }
    }
    SGB_CUDA(cudaStreamSynchronize(st));
  }

  // Work items of the whole-graph aggregation over the owned targets (the same
  // for every layer: in-list chunks of kChunk entries).
  struct InferPlan {
    DevBuf nch, nscan, nwork, sidx, rem, alive, scr, nscr, fetch;
    uint64_t total_items = 0, multi = 0;
  };
  InferPlan infer_plan() {
    const uint32_t lo = shard_lo, n = rows_owned();
    InferPlan pl;
    pl.nch.alloc_exact(sizeof(uint64_t) * std::max<uint32_t>(n, 1));
    pl.nscan.alloc_exact(sizeof(uint64_t) * std::max<uint32_t>(n, 1));
    {
      std::vector<uint32_t> lens(n);
      if (n) SGB_CUDA(copy_sync(st, lens.data(), in.len.as<uint32_t>() + lo, n * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost));
      for (uint32_t v = 0; v < n; ++v) {
        const uint64_t c = lens[v] == 0 ? 1 : (lens[v] + kChunk - 1) / kChunk;
        pl.total_items += c;
        pl.multi += c > 1;
      }
    }
    pl.nwork.alloc_exact(sizeof(uint64_t) * std::max<uint64_t>(pl.total_items, 1));
    pl.sidx.alloc_exact(sizeof(uint32_t) * N);
    pl.rem.alloc_exact(sizeof(uint32_t) * N);
    pl.alive.alloc_exact(sizeof(uint32_t) * N);
    pl.nscr.alloc_exact(sizeof(unsigned long long));
    pl.scr.alloc_exact(std::max<uint64_t>(1, pl.multi) * maxP * sizeof(int));
    pl.fetch.alloc_exact(sizeof(unsigned long long));
    SGB_CUDA(cudaMemsetAsync(pl.fetch.p, 0, sizeof(unsigned long long), st));
    if (n) {
      pdl_launch(k_node_chunks, grid_for(n), 256, 0, st, in.len.as<uint32_t>(), lo, n, kChunk, pl.nch.as<uint64_t>());
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, pl.nch.as<uint64_t>(), pl.nscan.as<uint64_t>(), n, st);
      cub::DeviceScan::ExclusiveSum(cub_temp(tb), tb, pl.nch.as<uint64_t>(), pl.nscan.as<uint64_t>(), n, st);
    }
    return pl;
  }

  // One whole-graph layer over the owned targets: a_l from the rows of m_in
  // (every shard's), then the layer's program with self rows `self_vb`, into
  // the virtual bases a_vb (pitch P[l]) and m_next_vb (pitch P[l + 1]).
  void infer_layer(InferPlan& pl, int l, const RowTable& m_in, const float* self_vb, float* a_vb, float* m_next_vb) {
    const uint32_t lo = shard_lo, n = rows_owned();
    if (!n) return;
    const uint32_t rows_chunk = std::max<uint32_t>(1, std::min<uint32_t>(n, 1u << 16));
    SGB_CUDA(cudaMemsetAsync(pl.nscr.p, 0, sizeof(unsigned long long), st));
    pdl_launch(k_node_work, grid_for(n), 256, 0, st, pl.nscan.as<uint64_t>(), pl.nch.as<uint64_t>(), lo, n,
               pl.nwork.as<uint64_t>(), pl.sidx.as<uint32_t>(), pl.rem.as<uint32_t>(), pl.alive.as<uint32_t>(),
               pl.nscr.as<unsigned long long>());
    if (pl.multi)
      pdl_launch(k_fill_int, sms * 4, 256, 0, st, pl.scr.as<int>(), pl.multi * P[l], is_max ? INT_MIN : INT_MAX);
    AggArgs A{};
    A.work = pl.nwork.as<uint64_t>();
    A.n_work = nullptr;
    A.n_work_host = pl.total_items;
    A.update = false;
    A.scratch_idx = pl.sidx.as<uint32_t>();
    A.remaining = pl.rem.as<uint32_t>();
    A.any_live = pl.alive.as<uint32_t>();
    A.scratch = pl.scr.as<int>();
    A.in_off = in.off.as<uint64_t>();
    A.in_len = in.len.as<uint32_t>();
    A.in_ent = pool.as<uint32_t>();
    A.msg = m_in;
    A.agg = reinterpret_cast<float4*>(a_vb);
    A.V = P[l] / 4;
    A.d = d[l];
    A.chunk = kChunk;
    A.fetch_ctr = pl.fetch.as<unsigned long long>();
    if (is_max) launch_aggregate<true>(A, A.V); else launch_aggregate<false>(A, A.V);
    for (uint32_t r0 = lo; r0 < lo + n; r0 += rows_chunk) {
      const uint32_t M = std::min(rows_chunk, lo + n - r0);
      uint32_t op_pitch = 0, od = 0;
      RowSrc x0{a_vb, nullptr, r0, P[l]};
      RowSrc self{self_vb, nullptr, r0, P[l]};
      const float* res = run_program(model->program(l - 1), x0, self, nullptr, M, rows_chunk, d[l], &op_pitch, &od,
                                     nullptr);
      pdl_launch(k_copy_rows, sms * 8, 256, 0, st, RowSrc{res, nullptr, 0, op_pitch},
                 RowDst{m_next_vb, nullptr, r0, P[l + 1]}, nullptr, M, od, nullptr);
      SGB_CUDA(cudaGetLastError());
    }
  }

  // Recomputes every alpha bound from a_l (after a whole-table rewrite).
  void refresh_abound() {
    for (int l = 2; l <= k && l < static_cast<int>(cmin.size()); ++l) {
      if (!cmin[l].p) continue;
      const size_t rows = rows_owned();
      const size_t n = rows * P[l];  // the allocations hold the owned rows
      DevBuf& colr = abcolr;
      pdl_launch(k_fill_int, 1, 256, 0, st, colr.as<int>(), P[l], INT_MAX);
      pdl_launch(k_fill_int, 1, 256, 0, st, colr.as<int>() + P[l], P[l], INT_MIN);
      if (is_max)
        pdl_launch(k_abound_range<true>, sms * 8, 256, 0, st, agg[l].as<float>(), n, P[l], colr.as<int>());
      else
        pdl_launch(k_abound_range<false>, sms * 8, 256, 0, st, agg[l].as<float>(), n, P[l], colr.as<int>());
      pdl_launch(k_abound_stats, 1, 256, 0, st, colr.as<int>(), P[l], abstat[l].as<float>());
      uint16_t* codes = abound[l].p ? abound[l].as<uint16_t>() : nullptr;
      if (is_max)
        pdl_launch(k_summarise_all<true>, sms * 8, 256, 0, st, agg[l].as<float>(), codes, cmin[l].as<float>(),
                   abstat[l].as<float>(), rows, P[l], d[l]);
      else
        pdl_launch(k_summarise_all<false>, sms * 8, 256, 0, st, agg[l].as<float>(), codes, cmin[l].as<float>(),
                   abstat[l].as<float>(), rows, P[l], d[l]);
      SGB_CUDA(cudaGetLastError());
    }
  }

  void alloc_tables(std::vector<DevBuf>& m, std::vector<DevBuf>& a) {
    m.clear();
    a.clear();
    m.resize(k + 2);
    a.resize(k + 1);
    // a sharded engine holds its own rows only (>= 256 bytes so every shard
    // has an allocation to share)
    const size_t rows = rows_owned();
    for (int l = 1; l <= k + 1; ++l) {
      const size_t bytes = std::max<size_t>(rows * P[l] * sizeof(float), 256);
      m[l].alloc_exact(bytes);
      SGB_CUDA(memset_sync(st, m[l].p, 0, bytes));
    }
    for (int l = 1; l <= k; ++l) {
      const size_t bytes = std::max<size_t>(rows * P[l] * sizeof(float), 256);
      a[l].alloc_exact(bytes);
      SGB_CUDA(memset_sync(st, a[l].p, 0, bytes));
    }
  }

  // Collective: every shard's allocation of m_1..m_k (the rows other shards read).
  std::vector<std::vector<const void*>> share_messages(const std::vector<DevBuf>& m) {
    std::vector<std::vector<const void*>> peers(k + 1);
    if (!sharded) return peers;
    for (int l = 1; l <= k; ++l) peers[l] = transport->share_device(m[l].p);
    return peers;
  }
  void unshare_messages(const std::vector<std::vector<const void*>>& peers) {
    if (!sharded) return;
    for (const auto& p : peers)
      if (!p.empty()) transport->unshare_device(p);
  }

  void load_checkpoints(const std::string& dir) {
    // CheckpointStore::load (checkpoint.cpp:166-203)
    std::ifstream manifest(dir + "/checkpoints.txt");
    if (!manifest) fail(Errc::io, "cannot open checkpoint manifest in " + dir);
    uint32_t nodes = 0;
    int layers = 0;
    size_t loaded = 0;
    std::string line;
    while (std::getline(manifest, line)) {
      std::istringstream ls(line);
      std::string kw;
      if (!(ls >> kw)) continue;
      if (kw == "nodes") {
        ls >> nodes;
      } else if (kw == "layers") {
        ls >> layers;
      } else if (kw == "msg" || kw == "agg") {
        int layer = 0;
        std::string name;
        if (!(ls >> layer >> name)) fail(Errc::format, "bad checkpoint manifest line");
        std::string path = (!name.empty() && name[0] == '/') ? name : dir + "/" + name;
        HostTensor t = read_matrix(path);
        const bool is_msg = kw == "msg";
        if (is_msg ? (layer < 1 || layer > k + 1) : (layer < 1 || layer > k))
          fail(Errc::invalid_argument, std::string(is_msg ? "message" : "aggregated") + " layer out of range: " +
                                           std::to_string(layer));
        if (t.dims[0] != N || t.dims[1] != d[layer])
          fail(Errc::dimension, "checkpoint tensor shape mismatch: " + name);
        upload_table(is_msg ? msg[layer] : agg[layer], P[layer], d[layer], t.data.data());
        ++loaded;
      } else {
        fail(Errc::format, "bad checkpoint manifest keyword: " + kw);
      }
    }
    if (nodes != N || layers != k) fail(Errc::dimension, "checkpoint manifest does not match graph/model");
    if (loaded != static_cast<size_t>(2 * k + 1)) fail(Errc::format, "checkpoint manifest is missing tensors");
  }

  void upload_table(DevBuf& t, uint32_t pitch, uint32_t dim, const float* host) {
    SGB_CUDA(copy2d_sync(st, t.p, pitch * sizeof(float), host, dim * sizeof(float), dim * sizeof(float), N,
                          cudaMemcpyHostToDevice));
  }

  void download_table(const DevBuf& t, uint32_t pitch, uint32_t dim, float* host) const {
    SGB_CUDA(copy2d_sync(st, host, dim * sizeof(float), t.p, pitch * sizeof(float), dim * sizeof(float), N,
                          cudaMemcpyDeviceToHost));
  }

  // ------------------------------------------------------------- timing

  // External records so they become event-record nodes when the round is
  // captured into a graph (a plain record would only become a dependency edge).
  void mark(int i) {
    if (!opts.profile_kernels || i >= 64) return;
    // the external flag is only valid inside a capture (sharded / k-hop /
    // baseline rounds run uncaptured)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SGB_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) {
      SGB_CUDA(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal));
    } else {
      SGB_CUDA(cudaEventRecord(ev[i], st));
      ev_marked |= 1ull << i;
    }
  }
  uint64_t ev_marked = 0;  // events recorded by an uncaptured round (the graph records all of its marks)
  // per-layer events live at 16 + 8 * (l - 1) + j (profiling covers up to 6 layers)
  void lmark(int l, int j) { mark(16 + 8 * (l - 1) + j); }
  double span(int a, int b) {
    if (ev_marked != ~0ull && (!((ev_marked >> a) & 1) || !((ev_marked >> b) & 1))) return 0.0;  // not in this round
    float ms = 0;
    SGB_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
    return ms;
  }

  // --------------------------------------------------------------- round

  template <bool IsMax>
  void launch_classify(const ClassifyArgs& A, uint32_t V) {
    const unsigned grid = static_cast<unsigned>(sms * grid_mult);
    // exact float4 columns per lane for 513..768-wide rows (602-d: 5 instead of 8,
    // 255 -> fewer registers, no spill)
    const uint32_t exact = (V + 31) / 32;
    if (exact == 5 || exact == 6) {
      if (exact == 5) pdl_launch(k_classify<IsMax, 5>, grid, 256, 0, st, A);
      else pdl_launch(k_classify<IsMax, 6>, grid, 256, 0, st, A);
      SGB_CUDA(cudaGetLastError());
      return;
    }
    switch (cpl_for(V)) {
      case 1: pdl_launch(k_classify<IsMax, 1>, grid, 256, 0, st, A); break;
      case 2: pdl_launch(k_classify<IsMax, 2>, grid, 256, 0, st, A); break;
      case 4: pdl_launch(k_classify<IsMax, 4>, grid, 256, 0, st, A); break;
      case 8: pdl_launch(k_classify<IsMax, 8>, grid, 256, 0, st, A); break;
      default: pdl_launch(k_classify<IsMax, 16>, grid, 256, 0, st, A); break;
    }
    SGB_CUDA(cudaGetLastError());
  }

  template <bool IsMax>
  void launch_filter(int l, uint32_t V, const RecSink& S, const AdjView& ov, unsigned long long* lctr,
                     const unsigned long long* ab, const SeedArgs& sd) {
    const unsigned grid = static_cast<unsigned>(sms * 8);
    const ExpItem* w = exp_work[l].as<ExpItem>();
    const unsigned long long* nw = ds(L(l, L_EXPWORK));
    const uint32_t* dp = dirty[l - 1].as<uint32_t>();
    const uint64_t* eb = exp_base[l - 1].as<uint64_t>();
    const float4* os = oldslab[l].as<float4>();
    const RowTable cu = msg_rows(l);
    const float4* ag = vb<float4>(agg[l], P[l] / 4);
    const uint2* bd = abound[l].p ? vb<uint2>(abound[l], P[l] / 4) : nullptr;
    const uint2* bs = thrtab[l].as<uint2>();
    const float* cm = (use_summary && cmin[l].p) ? vb<float>(cmin[l], 1) : nullptr;
    const float* as = abstat[l].as<float>();
    uint8_t* rf = run_flags.as<uint8_t>();
    const uint32_t* gt = opts.emit_changed_only ? changed[l - 1].as<uint32_t>() : nullptr;
    // UNR / min-blocks per SM chosen by measurement at C2 (256-d with bound codes:
    // 8 code rows in flight at 3 blocks/SM 67.5 us/round; 8 or 16 rows at 2
    // blocks/SM 78.8 / 75.3 us; 4 or 8 rows at 4 blocks/SM 67.2 / 68.5 us)
    switch (cpl_for(V)) {
      // (rows <= 128 floats keep 3 CTAs/SM and 8 alpha rows per exact-test step:
      // the 4-CTA variant's 2-row step cost C3 29.4 -> 33.1 us/round)
      case 1: pdl_launch(k_expand_filter<IsMax, 1, 8, 3>, grid, 256, 0, st, w, nw, dp, eb, ov, S, os, cu, ag, bd, bs, V, d[l], cm, as, rf, lctr, gt, sd, ab); break;
      case 2:
        if (!bd && filter_minb4) {  // scalar summary, no code rows: 4 CTAs/SM (C2 events 34.7 -> 31.7 us/round)
          pdl_launch(k_expand_filter<IsMax, 2, 8, 4, false>, grid, 256, 0, st, w, nw, dp, eb, ov, S, os, cu, ag, bd, bs, V, d[l], cm, as, rf, lctr, gt, sd, ab);
          break;
        }
        pdl_launch(k_expand_filter<IsMax, 2, 8, 3>, grid, 256, 0, st, w, nw, dp, eb, ov, S, os, cu, ag, bd, bs, V, d[l], cm, as, rf, lctr, gt, sd, ab); break;
      case 4: pdl_launch(k_expand_filter<IsMax, 4>, grid, 256, 0, st, w, nw, dp, eb, ov, S, os, cu, ag, bd, bs, V, d[l], cm, as, rf, lctr, gt, sd, ab); break;
      default: pdl_launch(k_expand_filter<IsMax, 8>, grid, 256, 0, st, w, nw, dp, eb, ov, S, os, cu, ag, bd, bs, V, d[l], cm, as, rf, lctr, gt, sd, ab); break;
    }
    SGB_CUDA(cudaGetLastError());
  }

  bool seeds_fused = false;  // layer 1's seed records are written by k_batch_group

  // Enqueues one whole round (no host sync). Returns nothing; results land in
  // the scalars/counters, copied back by the caller.
  void enqueue_round(const char* d_ops, const uint32_t* d_src, const uint32_t* d_dst, uint32_t B, uint32_t mult,
                     bool with_commit, bool with_layers = true) {
    const unsigned long long* ab = abort_flag();
    AdjView ov = out.view(pool.as<uint32_t>()), iv = in.view(pool.as<uint32_t>());
    // layer 1's seeds go into K1 when layer 1 follows in this round (sharded
    // rounds enqueue it separately; k-hop rounds run no layers)
    seeds_fused = B && B <= kGroupCap && (with_layers || sharded);
    if (!B || B > kGroupCap) {  // (k_batch_group initialises them itself)
      SGB_CUDA(cudaMemsetAsync(scal.p, 0, S_NUM * sizeof(unsigned long long), st));
      SGB_CUDA(cudaMemsetAsync(ds(S_ERR), 0xFF, sizeof(unsigned long long), st));
      SGB_CUDA(cudaMemsetAsync(ctr.p, 0, static_cast<size_t>(k + 1) * C_NUM * sizeof(unsigned long long), st));
    }
    mark(0);
    // ---- K1
    DelLists dl{del_head_out.as<uint32_t>(), del_head_in.as<uint32_t>(), del_pos.as<uint32_t>(),
                del_next.as<uint32_t>(), ds(S_DELREC)};
    if (B && B <= kGroupCap) {  // one-CTA hash grouping + validation (no sort)
      const uint32_t cap = B <= 1024 ? 1024u : (B <= 2048 ? 2048u : kGroupCap);
      // grouping, validation, relocation election, the gate, relocations, the
      // net ops and (when the layers follow) layer 1's seeds in one CTA
      const bool clu = use_k1_cluster && B <= kGroupCapCluster;
      const bool pre = !clu && use_k1_pre && B <= kGroupCapPre;
      pdl_launch(clu ? k_batch_cluster : (pre ? k_batch_group_pre : k_batch_group), clu ? kClusterK1 : 1,
          clu ? kClusterK1Threads : 1024,
          clu ? batch_cluster_smem(cap) : (pre ? batch_group_pre_smem(cap) : batch_group_smem(cap)), st,
          d_ops, d_src, d_dst, B, N, cap, hash(), ov, iv, b_keys.as<uint64_t>(), b_net.as<uint64_t>(), ds(S_ERR),
          reinterpret_cast<uint32_t*>(ds(S_BADOP)), ds(S_NET_INS), ds(S_NUM_NET), d_round.as<uint32_t>(),
          b_reloc.as<uint32_t>(), reinterpret_cast<const unsigned long long*>(pool_top.p), pool_cap, ds(S_ABORT),
          mult, ds(L(1, L_CURSOR)), L_STRIDE, static_cast<uint32_t>(k), pool_top.as<unsigned long long>(),
          b_touch_out.as<uint32_t>(), b_touch_in.as<uint32_t>(), dl, seeds_fused, sink(1, mult),
          ctr.as<unsigned long long>() + static_cast<size_t>(1) * C_NUM + C_SEEDS, scal.as<unsigned long long>(),
          static_cast<uint32_t>(S_NUM), ctr.as<unsigned long long>(), static_cast<uint32_t>((k + 1) * C_NUM));
    } else if (B) {
      pdl_launch(k_batch_keys, grid_for(B), 256, 0, st, d_ops, d_src, d_dst, B, N, key_bits(), b_keys.as<uint64_t>(),
                                                b_vals.as<uint32_t>(), ds(S_ERR),
                                                reinterpret_cast<uint32_t*>(ds(S_BADOP)));
      size_t tb = cub_tmp.cap;  // sized by prepare_round
      cub::DeviceRadixSort::SortPairs(cub_tmp.p, tb, b_keys.as<uint64_t>(), b_keys_s.as<uint64_t>(),
                                      b_vals.as<uint32_t>(), b_vals_s.as<uint32_t>(), static_cast<int>(B), 0,
                                      2 * key_bits(), st);
      pdl_launch(k_validate, grid_for(B), 256, 0, st, b_keys_s.as<uint64_t>(), b_vals_s.as<uint32_t>(), d_ops, B, N, key_bits(), hash(),
                                              ov, iv, b_net.as<uint64_t>(), ds(S_ERR), ds(S_NET_INS),
                                              ds(S_NUM_NET));
      pdl_launch(k_reloc_plan, grid_for(B), 256, 0, st, b_net.as<uint64_t>(), ds(S_NUM_NET), ov, iv, d_round.as<uint32_t>(),
                                                b_reloc.as<uint32_t>(), ds(S_NET_INS));
    }
    if (!B || B > kGroupCap)  // (k_batch_group gates small batches itself)
      pdl_launch(k_round_gate, 1, 1, 0, st, ds(S_ERR), ds(S_BADOP), ds(S_RELOC_DEMAND),
                                    reinterpret_cast<const unsigned long long*>(pool_top.p), pool_cap, ds(S_ABORT),
                                    ds(S_NUM_NET), mult, ds(L(1, L_CURSOR)), L_STRIDE, static_cast<uint32_t>(k));
    if (B > kGroupCap) {
      pdl_launch(k_relocate, grid_for(2ull * B * 32), 256, 0, st, b_reloc.as<uint32_t>(), ds(S_RELOC_N), ov, iv,
                                                         pool_top.as<unsigned long long>(), ab);
      pdl_launch(k_apply_net, grid_for(B), 256, 0, st, b_net.as<uint64_t>(), ds(S_NUM_NET), ov, iv, hash(), d_round.as<uint32_t>(),
                                               b_touch_out.as<uint32_t>(), b_touch_in.as<uint32_t>(), dl,
                                               ds(S_NET_INS), ab);
    }
    SGB_CUDA(cudaGetLastError());
    mark(2);

    // ---- layers
    for (int l = 1; l <= (with_layers ? k : 0); ++l) enqueue_layer(l, mult);
    if (with_commit) enqueue_commit();
  }

  // The record sink of layer l's generators.
  RecSink sink(int l, uint32_t mult) {
    const bool filtered = filtered_layer(l, mult);
    return RecSink{rec.as<uint64_t>(), ord.as<uint32_t>(), cnt.as<uint32_t>(), runs.as<uint32_t>(), ds(L(l, L_RUNS)),
                   ds(L(l, L_CURSOR)), filtered ? run_flags.as<uint8_t>() : nullptr, shard_lo, shard_hi,
                   filtered ? touched.as<uint32_t>() : nullptr};
  }

  // One layer of the round (engine.cpp:184-296): events, grouping, classify,
  // recompute, dirty list, combination, message write-back. Sharded engines
  // keep only records whose target they own and leave the next layer's
  // expansion planning to the shard exchange (shard_import).
  void enqueue_layer(int l, uint32_t mult) {
    const unsigned long long* ab = abort_flag();
    AdjView ov = out.view(pool.as<uint32_t>());
    const unsigned big = static_cast<unsigned>(sms * grid_mult);
    unsigned long long* lctr = ctr.as<unsigned long long>() + static_cast<size_t>(l) * C_NUM;
    const uint32_t V = P[l] / 4;
    lmark(l, 0);
    // pre-filtered expansion (k_expand_filter) on layers >= 2
    const bool filtered = filtered_layer(l, mult);
    const RecSink S = sink(l, mult);
    // cnt (per-target record counts) is zero here: k_collect_dirty clears every
    // touched entry at the end of each layer (and it starts zeroed)
    // seeds and SELF records fill their own record slots (seed range / cursor
    // tail) beside the expansion (reserved ranges): side stream
    // layer 1's seeds of batches <= kGroupCap were written by k_batch_group;
    // later layers' seeds by the expansion kernel itself
    if (l == 1 && !seeds_fused)
      pdl_launch(k_seed_records, sms * 2, 256, 0, st, b_net.as<uint64_t>(), ds(S_NUM_NET), mult, S,
                 lctr + C_SEEDS, ab);
    if (l > 1) {
      const SeedArgs sd{b_net.as<uint64_t>(), ds(S_NUM_NET), mult, S, lctr + C_SEEDS};
      const bool self_recs = model->has_user_ops();
      if (self_recs) fork();  // SELF records beside the expansion
      if (filtered) {
        RecSink Sf = S;
        Sf.exact = nullptr;
        if (is_max) launch_filter<true>(l, V, Sf, ov, lctr, ab, sd); else launch_filter<false>(l, V, Sf, ov, lctr, ab, sd);
      } else {
        pdl_launch(k_expand_records, big, 256, 0, st, exp_work[l].as<ExpItem>(), ds(L(l, L_EXPWORK)),
                                              dirty[l - 1].as<uint32_t>(), exp_base[l - 1].as<uint64_t>(), ov, mult,
                                              S, lctr + C_EVENTS,
                                              opts.emit_changed_only ? changed[l - 1].as<uint32_t>() : nullptr, sd,
                                              ab);
      }
      if (self_recs) {
        pdl_launch(k_self_records, sms * 2, 256, 0, st2, dirty[l - 1].as<uint32_t>(), changed[l - 1].as<uint32_t>(),
                                                 ds(L(l - 1, L_NDIRTY)), S, ab);
        join();
      }
    }
    lmark(l, 1);
    pdl_launch(k_alloc_runs, sms * 2, 256, 0, st, runs.as<uint32_t>(), ds(L(l, L_RUNS)), cnt.as<uint32_t>(),
                                         run_flags.as<uint8_t>(), filtered, off.as<uint32_t>(), ds(L(l, L_ALLOC)),
                                         lctr, ab);
    // K3 (the scatter also plans the classify segments)
    const uint32_t chunk = V > 64 ? chunk_wide : chunk_narrow;
    {
      ClassifyArgs A{};
      A.tmap = filtered ? touched.as<uint32_t>() : nullptr;
      A.rec = rec_s.as<uint64_t>();
      A.runs = runs.as<uint32_t>();
      A.off = off.as<uint32_t>();
      A.cnt = cnt.as<uint32_t>();
      A.num_runs = ds(L(l, L_RUNS));
      A.abort = ab;
      A.msg.cur = msg_rows(l);
      A.msg.old = l >= 2 ? oldslab[l].as<float4>() : nullptr;
      A.msg.stamp = l >= 2 ? stamp[l].as<uint32_t>() : nullptr;
      A.msg.slot = l >= 2 ? slot[l].as<uint32_t>() : nullptr;
      A.msg.net = b_net.as<uint64_t>();
      A.msg.dprev = l > 1 ? dirty[l - 1].as<uint32_t>() : nullptr;
      A.msg.round = d_round.as<uint32_t>();
      A.msg.V = V;
      A.agg = vb<float4>(agg[l], P[l] / 4);
      A.d = d[l];
      A.in_len = in.len.as<uint32_t>();
      A.in_new = in.n_new.as<uint32_t>();
      A.run_flags = run_flags.as<uint8_t>();
      A.seg = seg.as<uint4>();
      A.n_seg = ds(L(l, L_NSEG));
      A.cls_scratch = cls_scratch.as<int>();
      A.cls_slot = cls_slot.as<uint32_t>();
      A.cls_remaining = cls_remaining.as<uint32_t>();
      A.cls_flags = cls_flags.as<uint32_t>();
      A.n_cls_scratch = ds(L(l, L_NCLS));
      A.seg_next = nullptr;  // static assignment measured faster here than the dynamic queue
      A.work = work.as<uint64_t>();
      A.n_work = ds(L(l, L_NWORK));
      A.chunk = chunk;
      A.scratch = scratch.as<int>();
      A.scratch_idx = scratch_idx.as<uint32_t>();
      A.remaining = remaining.as<uint32_t>();
      A.any_live = any_live.as<uint32_t>();
      A.n_scratch = ds(L(l, L_NSCRATCH));
      A.ctr = lctr;
      if (use_sparse) {
        A.sp_target = sp_target.as<uint32_t>();
        A.sp_n = sp_n.as<uint32_t>();
        A.sp_dims = sp_dims.as<uint32_t>();
        A.sp_aold = sp_aold.as<float>();
        A.sp_acc = sp_acc.as<int>();
        A.sp_live = sp_live.as<uint32_t>();
        A.sp_changed = sp_changed.as<uint32_t>();
        A.n_sparse = ds(L(l, L_NSPARSE));
        A.swork = swork.as<uint64_t>();
        A.n_swork = ds(L(l, L_NSWORK));
        A.sp_remaining = sp_remaining.as<uint32_t>();
      }
      if (is_max)
        pdl_launch(k_scatter_plan<true>, big, 256, 0, st, rec.as<uint64_t>(), ord.as<uint32_t>(), ds(L(l, L_CURSOR)), A,
                                                  rec_s.as<uint64_t>(), filtered);
      else
        pdl_launch(k_scatter_plan<false>, big, 256, 0, st, rec.as<uint64_t>(), ord.as<uint32_t>(), ds(L(l, L_CURSOR)), A,
                                                   rec_s.as<uint64_t>(), filtered);
      SGB_CUDA(cudaGetLastError());
      lmark(l, 2);
      if (is_max) launch_classify<true>(A, V); else launch_classify<false>(A, V);
    }
    lmark(l, 3);
    // K4
    {
      AggArgs A{};
      A.work = work.as<uint64_t>();
      A.n_work = ds(L(l, L_NWORK));
      A.update = true;
      A.runs = runs.as<uint32_t>();
      A.abort = ab;
      A.run_flags = run_flags.as<uint8_t>();
      A.scratch_idx = scratch_idx.as<uint32_t>();
      A.remaining = remaining.as<uint32_t>();
      A.any_live = any_live.as<uint32_t>();
      A.scratch = scratch.as<int>();
      A.in_off = in.off.as<uint64_t>();
      A.in_len = in.len.as<uint32_t>();
      A.in_ent = pool.as<uint32_t>();
      A.msg = msg_rows(l);
      A.agg = vb<float4>(agg[l], V);
      A.V = V;
      A.d = d[l];
      A.chunk = chunk;
      A.fetch_ctr = lctr + (l == 1 ? C_FETCH_L1MSG : C_FETCH_OTHER);
      A.ctr = lctr;
      A.next = nullptr;
      if (use_sparse) fork();  // sparse recompute on the side stream, beside the dense one
      if (is_max) launch_aggregate<true>(A, V); else launch_aggregate<false>(A, V);
      if (use_sparse) {
        SparseArgs S{};
        S.swork = swork.as<uint64_t>();
        S.n_swork = ds(L(l, L_NSWORK));
        S.abort = ab;
        S.sp_target = sp_target.as<uint32_t>();
        S.sp_n = sp_n.as<uint32_t>();
        S.sp_dims = sp_dims.as<uint32_t>();
        S.sp_aold = sp_aold.as<float>();
        S.sp_acc = sp_acc.as<int>();
        S.sp_live = sp_live.as<uint32_t>();
        S.sp_changed = sp_changed.as<uint32_t>();
        S.n_sparse = ds(L(l, L_NSPARSE));
        S.sp_remaining = sp_remaining.as<uint32_t>();
        S.in_off = in.off.as<uint64_t>();
        S.in_len = in.len.as<uint32_t>();
        S.in_ent = pool.as<uint32_t>();
        S.msg = msg_rows(l);
        S.agg = vb<float>(agg[l], P[l]);
        S.P = P[l];
        S.run_flags = run_flags.as<uint8_t>();
        S.fetch_ctr = A.fetch_ctr;
        S.ctr = lctr;
        if (is_max) pdl_launch(k_recompute_sparse<true>, sms * grid_mult, 256, 0, st2, S);
        else pdl_launch(k_recompute_sparse<false>, sms * grid_mult, 256, 0, st2, S);
        SGB_CUDA(cudaGetLastError());
        join();
      }
    }
    lmark(l, 4);
    // K5
    const bool has_next = l < k;
    pdl_launch(k_collect_dirty, sms * 4, 256, 0, st, 
        runs.as<uint32_t>(), ds(L(l, L_RUNS)), run_flags.as<uint8_t>(), cnt.as<uint32_t>(),
        filtered ? touched.as<uint32_t>() : nullptr, !(has_next && filtered_layer(l + 1, mult)),
        dirty[l].as<uint32_t>(),
        ds(L(l, L_NDIRTY)), ov, has_next, mult, exp_base[l].as<uint64_t>(),
        has_next ? exp_work[l + 1].as<ExpItem>() : nullptr, has_next ? ds(L(l + 1, L_EXPWORK)) : nullptr,
        has_next ? ds(L(l + 1, L_CURSOR)) : nullptr, lctr, static_cast<uint32_t>(model->user_ops_in(l - 1)),
        l == 1, !sharded, changed[l].as<uint32_t>(), ab);
    SGB_CUDA(cudaGetLastError());
    lmark(l, 5);
    // K6 combination over the dirty rows, with K8 (write-back, pre-image,
    // change flag, stamps, next-layer thresholds) fused into its last GEMM
    uint32_t yp = 0, yd = 0;
    RowSrc x0{vb<float>(agg[l], P[l]), dirty[l].as<uint32_t>(), 0, P[l]};
    RowSrc self{vb<float>(msg[l], P[l]), dirty[l].as<uint32_t>(), 0, P[l]};
    uint16_t* bnd = abound[l].p ? vb<uint16_t>(abound[l], P[l]) : nullptr;
    // thresholds for the next layer's filter (sharded rounds: after the import)
    const bool thr_next = has_next && !sharded && filtered_layer(l + 1, mult) && thrtab[l + 1].p;
    WriteBack wb{};
    wb.table = vb<float>(msg[l + 1], P[l + 1]);
    wb.pitch = P[l + 1];
    wb.dirty = dirty[l].as<uint32_t>();
    wb.slab = has_next ? oldslab[l + 1].as<float>() : nullptr;
    wb.changed = changed[l].as<uint32_t>();
    wb.stamp = has_next ? stamp[l + 1].as<uint32_t>() : nullptr;
    wb.slot = has_next ? slot[l + 1].as<uint32_t>() : nullptr;
    wb.round = d_round.as<uint32_t>();
    wb.thr = thr_next ? thrtab[l + 1].as<uint16_t>() : nullptr;
    wb.tstat = thr_next ? abstat[l + 1].as<float>() : nullptr;
    wb.is_max = is_max;
    bool fused = false;
    const bool refresh = cmin.size() > static_cast<size_t>(l) && cmin[l].p;
    if (refresh) {  // the a_l codes and summaries of the dirty rows, beside the combination
      fork();
      auto* rc = is_max ? k_refresh_codes<true> : k_refresh_codes<false>;
      pdl_launch(rc, sms * 2, 256, 0, st2, dirty[l].as<uint32_t>(), ds(L(l, L_NDIRTY)), vb<float>(agg[l], P[l]), bnd,
                 vb<float>(cmin[l], 1), abstat[l].as<float>(), P[l], d[l], ab);
    }
    const float* Y = run_program(model->program(l - 1), x0, self, ds(L(l, L_NDIRTY)), 0, N, d[l], &yp, &yd, ab,
                                 use_fused_k8 ? &wb : nullptr, &fused);
    if (refresh) join();
    lmark(l, 6);
    if (!fused) {  // K8 write-back on its own
      auto* wm = is_max ? k_write_messages<true> : k_write_messages<false>;
      uint16_t* bnd8 = refresh ? nullptr : bnd;  // (codes already refreshed beside the GEMM)
      pdl_launch(wm, big, 256, 0, st, dirty[l].as<uint32_t>(), ds(L(l, L_NDIRTY)), Y, yp, vb<float>(msg[l + 1], P[l + 1]), P[l + 1],
                              d[l + 1], has_next ? oldslab[l + 1].as<float>() : nullptr,
                              has_next ? stamp[l + 1].as<uint32_t>() : nullptr,
                              has_next ? slot[l + 1].as<uint32_t>() : nullptr, d_round.as<uint32_t>(),
                              changed[l].as<uint32_t>(), ds(L(l, L_NCHANGED)), vb<float>(agg[l], P[l]), bnd8,
                              bnd8 ? abstat[l].as<float>() : nullptr, P[l],
                              thr_next ? thrtab[l + 1].as<uint16_t>() : nullptr,
                              thr_next ? abstat[l + 1].as<float>() : nullptr, ab);
    }
    SGB_CUDA(cudaGetLastError());
    if (sharded)  // this shard's own dirty count (the exchange replaces L_NDIRTY with the global one)
      SGB_CUDA(cudaMemcpyAsync(lctr + C_DIRTY, ds(L(l, L_NDIRTY)), 8, cudaMemcpyDeviceToDevice, st));
    lmark(l, 7);
  }

  // The round's scalars and counters go to the host BEFORE the graph commit
  // (DynamicGraph::commit, graph.cpp:108-111; checkpoint commit_round is the
  // stamp bump), and apply() waits for that copy only (ev_result): the commit
  // then runs behind the caller's return. Everything enqueued later on the
  // stream (the next round, readouts, saves) is ordered after it.
  void enqueue_commit() {
    const unsigned long long* ab = abort_flag();
    AdjView ov = out.view(pool.as<uint32_t>()), iv = in.view(pool.as<uint32_t>());
    SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaMemcpyAsync(h_ctr.p, ctr.p, static_cast<size_t>(k + 1) * C_NUM * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st));
    record_external(ev_result);
    mark(11);
    pdl_launch(k_commit, sms * 2, 256, 0, st, b_touch_out.as<uint32_t>(), b_touch_in.as<uint32_t>(),
               ds(S_NET_INS), ov, iv, hash(), del_head_out.as<uint32_t>(), del_head_in.as<uint32_t>(),
               del_pos.as<uint32_t>(), del_next.as<uint32_t>(), b_net.as<uint64_t>(), ds(S_NUM_NET), ab);
    SGB_CUDA(cudaGetLastError());
    mark(12);
  }

  // An event record that becomes an event-record node under stream capture.
  void record_external(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SGB_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) SGB_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else SGB_CUDA(cudaEventRecord(e, st));
  }

  RoundStats apply(const char* ops, const NodeId* src, const NodeId* dst, size_t count, bool on_device,
                   void* producer_stream);
  void baseline_counters(RoundStats& s);

  // ---- k-hop recompute comparator (EngineOptions::khop_recompute)
  DevBuf kh_reached, kh_members, kh_nch, kh_scan, kh_work, kh_scr;
  std::vector<uint64_t> kh_need;  // [l] = |need[l]|, l = 1..k+1 (need[k+1] = affected area)
  void khop_recompute();
};

// ------------------------------------------------------------------- ctor

DeviceEngine::DeviceEngine(const HostGraph& g, std::shared_ptr<const BoundModel> model, const float* features,
                           uint32_t rows, uint32_t cols, const char* ckpt_dir,
                           std::shared_ptr<ShardTransport> transport)
    : p_(new Impl) {
  std::string why;
  if (!cuda_device_available(&why)) fail(Errc::unknown, "no CUDA device available for the B200 engine: " + why);
  Impl& I = *p_;
  if (const char* dv = std::getenv("SGNN_B200_DEVICE")) I.device = std::atoi(dv);
  else SGB_CUDA(cudaGetDevice(&I.device));
  SGB_CUDA(cudaSetDevice(I.device));
  SGB_CUDA(cudaDeviceGetAttribute(&I.sms, cudaDevAttrMultiProcessorCount, I.device));
  SGB_CUDA(cudaDeviceGetAttribute(&I.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, I.device));
  SGB_CUDA(cudaStreamCreateWithFlags(&I.st, cudaStreamNonBlocking));
  SGB_CUDA(cudaStreamCreateWithFlags(&I.st2, cudaStreamNonBlocking));
  SGB_CUDA(cudaEventCreateWithFlags(&I.ev_fork, cudaEventDisableTiming));
  SGB_CUDA(cudaEventCreateWithFlags(&I.ev_join, cudaEventDisableTiming));
  SGB_CUDA(cudaEventCreateWithFlags(&I.ev_producer, cudaEventDisableTiming));
  SGB_CUDA(cudaEventCreateWithFlags(&I.ev_result, cudaEventDisableTiming));
  for (auto& e : I.ev) SGB_CUDA(cudaEventCreate(&e));
  I.ev_ready = true;
  I.model = std::move(model);
  I.N = g.num_nodes();
  I.shard_hi = I.N;
  if (I.N >= kMaxNodes) fail(Errc::unsupported_model, "device engine supports fewer than 2^29 nodes");
  if (transport) {
    // partitioned: the same bounds on every shard (from the same graph)
    if (ckpt_dir) fail(Errc::invalid_argument, "a sharded engine starts from full inference, not checkpoints");
    if (transport->world() > kMaxPeers) fail(Errc::invalid_argument, "at most 8 shards");
    std::vector<uint32_t> deg(I.N);
    for (uint32_t v = 0; v < I.N; ++v) deg[v] = static_cast<uint32_t>(g.in(v).size());
    I.bounds = shard_bounds(deg, transport->world());
    I.shard_rank = transport->rank();
    I.shard_world = transport->world();
    I.shard_lo = I.bounds[I.shard_rank];
    I.shard_hi = I.bounds[I.shard_rank + 1];
    I.sharded = true;  // a 1-shard group still runs the exchange (exercises the transport)
    I.transport = std::move(transport);
  }
  I.k = I.model->num_layers();
  I.is_max = I.model->agg() == Agg::Max;
  I.F = cols;
  I.d.assign(I.k + 2, 0);
  I.P.assign(I.k + 2, 0);
  for (int l = 1; l <= I.k + 1; ++l) {
    I.d[l] = I.model->message_dim(l);
    I.P[l] = pitch_of(I.d[l]);
    cpl_for(I.P[l] / 4);  // dimension limit check
    I.maxP = std::max(I.maxP, I.P[l]);
  }
  I.features.assign(features, features + static_cast<size_t>(rows) * cols);
  I.set_kernel_attributes();
  I.upload_graph(g);
  I.upload_weights();
  I.alloc_tables(I.msg, I.agg);
  I.stamp.resize(I.k + 2);
  I.slot.resize(I.k + 2);
  I.oldslab.resize(I.k + 2);
  for (int l = 2; l <= I.k; ++l) {
    I.stamp[l].alloc_exact(sizeof(uint32_t) * I.N);
    I.slot[l].alloc_exact(sizeof(uint32_t) * I.N);
    I.oldslab[l].alloc_exact(static_cast<size_t>(I.N) * I.P[l] * sizeof(float));
    SGB_CUDA(memset_sync(I.st, I.stamp[l].p, 0, sizeof(uint32_t) * I.N));
    // pitch padding of every pre-image row stays zero (the fused write-back
    // writes columns < d only)
    SGB_CUDA(memset_sync(I.st, I.oldslab[l].p, 0, static_cast<size_t>(I.N) * I.P[l] * sizeof(float)));
  }
  I.abound.resize(I.k + 1);
  I.abstat.resize(I.k + 1);
  I.thrtab.resize(I.k + 1);
  I.cmin.resize(I.k + 1);
  for (int l = 2; l <= I.k; ++l)
    if (cpl_for(I.P[l] / 4) <= 8) {  // filtered layers: grid + per-target summary
      I.abstat[l].alloc_exact(3 * sizeof(float) * I.P[l]);
      I.cmin[l].alloc_exact(std::max<size_t>(static_cast<size_t>(I.rows_owned()) * sizeof(float), 256));
    }
  // the summary settles what the per-position code rows would (C2: the code
  // stage settled none of the PAIRs the summary left open), so the N x pitch
  // code table and the per-source threshold rows exist only with the summary
  // off (the filter takes the source's normalised maximum from its rows)
  if (const char* f = std::getenv("SGNN_B200_SUMMARY")) I.use_summary = std::atoi(f) != 0;
  for (int l = 2; l <= I.k; ++l)
    if (!I.use_summary && cpl_for(I.P[l] / 4) >= 2 && cpl_for(I.P[l] / 4) <= 8) {  // widths whose filter reads codes
      I.abound[l].alloc_exact(std::max<size_t>(static_cast<size_t>(I.rows_owned()) * I.P[l] * sizeof(uint16_t), 256));
      I.thrtab[l].alloc_exact(static_cast<size_t>(I.N) * I.P[l] * sizeof(uint16_t));
      SGB_CUDA(memset_sync(I.st, I.thrtab[l].p, 0, static_cast<size_t>(I.N) * I.P[l] * sizeof(uint16_t)));
    }
  I.abcolr.alloc_exact(2 * sizeof(int) * I.maxP);
  I.dirty.resize(I.k + 1);
  I.changed.resize(I.k + 1);
  I.exp_base.resize(I.k + 1);
  I.exp_work.resize(I.k + 2);
  for (int l = 1; l <= I.k; ++l) {
    I.dirty[l].alloc_exact(sizeof(uint32_t) * I.N);
    I.changed[l].alloc_exact(sizeof(uint32_t) * I.N);
    I.exp_base[l].alloc_exact(sizeof(uint64_t) * I.N);
  }
  for (DevBuf* b : {&I.cnt, &I.off, &I.runs, &I.cls_slot, &I.cls_remaining, &I.cls_flags, &I.scratch_idx,
                    &I.remaining, &I.any_live, &I.sp_target, &I.sp_n, &I.sp_live, &I.sp_changed, &I.sp_remaining})
    b->alloc_exact(sizeof(uint32_t) * I.N);
  for (DevBuf* b : {&I.sp_dims, &I.sp_aold, &I.sp_acc}) b->alloc_exact(sizeof(uint32_t) * kSparseDims * I.N);
  I.touched.alloc_exact(sizeof(uint32_t) * (I.N / 16 + 1));
  SGB_CUDA(memset_sync(I.st, I.touched.p, 0, sizeof(uint32_t) * (I.N / 16 + 1)));
  I.run_flags.alloc_exact(I.N);
  SGB_CUDA(memset_sync(I.st, I.run_flags.p, 0, I.N));  // kept clear by k_collect_dirty
  SGB_CUDA(memset_sync(I.st, I.cnt.p, 0, sizeof(uint32_t) * I.N));  // likewise
  I.n_dirty_host.assign(I.k + 1, 0);
  I.S_NUM = S_GLOBAL + (I.k + 1) * L_STRIDE;
  I.scal.alloc_exact(I.S_NUM * sizeof(unsigned long long));
  I.h_scal.ensure(I.S_NUM * sizeof(unsigned long long));
  I.ctr.alloc_exact(static_cast<size_t>(I.k + 1) * C_NUM * sizeof(unsigned long long));
  I.h_ctr.ensure(static_cast<size_t>(I.k + 1) * C_NUM * sizeof(unsigned long long));
  I.d_round.alloc_exact(sizeof(uint32_t));
  I.h_round.ensure(sizeof(uint32_t));
  if (const char* g = std::getenv("SGNN_B200_GRAPHS")) I.use_graphs = std::atoi(g) != 0;
  if (const char* b = std::getenv("SGNN_B200_BULK")) I.use_bulk = std::atoi(b) != 0;
  if (const char* f = std::getenv("SGNN_B200_FILTER")) I.use_filter = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_SPARSE")) I.use_sparse = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_FUSED_K8")) I.use_fused_k8 = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_K1PRE")) I.use_k1_pre = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_GEMM_MAB")) I.gemm_m_ab = static_cast<uint32_t>(std::atoi(f));
  if (const char* f = std::getenv("SGNN_B200_K1CLUSTER")) I.use_k1_cluster = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_FILTER_MINB4")) I.filter_minb4 = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_TMA")) I.use_tma = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_DEVICE_EXCHANGE")) I.use_device_exchange = std::atoi(f) != 0;
  if (const char* f = std::getenv("SGNN_B200_TMA_STAGES")) I.tma_stages = std::atoi(f) == 3 ? 3 : 2;
  if (const char* f = std::getenv("SGNN_B200_GRID")) I.grid_mult = std::max(1, std::atoi(f));
  if (const char* f = std::getenv("SGNN_B200_BULK_GRID")) I.bulk_grid = std::max(1, std::atoi(f));
  if (const char* f = std::getenv("SGNN_B200_CHUNK")) I.chunk_narrow = std::max(8, std::atoi(f));
  if (const char* f = std::getenv("SGNN_B200_CHUNK_WIDE")) I.chunk_wide = std::max(8, std::atoi(f));
  if (const char* t = std::getenv("SGNN_B200_TRACE")) {
    I.trace = std::atoi(t) != 0;
    I.opts.profile_kernels = std::atoi(t) > 1;
  }
  I.ensure_capacity(1, 2);
  if (I.sharded) {
    // every shard's m_l allocation and pack buffers, read in place by the peers
    I.msg_peers = I.share_messages(I.msg);
    if (I.transport->peers_on_other_devices()) I.use_bulk = false;
    size_t rb_max = 16;
    for (int l = 1; l < I.k; ++l) rb_max = std::max(rb_max, shard_row_bytes(I.P[l + 1]));
    for (int b = 0; b < 2; ++b) {
      I.pack2[b].alloc_exact(static_cast<size_t>(I.rows_owned()) * rb_max + 256);
      I.pack_peers[b] = I.transport->share_device(I.pack2[b].p);
    }
    std::vector<unsigned long long> pt(2 * kMaxPeers, 0);
    for (int b = 0; b < 2; ++b)
      for (int r = 0; r < I.shard_world; ++r) pt[b * kMaxPeers + r] = reinterpret_cast<unsigned long long>(I.pack_peers[b][r]);
    I.pack_tab.alloc_exact(pt.size() * 8);
    SGB_CUDA(copy_sync(I.st, I.pack_tab.p, pt.data(), pt.size() * 8, cudaMemcpyHostToDevice));
    I.mbox.alloc_exact(MB_WORDS * 8ull);
    SGB_CUDA(memset_sync(I.st, I.mbox.p, 0, MB_WORDS * 8ull));
    I.xseq.alloc_exact(8);
    SGB_CUDA(memset_sync(I.st, I.xseq.p, 0, 8));
    const std::vector<const void*> bx = I.transport->share_device(I.mbox.p);
    I.boxes.world = static_cast<uint32_t>(I.shard_world);
    for (int r = 0; r < I.shard_world; ++r) I.boxes.box[r] = static_cast<const uint64_t*>(bx[r]);
    if (static_cast<size_t>(I.k + 1) * C_NUM > MB_CTR_N) I.use_device_exchange = false;
    I.d_imp.ensure(8ull * (3 * I.shard_world + 1));
    I.h_imp.ensure(8ull * (3 * I.shard_world + 1));
  }
  if (ckpt_dir)
    I.load_checkpoints(ckpt_dir);
  else
    I.full_inference(I.msg, I.agg, I.msg_peers);
  I.refresh_abound();
  SGB_CUDA(cudaDeviceSynchronize());
}

DeviceEngine::~DeviceEngine() = default;

void DeviceEngine::set_combination_mode(int mode) {
  Impl& I = *p_;
  if (mode < 0 || mode > 2)
    fail(Errc::invalid_argument, "combination_mode must be 0 (exact), 1 (3xTF32 tensor cores) or 2 (TF32)");
  if (mode == I.tc_mode) return;
  SGB_CUDA(cudaSetDevice(I.device));
  I.tc_mode = mode;
  if (I.graph.exec) SGB_CUDA(cudaGraphExecDestroy(I.graph.exec));
  I.graph = {};  // rounds are re-captured with the other GEMM
  // tables are recomputed so every stored message comes from the same arithmetic
  I.full_inference(I.msg, I.agg, I.msg_peers);
  I.refresh_abound();
}

int DeviceEngine::combination_mode() const { return p_->tc_mode; }

void DeviceEngine::shard_range(uint32_t* lo, uint32_t* hi) const {
  if (lo) *lo = p_->shard_lo;
  if (hi) *hi = p_->shard_hi;
}

std::vector<uint64_t> DeviceEngine::memory_bytes() const {
  const Impl& I = *p_;
  uint64_t tables = 0, graph = 0;
  for (const DevBuf& b : I.msg) tables += b.cap;
  for (const DevBuf& b : I.agg) tables += b.cap;
  for (const DevBuf& b : I.abound) tables += b.cap;
  for (const DevBuf& b : I.cmin) tables += b.cap;
  for (const DevBuf* b : {&I.pool, &I.h_slots, &I.out.off, &I.out.len, &I.out.cap, &I.out.n_new,
                          &I.out.n_del, &I.out.touch, &I.out.reloc, &I.in.off, &I.in.len, &I.in.cap, &I.in.n_new,
                          &I.in.n_del, &I.in.touch, &I.in.reloc})
    graph += b->cap;
  size_t free_b = 0, total_b = 0;
  SGB_CUDA(cudaSetDevice(I.device));
  SGB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  return {tables, graph, static_cast<uint64_t>(total_b - free_b)};
}

int DeviceEngine::device() const { return p_->device; }
bool DeviceEngine::sharded() const { return p_->sharded; }

EngineOptions& DeviceEngine::options() { return p_->opts; }
uint32_t DeviceEngine::num_nodes() const { return p_->N; }
uint64_t DeviceEngine::num_edges() const { return p_->E; }
int DeviceEngine::num_layers() const { return p_->k; }
const KernelTimes& DeviceEngine::kernel_times() const { return p_->kt; }
size_t DeviceEngine::launches_per_round() const { return p_->graph.kernel_nodes; }
void* DeviceEngine::stream() const { return p_->st; }

uint32_t DeviceEngine::dim(int layer, int stage) const {
  const Impl& I = *p_;
  if (stage == 0) {
    if (layer < 1 || layer > I.k + 1)
      fail(Errc::invalid_argument, "message layer out of range: " + std::to_string(layer));
  } else if (layer < 1 || layer > I.k) {
    fail(Errc::invalid_argument, "aggregated layer out of range: " + std::to_string(layer));
  }
  return I.d[layer];
}

// A sharded engine holds the rows of its own range of every table (the other
// shards hold theirs).
static void check_owned_rows(bool sharded, int layer, int stage, uint32_t lo, uint32_t hi, uint32_t slo,
                             uint32_t shi) {
  if (!sharded || lo >= hi) return;
  if (lo < slo || hi > shi)
    fail(Errc::invalid_argument, "rows [" + std::to_string(lo) + ", " + std::to_string(hi) + ") of " +
                                     (stage == 1 ? "aggregated" : "message") + " layer " + std::to_string(layer) +
                                     " are not owned by this shard [" + std::to_string(slo) + ", " +
                                     std::to_string(shi) + ")");
}

void DeviceEngine::read_row(int layer, int stage, NodeId node, float* out) const {
  const uint32_t dd = dim(layer, stage);
  const Impl& I = *p_;
  if (node >= I.N) fail(Errc::invalid_argument, "node id out of range");
  check_owned_rows(I.sharded, layer, stage, node, node + 1, I.shard_lo, I.shard_hi);
  const DevBuf& t = stage == 0 ? I.msg[layer] : I.agg[layer];
  SGB_CUDA(copy_sync(I.st, out, I.vb<float>(t, I.P[layer]) + static_cast<size_t>(node) * I.P[layer],
                     dd * sizeof(float), cudaMemcpyDeviceToHost));
}

void DeviceEngine::read_table(int layer, int stage, float* out) const { read_rows(layer, stage, 0, p_->N, out); }

void DeviceEngine::read_rows(int layer, int stage, uint32_t lo, uint32_t hi, float* out) const {
  const uint32_t dd = dim(layer, stage);
  const Impl& I = *p_;
  if (lo > hi || hi > I.N) fail(Errc::invalid_argument, "row range out of bounds");
  check_owned_rows(I.sharded, layer, stage, lo, hi, I.shard_lo, I.shard_hi);
  if (lo == hi) return;
  const DevBuf& t = stage == 0 ? I.msg[layer] : I.agg[layer];
  SGB_CUDA(copy2d_sync(I.st, out, dd * sizeof(float), I.vb<float>(t, I.P[layer]) + static_cast<size_t>(lo) * I.P[layer],
                       I.P[layer] * sizeof(float), dd * sizeof(float), hi - lo, cudaMemcpyDeviceToHost));
}

std::vector<NodeId> DeviceEngine::last_dirty(int layer) const {
  const Impl& I = *p_;
  if (layer < 1 || layer > I.k) fail(Errc::invalid_argument, "layer out of range: " + std::to_string(layer));
  std::vector<NodeId> v(I.n_dirty_host[layer]);
  if (!v.empty())
    SGB_CUDA(copy_sync(I.st, v.data(), I.dirty[layer].p, v.size() * sizeof(NodeId), cudaMemcpyDeviceToHost));
  std::sort(v.begin(), v.end());  // the reference's dirty lists are ascending (engine.cpp:209-228)
  return v;
}

void DeviceEngine::flush_l2() const {
  Impl& I = *p_;
  const size_t bytes = 256ull << 20;
  I.l2buf.ensure(bytes);
  pdl_launch(k_l2_flush, I.sms * 4, 256, 0, I.st, I.l2buf.as<uint4>(), bytes / sizeof(uint4), I.round);
  SGB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ round

RoundStats DeviceEngine::apply(const char* ops, const NodeId* src, const NodeId* dst, size_t count, bool on_device,
                               void* producer_stream) {
  return p_->apply(ops, src, dst, count, on_device, producer_stream);
}

RoundStats DeviceEngine::Impl::apply(const char* ops, const NodeId* src, const NodeId* dst, size_t count,
                                     bool on_device, void* producer_stream) {
  if (count > 0x3FFFFFFFull) fail(Errc::invalid_argument, "batch too large");
  const uint32_t B = static_cast<uint32_t>(count);
  SGB_CUDA(cudaSetDevice(device));
  PdlScope pdl_scope(!sharded);
  if (!on_device)
    for (size_t i = 0; i < count; ++i)
      if (ops[i] != '+' && ops[i] != '-') fail(Errc::invalid_argument, "op must be '+' or '-'");
  std::fill(n_dirty_host.begin(), n_dirty_host.end(), 0u);  // dirty_.assign (engine.cpp:176)
  ev_marked = 0;
  const uint32_t mult = opts.duplicate_seed_events ? 2u : 1u;
  if (2 * (E + h_tombs + B) > hcap) build_hash(std::max<uint64_t>(E / 4, 4ull * B));
  prepare_round(B, mult);
  *h_round.as<uint32_t>() = round;
  SGB_CUDA(cudaMemcpyAsync(d_round.p, h_round.p, sizeof(uint32_t), cudaMemcpyHostToDevice, st));

  const char* d_ops = ops;
  const uint32_t* d_src = src;
  const uint32_t* d_dst = dst;
  if (B && !on_device) {
    const size_t bytes = static_cast<size_t>(B) * 9;
    h_batch.ensure(bytes);
    char* hb = h_batch.as<char>();
    std::memcpy(hb, src, B * sizeof(uint32_t));
    std::memcpy(hb + 4 * static_cast<size_t>(B), dst, B * sizeof(uint32_t));
    std::memcpy(hb + 8 * static_cast<size_t>(B), ops, B);
    SGB_CUDA(cudaMemcpyAsync(b_src.p, hb, bytes, cudaMemcpyHostToDevice, st));
  } else if (B) {
    // device batch: staged into the engine's own buffer so a captured round
    // graph always reads the same addresses, after the producer's work
    if (producer_stream) {
      SGB_CUDA(cudaEventRecord(ev_producer, static_cast<cudaStream_t>(producer_stream)));
      SGB_CUDA(cudaStreamWaitEvent(st, ev_producer, 0));
    }
    uint32_t* bs = b_src.as<uint32_t>();
    SGB_CUDA(cudaMemcpyAsync(bs, src, B * 4ull, cudaMemcpyDeviceToDevice, st));
    SGB_CUDA(cudaMemcpyAsync(bs + B, dst, B * 4ull, cudaMemcpyDeviceToDevice, st));
    SGB_CUDA(cudaMemcpyAsync(bs + 2 * static_cast<size_t>(B), ops, B, cudaMemcpyDeviceToDevice, st));
  }
  if (B) {
    d_src = b_src.as<uint32_t>();
    d_dst = d_src + B;
    d_ops = reinterpret_cast<const char*>(d_src + 2 * static_cast<size_t>(B));
  }
  RoundStats stats;
  for (int attempt = 0;; ++attempt) {
    const bool baseline = opts.baseline_counters;
    const bool khop = opts.khop_recompute;
    if (sharded) {
      if (graph.B != B || graph.mult != mult || !graph.kernel_nodes) {
        // Launch count of a sharded round (graph segments between host-side
        // count exchanges): a capture that is never instantiated counts the
        // round's kernels; each exchange adds pack + import + plan.
        cudaGraph_t g = nullptr;
        SGB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        enqueue_round(d_ops, d_src, d_dst, B, mult, true);
        SGB_CUDA(cudaStreamEndCapture(st, &g));
        size_t nn = 0;
        SGB_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) SGB_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        size_t kn = 0;
        for (auto nd : nodes) {
          cudaGraphNodeType t;
          SGB_CUDA(cudaGraphNodeGetType(nd, &t));
          if (t == cudaGraphNodeTypeKernel) ++kn;
        }
        SGB_CUDA(cudaGraphDestroy(g));
        if (graph.exec) SGB_CUDA(cudaGraphExecDestroy(graph.exec));
        graph = {};
        graph.B = B;
        graph.mult = mult;
        graph.kernel_nodes = kn;
        for (int l = 1; l < k; ++l)  // pack + import + plan (+ thresholds) per exchange
          graph.kernel_nodes += 3 + ((filtered_layer(l + 1, mult) && thrtab[l + 1].p) ? 1 : 0);
      }
      // K1 (identical on every shard), then the layers without a host check of
      // the gate: a rejected batch aborts every kernel on every shard alike, so
      // the exchanges carry zero rows and the error is decoded after the round
      if (use_graphs && !opts.profile_kernels && use_device_exchange && !opts.baseline_counters) {
        sharded_round_device(d_ops, d_src, d_dst, B, mult);
        ev_marked = ~0ull;
      } else if (use_graphs && !opts.profile_kernels) {
        sharded_round_graphs(d_ops, d_src, d_dst, B, mult, stats);
        ev_marked = ~0ull;
      } else {
        enqueue_round(d_ops, d_src, d_dst, B, mult, false, false);
        sharded_layers(mult, stats);
      }
    } else if (!baseline && !khop && use_graphs) {
      if (!graph.exec || graph.B != B || graph.mult != mult || graph.profile != opts.profile_kernels ||
          graph.emit_gate != opts.emit_changed_only || graph.epoch != alloc_epoch().load()) {
        if (graph.exec) SGB_CUDA(cudaGraphExecDestroy(graph.exec));
        graph.exec = nullptr;
        cudaGraph_t g = nullptr;
        SGB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        enqueue_round(d_ops, d_src, d_dst, B, mult, true);
        SGB_CUDA(cudaStreamEndCapture(st, &g));
        {
          size_t nn = 0;
          SGB_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
          std::vector<cudaGraphNode_t> nodes(nn);
          if (nn) SGB_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
          graph.kernel_nodes = 0;
          for (auto nd : nodes) {
            cudaGraphNodeType t;
            SGB_CUDA(cudaGraphNodeGetType(nd, &t));
            if (t == cudaGraphNodeTypeKernel) ++graph.kernel_nodes;
          }
        }
        SGB_CUDA(cudaGraphInstantiate(&graph.exec, g, 0));
        SGB_CUDA(cudaGraphDestroy(g));
        graph.B = B;
        graph.mult = mult;
        graph.profile = opts.profile_kernels;
        graph.emit_gate = opts.emit_changed_only;
        graph.epoch = alloc_epoch().load();
      }
      SGB_CUDA(cudaGraphLaunch(graph.exec, st));
      ev_marked = ~0ull;  // the captured round records every mark
    } else {
      enqueue_round(d_ops, d_src, d_dst, B, mult, !baseline && !khop, !khop);
    }
    if (!sharded && (baseline || khop)) {
      SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      SGB_CUDA(cudaStreamSynchronize(st));
      if (!hs(S_ABORT)) {
        if (khop) {
          khop_recompute();
          refresh_abound();  // a_l rows rewritten outside K8
        }
        if (baseline) baseline_counters(stats);
      }
      enqueue_commit();
    }
    // the results (not the trailing graph commit) complete the call; profiled
    // rounds wait for every mark
    if (opts.profile_kernels) SGB_CUDA(cudaStreamSynchronize(st));
    else SGB_CUDA(cudaEventSynchronize(ev_result));
    if (hs(S_XERR))
      fail(Errc::unknown, "shard exchange timed out: a peer shard stopped applying rounds (the engine is unusable)");
    const unsigned long long ab = hs(S_ABORT);
    if (!ab) break;
    AdjView ov = out.view(pool.as<uint32_t>()), iv = in.view(pool.as<uint32_t>());
    if (B && B <= kGroupCap)  // grouped path: original 64-bit keys in batch order
      pdl_launch(k_reset_plan, grid_for(B), 256, 0, st, b_keys.as<uint64_t>(), B, N, 32, ov, iv);
    else if (B)
      pdl_launch(k_reset_plan, grid_for(B), 256, 0, st, b_keys_s.as<uint64_t>(), B, N, key_bits(), ov, iv);
    SGB_CUDA(cudaStreamSynchronize(st));
    if (ab == 3 && attempt < 4) {  // slab pool too small for this round's relocations: grow, replay
      uint64_t top = 0;
      SGB_CUDA(copy_sync(st, &top, pool_top.p, 8, cudaMemcpyDeviceToHost));
      grow_pool(hs(S_RELOC_DEMAND), top);
      continue;
    }
    if (hs(S_BADOP)) fail(Errc::invalid_argument, "op must be '+' or '-'");
    const unsigned long long err = hs(S_ERR);
    if (err == ~0ull) fail(Errc::unknown, "slab pool exhausted");
    const uint32_t seq = static_cast<uint32_t>(err >> 8);
    uint32_t s = 0, t = 0;
    if (on_device) {
      SGB_CUDA(copy_sync(st, &s, d_src + seq, 4, cudaMemcpyDeviceToHost));
      SGB_CUDA(copy_sync(st, &t, d_dst + seq, 4, cudaMemcpyDeviceToHost));
    } else {
      s = src[seq];
      t = dst[seq];
    }
    const std::string e = std::to_string(s) + "->" + std::to_string(t);
    switch (err & 0xFF) {
      case ERR_RANGE: fail(Errc::invalid_argument, "node id out of range: " + std::to_string(s >= N ? s : t));
      case ERR_DUP: fail(Errc::duplicate_edge, "insert of existing edge " + e);
      default: fail(Errc::missing_edge, "delete of missing edge " + e);
    }
  }

  // ---- bookkeeping and stats
  const uint64_t ins = hs(S_NET_INS), del = hs(S_NET_DEL), num_net = hs(S_NUM_NET);
  E = E + ins - del;
  in_entries += ins;
  out_entries += ins;
  h_tombs += del;
  stats.num_updates = count;
  stats.layers.resize(k);
  unsigned long long* hc = h_ctr.as<unsigned long long>();
  const bool khop = opts.khop_recompute;
  if (khop) {
    // k-hop comparator: every member of need[l+1] is a recompute target; its
    // self-message read (CountingApplyContext, baseline.cpp:199) is counted here.
    for (int l = 1; l <= k; ++l) {
      unsigned long long* c = hc + static_cast<size_t>(l) * C_NUM;
      c[C_TARGETS] = c[C_RECOMPUTES] = kh_need[l + 1];
      const unsigned long long self = model->user_ops_in(l - 1) > 0 ? kh_need[l + 1] : 0;
      c[l == 1 ? C_FETCH_L1MSG : C_FETCH_OTHER] += self;
    }
  }
  unsigned long long l1 = 0, other = 0;
  kt.recompute_bytes = kt.classify_bytes = kt.events_bytes = 0;
  kt.filter_entries = kt.filter_code_pairs = kt.filter_rows = 0;
  for (int l = 1; l <= k; ++l) {
    const unsigned long long* c = hc + static_cast<size_t>(l) * C_NUM;
    n_dirty_host[l] = static_cast<uint32_t>(hs(L(l, L_NDIRTY)));
    // seeds: all of them unless sharded (then the all-reduced owned counts)
    const uint64_t seed_rows = khop ? 0 : (sharded ? c[C_SEEDS] : num_net);
    LayerStats& Ls = stats.layers[l - 1];
    Ls.events = c[C_EVENTS] + seed_rows * mult;
    Ls.grouped_targets = c[C_TARGETS];
    Ls.user_targets = c[C_USER_TARGETS];
    Ls.no_deletion = c[C_NO_DEL];
    Ls.deletion_no_effect = c[C_DEL_NO_EFFECT];
    Ls.covered_reset = c[C_COVERED];
    Ls.exposed_reset = c[C_EXPOSED];
    Ls.recomputes = c[C_RECOMPUTES];
    Ls.dirty_nodes = sharded ? c[C_DIRTY] : n_dirty_host[l];
    const unsigned long long fl1 = c[C_FETCH_L1MSG] + (l == 1 ? seed_rows : 0);
    const unsigned long long fo = c[C_FETCH_OTHER] + (l == 1 ? 0 : seed_rows);
    Ls.fetch_rows = fl1 + fo;
    l1 += fl1;
    other += fo;
    // Algorithmic bytes: K3 reads one message row per Add/Del
    // (two per PAIR record), the 8-byte record and the target's alpha row, and
    // writes changed alpha rows; K4 reads every live in-neighbour row and its
    // in-list entry plus alpha_prev.
    const double row = 4.0 * d[l];
    kt.classify_bytes += c[C_EVROWS] * row + static_cast<double>(hs(L(l, L_CURSOR))) * 8.0 + c[C_TARGETS] * row +
                         c[C_AWRITES] * row;
    // K4: the dense path reads each live in-neighbour's whole row and in-list
    // entry; the sparse path reads the entry and one 4-byte value per uncovered
    // position, which moves a whole 32-byte sector (so counted at 32 B); both
    // read alpha_prev and write changed alpha rows.
    kt.recompute_bytes += c[C_RECOMP_ROWS] * (row + 4.0) + c[C_SPARSE_ROWS] * 4.0 + c[C_SPARSE_LOADS] * 32.0 +
                          c[C_EXPOSED] * row + c[C_AWRITES] * row;
    // K2/K7 events (SURVEY.md §8d per-unit bytes, what the algorithm must
    // move, not what L2 re-serves): on a filtered layer one alpha row per
    // grouped target (4 d_l), one 4-byte out-list entry per expanded entry and
    // the old + new rows of each dirty source (2 x 4 d_l); every layer writes
    // its 12-byte records (record + group ordinal) — seeds, kept PAIRs,
    // tombstones, new entries, SELF.
    const bool filt = filtered_layer(l, opts.duplicate_seed_events ? 2u : 1u);
    const double recs = static_cast<double>(hs(L(l, L_CURSOR)));
    if (filt) {
      kt.events_bytes += c[C_TARGETS] * row + c[C_FILTER_ENTS] * 4.0 + 2.0 * n_dirty_host[l - 1] * row + recs * 12.0;
      kt.filter_entries += c[C_FILTER_ENTS];
      kt.filter_code_pairs += c[C_FILTER_BROWS];
      kt.filter_rows += c[C_FILTER_ROWS];
    }
    else
      kt.events_bytes += c[C_EVENTS] * 4.0 + recs * 12.0;
  }
  if (model->has_prefix()) {
    stats.feature_fetches = 0;
    stats.checkpoint_fetches = l1 + other;
  } else {
    stats.feature_fetches = l1;
    stats.checkpoint_fetches = other;
  }
  if (opts.profile_kernels) {
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int l = 1; l <= k && l <= 6; ++l) {
      const int b = 16 + 8 * (l - 1);
      for (int j = 0; j < 7; ++j) t[j] += span(b + j, b + j + 1);
    }
    kt.graph_update = span(0, 2);
    kt.events = t[0];
    kt.sort_group = t[1];
    kt.classify = t[2];
    kt.recompute = t[3];
    kt.compact = t[4];
    kt.combine = t[5];
    kt.finalize = t[6];
    kt.commit = span(11, 12);
    kt.total = span(0, 12);
  }
  if (trace) {
    std::fprintf(stderr, "[sgnn trace] round %u:", round);
    for (int l = 1; l <= k; ++l)
      std::fprintf(stderr, " | l%d runs=%llu seg=%llu cls=%llu work=%llu scr=%llu dirty=%llu rec=%llu sparse=%llu swork=%llu",
                   l, hs(L(l, L_RUNS)), hs(L(l, L_NSEG)), hs(L(l, L_NCLS)), hs(L(l, L_NWORK)), hs(L(l, L_NSCRATCH)),
                   hs(L(l, L_NDIRTY)), hs(L(l, L_CURSOR)), hs(L(l, L_NSPARSE)), hs(L(l, L_NSWORK)));
    if (opts.profile_kernels)
      for (int l = 1; l <= k && l <= 6; ++l) {
        const int b = 16 + 8 * (l - 1);
        std::fprintf(stderr, " | l%d us ev=%.0f sort=%.0f cls=%.0f rec=%.0f col=%.0f comb=%.0f wr=%.0f", l,
                     1e3 * span(b, b + 1), 1e3 * span(b + 1, b + 2), 1e3 * span(b + 2, b + 3), 1e3 * span(b + 3, b + 4),
                     1e3 * span(b + 4, b + 5), 1e3 * span(b + 5, b + 6), 1e3 * span(b + 6, b + 7));
      }
    std::fprintf(stderr, "\n");
  }
  ++round;
  if (round == 0) round = 1;
  return stats;
}

// affected_area / affected_fetch_count / full_fetch_count (baseline.cpp:101-232)
// on the post-delta graph, before commit (live = entries without DEL).
void DeviceEngine::Impl::baseline_counters(RoundStats& s) {
  DevBuf reached, fa, fb, members;
  reached.alloc_exact((N + 3ull) & ~3ull);
  fa.alloc_exact(sizeof(uint32_t) * N + 4);
  fb.alloc_exact(sizeof(uint32_t) * N + 4);
  members.alloc_exact(sizeof(uint32_t) * N + 4);
  SGB_CUDA(cudaMemsetAsync(reached.p, 0, (N + 3ull) & ~3ull, st));
  SGB_CUDA(cudaMemsetAsync(ds(S_FRONT_A), 0, 8 * 4, st));
  AdjView ov = out.view(pool.as<uint32_t>()), iv = in.view(pool.as<uint32_t>());
  pdl_launch(k_seed_area, sms * 2, 256, 0, st, b_net.as<uint64_t>(), ds(S_NUM_NET), reached.as<uint8_t>(),
                                       fa.as<uint32_t>(), ds(S_FRONT_A));
  uint32_t* cur = fa.as<uint32_t>();
  uint32_t* nxt = fb.as<uint32_t>();
  unsigned long long* ncur = ds(S_FRONT_A);
  unsigned long long* nnxt = ds(S_FRONT_B);
  for (int h = 0; h < k; ++h) {  // forward k hops over current out-lists
    SGB_CUDA(cudaMemsetAsync(nnxt, 0, 8, st));
    pdl_launch(k_bfs_expand, sms * 8, 256, 0, st, cur, ncur, ov, reached.as<uint8_t>(), nxt, nnxt);
    std::swap(cur, nxt);
    std::swap(ncur, nnxt);
  }
  // |area(k)| and its member list (the first backward frontier)
  SGB_CUDA(cudaMemsetAsync(ds(S_COUNT), 0, 8 * 2, st));
  SGB_CUDA(cudaMemsetAsync(ds(S_FRONT_A), 0, 8 * 2, st));
  pdl_launch(k_need_count, sms * 4, 256, 0, st, reached.as<uint8_t>(), N, in.len.as<uint32_t>(), in.n_del.as<uint32_t>(), 0,
                                        ds(S_COUNT), ds(S_FRONT_A), members.as<uint32_t>());
  SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  SGB_CUDA(cudaStreamSynchronize(st));
  const unsigned long long area = hs(S_FRONT_A);
  // need sets backwards
  unsigned long long count = 0;
  cur = members.as<uint32_t>();
  ncur = ds(S_FRONT_A);
  nxt = fb.as<uint32_t>();
  nnxt = ds(S_FRONT_B);
  uint32_t* spare = fa.as<uint32_t>();
  for (int l = k; l >= 1; --l) {
    SGB_CUDA(cudaMemsetAsync(ds(S_COUNT), 0, 8 * 2, st));
    const uint32_t self = model->user_ops_in(l - 1) > 0 ? 1u : 0u;
    pdl_launch(k_need_count, sms * 4, 256, 0, st, reached.as<uint8_t>(), N, in.len.as<uint32_t>(), in.n_del.as<uint32_t>(),
                                          self, ds(S_COUNT), ds(S_COUNT2), nullptr);
    SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaStreamSynchronize(st));
    count += hs(S_COUNT) - 0;
    SGB_CUDA(cudaMemsetAsync(nnxt, 0, 8, st));
    pdl_launch(k_bfs_expand, sms * 8, 256, 0, st, cur, ncur, iv, reached.as<uint8_t>(), nxt, nnxt);
    uint32_t* t = cur;
    cur = nxt;
    nxt = (t == members.as<uint32_t>()) ? spare : t;
    std::swap(ncur, nnxt);
  }
  (void)0;
  if (model->has_prefix()) {
    SGB_CUDA(cudaMemsetAsync(ds(S_COUNT), 0, 8 * 2, st));
    pdl_launch(k_need_count, sms * 4, 256, 0, st, reached.as<uint8_t>(), N, in.len.as<uint32_t>(), in.n_del.as<uint32_t>(), 0,
                                          ds(S_COUNT2), ds(S_COUNT), nullptr);
    SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaStreamSynchronize(st));
    count += hs(S_COUNT);
  }
  unsigned long long full = model->has_prefix() ? N : 0;
  const uint64_t e_post = E + hs(S_NET_INS) - hs(S_NET_DEL);
  for (int l = 1; l <= k; ++l) full += e_post + (model->user_ops_in(l - 1) > 0 ? N : 0);
  s.has_baseline = true;
  s.affected_fetches = count;
  s.full_fetches = full;
  s.affected_area_nodes = area;
}

// baseline::affected_inference (baseline.cpp:177-207) on the device, on the
// post-delta graph before commit: area = k forward hops over current out-lists
// from the net delta's endpoints (affected_area, 101-130); need[l] = need[l+1] ∪
// in-neighbours (backward_need_sets, 139-166); then per layer l = 1..k every
// node of need[l+1] gets alpha re-aggregated over its whole current
// in-neighbourhood and its combination re-run — the same exact kernels as the
// whole-graph pass, so the tables equal the incremental path's bit for bit.
// Members are kept in one array in discovery order: need[l] is its prefix of
// length |need[l]|. Layer-1 messages are the (static) features; for prefix
// models the reference re-runs the prefix on need[1] with identical results,
// which this comparator counts but does not redo.
void DeviceEngine::Impl::khop_recompute() {
  AdjView ov = out.view(pool.as<uint32_t>()), iv = in.view(pool.as<uint32_t>());
  kh_reached.ensure((N + 3ull) & ~3ull);
  kh_members.ensure(sizeof(uint32_t) * N + 4);
  SGB_CUDA(cudaMemsetAsync(kh_reached.p, 0, (N + 3ull) & ~3ull, st));
  SGB_CUDA(cudaMemsetAsync(ds(S_FRONT_A), 0, 8 * 2, st));
  uint32_t* M = kh_members.as<uint32_t>();
  uint8_t* reached = kh_reached.as<uint8_t>();
  auto sync_scal = [&] {
    SGB_CUDA(cudaMemcpyAsync(h_scal.p, scal.p, S_NUM * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaStreamSynchronize(st));
  };
  pdl_launch(k_seed_area, sms * 2, 256, 0, st, b_net.as<uint64_t>(), ds(S_NUM_NET), reached, M, ds(S_FRONT_A));
  SGB_CUDA(cudaGetLastError());
  sync_scal();
  uint64_t total = hs(S_FRONT_A), begin = 0;
  // expand the frontier M[begin, total) (its size is in S_FRONT_A) into M[total, ...)
  auto hop = [&](const AdjView& a) {
    SGB_CUDA(cudaMemsetAsync(ds(S_FRONT_B), 0, 8, st));
    pdl_launch(k_bfs_expand, sms * 8, 256, 0, st, M + begin, ds(S_FRONT_A), a, reached, M + total, ds(S_FRONT_B));
    SGB_CUDA(cudaGetLastError());
    SGB_CUDA(cudaMemcpyAsync(ds(S_FRONT_A), ds(S_FRONT_B), 8, cudaMemcpyDeviceToDevice, st));
    sync_scal();
    begin = total;
    total += hs(S_FRONT_B);
  };
  for (int h = 0; h < k; ++h) hop(ov);
  kh_need.assign(k + 2, 0);
  kh_need[k + 1] = total;
  // backward: the first frontier is the whole area
  begin = 0;
  {
    const unsigned long long t = total;
    SGB_CUDA(copy_sync(st, ds(S_FRONT_A), &t, 8, cudaMemcpyHostToDevice));
  }
  for (int l = k; l >= 1; --l) {
    hop(iv);
    kh_need[l] = total;
  }
  // per-layer recompute of need[l+1]
  for (int l = 1; l <= k; ++l) {
    const uint32_t n = static_cast<uint32_t>(kh_need[l + 1]);
    if (n == 0) continue;
    unsigned long long* lctr = ctr.as<unsigned long long>() + static_cast<size_t>(l) * C_NUM;
    kh_nch.ensure(sizeof(uint64_t) * n);
    kh_scan.ensure(sizeof(uint64_t) * n);
    pdl_launch(k_list_chunks, grid_for(n), 256, 0, st, M, n, in.len.as<uint32_t>(), kChunk, kh_nch.as<uint64_t>());
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, kh_nch.as<uint64_t>(), kh_scan.as<uint64_t>(), n, st);
    cub::DeviceScan::ExclusiveSum(cub_temp(tb), tb, kh_nch.as<uint64_t>(), kh_scan.as<uint64_t>(), n, st);
    uint64_t last[2] = {0, 0};
    SGB_CUDA(copy_sync(st, &last[0], kh_scan.as<uint64_t>() + n - 1, 8, cudaMemcpyDeviceToHost));
    SGB_CUDA(copy_sync(st, &last[1], kh_nch.as<uint64_t>() + n - 1, 8, cudaMemcpyDeviceToHost));
    const uint64_t items = last[0] + last[1];
    kh_work.ensure(sizeof(uint64_t) * items);
    SGB_CUDA(cudaMemsetAsync(ds(S_COUNT), 0, 8, st));
    pdl_launch(k_list_work, grid_for(n), 256, 0, st, M, kh_scan.as<uint64_t>(), kh_nch.as<uint64_t>(), n,
                                             kh_work.as<uint64_t>(), scratch_idx.as<uint32_t>(),
                                             remaining.as<uint32_t>(), any_live.as<uint32_t>(), ds(S_COUNT));
    SGB_CUDA(cudaGetLastError());
    sync_scal();
    const uint64_t multi = hs(S_COUNT);
    if (multi) {
      kh_scr.ensure(multi * P[l] * sizeof(int));
      pdl_launch(k_fill_int, sms * 4, 256, 0, st, kh_scr.as<int>(), multi * P[l], is_max ? INT_MIN : INT_MAX);
    }
    AggArgs A{};
    A.work = kh_work.as<uint64_t>();
    A.n_work = nullptr;
    A.n_work_host = items;
    A.update = false;
    A.scratch_idx = scratch_idx.as<uint32_t>();
    A.remaining = remaining.as<uint32_t>();
    A.any_live = any_live.as<uint32_t>();
    A.scratch = kh_scr.as<int>();
    A.in_off = in.off.as<uint64_t>();
    A.in_len = in.len.as<uint32_t>();
    A.in_ent = pool.as<uint32_t>();
    A.msg = msg_rows(l);
    A.agg = agg[l].as<float4>();
    A.V = P[l] / 4;
    A.d = d[l];
    A.chunk = kChunk;
    A.fetch_ctr = lctr + (l == 1 ? C_FETCH_L1MSG : C_FETCH_OTHER);
    if (is_max) launch_aggregate<true>(A, A.V); else launch_aggregate<false>(A, A.V);
    uint32_t op_pitch = 0, od = 0;
    RowSrc x0{agg[l].as<float>(), M, 0, P[l]};
    RowSrc self{msg[l].as<float>(), M, 0, P[l]};
    const float* res = run_program(model->program(l - 1), x0, self, nullptr, n, N, d[l], &op_pitch, &od, nullptr);
    pdl_launch(k_copy_rows, sms * 8, 256, 0, st, RowSrc{res, nullptr, 0, op_pitch}, RowDst{msg[l + 1].as<float>(), M, 0, P[l + 1]},
                                         nullptr, n, od, nullptr);
    SGB_CUDA(cudaGetLastError());
  }
  // the prefix re-run on need[1] (counted, values unchanged)
  if (model->has_prefix()) {
    unsigned long long* c1 = ctr.as<unsigned long long>() + C_NUM;
    pdl_launch(k_add_u64, 1, 1, 0, st, c1 + C_FETCH_L1MSG, kh_need[1]);
    SGB_CUDA(cudaGetLastError());
  }
}

// --------------------------------------------------------- verify / save

// Layer by layer (baseline.cpp:234-256 verify_against_full): m_1 recomputed
// from the features and compared, then for every layer l the aggregate a_l and
// m_{l+1} recomputed from the engine's own m_l (every shard's rows) and
// compared. By induction over the layers this equals comparing against one
// from-scratch full inference, with two scratch tables instead of 2k + 1 (C4's
// per-GPU share would not fit the full set). A sharded engine checks its own
// rows; no collective is needed (it only reads tables that are final).
bool DeviceEngine::verify(uint32_t* layer, uint32_t* stage, uint32_t* node, uint32_t* index) const {
  Impl& I = *p_;
  SGB_CUDA(cudaSetDevice(I.device));
  const size_t rows = I.rows_owned();
  DevBuf ta, tm, res;
  ta.alloc_exact(std::max<size_t>(rows * I.maxP * sizeof(float), 256));
  tm.alloc_exact(std::max<size_t>(rows * I.maxP * sizeof(float), 256));
  res.alloc_exact(8);
  auto first_mismatch = [&](const DevBuf& got, const float* want, uint32_t l) -> unsigned long long {
    if (rows == 0) return ~0ull;
    SGB_CUDA(cudaMemsetAsync(res.p, 0xFF, 8, I.st));
    const unsigned g = std::min<unsigned>(grid_for(static_cast<uint64_t>(rows) * I.d[l]), I.sms * 16);
    pdl_launch(k_first_mismatch, g, 256, 0, I.st, got.as<float>(), want, static_cast<uint32_t>(rows), I.P[l], I.d[l],
               res.as<unsigned long long>());
    unsigned long long r = 0;
    SGB_CUDA(cudaMemcpyAsync(&r, res.p, 8, cudaMemcpyDeviceToHost, I.st));
    SGB_CUDA(cudaStreamSynchronize(I.st));
    return r;
  };
  auto report = [&](unsigned long long r, uint32_t l, uint32_t s) {
    if (layer) *layer = l;
    if (stage) *stage = s;
    if (node) *node = static_cast<uint32_t>(r >> 32) + I.shard_lo;
    if (index) *index = static_cast<uint32_t>(r);
    return false;
  };
  // m_1 (scratch pitch P[1] = the table's)
  std::vector<DevBuf> m1(2);
  m1[1] = std::move(tm);
  I.layer1_messages(m1[1]);
  unsigned long long r = first_mismatch(I.msg[1], m1[1].as<float>(), 1);
  tm = std::move(m1[1]);
  if (r != ~0ull) return report(r, 1, 0);
  Impl::InferPlan plan = I.infer_plan();
  for (int l = 1; l <= I.k; ++l) {
    const ptrdiff_t oa = static_cast<ptrdiff_t>(static_cast<size_t>(I.shard_lo) * I.P[l]);
    const ptrdiff_t om = static_cast<ptrdiff_t>(static_cast<size_t>(I.shard_lo) * I.P[l + 1]);
    I.infer_layer(plan, l, I.msg_rows(l), I.vb<float>(I.msg[l], I.P[l]), ta.as<float>() - oa, tm.as<float>() - om);
    r = first_mismatch(I.agg[l], ta.as<float>(), static_cast<uint32_t>(l));
    if (r != ~0ull) return report(r, static_cast<uint32_t>(l), 1);
    r = first_mismatch(I.msg[l + 1], tm.as<float>(), static_cast<uint32_t>(l + 1));
    if (r != ~0ull) return report(r, static_cast<uint32_t>(l + 1), 0);
  }
  return true;
}

void DeviceEngine::save_checkpoints(const std::string& dir) const {
  const Impl& I = *p_;
  if (I.sharded && I.shard_world > 1)
    fail(Errc::invalid_argument, "save_checkpoints on one shard of a sharded engine: aggregated and output tables "
                                 "are valid on their owners only (read them per shard with read_rows)");
  std::filesystem::create_directories(dir);
  std::ofstream manifest(dir + "/checkpoints.txt", std::ios::trunc);
  if (!manifest) fail(Errc::io, "cannot open for write: " + dir + "/checkpoints.txt");
  manifest << "nodes " << I.N << '\n' << "layers " << I.k << '\n';
  std::vector<float> host;
  for (int l = 1; l <= I.k + 1; ++l) {
    host.resize(static_cast<size_t>(I.N) * I.d[l]);
    I.download_table(I.msg[l], I.P[l], I.d[l], host.data());
    const std::string name = "msg_" + std::to_string(l) + ".tnsr";
    write_matrix(dir + "/" + name, I.N, I.d[l], host.data());
    manifest << "msg " << l << ' ' << name << '\n';
  }
  for (int l = 1; l <= I.k; ++l) {
    host.resize(static_cast<size_t>(I.N) * I.d[l]);
    I.download_table(I.agg[l], I.P[l], I.d[l], host.data());
    const std::string name = "agg_" + std::to_string(l) + ".tnsr";
    write_matrix(dir + "/" + name, I.N, I.d[l], host.data());
    manifest << "agg " << l << ' ' << name << '\n';
  }
  if (!manifest) fail(Errc::io, "write failed: checkpoint manifest");
}

void DeviceEngine::save_graph(const std::string& path) const {
  const Impl& I = *p_;
  std::vector<uint64_t> off(I.N);
  std::vector<uint32_t> len(I.N);
  SGB_CUDA(copy_sync(I.st, off.data(), I.out.off.p, I.N * 8ull, cudaMemcpyDeviceToHost));
  SGB_CUDA(copy_sync(I.st, len.data(), I.out.len.p, I.N * 4ull, cudaMemcpyDeviceToHost));
  uint64_t top = 0;
  SGB_CUDA(copy_sync(I.st, &top, I.pool_top.p, 8, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> pool(top);
  SGB_CUDA(copy_sync(I.st, pool.data(), I.pool.p, top * 4, cudaMemcpyDeviceToHost));
  std::vector<uint64_t> csr(I.N + 1, 0);
  for (uint32_t v = 0; v < I.N; ++v) csr[v + 1] = csr[v] + len[v];
  std::vector<NodeId> targets(csr[I.N]);
  for (uint32_t v = 0; v < I.N; ++v) {
    std::copy(pool.begin() + static_cast<long>(off[v]), pool.begin() + static_cast<long>(off[v] + len[v]),
              targets.begin() + static_cast<long>(csr[v]));
    std::sort(targets.begin() + static_cast<long>(csr[v]), targets.begin() + static_cast<long>(csr[v + 1]));
  }
  save_edge_list_csr(I.N, csr.data(), targets.data(), path);
}

}  // namespace sgb
