// Device-resident incremental engine (host-side interface; no CUDA types).
//
// One DeviceEngine owns, in HBM of one B200:
//   * the dynamic graph: out/in adjacency slabs with per-round DEL/NEW flags
//     (device/graph_store.cu) — replaces DynamicGraph (proj/src/core/graph.cpp);
//   * the checkpoint tables m_1..m_{k+1}, a_1..a_k (N x pitch fp32) plus the
//     per-round message pre-images — replaces CheckpointStore
//     (proj/src/core/checkpoint.cpp);
//   * the per-layer event machinery of Engine::process_update_round
//     (proj/src/core/engine.cpp:171-319), executed as sm_100a kernels.
// There is no CPU fallback: construction fails loudly without a CUDA device.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../host_graph.hpp"
#include "../model.hpp"
#include "../stats.hpp"

namespace sgb {

struct EngineOptions {
  bool duplicate_seed_events = false;  // engine.hpp:76-77 of the reference
  bool baseline_counters = false;
  bool profile_kernels = false;        // per-kernel-class CUDA-event timing (bench/roofline)
  // Comparator mode: each round recomputes the whole k-hop affected area from
  // scratch (baseline::affected_inference, proj/src/core/baseline.cpp:177-207)
  // instead of running the incremental event path. Same tables, bit for bit.
  bool khop_recompute = false;
  // North-star item 5 (not in the reference): a dirty node whose m_{l+1} is
  // bitwise unchanged emits no next-layer events. The reference emits Del/Add
  // for every dirty node (engine.cpp:276-283); such pairs cannot change any
  // aggregate, so tables and dirty sets stay identical while the event,
  // target, condition and fetch counters shrink. Off by default.
  bool emit_changed_only = false;
};

// Per-kernel-class device time of the last round (ms), when profile_kernels is on.
struct KernelTimes {
  double graph_update = 0, events = 0, sort_group = 0, classify = 0, recompute = 0, compact = 0, combine = 0,
         finalize = 0, commit = 0, total = 0;
  // Algorithmic bytes of the recompute (K4), classify (K3) and event-expansion
  // filter (K7, k_expand_filter) kernels in the last round.
  double recompute_bytes = 0, classify_bytes = 0, events_bytes = 0;
  // The filter's work in the last round (layers >= 2): out-list entries walked,
  // PAIRs tested against the alpha bound codes, and rows read (two source rows
  // per 32-entry task plus the exact alpha rows of PAIRs the codes left open).
  double filter_entries = 0, filter_code_pairs = 0, filter_rows = 0;
};

// Host-side collectives between the shards of one partitioned graph
// (owner-computes). One object per shard; every shard
// calls the same sequence. Device data never goes through the transport: each
// shard offers its allocations once (share_device) and reads the peers' rows
// and pack buffers in place through peer memory. Callers synchronize their own
// stream before a collective whenever the peers must see completed device work.
constexpr int kMaxShardsHost = 8;  // shards of one partitioned graph (one B200 box); dev_common.cuh kMaxPeers

class ShardTransport {
 public:
  virtual ~ShardTransport() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  virtual void barrier() = 0;
  // all[r] = shard r's value (a barrier: every shard has published).
  virtual std::vector<uint64_t> all_gather(uint64_t mine) = 0;
  // Element-wise sum over the shards, in place (every shard passes n values).
  virtual void allreduce_sum(unsigned long long* host, size_t n) = 0;
  // Collective: every shard offers one device allocation (its cudaMalloc base
  // pointer, on its own device); returns every shard's allocation as a device
  // address usable by this shard's kernels (the same device, peer access, or a
  // CUDA IPC mapping of another process's allocation).
  virtual std::vector<const void*> share_device(const void* base) = 0;
  // Releases the peer mappings share_device made for this allocation set.
  virtual void unshare_device(const std::vector<const void*>& peers) = 0;
  // True when some shard's memory lives on another GPU (valid after the first
  // share_device): peer rows are then NVLink loads, and the engine keeps its
  // gathers of other shards' rows on plain loads (no bulk-copy engine reads
  // of remote addresses, which only ran same-device in testing).
  virtual bool peers_on_other_devices() const = 0;
};

// `world` transports for shards living in one process (one host thread each),
// on the same or different devices (peer access is enabled between them).
std::vector<std::shared_ptr<ShardTransport>> make_local_shard_group(int world);
// Shards in separate processes of one host (one GPU each, or several on one
// GPU): barriers and small collectives through a POSIX shared-memory segment
// named `name` (created by rank 0), device allocations through CUDA IPC.
std::shared_ptr<ShardTransport> make_shm_transport(const std::string& name, int rank, int world,
                                                   double timeout_s = 600.0);

// Contiguous vertex ranges balancing sum(in-degree + 1) (a target's event and
// recompute work scales with its in-neighbourhood): bounds[r]..bounds[r+1].
std::vector<uint32_t> shard_bounds(const std::vector<uint32_t>& in_degree, int world);

class DeviceEngine {
 public:
  // features: rows x cols row-major (already NaN-checked and -0 flushed).
  // ckpt_dir != nullptr resumes from saved tables instead of full inference.
  // transport != nullptr: this engine is shard transport->rank() of a
  // partitioned graph (collective with the other shards' constructors): it owns
  // the vertex range shard_bounds() gives it and holds only those rows of every
  // table; ckpt_dir must then be null.
  DeviceEngine(const HostGraph& g, std::shared_ptr<const BoundModel> model, const float* features, uint32_t rows,
               uint32_t cols, const char* ckpt_dir, std::shared_ptr<ShardTransport> transport = nullptr);
  ~DeviceEngine();
  DeviceEngine(const DeviceEngine&) = delete;
  DeviceEngine& operator=(const DeviceEngine&) = delete;

  // One round. ops/src/dst are host pointers unless on_device. Throws Error on
  // an invalid batch, leaving graph and tables untouched.
  // on_device: ops/src/dst are device pointers. producer_stream (optional): the
  // cudaStream_t that wrote them; the engine's stream waits for it before the
  // batch is staged (otherwise the caller must have completed that work).
  RoundStats apply(const char* ops, const NodeId* src, const NodeId* dst, size_t count, bool on_device,
                   void* producer_stream = nullptr);

  EngineOptions& options();
  uint32_t num_nodes() const;
  uint64_t num_edges() const;
  int num_layers() const;
  uint32_t dim(int layer, int stage) const;  // validates like CheckpointStore::table
  void read_row(int layer, int stage, NodeId node, float* out) const;
  void read_table(int layer, int stage, float* out) const;  // rows x dim, packed
  // rows [lo, hi) x dim, packed. On a sharded engine the aggregated tables and
  // the output messages m_{k+1} are valid on their owner only: reading rows
  // outside the shard's range of those tables fails with invalid_argument.
  void read_rows(int layer, int stage, uint32_t lo, uint32_t hi, float* out) const;
  std::vector<NodeId> last_dirty(int layer) const;
  // Full inference on the current graph + bitwise compare; true when equal.
  // Collective on a sharded engine (every shard calls it; owned rows compared).
  bool verify(uint32_t* layer, uint32_t* stage, uint32_t* node, uint32_t* index) const;
  void save_checkpoints(const std::string& dir) const;
  void save_graph(const std::string& path) const;
  const KernelTimes& kernel_times() const;
  void shard_range(uint32_t* lo, uint32_t* hi) const;
  // [table bytes this engine holds, graph bytes, device memory in use (cudaMemGetInfo)].
  std::vector<uint64_t> memory_bytes() const;
  // 0 = exact (serial-k fp32, bit-identical to the reference; default),
  // 1 = tcgen05 kind::tf32 with 3xTF32 operand split (fp32-level tolerance),
  // 2 = tcgen05 kind::tf32 single pass. Switching recomputes all tables
  // (collective on a sharded engine).
  void set_combination_mode(int mode);
  int combination_mode() const;
  int device() const;
  bool sharded() const;
  // Kernel nodes of the captured round graph (0 before the first graph round).
  size_t launches_per_round() const;
  void flush_l2() const;
  void* stream() const;  // cudaStream_t

 private:
  struct Impl;
  std::unique_ptr<Impl> p_;
};

bool cuda_device_available(std::string* why);

}  // namespace sgb
