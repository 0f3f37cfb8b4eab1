// Shard transports for the owner-computes multi-GPU round.
//
// The reference is single-process; its per-layer targets are
// independent (engine.cpp:209-296 touches no cross-target state), so a round
// shards by target ownership with one exchange per layer boundary: every
// shard's dirty nodes of layer l with their previous and new m_{l+1} rows.
//
//   LocalTransport  shards in one process, one host thread each (tests on one
//                   B200, or several GPUs of one process): records are read in
//                   place from the peers' device buffers; host barriers order
//                   the phases.
//   NcclTransport   one process per GPU: counts all-gather, then an
//                   all-gather-v as one NCCL group of broadcasts (one root per
//                   shard, its own count), and a u64 all-reduce for the round
//                   counters — all ordered on the engine's stream.
//                   libnccl.so.2 is loaded at run time (torch's copy when torch
//                   is already in the process), so the engine library has no
//                   link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <vector>

#include "common.hpp"
#include "device/engine.hpp"

namespace sgb {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(Errc::unknown, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------- in-process

struct LocalShared {
  explicit LocalShared(int w) : world(w), ptrs(w), counts(w), sums(w) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void*> ptrs;
  std::vector<uint64_t> counts;
  std::vector<std::vector<unsigned long long>> sums;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
};

class LocalTransport final : public ShardTransport {
 public:
  LocalTransport(std::shared_ptr<LocalShared> sh, int r) : sh_(std::move(sh)), r_(r) {}
  int rank() const override { return r_; }
  int world() const override { return sh_->world; }

  void exchange(const void* send, const unsigned long long* d_count, size_t, void* stream,
                std::vector<const void*>& srcs, std::vector<uint64_t>& counts) override {
    unsigned long long n_local = 0;
    cuda_ok(cudaMemcpyAsync(&n_local, d_count, 8, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)),
            "shard count");
    cuda_ok(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "shard exchange");
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      sh_->ptrs[r_] = send;
      sh_->counts[r_] = n_local;
    }
    sh_->barrier();
    srcs = sh_->ptrs;
    counts = sh_->counts;
  }

  void exchange_done(void* stream) override {
    // peers read this shard's buffer in place: it must not change before every
    // importer is done
    cuda_ok(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "shard import");
    sh_->barrier();
  }

  void allreduce_sum(unsigned long long* dev, size_t n, void* stream) override {
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<unsigned long long> mine(n);
    cuda_ok(cudaMemcpyAsync(mine.data(), dev, n * 8, cudaMemcpyDeviceToHost, st), "allreduce d2h");
    cuda_ok(cudaStreamSynchronize(st), "allreduce d2h");
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      sh_->sums[r_] = mine;
    }
    sh_->barrier();
    std::fill(mine.begin(), mine.end(), 0ull);
    for (const auto& v : sh_->sums)
      for (size_t i = 0; i < n; ++i) mine[i] += v[i];
    sh_->barrier();  // every shard has read every contribution
    cuda_ok(cudaMemcpyAsync(dev, mine.data(), n * 8, cudaMemcpyHostToDevice, st), "allreduce h2d");
    cuda_ok(cudaStreamSynchronize(st), "allreduce h2d");
  }

 private:
  std::shared_ptr<LocalShared> sh_;
  int r_;
};

// ------------------------------------------------------------------- NCCL

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // SGNN_B200_NCCL names a specific libnccl; otherwise the process's already
    // loaded libnccl.so.2 (e.g. torch's) or the system one. RTLD_LOCAL: the
    // engine never exports NCCL symbols to later libraries.
    void* h = nullptr;
    if (const char* path = std::getenv("SGNN_B200_NCCL")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      const char* e = dlerror();
      a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp && a.error.empty()) a.error = std::string("libnccl lacks ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.all_gather, "ncclAllGather");
    sym(a.broadcast, "ncclBroadcast");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  if (!api.error.empty()) fail(Errc::unknown, api.error);
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(Errc::unknown, std::string("NCCL error in ") + what + ": " + nccl().error_string(r));
}

class NcclTransport final : public ShardTransport {
 public:
  NcclTransport(const uint8_t id[128], int rank, int world, int device) : r_(rank), w_(world) {
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&uid, id, 128);
    cuda_ok(cudaSetDevice(device), "nccl init");
    nccl_ok(nccl().comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
    cuda_ok(cudaMalloc(&d_counts_, 8ull * (world + 1)), "nccl counts");
    cuda_ok(cudaMallocHost(&h_counts_, 8ull * (world + 1)), "nccl counts");
  }
  ~NcclTransport() override {
    if (comm_) nccl().comm_destroy(comm_);
    if (recv_) cudaFree(recv_);
    if (d_counts_) cudaFree(d_counts_);
    if (h_counts_) cudaFreeHost(h_counts_);
  }
  int rank() const override { return r_; }
  int world() const override { return w_; }

  void exchange(const void* send, const unsigned long long* d_count, size_t row_bytes, void* stream,
                std::vector<const void*>& srcs, std::vector<uint64_t>& counts) override {
    auto st = static_cast<cudaStream_t>(stream);
    const auto& api = nccl();
    nccl_ok(api.all_gather(d_count, d_counts_, 1, ncclUint64, comm_, st), "counts all-gather");
    cuda_ok(cudaMemcpyAsync(h_counts_, d_counts_, 8ull * w_, cudaMemcpyDeviceToHost, st), "counts d2h");
    cuda_ok(cudaStreamSynchronize(st), "counts");
    counts.assign(h_counts_, h_counts_ + w_);
    const uint64_t total = std::accumulate(counts.begin(), counts.end(), 0ull);
    const size_t need = std::max<size_t>(total * row_bytes, 16);
    if (need > recv_cap_) {
      if (recv_) cuda_ok(cudaFree(recv_), "recv free");
      recv_cap_ = need + need / 4;
      cuda_ok(cudaMalloc(&recv_, recv_cap_), "recv alloc");
    }
    srcs.assign(w_, nullptr);
    nccl_ok(api.group_start(), "group start");
    uint64_t off = 0;
    for (int q = 0; q < w_; ++q) {
      uint8_t* dst = static_cast<uint8_t*>(recv_) + off * row_bytes;
      srcs[q] = dst;
      if (counts[q])
        nccl_ok(api.broadcast(q == r_ ? send : nullptr, dst, counts[q] * row_bytes, ncclUint8, q, comm_, st),
                "broadcast");
      off += counts[q];
    }
    nccl_ok(api.group_end(), "group end");
  }

  void exchange_done(void*) override {}  // the records were copied into this rank's own buffer

  void allreduce_sum(unsigned long long* dev, size_t n, void* stream) override {
    nccl_ok(nccl().all_reduce(dev, dev, n, ncclUint64, ncclSum, comm_, static_cast<cudaStream_t>(stream)),
            "counter all-reduce");
  }

 private:
  int r_, w_;
  ncclComm_t comm_ = nullptr;
  void* recv_ = nullptr;
  size_t recv_cap_ = 0;
  unsigned long long* d_counts_ = nullptr;
  unsigned long long* h_counts_ = nullptr;
};

}  // namespace

std::vector<std::shared_ptr<ShardTransport>> make_local_shard_group(int world) {
  if (world < 1) fail(Errc::invalid_argument, "shard count must be >= 1");
  auto sh = std::make_shared<LocalShared>(world);
  std::vector<std::shared_ptr<ShardTransport>> out;
  for (int r = 0; r < world; ++r) out.push_back(std::make_shared<LocalTransport>(sh, r));
  return out;
}

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId uid;
  nccl_ok(nccl().get_unique_id(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, 128);
}

std::shared_ptr<ShardTransport> make_nccl_transport(const uint8_t id[128], int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) fail(Errc::invalid_argument, "bad shard rank/world");
  return std::make_shared<NcclTransport>(id, rank, world, device);
}

std::vector<uint32_t> shard_bounds(const std::vector<uint32_t>& in_degree, int world) {
  if (world < 1) fail(Errc::invalid_argument, "shard count must be >= 1");
  const uint32_t n = static_cast<uint32_t>(in_degree.size());
  uint64_t total = 0;
  for (uint32_t d : in_degree) total += d + 1ull;
  std::vector<uint32_t> b(world + 1, n);
  b[0] = 0;
  uint64_t acc = 0;
  int r = 1;
  for (uint32_t v = 0; v < n && r < world; ++v) {
    acc += in_degree[v] + 1ull;
    while (r < world && acc * world >= total * static_cast<uint64_t>(r)) b[r++] = v + 1;
  }
  for (int q = 1; q <= world; ++q) b[q] = std::max(b[q], b[q - 1]);
  return b;
}

}  // namespace sgb
