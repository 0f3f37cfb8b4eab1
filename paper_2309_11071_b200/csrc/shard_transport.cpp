// Shard transports for the owner-computes multi-GPU round.
//
// The reference is single-process; its per-layer targets are
// independent (engine.cpp:209-296 touches no cross-target state), so a round
// shards by target ownership with one exchange per layer boundary. The tables
// are PARTITIONED (each shard holds its own rows) and every row, pre-image and
// pack buffer is read in place through peer memory, so the transport carries
// only host-side collectives: barriers, per-shard counts, the round counters,
// and the one-time sharing of device allocations.
//
//   LocalTransport  shards in one process, one host thread each (tests on one
//                   B200, or several GPUs of one process with peer access).
//   ShmTransport    one process per shard on one host (the 8 GPUs of one B200
//                   box, or several processes on one GPU): a POSIX shared-memory
//                   segment holds a generation barrier and the collective
//                   slots; device allocations are shared with CUDA IPC
//                   (cudaIpcGetMemHandle / cudaIpcOpenMemHandle), so peers'
//                   rows are NVLink loads. No NCCL on this path.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
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
  explicit LocalShared(int w) : world(w), vals(2, std::vector<uint64_t>(w)), ptrs(w), devs(w), sums(w) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<uint64_t>> vals;  // double-buffered by call parity
  std::vector<const void*> ptrs;
  std::vector<int> devs;
  std::vector<std::vector<unsigned long long>> sums;
  std::set<std::pair<int, int>> peer_enabled;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(600), [&] { return generation != g; })) {
      fail(Errc::unknown, "in-process shard barrier timed out (a shard failed or stopped calling collectives)");
    }
  }
};

class LocalTransport final : public ShardTransport {
 public:
  LocalTransport(std::shared_ptr<LocalShared> sh, int r) : sh_(std::move(sh)), r_(r) {}
  int rank() const override { return r_; }
  int world() const override { return sh_->world; }
  void barrier() override { sh_->barrier(); }

  std::vector<uint64_t> all_gather(uint64_t mine) override {
    // slot parity: a shard can only rewrite a buffer after every shard passed
    // the barrier of the call in between, i.e. finished reading it
    auto& buf = sh_->vals[calls_++ & 1];
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      buf[r_] = mine;
    }
    sh_->barrier();
    std::lock_guard<std::mutex> lk(sh_->mu);
    return buf;
  }

  void allreduce_sum(unsigned long long* host, size_t n) override {
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      sh_->sums[r_].assign(host, host + n);
    }
    sh_->barrier();
    std::vector<unsigned long long> acc(n, 0);
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      for (const auto& v : sh_->sums)
        for (size_t i = 0; i < n; ++i) acc[i] += v[i];
    }
    sh_->barrier();  // every shard has read every contribution
    std::copy(acc.begin(), acc.end(), host);
  }

  std::vector<const void*> share_device(const void* base) override {
    int dev = 0;
    cuda_ok(cudaGetDevice(&dev), "share_device");
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      sh_->ptrs[r_] = base;
      sh_->devs[r_] = dev;
    }
    sh_->barrier();
    std::vector<const void*> out;
    std::vector<int> devs;
    {
      std::lock_guard<std::mutex> lk(sh_->mu);
      out = sh_->ptrs;
      devs = sh_->devs;
    }
    // shards on other devices of this process: direct peer access (NVLink)
    for (int q = 0; q < world(); ++q) {
      if (devs[q] == dev) continue;
      std::lock_guard<std::mutex> lk(sh_->mu);
      if (!sh_->peer_enabled.insert({dev, devs[q]}).second) continue;
      int can = 0;
      cuda_ok(cudaDeviceCanAccessPeer(&can, dev, devs[q]), "peer query");
      if (!can) fail(Errc::unknown, "devices " + std::to_string(dev) + " and " + std::to_string(devs[q]) +
                                        " have no peer access: shards cannot read each other's rows");
      const cudaError_t e = cudaDeviceEnablePeerAccess(devs[q], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_ok(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
    }
    sh_->barrier();  // nobody reuses the slots before every shard has read them
    return out;
  }
  void unshare_device(const std::vector<const void*>&) override {}

  bool peers_on_other_devices() const override {
    std::lock_guard<std::mutex> lk(sh_->mu);
    for (int d : sh_->devs)
      if (d != sh_->devs[r_]) return true;
    return false;
  }

 private:
  std::shared_ptr<LocalShared> sh_;
  int r_;
  uint64_t calls_ = 0;
};

// ----------------------------------------------------------- shared memory

constexpr uint64_t kShmMagic = 0x53474e4e53484d31ull;  // "SGNNSHM1"
constexpr int kShmMaxWorld = kMaxShardsHost;
constexpr size_t kShmMaxVec = 1024;  // u64 values of one all-reduce

struct ShmSlot {
  uint64_t value[2];                     // all_gather, double-buffered by call parity
  unsigned long long vec[2][kShmMaxVec];  // allreduce contributions, likewise
  cudaIpcMemHandle_t handle;
  char bus_id[32];                       // PCI bus id of the shard's GPU (ordinals differ per process)
  int pid;
};

struct ShmSegment {
  std::atomic<uint64_t> magic;
  std::atomic<uint32_t> world;
  std::atomic<uint32_t> arrived;
  std::atomic<uint64_t> generation;
  std::atomic<uint32_t> joined;
  ShmSlot slot[kShmMaxWorld];
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "process-shared atomics need lock-free u64");

class ShmTransport final : public ShardTransport {
 public:
  ShmTransport(const std::string& name, int rank, int world, double timeout_s)
      : name_(name[0] == '/' ? name : "/" + name), r_(rank), w_(world), timeout_s_(timeout_s) {
    if (world < 1 || world > kShmMaxWorld || rank < 0 || rank >= world)
      fail(Errc::invalid_argument, "bad shard rank/world (1 <= world <= " + std::to_string(kShmMaxWorld) + ")");
    const size_t bytes = sizeof(ShmSegment);
    const auto t0 = std::chrono::steady_clock::now();
    if (rank == 0) {
      shm_unlink(name_.c_str());  // a stale segment of an earlier run
      fd_ = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd_ < 0) fail(Errc::io, "cannot create shared-memory segment " + name_);
      if (ftruncate(fd_, static_cast<off_t>(bytes)) != 0) fail(Errc::io, "cannot size shared-memory segment");
    } else {
      for (;;) {  // rank 0 creates it; wait until it exists at full size
        fd_ = shm_open(name_.c_str(), O_RDWR, 0600);
        struct stat sb {};
        if (fd_ >= 0 && fstat(fd_, &sb) == 0 && static_cast<size_t>(sb.st_size) >= bytes) break;
        if (fd_ >= 0) close(fd_);
        fd_ = -1;
        check_timeout(t0, "waiting for rank 0's shared-memory segment");
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0);
    if (p == MAP_FAILED) fail(Errc::io, "cannot map shared-memory segment " + name_);
    seg_ = static_cast<ShmSegment*>(p);
    if (rank == 0) {
      seg_->world.store(static_cast<uint32_t>(world));
      seg_->arrived.store(0);
      seg_->generation.store(0);
      seg_->joined.store(0);
      seg_->magic.store(kShmMagic, std::memory_order_release);
    } else {
      while (seg_->magic.load(std::memory_order_acquire) != kShmMagic) {
        check_timeout(t0, "waiting for rank 0 to initialise the shared-memory segment");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (seg_->world.load() != static_cast<uint32_t>(world))
        fail(Errc::invalid_argument, "shard world size differs from rank 0's");
    }
    seg_->slot[rank].pid = static_cast<int>(getpid());
    seg_->joined.fetch_add(1);
    barrier();
    if (rank == 0) shm_unlink(name_.c_str());  // every rank has it mapped; the name can go
  }

  ~ShmTransport() override {
    for (const void* p : opened_) cudaIpcCloseMemHandle(const_cast<void*>(p));
    if (seg_) munmap(seg_, sizeof(ShmSegment));
    if (fd_ >= 0) close(fd_);
  }

  int rank() const override { return r_; }
  int world() const override { return w_; }

  // Generation barrier: the last arriver resets the count, then bumps the
  // generation everybody else spins on (a process entering the next barrier
  // only does so after seeing the bump, i.e. after the reset).
  void barrier() override {
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t g = seg_->generation.load(std::memory_order_acquire);
    if (seg_->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(w_)) {
      seg_->arrived.store(0, std::memory_order_relaxed);
      seg_->generation.fetch_add(1, std::memory_order_acq_rel);
      return;
    }
    for (uint32_t spins = 0; seg_->generation.load(std::memory_order_acquire) == g; ++spins) {
      if (spins < 2048) continue;
      sched_yield();
      if ((spins & 1023) == 0) check_timeout(t0, "shard barrier");
    }
  }

  std::vector<uint64_t> all_gather(uint64_t mine) override {
    const int par = static_cast<int>(calls_++ & 1);
    seg_->slot[r_].value[par] = mine;
    barrier();
    std::vector<uint64_t> out(w_);
    for (int q = 0; q < w_; ++q) out[q] = seg_->slot[q].value[par];
    return out;
  }

  void allreduce_sum(unsigned long long* host, size_t n) override {
    if (n > kShmMaxVec) fail(Errc::invalid_argument, "all-reduce vector too long for the shared-memory slots");
    const int par = static_cast<int>(calls_++ & 1);
    std::memcpy(seg_->slot[r_].vec[par], host, n * sizeof(unsigned long long));
    barrier();
    std::fill(host, host + n, 0ull);
    for (int q = 0; q < w_; ++q)
      for (size_t i = 0; i < n; ++i) host[i] += seg_->slot[q].vec[par][i];
  }

  std::vector<const void*> share_device(const void* base) override {
    int dev = 0;
    cuda_ok(cudaGetDevice(&dev), "share_device");
    cuda_ok(cudaIpcGetMemHandle(&seg_->slot[r_].handle, const_cast<void*>(base)), "cudaIpcGetMemHandle");
    cuda_ok(cudaDeviceGetPCIBusId(seg_->slot[r_].bus_id, sizeof(seg_->slot[r_].bus_id), dev), "PCI bus id");
    barrier();
    std::vector<const void*> out(w_);
    for (int q = 0; q < w_; ++q) {
      if (q == r_) {
        out[q] = base;
        continue;
      }
      void* p = nullptr;
      cuda_ok(cudaIpcOpenMemHandle(&p, seg_->slot[q].handle, cudaIpcMemLazyEnablePeerAccess),
              "cudaIpcOpenMemHandle");
      out[q] = p;
      opened_.push_back(p);
    }
    barrier();  // the handle slots may be reused after this
    return out;
  }

  bool peers_on_other_devices() const override {
    for (int q = 0; q < w_; ++q)
      if (std::strncmp(seg_->slot[q].bus_id, seg_->slot[r_].bus_id, sizeof(seg_->slot[q].bus_id)) != 0) return true;
    return false;
  }

  void unshare_device(const std::vector<const void*>& peers) override {
    for (int q = 0; q < static_cast<int>(peers.size()); ++q) {
      if (q == r_ || !peers[q]) continue;
      auto it = std::find(opened_.begin(), opened_.end(), peers[q]);
      if (it == opened_.end()) continue;
      cudaIpcCloseMemHandle(const_cast<void*>(peers[q]));
      opened_.erase(it);
    }
  }

 private:
  void check_timeout(std::chrono::steady_clock::time_point t0, const char* what) const {
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (s > timeout_s_) fail(Errc::unknown, std::string("shared-memory shard transport timed out ") + what);
  }

  std::string name_;
  int r_, w_;
  double timeout_s_;
  int fd_ = -1;
  ShmSegment* seg_ = nullptr;
  uint64_t calls_ = 0;
  std::vector<const void*> opened_;
};

}  // namespace

std::vector<std::shared_ptr<ShardTransport>> make_local_shard_group(int world) {
  if (world < 1 || world > kMaxShardsHost)
    fail(Errc::invalid_argument, "shard count must be in 1.." + std::to_string(kMaxShardsHost));
  auto sh = std::make_shared<LocalShared>(world);
  std::vector<std::shared_ptr<ShardTransport>> out;
  for (int r = 0; r < world; ++r) out.push_back(std::make_shared<LocalTransport>(sh, r));
  return out;
}

std::shared_ptr<ShardTransport> make_shm_transport(const std::string& name, int rank, int world, double timeout_s) {
  if (name.empty() || name.find('/', 1) != std::string::npos)
    fail(Errc::invalid_argument, "shared-memory transport name must be a plain name");
  return std::make_shared<ShmTransport>(name, rank, world, timeout_s);
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
