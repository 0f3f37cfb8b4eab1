// Device-side vocabulary shared by the engine kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../common.hpp"

namespace sgb {

#define SGB_CUDA(expr)                                                                                  \
  do {                                                                                                  \
    cudaError_t err__ = (expr);                                                                         \
    if (err__ != cudaSuccess)                                                                           \
      ::sgb::fail(::sgb::Errc::unknown, std::string("CUDA error: ") + cudaGetErrorString(err__) + " at " + \
                                            __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

// Adjacency entries: node id in the low 30 bits, per-round state in the top two.
// A tombstone (DEL) was live before the round and is gone after it; a NEW entry
// was inserted this round. Previous-timestamp view = entries without NEW, current
// view = entries without DEL (the reference's neighbors_prev / neighbors,
// graph.cpp:81-106, without the O(|delta|) inversion).
constexpr uint32_t kNodeMask = 0x3FFFFFFFu;
constexpr uint32_t kFlagDel = 0x80000000u;
constexpr uint32_t kFlagNew = 0x40000000u;
constexpr uint32_t kMaxNodes = 1u << 29;

// Event record: target (32) | index (29) | type (3), sorted on the target bits.
// Seed records index the round's net-delta list; expansion records index the
// previous layer's dirty list, so the source's pre-image row is old_slab[index]
// with no per-node lookup; SELF records carry the target's own user event.
enum : uint32_t { EV_SEED_ADD = 0, EV_SEED_DEL = 1, EV_EXP_ADD = 2, EV_EXP_DEL = 3, EV_EXP_PAIR = 4, EV_SELF = 5 };
constexpr uint32_t kExpandChunk = 256;  // out-list entries per expansion work item
constexpr uint32_t kSparseDims = 8;     // exposed resets with <= this many uncovered positions: sparse recompute
constexpr uint32_t kAggBlockMax = 256;  // K4: most consecutive work items one warp takes in a large round
constexpr uint32_t kSparseChunk = 128;  // in-list entries per sparse recompute work item (C2: 128 beat 256 and 512)

// A message table whose rows are spread over the shards of a partitioned
// engine: shard r holds rows [lo[r], lo[r + 1]) in its
// own HBM, and every shard reaches every row through peer memory (the same
// device, NVLink P2P, or a CUDA IPC mapping of another process's allocation).
// base[r] is shard r's VIRTUAL base (its allocation minus lo[r] rows), so a row
// is base[owner] + v * pitch; an unpartitioned table is base[0] with lo[1..] =
// UINT32_MAX and parts = 1. The owner search (sharded tables only) is seven
// compares against kernel parameters.
constexpr int kMaxPeers = 8;
struct RowTable {
  const float* base[kMaxPeers];
  uint32_t lo[kMaxPeers];
  uint32_t parts;  // shards in the table (1: one allocation, no owner search)
  __device__ __forceinline__ const float* row(uint32_t v, uint32_t pitch) const {
    const float* b = base[0];
    // uniform branch: an unsharded gather is one multiply-add (the search
    // costs ~30 instructions and 14 constant loads per row; at C2 it was
    // most of the instruction stream of a 10^5-target recompute)
    if (parts > 1) {
#pragma unroll
      for (int r = 1; r < kMaxPeers; ++r)
        if (v >= lo[r]) b = base[r];
    }
    return b + static_cast<size_t>(v) * pitch;
  }
  __device__ __forceinline__ const float4* row4(uint32_t v, uint32_t V) const {
    return reinterpret_cast<const float4*>(row(v, 4 * V));
  }
};

// Record slot left by a generator for a target another shard owns.
constexpr uint64_t kNoRecord = ~0ull;

__host__ __device__ inline uint64_t make_record(uint32_t target, uint32_t index, uint32_t type) {
  return (static_cast<uint64_t>(target) << 32) | (static_cast<uint64_t>(index) << 3) | type;
}

// Per-run flag bits written by the classify kernel; RUN_EXACT is set by the
// event generators on targets that need the full group-and-classify path.
enum : uint8_t { RUN_GRP = 1, RUN_SELF = 2, RUN_EXPOSED = 4, RUN_DIRTY = 8, RUN_EXACT = 16 };

// Per-layer device counters (see stats.hpp; fetch split by layer-1 message rows).
enum : int {
  C_EVENTS = 0, C_TARGETS, C_USER_TARGETS, C_NO_DEL, C_DEL_NO_EFFECT, C_COVERED, C_EXPOSED, C_RECOMPUTES,
  C_DIRTY, C_FETCH_L1MSG, C_FETCH_OTHER,
  // measurement-only counters (algorithmic bytes of K2/K7, K3, K4)
  C_EVROWS, C_RECOMP_ROWS, C_AWRITES, C_SPARSE_LOADS, C_FILTER_ROWS, C_FILTER_ENTS,
  // sharded rounds: seeds whose target this shard owns (the host adds all
  // seeds itself when unsharded)
  C_SEEDS,
  C_SPARSE_ROWS,  // live in-neighbour rows visited by the sparse recompute
  C_FILTER_BROWS,  // 16-bit alpha bound rows read by the filter (one per PAIR entry)
  C_NUM
};

// Order-preserving float <-> int32 map for atomicMax/atomicMin reductions
// (valid because NaN is rejected at load and -0 is flushed everywhere).
__device__ __forceinline__ int f2o(float f) {
  int b = __float_as_int(f);
  return b >= 0 ? b : b ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float o2f(int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); }

template <bool IsMax>
__device__ __forceinline__ float sel(float acc, float v) {
  // reduce2 (reference tensor.hpp:19-21): keep acc on ties
  return IsMax ? (v > acc ? v : acc) : (v < acc ? v : acc);
}

// Vector form as single FMNMX instructions: with NaN rejected at load and -0
// flushed on every produced value, fmaxf/fminf select bitwise-identically to
// reduce2 (ties return equal bits either way).
template <bool IsMax>
__device__ __forceinline__ float4 sel4(float4 a, float4 v) {
  if (IsMax) return make_float4(fmaxf(a.x, v.x), fmaxf(a.y, v.y), fmaxf(a.z, v.z), fmaxf(a.w, v.w));
  return make_float4(fminf(a.x, v.x), fminf(a.y, v.y), fminf(a.z, v.z), fminf(a.w, v.w));
}

__device__ __forceinline__ bool neq4(float4 a, float4 b) {
  return __float_as_uint(a.x) != __float_as_uint(b.x) || __float_as_uint(a.y) != __float_as_uint(b.y) ||
         __float_as_uint(a.z) != __float_as_uint(b.z) || __float_as_uint(a.w) != __float_as_uint(b.w);
}

__device__ __forceinline__ float flushz(float x) { return x == 0.0f ? 0.0f : x; }

// 16-bit alpha bound codes for the filter (k_expand_filter). Values are
// oriented so that "inside alpha" means smaller: x = alpha for max, -alpha for
// min (negation is exact). Per layer and position i the table keeps a column
// base b_i and step s_i >= 0 (from the column range of the oriented a_l at the
// last whole-table refresh); code q in 1..65535 stands for the bound
// B(q) = b_i + q * s_i (separately rounded, monotone non-decreasing in q), code 0
// for -inf. Invariant: B(code) <= x. A PAIR whose oriented source value
// u = orient(max/min(old, new)) satisfies u < B(code) at every position has
// old and new strictly inside alpha (no tie, no beat: engine.cpp:45-87) and is
// settled from the codes alone (2 B per position instead of 4); the column
// step keeps the bound within ~range/65534 of alpha, where a bf16 rounding of
// alpha (relative 2^-8) failed for 91% of C2's PAIRs (rows with a small
// relative spread across nodes).
__device__ __forceinline__ float abound_at(uint32_t q, float base, float step) {
  return q == 0 ? -INFINITY : __fadd_rn(base, __fmul_rn(__uint2float_rn(q), step));
}
// Code of an oriented alpha value: some q with B(q) <= x (0 if none found).
// The estimate uses the reciprocal step (inv); only the B() checks decide.
// Codes stop at 65534 so that a threshold stored in 16 bits as
// min(threshold, 65535) still exceeds every code when the true threshold is
// 65536 ("never settled"): capping a code only costs pruning (B is monotone).
__device__ __forceinline__ uint32_t abound_code(float x, float base, float step, float inv) {
  const float t = __fmul_rn(__fsub_rn(x, base), inv);
  uint32_t q = !(t >= 1.0f) ? 0u : (t >= 65534.0f ? 65534u : static_cast<uint32_t>(t));
  if (q && abound_at(q, base, step) > x) {
    --q;
    if (q && abound_at(q, base, step) > x) q = 0;
  }
  return q;
}
// Threshold of an oriented source value: some q >= 1 with B(q) > u, 65536 if
// none found; a position is settled (u < alpha) when code >= threshold.
__device__ __forceinline__ uint32_t abound_threshold(float u, float base, float step, float inv) {
  const float t = __fmul_rn(__fsub_rn(u, base), inv);
  uint32_t q = !(t >= 0.0f) ? 1u : (t >= 65535.0f ? 65536u : static_cast<uint32_t>(t) + 1u);
  if (q <= 65535u && !(abound_at(q, base, step) > u)) {
    ++q;
    if (q <= 65535u && !(abound_at(q, base, step) > u)) q = 65536u;
  }
  return q;
}

// The filter's per-target scalar summary works on the same per-column grid,
// in floats: norm(x) = (x - base_c) * inv_c, a strictly increasing map per
// column for any finite base and positive inv (degenerate columns use inv 1).
// The target side is rounded down, the source side up, so
//   max_c norm_up(u[c]) < min_c norm_dn(alpha[c])  implies  u[c] < alpha[c] for every c
// (norm_dn(a) <= exact(a), exact(u) <= norm_up(u)); no 16-bit saturation or
// quantisation, so only PAIRs within float rounding of the boundary stay open.
__device__ __forceinline__ float colnorm_inv(float inv) { return inv > 0.0f && inv < INFINITY ? inv : 1.0f; }
__device__ __forceinline__ float norm_dn(float x, float base, float inv) {
  return __fmul_rd(__fsub_rd(x, base), colnorm_inv(inv));
}
__device__ __forceinline__ float norm_up(float x, float base, float inv) {
  return __fmul_ru(__fsub_ru(x, base), colnorm_inv(inv));
}

// 16-bit stored threshold of an oriented source value (see abound_code).
template <bool IsMax>
__device__ __forceinline__ uint16_t abound_threshold16(float o, float n, float base, float step, float inv) {
  const float u = IsMax ? fmaxf(o, n) : -fminf(o, n);
  const uint32_t t = abound_threshold(u, base, step, inv);
  return static_cast<uint16_t>(t > 65535u ? 65535u : t);
}

// Programmatic dependent launch (PDL). Every kernel starts with this: wait
// until the preceding kernel in the stream has completed and flushed its
// writes (a no-op when the launch carries no programmatic dependency), then
// let the next kernel's CTAs launch, so its launch latency and prologue hide
// behind this kernel's tail. Safe because every kernel waits before touching
// global memory, and dependents only launch once all of this grid's CTAs are
// resident (each triggers at entry). Round launches set the attribute
// (engine.cu pdl_launch).
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Warp-aggregated counter increment.
__device__ __forceinline__ void warp_add(unsigned long long* ctr, unsigned long long v) {
  unsigned long long s = v;
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(ctr, s);
}

inline uint32_t pitch_of(uint32_t d) { return (d + 3u) & ~3u; }

// Dynamic work distribution for warp-granular kernels: lane 0 takes `batch`
// items at a time from a global cursor, so warps that drew short items keep
// working instead of idling at the tail (static grid-stride assignment left
// ~20% of warp time waiting at block exit on skewed, power-law work).
struct WarpQueue {
  unsigned long long* cursor;  // null = static grid-stride over [0, n)
  uint64_t n;
  uint32_t batch;
  uint64_t cur, end, stride;
  __device__ __forceinline__ void init(unsigned long long* c, uint64_t count, uint32_t b) {
    cursor = c;
    n = count;
    batch = b;
    stride = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    cur = end = 0;
    if (!cursor) {
      cur = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
      end = ~0ull;
    }
  }
  __device__ __forceinline__ bool next(uint64_t& it) {
    if (!cursor) {
      if (cur >= n) return false;
      it = cur;
      cur += stride;
      return true;
    }
    if (cur >= end) {
      unsigned long long b = 0;
      if ((threadIdx.x & 31) == 0) b = atomicAdd(cursor, static_cast<unsigned long long>(batch));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (b >= n) return false;
      cur = b;
      end = b + batch < n ? b + batch : n;
    }
    it = cur++;
    return true;
  }
};

}  // namespace sgb

namespace sgb {

// ---- Blackwell bulk-copy (TMA engine, non-tensor) + mbarrier helpers -------
// A warp stages neighbour rows into a shared-memory ring with
// cp.async.bulk.shared::cluster.global (one instruction per row, completion
// counted in bytes on the slot's mbarrier), so dozens of KB per warp are in
// flight independently of the register file.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_row_load(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace sgb
