// K6 tensor-core mode: the combination GEMM on the 5th-generation tensor cores.
//
// Opt-in: sgnn_engine_set_option(e, "combination_mode", 1) = 3xTF32 (split
// operands, fp32-level accuracy), 2 = plain TF32 (one pass). The reference's
// matvec_affine (proj/src/core/tensor.cpp:41-53) sums w*x serially in fp32 with
// separately rounded products; tcgen05 kind::tf32 rounds both operands to TF32
// (10-bit mantissa) and accumulates in fp32 in its own order, so m_{l+1} moves in
// the last ~3 significant decimal digits. The mode therefore trades the exact
// mode's bit-parity (default) for tensor-core throughput within the tolerance
// tests/test_gpu_tc.py states (per value |err| <= 2e-5 * max(1, |exact|) for
// 3xTF32 and 1e-2 * max(1, |exact|) for TF32; max abs/rel error printed). It is deterministic: a row's result does not
// depend on its position in the tile, so incremental rounds, the k-hop
// comparator and verify() agree bit for bit among themselves in this mode.
//
// Kernel: CTA = 128 gathered rows x one N tile (<= 256 outputs, multiple of 16);
// 128 threads. Per 32-wide K chunk, every thread cp.asyncs 16-byte pieces of
// the gathered X rows and of W into a 3-stage (split: 2-stage) shared-memory ring laid out as
// the UMMA canonical K-major no-swizzle form (8-row x 16-byte core matrices:
// LBO = 128 B between K-adjacent cores, SBO = 1024 B between 8-row groups);
// one elected thread issues 4 (split: 12) x tcgen05.mma.cta_group::1.kind::tf32
// (M=128, N=tile, K=8) into a TMEM accumulator and tcgen05.commit arrives on the
// stage's mbarrier, which gates the reuse of that stage. Epilogue: each warp
// tcgen05.ld's its 32 TMEM lanes (= rows) 32 columns at a time, adds the bias,
// flushes -0, adds the SAGE residual, applies ReLU — the exact mode's order.
#pragma once

#include <cuda.h>  // CUtensorMap (the map itself is encoded on the host, engine.cu)

#include "combine_kernels.cuh"
#include "dev_common.cuh"

namespace sgb {

constexpr int kTcM = 128;      // rows per CTA (TMEM lanes)
constexpr int kTcK = 32;       // floats of K per stage
constexpr int kTcThreads = 128;

// SPLIT (3xTF32): each operand is split into a TF32 head and a TF32 tail
// (x = hi + lo, hi = rna_tf32(x), lo = x - hi exactly) and the product is
// accumulated as lo_a*hi_b + hi_a*lo_b + hi_a*hi_b — fp32-level accuracy from
// three tensor-core passes. Stages hold [A][B] and, when split, [A_lo][B_lo].
template <bool SPLIT>
struct TcCfg {
  static constexpr int kStages = SPLIT ? 2 : 3;
};
__host__ __device__ constexpr uint32_t tc_ntile(uint32_t n) {
  return n >= 256 ? 256u : ((n + 15u) & ~15u);
}
__host__ __device__ constexpr size_t tc_smem_bytes(uint32_t ntile, bool split) {
  return 1024 + static_cast<size_t>(split ? 2 : 3) * (kTcM + ntile) * kTcK * 4 * (split ? 2 : 1);
}

// Instruction descriptor, kind::tf32: D f32 (bits 4-5 = 1), A/B tf32 (7-9, 10-12
// = 2), both K-major (15, 16 = 0), N >> 3 at 17-22, M >> 4 at 24-28.
__host__ __device__ constexpr uint32_t tc_idesc(uint32_t m, uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// Shared-memory matrix descriptor: start address, LBO, SBO (all >> 4),
// version 1 (bit 46, sm_100), base offset 0, layout SWIZZLE_NONE (bits 61-63 = 0).
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Byte offset of the 16-byte piece (row r, K chunk kc) in a canonical tile.
__device__ __forceinline__ uint32_t tc_off(uint32_t r, uint32_t kc) {
  return (r >> 3) * 1024u + kc * 128u + (r & 7u) * 16u;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

template <bool SPLIT>
__global__ void __launch_bounds__(kTcThreads) k_gemm_tc(RowSrc X, const float* __restrict__ W, uint32_t ldw,
                                                        const float* __restrict__ bias, RowSrc R, bool has_residual,
                                                        RowDst Y, const unsigned long long* M_dev, uint32_t M_host,
                                                        uint32_t N, uint32_t K, bool relu,
                                                        const unsigned long long* abort) {
  pdl_prologue();
  extern __shared__ __align__(1024) unsigned char tsm[];
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  const uint32_t m0 = blockIdx.x * kTcM;
  if (m0 >= M || K == 0) return;
  const uint32_t ntile = tc_ntile(N);
  const uint32_t n0 = blockIdx.y * ntile;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tsm);            // kTcStages + 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tsm + 64);
  unsigned char* stage0 = tsm + 1024;
  constexpr int kTcStages = TcCfg<SPLIT>::kStages;
  const uint32_t a_bytes = kTcM * kTcK * 4, b_bytes = ntile * kTcK * 4;
  const uint32_t stage_bytes = (a_bytes + b_bytes) * (SPLIT ? 2 : 1);
  uint32_t tcols = 32;
  while (tcols < ntile) tcols <<= 1;
  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const uint32_t Kp = (K + 3u) & ~3u;  // rows/weights are zero-padded to a multiple of 4
  const uint32_t kt_n = (Kp + kTcK - 1) / kTcK;
  auto load = [&](uint32_t kt) {
    const uint32_t s = kt % kTcStages;
    const uint32_t sa = smem_u32(stage0 + s * stage_bytes), sb = sa + a_bytes;
    const uint32_t k0 = kt * kTcK;
    // A: 128 rows x 8 pieces
    for (uint32_t c = tid; c < kTcM * 8; c += kTcThreads) {
      const uint32_t r = c >> 3, kc = c & 7, k = k0 + kc * 4;
      const bool ok = m0 + r < M && k < Kp;
      const float* src = ok ? X.row(m0 + r) + k : X.base;
      cp_async16(sa + tc_off(r, kc), src, ok ? 16u : 0u);
    }
    // B: ntile weight rows x 8 pieces
    for (uint32_t c = tid; c < ntile * 8; c += kTcThreads) {
      const uint32_t r = c >> 3, kc = c & 7, k = k0 + kc * 4;
      const bool ok = n0 + r < N && k < Kp;
      const float* src = ok ? W + static_cast<size_t>(n0 + r) * ldw + k : W;
      cp_async16(sb + tc_off(r, kc), src, ok ? 16u : 0u);
    }
  };
  const uint32_t idesc = tc_idesc(kTcM, ntile);
  for (uint32_t p = 0; p + 1 < kTcStages; ++p) {
    if (p < kt_n) load(p);
    cp_async_commit();
  }
  for (uint32_t kt = 0; kt < kt_n; ++kt) {
    const uint32_t nxt = kt + kTcStages - 1;
    if (nxt < kt_n) {
      if (kt >= 1) mbar_wait(&bar[(kt - 1) % kTcStages], ((kt - 1) / kTcStages) & 1u);  // its MMAs drained the slot
      load(nxt);
    }
    cp_async_commit();
    cp_async_wait<kTcStages - 1>();
    if (SPLIT) {  // hi in place, lo into the stage's second half (same offsets)
      __syncthreads();
      float4* hi = reinterpret_cast<float4*>(stage0 + (kt % kTcStages) * stage_bytes);
      float4* lo = reinterpret_cast<float4*>(stage0 + (kt % kTcStages) * stage_bytes + a_bytes + b_bytes);
      for (uint32_t q = tid; q < (a_bytes + b_bytes) / 16; q += kTcThreads) {
        const float4 x = hi[q];
        const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        hi[q] = h;
        lo[q] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
      }
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = smem_u32(stage0 + (kt % kTcStages) * stage_bytes), sb = sa + a_bytes;
      const uint32_t la = sa + a_bytes + b_bytes, lb = la + a_bytes;
#pragma unroll
      for (uint32_t ks = 0; ks < kTcK / 8; ++ks) {
        const uint64_t ad = tc_sdesc(sa + ks * 256u, 128u, 1024u);
        const uint64_t bd = tc_sdesc(sb + ks * 256u, 128u, 1024u);
        const uint32_t acc = (kt | ks) ? 1u : 0u;
        if (SPLIT) {
          tc_mma(tmem, tc_sdesc(la + ks * 256u, 128u, 1024u), bd, idesc, acc);
          tc_mma(tmem, ad, tc_sdesc(lb + ks * 256u, 128u, 1024u), idesc, 1u);
          tc_mma(tmem, ad, bd, idesc, 1u);
        } else {
          tc_mma(tmem, ad, bd, idesc, acc);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar[kt % kTcStages]))
                   : "memory");
    }
  }
  // every MMA of this CTA has completed once the last stage's commit arrived
  mbar_wait(&bar[(kt_n - 1) % kTcStages], ((kt_n - 1) / kTcStages) & 1u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w owns TMEM lanes (rows) 32w .. 32w+31
  const uint32_t r = warp * 32 + lane;
  const bool row_ok = m0 + r < M;
  float* yrow = row_ok ? Y.row(m0 + r) : nullptr;
  const float* rrow = (row_ok && has_residual) ? R.row(m0 + r) : nullptr;
  for (uint32_t c0 = 0; c0 < ntile; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((warp * 32u) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!row_ok) continue;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t n = n0 + c0 + j;
      if (c0 + j >= ntile || n >= N) continue;
      float x = __uint_as_float(v[j]);
      if (bias) x = __fadd_rn(x, bias[n]);
      x = flushz(x);
      if (rrow) x = flushz(__fadd_rn(rrow[n], x));
      if (relu) x = x > 0.0f ? x : 0.0f;
      yrow[n] = x;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
}

// ---- TMA-fed variant (unsharded engines) ----------------------------------
// Same CTA tile, accumulation and epilogue as k_gemm_tc, but the operands are
// staged by the Tensor Memory Accelerator into the 128-byte-swizzled K-major
// layout (one 32-float K chunk = one 128-byte row per matrix row): W by one
// 2-D tile load per stage (box 32 x ntile); the gathered activation rows by
// cp.async.bulk.tensor ... tile::gather4 (four table rows per instruction, 32
// per stage), or one 2-D tile load when the rows are contiguous. One thread
// issues the copies and the MMAs; completion is counted in bytes on the
// stage's "full" mbarrier, reuse gated by the MMAs' tcgen05.commit. STAGES
// sizes the ring (2 stages of the TF32 kernel fit two CTAs per SM).
__host__ __device__ constexpr size_t tma_smem_bytes(uint32_t ntile, bool split, int stages) {
  return 1024 + static_cast<size_t>(stages) * (kTcM + ntile) * kTcK * 4 * (split ? 2 : 1);
}
__device__ __forceinline__ uint64_t tc_sdesc_sw128(uint32_t saddr) {
  // start >> 4, LBO 16 B (unused for swizzled K-major), SBO 1024 B (8 rows x
  // 128 B), version 1, layout SWIZZLE_128B (2) at bits 61-63
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (static_cast<uint64_t>(1024u >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y0, int32_t y1,
                                            int32_t y2, int32_t y3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(smem_u32(bar))
      : "memory");
}

template <bool SPLIT, int STAGES>
__global__ void __launch_bounds__(kTcThreads) k_gemm_tma(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB, RowSrc X,
                                                         const float* __restrict__ bias, RowSrc R, bool has_residual,
                                                         RowDst Y, const unsigned long long* M_dev, uint32_t M_host,
                                                         uint32_t N, uint32_t K, bool relu,
                                                         const unsigned long long* abort) {
  pdl_prologue();
  extern __shared__ __align__(1024) unsigned char tsm[];
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  const uint32_t m0 = blockIdx.x * kTcM;
  if (m0 >= M || K == 0) return;
  const uint32_t ntile = tc_ntile(N);
  const uint32_t n0 = blockIdx.y * ntile;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kS = STAGES;
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);        // [kS]
  uint64_t* done = full + 3;                                // [kS]
  uint64_t* accum = full + 6;                               // single use: every MMA of the tile done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tsm + 64);
  int32_t* rid = reinterpret_cast<int32_t*>(tsm + 128);     // the tile's 128 table rows
  unsigned char* stage0 = tsm + 1024;
  const uint32_t a_bytes = kTcM * kTcK * 4, b_bytes = ntile * kTcK * 4;
  const uint32_t stage_bytes = (a_bytes + b_bytes) * (SPLIT ? 2 : 1);
  uint32_t tcols = 32;
  while (tcols < ntile) tcols <<= 1;
  {
    const uint32_t m = m0 + tid < M ? m0 + tid : m0;  // rows past M repeat a valid one (discarded)
    rid[tid] = static_cast<int32_t>(X.ids ? X.ids[m] : X.offset + m);
  }
  if (tid == 0) {
    for (int i = 0; i < kS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done[i], 1);
    }
    mbar_init(accum, 1);
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const bool gather = X.ids != nullptr;
  const uint32_t Kp = (K + 3u) & ~3u;
  const uint32_t kt_n = (Kp + kTcK - 1) / kTcK;
  auto load = [&](uint32_t kt) {  // thread 0
    const uint32_t s = kt % kS;
    const uint32_t sa = smem_u32(stage0 + s * stage_bytes), sb = sa + a_bytes;
    const int32_t k0 = static_cast<int32_t>(kt * kTcK);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"(a_bytes + b_bytes)
                 : "memory");
    if (gather) {
#pragma unroll 4
      for (uint32_t g = 0; g < kTcM / 4; ++g)
        tma_gather4(sa + g * 512u, &tmA, k0, rid[4 * g], rid[4 * g + 1], rid[4 * g + 2], rid[4 * g + 3], &full[s]);
    } else {
      tma_load_2d(sa, &tmA, k0, rid[0], &full[s]);
    }
    tma_load_2d(sb, &tmB, k0, static_cast<int32_t>(n0), &full[s]);
  };
  const uint32_t idesc = tc_idesc(kTcM, ntile);
  if (tid == 0)
    for (uint32_t p = 0; p + 1 < kS && p < kt_n; ++p) load(p);
  for (uint32_t kt = 0; kt < kt_n; ++kt) {
    const uint32_t s = kt % kS;
    if (tid == 0) {
      const uint32_t nxt = kt + kS - 1;
      if (nxt < kt_n) {
        if (kt >= 1) mbar_wait(&done[(kt - 1) % kS], ((kt - 1) / kS) & 1u);  // its MMAs drained the slot
        load(nxt);
      }
    }
    if (SPLIT) {  // every thread: hi in place, lo into the stage's second half (layout-agnostic)
      mbar_wait(&full[s], (kt / kS) & 1u);
      float4* hi = reinterpret_cast<float4*>(stage0 + s * stage_bytes);
      float4* lo = reinterpret_cast<float4*>(stage0 + s * stage_bytes + a_bytes + b_bytes);
      for (uint32_t q = tid; q < (a_bytes + b_bytes) / 16; q += kTcThreads) {
        const float4 x = hi[q];
        const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        hi[q] = h;
        lo[q] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
      }
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      __syncthreads();
    } else if (tid == 0) {
      mbar_wait(&full[s], (kt / kS) & 1u);
    }
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = smem_u32(stage0 + s * stage_bytes), sb = sa + a_bytes;
      const uint32_t la = sa + a_bytes + b_bytes, lb = la + a_bytes;
#pragma unroll
      for (uint32_t ks = 0; ks < kTcK / 8; ++ks) {  // K = 8 tf32 = 32 bytes along the swizzled row
        const uint64_t ad = tc_sdesc_sw128(sa + ks * 32u), bd = tc_sdesc_sw128(sb + ks * 32u);
        const uint32_t acc = (kt | ks) ? 1u : 0u;
        if (SPLIT) {
          tc_mma(tmem, tc_sdesc_sw128(la + ks * 32u), bd, idesc, acc);
          tc_mma(tmem, ad, tc_sdesc_sw128(lb + ks * 32u), idesc, 1u);
          tc_mma(tmem, ad, bd, idesc, 1u);
        } else {
          tc_mma(tmem, ad, bd, idesc, acc);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&done[s]))
                   : "memory");
    }
  }
  // a dedicated single-use barrier for the epilogue: threads that skipped the
  // K loop cannot phase-track the per-stage barriers
  if (tid == 0)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(accum))
                 : "memory");
  mbar_wait(accum, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t r = warp * 32 + lane;
  const bool row_ok = m0 + r < M;
  float* yrow = row_ok ? Y.row(m0 + r) : nullptr;
  const float* rrow = (row_ok && has_residual) ? R.row(m0 + r) : nullptr;
  for (uint32_t c0 = 0; c0 < ntile; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((warp * 32u) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!row_ok) continue;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t n = n0 + c0 + j;
      if (c0 + j >= ntile || n >= N) continue;
      float x = __uint_as_float(v[j]);
      if (bias) x = __fadd_rn(x, bias[n]);
      x = flushz(x);
      if (rrow) x = flushz(__fadd_rn(rrow[n], x));
      if (relu) x = x > 0.0f ? x : 0.0f;
      yrow[n] = x;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
}

}  // namespace sgb
