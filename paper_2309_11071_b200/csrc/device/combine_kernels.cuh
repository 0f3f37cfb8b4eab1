// K6 — combination over the dirty rows (gathered-row GEMM, exact mode), and
// K7/K8 — message write-back with pre-image capture and change detection.
//
// Arithmetic contract (bit-exact with the reference CPU build):
//   matvec_affine (proj/src/core/tensor.cpp:41-53): acc starts at +0.0f, products
//     added in ascending column order, each product and each sum rounded
//     separately (no FMA), bias added after the loop, -0 flushed;
//   relu (tensor.cpp:55-58): x > 0 ? x : 0;
//   sage_self (hooks.cpp:24-29): x = flush(x + flush(W2 . m_self));
//   gin_self (hooks.cpp:31-36): x = flush(x + scale * m_self), scale = 1.0f + eps.
// Every output element is therefore one serial dot product; k_gemm_bulk tiles
// rows x outputs across the CTA and keeps each accumulator's k order; no
// multiply is ever contracted with its add (see the FMUL2/FADD2 note below).
#pragma once

#include "dev_common.cuh"

namespace sgb {

// Row addressing: row(m) = base + (ids ? ids[m] : offset + m) * pitch (floats).
struct RowSrc {
  const float* base;
  const uint32_t* ids;
  uint32_t offset;
  uint32_t pitch;
  __device__ __forceinline__ const float* row(uint32_t m) const {
    return base + static_cast<size_t>(ids ? ids[m] : offset + m) * pitch;
  }
};
struct RowDst {
  float* base;
  const uint32_t* ids;
  uint32_t offset;
  uint32_t pitch;
  __device__ __forceinline__ float* row(uint32_t m) const {
    return base + static_cast<size_t>(ids ? ids[m] : offset + m) * pitch;
  }
};

// K8 fused into the last GEMM of a layer's combination program: output row m
// (dirty position m, node dirty[m]) goes straight into the owner's row of
// m_{l+1} instead of a staging buffer. With `slab` (a next layer exists) the
// previous value is captured into the pre-image slab (the undo log,
// checkpoint.cpp:64-76), a bitwise change ORs into changed[m] (zeroed by K5;
// engine.cpp:273-287) and the node is stamped (read_prev, checkpoint.cpp:52-57);
// with `thr` the next layer's filter threshold of (old, new) is written too.
// Columns past d stay zero in both tables (the slab is zeroed at allocation).
struct WriteBack {
  float* table;            // m_{l+1}, virtual base (null: plain dense Y write)
  uint32_t pitch;
  const uint32_t* dirty;
  float* slab;             // pre-image slab of layer l+1, row m (null at the last layer)
  uint32_t* changed;
  uint32_t* stamp;
  uint32_t* slot;
  const uint32_t* round;
  uint16_t* thr;           // next layer's per-source thresholds (row m), or null
  const float* tstat;      // next layer's alpha grid (base, step, 1/step per column)
  bool is_max;
};

// ---- bulk-staged exact GEMM (the round's K6 path) -------------------------
// One launch serves every dirty-set size: the CTA picks its tile shape from the
// device-resident row count (no host sync, no idle variant launches inside the
// round graph). Operands are staged per K-chunk with cp.async.bulk into an
// NS-stage ring (completion counted in bytes on each stage's mbarrier), so the
// gathered rows of chunk c+NS stream in from HBM while chunk c is multiplied:
//   X: one bulk copy per gathered row (rows are contiguous, 16-byte aligned),
//      kept [row][k] with a 4-float pad per row (bank offset 4);
//   W: stored in HBM as 32-column panels, Wp[N/32][K][32] (uploaded once), so
//      a chunk of one panel is ONE contiguous bulk copy, kept [panel][k][32].
// (Per-row copies of a transposed W cost one bulk request per k and made the
// copy engine, not the arithmetic, the bound: ~38 cycles per request.)
// Arithmetic: scalar FMUL then FADD per product (the exact contract). Measured
// on B200: separate FMUL+FADD sustain 64 MAC/clk/SM, the packed f32x2 forms
// no more (FFMA2 issues at half rate; FMUL2+FADD2 also need an opaque barrier
// because ptxas contracts them into FFMA2 even with -fmad=false).
constexpr int kGemmCompute = 256;                 // 16 x 16 compute threads (8 warps)
constexpr int kGemmThreads = kGemmCompute + 32;   // + one producer warp
constexpr int kGemmStages = 6;

// BM x BN tile, 256 compute threads = 16 column threads x 16 row threads:
// thread (ty, tx) owns rows ty + 16*i (i < TM) and, in each 32-column panel q
// of the tile, the column pair (2*tx, 2*tx + 1). BM = 16*TM, BN = 16*TN.
// A ninth warp produces: it issues every chunk's bulk copies into the NS-stage
// ring as soon as the stage's previous contents are released (an `empty`
// mbarrier that each compute warp arrives on after its last read), and the
// compute warps wait only on the stage's `full` barrier (completion counted in
// bytes). No CTA-wide barrier per chunk: with one, 16 % of the stall samples
// were warps waiting for the slowest one at every chunk.
// Stage of the running chunk count gc (kept across tiles): gc % NS, fill gc / NS.
template <int BM, int BN, int TM, int TN, int KC>
__device__ __forceinline__ void gemm_bulk_tiles(float* smem, uint64_t* full, uint64_t* empty, const RowSrc& X,
                                                const float* __restrict__ Wp, const float* __restrict__ bias,
                                                const RowSrc& R, bool has_residual, const RowDst& Y, uint32_t M,
                                                uint32_t N, uint32_t K, bool relu, const WriteBack& wb) {
  static_assert(TN == 2 || TN == 4, "TN");
  static_assert(BN == 16 * TN && BM == 16 * TM, "16 x 16 threads");
  static_assert(BM + BN / 32 <= 96, "at most three copies per producer lane");
  constexpr int NS = kGemmStages;
  constexpr int XP = KC + 4;                 // X row pitch in shared memory (floats)
  constexpr int STAGE = BM * XP + KC * BN;   // floats per stage
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const uint32_t Kp = (K + 3u) & ~3u;
  const uint32_t chunks = (Kp + KC - 1) / KC;
  const uint32_t tiles_n = (N + BN - 1) / BN;
  const uint32_t tiles = ((M + BM - 1) / BM) * tiles_n;
  uint32_t gc = 0;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    const uint32_t rows_m = min(static_cast<uint32_t>(BM), M - m0);
    const uint32_t panels = min(static_cast<uint32_t>(BN / 32), (N - n0 + 31) / 32);
    if (tid >= kGemmCompute) {  // ---- producer warp
      const uint32_t lane = tid - kGemmCompute, ncopy = rows_m + panels;
      // this lane's copies (r = lane + 32 u), sources resolved once per tile
      const float* src[3];
      uint32_t dst[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const uint32_t r = lane + 32u * u;
        src[u] = nullptr;
        dst[u] = 0;
        if (r < rows_m) {
          src[u] = X.row(m0 + r);
          dst[u] = r * XP;
        } else if (r < ncopy) {
          const uint32_t q = r - rows_m;
          src[u] = Wp + static_cast<size_t>(n0 / 32 + q) * K * 32;
          dst[u] = BM * XP + q * KC * 32;
        }
      }
      for (uint32_t c = 0; c < chunks; ++c, ++gc) {
        const int st = gc % NS;
        const uint32_t f = gc / NS;
        if (f) mbar_wait(&empty[st], (f - 1) & 1u);  // the compute warps released fill f - 1
        const uint32_t k0 = c * KC;
        const uint32_t xbytes = min(static_cast<uint32_t>(KC), Kp - k0) * 4u;
        const uint32_t kw = min(static_cast<uint32_t>(KC), K - k0);  // panel rows: only k < K exist
        float* xs = smem + st * STAGE;
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])),
                       "r"(xbytes * rows_m + kw * 128u * panels)
                       : "memory");
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const uint32_t r = lane + 32u * u;
          if (r >= ncopy) continue;
          const bool row = r < rows_m;
          const float* sp = row ? src[u] + k0 : src[u] + static_cast<size_t>(k0) * 32;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(xs + dst[u])),
              "l"(sp), "r"(row ? xbytes : kw * 128u), "r"(smem_u32(&full[st]))
              : "memory");
        }
      }
      continue;
    }
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
    // the epilogue's operands that do not depend on the product (bias, and
    // the fused write-back's previous values) are loaded now, so their round
    // trips overlap the K loop instead of following it (the write-back's
    // compare was the kernel's largest single stall)
    float bv[TN], old[TM][TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const uint32_t n = n0 + 32 * (j / 2) + 2 * tx + (j % 2);
      bv[j] = bias && n < N ? bias[n] : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const uint32_t m = m0 + ty + 16 * i;
      const float* trow = wb.table && m < M ? wb.table + static_cast<size_t>(wb.dirty[m]) * wb.pitch : nullptr;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const uint32_t n = n0 + 32 * (j / 2) + 2 * tx + (j % 2);
        old[i][j] = trow && n < N ? trow[n] : 0.0f;
      }
    }
    for (uint32_t c = 0; c < chunks; ++c, ++gc) {
      const int st = gc % NS;
      mbar_wait(&full[st], (gc / NS) & 1u);
      const float* xs = smem + st * STAGE;
      const float* ws = xs + BM * XP;
      const uint32_t kc = min(static_cast<uint32_t>(KC), K - c * KC);
      // one 4-k group: X quads of the thread's rows, then per k the thread's
      // W column pairs; `ks` < 4 only in the last group of the last chunk
      auto group = [&](uint32_t g, int ks) {
        float4 xa[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) xa[i] = *reinterpret_cast<const float4*>(xs + (ty + 16 * i) * XP + 4 * g);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          if (s >= ks) break;
          float2 wv[TN / 2];
          const float* wrow = ws + (4 * g + s) * 32 + 2 * tx;
#pragma unroll
          for (int q = 0; q < TN / 2; ++q) wv[q] = *reinterpret_cast<const float2*>(wrow + q * KC * 32);
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float xv = s == 0 ? xa[i].x : (s == 1 ? xa[i].y : (s == 2 ? xa[i].z : xa[i].w));
#pragma unroll
            for (int q = 0; q < TN / 2; ++q) {
              acc[i][2 * q] = __fadd_rn(acc[i][2 * q], __fmul_rn(wv[q].x, xv));
              acc[i][2 * q + 1] = __fadd_rn(acc[i][2 * q + 1], __fmul_rn(wv[q].y, xv));
            }
          }
        }
      };
      const uint32_t full = kc >> 2;
#pragma unroll 4
      for (uint32_t g = 0; g < full; ++g) group(g, 4);
      if (kc & 3u) group(full, static_cast<int>(kc & 3u));
      __syncwarp();  // the warp is done with stage st
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const uint32_t m = m0 + ty + 16 * i;
      if (m >= M) continue;
      const float* rrow = has_residual ? R.row(m) : nullptr;
      float out[TN];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const uint32_t n = n0 + 32 * (j / 2) + 2 * tx + (j % 2);
        float v = acc[i][j];
        if (n < N) {
          if (bias) v = __fadd_rn(v, bv[j]);
          v = flushz(v);
          if (rrow) v = flushz(__fadd_rn(rrow[n], v));
          if (relu) v = v > 0.0f ? v : 0.0f;
        }
        out[j] = v;
      }
      if (!wb.table) {
        float* yrow = Y.row(m);
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const uint32_t n = n0 + 32 * (j / 2) + 2 * tx + (j % 2);
          if (n < N) yrow[n] = out[j];
        }
        continue;
      }
      // fused K8 (previous values loaded before the K loop)
      const uint32_t node = wb.dirty[m];
      float* trow = wb.table + static_cast<size_t>(node) * wb.pitch;
      bool diff = false;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const uint32_t n = n0 + 32 * (j / 2) + 2 * tx + (j % 2);
        if (n >= N) continue;
        trow[n] = out[j];
        if (wb.slab) {
          wb.slab[static_cast<size_t>(m) * wb.pitch + n] = old[i][j];
          diff |= __float_as_uint(old[i][j]) != __float_as_uint(out[j]);
          if (wb.thr) {
            const float b = wb.tstat[n], st = wb.tstat[wb.pitch + n], inv = wb.tstat[2 * wb.pitch + n];
            wb.thr[static_cast<size_t>(m) * wb.pitch + n] = wb.is_max
                                                                  ? abound_threshold16<true>(old[i][j], out[j], b, st, inv)
                                                                  : abound_threshold16<false>(old[i][j], out[j], b, st, inv);
          }
        }
      }
      if (wb.slab) {
        if (diff) atomicOr(&wb.changed[m], 1u);
        if (n0 == 0 && tx == 0) {
          wb.stamp[node] = *wb.round;
          wb.slot[node] = m;
        }
      }
    }
  }
}

// Tile shape by row count: M < m_ab -> 16x32 (1x2 per thread, 64-k chunks),
// M < m_bc -> 32x32 (2x2, 64-k chunks), else 64x64 (4x4, 32-k chunks); all
// fit gemm_bulk_smem() (~104 KB with 6 stages, two CTAs per SM: the deeper
// ring beat 4 stages at three CTAs per SM, C2 combine 47.0 -> 42.1 us/round,
// C3 40.0 -> 38.3; ncu had 23 % of stalls waiting on the ring).
__host__ __device__ constexpr size_t gemm_stage_bytes(int bm, int bn, int kc) {
  return 4ull * (static_cast<size_t>(bm) * (kc + 4) + static_cast<size_t>(kc) * bn);
}
__host__ __device__ constexpr size_t gemm_bulk_smem() {
  return 128 + kGemmStages * (gemm_stage_bytes(64, 64, 32) > gemm_stage_bytes(32, 32, 64) ? gemm_stage_bytes(64, 64, 32)
                                                                                       : gemm_stage_bytes(32, 32, 64));
}

__global__ void __launch_bounds__(kGemmThreads) k_gemm_bulk(RowSrc X, const float* __restrict__ Wp,
                                                            const float* __restrict__ bias, RowSrc R,
                                                            bool has_residual, RowDst Y,
                                                            const unsigned long long* M_dev, uint32_t M_host,
                                                            uint32_t m_ab, uint32_t m_bc, uint32_t N, uint32_t K,
                                                            bool relu, WriteBack wb, const unsigned long long* abort) {
  pdl_prologue();
  extern __shared__ __align__(128) unsigned char gsm[];
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  if (M == 0 || K == 0) return;
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm);
  uint64_t* empty = full + kGemmStages;
  float* smem = reinterpret_cast<float*>(gsm + 128);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGemmStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kGemmCompute / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (M < m_ab)
    gemm_bulk_tiles<16, 32, 1, 2, 64>(smem, full, empty, X, Wp, bias, R, has_residual, Y, M, N, K, relu, wb);
  else if (M < m_bc)
    gemm_bulk_tiles<32, 32, 2, 2, 64>(smem, full, empty, X, Wp, bias, R, has_residual, Y, M, N, K, relu, wb);
  else
    gemm_bulk_tiles<64, 64, 4, 4, 32>(smem, full, empty, X, Wp, bias, R, has_residual, Y, M, N, K, relu, wb);
}

// gin_self: Y = flush(X + scale * S) (elementwise, separately rounded).
__global__ void k_gin_self(RowSrc X, RowSrc S, float scale, RowDst Y, const unsigned long long* M_dev, uint32_t M_host, uint32_t d,
                           const unsigned long long* abort) {
  pdl_prologue();
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  const uint64_t total = static_cast<uint64_t>(M) * d;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t m = static_cast<uint32_t>(i / d), c = static_cast<uint32_t>(i % d);
    Y.row(m)[c] = flushz(__fadd_rn(X.row(m)[c], __fmul_rn(scale, S.row(m)[c])));
  }
}

__global__ void k_relu_rows(RowSrc X, RowDst Y, const unsigned long long* M_dev, uint32_t M_host, uint32_t d,
                           const unsigned long long* abort) {
  pdl_prologue();
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  const uint64_t total = static_cast<uint64_t>(M) * d;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t m = static_cast<uint32_t>(i / d), c = static_cast<uint32_t>(i % d);
    const float v = X.row(m)[c];
    Y.row(m)[c] = v > 0.0f ? v : 0.0f;
  }
}

__global__ void k_copy_rows(RowSrc X, RowDst Y, const unsigned long long* M_dev, uint32_t M_host, uint32_t d,
                           const unsigned long long* abort) {
  pdl_prologue();
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  const uint64_t total = static_cast<uint64_t>(M) * d;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t m = static_cast<uint32_t>(i / d), c = static_cast<uint32_t>(i % d);
    Y.row(m)[c] = X.row(m)[c];
  }
}

// Warp per dirty row: capture the pre-image of m_{l+1}[v] (undo log,
// checkpoint.cpp:64-76), write the new message, detect a bitwise change
// (engine.cpp:273-275, 287), stamp the node so prev/current views resolve.
//
// With `abound` (layers l >= 2 that the filter reads) the dirty row's 16-bit
// alpha bound row is refreshed from a_l: every
// alpha change of layer l is on a dirty node (engine.cpp:254-266), so the
// bounds stay valid for the next round's filter.
//
// With `thr` (the next layer is filtered against bound codes) the source's
// 16-bit per-position thresholds for layer l+1's filter are written too
// (row w, pitch `pitch`): threshold of max(old, new) (min: of -min) on layer
// l+1's alpha grid `tstat`, 0 past d (never blocks) — computed once per dirty
// source here instead of once per 32-entry filter task.
template <bool IsMax>
__global__ void k_write_messages(const uint32_t* dirty, const unsigned long long* n_p, const float* Y, uint32_t ypitch,
                                 float* table, uint32_t pitch, uint32_t d, float* old_slab, uint32_t* stamp,
                                 uint32_t* slot, const uint32_t* round_p, uint32_t* changed, unsigned long long* n_changed,
                                 const float* agg, uint16_t* abound, const float* abstat, uint32_t apitch,
                                 uint16_t* thr, const float* tstat, const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t n = *n_p;
  for (uint64_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
  const uint32_t v = dirty[w];
  // loads of 8 columns per lane are issued before any store (the buffers do
  // not alias, but the compiler cannot know): one L2 round trip per 256
  // columns instead of one per 32
  constexpr int U = 8;
  if (abound) {
    const float* ar = agg + static_cast<size_t>(v) * apitch;
    uint16_t* br = abound + static_cast<size_t>(v) * apitch;
    for (uint32_t c0 = lane; c0 < apitch; c0 += 32 * U) {
      float av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32u * u;
        av[u] = c < apitch ? ar[c] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32u * u;
        if (c < apitch)
          br[c] = static_cast<uint16_t>(
              abound_code(IsMax ? av[u] : -av[u], abstat[c], abstat[apitch + c], abstat[2 * apitch + c]));
      }
    }
  }
  float* row = table + static_cast<size_t>(v) * pitch;
  const float* y = Y + static_cast<size_t>(w) * ypitch;
  bool diff = false;
  if (old_slab) {
    float* o = old_slab + static_cast<size_t>(w) * pitch;
    for (uint32_t c0 = lane; c0 < pitch; c0 += 32 * U) {
      float ov[U], nv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32u * u;
        ov[u] = c < pitch ? row[c] : 0.0f;
        nv[u] = c < d ? y[c] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32u * u;
        if (c < pitch) {
          o[c] = ov[u];
          diff |= __float_as_uint(ov[u]) != __float_as_uint(nv[u]);
          row[c] = nv[u];
        }
      }
      if (thr) {
        uint16_t* tr = thr + static_cast<size_t>(w) * pitch;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = c0 + 32u * u;
          if (c < pitch)
            tr[c] = c < d ? abound_threshold16<IsMax>(ov[u], nv[u], tstat[c], tstat[pitch + c], tstat[2 * pitch + c])
                          : static_cast<uint16_t>(0);
        }
      }
    }
    diff = __any_sync(0xffffffffu, diff);
    if (lane == 0) {
      stamp[v] = *round_p;
      slot[v] = static_cast<uint32_t>(w);
      changed[w] = diff;
      if (diff) atomicAdd(n_changed, 1ull);
    }
  } else {
    for (uint32_t c0 = lane; c0 < d; c0 += 32 * U) {
      float nv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32u * u;
        nv[u] = c < d ? y[c] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32u * u;
        if (c < d) row[c] = nv[u];
      }
    }
  }
  }
}

// The alpha bound codes of the dirty rows of a_l and their row minimum (the
// filter's per-target scalar summary, below): warp per dirty row, beside the
// combination (it only reads a_l rows the GEMM also only reads). Every alpha
// change of a layer is on a dirty node (engine.cpp:254-266), so summaries stay
// valid for the next round's filter. `abound` may be null (rows of <= 128
// floats keep only the summary).
//
// Per-target summary: cmin[v] = min over positions c < d of norm_dn(alpha_v[c])
// (dev_common.cuh), the oriented alpha normalised per column on the code grid.
// The filter compares it with its PAIR source's umax = max_c norm_up(u[c]):
// umax < cmin gives u[c] < alpha[c] at every position — the PAIR lies strictly
// inside alpha and is settled from 4 bytes of the target. The per-column
// normalisation is what makes one scalar per row discriminate: measured on
// C2's layer-2 PAIRs the scalar test settles the same 99.8 % as the exact
// per-position test (profiles/r02/summary_probe_c2.json); the round-2 16-bit
// form (min code vs max threshold) settled 92 %, losing the rest to code
// quantisation and threshold saturation.
template <bool IsMax>
__device__ __forceinline__ void summarise_row(const float* ar, uint16_t* br, float* cmin_v, const float* abstat,
                                              uint32_t apitch, uint32_t d, uint32_t lane) {
  constexpr int U = 8;
  float mn = INFINITY;
  for (uint32_t c0 = lane; c0 < apitch; c0 += 32 * U) {
    float av[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t c = c0 + 32u * u;
      av[u] = c < apitch ? ar[c] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t c = c0 + 32u * u;
      if (c < apitch) {
        const float x = IsMax ? av[u] : -av[u];
        if (br) br[c] = static_cast<uint16_t>(abound_code(x, abstat[c], abstat[apitch + c], abstat[2 * apitch + c]));
        if (c < d) mn = fminf(mn, norm_dn(x, abstat[c], abstat[2 * apitch + c]));
      }
    }
  }
  for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) *cmin_v = mn;
}

template <bool IsMax>
__global__ void k_refresh_codes(const uint32_t* dirty, const unsigned long long* n_p, const float* agg,
                                uint16_t* abound, float* cmin, const float* abstat, uint32_t apitch, uint32_t d,
                                const unsigned long long* abort) {
  pdl_prologue();
  if (*abort) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t n = *n_p;
  for (uint64_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t v = dirty[w];
    summarise_row<IsMax>(agg + static_cast<size_t>(v) * apitch,
                         abound ? abound + static_cast<size_t>(v) * apitch : nullptr, cmin + v, abstat, apitch, d,
                         lane);
  }
}

// Whole-table summaries (after init, checkpoint load, a combination-mode switch
// or a k-hop round): warp per owned row, codes (when kept) and row minimum.
template <bool IsMax>
__global__ void k_summarise_all(const float* agg, uint16_t* abound, float* cmin, const float* abstat, size_t rows,
                                uint32_t apitch, uint32_t d) {
  pdl_prologue();
  const uint32_t lane = threadIdx.x & 31;
  for (size_t r = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5)
    summarise_row<IsMax>(agg + r * apitch, abound ? abound + r * apitch : nullptr, cmin + r, abstat, apitch, d, lane);
}

// Sharded rounds: the same thresholds for every imported dirty source (the
// owners' K8 computed them for their own rows only).
template <bool IsMax>
__global__ void k_source_thresholds(const uint32_t* dirty, const unsigned long long* n_p, const float* old_slab,
                                    RowTable table, uint32_t pitch, uint32_t d, uint16_t* thr, const float* tstat) {
  pdl_prologue();
  const uint64_t n = *n_p;
  const uint64_t total = n * pitch;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t w = i / pitch;
    const uint32_t c = static_cast<uint32_t>(i % pitch);
    const float o = old_slab[w * pitch + c], nv = table.row(dirty[w], pitch)[c];
    thr[i] = c < d ? abound_threshold16<IsMax>(o, nv, tstat[c], tstat[pitch + c], tstat[2 * pitch + c])
                   : static_cast<uint16_t>(0);
  }
}

// Whole-table refresh of the alpha bounds (after init, checkpoint load, a
// combination-mode switch or a k-hop round rewrote a_l outside K8): column
// range of the oriented table (ordered-int atomics into colr[0..P) = min,
// colr[P..2P) = max), then base/step/1/step per column, then every code.
template <bool IsMax>
__global__ void k_abound_range(const float* agg, size_t n, uint32_t pitch, int* colr) {
  pdl_prologue();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(i % pitch);
    const int o = f2o(IsMax ? agg[i] : -agg[i]);
    atomicMin(&colr[c], o);
    atomicMax(&colr[pitch + c], o);
  }
}
__global__ void k_abound_stats(const int* colr, uint32_t pitch, float* abstat) {
  pdl_prologue();
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < pitch; c += gridDim.x * blockDim.x) {
    float base = o2f(colr[c]);
    float step = __fdiv_rn(__fsub_rn(o2f(colr[pitch + c]), base), 65534.0f);
    if (!(fabsf(base) <= 3.0e38f) || !(step >= 0.0f && step <= 3.0e38f)) {  // no usable grid: never settles
      base = -INFINITY;
      step = 0.0f;
    }
    abstat[c] = base;
    abstat[pitch + c] = step;
    abstat[2 * pitch + c] = step > 0.0f ? __frcp_rn(step) : INFINITY;  // estimate only (abound_code)
  }
}
template <bool IsMax>
__global__ void k_abound_all(const float* agg, uint16_t* abound, const float* abstat, size_t n, uint32_t pitch) {
  pdl_prologue();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(i % pitch);
    abound[i] = static_cast<uint16_t>(
        abound_code(IsMax ? agg[i] : -agg[i], abstat[c], abstat[pitch + c], abstat[2 * pitch + c]));
  }
}

}  // namespace sgb
