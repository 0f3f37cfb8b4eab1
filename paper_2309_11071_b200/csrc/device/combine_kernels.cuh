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
// Every output element is therefore one serial dot product; the kernel tiles
// rows x outputs across the CTA (register micro-tiles, 32-deep k slabs
// double-buffered in shared memory) and keeps each accumulator's k order.
// __fmul_rn/__fadd_rn are never contracted into FFMA.
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

constexpr int GBK = 32;  // k-slab depth staged per pipeline step

// Y = epilogue(X . W^T): W is N x K row-major with pitch ldw (floats).
// epilogue: v = flush(acc [+ bias]); if residual: v = flush(R + v); if relu: relu(v).
// BM x BN output tile per CTA of (BM/TM)*(BN/TN) threads, TM x TN accumulators
// per thread; no split-K (that would change the summation order), so small
// dirty sets use small tiles to cover the SMs. k-slabs of GBK are fetched as
// float4 into registers one slab ahead (global latency overlaps the FMUL/FADD
// chains of the current slab) and stored k-major into a double-buffered
// shared tile, one barrier per slab. Every pitch is a multiple of 4 floats
// (pitch_of), so a float4 that starts below K stays inside its row.
// Rows come from a device-resident count (M_dev) so the launch needs no host
// sync; the CTA loops over tiles (persistent grid). A variant only runs when
// m_lo <= M < m_hi, so all variants can be enqueued into one graph.
template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) k_gemm_exact(
    RowSrc X, const float* __restrict__ W, uint32_t ldw, const float* __restrict__ bias, RowSrc R, bool has_residual,
    RowDst Y, const unsigned long long* M_dev, uint32_t M_host, uint32_t m_lo, uint32_t m_hi, uint32_t N, uint32_t K,
    bool relu, const unsigned long long* abort) {
  constexpr int T = (BM / TM) * (BN / TN);
  constexpr int K4 = GBK / 4;             // float4 per row per slab
  constexpr int XV = BM * K4 / T;         // X float4 loads per thread per slab
  constexpr int WV = BN * K4 / T;
  static_assert(XV >= 1 && WV >= 1 && XV * T == BM * K4 && WV * T == BN * K4, "tile/loader shape");
  static_assert(TM == 1 || TM == 2 || TM == 4, "TM");
  static_assert(TN == 1 || TN == 2 || TN == 4, "TN");
  if (abort && *abort) return;
  const uint32_t M = M_dev ? static_cast<uint32_t>(*M_dev) : M_host;
  if (M < m_lo || M >= m_hi) return;
  __shared__ __align__(16) float Xs[2][GBK][BM + 4];
  __shared__ __align__(16) float Ws[2][GBK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const uint32_t tiles_n = (N + BN - 1) / BN;
  const uint32_t tiles = ((M + BM - 1) / BM) * tiles_n;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    const float* xr[XV];
    const float* wr[WV];
#pragma unroll
    for (int q = 0; q < XV; ++q) {
      const int f = tid + q * T, row = f / K4;
      xr[q] = (m0 + row < M) ? X.row(m0 + row) : nullptr;
    }
#pragma unroll
    for (int q = 0; q < WV; ++q) {
      const int f = tid + q * T, row = f / K4;
      wr[q] = (n0 + row < N) ? W + static_cast<size_t>(n0 + row) * ldw : nullptr;
    }
    float4 xg[XV], wg[WV];
    auto fetch = [&](uint32_t k0) {
#pragma unroll
      for (int q = 0; q < XV; ++q) {
        const uint32_t kk = k0 + 4 * ((tid + q * T) % K4);
        xg[q] = (xr[q] && kk < K) ? __ldg(reinterpret_cast<const float4*>(xr[q] + kk)) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < WV; ++q) {
        const uint32_t kk = k0 + 4 * ((tid + q * T) % K4);
        wg[q] = (wr[q] && kk < K) ? __ldg(reinterpret_cast<const float4*>(wr[q] + kk)) : make_float4(0, 0, 0, 0);
      }
    };
    auto stage = [&](int buf) {
#pragma unroll
      for (int q = 0; q < XV; ++q) {
        const int f = tid + q * T, row = f / K4, k = 4 * (f % K4);
        Xs[buf][k + 0][row] = xg[q].x;
        Xs[buf][k + 1][row] = xg[q].y;
        Xs[buf][k + 2][row] = xg[q].z;
        Xs[buf][k + 3][row] = xg[q].w;
      }
#pragma unroll
      for (int q = 0; q < WV; ++q) {
        const int f = tid + q * T, row = f / K4, k = 4 * (f % K4);
        Ws[buf][k + 0][row] = wg[q].x;
        Ws[buf][k + 1][row] = wg[q].y;
        Ws[buf][k + 2][row] = wg[q].z;
        Ws[buf][k + 3][row] = wg[q].w;
      }
    };
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

    fetch(0);
    stage(0);
    __syncthreads();
    int buf = 0;
    for (uint32_t k0 = 0; k0 < K; k0 += GBK, buf ^= 1) {
      const bool more = k0 + GBK < K;
      if (more) fetch(k0 + GBK);
      const uint32_t kmax = min(static_cast<uint32_t>(GBK), K - k0);
#pragma unroll 8
      for (uint32_t k = 0; k < kmax; ++k) {
        float av[TM], bv[TN];
        if constexpr (TM == 4) {
          const float4 t = *reinterpret_cast<const float4*>(&Xs[buf][k][ty * 4]);
          av[0] = t.x; av[1] = t.y; av[2] = t.z; av[3] = t.w;
        } else if constexpr (TM == 2) {
          const float2 t = *reinterpret_cast<const float2*>(&Xs[buf][k][ty * 2]);
          av[0] = t.x; av[1] = t.y;
        } else {
          av[0] = Xs[buf][k][ty];
        }
        if constexpr (TN == 4) {
          const float4 t = *reinterpret_cast<const float4*>(&Ws[buf][k][tx * 4]);
          bv[0] = t.x; bv[1] = t.y; bv[2] = t.z; bv[3] = t.w;
        } else if constexpr (TN == 2) {
          const float2 t = *reinterpret_cast<const float2*>(&Ws[buf][k][tx * 2]);
          bv[0] = t.x; bv[1] = t.y;
        } else {
          bv[0] = Ws[buf][k][tx];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(bv[j], av[i]));
      }
      if (more) stage(buf ^ 1);
      __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const uint32_t m = m0 + ty * TM + i;
      if (m >= M) continue;
      float* yrow = Y.row(m);
      const float* rrow = has_residual ? R.row(m) : nullptr;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const uint32_t n = n0 + tx * TN + j;
        if (n >= N) continue;
        float v = acc[i][j];
        if (bias) v = __fadd_rn(v, bias[n]);
        v = flushz(v);
        if (rrow) v = flushz(__fadd_rn(rrow[n], v));
        if (relu) v = v > 0.0f ? v : 0.0f;
        yrow[n] = v;
      }
    }
  }
}

// gin_self: Y = flush(X + scale * S) (elementwise, separately rounded).
__global__ void k_gin_self(RowSrc X, RowSrc S, float scale, RowDst Y, const unsigned long long* M_dev, uint32_t M_host, uint32_t d,
                           const unsigned long long* abort) {
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
__global__ void k_write_messages(const uint32_t* dirty, const unsigned long long* n_p, const float* Y, uint32_t ypitch,
                                 float* table, uint32_t pitch, uint32_t d, float* old_slab, uint32_t* stamp,
                                 uint32_t* slot, const uint32_t* round_p, uint8_t* changed, unsigned long long* n_changed,
                                 const unsigned long long* abort) {
  if (*abort) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t n = *n_p;
  for (uint64_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
  const uint32_t v = dirty[w];
  float* row = table + static_cast<size_t>(v) * pitch;
  const float* y = Y + static_cast<size_t>(w) * ypitch;
  bool diff = false;
  if (old_slab) {
    float* o = old_slab + static_cast<size_t>(w) * pitch;
    for (uint32_t c = lane; c < pitch; c += 32) {
      const float oldv = row[c];
      const float newv = c < d ? y[c] : 0.0f;
      o[c] = oldv;
      diff |= __float_as_uint(oldv) != __float_as_uint(newv);
      row[c] = newv;
    }
    diff = __any_sync(0xffffffffu, diff);
    if (lane == 0) {
      stamp[v] = *round_p;
      slot[v] = static_cast<uint32_t>(w);
      changed[w] = diff;
      if (diff) atomicAdd(n_changed, 1ull);
    }
  } else {
    for (uint32_t c = lane; c < d; c += 32) row[c] = y[c];
  }
  }
}

}  // namespace sgb
