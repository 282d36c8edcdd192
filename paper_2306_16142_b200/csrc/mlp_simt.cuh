// fp32 MLP engine on CUDA cores (FFMA) -- the "fp32 mode" of the DDF MLP.
//
// Restates ddfield/neural.py:138-157 (forward_batch) and :229-249
// (input_gradient_batch) for one tile of M rows held in shared memory:
// activations live transposed as act[k][m] (rows contiguous), weight K-chunks
// stream from L2 into a [KC][NC] staging buffer, each thread owns an
// RM x 8 register tile.  Hidden-layer ReLU masks for the gradient are kept as
// bit words in shared memory (mask[l][n][m/32]).
//
// Exact fp32 arithmetic (no TF32): SURVEY App. B measured max|d|/rms <= 1e-5
// against the float64 reference, inside the 1e-4 tolerance.
#pragma once
#include "ddf_common.cuh"

namespace ddf {
namespace simt {

constexpr int NT = 256;          // threads per CTA
constexpr int TX = 16, TY = 16;  // thread grid over (cols, rows)
constexpr int KC = 32;           // K chunk staged per step
constexpr int NC = 128;          // N chunk (two groups of 64 columns)

template <int M, int KMAX>
struct Smem {
  static constexpr int RM = M / TY;
  static constexpr int ACT = KMAX * M;                  // floats per activation buffer
  static constexpr int MASK_WORDS = (DDF_MAX_LAYERS) * KMAX * (M / 32);
  static constexpr size_t bytes =
      sizeof(float) * (2 * ACT + KC * NC + M * 2) + sizeof(uint32_t) * MASK_WORDS +
      sizeof(double) * M * 8 + sizeof(int) * M * 2;
};

enum EpiMode : int { EPI_RELU = 0, EPI_RELU_MASK = 1, EPI_MASKMUL = 2, EPI_LINEAR = 3 };

// out[n][m] = epi( sum_k in[k][m] * Wkn[k][n] (+ bias[n]) )
// Wkn: [K][N] row-major in global memory (K, N multiples of 16).
template <int M>
__device__ __forceinline__ void gemm_layer(const float* __restrict__ Wkn, const float* __restrict__ bias,
                                           int K, int N, const float* act_in, float* act_out, float* ws,
                                           int mode, uint32_t* mask_out, const uint32_t* mask_in) {
  constexpr int RM = M / TY;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  for (int n0 = 0; n0 < N; n0 += NC) {
    const int nc = min(NC, N - n0);
    float acc[RM][8];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += KC) {
      const int kc = min(KC, K - k0);
      __syncthreads();
      for (int i = tid; i < kc * (NC / 4); i += NT) {
        const int k = i / (NC / 4), q = i % (NC / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q * 4 < nc) v = __ldg(reinterpret_cast<const float4*>(Wkn + (size_t)(k0 + k) * N + n0 + q * 4));
        *reinterpret_cast<float4*>(ws + k * NC + q * 4) = v;
      }
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < kc; ++k) {
        float a[RM];
        if constexpr (RM == 4) {
          float4 t = *reinterpret_cast<const float4*>(act_in + (k0 + k) * M + ty * 4);
          a[0] = t.x; a[1] = t.y; a[2] = t.z; a[3] = t.w;
        } else {
          float2 t = *reinterpret_cast<const float2*>(act_in + (k0 + k) * M + ty * 2);
          a[0] = t.x; a[1] = t.y;
        }
        const float4 w0 = *reinterpret_cast<const float4*>(ws + k * NC + tx * 4);
        const float4 w1 = *reinterpret_cast<const float4*>(ws + k * NC + 64 + tx * 4);
        const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
      }
    }
    // epilogue
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (c >= nc) continue;
      const int n = n0 + c;
      const float bn = (bias != nullptr) ? __ldg(bias + n) : 0.f;
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        const int m = ty * RM + i;
        float v = acc[i][j];
        if (mode == EPI_RELU || mode == EPI_RELU_MASK) {
          v = v + bn;
          const bool on = v > 0.f;
          v = on ? v : 0.f;
          bits |= (on ? 1u : 0u) << i;
        } else if (mode == EPI_MASKMUL) {
          const uint32_t w = mask_in[n * (M / 32) + (m >> 5)];
          v = ((w >> (m & 31)) & 1u) ? v : 0.f;
        }
        act_out[n * M + m] = v;
      }
      if (mode == EPI_RELU_MASK && bits) {
        const int m0 = ty * RM;
        atomicOr(&mask_out[n * (M / 32) + (m0 >> 5)], bits << (m0 & 31));
      }
    }
  }
  __syncthreads();
}

// Head (identity, N = 1): out[m] = sum_k act[k][m] * w[k] + b  (fp32).
// 4 threads per row for M = 64, 8 for M = 32.
template <int M>
__device__ __forceinline__ void head_dot(const float* __restrict__ w, float b, int K, const float* act,
                                         float* out) {
  constexpr int TPR = NT / M;
  const int m = threadIdx.x / TPR, part = threadIdx.x % TPR;
  float s = 0.f;
  for (int k = part; k < K; k += TPR) s = fmaf(act[k * M + m], __ldg(w + k), s);
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (part == 0) out[m] = s + b;
  __syncthreads();
}

}  // namespace simt
}  // namespace ddf
