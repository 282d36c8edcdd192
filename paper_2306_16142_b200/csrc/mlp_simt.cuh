// fp32 MLP engine on CUDA cores (FFMA) -- the "fp32 mode" of the DDF MLP.
//
// Restates ddfield/neural.py:138-157 (forward_batch) and :229-249
// (input_gradient_batch) for one tile of M rows held in shared memory:
// activations live transposed as act[k][m] (rows contiguous), weight K-chunks
// stream from L2 into double-buffered [KC][NC] stages (cp.async), each thread owns an
// 8 x 8 (or 8 x 4) register tile.  Hidden-layer ReLU masks for the gradient are kept as
// bit words in shared memory (mask[l][n][m/32]).
//
// Exact fp32 arithmetic (no TF32): SURVEY App. B measured max|d|/rms <= 1e-5
// against the float64 reference, inside the 1e-4 tolerance.
#pragma once
#include "ddf_common.cuh"

namespace ddf {
namespace simt {

constexpr int NT = 256;          // threads per CTA
constexpr int KC = 32;           // K chunk staged per step
constexpr int NC = 256;          // N chunk of a weight stage

template <int M, int KMAX>
struct Smem {
  static constexpr int ACT = KMAX * M;                  // floats per activation buffer
  static constexpr int MASK_WORDS = (DDF_MAX_LAYERS) * KMAX * (M / 32);
  static constexpr size_t bytes =
      sizeof(float) * (2 * ACT + 2 * KC * NC + M * 2) + sizeof(uint32_t) * MASK_WORDS +
      sizeof(double) * M * 8 + sizeof(int) * M * 2;
};

enum EpiMode : int { EPI_RELU = 0, EPI_RELU_MASK = 1, EPI_MASKMUL = 2, EPI_LINEAR = 3 };

// Weight K-chunk [kc][NC] of columns [n0, n0 + nc) -> shared memory with
// cp.async (16 B per copy; columns >= nc are zero-filled).
template <int NCT>
__device__ __forceinline__ void stage_weights(const float* __restrict__ Wkn, int N, int k0, int kc, int n0, int nc,
                                              float* dst) {
  for (int i = threadIdx.x; i < kc * (NCT / 4); i += NT) {
    const int k = i / (NCT / 4), q = i % (NCT / 4);
    const bool in = q * 4 < nc;
    const float* src = in ? Wkn + (size_t)(k0 + k) * N + n0 + q * 4 : Wkn;
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + k * NCT + q * 4);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(in ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// out[n][m] = epi( sum_k in[k][m] * Wkn[k][n] (+ bias[n]) )
// Wkn: [K][N] row-major in global memory (K, N multiples of 16).
// Register tile 8 rows x RN columns per thread: tx = tid % TXM owns rows
// {4 tx + i} and {M/2 + 4 tx + i} (i < 4), ty = tid / TXM owns columns
// {4 ty + j} (+ NCT/2 for the second four when RN = 8) of each chunk -- 64
// FFMA per four 16-byte shared loads at M = 64.  Weight chunks are double-buffered with
// cp.async and each k step's operands are loaded one step ahead.
template <int M, int NCT>
__device__ __forceinline__ void gemm_chunks(const float* __restrict__ Wkn, const float* __restrict__ bias,
                                            int K, int N, const float* act_in, float* act_out, float* ws,
                                            int mode, uint32_t* mask_out, const uint32_t* mask_in) {
  constexpr int RM = 8, TXM = M / RM, TYN = NT / TXM, RN = NCT / TYN;
  static_assert(RN == 4 || RN == 8, "register tile");
  const int tid = threadIdx.x, tx = tid % TXM, ty = tid / TXM;
  // rows {4 tx + i} and {M/2 + 4 tx + i}, i < 4: a warp's 16-byte loads and
  // stores of one half cover 128 contiguous bytes (no bank conflicts)
  const int m0 = tx * 4, mh = M / 2;
  const int nk = (K + KC - 1) / KC;
  auto col = [&](int j) { return RN == 8 ? (j < 4 ? ty * 4 + j : NCT / 2 + ty * 4 + (j - 4)) : ty * 4 + j; };
  for (int n0 = 0; n0 < N; n0 += NCT) {
    const int nc = min(NCT, N - n0);
    float acc[RM][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;
    stage_weights<NCT>(Wkn, N, 0, min(KC, K), n0, nc, ws);
    for (int c = 0; c < nk; ++c) {
      const int k0 = c * KC, kc = min(KC, K - k0);
      if (c + 1 < nk) {
        stage_weights<NCT>(Wkn, N, k0 + KC, min(KC, K - k0 - KC), n0, nc, ws + ((c + 1) & 1) * KC * NCT);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const float* wsc = ws + (c & 1) * KC * NCT + ty * 4;
      const float* ai = act_in + (size_t)k0 * M + m0;
      float4 a0 = *reinterpret_cast<const float4*>(ai), a1 = *reinterpret_cast<const float4*>(ai + mh);
      float4 w0 = *reinterpret_cast<const float4*>(wsc), w1 = w0;
      if constexpr (RN == 8) w1 = *reinterpret_cast<const float4*>(wsc + NCT / 2);
      auto kstep = [&](int k, bool more) {
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        if (more) {   // operands of step k + 1 in flight while step k computes
          a0 = *reinterpret_cast<const float4*>(ai + (k + 1) * M);
          a1 = *reinterpret_cast<const float4*>(ai + (k + 1) * M + mh);
          w0 = *reinterpret_cast<const float4*>(wsc + (k + 1) * NCT);
          if constexpr (RN == 8) w1 = *reinterpret_cast<const float4*>(wsc + (k + 1) * NCT + NCT / 2);
        }
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
      };
      if (kc == KC) {   // full chunk: unrolled, no per-step predicates
#pragma unroll
        for (int k = 0; k < KC; ++k) kstep(k, k + 1 < KC);
      } else {
#pragma unroll 4
        for (int k = 0; k < kc; ++k) kstep(k, k + 1 < kc);
      }
      __syncthreads();   // this buffer is refilled two chunks later
    }
    // epilogue: each half of a thread's rows of one column -> one vector store
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int cc = col(j);
      const bool live = cc < nc;
      const int n = n0 + (live ? cc : 0);
      const float bn = (live && bias != nullptr) ? __ldg(bias + n) : 0.f;
      float v[RM];
      uint32_t bits = 0;   // bit i: row (i < 4 ? m0 + i : mh + m0 + i - 4)
      uint32_t mw = 0u;
      if (mode == EPI_MASKMUL && live) {
        const uint32_t* mk = mask_in + n * (M / 32);
        const uint32_t lo = mk[m0 >> 5] >> (m0 & 31), hi = mk[(mh + m0) >> 5] >> ((mh + m0) & 31);
        mw = (lo & 15u) | ((hi & 15u) << 4);
      }
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        float x = acc[i][j];
        if (mode == EPI_RELU || mode == EPI_RELU_MASK) {
          x = x + bn;
          const bool on = x > 0.f;
          x = on ? x : 0.f;
          bits |= (on ? 1u : 0u) << i;
        } else if (mode == EPI_MASKMUL) {
          x = ((mw >> i) & 1u) ? x : 0.f;
        }
        v[i] = x;
      }
      if (live) {
        *reinterpret_cast<float4*>(act_out + n * M + m0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(act_out + n * M + mh + m0) = make_float4(v[4], v[5], v[6], v[7]);
      }
      if (mode == EPI_RELU_MASK) {
        // mask words: rows [0, 32) ... of each half, OR-ed over the TXM lanes of one row group
        uint32_t lo = (bits & 15u) << (m0 & 31), hi = ((bits >> 4) & 15u) << ((mh + m0) & 31);
#pragma unroll
        for (int o = 1; o < TXM; o <<= 1) {
          lo |= __shfl_xor_sync(0xffffffffu, lo, o);
          hi |= __shfl_xor_sync(0xffffffffu, hi, o);
        }
        if (live && tx == 0) {
          uint32_t* mk = mask_out + n * (M / 32);
          if constexpr (M == 64) {
            mk[0] = lo;
            mk[1] = hi;
          } else {
            mk[0] = lo | hi;
          }
        }
      }
    }
  }
  __syncthreads();
}

// 128-column chunks for layers at most 128 wide (no idle columns), 256 otherwise
template <int M>
__device__ __forceinline__ void gemm_layer(const float* __restrict__ Wkn, const float* __restrict__ bias,
                                           int K, int N, const float* act_in, float* act_out, float* ws,
                                           int mode, uint32_t* mask_out, const uint32_t* mask_in) {
  if constexpr (M == 64) {
    if (N <= 128) {
      gemm_chunks<M, 128>(Wkn, bias, K, N, act_in, act_out, ws, mode, mask_out, mask_in);
      return;
    }
  }
  gemm_chunks<M, NC>(Wkn, bias, K, N, act_in, act_out, ws, mode, mask_out, mask_in);
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
