// fp32-accurate DDF-MLP engine on the 5th-generation tensor cores: 3xTF32
// split precision (tcgen05.mma kind::tf32, fp32 accumulators in TMEM).
//
// The parity mode the SURVEY (App. B) specifies for configs 1-2: every fp32
// operand x is split as x = hi + lo with hi = tf32(x) (round to nearest) and
// lo = x - hi, and each layer accumulates  A_hi W_hi + A_hi W_lo + A_lo W_hi
// (the A_lo W_lo term is ~2^-22 relative and dropped).  The tensor core
// truncates fp32 operands to tf32 (measured, scratch/tf32_ts.cu), so the
// truncation of lo costs another ~2^-23.  Measured on B200: max |d - d_f64|
// / rms well inside the 1e-4 bound (tests/test_gpu_x3.py).
//
// One persistent CTA per SM, one 128-row tile in flight, ten warps:
//   warp 0      weight producer: per K-step of 8, a [W_hi | W_lo] chunk
//               (N rows x 32 B each, 32B-swizzled, built on the host from the
//               f64 effective weights) global -> shared with cp.async.bulk
//   warp 1      MMA issuer: per K-step  TS(A_hi, W_hi), TS(A_hi, W_lo),
//               SS(A_lo, W_hi)  with A_hi in TMEM (used twice; TS reads no
//               shared memory) and A_lo in shared memory (128B-swizzled fp32)
//   warps 2-9   row warps: encoding and per-layer epilogues
//
// TMEM holds two 256-column regions.  Step s (one dense layer) accumulates
// D_s in region s&1 and reads A_hi from region (s+1)&1.  The epilogue of step
// s works through D_s 32 columns at a time: TMEM -> registers -> bias, ReLU,
// masks -> split -> A_hi written back IN PLACE over the D_s columns it just
// read, A_lo into shared memory; then it releases that 32-column group to the
// MMA warp (a_ready[g]).  Step s+1's K-step k needs only group k/4, so the
// next layer's MMAs start after the first group and the epilogue runs under
// the tensor pipe.  Every write is ordered after the reads it replaces by the
// chain MMA s complete -> epilogue s -> MMA s+1 (see mlp_x3_kernel).
//
// Hidden widths up to 256 (configs 1, 2, 5); wider networks in fp32 mode run
// on the FFMA engine (mlp_simt.cuh).  The gradient program is the bf16
// engine's (mlp_umma.cuh): forward with ReLU bit masks, seed w_head * mask,
// backward chain with W^T images, input gradient out of the last step.
#pragma once
#include "mlp_umma.cuh"

namespace ddf {
namespace x3 {

using umma::Prog;
using umma::Step;
using umma::NetImage;
using umma::E_RELU_A;
using umma::E_HEAD;
using umma::E_RELU_MASK_A;
using umma::E_MASKG_A;
using umma::E_BWD_MASK_A;
using umma::E_BWD_OUT;
using umma::smem_u32;
using umma::mbar_init;
using umma::mbar_wait;
using umma::mbar_arrive;
using umma::mbar_expect_tx;
using umma::bulk_g2s;
using umma::tc_commit;
using umma::tc_after_sync;
using umma::tc_before_sync;
using umma::fence_async_smem;
using umma::sdesc;
using umma::named_sync;
using umma::st_shared_v4;
using umma::tmem_wait_ld;

constexpr int ROWS = 128;
constexpr int NTHREADS = 320;
constexpr int EPI_WARP0 = 2;
constexpr int N_EPI_WARPS = 8;
constexpr int MAXW = 256;            // widest padded hidden layer
constexpr int GROUPS = MAXW / 32;    // A column groups: 32 fp32 columns = one 128 B swizzled row
constexpr int REGION = 256;          // TMEM columns per region
constexpr int MASK_WORDS_PER_CTA = umma::MASK_WORDS_PER_CTA;

// kind::tf32 instruction descriptor: tf32 A/B (format 2), fp32 D, K-major, M = 128
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(ROWS >> 4) << 24);
}
// K-major, 32-byte swizzled canonical layout (one K-step of 8 fp32 per row):
// 8-row groups 256 B apart
__device__ __forceinline__ uint64_t sdesc32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;     // SBO
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;              // SWIZZLE_32B
  return d;
}
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// One K-step of the split product in a single asm block for the converged
// issuer warp (see umma::uni): TS(A_hi, W_hi), TS(A_hi, W_lo), SS(A_lo, W_hi)
// and the commit that frees the weight stage.  Descriptors travel as their low
// words; the high words (SBO, version, swizzle mode) are constants.
constexpr uint32_t SDESC32_HI = (uint32_t)((256 >> 4) | (1u << 14) | (6u << 29));
__device__ __forceinline__ void mma_x3_step_w(uint32_t tmem_d, uint32_t tmem_a, uint32_t bhi_lo, uint32_t blo_lo,
                                              uint32_t alo_lo, uint32_t id, uint32_t acc, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b64 bh, bl, al;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 q, %5, %5;\n\t"
      "mov.b64 bh, {%2, %8};\n\tmov.b64 bl, {%3, %8};\n\tmov.b64 al, {%4, %9};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bh, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bl, %5, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %5, q;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "r"(bhi_lo), "r"(blo_lo), "r"(alo_lo), "r"(id), "r"(acc), "r"(bar), "n"(SDESC32_HI),
      "n"(umma::SDESC_HI)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// tf32 round-to-nearest (ties away) of an fp32 value, as an fp32 bit pattern
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// One 32-column group of one row: hi parts -> TMEM (in place), lo parts ->
// the row's 128 B line of A_lo group g (128B swizzle), then release the group.
// x holds the 32 fp32 values.
__device__ __forceinline__ void put_group(const float (&x)[32], uint32_t tmem_cols, uint32_t alo_line, int r7) {
  uint32_t hi[32];
  float lo[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    hi[e] = tf32_rna(x[e]);
    lo[e] = x[e] - __uint_as_float(hi[e]);
  }
  tmem_st32(tmem_cols, hi);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(alo_line + (uint32_t)(((c ^ r7)) << 4), __float_as_uint(lo[4 * c]), __float_as_uint(lo[4 * c + 1]),
                 __float_as_uint(lo[4 * c + 2]), __float_as_uint(lo[4 * c + 3]));
}
// the MMA warp may read group g once every row warp of its column half has
// stored it: TMEM stores complete, shared stores visible to the async proxy
__device__ __forceinline__ void release_group(uint32_t bar, int lane) {
  tmem_wait_st();
  tc_before_sync();
  fence_async_smem();
  __syncwarp();
  if (lane == 0) mbar_arrive(bar);
}

// Network input columns [32 G, 32 G + 32) of one row, in f64 then split.  The
// first layer's inputs are split from the f64 encoding directly (hi = tf32(u),
// lo = fp32(u - hi)).  PE (EXTENSION, configs 3-5): [u0..u4, {sin(2^o pi u),
// cos(2^o pi u)} o = 0..5]; sincospi of 2^o u is exact argument scaling.
template <int G>
__device__ __forceinline__ void encode_group(bool pe, bool valid, const double (&u)[5], uint32_t tmem_cols,
                                             uint32_t alo_line, int r7) {
  double x[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) x[e] = 0.0;
  if (valid) {
#pragma unroll
    for (int j = 0; j < 5; ++j)
      if (j >= 32 * G && j < 32 * G + 32) x[j - 32 * G] = u[j];
    if (pe) {
#pragma unroll
      for (int o = 0; o < DDF_PE_OCTAVES; ++o)
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const int ks = 5 + 10 * o + j, kc = ks + 5;
          const bool ins = ks >= 32 * G && ks < 32 * G + 32, inc = kc >= 32 * G && kc < 32 * G + 32;
          if (ins || inc) {
            double s, c;
            sincospi(ldexp(u[j], o), &s, &c);
            if (ins) x[ks - 32 * G] = s;
            if (inc) x[kc - 32 * G] = c;
          }
        }
    }
  }
  uint32_t hi[32];
  float lo[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    hi[e] = tf32_rna((float)x[e]);
    lo[e] = (float)(x[e] - (double)__uint_as_float(hi[e]));
  }
  tmem_st32(tmem_cols, hi);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(alo_line + (uint32_t)(((c ^ r7)) << 4), __float_as_uint(lo[4 * c]), __float_as_uint(lo[4 * c + 1]),
                 __float_as_uint(lo[4 * c + 2]), __float_as_uint(lo[4 * c + 3]));
}

// Epilogue of one 32-column group (fully unrolled per kind).  Returns nothing;
// writes A (hi/lo) for the A-writing kinds, accumulates the head dot for E_HEAD.
template <int EPI>
__device__ __forceinline__ void epi_group(const Step& st, int c, int r, uint32_t tmem_d, uint32_t alo_line,
                                          uint32_t* my_masks, const float* head_w, float& head_part,
                                          const float* sparams) {
  uint32_t rg[32];
  DDF_TMEM_LD32(tmem_d, rg);
  float4 bq[8];
  uint32_t mq = 0u;
  if constexpr (EPI != E_BWD_MASK_A) {
#pragma unroll
    for (int k = 0; k < 8; ++k) bq[k] = *reinterpret_cast<const float4*>(sparams + (size_t)st.bias + c + 4 * k);
  } else {
    mq = my_masks[(st.mask_layer * 16 + (c >> 5)) * ROWS + r];
  }
  tmem_wait_ld();
  const float* bf = reinterpret_cast<const float*>(bq);
  float v[32];
  if constexpr (EPI == E_BWD_MASK_A) {
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = ((mq >> e) & 1u) ? __uint_as_float(rg[e]) : 0.f;
  } else if constexpr (EPI == E_RELU_A) {
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = fmaxf(__uint_as_float(rg[e]) + bf[e], 0.f);
  } else if constexpr (EPI == E_HEAD) {
#pragma unroll
    for (int e = 0; e < 32; e += 4) {
      const float4 hw = *reinterpret_cast<const float4*>(head_w + c + e);
      head_part = fmaf(fmaxf(__uint_as_float(rg[e]) + bf[e], 0.f), hw.x, head_part);
      head_part = fmaf(fmaxf(__uint_as_float(rg[e + 1]) + bf[e + 1], 0.f), hw.y, head_part);
      head_part = fmaf(fmaxf(__uint_as_float(rg[e + 2]) + bf[e + 2], 0.f), hw.z, head_part);
      head_part = fmaf(fmaxf(__uint_as_float(rg[e + 3]) + bf[e + 3], 0.f), hw.w, head_part);
    }
  } else {
    // ReLU mask bits of this row's 32 columns (neural.py:241 "h > 0")
    uint32_t mw = 0u;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float z = __uint_as_float(rg[e]) + bf[e];
      mw |= (z > 0.f ? 1u : 0u) << e;
      v[e] = fmaxf(z, 0.f);
    }
    if constexpr (EPI == E_RELU_MASK_A) {
      my_masks[(st.mask_layer * 16 + (c >> 5)) * ROWS + r] = mw;
    } else {   // E_MASKG_A: d/dh of the last hidden layer = w_head * mask
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        const float4 hw = *reinterpret_cast<const float4*>(head_w + c + e);
        v[e] = ((mw >> e) & 1u) ? hw.x : 0.f;
        v[e + 1] = ((mw >> (e + 1)) & 1u) ? hw.y : 0.f;
        v[e + 2] = ((mw >> (e + 2)) & 1u) ? hw.z : 0.f;
        v[e + 3] = ((mw >> (e + 3)) & 1u) ? hw.w : 0.f;
      }
    }
  }
  if constexpr (EPI != E_HEAD) put_group(v, tmem_d, alo_line, r & 7);
}

struct Smem {
  uint8_t* alo;      // A_lo: [GROUPS][128 rows][128 B], 1024-aligned
  uint8_t* stages;   // weight stages [n][W_hi N x 32 B | W_lo N x 32 B]
  uint64_t* bars;    // [0, GROUPS) a_ready, [GROUPS] acc, [GROUPS+1] pad, then full[S], empty[S]
  uint32_t* tmem_slot;
  float* red;        // [2][128] head partial sums
  float* params;     // current network's biases + head weights
};

template <class Op>
__global__ void __launch_bounds__(NTHREADS, 1)
mlp_x3_kernel(const FieldDev F, const Op op, uint32_t* __restrict__ mask_scratch, int n_stages, int alo_bytes,
              int stage_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base_ptr = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Smem S;
  S.alo = base_ptr;
  S.stages = base_ptr + alo_bytes;
  S.bars = reinterpret_cast<uint64_t*>(S.stages + (size_t)n_stages * stage_bytes);
  S.tmem_slot = reinterpret_cast<uint32_t*>(S.bars + GROUPS + 2 + 2 * n_stages);   // keeps params 16-B aligned
  S.red = reinterpret_cast<float*>(S.tmem_slot + 4);
  S.params = S.red + 2 * ROWS;

  const int warp = umma::uni((int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;   // warp index, provably warp-uniform
  const uint32_t bar0 = smem_u32(S.bars);
  auto BAR_A_READY = [&](int g) { return bar0 + 8u * g; };
  const uint32_t BAR_ACC = bar0 + 8u * GROUPS;
  auto BAR_FULL = [&](int s) { return bar0 + 8u * (GROUPS + 2 + s); };
  auto BAR_EMPTY = [&](int s) { return bar0 + 8u * (GROUPS + 2 + n_stages + s); };

  if (threadIdx.x == 0) {
    for (int g = 0; g < GROUPS; ++g) mbar_init(BAR_A_READY(g), 4);   // the 4 lane-quarter warps owning g
    mbar_init(BAR_ACC, 1);
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(BAR_FULL(s), 1);
      mbar_init(BAR_EMPTY(s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(S.tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *S.tmem_slot;
  const uint32_t alo_base = smem_u32(S.alo);
  const uint32_t st_base = smem_u32(S.stages);
  const int tiles = umma::n_tiles(F, op);

  if (warp == 0) {
    // ================================================= weight producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int j0, j1, base, nv;
        umma::tile_rows(F, op, t, j0, j1, base, nv);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_x3);
          const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
          const uint8_t* img = Op::kGrad ? P->img_grad : P->img_fwd;
          for (int s = 0; s < ns; ++s) {
            const Step st = umma::load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            const uint8_t* src = img + st.img_off;
            for (int kk = 0; kk < st.nchunk; ++kk) {
              mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
              mbar_expect_tx(BAR_FULL(stage), (uint32_t)st.chunk_bytes);
              bulk_g2s(st_base + (uint32_t)(stage * stage_bytes), src, (uint32_t)st.chunk_bytes, BAR_FULL(stage));
              src += st.chunk_bytes;
              if (++stage == n_stages) { stage = 0; phase ^= 1u; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer (whole warp, converged, on
    // warp-uniform values: umma::uni / umma::mbar_wait_u)
    {
      using umma::uni;
      using umma::mbar_wait_u;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t ar = 0u;                 // A_READY phase: every group completes one per step
      const uint32_t tmem_u = uni(tmem), bars_u = uni(bar0);
      const uint32_t alo0_lo = uni(umma::sdesc_lo(alo_base)), w0_lo = uni(umma::sdesc_lo(st_base));
      const uint32_t sstep = uni((uint32_t)stage_bytes >> 4);
      const int nst = uni(n_stages), tiles_u = uni(tiles);
      for (int t = blockIdx.x; t < tiles_u; t += gridDim.x) {
        int j0, j1, base, nv;
        umma::tile_rows(F, op, t, j0, j1, base, nv);
        j0 = uni(j0);
        j1 = uni(j1);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_x3);
          const int ns = uni(Op::kGrad ? P->n_grad : P->n_fwd);
          for (int s = 0; s < ns; ++s) {
            Step st = umma::load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            umma::uni_step(st);
            const uint32_t id = idesc_tf32(st.N);
            const uint32_t d_t = tmem_u + (uint32_t)((s & 1) * REGION);
            const uint32_t a_t = tmem_u + (uint32_t)(((s + 1) & 1) * REGION);
            const int ngr = (st.K + 31) >> 5;
            const uint32_t lo_off = (uint32_t)(st.N * 32) >> 4;   // W_lo block behind W_hi in a stage
            for (int kk = 0; kk < st.nchunk; ++kk) {
              const int g = kk >> 2;
              // A group g of this step: written by the previous epilogue (or the encoding)
              if ((kk & 3) == 0) mbar_wait_u(bars_u + 8u * (uint32_t)g, ar & 1u);
              mbar_wait_u(bars_u + 8u * (uint32_t)(GROUPS + 2 + stage), phase);
              tc_after_sync();
              const uint32_t bhi = w0_lo + (uint32_t)stage * sstep;
              const uint32_t alo = alo0_lo + (uint32_t)((g * ROWS * 128 + (kk & 3) * 32) >> 4);
              mma_x3_step_w(d_t, a_t + (uint32_t)(kk * 8), bhi, bhi + lo_off, alo, id, kk ? 1u : 0u,
                            bars_u + 8u * (uint32_t)(GROUPS + 2 + nst + stage));
              if (++stage == nst) { stage = 0; phase ^= 1u; }
            }
            // groups this step does not read: consume their release to keep phases in step
            for (int gg = ngr; gg < GROUPS; ++gg) mbar_wait_u(bars_u + 8u * (uint32_t)gg, ar & 1u);
            ++ar;
            umma::tc_commit_w(bars_u + 8u * (uint32_t)GROUPS);
          }
        }
      }
    }
  } else {
    // ================================================= row warps (encoding + epilogues)
    const int q = warp & 3;                    // TMEM lane quarter of this warp
    const int sub = (warp - EPI_WARP0) >> 2;   // column groups of this warp: g % 2 == sub
    const int r = q * 32 + lane;               // tile row == TMEM lane
    const int r7 = r & 7;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t alo_row = alo_base + (uint32_t)((r >> 3) * 1024 + r7 * 128);
    uint32_t* my_masks = mask_scratch + (size_t)blockIdx.x * MASK_WORDS_PER_CTA;
    uint32_t acc_ph = 0u;
    // this row of the next tile: list entry and path state (with its f64
    // direction -> angle trigonometry) fetched one tile ahead, issued once
    // the current tile's encoding is released
    int n_slot = 0;
    double n_pos[3] = {0.0, 0.0, 0.0}, n_u3 = 0.0, n_u4 = 0.0;
    auto fetch = [&](int tt) {
      if (tt < tiles) {
        int a0, a1, b0, c0;
        umma::tile_rows(F, op, tt, a0, a1, b0, c0);
        if (r < c0) {
          n_slot = op.slot(b0 + r);
          if constexpr (!Op::kRaw) op.load(n_slot, n_pos, n_u3, n_u4);
        }
      }
    };
    fetch(blockIdx.x);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int j0, j1, base, nv;
      umma::tile_rows(F, op, t, j0, j1, base, nv);
      const bool valid = r < nv;
      const int slot = valid ? n_slot : 0;
      double pos[3] = {n_pos[0], n_pos[1], n_pos[2]}, u3 = n_u3, u4 = n_u4;
      double best = 0.0;
      int bobj = 0;
      for (int j = j0; j < j1; ++j) {
        const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_x3);
        const NetDev& net = F.net[j];
        // this network's biases + head weights -> shared memory (every row warp
        // is past the previous program's last epilogue: see the head barrier)
        const int head_off = __ldg(&P->head_off);
        {
          const int nf = __ldg(&P->params_floats);
          const float4* src = reinterpret_cast<const float4*>(P->params);
          float4* dst = reinterpret_cast<float4*>(S.params);
          named_sync(1, N_EPI_WARPS * 32);
          for (int i = threadIdx.x - EPI_WARP0 * 32; i < (nf >> 2); i += N_EPI_WARPS * 32) dst[i] = __ldg(src + i);
          named_sync(1, N_EPI_WARPS * 32);
        }
        // ---- input encoding -> A_hi (TMEM region 1) + A_lo, groups g % 2 == sub
        const uint32_t enc_t = tmem + lane_addr + (uint32_t)REGION;
        const int k0 = P->k0;
        if constexpr (!Op::kRaw) {
          double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
          if (valid) row_u(F, j, pos, u3, u4, u);
          const bool pe = net.encoding == ENC_PE6;
          if (sub == 0) {
            encode_group<0>(pe, valid, u, enc_t, alo_row, r7);
            if (k0 > 64) encode_group<2>(pe, valid, u, enc_t + 64u, alo_row + 2u * ROWS * 128, r7);
          } else if (k0 > 32) {
            encode_group<1>(pe, valid, u, enc_t + 32u, alo_row + 1u * ROWS * 128, r7);
          }
        } else {
          for (int g = sub; g * 32 < k0; g += 2) {
            float x[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) x[e] = valid ? (float)op.raw(slot, 32 * g + e) : 0.f;
            put_group(x, enc_t + (uint32_t)(32 * g), alo_row + (uint32_t)(g * ROWS * 128), r7);
          }
        }
#pragma unroll
        for (int g = 0; g < GROUPS; ++g)
          if ((g & 1) == sub) release_group(BAR_A_READY(g), lane);
        if (j == j0) fetch(t + (int)gridDim.x);

        const int ns = Op::kGrad ? P->n_grad : P->n_fwd;
        float head_part = 0.f;
        for (int s = 0; s < ns; ++s) {
          const Step st = umma::load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
          const int epi = st.epi;
          const uint32_t d_t = tmem + lane_addr + (uint32_t)((s & 1) * REGION);
          mbar_wait(BAR_ACC, acc_ph & 1u);
          ++acc_ph;
          tc_after_sync();
          if (epi == E_BWD_OUT) {
            if (sub == 0) {
              // d pred / d inputs for this row: st.N (>= k0) fp32 columns
              float gin[96];
#pragma unroll
              for (int c = 0; c < 96; c += 16) {
                if (c < st.N) {
                  uint32_t rg[16];
                  DDF_TMEM_LD16(d_t + (uint32_t)c, rg);
                  tmem_wait_ld();
#pragma unroll
                  for (int e = 0; e < 16; ++e) gin[c + e] = __uint_as_float(rg[e]);
                }
              }
              if constexpr (Op::kGrad) {
                if (valid) {
                  if constexpr (Op::kRaw) {
                    op.store_grad_raw(slot, [&](int k) { return (double)gin[k]; });
                  } else {
                    double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                    row_u(F, j, pos, u3, u4, u);
                    double g5[5];
                    pe_chain(net, u, [&](int k) { return (double)gin[k]; }, g5);
                    op.store_grad(slot, g5);
                  }
                }
              }
            }
            tc_before_sync();
            continue;
          }
          const int ng = (st.N + 31) >> 5;
          const float* hw = S.params + head_off;
          for (int g = sub; g < GROUPS; g += 2) {
            if (g < ng) {
              const int c = 32 * g;
              const uint32_t tc = d_t + (uint32_t)c, al = alo_row + (uint32_t)(g * ROWS * 128);
              switch (epi) {
                case E_RELU_A: epi_group<E_RELU_A>(st, c, r, tc, al, my_masks, hw, head_part, S.params); break;
                case E_RELU_MASK_A: epi_group<E_RELU_MASK_A>(st, c, r, tc, al, my_masks, hw, head_part, S.params); break;
                case E_MASKG_A: epi_group<E_MASKG_A>(st, c, r, tc, al, my_masks, hw, head_part, S.params); break;
                case E_BWD_MASK_A: epi_group<E_BWD_MASK_A>(st, c, r, tc, al, my_masks, hw, head_part, S.params); break;
                default: epi_group<E_HEAD>(st, c, r, tc, al, my_masks, hw, head_part, S.params); break;
              }
            }
            if (epi != E_HEAD) release_group(BAR_A_READY(g), lane);
          }
          tc_before_sync();
          if (epi == E_HEAD) {
            S.red[sub * ROWS + r] = head_part;
            named_sync(1, N_EPI_WARPS * 32);
            if (sub == 0) {
              double p = (double)(S.red[r] + S.red[ROWS + r] + P->head_b);
              if (F.composite) p = dmul(net.scale, p);
              if (j == j0 || p < best) { best = p; bobj = j; }
            }
            named_sync(1, N_EPI_WARPS * 32);
          }
        }
      }
      if constexpr (!Op::kGrad) {
        if (sub == 0 && valid) op.store_fwd(slot, best, bobj);
      }
    }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ================================================================== two tiles in flight (<= 128 wide)
// Networks whose hidden layers are at most 128 wide (config 1, the UDF scan)
// leave half of TMEM and of the A_lo buffer unused in mlp_x3_kernel, and with
// one tile per CTA the tensor pipe idles through every epilogue (measured:
// ~23 K cycles per tile against 9.6 K of MMAs).  Here two 128-row tiles
// ("slots" X, Y) run the layers in lock-step, as in the bf16 ping-pong
// engine: the MMA warp issues layer s of X, then layer s of Y, while the row
// warps run X's epilogue.  Slot sl owns TMEM columns [256 sl, 256 sl + 256):
// D_s in its 128-column region s & 1, A_hi in the other; its own A_lo buffer,
// barriers, ReLU-mask scratch and staged params.  A slot's A is released
// once per step (all groups at once): by the time the issuer returns to the
// slot its epilogue is done, so the group-by-group release of the one-tile
// kernel buys nothing here.
constexpr int PP_REGION = 128;
constexpr int PP_GROUPS = PP_REGION / 32;

template <class Op>
__global__ void __launch_bounds__(NTHREADS, 1)
mlp_x3pp_kernel(const FieldDev F, const Op op, uint32_t* __restrict__ mask_scratch, int n_stages, int alo_bytes,
                int stage_bytes, int params_bytes) {
  using umma::uni;
  using umma::mbar_wait_u;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base_ptr = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* alo = base_ptr;                                        // [2 slots][alo_bytes]
  uint8_t* stages = base_ptr + 2 * (size_t)alo_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)n_stages * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 + 2 * n_stages);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);           // [2 slots][2 subs][128]
  float* sparams = red + 4 * ROWS;                                // [2 slots][params_bytes/4]
  const int pfl = params_bytes >> 2;

  const int warp = uni((int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(bars);
  auto BAR_A_READY = [&](int sl) { return bar0 + 8u * sl; };
  auto BAR_ACC = [&](int sl) { return bar0 + 8u * (2 + sl); };
  auto BAR_FULL = [&](int st_) { return bar0 + 8u * (4 + st_); };
  auto BAR_EMPTY = [&](int st_) { return bar0 + 8u * (4 + n_stages + st_); };

  if (threadIdx.x == 0) {
    for (int sl = 0; sl < 2; ++sl) {
      mbar_init(BAR_A_READY(sl), N_EPI_WARPS);
      mbar_init(BAR_ACC(sl), 1);
    }
    for (int st_ = 0; st_ < n_stages; ++st_) {
      mbar_init(BAR_FULL(st_), 1);
      mbar_init(BAR_EMPTY(st_), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t alo_base = smem_u32(alo);
  const uint32_t st_base = smem_u32(stages);
  const int pairs = umma::pp_pairs(F, op);

  if (warp == 0) {
    // ================================================= weight producer: each step once per slot
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        int j0, j1, base, nv;
        umma::pp_rows(F, op, pr, 0, j0, j1, base, nv);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_x3);
          const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
          const uint8_t* img = Op::kGrad ? P->img_grad : P->img_fwd;
          for (int s = 0; s < ns; ++s) {
            const Step st = umma::load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            for (int sl = 0; sl < 2; ++sl) {
              const uint8_t* src = img + st.img_off;
              for (int kk = 0; kk < st.nchunk; ++kk) {
                mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
                mbar_expect_tx(BAR_FULL(stage), (uint32_t)st.chunk_bytes);
                bulk_g2s(st_base + (uint32_t)(stage * stage_bytes), src, (uint32_t)st.chunk_bytes, BAR_FULL(stage));
                src += st.chunk_bytes;
                if (++stage == n_stages) { stage = 0; phase ^= 1u; }
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer (whole warp, converged, uniform)
    int stage = 0;
    uint32_t phase = 0;
    uint32_t ar = 0u;
    const uint32_t tmem_u = uni(tmem), bars_u = uni(bar0);
    const uint32_t alo0_lo = uni(umma::sdesc_lo(alo_base)), w0_lo = uni(umma::sdesc_lo(st_base));
    const uint32_t alo_step = uni((uint32_t)alo_bytes >> 4), sstep = uni((uint32_t)stage_bytes >> 4);
    const int nst = uni(n_stages), pairs_u = uni(pairs);
    for (int pr = blockIdx.x; pr < pairs_u; pr += gridDim.x) {
      int j0, j1, base, nv;
      umma::pp_rows(F, op, pr, 0, j0, j1, base, nv);
      j0 = uni(j0);
      j1 = uni(j1);
      for (int j = j0; j < j1; ++j) {
        const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_x3);
        const int ns = uni(__ldg(Op::kGrad ? &P->n_grad : &P->n_fwd));
        for (int s = 0; s < ns; ++s) {
          Step st = umma::load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
          umma::uni_step(st);
          const uint32_t id = idesc_tf32(st.N);
          const uint32_t lo_off = (uint32_t)(st.N * 32) >> 4;   // W_lo block behind W_hi in a stage
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            mbar_wait_u(bars_u + 8u * sl, ar & 1u);   // the slot's A (hi in TMEM, lo in shared memory)
            tc_after_sync();
            const uint32_t d_t = tmem_u + (uint32_t)(sl * 256 + (s & 1) * PP_REGION);
            const uint32_t a_t = tmem_u + (uint32_t)(sl * 256 + ((s + 1) & 1) * PP_REGION);
            const uint32_t alo_sl = alo0_lo + (uint32_t)sl * alo_step;
            for (int kk = 0; kk < st.nchunk; ++kk) {
              mbar_wait_u(bars_u + 8u * (uint32_t)(4 + stage), phase);
              tc_after_sync();
              const uint32_t bhi = w0_lo + (uint32_t)stage * sstep;
              const uint32_t al = alo_sl + (uint32_t)(((kk >> 2) * ROWS * 128 + (kk & 3) * 32) >> 4);
              mma_x3_step_w(d_t, a_t + (uint32_t)(kk * 8), bhi, bhi + lo_off, al, id, kk ? 1u : 0u,
                            bars_u + 8u * (uint32_t)(4 + nst + stage));
              if (++stage == nst) { stage = 0; phase ^= 1u; }
            }
            umma::tc_commit_w(bars_u + 8u * (uint32_t)(2 + sl));
          }
          ++ar;
        }
      }
    }
  } else {
    // ================================================= row warps (both slots in turn)
    const int q = warp & 3;
    const int sub = (warp - EPI_WARP0) >> 2;   // column groups of this warp: g % 2 == sub
    const int r = q * 32 + lane;
    const int r7 = r & 7;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t acc_ph[2] = {0u, 0u};
    // this row of the next pair of tiles, fetched one pair ahead
    int n_slot[2] = {0, 0};
    double n_pos[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}}, n_u3[2] = {0.0, 0.0}, n_u4[2] = {0.0, 0.0};
    auto fetch = [&](int pp) {
      if (pp < pairs) {
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          int a0, a1, b0, c0;
          umma::pp_rows(F, op, pp, sl, a0, a1, b0, c0);
          if (r < c0) {
            n_slot[sl] = op.slot(b0 + r);
            if constexpr (!Op::kRaw) op.load(n_slot[sl], n_pos[sl], n_u3[sl], n_u4[sl]);
          }
        }
      }
    };
    // a slot's A complete: TMEM stores done, shared stores visible to the async proxy
    auto release = [&](int sl) {
      tmem_wait_st();
      tc_before_sync();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR_A_READY(sl));
    };
    fetch(blockIdx.x);
    for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
      int j0 = 0, j1 = 0;
      int slot_id[2] = {0, 0};
      bool valid[2] = {false, false};
      double pos[2][3], u3[2], u4[2], best[2] = {0.0, 0.0};
      int bobj[2] = {0, 0};
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        int base, nv;
        umma::pp_rows(F, op, pr, sl, j0, j1, base, nv);
        valid[sl] = r < nv;
        slot_id[sl] = valid[sl] ? n_slot[sl] : 0;
        pos[sl][0] = n_pos[sl][0]; pos[sl][1] = n_pos[sl][1]; pos[sl][2] = n_pos[sl][2];
        u3[sl] = n_u3[sl];
        u4[sl] = n_u4[sl];
      }
      for (int j = j0; j < j1; ++j) {
        const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_x3);
        const NetDev& net = F.net[j];
        const int head_off = __ldg(&P->head_off);
        const int k0 = P->k0;
        const bool pe = net.encoding == ENC_PE6;
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          {   // params of this network for the slot (the slot's previous network is done)
            const int nf = __ldg(&P->params_floats);
            const float4* src = reinterpret_cast<const float4*>(P->params);
            float4* dst = reinterpret_cast<float4*>(sparams + sl * pfl);
            named_sync(1, N_EPI_WARPS * 32);
            for (int i = threadIdx.x - EPI_WARP0 * 32; i < (nf >> 2); i += N_EPI_WARPS * 32) dst[i] = __ldg(src + i);
            named_sync(1, N_EPI_WARPS * 32);
          }
          // ---- input encoding -> A_hi (the slot's region 1) + A_lo, groups g % 2 == sub
          const uint32_t enc_t = tmem + lane_addr + (uint32_t)(sl * 256 + PP_REGION);
          const uint32_t alo_row = alo_base + (uint32_t)(sl * alo_bytes) + (uint32_t)((r >> 3) * 1024 + r7 * 128);
          if constexpr (!Op::kRaw) {
            double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (valid[sl]) row_u(F, j, pos[sl], u3[sl], u4[sl], u);
            if (sub == 0) {
              encode_group<0>(pe, valid[sl], u, enc_t, alo_row, r7);
              if (k0 > 64) encode_group<2>(pe, valid[sl], u, enc_t + 64u, alo_row + 2u * ROWS * 128, r7);
            } else if (k0 > 32) {
              encode_group<1>(pe, valid[sl], u, enc_t + 32u, alo_row + 1u * ROWS * 128, r7);
            }
          } else {
            for (int g = sub; g * 32 < k0; g += 2) {
              float x[32];
#pragma unroll
              for (int e = 0; e < 32; ++e) x[e] = valid[sl] ? (float)op.raw(slot_id[sl], 32 * g + e) : 0.f;
              put_group(x, enc_t + (uint32_t)(32 * g), alo_row + (uint32_t)(g * ROWS * 128), r7);
            }
          }
          release(sl);
        }
        if (j == j0) fetch(pr + (int)gridDim.x);

        const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
        float head_part[2] = {0.f, 0.f};
        for (int s = 0; s < ns; ++s) {
          const Step st = umma::load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
          const int epi = st.epi;
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            mbar_wait(BAR_ACC(sl), acc_ph[sl] & 1u);
            ++acc_ph[sl];
            tc_after_sync();
            const uint32_t d_t = tmem + lane_addr + (uint32_t)(sl * 256 + (s & 1) * PP_REGION);
            const uint32_t alo_row = alo_base + (uint32_t)(sl * alo_bytes) + (uint32_t)((r >> 3) * 1024 + r7 * 128);
            uint32_t* my_masks = mask_scratch + ((size_t)blockIdx.x * 2 + sl) * MASK_WORDS_PER_CTA;
            const float* sp = sparams + sl * pfl;
            if (epi == E_BWD_OUT) {
              if (sub == 0) {
                float gin[96];
#pragma unroll
                for (int c = 0; c < 96; c += 16) {
                  if (c < st.N) {
                    uint32_t rg[16];
                    DDF_TMEM_LD16(d_t + (uint32_t)c, rg);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) gin[c + e] = __uint_as_float(rg[e]);
                  }
                }
                if constexpr (Op::kGrad) {
                  if (valid[sl]) {
                    if constexpr (Op::kRaw) {
                      op.store_grad_raw(slot_id[sl], [&](int k) { return (double)gin[k]; });
                    } else {
                      double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                      row_u(F, j, pos[sl], u3[sl], u4[sl], u);
                      double g5[5];
                      pe_chain(net, u, [&](int k) { return (double)gin[k]; }, g5);
                      op.store_grad(slot_id[sl], g5);
                    }
                  }
                }
              }
              tc_before_sync();
              continue;
            }
            const int ng = (st.N + 31) >> 5;
            const float* hw = sp + head_off;
            for (int g = sub; g < PP_GROUPS; g += 2) {
              if (g < ng) {
                const int c = 32 * g;
                const uint32_t tc = d_t + (uint32_t)c, al = alo_row + (uint32_t)(g * ROWS * 128);
                switch (epi) {
                  case E_RELU_A: epi_group<E_RELU_A>(st, c, r, tc, al, my_masks, hw, head_part[sl], sp); break;
                  case E_RELU_MASK_A: epi_group<E_RELU_MASK_A>(st, c, r, tc, al, my_masks, hw, head_part[sl], sp); break;
                  case E_MASKG_A: epi_group<E_MASKG_A>(st, c, r, tc, al, my_masks, hw, head_part[sl], sp); break;
                  case E_BWD_MASK_A: epi_group<E_BWD_MASK_A>(st, c, r, tc, al, my_masks, hw, head_part[sl], sp); break;
                  default: epi_group<E_HEAD>(st, c, r, tc, al, my_masks, hw, head_part[sl], sp); break;
                }
              }
            }
            if (epi != E_HEAD) {
              release(sl);
            } else {
              tc_before_sync();
              float* rd = red + sl * 2 * ROWS;
              rd[sub * ROWS + r] = head_part[sl];
              named_sync(1, N_EPI_WARPS * 32);
              if (sub == 0) {
                double pv = (double)(rd[r] + rd[ROWS + r] + P->head_b);
                if (F.composite) pv = dmul(net.scale, pv);
                if (j == j0 || pv < best[sl]) { best[sl] = pv; bobj[sl] = j; }
              }
              named_sync(1, N_EPI_WARPS * 32);
            }
          }
        }
      }
      if constexpr (!Op::kGrad) {
#pragma unroll
        for (int sl = 0; sl < 2; ++sl)
          if (sub == 0 && valid[sl]) op.store_fwd(slot_id[sl], best[sl], bobj[sl]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------ host side
inline int pad_to(int x, int m) { return (x + m - 1) / m * m; }

// nearest tf32 (ties away, as cvt.rna) of an fp32 value
inline float host_tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u += 0x1000u;
  u &= 0xFFFFE000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

// Append the K-steps of one step: B[n][k] = src(n, k) (f64), n < N, k < K.
// Per K-step of 8: W_hi block then W_lo block, each N rows x 32 B with the
// 32-byte swizzle (16-byte half h of row n at h ^ ((n >> 2) & 1)).
template <class Src>
inline void append_ksteps(std::vector<float>& img, Step& st, Src src) {
  st.img_off = (long long)img.size() * 4;
  const int N = st.N;
  for (int kk = 0; kk < st.nchunk; ++kk) {
    const size_t base = img.size();
    img.resize(base + (size_t)2 * N * 8, 0.f);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < 8; ++k) {
        const int gk = kk * 8 + k;
        const double w = gk < st.K ? src(n, gk) : 0.0;
        const float hi = host_tf32_rna((float)w);
        const float lo = (float)(w - (double)hi);
        const size_t off = (size_t)(n >> 3) * 64 + (size_t)(n & 7) * 8 + (size_t)((((k >> 2) ^ ((n >> 2) & 1)) << 2) + (k & 3));
        img[base + off] = hi;
        img[base + (size_t)N * 8 + off] = lo;
      }
  }
}

inline Step make_step(int K, int N, int epi) {
  Step s{};
  s.K = K; s.N = N; s.nh = 1; s.epi = epi;
  s.rows = N;
  s.nchunk = K / 8;
  s.chunk_bytes = 2 * N * 32;
  s.mask_layer = -1;
  s.bias = nullptr;
  return s;
}

// Can this network run on the 3xTF32 engine?  (hidden widths <= 256, input <= 96)
inline bool supports(const int32_t* widths, int32_t n_widths) {
  const int L = n_widths - 1;
  if (L < 2 || widths[0] > 96) return false;
  for (int l = 1; l < L; ++l)
    if (pad_to(widths[l], 32) > MAXW) return false;
  return true;
}

// Build forward and gradient programs + 3xTF32 images for one network.
// weights: concat of W_l (out, in) row-major float64; biases: concat of b_l.
inline int build_image(const int32_t* widths, int32_t n_widths, const double* weights, const double* biases,
                       NetImage* out, std::string* err) {
  const int L = n_widths - 1;
  out->in_width = widths[0];
  if (!supports(widths, n_widths)) { *err = "3xTF32 engine: hidden widths up to 256, input up to 96"; return 1; }
  std::vector<int> wp(n_widths);
  wp[0] = pad_to(widths[0], 8);
  for (int l = 1; l < L; ++l) wp[l] = pad_to(widths[l], 32);
  wp[L] = 1;
  // f64 effective weights, padded (host), row-major (out, in)
  std::vector<std::vector<double>> W(L);
  std::vector<std::vector<float>> B(L);
  size_t wo = 0, bo = 0;
  for (int l = 0; l < L; ++l) {
    const int in = widths[l], o = widths[l + 1];
    W[l].assign((size_t)wp[l + 1] * wp[l], 0.0);
    B[l].assign(wp[l + 1], 0.f);
    for (int a = 0; a < o; ++a) {
      for (int k = 0; k < in; ++k) W[l][(size_t)a * wp[l] + k] = weights[wo + (size_t)a * in + k];
      B[l][a] = (float)biases[bo + a];
    }
    wo += (size_t)o * in;
    bo += o;
  }
  Prog& P = out->host;
  std::memset(&P, 0, sizeof(P));
  P.k0 = wp[0];
  P.in_width = widths[0];
  P.encoding = widths[0] == 65 ? ENC_PE6 : ENC_RAW5;
  P.head_b = B[L - 1][0];
  int maxh = 0;
  for (int l = 1; l < L; ++l) maxh = std::max(maxh, wp[l]);
  P.max_hidden = maxh;
  std::vector<float> params;   // hidden-layer biases then head weights (fp32, multiples of 4 floats)
  std::vector<size_t> bias_off(L);
  for (int l = 0; l < L - 1; ++l) { bias_off[l] = params.size(); params.insert(params.end(), B[l].begin(), B[l].end()); }
  const size_t head_off = params.size();
  for (int k = 0; k < wp[L - 1]; ++k) params.push_back((float)W[L - 1][k]);
  while (params.size() % 4) params.push_back(0.f);

  std::vector<float> img;
  P.n_fwd = L - 1;
  for (int l = 0; l < L - 1; ++l) {
    Step s = make_step(wp[l], wp[l + 1], l == L - 2 ? E_HEAD : E_RELU_A);
    const std::vector<double>& w = W[l];
    const int K = wp[l];
    append_ksteps(img, s, [&](int n, int k) { return w[(size_t)n * K + k]; });
    s.bias = reinterpret_cast<const float*>(bias_off[l]);
    P.fwd[l] = s;
  }
  const size_t fwd_floats = img.size();
  std::vector<float> gimg;
  int gs = 0;
  for (int l = 0; l < L - 1; ++l) {
    Step s = make_step(wp[l], wp[l + 1], l == L - 2 ? E_MASKG_A : E_RELU_MASK_A);
    s.mask_layer = l;
    const std::vector<double>& w = W[l];
    const int K = wp[l];
    append_ksteps(gimg, s, [&](int n, int k) { return w[(size_t)n * K + k]; });
    s.bias = reinterpret_cast<const float*>(bias_off[l]);
    P.grad[gs++] = s;
  }
  // backward: layer l maps d z_l (width wp[l+1]) to d h_l (width wp[l]) with B[n][k] = W_l[k][n];
  // the last step's N (input gradient) is padded to 16 (MMA N granularity at M = 128)
  for (int l = L - 2; l >= 0; --l) {
    const bool last = l == 0;
    Step s = make_step(wp[l + 1], last ? pad_to(widths[0], 16) : wp[l], last ? E_BWD_OUT : E_BWD_MASK_A);
    s.mask_layer = l - 1;
    const std::vector<double>& w = W[l];
    const int Kin = wp[l];
    append_ksteps(gimg, s, [&](int n, int k) { return n < Kin ? w[(size_t)k * Kin + n] : 0.0; });
    P.grad[gs++] = s;
  }
  P.n_grad = gs;
  if (gs > 2 * DDF_MAX_LAYERS) { *err = "too many layers"; return 1; }
  P.kmax = 0;
  P.max_chunk_bytes = 0;
  for (int i = 0; i < P.n_fwd; ++i) { P.kmax = std::max(P.kmax, std::max(P.fwd[i].K, P.fwd[i].N)); P.max_chunk_bytes = std::max(P.max_chunk_bytes, P.fwd[i].chunk_bytes); }
  for (int i = 0; i < P.n_grad; ++i) { P.kmax = std::max(P.kmax, std::max(P.grad[i].K, P.grad[i].N)); P.max_chunk_bytes = std::max(P.max_chunk_bytes, P.grad[i].chunk_bytes); }
  // upload
  const size_t total = (fwd_floats + gimg.size()) * 4;
  if (cudaMalloc(&out->img, total) != cudaSuccess) { *err = "cudaMalloc (weight image) failed"; return 4; }
  cudaMemcpy(out->img, img.data(), fwd_floats * 4, cudaMemcpyHostToDevice);
  cudaMemcpy((uint8_t*)out->img + fwd_floats * 4, gimg.data(), gimg.size() * 4, cudaMemcpyHostToDevice);
  if (cudaMalloc(&out->params, params.size() * 4) != cudaSuccess) { *err = "cudaMalloc (params) failed"; return 4; }
  cudaMemcpy(out->params, params.data(), params.size() * 4, cudaMemcpyHostToDevice);
  const float* pdev = reinterpret_cast<const float*>(out->params);
  for (int i = 0; i < P.n_grad; ++i) P.grad[i].bias = nullptr;
  for (int l = 0; l < L - 1; ++l) {
    P.fwd[l].bias = reinterpret_cast<const float*>(bias_off[l]);
    P.grad[l].bias = reinterpret_cast<const float*>(bias_off[l]);
  }
  P.head_w = pdev + head_off;
  P.params = pdev;
  P.head_off = (int)head_off;
  P.params_floats = (int)params.size();
  P.img_fwd = reinterpret_cast<const uint8_t*>(out->img);
  P.img_grad = reinterpret_cast<const uint8_t*>(out->img) + fwd_floats * 4;
  if (cudaMalloc(&out->dev, sizeof(Prog)) != cudaSuccess) { *err = "cudaMalloc (program) failed"; return 4; }
  if (cudaMemcpy(out->dev, &P, sizeof(Prog), cudaMemcpyHostToDevice) != cudaSuccess) { *err = "upload failed"; return 4; }
  return 0;
}

template <class Op>
int launch(const FieldDev& F, const std::vector<NetImage>& images, const Op& op, int max_rows, int sm_count,
           uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  int kmax = 0, chunk = 0, params_bytes = 0;
  for (int j = 0; j < F.n_obj; ++j) {
    kmax = std::max(kmax, images[j].host.kmax);
    chunk = std::max(chunk, images[j].host.max_chunk_bytes);
    params_bytes = std::max(params_bytes, images[j].host.params_floats * 4);
  }
  int maxh = 0;
  for (int j = 0; j < F.n_obj; ++j) maxh = std::max(maxh, images[j].host.max_hidden);
  if (maxh <= PP_REGION && kmax <= PP_REGION) {
    // two tiles per CTA in lock-step (mlp_x3pp_kernel)
    const int alo_bytes = ROWS * pad_to(kmax, 32) * 4;
    const int extra = 1024 /*align*/ + 8 * (4 + 2 * 12) + 16 + 4 * ROWS * 4 + 2 * params_bytes;
    const int n_stages = std::min(12, (umma::SMEM_LIMIT - 2 * alo_bytes - extra) / chunk);
    if (n_stages < 2) { *err = "3xTF32 two-tile engine: not enough shared memory for the weight pipeline"; return 1; }
    const size_t smem = 2 * (size_t)alo_bytes + (size_t)n_stages * chunk + extra;
    auto kern = mlp_x3pp_kernel<Op>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
    const int pairs_max = ((max_rows + ROWS - 1) / ROWS + 1) / 2 + (Op::kGrad ? F.n_obj : 0);
    const int grid = std::max(1, std::min(pairs_max, sm_count));
    kern<<<grid, NTHREADS, smem, st>>>(F, op, mask_scratch, n_stages, alo_bytes, chunk, params_bytes);
    e = cudaGetLastError();
    if (e != cudaSuccess) { *err = std::string("mlp_x3pp_kernel launch: ") + cudaGetErrorString(e); return 4; }
    return 0;
  }
  const int alo_bytes = ROWS * pad_to(kmax, 32) * 4;
  const int extra = 1024 /*align*/ + 8 * (GROUPS + 2 + 2 * 12) + 16 + 2 * ROWS * 4 + params_bytes;
  int n_stages = std::min(12, (umma::SMEM_LIMIT - alo_bytes - extra) / chunk);
  if (n_stages < 2) { *err = "3xTF32 engine: not enough shared memory for the weight pipeline"; return 1; }
  const size_t smem = (size_t)alo_bytes + (size_t)n_stages * chunk + extra;
  auto kern = mlp_x3_kernel<Op>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
  const int tiles_max = (max_rows + ROWS - 1) / ROWS + (Op::kGrad ? F.n_obj : 0);
  const int grid = std::max(1, std::min(tiles_max, sm_count));
  kern<<<grid, NTHREADS, smem, st>>>(F, op, mask_scratch, n_stages, alo_bytes, chunk);
  e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("mlp_x3_kernel launch: ") + cudaGetErrorString(e); return 4; }
  return 0;
}

}  // namespace x3
}  // namespace ddf
