// bf16 DDF-MLP engine on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// One persistent CTA per SM, 128-row tiles (the UMMA M = 128 datapath), ten
// warps:
//   warp 0      weight producer: streams UMMA-ready weight chunks (pre-swizzled
//               on the host) global->shared with cp.async.bulk + mbarrier tx
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (kind::f16,
//               bf16 x bf16 -> fp32 in TMEM), commits to mbarriers
//   warps 2-9   row warps: input encoding in registers -> A tile in shared
//               memory; per layer the TMEM->register epilogue (bias + ReLU /
//               ReLU masks / gradient masks) writes the next layer's bf16 A
//               tile back into shared memory; the last epilogue hands the
//               distance (or input gradient) to the row op.
//
// Activations never leave the SM.  Each dense layer is split into two
// N-halves whose accumulators sit side by side in TMEM (<= 512 fp32 columns);
// the epilogue of half 0 overwrites A columns [0, N/2) as soon as the MMAs of
// half 1 have read them (a_free barriers), so one A buffer (128 x 512 bf16)
// suffices and the tensor pipe stays busy while the epilogue runs.
//
// Gradient programs (neural.py:229-249) run the hidden layers forward storing
// ReLU bit masks (one u32 per row per 32 columns, per-CTA global scratch),
// seed d/dh of the last hidden layer with w_head * mask, then run the
// backward chain d_h <- (d_h * mask) @ W on the tensor cores with W^T images.
#pragma once
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "ddf_common.cuh"
#include "field_kernels.cuh"

namespace ddf {
namespace umma {

constexpr int ROWS = 128;
// Pipeline wait-cycle counters (diagnostics): compiled in with -DDDF_PIPE_STATS=1
#ifndef DDF_PIPE_STATS
#define DDF_PIPE_STATS 0
#endif
constexpr bool kStats = DDF_PIPE_STATS != 0;
// DDF_DEBUG_UMMA bits that skip work (timing experiments, wrong results):
// honoured only in the diagnostics build (-DDDF_PIPE_STATS=1, scratch/).
// -DDDF_ALLOW_DBG=1 honours them without the counters (timeline builds).
#ifndef DDF_ALLOW_DBG
#define DDF_ALLOW_DBG 0
#endif
constexpr int kUnsafeDbg = 1 | 8 | 128 | 1024 | 2048;
inline int debug_bits() {
  static const int raw = getenv("DDF_DEBUG_UMMA") ? atoi(getenv("DDF_DEBUG_UMMA")) : 0;
  return (kStats || DDF_ALLOW_DBG) ? raw : (raw & ~kUnsafeDbg);
}
static __device__ unsigned long long g_dbg[16];   // per translation unit (engines.h sums them)
// Event timeline of CTA 0 (diagnostics build -DDDF_TRACE=1): entries
// (clock64 << 16) | tag, tag = event | step << 5 | half << 11 | role << 12,
// recorded for the tiles CTA 0 runs as its TRACE_TILE0-th and next ones.
#ifndef DDF_TRACE
#define DDF_TRACE 0
#endif
constexpr bool kTrace = DDF_TRACE != 0;
// Each recording thread owns a TRACE_PER_ROLE slice (plain stores, no
// atomics, so the timeline is not perturbed by round trips); the reader
// compacts the slices.
constexpr int TRACE_CAP = 16384, TRACE_PER_ROLE = 4096, TRACE_TILE0 = 3, TRACE_TILES = 2;
static __device__ unsigned long long g_trace[TRACE_CAP];
struct TraceCursor {
  int role, n;
  __device__ void ev(bool on, int e, int step, int half) {
    if (kTrace && on && n < TRACE_PER_ROLE)
      g_trace[role * TRACE_PER_ROLE + n++] =
          ((unsigned long long)clock64() << 16) | (unsigned)(e | (step << 5) | (half << 11) | (role << 12));
  }
};
#define DDF_DBG_T0() long long _t0 = kStats ? clock64() : 0
#define DDF_DBG_ADD(i) do { if (kStats) dbg_acc[i] += (unsigned long long)(clock64() - _t0); } while (0)
#define DDF_DBG_FLUSH() do { if (kStats) for (int _i = 0; _i < 16; ++_i) if (dbg_acc[_i]) atomicAdd(&g_dbg[_i], dbg_acc[_i]); } while (0)
constexpr int NTHREADS = 320;
constexpr int EPI_WARP0 = 2;
constexpr int N_EPI_WARPS = 8;
constexpr int MASK_WORDS_PER_CTA = DDF_MAX_LAYERS * 16 * ROWS;   // u32: [layer][col/32][row]

// E_MASKG_HEAD_A exists only inside fused trace+gradient kernels (Op::kFused):
// the gradient program's E_MASKG_A step that also forms the identity head.
enum Epi : int { E_RELU_A = 0, E_HEAD = 1, E_RELU_MASK_A = 2, E_MASKG_A = 3, E_BWD_MASK_A = 4, E_BWD_OUT = 5,
                 E_MASKG_HEAD_A = 6 };
__host__ __device__ inline bool writes_a(int e) {
  return e == E_RELU_A || e == E_RELU_MASK_A || e == E_MASKG_A || e == E_BWD_MASK_A || e == E_MASKG_HEAD_A;
}

struct __align__(16) Step {
  int K, N, nh, epi;
  int nchunk;          // 64-wide K chunks per half
  int rows;            // N / nh (MMA N)
  int chunk_bytes;     // rows * 128
  int mask_layer;      // E_RELU_MASK_A: layer stored; E_BWD_MASK_A: layer applied
  long long img_off;   // byte offset of the step's first chunk in the image
  const float* bias;   // holds the float offset of the bias in Prog::params (no bias: unused)
};
static_assert(sizeof(Step) == 48, "Step is loaded as three 16-byte vectors");

// One step descriptor -> registers with three independent 16-byte loads (the
// roles would otherwise re-read fields after every barrier asm, and with
// 227 KB of shared memory carved out those loads miss L1).
__device__ __forceinline__ Step load_step(const Step* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  Step s;
  s.K = a.x; s.N = a.y; s.nh = a.z; s.epi = a.w;
  s.nchunk = b.x; s.rows = b.y; s.chunk_bytes = b.z; s.mask_layer = b.w;
  s.img_off = (long long)(((unsigned long long)(unsigned)c.y << 32) | (unsigned)c.x);
  s.bias = reinterpret_cast<const float*>(((unsigned long long)(unsigned)c.w << 32) | (unsigned)c.z);
  return s;
}

// Warp-uniform copy of a value every lane of a converged warp already agrees
// on.  ptxas keeps the result of redux.sync in a uniform register and then
// computes everything derived from it (descriptor advances, loop counters,
// barrier addresses) on the uniform datapath, so a tcgen05.mma whose operands
// all come from such values is issued as one uniform instruction: no ELECT /
// R2UR.BROADCAST waterfall per operand (~45 SASS instructions per four-MMA
// block otherwise, which paced the N = 128 engines).  Used by the MMA
// issuer warps on values loaded from memory (step descriptors, the TMEM
// base address), which the compiler must otherwise assume differ per lane.
__device__ __forceinline__ uint32_t uni(uint32_t x) { return __reduce_or_sync(0xffffffffu, x); }
__device__ __forceinline__ int uni(int x) { return (int)__reduce_or_sync(0xffffffffu, (uint32_t)x); }
// the fields of a step the MMA issuer uses, warp-uniform
__device__ __forceinline__ void uni_step(Step& st) {
  st.K = uni(st.K); st.N = uni(st.N); st.nh = uni(st.nh); st.epi = uni(st.epi);
  st.nchunk = uni(st.nchunk); st.rows = uni(st.rows);
}

// Bias folded into the accumulator (ping-pong and quad programs, hidden widths
// <= 256).  The epilogue's shared-memory traffic competes with the MMAs'
// operand fetch (profiles/r2_exp_epilogue_cost.txt), and a third of it was
// the broadcast bias loads.  Each forward-type step of these programs carries
// one more weight chunk whose K columns 0..2 hold the bias split into three
// bf16 pieces (hi + mid + lo = the fp32 bias to ~2^-24), and the issuer adds
// one K = 16 MMA of it against a constant A block whose columns 0..2 are 1:
// D += 1 * b_hi + 1 * b_mid + 1 * b_lo.  The epilogue then reads z, not z - b.
__host__ __device__ inline bool step_has_bias(int epi) {
  return epi == E_RELU_A || epi == E_HEAD || epi == E_RELU_MASK_A || epi == E_MASKG_A;
}
struct Prog {
  int n_fwd, n_grad;
  int k0;              // padded input width (multiple of 16)
  int in_width;        // unpadded input width
  int encoding;
  int kmax;            // widest A tile (columns)
  int max_chunk_bytes;
  int pp;              // 1: two-tile ping-pong program (hidden widths <= 256, one N-half per step)
  int max_hidden;      // widest padded hidden layer (<= 128: four-slot quad kernel)
  int fold;            // 1: forward-type steps carry a bias chunk (quad programs: after the K chunks; wide ones: per N-half, ahead)
  int chunk_k;         // K columns per weight chunk: 64, or 32 for 256-wide ping-pong programs
  float head_b;
  const float* head_w; // fp32, padded last hidden width
  const float* params; // fp32 block: hidden-layer biases then head weights (staged in shared memory)
  int params_floats;   // multiple of 4
  int head_off;        // float offset of the head weights in the block
  const uint8_t* img_fwd;
  const uint8_t* img_grad;
  Step fwd[DDF_MAX_LAYERS];
  Step grad[2 * DDF_MAX_LAYERS];
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// The same wait for a converged warp, leaving on a warp vote: the loop's exit
// is warp-uniform by construction, so the compiler keeps the code after it
// on the uniform datapath (see uni below); a per-lane exit makes ptxas treat
// everything downstream as potentially divergent.
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "vote.sync.all.pred q, p, 0xffffffff;\n\t"
      "@!q bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
#ifdef DDF_EXP_NOFENCE
// timing experiment only (racy): what does the generic -> async proxy fence cost the row warps?
__device__ __forceinline__ void fence_async_smem() {}
#else
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
#endif

// K-major, 128-byte swizzled canonical layout: 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: bf16 A/B, fp32 D, K-major A and B, M = 128
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(ROWS >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

// One 64-wide K chunk (four K = 16 MMAs) in a single asm block, optionally
// followed by a commit.  The issuing thread is lane 0 of a divergent warp, so
// every asm block with tcgen05 operands costs an ELECT / R2UR.BROADCAST
// waterfall; one block per chunk instead of one per MMA (plus per-MMA
// descriptor rebuilds) cut the issuer's instruction stream ~4x -- it, not
// the tensor pipe, paced the 512-wide engine (ncu source page: ~90 issue
// cycles per 128-cycle MMA).  Descriptors advance by 32 B (2 in the >> 4
// address field) per K step.
__device__ __forceinline__ void mma_k64(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %3, %3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_k64_commit(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc,
                                               uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %3, %3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n\t"
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(id), "r"(acc), "r"(bar)
      : "memory");
}

// Warp-wide variants: all 32 lanes of the issuing warp execute them in
// converged code (so the compiler keeps descriptors in uniform registers
// without an ELECT / R2UR.BROADCAST waterfall) and one lane, chosen by
// elect.sync inside the asm, issues.
// Descriptors travel as their low 32 bits (start address >> 4, LBO): the
// high word (SBO = 1024 B, version, 128-byte swizzle) is the same for every
// operand here, so the K-step advances are 32-bit adds.
constexpr uint32_t SDESC_HI = (uint32_t)((1024 >> 4) | (1u << 14) | (2u << 29));
__device__ __forceinline__ uint32_t sdesc_lo(uint32_t saddr) { return ((saddr & 0x3FFFFu) >> 4) | (1u << 16); }
// The constant A block: 128 rows x 32 B, 32-byte swizzle (16-byte half h of
// row r at h ^ ((r >> 2) & 1)), columns 0..2 = 1.0 bf16, the rest 0.
constexpr int ONES_BYTES = ROWS * 32;
constexpr uint32_t SDESC32B_HI = (uint32_t)((256 >> 4) | (1u << 14) | (6u << 29));   // SBO 256 B, version, SWIZZLE_32B
__device__ __forceinline__ void write_ones_block(uint8_t* ones, int tid, int nthreads) {
  for (int r = tid; r < ROWS; r += nthreads) {
    uint4* row = reinterpret_cast<uint4*>(ones + r * 32);
    const int h0 = (r >> 2) & 1;
    row[h0] = make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u);   // bf16 1, 1, 1, 0, 0, 0, 0, 0
    row[h0 ^ 1] = make_uint4(0u, 0u, 0u, 0u);
  }
}
// the fold's MMA: A = the ones block, B = the bias chunk (both one K = 16 step, 32-byte swizzle)
__device__ __forceinline__ void mma_bias_w(uint32_t tmem_d, uint32_t ones_lo, uint32_t db_lo, uint32_t id,
                                           uint32_t acc = 1u) {
  asm volatile(
      "{\n\t.reg .pred q, e;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 q, %4, 0;\n\t"
      "mov.b64 a, {%1, %5};\n\tmov.b64 b, {%2, %5};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t}" ::"r"(tmem_d),
      "r"(ones_lo), "r"(db_lo), "r"(id), "r"(acc), "n"(SDESC32B_HI)
      : "memory");
}

__device__ __forceinline__ void mma_k64_commit_w(uint32_t tmem_d, uint32_t da, uint32_t db, uint32_t id,
                                                 uint32_t acc, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
      ".reg .b64 a0, a1, a2, a3, b0, b1, b2, b3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %3, %3;\n\t"
      "add.u32 x1, %1, 2;\n\tadd.u32 x2, %1, 4;\n\tadd.u32 x3, %1, 6;\n\t"
      "add.u32 y1, %2, 2;\n\tadd.u32 y2, %2, 4;\n\tadd.u32 y3, %2, 6;\n\t"
      "mov.b64 a0, {%1, %6};\n\tmov.b64 a1, {x1, %6};\n\tmov.b64 a2, {x2, %6};\n\tmov.b64 a3, {x3, %6};\n\t"
      "mov.b64 b0, {%2, %6};\n\tmov.b64 b1, {y1, %6};\n\tmov.b64 b2, {y2, %6};\n\tmov.b64 b3, {y3, %6};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(tmem_d),
      "r"(da), "r"(db), "r"(id), "r"(acc), "r"(bar), "n"(SDESC_HI)
      : "memory");
}
__device__ __forceinline__ void mma_k64_w(uint32_t tmem_d, uint32_t da, uint32_t db, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
      ".reg .b64 a0, a1, a2, a3, b0, b1, b2, b3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %3, %3;\n\t"
      "add.u32 x1, %1, 2;\n\tadd.u32 x2, %1, 4;\n\tadd.u32 x3, %1, 6;\n\t"
      "add.u32 y1, %2, 2;\n\tadd.u32 y2, %2, 4;\n\tadd.u32 y3, %2, 6;\n\t"
      "mov.b64 a0, {%1, %5};\n\tmov.b64 a1, {x1, %5};\n\tmov.b64 a2, {x2, %5};\n\tmov.b64 a3, {x3, %5};\n\t"
      "mov.b64 b0, {%2, %5};\n\tmov.b64 b1, {y1, %5};\n\tmov.b64 b2, {y2, %5};\n\tmov.b64 b3, {y3, %5};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n\t}" ::"r"(tmem_d),
      "r"(da), "r"(db), "r"(id), "r"(acc), "n"(SDESC_HI)
      : "memory");
}
// One 32-wide K chunk of a ping-pong program (two K = 16 MMAs) and the commit
// that frees its stage: A in the 128-byte swizzle (the A tile), B in the
// 64-byte swizzle (SBO 512 B).
constexpr uint32_t SDESC64B_HI = (uint32_t)((512 >> 4) | (1u << 14) | (4u << 29));
__device__ __forceinline__ void mma_k32_commit_w(uint32_t tmem_d, uint32_t da, uint32_t db, uint32_t id,
                                                 uint32_t acc, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 x1, y1;\n\t"
      ".reg .b64 a0, a1, b0, b1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %3, %3;\n\t"
      "add.u32 x1, %1, 2;\n\tadd.u32 y1, %2, 2;\n\t"
      "mov.b64 a0, {%1, %6};\n\tmov.b64 a1, {x1, %6};\n\t"
      "mov.b64 b0, {%2, %7};\n\tmov.b64 b1, {y1, %7};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(tmem_d),
      "r"(da), "r"(db), "r"(id), "r"(acc), "r"(bar), "n"(SDESC_HI), "n"(SDESC64B_HI)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tc_commit_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

#define DDF_TMEM_LD32(taddr, r)                                                                                   \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
      : "r"(taddr))
#define DDF_TMEM_LD16(taddr, r)                                                                                   \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"    \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])     \
      : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// relu + round-to-nearest bf16 + pack in one instruction (exact: rounding
// preserves sign, so relu(round(x)) == round(relu(x))); a -> low half
__device__ __forceinline__ uint32_t pack_bf16_relu(float a, float b) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(b), "f"(a));
  return d;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
// byte offset of the 16-byte chunk (8 columns starting at col) of row r in a
// [K/64][128 rows][128 B] swizzled A tile
__device__ __forceinline__ uint32_t a_off(int r, int col) {
  const int kb = col >> 6, cc = (col & 63) >> 3;
  return (uint32_t)(kb * (ROWS * 128) + (r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4));
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// One epilogue half for one warp: its NM 32-column chunks of the accumulator
// -> registers -> (bias, ReLU, masks, head dot) -> packed bf16 -> A tile.  The
// first two packed chunks are held until the A columns are free (a_free),
// later chunks store directly.  Specialised per epilogue kind and chunk count
// so each fully unrolled loop carries only the arithmetic it needs.
template <int EPI, int NM, bool FOLD = false>
__device__ __forceinline__ void epi_chunks(const Step& st, int c_first, int r, uint32_t tmem_row, uint32_t a_row,
                                           uint32_t* my_masks, const float* head_w, float& head_part,
                                           uint32_t bar_free, uint32_t& free_ph, const float* sparams,
                                           const uint32_t (&mpre)[4]) {
  constexpr bool WA = EPI == E_RELU_A || EPI == E_RELU_MASK_A || EPI == E_MASKG_A || EPI == E_BWD_MASK_A ||
                     EPI == E_MASKG_HEAD_A;
  constexpr bool BIAS = EPI != E_BWD_MASK_A && !FOLD;   // FOLD: the bias is already in the accumulator
  constexpr int HOLD = NM < 2 ? NM : 2;
  const int r7 = r & 7;
  uint32_t hold[HOLD > 0 ? HOLD : 1][16];
  auto store = [&](int c, const uint32_t* pk) {
#ifdef DDF_EXP_NOST
    // timing experiment only (wrong results): no A-tile stores, what do they cost the MMAs beside them?
    if (pk[0] == 0x12345678u && pk[7] == 0x9abcdef0u) st_shared_v4(a_row, pk[0], pk[1], pk[2], pk[3]);
    return;
#endif
    // 4 x 16 B of one row into the 128B-swizzled A tile (row base a_row)
    const uint32_t blk = a_row + (uint32_t)((c >> 6) * (ROWS * 128));
    const int cc0 = (c & 63) >> 3;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      st_shared_v4(blk + (uint32_t)(((cc0 + e) ^ r7) << 4), pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
  };
  // chunk i's epilogue once its accumulator registers are loaded
  // biases and head weights live in shared memory: explicit ld.shared (short
  // scoreboard) rather than generic loads, issued before the TMEM wait
  const uint32_t bias_s = smem_u32(sparams) + 4u * (uint32_t)(size_t)st.bias;
  const uint32_t head_s = smem_u32(head_w);
  auto load_bias = [&](int c, float4 (&bq)[8]) {
#ifdef DDF_EXP_NOBIAS
    if constexpr (false) {
#else
    if constexpr (BIAS) {
#endif
  #pragma unroll
      for (int k = 0; k < 8; ++k) bq[k] = ld_shared_f4(bias_s + 4u * (uint32_t)(c + 4 * k));
    }
  };
  // z = accumulator + bias.  DDF_EXP_NOBIAS (timing experiment only, exact
  // only for zero biases) drops the add to measure what it costs
  auto zb = [](uint32_t acc, float b) {
#ifdef DDF_EXP_NOBIAS
    (void)b;
    return __uint_as_float(acc);
#else
    if constexpr (FOLD) return __uint_as_float(acc);
    else return __uint_as_float(acc) + b;
#endif
  };
  auto proc = [&](const int i, const int c, const uint32_t (&rg)[32], const float4 (&bq)[8]) {
      uint32_t mq = 0u;
      if constexpr (EPI == E_BWD_MASK_A) mq = mpre[i];   // prefetched before the accumulator wait
      const float* bf = reinterpret_cast<const float*>(bq);
      uint32_t pkd[16];
      if constexpr (EPI == E_BWD_MASK_A) {
  #pragma unroll
        for (int e = 0; e < 16; ++e)
          pkd[e] = pack_bf16(((mq >> (2 * e)) & 1u) ? __uint_as_float(rg[2 * e]) : 0.f,
                             ((mq >> (2 * e + 1)) & 1u) ? __uint_as_float(rg[2 * e + 1]) : 0.f);
      } else if constexpr (EPI == E_RELU_A) {
  #pragma unroll
        for (int e = 0; e < 16; ++e)
          pkd[e] = pack_bf16_relu(zb(rg[2 * e], bf[2 * e]), zb(rg[2 * e + 1], bf[2 * e + 1]));
      } else if constexpr (EPI == E_HEAD) {
  #pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 hw = ld_shared_f4(head_s + 4u * (uint32_t)(c + e));
          head_part = fmaf(fmaxf(zb(rg[e], bf[e]), 0.f), hw.x, head_part);
          head_part = fmaf(fmaxf(zb(rg[e + 1], bf[e + 1]), 0.f), hw.y, head_part);
          head_part = fmaf(fmaxf(zb(rg[e + 2], bf[e + 2]), 0.f), hw.z, head_part);
          head_part = fmaf(fmaxf(zb(rg[e + 3], bf[e + 3]), 0.f), hw.w, head_part);
        }
      } else {
        // ReLU mask bits of this row's 32 columns (neural.py:241 "h > 0")
        uint32_t mw = 0u;
        float v[32];
  #pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float z = zb(rg[e], bf[e]);
          mw |= (z > 0.f ? 1u : 0u) << e;
          // E_RELU_MASK_A packs with the relu-rounding convert (exact, see
          // pack_bf16_relu), so it keeps z and skips the FMNMX
          v[e] = EPI == E_RELU_MASK_A ? z : fmaxf(z, 0.f);
        }
        if constexpr (EPI == E_RELU_MASK_A) {
          my_masks[(st.mask_layer * 16 + (c >> 5)) * ROWS + r] = mw;
  #pragma unroll
          for (int e = 0; e < 16; ++e) pkd[e] = pack_bf16_relu(v[2 * e], v[2 * e + 1]);
        } else {   // E_MASKG_A: d/dh of the last hidden layer = w_head * mask
  #pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 hw = ld_shared_f4(head_s + 4u * (uint32_t)(c + e));
            if constexpr (EPI == E_MASKG_HEAD_A) {
              // the identity head of the forward, in E_HEAD's order (same fp32 result)
              head_part = fmaf(v[e], hw.x, head_part);
              head_part = fmaf(v[e + 1], hw.y, head_part);
              head_part = fmaf(v[e + 2], hw.z, head_part);
              head_part = fmaf(v[e + 3], hw.w, head_part);
            }
            v[e] = ((mw >> e) & 1u) ? hw.x : 0.f;
            v[e + 1] = ((mw >> (e + 1)) & 1u) ? hw.y : 0.f;
            v[e + 2] = ((mw >> (e + 2)) & 1u) ? hw.z : 0.f;
            v[e + 3] = ((mw >> (e + 3)) & 1u) ? hw.w : 0.f;
          }
  #pragma unroll
          for (int e = 0; e < 16; ++e) pkd[e] = pack_bf16(v[2 * e], v[2 * e + 1]);
        }
      }
      if constexpr (WA) {
        if (i < HOLD) {
  #pragma unroll
          for (int e = 0; e < 16; ++e) hold[i][e] = pkd[e];
        }
        if (i == HOLD - 1) {
          mbar_wait(bar_free, free_ph & 1u);
          ++free_ph;
  #pragma unroll
          for (int q2 = 0; q2 < HOLD; ++q2) store(c_first + q2 * 64, hold[q2]);
        } else if (i >= HOLD) {
          store(c, pkd);
        }
      }
  
  };
  // TMEM loads are software-pipelined one chunk ahead: chunk i + 1's load is
  // in flight while chunk i is processed (8 warps share the SM's TMEM read
  // port, so the next read overlaps this chunk's math and stores instead of
  // alternating with them).  tcgen05.wait::ld waits for every outstanding
  // load, hence one chunk of look-ahead.
  uint32_t rg[2][32];
#ifdef DDF_EXP_NOLD
  // timing experiment only (wrong results): no accumulator loads, what does the TMEM read port cost?
#pragma unroll
  for (int e = 0; e < 32; ++e) { rg[0][e] = (uint32_t)(r * 977 + e); rg[1][e] = (uint32_t)(r * 131 + e); }
#undef DDF_TMEM_LD32
#define DDF_TMEM_LD32(taddr, r_) ((void)0)
#endif
  if constexpr (NM > 0) {
    DDF_TMEM_LD32(tmem_row + (uint32_t)c_first, rg[0]);
    tmem_wait_ld();
  }
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    if (i + 1 < NM) DDF_TMEM_LD32(tmem_row + (uint32_t)(c_first + (i + 1) * 64), rg[(i + 1) & 1]);
    float4 bq[8];
    load_bias(c_first + i * 64, bq);
    proc(i, c_first + i * 64, rg[i & 1], bq);
    if (i + 1 < NM) tmem_wait_ld();
  }
  if constexpr (WA && NM == 0) ++free_ph;   // no columns in this half: keep the phase count in step
}

template <int EPI, bool FOLD = false>
__device__ __forceinline__ void epi_half(int nmine, const Step& st, int c_first, int r, uint32_t tmem_row,
                                         uint32_t a_row, uint32_t* my_masks, const float* head_w, float& head_part,
                                         uint32_t bar_free, uint32_t& free_ph, const float* sp,
                                         const uint32_t (&mpre)[4]) {
  switch (nmine) {
    case 0: epi_chunks<EPI, 0, FOLD>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, bar_free, free_ph, sp, mpre); break;
    case 1: epi_chunks<EPI, 1, FOLD>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, bar_free, free_ph, sp, mpre); break;
    case 2: epi_chunks<EPI, 2, FOLD>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, bar_free, free_ph, sp, mpre); break;
    case 3: epi_chunks<EPI, 3, FOLD>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, bar_free, free_ph, sp, mpre); break;
    default: epi_chunks<EPI, 4, FOLD>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, bar_free, free_ph, sp, mpre); break;
  }
}

// ------------------------------------------------------------------ input encoding
// bf16 A-tile columns [LO, HI) of one row from its 5 encoded inputs u.  The
// 6-octave sin/cos encoding (EXTENSION, configs 3-5) takes one sincospif per
// input and the double-angle recurrence sin 2x = 2 sin x cos x,
// cos 2x = (cos x - sin x)(cos x + sin x) for the higher octaves: fp32 error
// ~2^o ulp, far below the bf16 operand rounding.
__device__ __forceinline__ void pe_tables(const double u[5], float (&sn)[DDF_PE_OCTAVES][5],
                                          float (&cs)[DDF_PE_OCTAVES][5]) {
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    float sv, cv;
    sincospif((float)u[j], &sv, &cv);
    sn[0][j] = sv;
    cs[0][j] = cv;
#pragma unroll
    for (int o = 1; o < DDF_PE_OCTAVES; ++o) {
      const float s2 = 2.f * sv * cv, c2 = (cv - sv) * (cv + sv);
      sv = s2;
      cv = c2;
      sn[o][j] = sv;
      cs[o][j] = cv;
    }
  }
}
// Chain rule through the 65-D encoding for the tensor-core engines: the same
// fp32 sin/cos tables as the forward encoding (one sincospif per input and
// the double-angle recurrence), fp32 accumulation.  The gradient entering
// here is already fp32 from TMEM; the f64 restatement (field_kernels.cuh
// pe_chain) is kept for the fp32 SIMT parity engine.
template <class G>
__device__ __forceinline__ void pe_chain_tc(bool pe, const double u[5], G g, double out[5]) {
  float acc[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) acc[j] = g(j);
  if (pe) {
    float sn[DDF_PE_OCTAVES][5], cs[DDF_PE_OCTAVES][5];
    pe_tables(u, sn, cs);
#pragma unroll
    for (int o = 0; o < DDF_PE_OCTAVES; ++o) {
      const float f = (float)(1 << o) * 3.14159265358979f;
#pragma unroll
      for (int j = 0; j < 5; ++j)
        acc[j] = fmaf(f * cs[o][j], g(5 + 10 * o + j), fmaf(-f * sn[o][j], g(5 + 10 * o + 5 + j), acc[j]));
    }
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) out[j] = (double)acc[j];
}

template <int LO, int HI>
__device__ __forceinline__ void store_encoding(bool pe, bool valid, const double u[5], uint32_t a_tile, int r) {
  float sn[DDF_PE_OCTAVES][5], cs[DDF_PE_OCTAVES][5];
  if (pe && valid) pe_tables(u, sn, cs);
#pragma unroll
  for (int c = LO; c < HI; c += 8) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = c + e;
      float x = 0.f;
      if (valid) {
        if (k < 5) {
          x = (float)u[k];
        } else if (pe && k < 5 + 10 * DDF_PE_OCTAVES) {
          const int o = (k - 5) / 10, rr = (k - 5) % 10;
          x = rr < 5 ? sn[o][rr] : cs[o][rr - 5];
        }
      }
      v[e] = x;
    }
    st_shared_v4(a_tile + a_off(r, c), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                 pack_bf16(v[6], v[7]));
  }
}
// the row's half of the input columns: k0 = 16 (5 raw inputs) or 80 (65 PE inputs)
__device__ __forceinline__ void encode_row(int k0, int sub, bool pe, bool valid, const double u[5], uint32_t a_tile,
                                           int r) {
  if (k0 == 16) {
    if (sub == 0) store_encoding<0, 8>(false, valid, u, a_tile, r);
    else store_encoding<8, 16>(false, valid, u, a_tile, r);
  } else {
    if (sub == 0) store_encoding<0, 40>(pe, valid, u, a_tile, r);
    else store_encoding<40, 80>(pe, valid, u, a_tile, r);
  }
}

// ------------------------------------------------------------------ tiles
// Forward: tile t covers list rows [128 t, 128 t + 128) and runs every object.
// Gradient: tiles enumerate (object, 128-row block) over the object segments.
template <class Op>
__device__ __forceinline__ int n_tiles(const FieldDev& F, const Op& op) {
  if constexpr (Op::kGrad) {
    int t = 0;
    for (int j = 0; j < F.n_obj; ++j) t += (op.seg_end(j) - op.seg_begin(j) + ROWS - 1) / ROWS;
    return t;
  } else {
    return (op.total() + ROWS - 1) / ROWS;
  }
}
template <class Op>
__device__ __forceinline__ void tile_rows(const FieldDev& F, const Op& op, int t, int& j0, int& j1, int& base, int& nv) {
  if constexpr (Op::kGrad) {
    int j = 0;
    for (;; ++j) {
      const int c = (op.seg_end(j) - op.seg_begin(j) + ROWS - 1) / ROWS;
      if (t < c || j == F.n_obj - 1) break;
      t -= c;
    }
    base = op.seg_begin(j) + t * ROWS;
    nv = min(ROWS, op.seg_end(j) - base);
    j0 = j;
    j1 = j + 1;
  } else {
    base = t * ROWS;
    nv = min(ROWS, op.total() - base);
    j0 = 0;
    j1 = F.n_obj;
  }
}

struct Smem {
  uint8_t* a;           // A tile, 1024-aligned
  uint8_t* stages;      // weight stages
  uint64_t* bars;       // [0..1] a_ready, [2..3] acc_ready, [4..5] a_free, [6..6+S) w_full, [..+S) w_empty
  uint32_t* tmem_slot;
  float* red;           // [2][128] head partial sums
  float* params;        // current network's biases + head weights
};

// ------------------------------------------------------------------ kernel
template <class Op>
__global__ void __launch_bounds__(NTHREADS, 1)
mlp_kernel(const FieldDev F, const Op op, uint32_t* __restrict__ mask_scratch, int n_stages, int a_bytes,
           int stage_bytes, int params_bytes, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // fused trace+gradient (Op::kFused): the gradient program, whose last
  // forward epilogue also forms the head and hands the distance to the row op
  constexpr bool kProgG = Op::kGrad || Op::kFused;
  uint8_t* base_ptr = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Smem S;
  S.a = base_ptr;
  S.stages = base_ptr + a_bytes;
  S.bars = reinterpret_cast<uint64_t*>(S.stages + (size_t)((dbg & 8) ? 1 : n_stages) * stage_bytes);
  S.tmem_slot = reinterpret_cast<uint32_t*>(S.bars + 6 + 2 * n_stages);
  S.red = reinterpret_cast<float*>(S.tmem_slot + 4);
  S.params = S.red + 2 * ROWS;
  // the bias fold's constant A block (step_has_bias), aligned to its 256-byte swizzle atom
  uint8_t* ones = reinterpret_cast<uint8_t*>(((uintptr_t)(S.params + (params_bytes >> 2)) + 255) & ~(uintptr_t)255);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(S.bars);
  auto BAR_A_READY = [&](int h) { return bar0 + 8u * (0 + h); };
  auto BAR_ACC = [&](int h) { return bar0 + 8u * (2 + h); };
  auto BAR_A_FREE = [&](int h) { return bar0 + 8u * (4 + h); };
  auto BAR_FULL = [&](int s) { return bar0 + 8u * (6 + s); };
  auto BAR_EMPTY = [&](int s) { return bar0 + 8u * (6 + n_stages + s); };

  if (threadIdx.x == 0) {
    for (int h = 0; h < 2; ++h) {
      mbar_init(BAR_A_READY(h), N_EPI_WARPS);
      mbar_init(BAR_ACC(h), 1);
      mbar_init(BAR_A_FREE(h), 1);
    }
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
  write_ones_block(ones, threadIdx.x, blockDim.x);
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *S.tmem_slot;
  const uint32_t a_base = smem_u32(S.a);
  const uint32_t st_base = smem_u32(S.stages);
  const int tiles = n_tiles(F, op);
  const int sstride = (dbg & 8) ? 0 : stage_bytes;   // dbg 8: all stages alias one buffer (timing only)
  unsigned long long dbg_acc[16];
  if (kStats)
    for (int i = 0; i < 16; ++i) dbg_acc[i] = 0ull;

  if (warp == 0) {
    // ================================================= weight producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int j0, j1, base, nv;
        tile_rows(F, op, t, j0, j1, base, nv);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = __ldg(kProgG ? &P->n_grad : &P->n_fwd);
          const uint8_t* img = kProgG ? P->img_grad : P->img_fwd;
          for (int s = 0; s < ns; ++s) {
            const Step st = load_step(kProgG ? &P->grad[s] : &P->fwd[s]);
            const uint8_t* src = img + st.img_off;
            const bool fold = step_has_bias(st.epi);   // wide programs carry a bias chunk ahead of each N-half
            const int per_half = st.nchunk + (fold ? 1 : 0);
            const int nck = st.nh * per_half;
            for (int c = 0; c < nck; ++c) {
              const uint32_t bytes = (fold && c % per_half == 0) ? (uint32_t)(st.rows * 32) : (uint32_t)st.chunk_bytes;
              {
                DDF_DBG_T0();
                mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
                DDF_DBG_ADD(6);
              }
              if (dbg & 1) {   // timing experiment only: no weight traffic (wrong results)
                mbar_arrive(BAR_FULL(stage));
              } else {
                mbar_expect_tx(BAR_FULL(stage), bytes);
                bulk_g2s(st_base + (uint32_t)(stage * sstride), src, bytes, BAR_FULL(stage));
              }
              src += bytes;
              if (++stage == n_stages) { stage = 0; phase ^= 1u; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer
    // The whole warp runs this loop in converged, warp-uniform control flow;
    // each tcgen05 instruction is issued by one elected lane.  The chunk loop
    // carries only the weight wait, the four-MMA issue and the ring advance:
    // the issuing thread's instruction latency, not the tensor pipe, had
    // paced this engine (~750 cycles per 512-cycle chunk with per-chunk
    // bookkeeping in a lane-0 branch).
    {
      DDF_DBG_T0();
      TraceCursor tcur{1, 0};
      int stage = 0;
      uint32_t phase = 0;
      uint32_t ar[2] = {0u, 0u};
      const uint64_t da0 = sdesc(a_base), db0 = sdesc(st_base);
      const uint32_t da0_lo = sdesc_lo(a_base), db0_lo = sdesc_lo(st_base);
      const uint32_t sstep = (uint32_t)sstride >> 4;
      const uint32_t ones_lo = sdesc_lo(smem_u32(ones));
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int j0, j1, base, nv;
        tile_rows(F, op, t, j0, j1, base, nv);
        const bool trc = kTrace && blockIdx.x == 0 && lane == 0 &&
                         (t - (int)blockIdx.x) / (int)gridDim.x >= TRACE_TILE0 &&
                         (t - (int)blockIdx.x) / (int)gridDim.x < TRACE_TILE0 + TRACE_TILES;
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = kProgG ? P->n_grad : P->n_fwd;
          int prev_rows = 1 << 30;
          for (int s = 0; s < ns; ++s) {
            const Step st = load_step(kProgG ? &P->grad[s] : &P->fwd[s]);
            const uint32_t id = idesc(st.rows);
            const bool wa = writes_a(st.epi);
            const bool fold = step_has_bias(st.epi);
            // chunks [0, kc1) read A columns < K/2 (A_READY(0)), the rest also
            // columns >= K/2 (A_READY(1)); in the last N-half, A_FREE(0) follows
            // chunk c0 (the last reading A columns < N/2) and A_FREE(1) the last
            const int kc1 = min(st.nchunk, (st.K >> 1) >> 6);
            const int c0 = min(st.nchunk - 1, ((st.N >> 1) - 1) >> 6);
            const int nfull = st.K >> 6;                 // chunks of four K = 16 MMAs
            bool waited0 = false, waited1 = false;
            auto wait_a = [&](int which) {
              DDF_DBG_T0();
              tcur.ev(trc, which ? 3 : 1, s, 0);
              mbar_wait(BAR_A_READY(which), ar[which] & 1u);
              ++ar[which];
              tcur.ev(trc, which ? 4 : 2, s, 0);
              if (lane == 0) DDF_DBG_ADD(0);
            };
            if (st.rows > prev_rows) {
              // half 0 of this step would overwrite TMEM columns of the previous
              // step's half 1: wait until both previous epilogue halves are done
              wait_a(0); wait_a(1);
              waited0 = waited1 = true;
            }
            prev_rows = st.rows;
            for (int h = 0; h < st.nh; ++h) {
              const uint32_t td = tmem + (uint32_t)(h * st.rows);
              const bool last_half = h == st.nh - 1;
              // chunk segments: [kc_a, kc_b) issued back to back, the waits and
              // A_FREE commits between segments
              int kc = 0;
              while (kc < st.nchunk) {
                if (kc == 0 && !waited0) { wait_a(0); waited0 = true; }
                if (kc >= kc1 && !waited1) { wait_a(1); waited1 = true; }
                if (kc == 0 && fold) {
                  // the half's accumulator starts as its bias (ones block x bias chunk), the K chunks add to it
                  mbar_wait(BAR_FULL(stage), phase);
                  tc_after_sync();
                  mma_bias_w(td, ones_lo, db0_lo + (uint32_t)stage * sstep, id, 0u);
                  tc_commit_w(BAR_EMPTY(stage));
                  if (++stage == n_stages) { stage = 0; phase ^= 1u; }
                }
                int kend = st.nchunk;
                if (!waited1 && kc1 > kc) kend = min(kend, kc1);
                if (wa && last_half && c0 >= kc) kend = min(kend, c0 + 1);
                const int kfull = min(kend, nfull);
                if (kc == 0) tcur.ev(trc, 6, s, h);
                for (; kc < kfull; ++kc) {
                  mbar_wait(BAR_FULL(stage), phase);
                  tc_after_sync();
                  if (kStats && (dbg & 128)) {   // dbg 128: timing experiment only, no MMAs (wrong results)
                    tc_commit_w(BAR_EMPTY(stage));
                  } else {
                    mma_k64_commit_w(td, da0_lo + (uint32_t)(kc * (ROWS * 128 / 16)), db0_lo + (uint32_t)stage * sstep,
                                     id, (kc || fold) ? 1u : 0u, BAR_EMPTY(stage));
                  }
                  tcur.ev(trc, 8, s, h);                  // 8: K chunk issued
                  if (++stage == n_stages) { stage = 0; phase ^= 1u; }
                }
                if (kc < kend) {
                  // the partial last chunk (K not a multiple of 64: the input layer)
                  mbar_wait(BAR_FULL(stage), phase);
                  tc_after_sync();
                  const int nks = (st.K - kc * 64 + 15) >> 4;
                  const uint64_t da = da0 + (uint64_t)(kc * (ROWS * 128 / 16));
                  const uint64_t db = db0 + (uint64_t)(stage * sstep);
                  for (int ks = 0; ks < nks; ++ks) mma_bf16_w(td, da + 2 * ks, db + 2 * ks, id, (kc | ks || fold) ? 1u : 0u);
                  tc_commit_w(BAR_EMPTY(stage));
                  if (++stage == n_stages) { stage = 0; phase ^= 1u; }
                  ++kc;
                }
                if (wa && last_half) {
                  if (kc == c0 + 1) tc_commit_w(BAR_A_FREE(0));
                  if (kc == st.nchunk) tc_commit_w(BAR_A_FREE(1));
                }
              }
              tc_commit_w(BAR_ACC(h));
              tcur.ev(trc, 7, s, h);                       // 7: last chunk of the half issued
            }
            if (kStats && lane == 0) atomicAdd(&g_dbg[5], 1ull);
            if (!waited1) wait_a(1);   // keep phases in step
          }
        }
      }
      if (lane == 0) DDF_DBG_ADD(4);
    }
  } else {
    // ================================================= row warps (encoding + epilogues)
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int sub = (warp - EPI_WARP0) >> 2;   // column split between the two warps of a quarter
    const int r = q * 32 + lane;         // tile row == TMEM lane
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t a_row = a_base + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);   // this row in every A k-block
    uint32_t* my_masks = mask_scratch + (size_t)blockIdx.x * MASK_WORDS_PER_CTA;
    uint32_t acc_ph[2] = {0u, 0u}, free_ph[2] = {0u, 0u};
    TraceCursor tcur{warp == EPI_WARP0 ? 2 : 3, 0};
    int staged_j = -1;   // network whose params are in shared memory
    // this row of the next tile: list entry and path state fetched one tile
    // ahead (issued once the current tile's encoding is stored, so the two
    // dependent global round trips overlap the first layer's MMAs instead of
    // sitting between tiles with the tensor pipe idle)
    int n_slot = 0;
    double n_pos[3] = {0.0, 0.0, 0.0}, n_az = 0.0, n_pol = 0.0;
    auto fetch = [&](int tt) {
      if (tt < tiles) {
        int a0, a1, b0, c0;
        tile_rows(F, op, tt, a0, a1, b0, c0);
        if (r < c0) {
          n_slot = op.slot(b0 + r);
          if constexpr (!Op::kRaw) op.load(n_slot, n_pos, n_az, n_pol);
        }
      }
    };
    fetch(blockIdx.x);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int j0, j1, base, nv;
      tile_rows(F, op, t, j0, j1, base, nv);
      const bool valid = r < nv;
      const int slot = valid ? n_slot : 0;
      const bool trc = kTrace && blockIdx.x == 0 && lane == 0 && (warp == EPI_WARP0 || warp == EPI_WARP0 + 7) &&
                       (t - (int)blockIdx.x) / (int)gridDim.x >= TRACE_TILE0 &&
                       (t - (int)blockIdx.x) / (int)gridDim.x < TRACE_TILE0 + TRACE_TILES;
      tcur.ev(trc, 16, 0, 0);                                  // 16: tile start (encoding begins)
      double pos[3] = {n_pos[0], n_pos[1], n_pos[2]}, az = n_az, pol = n_pol;
      double best = 0.0;
      int bobj = 0;
      for (int j = j0; j < j1; ++j) {
        const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
        const NetDev& net = F.net[j];
        // this network's biases + head weights -> shared memory, only when the
        // network changes (a single-network field stages them once per launch;
        // every epilogue warp is past the previous network's last use: HEAD
        // ends in a named barrier, gradient programs end with BWD_OUT which
        // reads none)
        const int head_off = __ldg(&P->head_off);
        if (j != staged_j) {
          staged_j = j;
          const int nf = __ldg(&P->params_floats);
          const float4* src = reinterpret_cast<const float4*>(P->params);
          float4* dst = reinterpret_cast<float4*>(S.params);
          named_sync(1, N_EPI_WARPS * 32);
          for (int i = threadIdx.x - EPI_WARP0 * 32; i < (nf >> 2); i += N_EPI_WARPS * 32) dst[i] = __ldg(src + i);
          named_sync(1, N_EPI_WARPS * 32);
        }
        double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if constexpr (!Op::kRaw) {
          if (valid) row_u(F, j, pos, az, pol, u);
        }
        // ---- input encoding -> A columns [sub*k0/2, (sub+1)*k0/2)
        if constexpr (!Op::kRaw) {
          encode_row(P->k0, sub, net.encoding == ENC_PE6, valid, u, a_base, r);
        } else {
          const int k0 = P->k0, half = k0 >> 1;
          for (int c = sub * half; c < (sub + 1) * half; c += 8) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = valid ? (float)op.raw(slot, c + e) : 0.f;
            st_shared_v4(a_base + a_off(r, c), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                         pack_bf16(v[6], v[7]));
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) { mbar_arrive(BAR_A_READY(0)); mbar_arrive(BAR_A_READY(1)); }
        tcur.ev(trc, 20, 0, 0);                        // 20: encoding stored
        if (j == j0) fetch(t + gridDim.x);

        const int ns = kProgG ? P->n_grad : P->n_fwd;
        float head_part = 0.f;
        for (int s = 0; s < ns; ++s) {
          const Step st = load_step(kProgG ? &P->grad[s] : &P->fwd[s]);
          const int epi = st.epi;
          const bool wa = writes_a(epi);
          for (int h = 0; h < st.nh; ++h) {
            const int col0 = h * st.rows;
            const int c_first = col0 + sub * 32;
            // ReLU mask words of the backward epilogue: load before the wait
            uint32_t mpre[4] = {0u, 0u, 0u, 0u};
            if (epi == E_BWD_MASK_A) {
              const int nm = (st.rows - sub * 32 + 63) >> 6;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (i < nm) mpre[i] = my_masks[(st.mask_layer * 16 + ((c_first + 64 * i) >> 5)) * ROWS + r];
            }
            {
              DDF_DBG_T0();
              tcur.ev(trc, 17, s, h);                  // 17: wait for the accumulator begins
              mbar_wait(BAR_ACC(h), acc_ph[h] & 1u);
              tcur.ev(trc, 18, s, h);                  // 18: accumulator ready
              if (threadIdx.x == EPI_WARP0 * 32) DDF_DBG_ADD(2);
            }
            ++acc_ph[h];
            tc_after_sync();
            if ((kStats || DDF_ALLOW_DBG) && (dbg & 2048)) {   // dbg 2048: timing only, no epilogue (wrong results)
              tc_before_sync();
              if (wa) {
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(BAR_A_READY(h));
              }
              continue;
            }
            if (epi == E_BWD_OUT) {
              if (sub == 0) {
                // d pred / d inputs for this row: st.rows (= k0) fp32 columns
                float g[128];
                for (int c = 0; c < st.rows; c += 16) {
                  uint32_t rg[16];
                  DDF_TMEM_LD16(tmem + lane_addr + (uint32_t)c, rg);
                  tmem_wait_ld();
#pragma unroll
                  for (int e = 0; e < 16; ++e) g[c + e] = __uint_as_float(rg[e]);
                }
                if constexpr (kProgG) {
                  if (valid) {
                    if constexpr (Op::kRaw) {
                      op.store_grad_raw(slot, [&](int k) { return (double)g[k]; });
                    } else {
                      double g5[5];
                      pe_chain_tc(net.encoding == ENC_PE6, u, [&](int k) { return g[k]; }, g5);
                      op.store_grad(slot, g5);
                    }
                  }
                }
              }
              tc_before_sync();
              continue;
            }
            // TMEM -> registers -> epilogue math -> packed bf16, all before the A
            // columns are free; only the shared stores wait for a_free
            const int nmine = (st.rows - sub * 32 + 63) >> 6;   // 32-col chunks of this warp
            const long long t_epi = kStats ? clock64() : 0;
            switch (epi) {
              case E_RELU_A:
                epi_half<E_RELU_A, true>(nmine, st, c_first, r, tmem + lane_addr, a_row, my_masks, S.params + head_off, head_part, BAR_A_FREE(h), free_ph[h], S.params, mpre);
                break;
              case E_RELU_MASK_A:
                epi_half<E_RELU_MASK_A, true>(nmine, st, c_first, r, tmem + lane_addr, a_row, my_masks, S.params + head_off, head_part, BAR_A_FREE(h), free_ph[h], S.params, mpre);
                break;
              case E_MASKG_A:
                if constexpr (Op::kFused)
                  epi_half<E_MASKG_HEAD_A, true>(nmine, st, c_first, r, tmem + lane_addr, a_row, my_masks, S.params + head_off, head_part, BAR_A_FREE(h), free_ph[h], S.params, mpre);
                else
                epi_half<E_MASKG_A, true>(nmine, st, c_first, r, tmem + lane_addr, a_row, my_masks, S.params + head_off, head_part, BAR_A_FREE(h), free_ph[h], S.params, mpre);
                break;
              case E_BWD_MASK_A:
                epi_half<E_BWD_MASK_A, true>(nmine, st, c_first, r, tmem + lane_addr, a_row, my_masks, S.params + head_off, head_part, BAR_A_FREE(h), free_ph[h], S.params, mpre);
                break;
              default:
                epi_half<E_HEAD, true>(nmine, st, c_first, r, tmem + lane_addr, a_row, my_masks, S.params + head_off, head_part, BAR_A_FREE(h), free_ph[h], S.params, mpre);
                break;
            }
            if (kStats && threadIdx.x == EPI_WARP0 * 32) dbg_acc[7] += (unsigned long long)(clock64() - t_epi);
            tc_before_sync();
            if (wa) {
              fence_async_smem();
              __syncwarp();
              if (lane == 0) mbar_arrive(BAR_A_READY(h));
            }
            tcur.ev(trc, 19, s, h);                    // 19: epilogue of the half done
          }
          if (epi == E_HEAD || (Op::kFused && epi == E_MASKG_A)) {
            S.red[sub * ROWS + r] = head_part;
            named_sync(1, N_EPI_WARPS * 32);
            if (sub == 0) {
              double p = (double)(S.red[r] + S.red[ROWS + r] + P->head_b);
              if (F.composite) p = dmul(net.scale, p);
              if (j == j0 || p < best) { best = p; bobj = j; }
              // fused: the row op sees the distance before the backward's
              // E_BWD_OUT (same thread) decides whether to keep the gradient
              if constexpr (Op::kFused) {
                if (valid) op.store_fwd(slot, best, bobj);
              }
            }
            named_sync(1, N_EPI_WARPS * 32);
          }
        }
      }
      if constexpr (!Op::kGrad && !Op::kFused) {
        if (sub == 0 && valid) op.store_fwd(slot, best, bobj);
      }
    }
  }
  if (lane == 0 && (warp == 0 || warp == 1 || warp == EPI_WARP0)) DDF_DBG_FLUSH();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}


// ================================================================== ping-pong
// Networks whose hidden layers are at most 256 wide run two 128-row tiles
// ("slots" X, Y) through the layers in lock-step: the MMA warp issues layer s
// of X (one full-N chain, N <= 256), then layer s of Y, then s+1 of X...  The
// epilogue of X's layer s (TMEM -> bias/ReLU -> bf16 A_X) overlaps the MMAs of
// Y's layer s, so the tensor pipe never waits for an epilogue.  TMEM: X in
// columns [0, 256), Y in [256, 512).  Each slot has its own A tile, barriers,
// ReLU-mask scratch and staged params.  The MMAs of a slot's step complete
// before its epilogue writes the slot's A tile, so no a_free barriers exist.

// One warp's NM 32-column chunks (STRIDE columns apart) of a slot's accumulator.
// TMEM loads run one chunk ahead of the arithmetic (the chain TMEM load ->
// bias/ReLU/pack -> shared stores is latency-bound when run back to back),
// biases and head weights come through explicit ld.shared.
template <int EPI, int NM, int STRIDE = 64>
__device__ __forceinline__ void epi_direct(const Step& st, int c_first, int r, uint32_t tmem_row, uint32_t a_row,
                                           uint32_t* my_masks, const float* head_w, float& head_part,
                                           const float* sparams) {
  const int r7 = r & 7;
  (void)sparams;
  uint32_t rgb[2][32];
  DDF_TMEM_LD32(tmem_row + (uint32_t)c_first, rgb[0]);
  uint32_t mq_next = 0u;
  if constexpr (EPI == E_BWD_MASK_A) mq_next = my_masks[(st.mask_layer * 16 + (c_first >> 5)) * ROWS + r];
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const int c = c_first + i * STRIDE;
    if (i + 1 < NM) DDF_TMEM_LD32(tmem_row + (uint32_t)(c + STRIDE), rgb[(i + 1) & 1]);
    const uint32_t(&rg)[32] = rgb[i & 1];
    // no bias here: it is already in the accumulator (step_has_bias)
    const uint32_t mq = mq_next;
    if constexpr (EPI == E_BWD_MASK_A) {
      if (i + 1 < NM) mq_next = my_masks[(st.mask_layer * 16 + ((c + STRIDE) >> 5)) * ROWS + r];
    }
    uint32_t pkd[16];
    if constexpr (EPI == E_BWD_MASK_A) {
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pkd[e] = pack_bf16(((mq >> (2 * e)) & 1u) ? __uint_as_float(rg[2 * e]) : 0.f,
                           ((mq >> (2 * e + 1)) & 1u) ? __uint_as_float(rg[2 * e + 1]) : 0.f);
    } else if constexpr (EPI == E_RELU_A) {
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pkd[e] = pack_bf16_relu(__uint_as_float(rg[2 * e]), __uint_as_float(rg[2 * e + 1]));
    } else if constexpr (EPI == E_HEAD) {
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        const float4 hw = __ldg(reinterpret_cast<const float4*>(head_w + c + e));
        head_part = fmaf(fmaxf(__uint_as_float(rg[e]), 0.f), hw.x, head_part);
        head_part = fmaf(fmaxf(__uint_as_float(rg[e + 1]), 0.f), hw.y, head_part);
        head_part = fmaf(fmaxf(__uint_as_float(rg[e + 2]), 0.f), hw.z, head_part);
        head_part = fmaf(fmaxf(__uint_as_float(rg[e + 3]), 0.f), hw.w, head_part);
      }
    } else {
      uint32_t mw = 0u;
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float z = __uint_as_float(rg[e]);
        mw |= (z > 0.f ? 1u : 0u) << e;
        v[e] = z;
      }
      if constexpr (EPI == E_RELU_MASK_A) {
        my_masks[(st.mask_layer * 16 + (c >> 5)) * ROWS + r] = mw;
#pragma unroll
        for (int e = 0; e < 16; ++e) pkd[e] = pack_bf16_relu(v[2 * e], v[2 * e + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 hw = __ldg(reinterpret_cast<const float4*>(head_w + c + e));
          v[e] = ((mw >> e) & 1u) ? hw.x : 0.f;
          v[e + 1] = ((mw >> (e + 1)) & 1u) ? hw.y : 0.f;
          v[e + 2] = ((mw >> (e + 2)) & 1u) ? hw.z : 0.f;
          v[e + 3] = ((mw >> (e + 3)) & 1u) ? hw.w : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) pkd[e] = pack_bf16(v[2 * e], v[2 * e + 1]);
      }
    }
    if constexpr (EPI != E_HEAD) {
      const uint32_t blk = a_row + (uint32_t)((c >> 6) * (ROWS * 128));
      const int cc0 = (c & 63) >> 3;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        st_shared_v4(blk + (uint32_t)(((cc0 + e) ^ r7) << 4), pkd[4 * e], pkd[4 * e + 1], pkd[4 * e + 2],
                     pkd[4 * e + 3]);
    }
    if (i + 1 < NM) tmem_wait_ld();
  }
}

template <int EPI>
__device__ __forceinline__ void epi_direct_n(int nm, const Step& st, int c_first, int r, uint32_t tmem_row,
                                             uint32_t a_row, uint32_t* my_masks, const float* head_w,
                                             float& head_part, const float* sp) {
  switch (nm) {
    case 1: epi_direct<EPI, 1>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, sp); break;
    case 2: epi_direct<EPI, 2>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, sp); break;
    case 3: epi_direct<EPI, 3>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, sp); break;
    case 4: epi_direct<EPI, 4>(st, c_first, r, tmem_row, a_row, my_masks, head_w, head_part, sp); break;
    default: break;
  }
}

// Pack p of a CTA (NS tiles) -> (objects, row block) of slot `sl`.  Gradient
// passes pad each object's tile count to a multiple of NS so all slots of a
// pack run the same network.
template <class Op, int NS = 2>
__device__ __forceinline__ int pp_pairs(const FieldDev& F, const Op& op) {
  if constexpr (Op::kGrad) {
    int t = 0;
    for (int j = 0; j < F.n_obj; ++j) t += ((op.seg_end(j) - op.seg_begin(j) + ROWS - 1) / ROWS + NS - 1) / NS;
    return t;
  } else {
    return ((op.total() + ROWS - 1) / ROWS + NS - 1) / NS;
  }
}
template <class Op, int NS = 2>
__device__ __forceinline__ void pp_rows(const FieldDev& F, const Op& op, int p, int sl, int& j0, int& j1, int& base,
                                        int& nv) {
  if constexpr (Op::kGrad) {
    int j = 0;
    for (;; ++j) {
      const int c = ((op.seg_end(j) - op.seg_begin(j) + ROWS - 1) / ROWS + NS - 1) / NS;
      if (p < c || j == F.n_obj - 1) break;
      p -= c;
    }
    base = op.seg_begin(j) + (NS * p + sl) * ROWS;
    nv = max(0, min(ROWS, op.seg_end(j) - base));
    j0 = j;
    j1 = j + 1;
  } else {
    base = (NS * p + sl) * ROWS;
    nv = max(0, min(ROWS, op.total() - base));
    j0 = 0;
    j1 = F.n_obj;
  }
}

template <class Op>
__global__ void __launch_bounds__(NTHREADS, 1)
mlp_pp_kernel(const FieldDev F, const Op op, uint32_t* __restrict__ mask_scratch, int n_stages, int a_bytes,
              int stage_bytes, int params_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base_ptr = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* a_tiles = base_ptr;                                   // [2][a_bytes]
  uint8_t* stages = base_ptr + 2 * (size_t)a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)n_stages * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 + 2 * n_stages);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);           // [2 slots][2 subs][128]
  (void)params_bytes;   // nothing of a network's params is staged: biases are folded, head weights read in place
  // the bias fold's constant A block, aligned to its 256-byte swizzle atom
  uint8_t* ones = reinterpret_cast<uint8_t*>(((uintptr_t)(red + 4 * ROWS) + 255) & ~(uintptr_t)255);

  const int warp = uni((int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;   // warp index, provably warp-uniform
  const uint32_t bar0 = smem_u32(bars);
  auto BAR_A_READY = [&](int sl) { return bar0 + 8u * sl; };
  auto BAR_ACC = [&](int sl) { return bar0 + 8u * (2 + sl); };
  auto BAR_FULL = [&](int s) { return bar0 + 8u * (4 + s); };
  auto BAR_EMPTY = [&](int s) { return bar0 + 8u * (4 + n_stages + s); };

  if (threadIdx.x == 0) {
    for (int sl = 0; sl < 2; ++sl) {
      mbar_init(BAR_A_READY(sl), N_EPI_WARPS);
      mbar_init(BAR_ACC(sl), 1);
    }
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(BAR_FULL(s), 1);
      mbar_init(BAR_EMPTY(s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  write_ones_block(ones, threadIdx.x, blockDim.x);
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base0 = smem_u32(a_tiles);
  const uint32_t st_base = smem_u32(stages);
  const int pairs = pp_pairs(F, op);

  if (warp == 0) {
    // ================================================= weight producer (each step streamed once per slot)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        int j0, j1, base, nv;
        pp_rows(F, op, pr, 0, j0, j1, base, nv);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
          const uint8_t* img = Op::kGrad ? P->img_grad : P->img_fwd;
          for (int s = 0; s < ns; ++s) {
            const Step st = load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            const int nck = st.nchunk + (step_has_bias(st.epi) ? 1 : 0);   // + the bias chunk (rows x 32 B)
            for (int sl = 0; sl < 2; ++sl) {
              const uint8_t* src = img + st.img_off;
              for (int c = 0; c < nck; ++c) {
                const uint32_t bytes = c < st.nchunk ? (uint32_t)st.chunk_bytes : (uint32_t)(st.rows * 32);
                mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
                mbar_expect_tx(BAR_FULL(stage), bytes);
                bulk_g2s(st_base + (uint32_t)(stage * stage_bytes), src, bytes, BAR_FULL(stage));
                src += st.chunk_bytes;
                if (++stage == n_stages) { stage = 0; phase ^= 1u; }
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer (whole warp, converged, on
    // warp-uniform values: see uni / mbar_wait_u)
    {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t ar = 0u;                              // A_READY phase: each slot completes one per step
      const uint32_t tmem_u = uni(tmem), bars_u = uni(bar0);
      const uint32_t a0_lo = uni(sdesc_lo(a_base0)), db0_lo = uni(sdesc_lo(st_base));
      const uint32_t a_step = uni((uint32_t)a_bytes >> 4), sstep = uni((uint32_t)stage_bytes >> 4);
      const int nst = uni(n_stages), pairs_u = uni(pairs);
      const uint32_t ones_lo = uni(sdesc_lo(smem_u32(ones)));
      TraceCursor tcur{1, 0};
      for (int pr = blockIdx.x; pr < pairs_u; pr += gridDim.x) {
        int j0, j1, base, nv;
        pp_rows(F, op, pr, 0, j0, j1, base, nv);
        j0 = uni(j0);
        j1 = uni(j1);
        const bool trc = kTrace && blockIdx.x == 0 && lane == 0 && (pr - (int)blockIdx.x) / (int)gridDim.x >= TRACE_TILE0 &&
                         (pr - (int)blockIdx.x) / (int)gridDim.x < TRACE_TILE0 + TRACE_TILES;
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = uni(__ldg(Op::kGrad ? &P->n_grad : &P->n_fwd));
          const bool k32 = uni(__ldg(&P->chunk_k)) == 32;   // 256-wide programs: chunks of 32 K columns
          for (int s = 0; s < ns; ++s) {
            Step st = load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            uni_step(st);
            const uint32_t id = idesc(st.rows);
            const int nfull = k32 ? st.K >> 5 : st.K >> 6;   // chunks of two / four K = 16 MMAs
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              // this slot's A tile (and its TMEM columns) are ready
              tcur.ev(trc, 1, s * 2 + sl, 0);                // 1: wait for the slot's A tile begins
              mbar_wait_u(bars_u + 8u * sl, ar & 1u);
              tcur.ev(trc, 2, s * 2 + sl, 0);                // 2: A tile ready
              tc_after_sync();
              const uint32_t da_lo = a0_lo + (uint32_t)sl * a_step;
              const uint32_t td = tmem_u + (uint32_t)(sl * 256);
              for (int kc = 0; kc < st.nchunk; ++kc) {
                mbar_wait_u(bars_u + 8u * (uint32_t)(4 + stage), phase);
                tc_after_sync();
                const uint32_t db = db0_lo + (uint32_t)stage * sstep;
                const uint32_t bar_empty = bars_u + 8u * (uint32_t)(4 + nst + stage);
                if (k32) {
                  // chunk kc = A columns [32 kc, 32 kc + 32): k-block kc / 2 of the A tile, its half kc & 1
                  const uint32_t da = da_lo + (uint32_t)((kc >> 1) * (ROWS * 128 / 16) + (kc & 1) * 4);
                  if (kc < nfull) {
                    mma_k32_commit_w(td, da, db, id, kc ? 1u : 0u, bar_empty);
                  } else {   // a last chunk of 16 K columns (the input layer)
                    mma_bf16_w(td, ((uint64_t)SDESC_HI << 32) | da, ((uint64_t)SDESC64B_HI << 32) | db, id, kc ? 1u : 0u);
                    tc_commit_w(bar_empty);
                  }
                } else {
                  const uint32_t da = da_lo + (uint32_t)(kc * (ROWS * 128 / 16));
                  if (kc < nfull) {
                    mma_k64_commit_w(td, da, db, id, kc ? 1u : 0u, bar_empty);
                  } else {
                    const int nks = (st.K - kc * 64 + 15) >> 4;
                    for (int ks = 0; ks < nks; ++ks)
                      mma_bf16_w(td, ((uint64_t)SDESC_HI << 32) | (da + 2 * ks), ((uint64_t)SDESC_HI << 32) | (db + 2 * ks), id,
                                 (kc | ks) ? 1u : 0u);
                    tc_commit_w(bar_empty);
                  }
                }
                if (++stage == nst) { stage = 0; phase ^= 1u; }
              }
              if (step_has_bias(st.epi)) {   // D += bias (the step's last chunk, see step_has_bias)
                mbar_wait_u(bars_u + 8u * (uint32_t)(4 + stage), phase);
                tc_after_sync();
                mma_bias_w(td, ones_lo, db0_lo + (uint32_t)stage * sstep, id);
                tc_commit_w(bars_u + 8u * (uint32_t)(4 + nst + stage));
                if (++stage == nst) { stage = 0; phase ^= 1u; }
              }
              tc_commit_w(bars_u + 8u * (uint32_t)(2 + sl));
              tcur.ev(trc, 7, s * 2 + sl, 0);                // 7: the slot's layer issued
            }
            ++ar;
          }
        }
      }
    }
  } else {
    // ================================================= row warps
    const int q = warp & 3;
    const int sub = (warp - EPI_WARP0) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t acc_ph[2] = {0u, 0u};
    // this row of the next pair of tiles: list entries and path state fetched
    // one pair ahead (issued once the current encodings are stored), so the
    // dependent global round trips overlap the first layer's MMAs
    int n_slot[2] = {0, 0};
    double n_pos[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}}, n_az[2] = {0.0, 0.0}, n_pol[2] = {0.0, 0.0};
    auto fetch = [&](int pp) {
      if (pp < pairs) {
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          int a0, a1, b0, c0;
          pp_rows(F, op, pp, sl, a0, a1, b0, c0);
          if (r < c0) {
            n_slot[sl] = op.slot(b0 + r);
            if constexpr (!Op::kRaw) op.load(n_slot[sl], n_pos[sl], n_az[sl], n_pol[sl]);
          }
        }
      }
    };
    fetch(blockIdx.x);
    TraceCursor tcur{warp == EPI_WARP0 ? 2 : 3, 0};
    for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
      const bool trc = kTrace && blockIdx.x == 0 && lane == 0 && (warp == EPI_WARP0 || warp == EPI_WARP0 + 7) &&
                       (pr - (int)blockIdx.x) / (int)gridDim.x >= TRACE_TILE0 &&
                       (pr - (int)blockIdx.x) / (int)gridDim.x < TRACE_TILE0 + TRACE_TILES;
      tcur.ev(trc, 16, 0, 0);                                    // 16: pair of tiles starts
      int j0 = 0, j1 = 0;
      int slot_id[2] = {0, 0};
      bool valid[2] = {false, false};
      double pos[2][3], az[2], pol[2], best[2] = {0.0, 0.0};
      int bobj[2] = {0, 0};
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        int base, nv;
        pp_rows(F, op, pr, sl, j0, j1, base, nv);
        valid[sl] = r < nv;
        slot_id[sl] = valid[sl] ? n_slot[sl] : 0;
        pos[sl][0] = n_pos[sl][0]; pos[sl][1] = n_pos[sl][1]; pos[sl][2] = n_pos[sl][2];
        az[sl] = n_az[sl];
        pol[sl] = n_pol[sl];
      }
      for (int j = j0; j < j1; ++j) {
        const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
        const NetDev& net = F.net[j];
        const int head_off = __ldg(&P->head_off);
        const int k0 = P->k0, halfk = k0 >> 1;
        double u[2][5];
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          for (int e = 0; e < 5; ++e) u[sl][e] = 0.0;
          if constexpr (!Op::kRaw) {
            if (valid[sl]) row_u_bf16(F, j, pos[sl], az[sl], pol[sl], u[sl]);
          }
          const uint32_t a_slot = a_base0 + (uint32_t)(sl * a_bytes);
          if constexpr (!Op::kRaw) {
            encode_row(k0, sub, net.encoding == ENC_PE6, valid[sl], u[sl], a_slot, r);
          } else {
            for (int c = sub * halfk; c < (sub + 1) * halfk; c += 8) {
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = valid[sl] ? (float)op.raw(slot_id[sl], c + e) : 0.f;
              st_shared_v4(a_slot + a_off(r, c), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                           pack_bf16(v[6], v[7]));
            }
          }
          fence_async_smem();
          tc_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR_A_READY(sl));
          tcur.ev(trc, 20, sl, 0);                               // 20: the slot's encoding stored
        }
        if (j == j0) fetch(pr + (int)gridDim.x);

        const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
        float head_part[2] = {0.f, 0.f};
        for (int s = 0; s < ns; ++s) {
          const Step st = load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
          const int epi = st.epi;
          // the head weights of this warp's columns (read in place by the HEAD / MASKG epilogue) into
          // L1 while the step's MMAs run: a first touch costs an L2 round trip per 32-column chunk
          if (epi == E_HEAD || epi == E_MASKG_A) {
            const int nm = (st.rows - sub * 32 + 63) >> 6;
            if (lane < 8 * nm) {
              const float* hp = P->params + head_off + sub * 32 + 64 * (lane >> 3) + 4 * (lane & 7);
              asm volatile("prefetch.global.L1 [%0];" ::"l"(hp));
            }
          }
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            tcur.ev(trc, 17, s * 2 + sl, 0);                     // 17: wait for the accumulator begins
            mbar_wait(BAR_ACC(sl), acc_ph[sl] & 1u);
            tcur.ev(trc, 18, s * 2 + sl, 0);                     // 18: accumulator ready
            ++acc_ph[sl];
            tc_after_sync();
            const uint32_t tmem_row = tmem + lane_addr + (uint32_t)(sl * 256);
            uint32_t* my_masks = mask_scratch + ((size_t)blockIdx.x * 2 + sl) * MASK_WORDS_PER_CTA;
            if (epi == E_BWD_OUT) {
              if (sub == 0) {
                float g[128];
                for (int c = 0; c < st.rows; c += 16) {
                  uint32_t rg[16];
                  DDF_TMEM_LD16(tmem_row + (uint32_t)c, rg);
                  tmem_wait_ld();
#pragma unroll
                  for (int e = 0; e < 16; ++e) g[c + e] = __uint_as_float(rg[e]);
                }
                if constexpr (Op::kGrad) {
                  if (valid[sl]) {
                    if constexpr (Op::kRaw) {
                      op.store_grad_raw(slot_id[sl], [&](int k) { return (double)g[k]; });
                    } else {
                      double g5[5];
                      pe_chain_tc(net.encoding == ENC_PE6, u[sl], [&](int k) { return g[k]; }, g5);
                      op.store_grad(slot_id[sl], g5);
                    }
                  }
                }
              }
              tc_before_sync();
              continue;
            }
            const uint32_t a_row = a_base0 + (uint32_t)(sl * a_bytes) + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
            const int nm = (st.rows - sub * 32 + 63) >> 6;
            const float* sp = P->params;   // global: only the head weights are read (bias folded)
            switch (epi) {
              case E_RELU_A: epi_direct_n<E_RELU_A>(nm, st, sub * 32, r, tmem_row, a_row, my_masks, sp + head_off, head_part[sl], sp); break;
              case E_RELU_MASK_A: epi_direct_n<E_RELU_MASK_A>(nm, st, sub * 32, r, tmem_row, a_row, my_masks, sp + head_off, head_part[sl], sp); break;
              case E_MASKG_A: epi_direct_n<E_MASKG_A>(nm, st, sub * 32, r, tmem_row, a_row, my_masks, sp + head_off, head_part[sl], sp); break;
              case E_BWD_MASK_A: epi_direct_n<E_BWD_MASK_A>(nm, st, sub * 32, r, tmem_row, a_row, my_masks, sp + head_off, head_part[sl], sp); break;
              default: epi_direct_n<E_HEAD>(nm, st, sub * 32, r, tmem_row, a_row, my_masks, sp + head_off, head_part[sl], sp); break;
            }
            tc_before_sync();
            if (writes_a(epi)) {
              fence_async_smem();
              __syncwarp();
              if (lane == 0) mbar_arrive(BAR_A_READY(sl));
            } else if (epi == E_HEAD) {
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
            tcur.ev(trc, 19, s * 2 + sl, 0);                     // 19: epilogue done
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
// ================================================================== quad
// Networks whose hidden layers are at most 128 wide (config 1, the UDF scan)
// run four 128-row tiles ("slots") per CTA, TMEM columns [128 sl, 128 sl + 128).
// A layer of one slot is only 8 N=128 MMAs (~700 cycles), shorter than one
// epilogue, so two slots in flight leave the tensor pipe waiting.  Here each
// group of four row warps owns two slots (group g: slots g and g + 2) and runs
// whole rows (all columns; the head dot stays in registers, no cross-warp
// reduction), so the two groups' epilogues overlap each other and the MMAs
// of the other slots.  Weight chunks are streamed once per layer and shared by
// the four slots (chunk-major MMA order); params are staged only when the
// network changes.
constexpr int QS = 4;                                    // most slots per CTA (mask scratch sizing)

// Epilogue in 16-column pieces with the next piece's TMEM load in flight while
// this one is processed: one warp's NM 32-column chunks, STRIDE columns apart
// from c_first.  The per-piece chain (TMEM load -> bias, ReLU, pack -> shared
// stores) is latency-bound (~700 cycles per 32 columns when run back to back,
// ~80 instructions issued), and kernels with 16 row warps have 96 registers
// per thread, so the pipeline holds 2 x 16 accumulator registers instead of
// 1 x 32.  WAIT_FREE: the A columns may be overwritten only once the MMAs that
// read them have completed (bar_free, the > 256-wide engines' a_free); the
// wait sits before the first store, after the first piece's arithmetic.
struct NoMid {
  __device__ __forceinline__ void operator()() const {}
};
// mid(): called once the first 32-column chunk is stored (NM == 2 only), for
// engines that release the A columns of a part in two steps.
template <int EPI, int NM, int STRIDE, bool WAIT_FREE, class Mid = NoMid>
__device__ __forceinline__ void epi_cols16(const Step& st, int c_first, int r, uint32_t tmem_row, uint32_t a_row,
                                           uint32_t* my_masks, const float* head_w, float& head_part,
                                           const float* sparams, uint32_t bar_free, uint32_t& free_ph,
                                           Mid mid = Mid()) {
  constexpr bool WA = EPI != E_HEAD;
  constexpr bool HEAD_DOT = EPI == E_HEAD || EPI == E_MASKG_HEAD_A;
  const int r7 = r & 7;
  (void)sparams;
  const uint32_t head_s = smem_u32(head_w);
  uint32_t rg[2][16];
  uint32_t mw = 0u, mq = 0u;
  if constexpr (NM > 0) {
    DDF_TMEM_LD16(tmem_row + (uint32_t)c_first, rg[0]);
    tmem_wait_ld();
  }
#pragma unroll
  for (int i = 0; i < 2 * NM; ++i) {
    const int c = c_first + (i >> 1) * STRIDE + (i & 1) * 16;
    if (i + 1 < 2 * NM)
      DDF_TMEM_LD16(tmem_row + (uint32_t)(c_first + ((i + 1) >> 1) * STRIDE + ((i + 1) & 1) * 16), rg[(i + 1) & 1]);
    const uint32_t(&x)[16] = rg[i & 1];
    // no bias here: it is already in the accumulator (step_has_bias)
    if constexpr (EPI == E_BWD_MASK_A) {
      if ((i & 1) == 0) mq = my_masks[(st.mask_layer * 16 + (c >> 5)) * ROWS + r];
    }
    uint32_t pkd[8];
    if constexpr (EPI == E_BWD_MASK_A) {
      const uint32_t m = mq >> (16 * (i & 1));
#pragma unroll
      for (int e = 0; e < 8; ++e)
        pkd[e] = pack_bf16(((m >> (2 * e)) & 1u) ? __uint_as_float(x[2 * e]) : 0.f,
                           ((m >> (2 * e + 1)) & 1u) ? __uint_as_float(x[2 * e + 1]) : 0.f);
    } else if constexpr (EPI == E_RELU_A) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        pkd[e] = pack_bf16_relu(__uint_as_float(x[2 * e]), __uint_as_float(x[2 * e + 1]));
    } else if constexpr (EPI == E_HEAD) {
#pragma unroll
      for (int e = 0; e < 16; e += 4) {
        const float4 hw = ld_shared_f4(head_s + 4u * (uint32_t)(c + e));
        head_part = fmaf(fmaxf(__uint_as_float(x[e]), 0.f), hw.x, head_part);
        head_part = fmaf(fmaxf(__uint_as_float(x[e + 1]), 0.f), hw.y, head_part);
        head_part = fmaf(fmaxf(__uint_as_float(x[e + 2]), 0.f), hw.z, head_part);
        head_part = fmaf(fmaxf(__uint_as_float(x[e + 3]), 0.f), hw.w, head_part);
      }
    } else {
      // ReLU mask bits (neural.py:241 "h > 0"), one u32 per 32 columns
      uint32_t mh = 0u;
      float v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float z = __uint_as_float(x[e]);
        mh |= (z > 0.f ? 1u : 0u) << e;
        v[e] = z;
      }
      mw |= mh << (16 * (i & 1));
      if constexpr (EPI == E_RELU_MASK_A) {
        if (i & 1) { my_masks[(st.mask_layer * 16 + (c >> 5)) * ROWS + r] = mw; mw = 0u; }
#pragma unroll
        for (int e = 0; e < 8; ++e) pkd[e] = pack_bf16_relu(v[2 * e], v[2 * e + 1]);
      } else {   // E_MASKG_A / E_MASKG_HEAD_A: d/dh of the last hidden layer = w_head * mask
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          const float4 hw = ld_shared_f4(head_s + 4u * (uint32_t)(c + e));
          if constexpr (HEAD_DOT) {
            // the identity head of the forward, in E_HEAD's order (same fp32 result)
            head_part = fmaf(fmaxf(v[e], 0.f), hw.x, head_part);
            head_part = fmaf(fmaxf(v[e + 1], 0.f), hw.y, head_part);
            head_part = fmaf(fmaxf(v[e + 2], 0.f), hw.z, head_part);
            head_part = fmaf(fmaxf(v[e + 3], 0.f), hw.w, head_part);
          }
          v[e] = ((mh >> e) & 1u) ? hw.x : 0.f;
          v[e + 1] = ((mh >> (e + 1)) & 1u) ? hw.y : 0.f;
          v[e + 2] = ((mh >> (e + 2)) & 1u) ? hw.z : 0.f;
          v[e + 3] = ((mh >> (e + 3)) & 1u) ? hw.w : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) pkd[e] = pack_bf16(v[2 * e], v[2 * e + 1]);
      }
    }
    if constexpr (WA) {
      if constexpr (WAIT_FREE) {
        if (i == 0) {
          mbar_wait(bar_free, free_ph & 1u);
          ++free_ph;
        }
      }
      const uint32_t blk = a_row + (uint32_t)((c >> 6) * (ROWS * 128));
      const int cc0 = (c & 63) >> 3;
      st_shared_v4(blk + (uint32_t)(((cc0) ^ r7) << 4), pkd[0], pkd[1], pkd[2], pkd[3]);
      st_shared_v4(blk + (uint32_t)(((cc0 + 1) ^ r7) << 4), pkd[4], pkd[5], pkd[6], pkd[7]);
      if constexpr (NM == 2) {
        if (i == 1) mid();
      }
    }
    if (i + 1 < 2 * NM) tmem_wait_ld();
  }
  if constexpr (WA && WAIT_FREE && NM == 0) ++free_ph;   // no columns in this part: keep the phase count in step
}

// the quad engine's whole-row epilogue: NCH 16-column pieces from column 0
template <int EPI, int NCH>
__device__ __forceinline__ void epi_rows16(const Step& st, int r, uint32_t tmem_row, uint32_t a_row, uint32_t* my_masks,
                                           const float* head_w, float& head_part, const float* sparams) {
  uint32_t unused = 0u;
  epi_cols16<EPI, NCH / 2, 32, false>(st, 0, r, tmem_row, a_row, my_masks, head_w, head_part, sparams, 0u, unused);
}

template <int EPI>
__device__ __forceinline__ void epi_rows_n(int nm, const Step& st, int r, uint32_t tmem_row, uint32_t a_row,
                                           uint32_t* my_masks, const float* head_w, float& head_part,
                                           const float* sp) {
  switch (nm) {   // nm: 32-column groups of the layer (64 / 128 wide)
    case 2: epi_rows16<EPI, 4>(st, r, tmem_row, a_row, my_masks, head_w, head_part, sp); break;
    case 4: epi_rows16<EPI, 8>(st, r, tmem_row, a_row, my_masks, head_w, head_part, sp); break;
    default: break;
  }
}

__device__ __forceinline__ void encode_row_full(int k0, bool pe, bool valid, const double u[5], uint32_t a_tile,
                                                int r) {
  if (k0 == 16) store_encoding<0, 16>(false, valid, u, a_tile, r);
  else store_encoding<0, 80>(pe, valid, u, a_tile, r);
}

template <class Op, int NSL>
__global__ void __launch_bounds__((EPI_WARP0 + 4 * NSL) * 32, 1)
mlp_quad_kernel(const FieldDev F, const Op op, uint32_t* __restrict__ mask_scratch, int n_stages, int a_bytes,
                int stage_bytes, int params_bytes, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base_ptr = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* a_tiles = base_ptr;                                   // [NSL][a_bytes]
  uint8_t* stages = base_ptr + NSL * (size_t)a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)n_stages * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NSL + 2 * n_stages);
  float* sparams = reinterpret_cast<float*>(tmem_slot + 4);      // one copy: [params_bytes/4]
  // the bias fold's constant A block, aligned to its 256-byte swizzle atom
  uint8_t* ones = reinterpret_cast<uint8_t*>(((uintptr_t)(sparams + (params_bytes >> 2)) + 255) & ~(uintptr_t)255);

  const int warp = uni((int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;   // warp index, provably warp-uniform
  const uint32_t bar0 = smem_u32(bars);
  auto BAR_A_READY = [&](int sl) { return bar0 + 8u * sl; };
  auto BAR_ACC = [&](int sl) { return bar0 + 8u * (NSL + sl); };
  auto BAR_FULL = [&](int s) { return bar0 + 8u * (2 * NSL + s); };
  auto BAR_EMPTY = [&](int s) { return bar0 + 8u * (2 * NSL + n_stages + s); };

  if (threadIdx.x == 0) {
    for (int sl = 0; sl < NSL; ++sl) {
      mbar_init(BAR_A_READY(sl), N_EPI_WARPS / 2);
      mbar_init(BAR_ACC(sl), 1);
    }
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(BAR_FULL(s), 1);
      mbar_init(BAR_EMPTY(s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  write_ones_block(ones, threadIdx.x, blockDim.x);
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base0 = smem_u32(a_tiles);
  const uint32_t st_base = smem_u32(stages);
  const int packs = pp_pairs<Op, NSL>(F, op);
  unsigned long long dbg_acc[16];
  if (kStats)
    for (int i = 0; i < 16; ++i) dbg_acc[i] = 0ull;

  if (warp == 0) {
    // ================================================= weight producer: each chunk once per layer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int pk = blockIdx.x; pk < packs; pk += gridDim.x) {
        int j0, j1, base, nv;
        pp_rows<Op, NSL>(F, op, pk, 0, j0, j1, base, nv);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
          const uint8_t* img = Op::kGrad ? P->img_grad : P->img_fwd;
          for (int s = 0; s < ns; ++s) {
            const Step st = load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            const int nck = st.nchunk + (step_has_bias(st.epi) ? 1 : 0);   // + the bias chunk (rows x 32 B)
            for (int c = 0; c < nck; ++c) {
              const uint8_t* src = img + st.img_off + (size_t)c * st.chunk_bytes;
              const uint32_t bytes = c < st.nchunk ? (uint32_t)st.chunk_bytes : (uint32_t)(st.rows * 32);
              DDF_DBG_T0();
              mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
              DDF_DBG_ADD(6);
              mbar_expect_tx(BAR_FULL(stage), bytes);
              bulk_g2s(st_base + (uint32_t)(stage * stage_bytes), src, bytes, BAR_FULL(stage));
              if (++stage == n_stages) { stage = 0; phase ^= 1u; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer: slot-major within a layer.
    // Layer s of slot 0 (all its K chunks), then of slot 1, ...: slot 0's
    // accumulator is committed after its own 8 MMAs, so its epilogue runs
    // under the MMAs of slots 1-3 and its next layer can follow slot 3's
    // directly.  (Chunk-major order committed all four accumulators at the
    // end of the layer: MMA phase, then epilogue phase, nothing overlapped.)
    // The layer's weight chunks stay in the ring until slot NSL-1 has read
    // them (nchunk <= 2 stages; the ring has >= 4).  The whole warp runs this
    // loop converged; one elected lane issues (see mma_k64_commit_w).
    {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t ar = 0u;                              // A_READY phase: every slot completes one per step
      const long long t_all = kStats ? clock64() : 0;
      const uint32_t tmem_u = uni(tmem);
      const uint32_t a0_lo = uni(sdesc_lo(a_base0)), db0_lo = uni(sdesc_lo(st_base));
      const uint32_t a_step = uni((uint32_t)a_bytes >> 4), sstep = uni((uint32_t)stage_bytes >> 4);
      const uint32_t bars_u = uni(bar0);
      const int nst = uni(n_stages), packs_u = uni(packs);
      const uint32_t ones_lo = uni(sdesc_lo(smem_u32(ones)));
      TraceCursor tcur{1, 0};
      for (int pk = blockIdx.x; pk < packs_u; pk += gridDim.x) {
        int j0, j1, base, nv;
        pp_rows<Op, NSL>(F, op, pk, 0, j0, j1, base, nv);
        j0 = uni(j0);
        j1 = uni(j1);
        const bool trc = kTrace && blockIdx.x == 0 && lane == 0 && (pk - (int)blockIdx.x) / (int)gridDim.x >= TRACE_TILE0 &&
                         (pk - (int)blockIdx.x) / (int)gridDim.x < TRACE_TILE0 + TRACE_TILES;
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = uni(__ldg(Op::kGrad ? &P->n_grad : &P->n_fwd));
          for (int s = 0; s < ns; ++s) {
            Step st = load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
            uni_step(st);
            const uint32_t id = idesc(st.rows);
            const int nfull = st.K >> 6;                 // chunks of four K = 16 MMAs
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl) {
              {
                // this slot's A tile is written and its TMEM columns are read out
                DDF_DBG_T0();
                tcur.ev(trc, 1, s * NSL + sl, 0);            // 1: wait for the slot's A tile begins
                mbar_wait_u(bars_u + 8u * sl, ar & 1u);
                tcur.ev(trc, 2, s * NSL + sl, 0);            // 2: A tile ready
                if (lane == 0) DDF_DBG_ADD(0);
              }
              tc_after_sync();
              const uint32_t da_lo = a0_lo + (uint32_t)sl * a_step;
              const uint32_t td = tmem_u + (uint32_t)(sl * (512 / NSL));
              int stg = stage;
              uint32_t ph = phase;
              for (int kc = 0; kc < st.nchunk; ++kc) {
                if (sl == 0) {
                  DDF_DBG_T0();
                  mbar_wait_u(bars_u + 8u * (uint32_t)(2 * NSL + stg), ph);
                  if (lane == 0) DDF_DBG_ADD(1);
                  tc_after_sync();
                }
                const uint32_t da = da_lo + (uint32_t)(kc * (ROWS * 128 / 16));
                const uint32_t db = db0_lo + (uint32_t)stg * sstep;
                if (kc < nfull) {
                  mma_k64_w(td, da, db, id, kc ? 1u : 0u);
                } else {
                  const int nks = (st.K - kc * 64 + 15) >> 4;
                  for (int ks = 0; ks < nks; ++ks)
                    mma_bf16_w(td, ((uint64_t)SDESC_HI << 32) | (da + 2 * ks), ((uint64_t)SDESC_HI << 32) | (db + 2 * ks), id,
                               (kc | ks) ? 1u : 0u);
                }
                if (++stg == nst) { stg = 0; ph ^= 1u; }
              }
              if (step_has_bias(st.epi)) {   // D += bias: the chunk after the K chunks, shared by the slots
                if (sl == 0) {
                  mbar_wait_u(bars_u + 8u * (uint32_t)(2 * NSL + stg), ph);
                  tc_after_sync();
                }
                mma_bias_w(td, ones_lo, db0_lo + (uint32_t)stg * sstep, id);
              }
              tc_commit_w(bars_u + 8u * (uint32_t)(NSL + sl));
              tcur.ev(trc, 7, s * NSL + sl, 0);              // 7: the slot's layer issued
            }
            ++ar;
            const int nck = st.nchunk + (step_has_bias(st.epi) ? 1 : 0);
            for (int kc = 0; kc < nck; ++kc) {           // every slot has read the layer's chunks
              tc_commit_w(bars_u + 8u * (uint32_t)(2 * NSL + nst + stage));
              if (++stage == nst) { stage = 0; phase ^= 1u; }
            }
          }
        }
      }
      if (kStats && lane == 0) dbg_acc[4] += (unsigned long long)(clock64() - t_all);
    }
  } else {
    // ================================================= row warps: group g (four warps, one per TMEM
    // lane quarter) owns slot g, so the four slots' epilogues run concurrently
    const int q = warp & 3;
    const int sl = (warp - EPI_WARP0) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t tmem_row = tmem + lane_addr + (uint32_t)(sl * (512 / NSL));
    const uint32_t a_slot = a_base0 + (uint32_t)(sl * a_bytes);
    const uint32_t a_row = a_slot + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
    uint32_t* my_masks = mask_scratch + ((size_t)blockIdx.x * NSL + sl) * MASK_WORDS_PER_CTA;
    uint32_t acc_ph = 0u;
    int staged = -1;
    const bool w0 = kStats && threadIdx.x == EPI_WARP0 * 32;
    const long long t_rows = kStats ? clock64() : 0;
    TraceCursor tcur{q == 0 && sl == 0 ? 2 : 3, 0};
    // this row of the slot's next tile: list entry and path state (with its
    // f64 direction -> angle trigonometry) fetched one pack ahead, issued
    // once the current pack's encoding is stored, so the loads and the trig
    // run while the row warp would otherwise wait for layer accumulators
    int n_slot = 0;
    double n_pos[3] = {0.0, 0.0, 0.0}, n_az = 0.0, n_pol = 0.0;
    auto fetch = [&](int pp) {
      if (pp < packs) {
        int a0, a1, b0, c0;
        pp_rows<Op, NSL>(F, op, pp, sl, a0, a1, b0, c0);
        if (r < c0) {
          n_slot = op.slot(b0 + r);
          if constexpr (!Op::kRaw) op.load(n_slot, n_pos, n_az, n_pol);
        }
      }
    };
    fetch(blockIdx.x);
    for (int pk = blockIdx.x; pk < packs; pk += gridDim.x) {
      long long t_ph = kStats ? clock64() : 0;
      int j0, j1, base, nv;
      pp_rows<Op, NSL>(F, op, pk, sl, j0, j1, base, nv);
      const bool trc = kTrace && blockIdx.x == 0 && lane == 0 && q == 0 && (sl == 0 || sl == NSL - 1) &&
                       (pk - (int)blockIdx.x) / (int)gridDim.x >= TRACE_TILE0 &&
                       (pk - (int)blockIdx.x) / (int)gridDim.x < TRACE_TILE0 + TRACE_TILES;
      tcur.ev(trc, 16, sl, 0);                                   // 16: pack start
      const bool valid = r < nv;
      const int slot_id = valid ? n_slot : 0;
      double pos[3] = {n_pos[0], n_pos[1], n_pos[2]}, az = n_az, pol = n_pol, best = 0.0;
      int bobj = 0;
      if (w0) { dbg_acc[3] += (unsigned long long)(clock64() - t_ph); t_ph = clock64(); }
      for (int j = j0; j < j1; ++j) {
        const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
        const NetDev& net = F.net[j];
        const int head_off = __ldg(&P->head_off);
        const int k0 = P->k0;
        if (j != staged) {
          // every row warp is past its last read of the previous network's params
          const int nf = __ldg(&P->params_floats);
          const float4* src = reinterpret_cast<const float4*>(P->params);
          float4* dst = reinterpret_cast<float4*>(sparams);
          named_sync(1, (4 * NSL) * 32);
          for (int i = threadIdx.x - EPI_WARP0 * 32; i < (nf >> 2); i += (4 * NSL) * 32) dst[i] = __ldg(src + i);
          named_sync(1, (4 * NSL) * 32);
          staged = j;
          if (w0) { dbg_acc[8] += (unsigned long long)(clock64() - t_ph); t_ph = clock64(); }
        }
        double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if constexpr (!Op::kRaw) {
          if (valid) row_u(F, j, pos, az, pol, u);
          encode_row_full(k0, net.encoding == ENC_PE6, valid, u, a_slot, r);
        } else {
          for (int c = 0; c < k0; c += 8) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = valid ? (float)op.raw(slot_id, c + e) : 0.f;
            st_shared_v4(a_slot + a_off(r, c), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                         pack_bf16(v[6], v[7]));
          }
        }
        fence_async_smem();
        tc_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR_A_READY(sl));
        tcur.ev(trc, 20, sl, 0);                                 // 20: encoding stored
        if (j == j0) fetch(pk + (int)gridDim.x);
        if (w0) { dbg_acc[5] += (unsigned long long)(clock64() - t_ph); t_ph = clock64(); }

        const int ns = __ldg(Op::kGrad ? &P->n_grad : &P->n_fwd);
        float head_part = 0.f;
        for (int s = 0; s < ns; ++s) {
          const Step st = load_step(Op::kGrad ? &P->grad[s] : &P->fwd[s]);
          const int epi = st.epi;
          tcur.ev(trc, 17, s * NSL + sl, 0);                     // 17: wait for the accumulator begins
          mbar_wait(BAR_ACC(sl), acc_ph & 1u);
          tcur.ev(trc, 18, s * NSL + sl, 0);                     // 18: accumulator ready
          if (w0) { dbg_acc[2] += (unsigned long long)(clock64() - t_ph); t_ph = clock64(); }
          ++acc_ph;
          tc_after_sync();
          if (epi == E_BWD_OUT) {
            float gr[128];
            for (int c = 0; c < st.rows; c += 16) {
              uint32_t rg[16];
              DDF_TMEM_LD16(tmem_row + (uint32_t)c, rg);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 16; ++e) gr[c + e] = __uint_as_float(rg[e]);
            }
            if constexpr (Op::kGrad) {
              if (valid) {
                if constexpr (Op::kRaw) {
                  op.store_grad_raw(slot_id, [&](int kk) { return (double)gr[kk]; });
                } else {
                  double g5[5];
                  pe_chain_tc(net.encoding == ENC_PE6, u, [&](int kk) { return gr[kk]; }, g5);
                  op.store_grad(slot_id, g5);
                }
              }
            }
            tc_before_sync();
            continue;
          }
          const int nm = (dbg & 1024) ? 0 : st.rows >> 5;   // dbg 1024: timing only, no epilogue arithmetic
          switch (epi) {
            case E_RELU_A: epi_rows_n<E_RELU_A>(nm, st, r, tmem_row, a_row, my_masks, sparams + head_off, head_part, sparams); break;
            case E_RELU_MASK_A: epi_rows_n<E_RELU_MASK_A>(nm, st, r, tmem_row, a_row, my_masks, sparams + head_off, head_part, sparams); break;
            case E_MASKG_A: epi_rows_n<E_MASKG_A>(nm, st, r, tmem_row, a_row, my_masks, sparams + head_off, head_part, sparams); break;
            case E_BWD_MASK_A: epi_rows_n<E_BWD_MASK_A>(nm, st, r, tmem_row, a_row, my_masks, sparams + head_off, head_part, sparams); break;
            default: epi_rows_n<E_HEAD>(nm, st, r, tmem_row, a_row, my_masks, sparams + head_off, head_part, sparams); break;
          }
          tc_before_sync();
          if (writes_a(epi)) {
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR_A_READY(sl));
          } else if (epi == E_HEAD) {
            double pv = (double)(head_part + P->head_b);
            if (F.composite) pv = dmul(net.scale, pv);
            if (j == j0 || pv < best) { best = pv; bobj = j; }
          }
          tcur.ev(trc, 19, s * NSL + sl, 0);                     // 19: epilogue done
          if (w0) { dbg_acc[7] += (unsigned long long)(clock64() - t_ph); t_ph = clock64(); }
        }
      }
      if constexpr (!Op::kGrad) {
        if (valid) op.store_fwd(slot_id, best, bobj);
      }
      if (w0) dbg_acc[10] += (unsigned long long)(clock64() - t_ph);
    }
    if (w0) dbg_acc[9] += (unsigned long long)(clock64() - t_rows);
  }
  if (kStats && lane == 0 && (warp == 0 || warp == 1 || warp == EPI_WARP0)) DDF_DBG_FLUSH();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// TMA descriptors of one network's weight image (forward + gradient
// programs back to back), viewed as rows of 128 bytes: boxes of 128 rows
// (16 KB, a stage) and of 8 rows (the N = 80 backward output step).
struct Tmaps {
  CUtensorMap box128, box8;        // the image as rows of 128 bytes: boxes of 128 and of 8 rows
  CUtensorMap b32_128, b32_8;      // the image as rows of 32 bytes (bias chunks): boxes of 128 and of 8 rows
};

struct NetImage {
  void* dev = nullptr;       // Prog (device)
  void* img = nullptr;       // fwd + grad images
  void* params = nullptr;    // biases + head weights (fp32)
  int in_width = 0;
  Prog host{};
  Tmaps tmaps{};             // over img (networks wider than 256: the CTA-pair engine, mlp_2sm.cuh)
};

// Tensor maps over a network's weight image (rows of 128 bytes), built once
// per image on the host through the driver entry point (no libcuda link).
inline int make_weight_tmaps(const void* img, size_t bytes, Tmaps* out, std::string* err) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      *err = "cuTensorMapEncodeTiled unavailable";
      return 4;
    }
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint32_t estr[2] = {1, 1};
  for (int v = 0; v < 2; ++v) {         // v = 0: rows of 128 bytes, v = 1: rows of 32 bytes
    const cuuint64_t row_u64 = v == 0 ? 16 : 4;
    const cuuint64_t dims[2] = {row_u64, (cuuint64_t)(bytes / (row_u64 * 8))};
    const cuuint64_t strides[1] = {row_u64 * 8};
    for (int b = 0; b < 2; ++b) {
      const cuuint32_t box[2] = {(cuuint32_t)row_u64, b == 0 ? 128u : 8u};
      CUtensorMap* tm = v == 0 ? (b == 0 ? &out->box128 : &out->box8) : (b == 0 ? &out->b32_128 : &out->b32_8);
      CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(img), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { *err = "cuTensorMapEncodeTiled failed"; return 4; }
    }
  }
  return 0;
}



inline int pad_to(int x, int m) { return (x + m - 1) / m * m; }

inline void append_bias_rows(std::vector<uint16_t>& img, int rows, const float* bias);

// Append the chunks of one step: B[n][k] = src(n, k), n < N (rows), k < K.
// half_bias (wide programs, nh = 2, bias folded): the bias chunk of each
// N-half goes ahead of that half's K chunks.
// ck = 64: chunks of 64 K columns, rows of 128 B in the 128-byte swizzle.
// ck = 32 (ping-pong programs): chunks of 32 K columns, rows of 64 B in the
// 64-byte swizzle (16-byte unit u of row n at u ^ ((n >> 1) & 3)): half the
// stage size, so the weight ring holds five stages beside the two A tiles
// instead of two.
template <class Src>
inline void append_chunks(std::vector<uint16_t>& img, Step& st, Src src, const float* half_bias = nullptr,
                          int ck = 64) {
  st.img_off = (long long)img.size() * 2;
  for (int h = 0; h < st.nh; ++h) {
    if (half_bias) append_bias_rows(img, st.rows, half_bias + h * st.rows);
    for (int kc = 0; kc < st.nchunk; ++kc) {
      const size_t base = img.size();
      img.resize(base + (size_t)st.rows * ck, 0);
      for (int n = 0; n < st.rows; ++n)
        for (int k = 0; k < ck; ++k) {
          const int gn = h * st.rows + n, gk = kc * ck + k;
          const float v = (gk < st.K) ? src(gn, gk) : 0.f;
          __nv_bfloat16 b = __float2bfloat16_rn(v);
          const size_t off = ck == 64
              ? (size_t)(n >> 3) * 512 + (size_t)(n & 7) * 64 + (size_t)((((k >> 3) ^ (n & 7)) << 3) + (k & 7))
              : (size_t)n * 32 + (size_t)((((k >> 3) ^ ((n >> 1) & 3)) << 3) + (k & 7));
          std::memcpy(&img[base + off], &b, 2);
        }
    }
  }
}

// The bias chunk of a folded step (see step_has_bias): rows x 16 bf16 (one
// K = 16 step, 32 B per row, 32-byte swizzle: 16-byte half h of row n at
// h ^ ((n >> 2) & 1)), columns 0..2 of row n = the three bf16 pieces of
// bias[n].  It follows the step's K chunks in the image.
inline int bias_chunk_bytes(int rows) { return rows * 32; }
inline void append_bias_chunk(std::vector<uint16_t>& img, const Step& st, const std::vector<float>& bias) {
  append_bias_rows(img, st.rows, bias.data());
}
inline void append_bias_rows(std::vector<uint16_t>& img, int rows, const float* bias) {
  const size_t base = img.size();
  img.resize(base + (size_t)rows * 16, 0);
  for (int n = 0; n < rows; ++n) {
    float rem = bias[n];
    for (int k = 0; k < 3; ++k) {
      const __nv_bfloat16 b = __float2bfloat16_rn(rem);
      rem -= __bfloat162float(b);
      const size_t off = (size_t)n * 16 + (size_t)((((k >> 3) ^ ((n >> 2) & 1)) << 3) + (k & 7));
      std::memcpy(&img[base + off], &b, 2);
    }
  }
}

inline Step make_step(int K, int N, int nh, int epi, int ck = 64) {
  Step s{};
  s.K = K; s.N = N; s.nh = nh; s.epi = epi;
  s.rows = N / nh;
  s.nchunk = (K + ck - 1) / ck;
  s.chunk_bytes = s.rows * ck * 2;
  s.mask_layer = -1;
  s.bias = nullptr;
  return s;
}

// Build forward and gradient programs + UMMA images for one network.
// weights: concat of W_l (out, in) row-major float64; biases: concat of b_l.
inline int build_image(const int32_t* widths, int32_t n_widths, const double* weights, const double* biases,
                       NetImage* out, std::string* err) {
  const int L = n_widths - 1;
  out->in_width = widths[0];
  if (L < 2) { *err = "bf16 engine needs at least one hidden layer"; return 1; }
  std::vector<int> wp(n_widths);
  wp[0] = pad_to(widths[0], 16);
  for (int l = 1; l < L; ++l) wp[l] = pad_to(widths[l], 64);
  wp[L] = 1;
  for (int l = 1; l < L; ++l)
    if (wp[l] > 512) { *err = "bf16 engine supports hidden widths up to 512"; return 1; }
  if (wp[0] > 128) { *err = "bf16 engine supports input widths up to 128"; return 1; }
  // host copies of effective weights, padded
  std::vector<std::vector<float>> W(L), B(L);
  size_t wo = 0, bo = 0;
  for (int l = 0; l < L; ++l) {
    const int in = widths[l], o = widths[l + 1];
    W[l].assign((size_t)wp[l + 1] * wp[l], 0.f);
    B[l].assign(wp[l + 1], 0.f);
    for (int a = 0; a < o; ++a) {
      for (int k = 0; k < in; ++k) W[l][(size_t)a * wp[l] + k] = (float)weights[wo + (size_t)a * in + k];
      B[l][a] = (float)biases[bo + a];
    }
    wo += (size_t)o * in;
    bo += o;
  }
  int maxh = 0;
  for (int l = 1; l < L; ++l) maxh = std::max(maxh, wp[l]);
  const int split = maxh <= 256 ? 1 : 2;   // <= 256: full-N MMAs, two tiles in flight (ping-pong kernel)
  Prog& P = out->host;
  std::memset(&P, 0, sizeof(P));
  P.pp = split == 1;
  // Ping-pong programs at 256 wide: 32-column chunks.  With 64-column (32 KB) chunks only two stages fit
  // beside the two 64 KB A tiles and the weight stream is latency-starved; 16 KB stages give five
  // (5->8x256 forward 1300 -> 1401 TF/s).  At 192 wide five 24 KB stages fit already and the extra
  // barrier round per two MMAs costs more than it hides (788 -> 659 TF/s), so those keep 64.
  const int ck = (split == 1 && maxh > 192) ? 32 : 64;
  P.chunk_k = ck;
  P.fold = 1;   // every bf16 program: quad / ping-pong (chunk after the K chunks) and wide (per N-half, ahead)   // quad programs (chunk after the K chunks) and wide ones (per N-half, ahead)
  P.max_hidden = maxh;
  P.k0 = wp[0];
  P.in_width = widths[0];
  P.encoding = widths[0] == 65 ? ENC_PE6 : ENC_RAW5;
  P.head_b = B[L - 1][0];
  // fp32 params: biases of hidden layers then head weights
  std::vector<float> params;   // every vector starts at a multiple of 4 floats (wp[] are multiples of 16)
  std::vector<size_t> bias_off(L);
  for (int l = 0; l < L - 1; ++l) { bias_off[l] = params.size(); params.insert(params.end(), B[l].begin(), B[l].end()); }
  const size_t head_off = params.size();
  params.insert(params.end(), W[L - 1].begin(), W[L - 1].begin() + wp[L - 1]);
  while (params.size() % 4) params.push_back(0.f);

  std::vector<uint16_t> img;
  // forward program: hidden layers 0..L-2, the last one fused with the head
  P.n_fwd = L - 1;
  for (int l = 0; l < L - 1; ++l) {
    Step s = make_step(wp[l], wp[l + 1], split, l == L - 2 ? E_HEAD : E_RELU_A, ck);
    const std::vector<float>& w = W[l];
    const int K = wp[l];
    append_chunks(img, s, [&](int n, int k) { return w[(size_t)n * K + k]; }, P.fold && split == 2 ? B[l].data() : nullptr, ck);
    if (P.fold && split == 1) append_bias_chunk(img, s, B[l]);
    s.bias = reinterpret_cast<const float*>(bias_off[l]);   // patched to device below
    P.fwd[l] = s;
  }
  const size_t fwd_bytes = img.size() * 2;
  std::vector<uint16_t> gimg;
  int gs = 0;
  for (int l = 0; l < L - 1; ++l) {
    Step s = make_step(wp[l], wp[l + 1], split, l == L - 2 ? E_MASKG_A : E_RELU_MASK_A, ck);
    s.mask_layer = l;
    const std::vector<float>& w = W[l];
    const int K = wp[l];
    append_chunks(gimg, s, [&](int n, int k) { return w[(size_t)n * K + k]; }, P.fold && split == 2 ? B[l].data() : nullptr, ck);
    if (P.fold && split == 1) append_bias_chunk(gimg, s, B[l]);
    s.bias = reinterpret_cast<const float*>(bias_off[l]);
    P.grad[gs++] = s;
  }
  // backward: layer l maps d z_l (width wp[l+1]) to d h_l (width wp[l]) with B[n][k] = W_l[k][n]
  for (int l = L - 2; l >= 0; --l) {
    const bool last = l == 0;
    Step s = make_step(wp[l + 1], wp[l], last ? 1 : split, last ? E_BWD_OUT : E_BWD_MASK_A, ck);
    s.mask_layer = l - 1;
    const std::vector<float>& w = W[l];
    const int Kin = wp[l];
    append_chunks(gimg, s, [&](int n, int k) { return w[(size_t)k * Kin + n]; }, nullptr, ck);
    P.grad[gs++] = s;
  }
  P.n_grad = gs;
  if (gs > 2 * DDF_MAX_LAYERS) { *err = "too many layers"; return 1; }
  P.kmax = 0;
  P.max_chunk_bytes = 0;
  for (int i = 0; i < P.n_fwd; ++i) { P.kmax = std::max(P.kmax, std::max(P.fwd[i].K, P.fwd[i].N)); P.max_chunk_bytes = std::max(P.max_chunk_bytes, P.fwd[i].chunk_bytes); }
  for (int i = 0; i < P.n_grad; ++i) { P.kmax = std::max(P.kmax, std::max(P.grad[i].K, P.grad[i].N)); P.max_chunk_bytes = std::max(P.max_chunk_bytes, P.grad[i].chunk_bytes); }
  // upload
  const size_t total = fwd_bytes + gimg.size() * 2;
  if (cudaMalloc(&out->img, total) != cudaSuccess) { *err = "cudaMalloc (weight image) failed"; return 4; }
  cudaMemcpy(out->img, img.data(), fwd_bytes, cudaMemcpyHostToDevice);
  cudaMemcpy((uint8_t*)out->img + fwd_bytes, gimg.data(), gimg.size() * 2, cudaMemcpyHostToDevice);
  if (cudaMalloc(&out->params, params.size() * 4) != cudaSuccess) { *err = "cudaMalloc (params) failed"; return 4; }
  cudaMemcpy(out->params, params.data(), params.size() * 4, cudaMemcpyHostToDevice);
  const float* pdev = reinterpret_cast<const float*>(out->params);
  // steps carry the float offset of their bias inside the params block
  // (staged in shared memory by the kernel)
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
  P.img_grad = reinterpret_cast<const uint8_t*>(out->img) + fwd_bytes;
  if (!P.pp)
    if (int rc = make_weight_tmaps(out->img, total, &out->tmaps, err)) return rc;
  if (cudaMalloc(&out->dev, sizeof(Prog)) != cudaSuccess) { *err = "cudaMalloc (program) failed"; return 4; }
  if (cudaMemcpy(out->dev, &P, sizeof(Prog), cudaMemcpyHostToDevice) != cudaSuccess) { *err = "upload failed"; return 4; }
  return 0;
}

inline void free_image(NetImage* im) {
  if (im->dev) cudaFree(im->dev);
  if (im->img) cudaFree(im->img);
  if (im->params) cudaFree(im->params);
  im->dev = im->img = im->params = nullptr;
}

constexpr int SMEM_LIMIT = 232448;   // 227 KB opt-in per CTA

template <class Op>
int launch_pp(const FieldDev& F, const std::vector<NetImage>& images, const Op& op, int max_rows, int sm_count,
              uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  int kmax = 0, chunk = 0, params_bytes = 0;
  for (int j = 0; j < F.n_obj; ++j) {
    kmax = std::max(kmax, images[j].host.kmax);
    chunk = std::max(chunk, images[j].host.max_chunk_bytes);
    params_bytes = std::max(params_bytes, images[j].host.params_floats * 4);
  }
  const int a_bytes = ROWS * pad_to(kmax, 64) * 2;
  const int extra = 1024 + 8 * (4 + 2 * 8) + 16 + 4 * ROWS * 4 + ONES_BYTES + 256;
  int n_stages = std::min(8, (SMEM_LIMIT - 2 * a_bytes - extra) / chunk);
  if (n_stages < 2) { *err = "bf16 ping-pong engine: not enough shared memory"; return 1; }
  const size_t smem = 2 * (size_t)a_bytes + (size_t)n_stages * chunk + extra;
  auto kern = mlp_pp_kernel<Op>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
  const int pairs_max = ((max_rows + ROWS - 1) / ROWS + 1) / 2 + (Op::kGrad ? F.n_obj : 0);
  const int grid = std::max(1, std::min(pairs_max, sm_count));
  kern<<<grid, NTHREADS, smem, st>>>(F, op, mask_scratch, n_stages, a_bytes, chunk, params_bytes);
  e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("mlp_pp_kernel launch: ") + cudaGetErrorString(e); return 4; }
  return 0;
}

template <class Op, int NSL>
int launch_quad(const FieldDev& F, const std::vector<NetImage>& images, const Op& op, int max_rows, int sm_count,
                uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  int kmax = 0, chunk = 0, params_bytes = 0;
  for (int j = 0; j < F.n_obj; ++j) {
    kmax = std::max(kmax, images[j].host.kmax);
    chunk = std::max(chunk, images[j].host.max_chunk_bytes);
    params_bytes = std::max(params_bytes, images[j].host.params_floats * 4);
  }
  const int a_bytes = ROWS * pad_to(kmax, 64) * 2;
  const int extra = 1024 + 8 * (2 * NSL + 2 * 8) + 16 + params_bytes + ONES_BYTES + 256;
  int n_stages = std::min(8, (SMEM_LIMIT - NSL * a_bytes - extra) / chunk);
  // a layer's chunks (at most two K chunks and the bias chunk) stay in the ring until the last slot has read them
  if (n_stages < 4) { *err = "bf16 quad engine: not enough shared memory"; return 1; }
  const size_t smem = NSL * (size_t)a_bytes + (size_t)n_stages * chunk + extra;
  auto kern = mlp_quad_kernel<Op, NSL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
  const int packs_max = ((max_rows + ROWS - 1) / ROWS + NSL - 1) / NSL + (Op::kGrad ? F.n_obj : 0);
  const int grid = std::max(1, std::min(packs_max, sm_count));
  const int dbg = debug_bits();
  kern<<<grid, (EPI_WARP0 + 4 * NSL) * 32, smem, st>>>(F, op, mask_scratch, n_stages, a_bytes, chunk, params_bytes, dbg);
  e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("mlp_quad_kernel launch: ") + cudaGetErrorString(e); return 4; }
  return 0;
}

template <class Op>
int launch(const FieldDev& F, const std::vector<NetImage>& images, const Op& op, int max_rows, int sm_count,
           uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  int maxh = 0;
  bool all_pp = true;
  for (int j = 0; j < F.n_obj; ++j) {
    all_pp = all_pp && images[j].host.pp;
    maxh = std::max(maxh, images[j].host.max_hidden);
  }
  // <= 128 wide: four slots, one row-warp group per slot.  129..256 wide: the
  // ping-pong engine below (a two-slot group-per-slot variant measured slower:
  // 880 vs 1065 TF/s forward on 5->8x256, c5 60.1 M vs 69.6 M path samples/s).
  // Quad programs carry folded bias chunks (step_has_bias), which only the
  // quad kernel consumes.
  if constexpr (Op::kFused) {
    // fused trace+gradient exists for the > 256-wide single-tile engine only
    if (all_pp || F.n_obj != 1) { *err = "fused trace+gradient needs one network wider than 256"; return 1; }
  } else {
  if (all_pp && maxh <= 128)
    return launch_quad<Op, 4>(F, images, op, max_rows, sm_count, mask_scratch, st, err);
  bool pp = true, any_pp = false;
  for (int j = 0; j < F.n_obj; ++j) {
    pp = pp && images[j].host.pp;
    any_pp = any_pp || images[j].host.pp;
  }
  if (any_pp && !pp) { *err = "bf16 engine: networks of one field must all be <= 256 or all > 256 wide"; return 1; }
  if (pp) return launch_pp<Op>(F, images, op, max_rows, sm_count, mask_scratch, st, err);
  }
  int kmax = 0, chunk = 0, params_bytes = 0;
  for (int j = 0; j < F.n_obj; ++j) {
    kmax = std::max(kmax, images[j].host.kmax);
    chunk = std::max(chunk, images[j].host.max_chunk_bytes);
    params_bytes = std::max(params_bytes, images[j].host.params_floats * 4);
  }
  const int a_bytes = ROWS * pad_to(kmax, 64) * 2;
  const int extra = 1024 /*align*/ + 8 * (6 + 2 * 8) + 16 + 2 * ROWS * 4 + params_bytes + ONES_BYTES + 256;
  int n_stages = (SMEM_LIMIT - a_bytes - extra) / chunk;
  n_stages = std::min(n_stages, 8);
  if (n_stages < 2) { *err = "bf16 engine: not enough shared memory for the weight pipeline"; return 1; }
  const int dbg = debug_bits();
  if (dbg & 8) n_stages = 8;
  if (dbg & 256) n_stages = std::min(n_stages, 2);
  const size_t smem = (size_t)a_bytes + (size_t)((dbg & 8) ? 1 : n_stages) * chunk + extra;
  auto kern = mlp_kernel<Op>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
  const int tiles_max = (max_rows + ROWS - 1) / ROWS + (Op::kGrad ? F.n_obj : 0);
  const int grid = std::max(1, std::min(tiles_max, sm_count));
  kern<<<grid, NTHREADS, smem, st>>>(F, op, mask_scratch, n_stages, a_bytes, chunk, params_bytes, dbg);
  e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("mlp_kernel launch: ") + cudaGetErrorString(e); return 4; }
  return 0;
}

}  // namespace umma
}  // namespace ddf
