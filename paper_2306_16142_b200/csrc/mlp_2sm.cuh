// bf16 DDF-MLP engine for hidden layers wider than 256 on a CTA pair
// (tcgen05.mma.cta_group::2): configs 3 and 4.
//
// Why a pair.  The single-CTA engine (mlp_umma.cuh mlp_kernel) streams every
// weight chunk from L2 once per 128-row tile: 32 KB per 512 MMA cycles per SM,
// ~9.5 KB/cycle for the chip, above the ~6.3 KB/cycle the L2 -> SM path
// delivers, and only three 32-KB stages fit beside the 128 KB A tile, too few
// to hide the copy latency.  Measured on that engine: weights switched off
// (timing experiment) lifted the 512-wide forward from 1251 to 1487 TF/s.
//
// Here two CTAs on the two SMs of a TPC run one M = 256 MMA: each CTA keeps
// its own 128-row A tile and TMEM accumulator (rows 128 r .. 128 r + 127 of
// the pair's 256-row tile) and holds HALF of every weight chunk (N/2 rows of
// B).  Per SM the weight stream halves, each stage is 16 KB, so six stages
// fit, and each weight byte feeds 256 rows.
//
//   warp 0      weight producer (both CTAs): its half of each chunk by TMA
//               (cp.async.bulk.tensor.2d.cta_group::2) into its own stage
//               buffer, completion signalled on the LEADER's FULL barrier
//   warp 1      leader CTA: the MMA issuer (whole warp, elected lane);
//               commits multicast to both CTAs (EMPTY, ACC, A_FREE)
//   warps 2-9   row warps (both CTAs): encoding and epilogues exactly as in
//               mlp_kernel, on their own TMEM and A tile; A_READY arrivals go
//               to the leader's barrier (remote arrive, cluster release)
//
// Tiles go to pairs: pair p takes tiles 2 tp + r for tp = p, p + npairs, ...;
// the second CTA of the last pair may see an empty tile (no valid rows) and
// still runs the program so both CTAs stay in step.
#pragma once
#include "mlp_umma.cuh"

namespace ddf {
namespace umma {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the leader CTA's copy of a barrier at the same offset (cluster address)
__device__ __forceinline__ uint32_t leader_addr(uint32_t bar) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(bar));
  return r;
}
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(bar)) : "memory");
}
// wait with cluster-scope acquire: the peer's A-tile writes, released by its
// arrive, are visible before the MMAs read them
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "vote.sync.all.pred q, p, 0xffffffff;\n\t"
      "@!q bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// one box of the weight image -> this CTA's stage buffer, transaction bytes
// counted on the leader's FULL barrier (the peer bit of the address cleared)
__device__ __forceinline__ void tma_box_pair(uint32_t dst, const CUtensorMap* tm, int row, uint32_t full_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(row), "r"(full_bar & 0xFEFFFFFFu)
      : "memory");
}
// kind::f16 instruction descriptor for the pair: M = 256
__device__ __forceinline__ uint32_t idesc2(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
__device__ __forceinline__ void mma2_k64_commit_w(uint32_t tmem_d, uint32_t da, uint32_t db, uint32_t id,
                                                  uint32_t acc, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
      ".reg .b64 a0, a1, a2, a3, b0, b1, b2, b3;\n\t.reg .b16 m;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %3, %3;\n\t"
      "mov.b16 m, 3;\n\t"
      "add.u32 x1, %1, 2;\n\tadd.u32 x2, %1, 4;\n\tadd.u32 x3, %1, 6;\n\t"
      "add.u32 y1, %2, 2;\n\tadd.u32 y2, %2, 4;\n\tadd.u32 y3, %2, 6;\n\t"
      "mov.b64 a0, {%1, %6};\n\tmov.b64 a1, {x1, %6};\n\tmov.b64 a2, {x2, %6};\n\tmov.b64 a3, {x3, %6};\n\t"
      "mov.b64 b0, {%2, %6};\n\tmov.b64 b1, {y1, %6};\n\tmov.b64 b2, {y2, %6};\n\tmov.b64 b3, {y3, %6};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], m;\n\t}"
      ::"r"(tmem_d), "r"(da), "r"(db), "r"(id), "r"(acc), "r"(bar), "n"(SDESC_HI)
      : "memory");
}
__device__ __forceinline__ void mma2_bf16_w(uint32_t tmem_d, uint32_t da, uint32_t db, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 a, {%1, %5};\n\tmov.b64 b, {%2, %5};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(da), "r"(db), "r"(id), "r"(acc), "n"(SDESC_HI));
}
// the bias fold's MMA for the pair (see mlp_umma.cuh step_has_bias): A = each CTA's ones block,
// B = each CTA's half of the bias chunk, both one K = 16 step in the 32-byte swizzle
__device__ __forceinline__ void mma2_bias_w(uint32_t tmem_d, uint32_t ones_lo, uint32_t db_lo, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred q, e;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 q, %4, 0;\n\t"
      "mov.b64 a, {%1, %5};\n\tmov.b64 b, {%2, %5};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, q;\n\t}" ::"r"(tmem_d),
      "r"(ones_lo), "r"(db_lo), "r"(id), "r"(acc), "n"(SDESC32B_HI)
      : "memory");
}
// MMA completion -> the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void tc_commit2_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar)
      : "memory");
}

// tile_rows for tile indices past the last tile (the idle half of the last
// pair): no valid rows, the first network
template <class Op>
__device__ __forceinline__ void tile_rows2(const FieldDev& F, const Op& op, int t, int tiles, int& j0, int& j1,
                                           int& base, int& nv) {
  if (t < tiles) {
    tile_rows(F, op, t, j0, j1, base, nv);
  } else {
    j0 = 0; j1 = 1; base = 0; nv = 0;
  }
}

template <class Op>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
mlp2_kernel(const FieldDev F, const Op op, uint32_t* __restrict__ mask_scratch, int n_stages, int a_bytes,
            int stage_bytes, int params_bytes, const __grid_constant__ Tmaps tm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr bool kProgG = Op::kGrad || Op::kFused;
  uint8_t* base_ptr = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Smem S;
  S.a = base_ptr;
  S.stages = base_ptr + a_bytes;
  S.bars = reinterpret_cast<uint64_t*>(S.stages + (size_t)n_stages * stage_bytes);
  S.tmem_slot = reinterpret_cast<uint32_t*>(S.bars + 6 + 2 * n_stages);
  S.red = reinterpret_cast<float*>(S.tmem_slot + 4);
  S.params = S.red + 2 * ROWS;
  // the bias fold's constant A block, aligned to its 256-byte swizzle atom
  uint8_t* ones = reinterpret_cast<uint8_t*>(((uintptr_t)(S.params + (params_bytes >> 2)) + 255) & ~(uintptr_t)255);

  const int warp = uni((int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;   // warp index, provably warp-uniform
  const uint32_t rank = cluster_ctarank();
  const int pair = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);
  const uint32_t bar0 = smem_u32(S.bars);
  auto BAR_A_READY = [&](int h) { return bar0 + 8u * (0 + h); };
  auto BAR_ACC = [&](int h) { return bar0 + 8u * (2 + h); };
  auto BAR_A_FREE = [&](int h) { return bar0 + 8u * (4 + h); };
  auto BAR_FULL = [&](int s) { return bar0 + 8u * (6 + s); };
  auto BAR_EMPTY = [&](int s) { return bar0 + 8u * (6 + n_stages + s); };

  if (threadIdx.x == 0) {
    for (int h = 0; h < 2; ++h) {
      mbar_init(BAR_A_READY(h), 2 * N_EPI_WARPS);   // the leader's counts both CTAs' row warps
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
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(S.tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  write_ones_block(ones, threadIdx.x, blockDim.x);
  fence_async_smem();
  tc_before_sync();
  cluster_sync_all();   // both CTAs' barriers initialised before any remote arrive or multicast commit
  tc_after_sync();
  const uint32_t tmem = *S.tmem_slot;
  const uint32_t a_base = smem_u32(S.a);
  const uint32_t st_base = smem_u32(S.stages);
  const int tiles = n_tiles(F, op);
  const int pairs_total = (tiles + 1) >> 1;
  unsigned long long dbg_acc[16];
  if (kStats)
    for (int i = 0; i < 16; ++i) dbg_acc[i] = 0ull;

  if (warp == 0) {
    // ================================================= weight producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tp = pair; tp < pairs_total; tp += npairs) {
        int j0, j1, base, nv;
        tile_rows2(F, op, 2 * tp + (int)rank, tiles, j0, j1, base, nv);
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = __ldg(kProgG ? &P->n_grad : &P->n_fwd);
          const int img_row0 = kProgG ? (int)((P->img_grad - P->img_fwd) >> 7) : 0;
          for (int s = 0; s < ns; ++s) {
            const Step st = load_step(kProgG ? &P->grad[s] : &P->fwd[s]);
            const int half_rows = st.rows >> 1;
            const bool fold = step_has_bias(st.epi);   // a bias chunk (rows x 32 B) ahead of each N-half
            // this CTA's half of every chunk: rows [rank * half, (rank + 1) * half)
            int base_row = img_row0 + (int)(st.img_off >> 7);   // in rows of 128 bytes
            for (int h = 0; h < st.nh; ++h) {
              if (fold) {
                mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
                const uint32_t dst = st_base + (uint32_t)(stage * stage_bytes);
                if (rank == 0) mbar_expect_tx(BAR_FULL(stage), (uint32_t)(st.rows * 32));   // both halves
                const int row32 = 4 * base_row + (int)rank * half_rows;                      // in rows of 32 bytes
                int r0 = 0;
                for (; r0 + 128 <= half_rows; r0 += 128) tma_box_pair(dst + (uint32_t)(r0 * 32), &tm.b32_128, row32 + r0, BAR_FULL(stage));
                for (; r0 < half_rows; r0 += 8) tma_box_pair(dst + (uint32_t)(r0 * 32), &tm.b32_8, row32 + r0, BAR_FULL(stage));
                base_row += st.rows >> 2;
                if (++stage == n_stages) { stage = 0; phase ^= 1u; }
              }
              for (int c = 0; c < st.nchunk; ++c) {
                mbar_wait(BAR_EMPTY(stage), phase ^ 1u);
                const uint32_t dst = st_base + (uint32_t)(stage * stage_bytes);
                if (rank == 0) mbar_expect_tx(BAR_FULL(stage), (uint32_t)st.chunk_bytes);   // both halves
                const int row = base_row + (int)rank * half_rows;
                int r0 = 0;
                for (; r0 + 128 <= half_rows; r0 += 128) tma_box_pair(dst + (uint32_t)(r0 * 128), &tm.box128, row + r0, BAR_FULL(stage));
                for (; r0 < half_rows; r0 += 8) tma_box_pair(dst + (uint32_t)(r0 * 128), &tm.box8, row + r0, BAR_FULL(stage));
                base_row += st.rows;
                if (++stage == n_stages) { stage = 0; phase ^= 1u; }
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer (leader CTA, whole warp)
    // The whole warp runs this loop converged on warp-uniform values (uni,
    // mbar_wait_u: mlp_umma.cuh), so the tcgen05 instructions are issued from
    // uniform registers without per-operand ELECT / R2UR waterfalls.
    if (rank == 0) {
      TraceCursor tcur{1, 0};
      int stage = 0;
      uint32_t phase = 0;
      uint32_t ar[2] = {0u, 0u};
      const uint32_t tmem_u = uni(tmem), bars_u = uni(bar0);
      const uint32_t da0_lo = uni(sdesc_lo(a_base)), db0_lo = uni(sdesc_lo(st_base));
      const uint32_t sstep = uni((uint32_t)stage_bytes >> 4);
      const uint32_t ones_lo = uni(sdesc_lo(smem_u32(ones)));
      const int nst = uni(n_stages), pairs_u = uni(pairs_total);
      auto UB_A_READY = [&](int h) { return bars_u + 8u * (0 + h); };
      auto UB_ACC = [&](int h) { return bars_u + 8u * (2 + h); };
      auto UB_A_FREE = [&](int h) { return bars_u + 8u * (4 + h); };
      auto UB_FULL = [&](int st_) { return bars_u + 8u * (uint32_t)(6 + st_); };
      auto UB_EMPTY = [&](int st_) { return bars_u + 8u * (uint32_t)(6 + nst + st_); };
      for (int tp = pair; tp < pairs_u; tp += npairs) {
        int j0, j1, base, nv;
        tile_rows2(F, op, 2 * tp, tiles, j0, j1, base, nv);
        j0 = uni(j0);
        j1 = uni(j1);
        const bool trc = kTrace && pair == 0 && lane == 0 && (tp - pair) / npairs >= TRACE_TILE0 &&
                         (tp - pair) / npairs < TRACE_TILE0 + TRACE_TILES;
        for (int j = j0; j < j1; ++j) {
          const Prog* P = reinterpret_cast<const Prog*>(F.net[j].wimg_fwd);
          const int ns = uni(kProgG ? P->n_grad : P->n_fwd);
          int prev_rows = 1 << 30;
          for (int s = 0; s < ns; ++s) {
            Step st = load_step(kProgG ? &P->grad[s] : &P->fwd[s]);
            uni_step(st);
            const uint32_t id = idesc2(st.rows);
            const bool wa = writes_a(st.epi);
            const bool fold = step_has_bias(st.epi);
            const int kc1 = min(st.nchunk, (st.K >> 1) >> 6);
            const int c0 = min(st.nchunk - 1, ((st.N >> 1) - 1) >> 6);
            const int nfull = st.K >> 6;
            bool waited0 = false, waited1 = false;
            auto wait_a = [&](int which) {
              tcur.ev(trc, which ? 3 : 1, s, 0);
              mbar_wait_cluster(UB_A_READY(which), ar[which] & 1u);
              ++ar[which];
              tcur.ev(trc, which ? 4 : 2, s, 0);
            };
            if (st.rows > prev_rows) { wait_a(0); wait_a(1); waited0 = waited1 = true; }
            prev_rows = st.rows;
            for (int h = 0; h < st.nh; ++h) {
              const uint32_t td = tmem_u + (uint32_t)(h * st.rows);
              const bool last_half = h == st.nh - 1;
              int kc = 0;
              while (kc < st.nchunk) {
                if (kc == 0 && !waited0) { wait_a(0); waited0 = true; }
                if (kc >= kc1 && !waited1) { wait_a(1); waited1 = true; }
                if (kc == 0 && fold) {
                  // the half's accumulator starts as its bias (ones block x bias chunk), the K chunks add to it
                  mbar_wait_u(UB_FULL(stage), phase);
                  tc_after_sync();
                  mma2_bias_w(td, ones_lo, db0_lo + (uint32_t)stage * sstep, id, 0u);
                  tc_commit2_w(UB_EMPTY(stage));
                  if (++stage == nst) { stage = 0; phase ^= 1u; }
                }
                int kend = st.nchunk;
                if (!waited1 && kc1 > kc) kend = min(kend, kc1);
                if (wa && last_half && c0 >= kc) kend = min(kend, c0 + 1);
                const int kfull = min(kend, nfull);
                if (kc == 0) tcur.ev(trc, 6, s, h);
                for (; kc < kfull; ++kc) {
                  mbar_wait_u(UB_FULL(stage), phase);
                  tc_after_sync();
                  mma2_k64_commit_w(td, da0_lo + (uint32_t)(kc * (ROWS * 128 / 16)), db0_lo + (uint32_t)stage * sstep,
                                    id, (kc || fold) ? 1u : 0u, UB_EMPTY(stage));
                  tcur.ev(trc, 8, s, h);
                  if (++stage == nst) { stage = 0; phase ^= 1u; }
                }
                if (kc < kend) {   // the partial last chunk (the input layer's K = 80)
                  mbar_wait_u(UB_FULL(stage), phase);
                  tc_after_sync();
                  const int nks = (st.K - kc * 64 + 15) >> 4;
                  const uint32_t da = da0_lo + (uint32_t)(kc * (ROWS * 128 / 16));
                  const uint32_t db = db0_lo + (uint32_t)stage * sstep;
                  for (int ks = 0; ks < nks; ++ks) mma2_bf16_w(td, da + 2 * ks, db + 2 * ks, id, (kc | ks || fold) ? 1u : 0u);
                  tc_commit2_w(UB_EMPTY(stage));
                  if (++stage == nst) { stage = 0; phase ^= 1u; }
                  ++kc;
                }
                if (wa && last_half) {
                  if (kc == c0 + 1) tc_commit2_w(UB_A_FREE(0));
                  if (kc == st.nchunk) tc_commit2_w(UB_A_FREE(1));
                }
              }
              tc_commit2_w(UB_ACC(h));
              tcur.ev(trc, 7, s, h);
            }
            if (!waited1) wait_a(1);   // keep phases in step
          }
        }
      }
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
        tile_rows2(F, op, tt, tiles, a0, a1, b0, c0);
        if (r < c0) {
          n_slot = op.slot(b0 + r);
          if constexpr (!Op::kRaw) op.load(n_slot, n_pos, n_az, n_pol);
        }
      }
    };
    fetch(2 * pair + (int)rank);
    for (int tp = pair; tp < pairs_total; tp += npairs) {
      const int t = 2 * tp + (int)rank;
      int j0, j1, base, nv;
      tile_rows2(F, op, t, tiles, j0, j1, base, nv);
      const bool valid = r < nv;
      const int slot = valid ? n_slot : 0;
      const bool trc = kTrace && pair == 0 && rank == 0 && lane == 0 && (warp == EPI_WARP0 || warp == EPI_WARP0 + 7) &&
                       (tp - pair) / npairs >= TRACE_TILE0 && (tp - pair) / npairs < TRACE_TILE0 + TRACE_TILES;
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
        if (lane == 0) { mbar_arrive_leader(BAR_A_READY(0)); mbar_arrive_leader(BAR_A_READY(1)); }
        tcur.ev(trc, 20, 0, 0);                        // 20: encoding stored
        if (j == j0) fetch(t + 2 * npairs);

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
              if (lane == 0) mbar_arrive_leader(BAR_A_READY(h));
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
  __syncwarp();
  tc_before_sync();
  cluster_sync_all();   // no CTA leaves while its pair still reads its shared memory or TMEM
  tc_after_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// The pair engine takes one network wider than 256 (the single-tile engine's
// domain) on an even grid of CTA pairs.
template <class Op>
int launch_2sm(const FieldDev& F, const NetImage& im, const Op& op, int max_rows, int sm_count,
               uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  const int a_bytes = ROWS * pad_to(im.host.kmax, 64) * 2;
  const int params_bytes = im.host.params_floats * 4;
  const int stage_bytes = 16384;
  const int extra = 1024 /*align*/ + 8 * (6 + 2 * 8) + 16 + 2 * ROWS * 4 + params_bytes + ONES_BYTES + 256;
  const int n_stages = std::min(8, (SMEM_LIMIT - a_bytes - extra) / stage_bytes);
  if (n_stages < 2) { *err = "bf16 pair engine: not enough shared memory for the weight pipeline"; return 1; }
  const size_t smem = (size_t)a_bytes + (size_t)n_stages * stage_bytes + extra;
  auto kern = mlp2_kernel<Op>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
  const int tiles_max = (max_rows + ROWS - 1) / ROWS + (Op::kGrad ? F.n_obj : 0);
  const int npairs = std::max(1, std::min((tiles_max + 1) / 2, sm_count / 2));
  kern<<<2 * npairs, NTHREADS, smem, st>>>(F, op, mask_scratch, n_stages, a_bytes, stage_bytes, params_bytes, im.tmaps);
  e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("mlp2_kernel launch: ") + cudaGetErrorString(e); return 4; }
  return 0;
}

}  // namespace umma
}  // namespace ddf
