// What slows the engines' MMA issue below the tensor-pipe rate?  The 512-wide
// engine's issue pattern rebuilt step by step on an otherwise empty SM:
//   mode 0: issuer alone, S = 3 chunks ahead of completion (mma_lag.cu)
//   bit 1: a producer thread between completion and the next chunk (waits
//          EMPTY(stage), arrives FULL(stage); the issuer waits FULL)
//   bit 2: 8 row warps: per 8-chunk half they wait ACC(h) (committed after the
//          half) and arrive A_READY(h); the issuer waits A_READY(0) before a
//          layer's first chunk and A_READY(1) before its fifth
// Cycles per MMA (N = 256, M = 128, K = 16; floor 128).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d; }
__device__ __forceinline__ void mma4(uint32_t td, uint64_t da, uint64_t db, uint32_t id, uint32_t acc, uint32_t bar) {
  asm volatile("{\n\t.reg .pred p, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, %3, %3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n\t"
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}"
      :: "r"(td), "l"(da), "l"(db), "r"(id), "r"(acc), "r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory"); }
constexpr int S = 3;
__global__ void k(int layers, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t full[S], empty[S], accb[2], aready[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[i])));
                                  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&empty[i]))); }
    for (int i = 0; i < 2; ++i) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&accb[i])));
                                  asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" :: "r"(smem_u32(&aready[i]))); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (mode & 4) {   // operands filled with random bf16 in [-1, 1) (the engines' data) instead of leftover bytes
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
    for (int i = threadIdx.x; i < 224 * 1024 / 4; i += blockDim.x) {
      x ^= x << 13; x ^= x >> 17; x ^= x << 5;
      const uint32_t lo = 0x3F80u | (x & 0x807Fu), hi = 0x3F00u | ((x >> 16) & 0x807Fu);   // +-[0.5, 2)
      reinterpret_cast<uint32_t*>(base)[i] = lo | (hi << 16);
    }
  } else if (mode & 8) {
    for (int i = threadIdx.x; i < 224 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0u;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int nchunk = layers * 16;
  if (warp == 0 && lane == 0 && (mode & 1)) {          // producer
    uint32_t ph = 0; int st = 0;
    for (int c = 0; c < nchunk; ++c) {
      wait(smem_u32(&empty[st]), ph ^ 1u);
      arrive(smem_u32(&full[st]));
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {                 // issuer
    const uint64_t da0 = sdesc(smem_u32(base)), db0 = sdesc(smem_u32(base + 131072));
    uint32_t ph = 0, ar[2] = {0, 0}; int st = 0;
    uint32_t eph[S] = {0, 0, 0};
    long long t0 = clock64();
    for (int l = 0; l < layers; ++l) {
      for (int h = 0; h < 2; ++h) {
        for (int kc = 0; kc < 8; ++kc) {
          const int c = (l * 2 + h) * 8 + kc;
          if ((mode & 2) && h == 0 && kc == 0 && l > 0) { wait(smem_u32(&aready[0]), ar[0] & 1u); ++ar[0]; }
          if ((mode & 2) && h == 0 && kc == 4 && l > 0) { wait(smem_u32(&aready[1]), ar[1] & 1u); ++ar[1]; }
          if (mode & 1) { wait(smem_u32(&full[st]), ph); }
          else if (c >= S) { wait(smem_u32(&empty[st]), eph[st] & 1u); ++eph[st]; }
          asm volatile("tcgen05.fence::after_thread_sync;");
          mma4(tmem + (uint32_t)(h * 256), da0 + (uint64_t)(kc * 1024), db0 + (uint64_t)(st * 2048), id,
               kc ? 1u : 0u, smem_u32(&empty[st]));
          if (++st == S) { st = 0; ph ^= 1u; }
        }
        commit(smem_u32(&accb[h]));
      }
    }
    wait(smem_u32(&accb[1]), (uint32_t)((layers - 1) & 1));
    long long t1 = clock64();
    atomicAdd(out, (unsigned long long)(t1 - t0));
  } else if (warp >= 2 && (mode & 2)) {                 // row warps
    for (int l = 0; l < layers; ++l)
      for (int h = 0; h < 2; ++h) {
        wait(smem_u32(&accb[h]), (uint32_t)(l & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        __syncwarp();
        if (lane == 0 && l + 1 < layers) arrive(smem_u32(&aready[h]));
      }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  const int runs[][2] = {{0, 256}, {8, 256}, {4, 256}, {7, 256}, {8, 16384}, {4, 16384}, {7, 16384}};
  for (const auto& r : runs) {
    const int mode = r[0], layers = r[1];
    cudaMemset(d, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 320, 225 * 1024>>>(layers, mode, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)cyc / 148 / ((double)layers * 64);
    printf("mode %d (producer %d, row warps %d, data %s), %6d layers, %8.2f ms: %.1f cycles/MMA, %.0f TF/s, SM clock %.0f MHz %s\n",
           mode, mode & 1, (mode >> 1) & 1, (mode & 4) ? "random" : (mode & 8) ? "zeros" : "leftover", layers, ms, per, 2.0 * 128 * 256 * 16 * 64.0 * layers * 148 / (ms * 1e-3) / 1e12,
           (double)cyc / 148 / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
