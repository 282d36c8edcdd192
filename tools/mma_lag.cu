// tcgen05.mma throughput when the issuer may run only S chunks (of 4 K=16
// MMAs, N=256) ahead of completion: chunk k is issued after the commit of
// chunk k-S has arrived, as a weight ring of S stages allows.  Prints cycles
// per MMA for S = 1..8 (the engines' 512-wide ring has S = 3).
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
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(bar), "r"(par) : "memory");
}
__global__ void k(int nchunk, int S, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot; __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 32) {
    const uint64_t da0 = sdesc(smem_u32(base)), db0 = sdesc(smem_u32(base + 131072));
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = clock64();
    for (int c = 0; c < nchunk; ++c) {
      const int s = c % S;
      if (c >= S) { wait(smem_u32(&bar[s]), ph[s] & 1u); ++ph[s]; asm volatile("tcgen05.fence::after_thread_sync;"); }
      const uint32_t td = tmem + (uint32_t)(((c >> 3) & 1) * 256);
      mma4(td, da0 + (uint64_t)((c & 7) * 1024), db0 + (uint64_t)((c % 3) * 2048), id, (c & 7) ? 1u : 0u, smem_u32(&bar[s]));
    }
    for (int c = nchunk - S; c < nchunk; ++c) { const int s = c % S; wait(smem_u32(&bar[s]), ph[s] & 1u); ++ph[s]; }
    long long t1 = clock64();
    atomicAdd(out, (unsigned long long)(t1 - t0));
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  for (int S = 1; S <= 8; ++S) {
    const int nchunk = 4096;
    cudaMemset(d, 0, 8);
    k<<<148, 64, 225 * 1024>>>(nchunk, S, d);
    cudaDeviceSynchronize();
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("S=%d chunks in flight: %.1f cycles/MMA (N=256 floor 128) %s\n", S, (double)cyc / 148 / (nchunk * 4),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
