// Raw tcgen05.mma throughput: one CTA per SM issues NMMA back-to-back MMAs
// (M=128, N=var, K=16, bf16 SS) into TMEM, commit every 4, optional wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d; }
__global__ void k(int nmma, int n, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot; __shared__ __align__(8) uint64_t bar; __shared__ __align__(8) uint64_t bar2;
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar2))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t a = smem_u32(base), b = smem_u32(base + 131072);
  if ((mode & 16) && threadIdx.x >= 64) {   // 8 warps storing 16-byte vectors into a separate region
    const uint32_t w = smem_u32(base + 163840) + (threadIdx.x - 64) * 16;
    for (int it = 0; it < nmma * 2; ++it)
      asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" :: "r"(w + (uint32_t)((it & 7) * 4096)), "r"(it) : "memory");
  }
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < nmma; ++i) {
      const uint32_t kc = (mode & 8) ? (uint32_t)((i >> 2) & 1) * 16384u : 0u;
      const uint32_t sl = (mode & 8) ? (uint32_t)((i >> 3) & 3) * 32768u : 0u;
      uint64_t ad = sdesc(a + sl + kc + (i & 3) * 32), bd = sdesc(b + kc + (i & 3) * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                   :: "r"(tmem + (uint32_t)((mode & 2) ? ((i >> 2) & 1) * n : 0)), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i & 3)));
      if ((i & 3) == 3 && (mode & 4)) {   // a pre-completed barrier wait per chunk
        asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(smem_u32(&bar2)), "r"(1u) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if ((i & 3) == 3 && (mode & 1)) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
    // wait for the last phase: count commits
    int ncommit = ((mode & 1) ? nmma / 4 : 0) + 1;
    uint32_t par = (ncommit - 1) & 1;
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(smem_u32(&bar)), "r"(par) : "memory");
    long long t1 = clock64();
    atomicAdd(out, (unsigned long long)(t1 - t0));
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int ns[] = {64, 128, 256};
  for (int mode : {1, 9, 17, 25}) for (int n : ns) {
    int nmma = 4096;
    cudaMemset(d, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 320, 220 * 1024>>>(nmma, n, mode, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    double per = (double)cyc / 148 / nmma;
    double tf = 2.0 * 128 * n * 16 * nmma * 148 / (ms * 1e-3) / 1e12;
    printf("mode %d (commit/4=%d, alt-tmem=%d) N=%3d: %.1f cycles/MMA (ideal %d), %.0f TF/s by events (%s)\n", mode, mode & 1, (mode >> 1) & 1, n, per, 128 * n / 256, tf, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
