#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d; }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(bar), "r"(par) : "memory"); }
__global__ void k(int n, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot; __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t a = smem_u32(base), b = smem_u32(base + 65536);
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    int counts[] = {1, 4, 16, 64};
    for (int ci = 0; ci < 4; ++ci) {
      for (int rep = 0; rep < 3; ++rep) {
        long long t0 = clock64();
        for (int i = 0; i < counts[ci]; ++i) {
          uint64_t ad = sdesc(a + (i & 3) * 32), bd = sdesc(b + (i & 3) * 32);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)i));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
        wait(smem_u32(&bar), ph); ph ^= 1;
        long long t1 = clock64();
        if (rep == 2 && blockIdx.x == 0) out[ci] = t1 - t0;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {128, 256}) {
    for (int g : {1, 148}) {
      k<<<g, 128, 200 * 1024>>>(n, d); cudaDeviceSynchronize();
      unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("N=%d grid=%d: issue+commit+wait cycles for 1/4/16/64 MMAs: %llu %llu %llu %llu\n", n, g, h[0], h[1], h[2], h[3]);
    }
  }
  return 0;
}
