// Epilogue instruction-stream microbenchmark: 8 warps (2 per TMEM lane
// quarter) repeatedly do LDTM.x32 -> +bias, ReLU -> bf16 pack -> 4 x STS.128
// into a 128B-swizzled tile, no barriers.  Cycles per 32-column chunk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) { __nv_bfloat162 v = __floats2bfloat162_rn(a, b); return *reinterpret_cast<uint32_t*>(&v); }
#define LD32(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
 : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr))
__global__ void k(int iters, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ float bias[512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  for (int i = threadIdx.x; i < 512; i += blockDim.x) bias[i] = 0.001f * i;
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const int q = warp & 3, sub = warp >> 2, r = q * 32 + lane;
  const uint32_t a_row = smem_u32(sm) + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
  const int r7 = r & 7;
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = 0; i < 4; ++i) {
      const int c = sub * 32 + i * 64 + ((it & 1) << 8);
      uint32_t rg[32];
      if (mode & 1) { for (int e = 0; e < 32; ++e) rg[e] = it + e; }
      else { LD32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, rg); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pk[e] = pack_bf16(fmaxf(__uint_as_float(rg[2 * e]) + bias[c + 2 * e], 0.f), fmaxf(__uint_as_float(rg[2 * e + 1]) + bias[c + 2 * e + 1], 0.f));
      if (!(mode & 2)) {
        const uint32_t blk = a_row + (uint32_t)((c >> 6) * 16384);
        const int cc0 = (c & 63) >> 3;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(blk + (uint32_t)(((cc0 + e) ^ r7) << 4)), "r"(pk[4*e]), "r"(pk[4*e+1]), "r"(pk[4*e+2]), "r"(pk[4*e+3]) : "memory");
      } else { for (int e = 0; e < 16; ++e) acc ^= pk[e]; }
    }
  }
  long long t1 = clock64();
  if (lane == 0 && warp == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
  if (acc == 12345) out[1] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[] = {"LDTM+math+STS", "regs+math+STS", "LDTM+math", "regs+math"};
  for (int mode = 0; mode < 4; ++mode) for (int nw : {8, 4}) {
    cudaMemset(d, 0, 16);
    int iters = 2000;
    k<<<148, nw * 32, 140 * 1024>>>(iters, mode, d); cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-16s warps=%d: %.1f cycles per 32-col chunk per warp (%s)\n", names[mode], nw, (double)c / 148 / (iters * 4), cudaGetErrorString(cudaGetLastError()));
  }
}
