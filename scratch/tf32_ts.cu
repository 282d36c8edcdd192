// tcgen05.mma kind::tf32 probe: (1) correctness of the SS (A in shared memory)
// and TS (A in TMEM) forms against a host reference, with the A layout in TMEM
// as lane = row, column = k (one fp32 per column); (2) how the tensor core
// treats the low 13 mantissa bits of fp32 operands (truncate vs round);
// (3) issue cost per instruction, M = 128, N = 128/256, K = 8, SS vs TS.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d; }
__host__ __device__ inline uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// byte offset of element (r, k) of a [rows][32] fp32 K-major 128B-swizzled tile
__host__ __device__ inline uint32_t swz(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4);
}
__host__ __device__ inline uint32_t swz32(int r, int k) {
  return (uint32_t)((r >> 3) * 256 + (r & 7) * 32 + ((((k >> 2) ^ ((r >> 2) & 1))) << 4) + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t sdesc32(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr & 0x3FFFFu) >> 4); d |= (uint64_t)1 << 16; d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)6 << 61; return d; }
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(bar), "r"(par) : "memory");
}
// A: 128 x 32 fp32, B: 256 x 32 fp32 (row-major, K contiguous). D: 128 x 256 fp32.
// mode 0: SS, mode 1: TS.  nrep > 1: timing, D accumulates garbage.
__global__ void k(const float* A, const float* B, float* D, int mode, int n, int nrep, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot; __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  // A and B -> shared (swizzled); A also -> TMEM columns [256, 288)
  uint8_t* sa = base; uint8_t* sb = base + 16384;
  for (int i = tid; i < 128 * 32; i += blockDim.x) { int r = i / 32, kk = i % 32; *(float*)(sa + swz(r, kk)) = A[i]; }
  for (int i = tid; i < 256 * 32; i += blockDim.x) { int r = i / 32, kk = i % 32; *(float*)(sb + swz(r, kk)) = B[i]; }
  uint8_t* sb32 = base + 65536;   // [K/8][256 rows][32 B], 32B swizzle
  for (int i = tid; i < 256 * 32; i += blockDim.x) { int r = i / 32, kk = i % 32;
    *(float*)(sb32 + (kk >> 3) * 8192 + swz32(r, kk & 7)) = B[i]; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (warp < 4) {
    const int r = warp * 32 + lane;
    uint32_t v[32];
    for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(A[r * 32 + e]);
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 256u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 :: "r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                 "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                 "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t id = idesc_tf32(n);
    long long t0 = clock64();
    for (int rep = 0; rep < nrep; ++rep)
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t bd = (mode >= 2) ? sdesc32(smem_u32(sb32) + ks * 8192) : sdesc(smem_u32(sb) + ks * 32);
        const uint32_t acc = (rep | ks) ? 1u : 0u;
        if (mode == 4) {   // 3xTF32 pattern: TS(hi, Whi) + TS(hi, Wlo) + SS(lo, Whi), Wlo = next K block
          const uint64_t bl = sdesc32(smem_u32(sb32) + ((ks + 1) & 3) * 8192);
          const uint64_t ad = sdesc(smem_u32(sa) + ks * 32);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       :: "r"(tmem), "r"(tmem + 256u + (uint32_t)(ks * 8)), "l"(bd), "r"(id), "r"(acc));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       :: "r"(tmem), "r"(tmem + 256u + (uint32_t)(ks * 8)), "l"(bl), "r"(id), "r"(1u));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       :: "r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(1u));
        } else if (mode == 0 || mode == 2) {
          const uint64_t ad = sdesc(smem_u32(sa) + ks * 32);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       :: "r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        } else {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       :: "r"(tmem), "r"(tmem + 256u + (uint32_t)(ks * 8)), "l"(bd), "r"(id), "r"(acc));
        }
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
    wait_bar(smem_u32(&bar), 0);
    long long t1 = clock64();
    if (cyc) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4 && D) {
    const int r = warp * 32 + lane;
    for (int c = 0; c < n; c += 32) {
      uint32_t v[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
                   "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int e = 0; e < 32; ++e) D[r * 256 + c + e] = __uint_as_float(v[e]);
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
static float rn_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x1000u + ((u >> 13) & 1u) - 1u; u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
static float rna_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
int main() {
  std::mt19937 g(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> A(128 * 32), B(256 * 32), D(128 * 256);
  for (auto& x : A) x = U(g);
  for (auto& x : B) x = U(g);
  float *dA, *dB, *dD; unsigned long long* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    k<<<1, 128, 140 * 1024>>>(dA, dB, dD, mode, 256, 1, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err_t = 0, err_rn = 0, err_rna = 0, err_f = 0, mx = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 256; ++c) {
        double st = 0, sr = 0, sa = 0, sf = 0;
        for (int kk = 0; kk < 32; ++kk) {
          st += (double)trunc_tf32(A[r * 32 + kk]) * trunc_tf32(B[c * 32 + kk]);
          sr += (double)rn_tf32(A[r * 32 + kk]) * rn_tf32(B[c * 32 + kk]);
          sa += (double)rna_tf32(A[r * 32 + kk]) * rna_tf32(B[c * 32 + kk]);
          sf += (double)A[r * 32 + kk] * B[c * 32 + kk];
        }
        const double d = D[r * 256 + c];
        err_t = fmax(err_t, fabs(d - st)); err_rn = fmax(err_rn, fabs(d - sr)); err_rna = fmax(err_rna, fabs(d - sa));
        err_f = fmax(err_f, fabs(d - sf)); mx = fmax(mx, fabs(sf));
      }
    printf("%s%s (%s): max|D| %.3f  max err vs trunc-tf32 %.3g, vs rn-tf32 %.3g, vs rna-tf32 %.3g, vs fp32 %.3g\n",
           (mode & 1) ? "TS" : "SS", mode >= 2 ? "/B-sw32" : "", cudaGetErrorString(e), mx, err_t, err_rn, err_rna, err_f);
  }
  for (int mode = 0; mode < 5; ++mode)
    for (int n : {128, 256}) {
      const int nrep = 2048;
      cudaMemset(dc, 0, 8);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<148, 128, 140 * 1024>>>(dA, dB, nullptr, mode, n, nrep, dc);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      const double per = (double)cyc / 148 / (nrep * 4) / (mode == 4 ? 3 : 1);
      const double tf = 2.0 * 128 * n * 8 * nrep * 4 * 148 * (mode == 4 ? 3 : 1) / (ms * 1e-3) / 1e12;
      printf("mode %d %s N=%d: %.1f cycles per K=8 MMA, %.0f TF/s tf32 by events (%s)\n", mode, (mode & 1) ? "TS" : "SS", n, per, tf,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
