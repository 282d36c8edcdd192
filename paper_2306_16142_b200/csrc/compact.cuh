// Stable stream compaction of per-slot flags into ascending slot lists --
// the device form of the reference's np.nonzero(alive) (field.py:277,
// render.py:225).  Optionally buckets the survivors by object id (stable
// within each bucket) so a gradient pass can run one network per tile.
//
//   pass 1  count      per 1024-slot block, per object (warp ballot + popc)
//   pass 2  scan       one CTA: exclusive scan of block counts -> offsets,
//                      segment table seg[0..n_obj], total -> *count
//   pass 3  scatter    warp ballot ranks + per-warp prefix -> list
// HBM traffic: flags (1 B) + obj (4 B, bucketed only) read twice, 4 B written
// per survivor.
#pragma once
#include "ddf_common.cuh"

namespace ddf {
namespace compact {

constexpr int NT = 256;
constexpr int IPT = 4;
constexpr int BLOCK_ITEMS = NT * IPT;

// sel (nullable): only slots whose sel byte equals sel_val are taken
__device__ __forceinline__ bool take(const uint8_t* flags, const uint8_t* sel, int sel_val, const int* obj, int idx,
                                     int n, int j) {
  return idx < n && flags[idx] && (sel == nullptr || sel[idx] == sel_val) && (obj == nullptr || obj[idx] == j);
}

__global__ void __launch_bounds__(NT) count_kernel(const uint8_t* __restrict__ flags, const uint8_t* __restrict__ sel,
                                                   int sel_val, const int* __restrict__ obj, int n, int n_obj,
                                                   int* __restrict__ block_counts) {
  __shared__ int cnt[DDF_MAX_OBJECTS];
  if (threadIdx.x < DDF_MAX_OBJECTS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * BLOCK_ITEMS;
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < n_obj; ++j) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const unsigned b = __ballot_sync(0xffffffffu, take(flags, sel, sel_val, obj, base + i * NT + threadIdx.x, n, j));
      c += __popc(b);
    }
    if (lane == 0 && c) atomicAdd(&cnt[j], c);
  }
  __syncthreads();
  if (threadIdx.x < n_obj) block_counts[blockIdx.x * n_obj + threadIdx.x] = cnt[threadIdx.x];
}

// one CTA of 1024 threads; block_counts -> block offsets (in place)
__global__ void __launch_bounds__(1024) scan_kernel(int* __restrict__ block_counts, int nblocks, int n_obj,
                                                    int* __restrict__ seg, int* __restrict__ count,
                                                    unsigned long long* __restrict__ rows_acc,
                                                    unsigned long long* __restrict__ rows_acc2) {
  __shared__ int part[1024];
  __shared__ int seg_base;
  if (threadIdx.x == 0) seg_base = 0;
  __syncthreads();
  const int per = (nblocks + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(nblocks, b0 + per);
  for (int j = 0; j < n_obj; ++j) {
    int s = 0;
    for (int b = b0; b < b1; ++b) s += block_counts[b * n_obj + j];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {       // Hillis-Steele inclusive scan
      const int v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += v;
      __syncthreads();
    }
    int run = seg_base + part[threadIdx.x] - s;      // exclusive
    for (int b = b0; b < b1; ++b) {
      const int c = block_counts[b * n_obj + j];
      block_counts[b * n_obj + j] = run;
      run += c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      seg[j] = seg_base;
      seg_base += part[1023];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    seg[n_obj] = seg_base;
    *count = seg_base;
    if (rows_acc) *rows_acc += (unsigned long long)seg_base;
    if (rows_acc2) *rows_acc2 += (unsigned long long)seg_base;
  }
}

__global__ void __launch_bounds__(NT) scatter_kernel(const uint8_t* __restrict__ flags, const uint8_t* __restrict__ sel,
                                                     int sel_val, const int* __restrict__ obj,
                                                     int n, int n_obj, const int* __restrict__ block_offsets,
                                                     int* __restrict__ list) {
  __shared__ int warp_cnt[NT / 32];
  const int base = blockIdx.x * BLOCK_ITEMS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int j = 0; j < n_obj; ++j) {
    int run = block_offsets[blockIdx.x * n_obj + j];
    for (int i = 0; i < IPT; ++i) {
      const int idx = base + i * NT + threadIdx.x;
      const bool t = take(flags, sel, sel_val, obj, idx, n, j);
      const unsigned b = __ballot_sync(0xffffffffu, t);
      if (lane == 0) warp_cnt[warp] = __popc(b);
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) {
        const int c = warp_cnt[w];
        before += (w < warp) ? c : 0;
        total += c;
      }
      if (t) list[run + before + __popc(b & lt)] = idx;
      run += total;
      __syncthreads();
    }
  }
}

}  // namespace compact
}  // namespace ddf
