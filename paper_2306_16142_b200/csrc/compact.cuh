// Stable stream compaction of per-slot flags into ascending slot lists --
// the device form of the reference's np.nonzero(alive) (field.py:277,
// render.py:225).  Optionally buckets the survivors by object id (stable
// within each bucket) so a gradient pass can run one network per tile.
//
//   pass 1  count      per 1024-slot block, per object (warp ballot + popc)
//   pass 2  scan       one CTA: exclusive scan of block counts -> offsets,
//                      segment table seg[0..n_obj], total -> *count
//   pass 3  scatter    match-any ranks per object + per-warp prefix -> list
// HBM traffic: flags (1 B) + obj (4 B, bucketed only) read twice (once per
// pass, whatever the object count), 4 B written per survivor.
//
// Unbucketed lists (one segment) take the single-pass kernel instead:
// onepass_kernel reads the flags once and finds its block's offset by
// decoupled look-back over the predecessors' published counts.
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
  // each slot's flag and object id are read once; the per-object ballots
  // below work on registers (-1 = not taken)
  int oid[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int idx = base + i * NT + threadIdx.x;
    oid[i] = take(flags, sel, sel_val, nullptr, idx, n, 0) ? (obj ? obj[idx] : 0) : -1;
  }
  for (int j = 0; j < n_obj; ++j) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i) c += __popc(__ballot_sync(0xffffffffu, oid[i] == j));
    if (lane == 0 && c) atomicAdd(&cnt[j], c);
  }
  __syncthreads();
  if (threadIdx.x < n_obj) block_counts[blockIdx.x * n_obj + threadIdx.x] = cnt[threadIdx.x];
}

// one CTA of 1024 threads; block_counts -> block offsets (in place)
__global__ void __launch_bounds__(1024) scan_kernel(int* __restrict__ block_counts, int nblocks, int n_obj,
                                                    int* __restrict__ seg, int* __restrict__ count,
                                                    unsigned long long* __restrict__ rows_acc,
                                                    unsigned long long* __restrict__ rows_acc2,
                                                    unsigned long long* __restrict__ rows_acc3) {
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
    if (rows_acc3) *rows_acc3 += (unsigned long long)seg_base;
  }
}

__global__ void __launch_bounds__(NT) scatter_kernel(const uint8_t* __restrict__ flags, const uint8_t* __restrict__ sel,
                                                     int sel_val, const int* __restrict__ obj,
                                                     int n, int n_obj, const int* __restrict__ block_offsets,
                                                     int* __restrict__ list) {
  // one pass over the block for every object: __match_any_sync groups a
  // warp's lanes by object id; wc[i][w][j] = slots of object j in warp w's
  // i-th 32-slot row.  A slot's position is its object's block offset plus
  // the same-object slots before it in index order (i, warp, lane).
  __shared__ int wc[IPT][NT / 32][DDF_MAX_OBJECTS];
  const int base = blockIdx.x * BLOCK_ITEMS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int k = threadIdx.x; k < IPT * (NT / 32) * DDF_MAX_OBJECTS; k += NT) (&wc[0][0][0])[k] = 0;
  __syncthreads();
  int oid[IPT];
  unsigned grp[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int idx = base + i * NT + threadIdx.x;
    int o = take(flags, sel, sel_val, nullptr, idx, n, 0) ? (obj ? obj[idx] : 0) : -1;
    if (o >= n_obj) o = -1;   // ids outside [0, n_obj) are never listed
    oid[i] = o;
    grp[i] = __match_any_sync(0xffffffffu, o);
    if (o >= 0 && (grp[i] & lt) == 0u) wc[i][warp][o] = __popc(grp[i]);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int j = oid[i];
    if (j < 0) continue;
    int pos = block_offsets[blockIdx.x * n_obj + j] + __popc(grp[i] & lt);
#pragma unroll
    for (int i2 = 0; i2 < IPT; ++i2)
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) pos += (i2 < i || (i2 == i && w < warp)) ? wc[i2][w][j] : 0;
    list[pos] = base + i * NT + threadIdx.x;
  }
}

// ---------------------------------------------------------------- single pass
// state[b] (zeroed before the launch, with the ticket counter at state[nb]):
// bits 32-33 = 1 aggregate published, 2 inclusive prefix published; bits 0-31
// the count.  Blocks take tickets in launch order, so every predecessor a
// block waits on is already resident and never waits on a successor.
constexpr unsigned long long ST_AGG = 1ull << 32, ST_INC = 2ull << 32;

__device__ __forceinline__ unsigned long long ld_state(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_state(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int OP_IPT = 32;                  // contiguous slots per thread
constexpr int OP_ITEMS = NT * OP_IPT;       // 8192 slots per block: a short look-back chain
// state: nb block words, the ticket counter (state[nb]) and a finished-blocks
// counter (state[nb + 1]).  The kernel expects them all zero and leaves them
// all zero: the last block to finish (every block's look-back has ended by
// then) clears them, so a call needs no memset launch ahead of it and a
// captured graph replays without one.
constexpr int OP_STATE_EXTRA = 2;

__global__ void __launch_bounds__(NT) onepass_kernel(const uint8_t* __restrict__ flags, const uint8_t* __restrict__ sel,
                                                     int sel_val, int n, int nb, unsigned long long* state,
                                                     int* __restrict__ list, int* __restrict__ seg,
                                                     int* __restrict__ count, unsigned long long* rows_acc,
                                                     unsigned long long* rows_acc2,
                                                     unsigned long long* rows_acc3) {
  __shared__ int warp_tot[NT / 32];
  __shared__ int s_ticket, s_excl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_ticket = (int)atomicAdd(&state[nb], 1ull);
  __syncthreads();
  const int b = s_ticket;
  const int base = b * OP_ITEMS + threadIdx.x * OP_IPT;
  // this thread's 32 slots as a bit mask (vector loads when fully in range)
  uint32_t bits = 0u;
  if (base + OP_IPT <= n && (((uintptr_t)(flags + base) | (uintptr_t)(sel ? sel + base : nullptr)) & 15u) == 0) {
    const uint4* fv = reinterpret_cast<const uint4*>(flags + base);
    const uint4 f0 = __ldg(fv), f1 = __ldg(fv + 1);
    const uint32_t fw[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
    uint32_t sw[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (sel) {
      const uint4* sv = reinterpret_cast<const uint4*>(sel + base);
      const uint4 s0 = __ldg(sv), s1 = __ldg(sv + 1);
      sw[0] = s0.x; sw[1] = s0.y; sw[2] = s0.z; sw[3] = s0.w; sw[4] = s1.x; sw[5] = s1.y; sw[6] = s1.z; sw[7] = s1.w;
    }
#pragma unroll
    for (int e = 0; e < OP_IPT; ++e) {
      const bool fl = ((fw[e >> 2] >> (8 * (e & 3))) & 0xffu) != 0u;
      const bool sl = !sel || (int)((sw[e >> 2] >> (8 * (e & 3))) & 0xffu) == sel_val;
      bits |= (fl && sl ? 1u : 0u) << e;
    }
  } else {
    for (int e = 0; e < OP_IPT; ++e) bits |= (take(flags, sel, sel_val, nullptr, base + e, n, 0) ? 1u : 0u) << e;
  }
  const int cnt = __popc(bits);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int wt = lane < NT / 32 ? warp_tot[lane] : 0;
    int agg = wt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(0xffffffffu, agg, o);
    if (b == 0) {
      if (lane == 0) {
        st_state(&state[0], ST_INC | (unsigned)agg);
        s_excl = 0;
      }
    } else {
      if (lane == 0) st_state(&state[b], ST_AGG | (unsigned)agg);
      int excl = 0;
      int p = b - 1 - lane;   // this lane's predecessor in the current window
      while (true) {
        unsigned long long v = ST_INC;   // before block 0: an inclusive prefix of 0
        if (p >= 0) {
          do { v = ld_state(&state[p]); } while ((v >> 32) == 0ull);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (v >> 32) == 2ull);
        // lanes up to and including the nearest inclusive prefix contribute
        const int stop = inc ? __ffs(inc) - 1 : 31;
        int val = lane <= stop ? (int)(v & 0xffffffffu) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (inc) break;
        p -= 32;
      }
      if (lane == 0) {
        st_state(&state[b], ST_INC | (unsigned)(excl + agg));
        s_excl = excl;
      }
    }
  }
  __syncthreads();
  int before = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) before += (w < warp) ? warp_tot[w] : 0;
  int pos = s_excl + before + incl - cnt;
  while (bits) {
    const int e = __ffs(bits) - 1;
    list[pos++] = base + e;
    bits &= bits - 1u;
  }
  if (b == nb - 1 && threadIdx.x == NT - 1) {   // the last thread of the last block ends at the total
    seg[0] = 0;
    seg[1] = pos;
    *count = pos;
    if (rows_acc) *rows_acc += (unsigned long long)pos;
    if (rows_acc2) *rows_acc2 += (unsigned long long)pos;
    if (rows_acc3) *rows_acc3 += (unsigned long long)pos;
  }
  // self-cleaning: this block no longer reads any state word (its look-back
  // ended before the barrier above); the block that finishes last resets them
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&state[nb + 1], 1ull) == (unsigned long long)(nb - 1);
  }
  __syncthreads();
  if (s_last)
    for (int i = threadIdx.x; i < nb + OP_STATE_EXTRA; i += NT) state[i] = 0ull;
}

}  // namespace compact
}  // namespace ddf
