// Shared body of the engine translation units (eng_*.cu): definitions of the
// engines.h entry points; each TU instantiates them for its share of the row
// ops.  Kernels of wavefront.cuh / udf.cuh stay in ddf_api.cu (DDF_OPS_ONLY).
#pragma once
#define DDF_OPS_ONLY 1
#include "engines.h"
#include "mlp_2sm.cuh"
#include "mlp_x3.cuh"

namespace ddf {
namespace engines {

template <class Op>
int umma_launch(const FieldDev& F, const std::vector<umma::NetImage>& images, const Op& op, int max_rows,
                int sm_count, uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  // one network wider than 256: the CTA-pair engine (mlp_2sm.cuh); DDF_DEBUG_UMMA
  // bit 4096 keeps the single-CTA engine (A/B timing)
  if (F.n_obj == 1 && images.size() == 1 && !images[0].host.pp && !(umma::debug_bits() & 4096) && sm_count >= 2)
    return umma::launch_2sm<Op>(F, images[0], op, max_rows, sm_count, mask_scratch, st, err);
  return umma::launch<Op>(F, images, op, max_rows, sm_count, mask_scratch, st, err);
}

template <class Op>
int x3_launch(const FieldDev& F, const std::vector<umma::NetImage>& images, const Op& op, int max_rows,
              int sm_count, uint32_t* mask_scratch, cudaStream_t st, std::string* err) {
  return x3::launch<Op>(F, images, op, max_rows, sm_count, mask_scratch, st, err);
}

template <int M, int KMAX>
size_t simt_smem() {
  return sizeof(double) * M * 8 + sizeof(float) * (2 * KMAX * M + 2 * simt::KC * simt::NC + 2 * M) +
         sizeof(uint32_t) * DDF_MAX_LAYERS * KMAX * (M / 32) + sizeof(int) * 2 * M;
}

template <class Op, int M, int KMAX>
int simt_run(const FieldDev& F, const Op& op, int max_rows, int sm_count, cudaStream_t st, std::string* err) {
  const size_t sm = simt_smem<M, KMAX>();
  void (*kern)(const FieldDev, const Op);
  if constexpr (Op::kGrad) kern = simt::grad_kernel<M, KMAX, Op>;
  else kern = simt::forward_kernel<M, KMAX, Op>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) { *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return 4; }
  const int tiles = (max_rows + M - 1) / M + (Op::kGrad ? F.n_obj : 0);
  const int grid = std::max(1, std::min(tiles, sm_count));
  kern<<<grid, simt::NT, sm, st>>>(F, op);
  e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("simt kernel launch: ") + cudaGetErrorString(e); return 4; }
  return 0;
}

template <class Op>
int simt_launch(const FieldDev& F, const Op& op, int max_rows, int max_width, int sm_count, cudaStream_t st,
                std::string* err) {
  if (max_width <= 256) return simt_run<Op, 64, 256>(F, op, max_rows, sm_count, st, err);
  if (max_width <= 512) return simt_run<Op, 32, 512>(F, op, max_rows, sm_count, st, err);
  *err = "fp32 engine supports layer widths up to 512";
  return 1;
}

}  // namespace engines
}  // namespace ddf

#define DDF_INST_UMMA(OP)                                                                                     \
  template int ddf::engines::umma_launch<OP>(const ddf::FieldDev&, const std::vector<ddf::umma::NetImage>&,  \
                                             const OP&, int, int, uint32_t*, cudaStream_t, std::string*);
#define DDF_INST_X3(OP)                                                                                       \
  template int ddf::engines::x3_launch<OP>(const ddf::FieldDev&, const std::vector<ddf::umma::NetImage>&,    \
                                           const OP&, int, int, uint32_t*, cudaStream_t, std::string*);
#define DDF_INST_SIMT(OP)                                                                                     \
  template int ddf::engines::simt_launch<OP>(const ddf::FieldDev&, const OP&, int, int, int, cudaStream_t,   \
                                             std::string*);

// the diagnostics counters and event trace of this TU's module, under
// TU-specific names
#define DDF_UMMA_DEBUG_READER(NAME)                                                                         \
  namespace ddf { namespace engines {                                                                       \
  void NAME(unsigned long long* acc, bool reset) {                                                          \
    unsigned long long h[16];                                                                               \
    if (cudaMemcpyFromSymbol(h, umma::g_dbg, sizeof(h)) != cudaSuccess) return;                             \
    for (int i = 0; i < 16; ++i) acc[i] += h[i];                                                            \
    if (reset) {                                                                                            \
      for (int i = 0; i < 16; ++i) h[i] = 0;                                                                \
      cudaMemcpyToSymbol(umma::g_dbg, h, sizeof(h));                                                        \
    }                                                                                                       \
  }                                                                                                         \
  int NAME##_trace(unsigned long long* out, int cap, bool reset) {                                          \
    std::vector<unsigned long long> all(umma::TRACE_CAP);                                                   \
    if (cudaMemcpyFromSymbol(all.data(), umma::g_trace, sizeof(unsigned long long) * umma::TRACE_CAP) !=    \
        cudaSuccess) return 0;                                                                              \
    int n = 0;                                                                                              \
    for (unsigned long long v : all)                                                                        \
      if (v && n < cap) out[n++] = v;                                                                       \
    if (reset) {                                                                                            \
      std::vector<unsigned long long> z(umma::TRACE_CAP, 0ull);                                             \
      cudaMemcpyToSymbol(umma::g_trace, z.data(), sizeof(unsigned long long) * umma::TRACE_CAP);            \
    }                                                                                                       \
    return n;                                                                                               \
  } } }
