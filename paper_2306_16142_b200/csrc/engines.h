// The MLP engines behind run_mlp (ddf_api.cu), compiled in their own
// translation units (eng_*.cu) so the library builds in parallel.  Each
// engine entry is a template declared here and explicitly instantiated for
// every row op in exactly one eng_*.cu; ddf_api.cu only calls it.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "ddf_common.cuh"
#include "field_kernels.cuh"
#include "mlp_umma.cuh"
#include "udf.cuh"
#include "wavefront.cuh"

namespace ddf {
namespace engines {

// bf16 tcgen05 engines (mlp_umma.cuh): 0 ok, 1 usage, 4 CUDA (message in *err)
template <class Op>
int umma_launch(const FieldDev& F, const std::vector<umma::NetImage>& images, const Op& op, int max_rows,
                int sm_count, uint32_t* mask_scratch, cudaStream_t st, std::string* err);
// 3xTF32 tcgen05 engine (mlp_x3.cuh), same contract
template <class Op>
int x3_launch(const FieldDev& F, const std::vector<umma::NetImage>& images, const Op& op, int max_rows,
              int sm_count, uint32_t* mask_scratch, cudaStream_t st, std::string* err);
// exact-fp32 FFMA engine (mlp_simt.cuh, field_kernels.cuh): max_width <= 512
template <class Op>
int simt_launch(const FieldDev& F, const Op& op, int max_rows, int max_width, int sm_count, cudaStream_t st,
                std::string* err);

// diagnostics counters of the tcgen05 engines (DDF_PIPE_STATS builds), summed
// over the engine translation units
void umma_debug_counters(unsigned long long* out16, bool reset);
// the event timeline of CTA 0 (DDF_TRACE builds): entries written, <= cap
int umma_debug_trace(unsigned long long* out, int cap, bool reset);

}  // namespace engines
}  // namespace ddf

// every row op the engines serve; X(op, has_fused_engine)
#define DDF_ENGINE_OPS(X) \
  X(ddf::RawForwardOp)    \
  X(ddf::RawGradOp)       \
  X(ddf::QueryOp)         \
  X(ddf::TraceStepOp)     \
  X(ddf::NormalOp)        \
  X(ddf::GradOutOp)       \
  X(ddf::udf::ScanOp)     \
  X(ddf::udf::ProbeOp)
