// bf16 tcgen05 engine (placeholder until the UMMA kernels land).
#pragma once
#include <string>
#include "ddf_common.cuh"
namespace ddf {
namespace umma {
struct NetImage { void* dev = nullptr; int in_width = 0; };
inline int build_image(const int32_t* widths, int32_t, const double*, const double*, NetImage* img, std::string*) {
  img->in_width = widths[0];
  img->dev = nullptr;
  return 0;
}
inline void free_image(NetImage* img) { if (img->dev) cudaFree(img->dev); img->dev = nullptr; }
template <class Op>
int launch(const FieldDev&, const Op&, int, bool, int, cudaStream_t, std::string* err) {
  *err = "bf16 tcgen05 engine not built yet";
  return 1;
}
}  // namespace umma
}  // namespace ddf
