// tcgen05 bf16 engines for the UDF row ops (see engines.h)
#include "eng_common.cuh"
DDF_INST_UMMA(ddf::udf::ScanOp)
DDF_INST_UMMA(ddf::udf::ProbeOp)
DDF_UMMA_DEBUG_READER(umma_debug_c)

namespace ddf {
namespace engines {
void umma_debug_a(unsigned long long*, bool);
void umma_debug_b(unsigned long long*, bool);
int umma_debug_a_trace(unsigned long long*, int, bool);
int umma_debug_b_trace(unsigned long long*, int, bool);
int umma_debug_trace(unsigned long long* out, int cap, bool reset) {
  int n = umma_debug_a_trace(out, cap, reset);
  n += umma_debug_b_trace(out + n, cap - n, reset);
  n += umma_debug_c_trace(out + n, cap - n, reset);
  return n;
}
void umma_debug_counters(unsigned long long* out16, bool reset) {
  for (int i = 0; i < 16; ++i) out16[i] = 0;
  umma_debug_a(out16, reset);
  umma_debug_b(out16, reset);
  umma_debug_c(out16, reset);
}
}  // namespace engines
}  // namespace ddf
