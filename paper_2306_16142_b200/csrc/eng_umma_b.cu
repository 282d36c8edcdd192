// tcgen05 bf16 engines for the render's row ops (see engines.h)
#include "eng_common.cuh"
DDF_INST_UMMA(ddf::TraceStepOp)
DDF_INST_UMMA(ddf::GradOutOp)
DDF_INST_UMMA(ddf::TraceGradOp)
DDF_UMMA_DEBUG_READER(umma_debug_b)
