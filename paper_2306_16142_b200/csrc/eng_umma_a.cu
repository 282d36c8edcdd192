// tcgen05 bf16 engines for the protocol row ops (see engines.h)
#include "eng_common.cuh"
DDF_INST_UMMA(ddf::RawForwardOp)
DDF_INST_UMMA(ddf::RawGradOp)
DDF_INST_UMMA(ddf::QueryOp)
DDF_INST_UMMA(ddf::NormalOp)
DDF_UMMA_DEBUG_READER(umma_debug_a)
