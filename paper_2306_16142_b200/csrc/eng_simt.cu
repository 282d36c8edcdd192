// exact-fp32 FFMA engine for every row op (see engines.h)
#include "eng_common.cuh"
DDF_ENGINE_OPS(DDF_INST_SIMT)
