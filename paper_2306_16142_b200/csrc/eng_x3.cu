// 3xTF32 tcgen05 engine for every row op (see engines.h)
#include "eng_common.cuh"
DDF_ENGINE_OPS(DDF_INST_X3)
