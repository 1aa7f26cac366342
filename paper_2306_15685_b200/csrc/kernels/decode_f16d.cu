// Decode kernel instantiations: group F16D (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_F16D(AB_DECODE_INSTANCE)
