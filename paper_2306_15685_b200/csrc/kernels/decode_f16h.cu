// Decode kernel instantiations: group F16H (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_F16H(AB_DECODE_INSTANCE)
