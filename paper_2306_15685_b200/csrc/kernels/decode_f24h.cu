// Decode kernel instantiations: group F24H (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_F24H(AB_DECODE_INSTANCE)
