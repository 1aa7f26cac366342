// Decode kernel instantiations: group F16C (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_F16C(AB_DECODE_INSTANCE)
