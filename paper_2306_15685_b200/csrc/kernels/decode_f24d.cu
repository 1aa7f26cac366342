// Decode kernel instantiations: group F24D (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_F24D(AB_DECODE_INSTANCE)
