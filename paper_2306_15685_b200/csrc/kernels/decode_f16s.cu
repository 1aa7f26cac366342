// Decode kernel instantiations: group F16S (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_F16S(AB_DECODE_INSTANCE)
