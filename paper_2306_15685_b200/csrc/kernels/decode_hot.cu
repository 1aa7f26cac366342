// Decode kernel instantiations: group HOT (csrc/decode_instances.h).
#include "../decode_kernel.cuh"
#include "../decode_instances.h"

AB_DECODE_HOT(AB_DECODE_INSTANCE)
