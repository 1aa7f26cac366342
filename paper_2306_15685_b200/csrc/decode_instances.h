// The decode kernel's instantiations, one group per translation unit
// (csrc/kernels/*.cu): each unit compiles only its group, so the hot C3
// kernel (256 threads, 16-byte records, direct table, f32 scores) is
// optimised on its own, and the units build in parallel.  The host ABI
// (arcboost_b200.cu) declares them extern and launches them.
#pragma once

#define AB_DECODE_HOT(X) X(256, Fmt16<false>, float)
#define AB_DECODE_F16D(X)                                                                               \
  X(512, Fmt16<false>, float) X(1024, Fmt16<false>, float) X(256, Fmt16<false>, double)               \
  X(512, Fmt16<false>, double) X(1024, Fmt16<false>, double)
#define AB_DECODE_F16H(X)                                                                               \
  X(256, Fmt16<true>, float) X(512, Fmt16<true>, float) X(1024, Fmt16<true>, float)                   \
  X(256, Fmt16<true>, double) X(512, Fmt16<true>, double) X(1024, Fmt16<true>, double)
#define AB_DECODE_F24D(X)                                                                               \
  X(256, Fmt24<false>, float) X(512, Fmt24<false>, float) X(1024, Fmt24<false>, float)                \
  X(256, Fmt24<false>, double) X(512, Fmt24<false>, double) X(1024, Fmt24<false>, double)
#define AB_DECODE_F24H(X)                                                                               \
  X(256, Fmt24<true>, float) X(512, Fmt24<true>, float) X(1024, Fmt24<true>, float)                   \
  X(256, Fmt24<true>, double) X(512, Fmt24<true>, double) X(1024, Fmt24<true>, double)
// small graphs, 1024-thread CTAs: the token table in shared memory
#define AB_DECODE_F16S(X) X(1024, Fmt16S, float) X(1024, Fmt16S, double)
// ... a channel per thread-block cluster (C1 / C2: few channels)
#define AB_DECODE_F16C(X) X(1024, Fmt16SC2, float) X(1024, Fmt16SC4, float) X(1024, Fmt16SC8, float) X(1024, Fmt16SC16, float)
#define AB_DECODE_ALL(X)                                                                                \
  AB_DECODE_HOT(X) AB_DECODE_F16D(X) AB_DECODE_F16H(X) AB_DECODE_F24D(X) AB_DECODE_F24H(X) AB_DECODE_F16S(X) \
  AB_DECODE_F16C(X)

#define AB_DECODE_EXTERN(B, F, S) \
  extern template __global__ void ab::decode_kernel<B, ab::F, S>(const __grid_constant__ ab::DecodeParams);
#define AB_DECODE_INSTANCE(B, F, S) \
  template __global__ void ab::decode_kernel<B, ab::F, S>(const __grid_constant__ ab::DecodeParams);
