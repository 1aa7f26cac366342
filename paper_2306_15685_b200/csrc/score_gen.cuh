// Synthetic score generation on the device ("generation on
// device"): the uniform cost streams the reference's tooling and the
// benchmark draw on the host with numpy — `np.random.default_rng(seed)
// .uniform(low, high, n)` (PCG64, XSL-RR 128/64; synth.py:156-195 scores,
// harness.py:374 per-utterance streams) — reproduced bit for bit, so a
// [C, T, L] cost tensor is produced in HBM instead of being copied there.
//
// numpy's PCG64 step: state = state * M + inc (mod 2^128), output the
// XSL-RR of the NEW state: rotr64(hi ^ lo, hi >> 58).  uniform(low, high) =
// low + (high - low) * ((x >> 11) * 2^-53), rounded step by step (no FMA).
// Each thread jumps its stream ahead to its chunk (Brown's O(log n) LCG
// advance) and generates the chunk sequentially.
#pragma once
#include <cstdint>

namespace ab {

struct U128 {
  unsigned long long hi, lo;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

constexpr unsigned long long PCG_MULT_HI = 2549297995355413924ull; // 0x2360ED051FC65DA4
constexpr unsigned long long PCG_MULT_LO = 4865540595714422341ull; // 0x4385DF649FCCF645

// state after `delta` more steps (pcg_advance_lcg_128)
__device__ __forceinline__ U128 pcg_advance(U128 state, U128 inc, unsigned long long delta) {
  U128 acc_mult{0, 1}, acc_plus{0, 0}, cur_mult{PCG_MULT_HI, PCG_MULT_LO}, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}

__device__ __forceinline__ unsigned long long pcg_next(U128 &state, U128 inc) {
  state = add128(mul128(state, U128{PCG_MULT_HI, PCG_MULT_LO}), inc);
  const unsigned long long x = state.hi ^ state.lo;
  const unsigned rot = (unsigned)(state.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int GEN_CHUNK = 64; // values per thread

// streams[s] = {state_hi, state_lo, inc_hi, inc_lo}; out[s * n + k] = value k of stream s
template <typename T>
__global__ void __launch_bounds__(256) uniform_kernel(const unsigned long long *__restrict__ streams, int n_streams,
                                                      long long n, double low, double range, double offset,
                                                      T *__restrict__ out) {
  const long long chunks = (n + GEN_CHUNK - 1) / GEN_CHUNK;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= chunks * n_streams) return;
  const int s = (int)(gid / chunks);
  const long long c = gid - (long long)s * chunks;
  U128 st{streams[4 * s], streams[4 * s + 1]};
  const U128 inc{streams[4 * s + 2], streams[4 * s + 3]};
  const long long k0 = c * GEN_CHUNK;
  st = pcg_advance(st, inc, (unsigned long long)k0);
  const long long k1 = k0 + GEN_CHUNK < n ? k0 + GEN_CHUNK : n;
  T *o = out + (size_t)s * (size_t)n;
  for (long long k = k0; k < k1; ++k) {
    const double u = (double)(pcg_next(st, inc) >> 11) * (1.0 / 9007199254740992.0);
    const double v = __dadd_rn(offset, __dadd_rn(low, __dmul_rn(range, u)));
    o[k] = (T)v;
  }
}

} // namespace ab
