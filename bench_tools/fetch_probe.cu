// DRAM bytes moved per random access (run under ncu with dram__bytes_read.sum /
// dram__bytes_write.sum): how much of a 128-byte line a random 16/32/64-byte
// load (or CAS-128) really fetches, with each load flavour and each
// cudaLimitMaxL2FetchGranularity setting.  The decoder's token-table values,
// arc records and frontier-row reads are random 16-32 B accesses, so this
// factor multiplies most of its DRAM traffic.
//   kernel rd<W, MODE>: W bytes per access (W/16 x 16-B loads, W-aligned);
//   MODE 0 ld.global.cg, 1 ld.global.nc, 2 ld.global.cg with an L2 evict_first policy,
//   3 ld.global.relaxed.gpu (an L1-bypassing plain load), 4 atom.cas.b128.
// Each launch does 256 threads x 1184 CTAs x 64 accesses (19.4 M) over a
// 32 GB footprint.  Launch order: see the stdout lines.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 31; x *= 0x7fb5d329728ea185ull; x ^= x >> 27; x *= 0x81dadef4bc2dd44dull; x ^= x >> 33;
  return x;
}

template <int W, int MODE>
__global__ void rd(uint4 *base, uint64_t nslots, uint64_t seed, unsigned long long *sink) {
  constexpr int V = W / 16;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = mix(seed ^ t);
  unsigned acc = 0;
  for (int it = 0; it < 16; ++it) {
    uint4 v[4][V];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      h = h * 6364136223846793005ull + 1442695040888963407ull;
      uint4 *p = base + ((h >> 16) % nslots) * V;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (MODE == 0) v[u][k] = __ldcg(p + k);
        else if (MODE == 1) v[u][k] = __ldg(p + k);
        else if (MODE == 2) {
          uint4 r;
          uint64_t pol;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
          asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p + k), "l"(pol));
          v[u][k] = r;
        } else if (MODE == 3) {
          uint4 r;
          asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p + k));
          v[u][k] = r;
        } else {
          unsigned long long r0, r1, e0 = 0, e1 = 0, d0 = t, d1 = it;
          asm volatile("{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
                       " atom.global.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
                       : "=l"(r0), "=l"(r1) : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(p + k) : "memory");
          v[u][k] = make_uint4((unsigned)r0, (unsigned)r1, 0, 0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < V; ++k) acc += v[u][k].x;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int W, int MODE> static void run(uint4 *buf, size_t bytes, unsigned long long *sink, const char *what) {
  rd<W, MODE><<<1184, 256>>>(buf, bytes / W, 12345 + W * 7 + MODE, sink);
  cudaDeviceSynchronize();
  printf("launch rd<%d,%d> %s\n", W, MODE, what);
}

int main() {
  const size_t bytes = 32ull << 30;
  uint4 *buf;
  unsigned long long *sink;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 8) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  cudaDeviceSynchronize();
  size_t g0 = 0;
  cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity);
  printf("default L2 fetch granularity limit %zu\n", g0);
  run<16, 0>(buf, bytes, sink, "cg default");
  run<16, 1>(buf, bytes, sink, "nc default");
  run<16, 2>(buf, bytes, sink, "cg evict_first default");
  run<16, 3>(buf, bytes, sink, "relaxed.gpu default");
  run<16, 4>(buf, bytes, sink, "cas128 default");
  run<32, 0>(buf, bytes, sink, "cg 32B default");
  run<64, 0>(buf, bytes, sink, "cg 64B default");
  for (int g : {32, 64, 128}) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("set limit %d -> %s, reads back %zu\n", g, cudaGetErrorString(e), got);
    run<16, 0>(buf, bytes, sink, "cg");
    run<16, 1>(buf, bytes, sink, "nc");
    run<16, 4>(buf, bytes, sink, "cas128");
  }
  return 0;
}
