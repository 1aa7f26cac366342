// Probe: is random-access throughput bound by DRAM or by per-SM outstanding
// misses?  Random 16-B loads over an L2-resident (32 MB) and an HBM (64 GB)
// footprint, .cg vs .nc, and 1/4/8 loads per 128-B line per lane.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int UNR, int NC, int PER>
__global__ void rd(const uint4 *base, uint64_t mask_lines, int iters, uint64_t seed, unsigned long long *sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = (seed ^ t) * 0x9E3779B97F4A7C15ull;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 v[UNR][PER];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      h = h * 6364136223846793005ull + 1442695040888963407ull;
      const uint4 *p = base + ((h >> 20) & mask_lines) * 8; // 128-B line
#pragma unroll
      for (int q = 0; q < PER; ++q) v[u][q] = NC ? __ldg(p + q * (8 / PER)) : __ldcg(p + q * (8 / PER));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int q = 0; q < PER; ++q) acc += v[u][q].x;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <typename K> static float timeit(K k) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k();
  cudaEventRecord(e0);
  k();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  const size_t bytes = 64ull << 30;
  uint4 *buf;
  unsigned long long *sink;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 8) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{");
  const char *sep = "";
  for (size_t fp : {(size_t)32 << 20, bytes}) {
    const uint64_t ml = fp / 128 - 1;
    const char *fn = fp < (1ull << 30) ? "L2" : "HBM";
    for (int bps : {1, 8}) {
      const int threads = 256, blocks = sms * bps, iters = 16;
      const double lanes = (double)threads * blocks * iters * 4;
      float ms;
      ms = timeit([&] { rd<4, 0, 1><<<blocks, threads>>>(buf, ml, iters, 1, sink); });
      printf("%s\"%s_cg_1per_b%d_Greq_s\": %.1f", sep, fn, bps, lanes / ms / 1e6); sep = ", ";
      ms = timeit([&] { rd<4, 1, 1><<<blocks, threads>>>(buf, ml, iters, 2, sink); });
      printf(", \"%s_nc_1per_b%d_Greq_s\": %.1f", fn, bps, lanes / ms / 1e6);
      ms = timeit([&] { rd<4, 0, 4><<<blocks, threads>>>(buf, ml, iters, 3, sink); });
      printf(", \"%s_cg_4per_b%d_Gline_s\": %.1f", fn, bps, lanes / ms / 1e6);
      ms = timeit([&] { rd<4, 0, 8><<<blocks, threads>>>(buf, ml, iters, 4, sink); });
      printf(", \"%s_cg_8per_b%d_Gline_s\": %.1f", fn, bps, lanes / ms / 1e6);
    }
  }
  printf("}\n");
  return 0;
}
