// Random-access HBM ceiling on this GPU: the roofline the decoder's table and
// graph traffic runs against (random 32-byte sectors over a footprint far
// above L2), next to the streaming copy number MEASURED_PEAKS.json quotes.
//   read16 : random 16-B loads (one 32-B sector fetched per load)
//   cas16  : random 16-B CAS-128 (read-modify-write of one sector)
// Each thread keeps UNR independent accesses in flight; prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 31; x *= 0x7fb5d329728ea185ull; x ^= x >> 27; x *= 0x81dadef4bc2dd44dull; x ^= x >> 33;
  return x;
}

template <int UNR>
__global__ void read16(const uint4 *base, uint64_t mask, int iters, uint64_t seed, unsigned long long *sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = mix(seed ^ t);
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      h = h * 6364136223846793005ull + 1442695040888963407ull;
      v[u] = __ldcg(base + ((h >> 20) & mask));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int UNR>
__global__ void cas16(uint4 *base, uint64_t mask, int iters, uint64_t seed, unsigned long long *sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = mix(seed ^ t);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned long long r0[UNR], r1[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      h = h * 6364136223846793005ull + 1442695040888963407ull;
      uint4 *p = base + ((h >> 20) & mask);
      unsigned long long e0 = 0, e1 = 0, d0 = t, d1 = it;
      asm volatile("{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
                   " atom.global.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
                   : "=l"(r0[u]), "=l"(r1[u]) : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(p) : "memory");
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += r0[u] ^ r1[u];
  }
  if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

__global__ void stream_copy(const uint4 *a, uint4 *b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
}

template <typename K>
static float timeit(K k) {
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
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 8) != cudaSuccess) {
    printf("{\"error\": \"alloc\"}\n");
    return 1;
  }
  cudaMemset(buf, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t mask = bytes / 16 - 1;
  const int iters = 32;
  printf("{\"sector_bytes\": 32");
  for (int fp_gb : {1, 4, 16, 32, 64}) {
    const uint64_t fmask = ((uint64_t)fp_gb << 30) / 16 - 1;
    const int threads = 256, blocks = sms * 8;
    const double n = (double)threads * blocks * iters;
    float ms = timeit([&] { read16<4><<<blocks, threads>>>(buf, fmask, iters * 2, 7 + fp_gb, sink); });
    printf(", \"read16_%dGB_Gsect_s\": %.2f", fp_gb, n * 8 / ms / 1e6);
    ms = timeit([&] { cas16<4><<<blocks, threads>>>(buf, fmask, iters * 2, 9 + fp_gb, sink); });
    printf(", \"cas16_%dGB_Gop_s\": %.2f", fp_gb, n * 8 / ms / 1e6);
  }
  (void)mask;
  const uint64_t n = (8ull << 30) / 16;
  float ms = timeit([&] { stream_copy<<<sms * 16, 512>>>(buf, buf + n, n); });
  printf(", \"stream_copy_GBps\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
