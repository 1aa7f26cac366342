// Random-access HBM ceiling on this GPU: the roofline the decoder's table and
// graph traffic actually runs against (random 32-byte sectors, not streaming).
//   read32   : random 32-B sector reads (ld.global.cg.v4 x2 of one sector)
//   read16   : random 16-B reads (one sector fetched per access)
//   cas16    : random 16-B CAS-128 (read-modify-write of one sector)
//   stream   : coalesced copy (the MEASURED_PEAKS-style streaming number)
// Footprint 64 GB (far above L2); each thread issues UNR independent accesses
// per iteration.  Prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

template <int UNR>
__global__ void read32(const uint4 *base, uint64_t nsec, int iters, uint64_t seed, unsigned long long *sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 v[UNR][2];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t s = mix(seed ^ (t * 1315423911ull + it * UNR + u)) % nsec;
      v[u][0] = __ldcg(base + 2 * s);
      v[u][1] = __ldcg(base + 2 * s + 1);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u][0].x ^ v[u][1].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int UNR>
__global__ void read16(const uint4 *base, uint64_t n16, int iters, uint64_t seed, unsigned long long *sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = __ldcg(base + mix(seed ^ (t * 2654435761ull + it * UNR + u)) % n16);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int UNR>
__global__ void cas16(uint4 *base, uint64_t n16, int iters, uint64_t seed, unsigned long long *sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned long long r0[UNR], r1[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t i = mix(seed ^ (t * 40503ull + it * UNR + u)) % n16;
      unsigned long long e0 = 0, e1 = 0, d0 = t, d1 = it;
      asm volatile("{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
                   " atom.global.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
                   : "=l"(r0[u]), "=l"(r1[u]) : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(base + i) : "memory");
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

int main() {
  const size_t bytes = 64ull << 30;
  uint4 *buf;
  unsigned long long *sink;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 0, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8, iters = 64;
  const uint64_t accesses = (uint64_t)threads * blocks * iters * 8;
  float ms;
  printf("{");
  // read32: sectors per second
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    read32<8><<<blocks, threads>>>(buf, bytes / 32, iters, 17 + rep, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"read32_GBps\": %.1f, \"read32_Gsectors_per_s\": %.2f, ", accesses * 32.0 / ms / 1e6, accesses / ms / 1e6);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    read16<8><<<blocks, threads>>>(buf, bytes / 16, iters, 29 + rep, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"read16_Gaccesses_per_s\": %.2f, ", accesses / ms / 1e6);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cas16<8><<<blocks, threads>>>(buf, bytes / 16, iters, 31 + rep, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"cas16_Gops_per_s\": %.2f, ", accesses / ms / 1e6);
  const uint64_t n = (8ull << 30) / 16;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    stream_copy<<<sms * 16, 512>>>(buf, buf + n, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"stream_copy_GBps\": %.1f, \"footprint_GB\": 64, \"threads\": %d}\n", 2.0 * n * 16 / ms / 1e6, threads * blocks);
  CK(cudaGetLastError());
  return 0;
}
