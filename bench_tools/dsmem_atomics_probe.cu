// Which atomics are atomic on a peer CTA's shared memory (DSMEM) through a
// generic address (cooperative_groups map_shared_rank) on this GPU: 512
// threads of a 2-CTA cluster hit the leader's variables.  Found on sm_100:
// 64-bit atomicMin is not (the decode kernel keeps per-CTA minima instead).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
struct V {
  unsigned long long mn64, add64, cas64;
  unsigned int mn32, add32, or32, cas32;
  int mx32;
  unsigned long long c128[2];
};
__global__ void __cluster_dims__(2, 1, 1) k(V *out) {
  __shared__ V v;
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) {
    v.mn64 = ~0ull; v.add64 = 0; v.cas64 = 0; v.mn32 = ~0u; v.add32 = 0; v.or32 = 0; v.cas32 = 0; v.mx32 = -1;
    v.c128[0] = v.c128[1] = 0;
  }
  cl.sync();
  V *p = cl.map_shared_rank(&v, 0);
  const unsigned t = cl.block_rank() * blockDim.x + threadIdx.x; // 0..511
  atomicMin(&p->mn64, 1000000ull + (511 - t));
  atomicAdd(&p->add64, 1ull);
  atomicMin(&p->mn32, 1000u + (511 - t));
  atomicAdd(&p->add32, 1u);
  atomicOr(&p->or32, 1u << (t & 31));
  atomicMax(&p->mx32, (int)t);
  unsigned long long o = p->cas64, n;
  while ((n = atomicCAS(&p->cas64, o, o + 1)) != o) o = n;
  unsigned int o32 = p->cas32, n32;
  while ((n32 = atomicCAS(&p->cas32, o32, o32 + 1)) != o32) o32 = n32;
  unsigned long long e0 = p->c128[0], e1 = p->c128[1];
  while (true) { // 128-bit CAS increment of both halves
    unsigned long long r0, r1;
    asm volatile("{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
                 " atom.relaxed.cluster.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
                 : "=l"(r0), "=l"(r1) : "l"(e0), "l"(e1), "l"(e0 + 1), "l"(e1 + 2), "l"(&p->c128[0]) : "memory");
    if (r0 == e0 && r1 == e1) break;
    e0 = r0; e1 = r1;
  }
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) *out = v;
}
int main() {
  V *d, h;
  cudaMalloc(&d, sizeof(V));
  k<<<2, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, sizeof(V), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  printf("min64 %llu (want 1000000) add64 %llu (512) cas64 %llu (512)\n", h.mn64, h.add64, h.cas64);
  printf("min32 %u (want 1000) add32 %u (512) or32 %x (ffffffff) max32 %d (511) cas32 %u (512)\n", h.mn32, h.add32, h.or32, h.mx32, h.cas32);
  printf("cas128 %llu %llu (512 1024)\n", h.c128[0], h.c128[1]);
}
