// Cost of the synchronisation a cluster channel (decode_kernel, Fmt16SC)
// does per pass, on this GPU: clusters of CL CTAs x 1024 threads, ITERS
// back-to-back operations, clock64 per operation:
//   bar_rel_acq  barrier.cluster.arrive.release + wait.acquire (csync)
//   bar_relaxed  barrier.cluster.arrive.relaxed + wait (no memory ordering)
//   fence_bar    fence.acq_rel.cluster + relaxed barrier
//   syncthreads  the CTA barrier
//   rem_atom     one warp-aggregated atomicAdd per warp on the leader's shared counter
//   rem_load     a load of the leader's shared counter (dependent chain)
// With and without outstanding global stores before each barrier (st).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_sync_probe cluster_sync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int ITERS = 2000;

template <int CL, int MODE, bool ST>
__global__ void __launch_bounds__(1024) k(long long *out, unsigned *gbuf) {
  __shared__ unsigned cnt;
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) cnt = 0;
  cl.sync();
  unsigned *lead = cl.map_shared_rank(&cnt, 0);
  unsigned acc = 0;
  const unsigned gid = (blockIdx.x * 1024 + threadIdx.x) * 33u;
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    if (ST) gbuf[(gid + i * 4099u) & ((1u << 24) - 1)] = i; // a scattered store in flight
    if (MODE == 0) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (MODE == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    } else if (MODE == 2) {
      asm volatile("fence.acq_rel.cluster;\n\tbarrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    } else if (MODE == 3) {
      __syncthreads();
    } else if (MODE == 4) {
      if ((threadIdx.x & 31) == 0) acc += atomicAdd(lead, 1u);
      __syncwarp();
    } else if (MODE == 5) {
      acc += *(volatile unsigned *)(lead + (acc & 0)) ;
    }
  }
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / ITERS + (acc == 0xFFFFFFFFu);
}

template <int CL, int MODE, bool ST> void run(const char *name, long long *d, unsigned *g, int clusters) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * clusters);
  cfg.blockDim = dim3(1024);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = CL;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k<CL, MODE, ST>, d, g);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * CL * clusters, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < CL * clusters; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("CL=%d clusters=%3d %-12s stores=%d  %6lld cycles/op  %s\n", CL, clusters, name, (int)ST, mx,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int CL> void all(long long *d, unsigned *g, int clusters) {
  run<CL, 0, false>("bar_rel_acq", d, g, clusters);
  run<CL, 0, true>("bar_rel_acq", d, g, clusters);
  run<CL, 1, false>("bar_relaxed", d, g, clusters);
  run<CL, 1, true>("bar_relaxed", d, g, clusters);
  run<CL, 2, true>("fence_bar", d, g, clusters);
  run<CL, 3, false>("syncthreads", d, g, clusters);
  run<CL, 3, true>("syncthreads", d, g, clusters);
  run<CL, 4, false>("rem_atom", d, g, clusters);
  run<CL, 5, false>("rem_load", d, g, clusters);
}

int main() {
  long long *d;
  unsigned *g;
  cudaMalloc(&d, 256 * sizeof(long long));
  cudaMalloc(&g, (1u << 24) * sizeof(unsigned));
  all<8>(d, g, 1);
  all<2>(d, g, 1);
  all<2>(d, g, 64);
  return 0;
}
