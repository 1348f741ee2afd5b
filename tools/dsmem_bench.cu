// Distributed-shared-memory gather bandwidth on B200 (decides whether a
// cluster-resident m = 4096 codebook can beat the L2 gathers of the staged
// decode kernel).  Clusters of C CTAs (one per SM, 128 KB of shared memory
// each); every warp gathers 64-byte centroids (4 lanes x 16 B, 8 centroids
// per instruction, as the staged kernel's d32 gathers) from random offsets of
// random CTAs of its cluster (ld.shared::cluster), or from its own CTA
// (local baseline).  Prints bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_bench tools/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int SMEM = 128 * 1024;

__global__ void gather_kernel(int iters, int remote, unsigned long long *cycles, uint32_t *sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int nblk = cl.num_blocks();
  for (int i = threadIdx.x; i < SMEM / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  cl.sync();
  const int lane = threadIdx.x & 31;
  uint32_t x = (blockIdx.x * 977 + threadIdx.x * 131 + 7) * 2654435761u;
  uint32_t acc = 0;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // 8 centroids per instruction: lanes 4c..4c+3 read centroid c's 64 bytes
    x = x * 1664525u + 1013904223u;
    const uint32_t cent = __shfl_sync(0xffffffffu, x, lane & ~3) >> 20;   // 0..4095: 64 B each... wrap to 128 KB
    const uint32_t off = ((cent & 2047) << 6) + (lane & 3) * 16;
    const int peer = remote ? (int)((__shfl_sync(0xffffffffu, x, lane & ~3) >> 8) % nblk) : (int)cl.block_rank();
    uint32_t addr = base + off, raddr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(addr), "r"(peer));
    uint32_t a0, a1, a2, a3;
    asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(raddr));
    acc += a0 ^ a1 ^ a2 ^ a3;
  }
  unsigned long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  int dev = 0;
  cudaSetDevice(dev);
  cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  unsigned long long *cyc;
  uint32_t *sink;
  cudaMalloc(&cyc, 1024 * sizeof(unsigned long long));
  cudaMalloc(&sink, 4);
  const int iters = 4096;
  for (int C : {1, 2, 4, 8}) {
    for (int remote : {0, 1}) {
      for (int threads : {256, 512}) {
        cudaLaunchConfig_t cfg = {};
        const int grid = (148 / C) * C;
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaLaunchKernelEx(&cfg, gather_kernel, iters, remote, cyc, sink);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, gather_kernel, iters, remote, cyc, sink);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[1024];
        cudaMemcpy(h, cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes_per_cta = (double)iters * threads * 16;
        printf("cluster %d remote %d threads %d: %s  %.1f B/clk/SM (max CTA cycles %.0f), %.1f GB/s total (%.3f ms)\n", C,
               remote, threads, cudaGetErrorString(err), bytes_per_cta / mx, mx, bytes_per_cta * grid / (ms * 1e6), ms);
      }
    }
  }
  return 0;
}
