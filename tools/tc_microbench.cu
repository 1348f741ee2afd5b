// tcgen05.mma issue-rate microbenchmark on one SM: back-to-back kind::f16
// MMAs (M = 128, K = 16, fp32 accumulate) for N in {64, 128, 256}, A from
// shared memory or TMEM, B from shared memory; prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_microbench tools/tc_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int N, bool A_TMEM>
__global__ void bench(unsigned long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_addr;
  __shared__ __align__(8) unsigned long long bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_addr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_addr;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t a = desc(smem_u32(sm)), b = desc(smem_u32(sm + 32768));
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (A_TMEM)
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                "r"(tmem + 256 + 8 * k), "l"(b + 2 * k), "r"(idesc), "r"(1));
          else
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(a + 2 * k), "l"(b + 2 * k), "r"(idesc), "r"(1));
        }
      }
      __syncwarp();
    }
    if (lane == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    __syncwarp();
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
    unsigned long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool A_TMEM>
void run(const char *name) {
  unsigned long long *d, h;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  cudaFuncSetAttribute(bench<N, A_TMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  bench<N, A_TMEM><<<1, 128, 96 * 1024>>>(d, 10);
  bench<N, A_TMEM><<<1, 128, 96 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * 8.0);
  const double flop = 2.0 * 128 * N * 16;
  printf("%-24s N=%3d  %7.1f clk/MMA  %7.0f flop/clk  (%s)\n", name, N, per, flop / per,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, false>("A smem, B smem");
  run<128, false>("A smem, B smem");
  run<256, false>("A smem, B smem");
  run<64, true>("A tmem, B smem");
  run<128, true>("A tmem, B smem");
  run<256, true>("A tmem, B smem");
  return 0;
}
