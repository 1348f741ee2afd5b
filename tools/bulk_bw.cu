// Aggregate L2 -> shared-memory bulk-copy bandwidth: every CTA (one per SM)
// streams CHUNK-byte cp.async.bulk copies from an L2-resident buffer through
// a ring of S stages; prints TB/s for a few (CHUNK, S) combinations.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw tools/bulk_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void bw(const uint8_t *src, size_t src_bytes, int chunk, int stages, int iters, unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bar[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = src_bytes / chunk;
  size_t c = (size_t)blockIdx.x * 7919 % nchunks;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    if (it >= stages) {
      const uint32_t parity = ((it / stages) - 1) & 1;
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(&bar[s])), "r"(parity)
            : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm + (size_t)s * chunk)),
        "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(&bar[s]))
        : "memory");
    c = (c + 148) % nchunks;
  }
  for (int s = 0; s < stages; ++s) {
    const int last = iters - 1 - ((iters - 1 - s) % stages);
    if (last < 0) continue;
    const uint32_t parity = (last / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar[s])), "r"(parity)
          : "memory");
  }
  sink[blockIdx.x] = sm[0];
}

int main() {
  const size_t bytes = 64ull << 20;   // L2-resident working set
  uint8_t *src;
  unsigned long long *sink;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaMalloc(&sink, 8 * 1024);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int cfg[][2] = {{16384, 2}, {16384, 4}, {16384, 8}, {32768, 2}, {32768, 4}, {65536, 2}, {65536, 3}};
  for (auto &c : cfg) {
    const int chunk = c[0], stages = c[1], iters = 2000;
    const int smem = chunk * stages;
    cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bw<<<sms, 32, smem>>>(src, bytes, chunk, stages, 50, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bw<<<sms, 32, smem>>>(src, bytes, chunk, stages, iters, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double tbs = (double)sms * iters * chunk / (ms * 1e-3) / 1e12;
    printf("chunk %6d B x %d stages: %.2f TB/s (%.1f B/clk/SM at 1.9 GHz) %s\n", chunk, stages, tbs,
           tbs * 1e12 / sms / 1.9e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
