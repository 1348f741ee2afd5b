// TMA gather throughput on B200: can `cp.async.bulk.tensor.2d ... tile::gather4`
// (4 arbitrary 64-byte rows of an L2-resident codebook per request, written to
// shared memory by the TMA engine, off the LSU pipe) feed the staged decode
// kernel's m = 4096 centroid gathers faster than per-lane cp.async?
// Each warp's elected lane streams random requests through an 8-slot ring
// (one mbarrier per slot); rows per clock per SM are reported for
//   gather4 (4 rows / request), 1D cp.async.bulk (1 row / request),
//   per-lane cp.async 16 B (the staged kernel's current gather, 8 rows / instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather4_bench tools/gather4_bench.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>

#ifndef SLOTS_N
#define SLOTS_N 8
#endif
constexpr int ROWS = 8192, ROWB = 64, SLOTS = SLOTS_N;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void gather_kernel(const __grid_constant__ CUtensorMap map, const uint8_t *table, int iters,
                              unsigned long long *cycles, uint32_t *sink) {
  __shared__ __align__(128) uint8_t ring[8][SLOTS][256];
  __shared__ __align__(8) unsigned long long bar[8][SLOTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int s = 0; s < SLOTS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t x = (blockIdx.x * 7919u + warp * 104729u + 12345u) * 2654435761u;
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % SLOTS;
    if (MODE == 2) {   // per-lane cp.async: 32 lanes x 16 B = 8 rows
      x = x * 1664525u + 1013904223u;
      const uint32_t row = __shfl_sync(0xffffffffu, x >> 13, lane & ~3) & (ROWS - 1);
      const uint8_t *src = table + (size_t)row * ROWB + (lane & 3) * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(&ring[warp][s][0]) + ((lane * 16) & 255)),
                   "l"(src));
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group %0;" ::"n"(SLOTS - 2));
      continue;
    }
    if (lane == 0) {
      if (it >= SLOTS) {   // slot reuse: wait for its previous fill
        const uint32_t ph = ((it / SLOTS) - 1) & 1;
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                     ::"r"(su32(&bar[warp][s])), "r"(ph) : "memory");
        acc += ring[warp][s][it & 63];
      }
      x = x * 1664525u + 1013904223u;
      if (MODE == 0) {
        const int r0 = (x >> 3) & (ROWS - 1), r1 = (x >> 7) & (ROWS - 1), r2 = (x >> 11) & (ROWS - 1),
                  r3 = (x >> 15) & (ROWS - 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp][s])), "r"(256)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5, %6}], [%7];" ::"r"(su32(&ring[warp][s][0])),
            "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&bar[warp][s]))
            : "memory");
      } else {
        const int r0 = (x >> 3) & (ROWS - 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp][s])), "r"(ROWB)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(&ring[warp][s][0])),
            "l"(table + (size_t)r0 * ROWB), "r"(ROWB), "r"(su32(&bar[warp][s]))
            : "memory");
      }
    }
    __syncwarp();
  }
  if (MODE == 2) asm volatile("cp.async.wait_all;");
  if (MODE != 2 && lane == 0)
    for (int k = 0; k < SLOTS; ++k) {   // drain
      const int it = iters - SLOTS + k, s = it % SLOTS;
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                   ::"r"(su32(&bar[warp][s])), "r"((uint32_t)((it / SLOTS) & 1)) : "memory");
    }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345u) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint8_t *table;
  cudaMalloc(&table, (size_t)ROWS * ROWB);
  cudaMemset(table, 1, (size_t)ROWS * ROWB);
  unsigned long long *cyc;
  uint32_t *sink;
  cudaMalloc(&cyc, 1024 * sizeof(unsigned long long));
  cudaMalloc(&sink, 4);
  CUtensorMap map;
  cuuint64_t dims[2] = {32, ROWS};            // fp16 columns, rows
  cuuint64_t strides[1] = {ROWB};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, table, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map encode: %d\n", (int)r);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {1, 2, 4, 8}) {
      void (*k)(const CUtensorMap, const uint8_t *, int, unsigned long long *, uint32_t *) =
          mode == 0 ? gather_kernel<0> : mode == 1 ? gather_kernel<1> : gather_kernel<2>;
      k<<<148, 32 * warps>>>(map, table, iters, cyc, sink);   // warm-up (L2)
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<148, 32 * warps>>>(map, table, iters, cyc, sink);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double rows_per_req = mode == 0 ? 4 : mode == 1 ? 1 : 8;
      const double rows = (double)iters * warps * rows_per_req;
      printf("%-10s warps %d: %s  %.3f rows/clk/SM  (%.1f clk per request per SM, %.3f ms)\n",
             mode == 0 ? "gather4" : mode == 1 ? "bulk1d" : "cp.async", warps, cudaGetErrorString(e), rows / mx,
             mx / ((double)iters * warps), ms);
    }
  }
  return 0;
}
