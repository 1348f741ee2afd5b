// Tensor-core VQ encoder for d = 128, d_sub = 8, m <= 256 (the 1-bit d8m256
// configuration) with bf16 / fp16 inputs.  Reference: vq.encode_rows (vq.py:226-232) ->
// assign_nearest (_ckernels.pyx:134-163): strict-< argmin of the squared
// distance over the centroids, lowest index on ties.
//
// One token row (16 groups x 8 dims) is one m16 tile: row r = group r.  The
// distance to centroid c is evaluated as d'(c) = |c|^2 - 2 x.c (|x|^2 is
// the same for every centroid) with m16n8k16 + m16n8k8 MMAs:
//   * A = -2x (exact in the input's 16-bit format),
//   * B = the centroids split into three 16-bit parts c = hi + mid + lo
//     (24 mantissa bits: the fp32 centroid exactly), K rows [hi; mid] in the
//     k16 MMA and lo in the k8 MMA,
//   * C = |c|^2 (fp32), so D = d'(c) with fp32 accumulation.
// The error of d' is ~2^-23 (|x|^2 + |c|^2): below the parity bound of
// SURVEY.md §8c (codes must match where the fp64 margin exceeds
// 1e-6 (|x|^2 + max|c|^2)).  A warp keeps the whole split codebook in
// registers (96 per lane), the norms come from 1 KB of shared memory
// (broadcast reads), and the warp streams token rows.
#include "common.cuh"

namespace antkv {

constexpr int EM_WARPS = 8;

template <bool BF16>
__device__ __forceinline__ uint32_t pack16(float a, float b) {
  if (BF16) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&v);
  }
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

template <bool BF16>
__device__ __forceinline__ float round16(float a) {
  return BF16 ? __bfloat162float(__float2bfloat16_rn(a)) : __half2float(__float2half_rn(a));
}

// hi / mid / lo 16-bit parts of (a, b): a = hi + mid + lo to fp32 precision
template <bool BF16>
__device__ __forceinline__ void split3(float a, float b, uint32_t &hi, uint32_t &mid, uint32_t &lo) {
  const float ah = round16<BF16>(a), bh = round16<BF16>(b);
  const float ar = a - ah, br = b - bh;
  const float am = round16<BF16>(ar), bm = round16<BF16>(br);
  hi = pack16<BF16>(ah, bh);
  mid = pack16<BF16>(am, bm);
  lo = pack16<BF16>(ar - am, br - bm);
}

template <bool BF16>
__device__ __forceinline__ void mma_k16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0,
                                        uint32_t b1) {
  if (BF16)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%4,%5}, {%6,%7}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%4,%5}, {%6,%7}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
}

template <bool BF16>
__device__ __forceinline__ void mma_k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  if (BF16)
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

__device__ __forceinline__ void store_code_any(void *codes, int64_t off, int code_bytes, int v) {
  if (code_bytes == 1) reinterpret_cast<uint8_t *>(codes)[off] = static_cast<uint8_t>(v);
  else if (code_bytes == 2) reinterpret_cast<uint16_t *>(codes)[off] = static_cast<uint16_t>(v);
  else if (code_bytes == 4) reinterpret_cast<int32_t *>(codes)[off] = v;
  else reinterpret_cast<int64_t *>(codes)[off] = v;
}

// grid = (ceil(rows / (EM_WARPS * tpw)), nsets); set s reads
// X + s * x_set_stride, codebook (s % cb_mod) and writes codes like
// launch_encode (tile / row strides).
template <bool BF16>
__global__ void __launch_bounds__(EM_WARPS * 32, 1)
vq_encode_mma_kernel(const uint16_t *__restrict__ X, int64_t rows, int64_t x_set_stride,
                     const float *__restrict__ codebooks, int cb_mod, int m,
                     void *__restrict__ codes, int code_bytes, int64_t code_set_stride,
                     int64_t code_tile_stride, int64_t code_row_stride, int tpw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int set = blockIdx.y;
  const float *cb = codebooks + (int64_t)(set % cb_mod) * m * 8;
  // |c|^2 per centroid in shared memory (+inf beyond m), the split codebook
  // in B-fragment order in registers
  __shared__ __align__(16) float snorm[256];
  for (int cc = threadIdx.x; cc < 256; cc += blockDim.x) {
    float s = INFINITY;
    if (cc < m) {
      const float4 p = *reinterpret_cast<const float4 *>(cb + cc * 8);
      const float4 q = *reinterpret_cast<const float4 *>(cb + cc * 8 + 4);
      s = p.x * p.x;
      s = fmaf(p.y, p.y, s);
      s = fmaf(p.z, p.z, s);
      s = fmaf(p.w, p.w, s);
      s = fmaf(q.x, q.x, s);
      s = fmaf(q.y, q.y, s);
      s = fmaf(q.z, q.z, s);
      s = fmaf(q.w, q.w, s);
    }
    snorm[cc] = s;
  }
  uint32_t bh[32], bm[32], bl[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int col = 8 * j + g;
    float c0 = 0.f, c1 = 0.f;
    if (col < m) {
      const float2 v = *reinterpret_cast<const float2 *>(cb + col * 8 + 2 * t);
      c0 = v.x;
      c1 = v.y;
    }
    split3<BF16>(c0, c1, bh[j], bm[j], bl[j]);
  }
  __syncthreads();
  const uint16_t *xs = X + set * x_set_stride;
  const int64_t r0 = ((int64_t)blockIdx.x * EM_WARPS + warp) * tpw;
  const int64_t r1 = min(rows, r0 + tpw);
  // A = -2 x: rows g / g+8 = groups, k = dims 2t, 2t+1 (exact scaling)
  const uint32_t neg2 = 0xC000C000u;   // (-2, -2): the same bits in bf16 and fp16
  uint32_t xa = 0, xb = 0;
  if (r0 < r1) {
    xa = *reinterpret_cast<const uint32_t *>(xs + r0 * 128 + g * 8 + 2 * t);
    xb = *reinterpret_cast<const uint32_t *>(xs + r0 * 128 + (g + 8) * 8 + 2 * t);
  }
  for (int64_t r = r0; r < r1; ++r) {
    uint32_t a0, a1;
    if (BF16) {
      __nv_bfloat162 p = __hmul2(*reinterpret_cast<__nv_bfloat162 *>(&xa),
                                 *reinterpret_cast<const __nv_bfloat162 *>(&neg2));
      __nv_bfloat162 q = __hmul2(*reinterpret_cast<__nv_bfloat162 *>(&xb),
                                 *reinterpret_cast<const __nv_bfloat162 *>(&neg2));
      a0 = *reinterpret_cast<uint32_t *>(&p);
      a1 = *reinterpret_cast<uint32_t *>(&q);
    } else {
      __half2 p = __hmul2(*reinterpret_cast<__half2 *>(&xa), *reinterpret_cast<const __half2 *>(&neg2));
      __half2 q = __hmul2(*reinterpret_cast<__half2 *>(&xb), *reinterpret_cast<const __half2 *>(&neg2));
      a0 = *reinterpret_cast<uint32_t *>(&p);
      a1 = *reinterpret_cast<uint32_t *>(&q);
    }
    if (r + 1 < r1) {   // prefetch the next token row
      xa = *reinterpret_cast<const uint32_t *>(xs + (r + 1) * 128 + g * 8 + 2 * t);
      xb = *reinterpret_cast<const uint32_t *>(xs + (r + 1) * 128 + (g + 8) * 8 + 2 * t);
    }
    float best0 = INFINITY, best1 = INFINITY;
    int bi0 = 0, bi1 = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float2 nn = *reinterpret_cast<const float2 *>(&snorm[8 * j + 2 * t]);
      float d[4] = {nn.x, nn.y, nn.x, nn.y};
      mma_k16<BF16>(d, a0, a1, bh[j], bm[j]);
      mma_k8<BF16>(d, a0, a1, bl[j]);
      // columns 8j + 2t (< 8j + 2t + 1): strict < keeps the lowest index
      if (d[0] < best0) { best0 = d[0]; bi0 = 8 * j + 2 * t; }
      if (d[1] < best0) { best0 = d[1]; bi0 = 8 * j + 2 * t + 1; }
      if (d[2] < best1) { best1 = d[2]; bi1 = 8 * j + 2 * t; }
      if (d[3] < best1) { best1 = d[3]; bi1 = 8 * j + 2 * t + 1; }
    }
    // reduce over the 4 lanes of a row: smaller distance, then lower index
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      const float ob0 = __shfl_xor_sync(0xffffffffu, best0, o);
      const int oi0 = __shfl_xor_sync(0xffffffffu, bi0, o);
      const float ob1 = __shfl_xor_sync(0xffffffffu, best1, o);
      const int oi1 = __shfl_xor_sync(0xffffffffu, bi1, o);
      if (ob0 < best0 || (ob0 == best0 && oi0 < bi0)) { best0 = ob0; bi0 = oi0; }
      if (ob1 < best1 || (ob1 == best1 && oi1 < bi1)) { best1 = ob1; bi1 = oi1; }
    }
    if (t == 0) {
      const int64_t base = set * code_set_stride + (r >> 4) * code_tile_stride + (r & 15) * code_row_stride;
      store_code_any(codes, base + g, code_bytes, bi0);
      store_code_any(codes, base + g + 8, code_bytes, bi1);
    }
  }
}

// Returns ANTKV_EUNSUPPORTED (nothing launched) when the configuration is not
// the tensor-core one; the caller then runs the exhaustive float32 encoder.
int launch_encode_mma(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride,
                      int nsets, const float *codebooks, int cb_mod, int m, int d_sub,
                      void *codes, int code_bytes, int64_t code_set_stride,
                      int64_t code_tile_stride, int64_t code_row_stride, const float *d2,
                      cudaStream_t st) {
  if (d != 128 || d_sub != 8 || m > 256 || m < 1 || d2 != nullptr) return ANTKV_EUNSUPPORTED;
  if (dtype != ANTKV_BF16 && dtype != ANTKV_F16) return ANTKV_EUNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(X) & 3) || (x_set_stride & 1) ||
      (reinterpret_cast<uintptr_t>(codebooks) & 15))
    return ANTKV_EUNSUPPORTED;
  if (rows == 0 || nsets == 0) return ANTKV_OK;
  // one wave of one 8-warp CTA per SM: CTAs per set = 148 / nsets, rows
  // split evenly over their warps (at least 16 per warp so the per-warp
  // codebook split stays amortised)
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t cps = nsets >= sms ? 1 : sms / nsets;
  int64_t tpw = (rows + cps * EM_WARPS - 1) / (cps * EM_WARPS);
  if (tpw < 16) tpw = 16;
  dim3 grid(ceil_div(rows, EM_WARPS * tpw), nsets);
  const uint16_t *Xh = reinterpret_cast<const uint16_t *>(X);
  if (dtype == ANTKV_BF16)
    vq_encode_mma_kernel<true><<<grid, EM_WARPS * 32, 0, st>>>(
        Xh, rows, x_set_stride, codebooks, cb_mod, m, codes, code_bytes, code_set_stride,
        code_tile_stride, code_row_stride, (int)tpw);
  else
    vq_encode_mma_kernel<false><<<grid, EM_WARPS * 32, 0, st>>>(
        Xh, rows, x_set_stride, codebooks, cb_mod, m, codes, code_bytes, code_set_stride,
        code_tile_stride, code_row_stride, (int)tpw);
  ANTKV_LAUNCH_CHECK("vq_encode_mma_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
