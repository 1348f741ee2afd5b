// Tensor-core VQ encoder for sub-vectors of 16, 32 or 64 dims and any
// codebook size (config #3's d32m4096, d16m4096, d16m256 ...) with bf16 /
// fp16 inputs.  Reference: vq.encode_rows (vq.py:226-232) -> assign_nearest
// (_ckernels.pyx:134-163): strict-< argmin of the squared distance, lowest
// index on ties.  encode_mma.cu holds the d_sub = 8, m <= 256 variant whose
// split codebook fits in registers.
//
// A sub-vector is a GEMM row: D[row][c] = |c|^2 - 2 x.c over every centroid
// c, with m16n8k16 MMAs and float32 accumulation:
//   * A = -2 x (exact in the input's 16-bit format), k = the d_sub dims;
//   * B = the centroid split into three 16-bit parts hi + mid + lo (the fp32
//     centroid to 24 bits), three MMAs per k-step;
//   * C = |c|^2 (fp32; +inf beyond m).
// The error of D is ~2^-23 (|x|^2 + |c|^2), inside SURVEY §8c's parity bound.
// Each warp holds the A fragments of RT = 4 row tiles (64 sub-vectors); the
// CTA streams the codebook in 128-centroid chunks that its threads split into
// shared memory (rows padded to an odd number of 16-byte units, so the eight
// row addresses of an ldmatrix phase hit distinct bank groups); every B
// fragment loaded by ldmatrix feeds RT MMAs.  The running argmin lives in
// registers (rows g, g + 8 of each tile, columns 2t, 2t + 1 per lane).
#include <stdlib.h>

#include "common.cuh"

namespace antkv {

namespace {

constexpr int ET_WARPS = 8;
// 16-row tiles per warp: every B fragment feeds RT MMAs (8 measured best for
// d_sub = 32, 4 for 16 and 64)
__host__ __device__ constexpr int et_rt(int ds) { return ds == 32 ? 8 : 4; }
constexpr int ET_CN = 128;               // centroids per shared-memory chunk

template <bool BF16>
__device__ __forceinline__ uint32_t pk16(float a, float b) {
  if (BF16) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&v);
  }
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

template <bool BF16>
__device__ __forceinline__ float r16(float a) {
  return BF16 ? __bfloat162float(__float2bfloat16_rn(a)) : __half2float(__float2half_rn(a));
}

template <bool BF16>
__device__ __forceinline__ void mma16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if (BF16)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm2(uint32_t addr, uint32_t &r0, uint32_t &r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}

__device__ __forceinline__ void store_code_u(void *codes, int64_t off, int code_bytes, int v) {
  if (code_bytes == 1) reinterpret_cast<uint8_t *>(codes)[off] = static_cast<uint8_t>(v);
  else if (code_bytes == 2) reinterpret_cast<uint16_t *>(codes)[off] = static_cast<uint16_t>(v);
  else if (code_bytes == 4) reinterpret_cast<int32_t *>(codes)[off] = v;
  else reinterpret_cast<int64_t *>(codes)[off] = v;
}

// grid = (ceil(rows * G / (ET_WARPS * RT * 16)), nsets); set s reads
// X + s * x_set_stride, codebook (s % cb_mod) and writes the code of
// (row r, group g) at s * code_set_stride + (r / 16) * code_tile_stride +
// (r % 16) * code_row_stride + g (launch_encode's layout).
template <bool BF16, int DS>
__global__ void __launch_bounds__(ET_WARPS * 32, 1)
vq_encode_tc_kernel(const uint16_t *__restrict__ X, int64_t rows, int G, int64_t x_set_stride,
                    const float *__restrict__ codebooks, int cb_mod, int m, void *__restrict__ codes,
                    int code_bytes, int64_t code_set_stride, int64_t code_tile_stride,
                    int64_t code_row_stride) {
  constexpr int KS = DS / 16;                      // k16 steps per sub-vector
  constexpr int RT = et_rt(DS);                    // 16-row tiles per warp
  constexpr int UNITS = 3 * DS / 8;                // 16-byte units of a split centroid
  constexpr int PU = UNITS | 1;                    // padded to an odd count
  constexpr int PITCH = PU * 16;
  constexpr int CN = DS >= 64 ? ET_CN / 2 : ET_CN;   // static shared memory stays under 48 KB
  __shared__ __align__(16) uint8_t sb[CN * PITCH];
  __shared__ float snorm[CN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int set = blockIdx.y;
  const float *cb = codebooks + (int64_t)(set % cb_mod) * m * DS;
  const int64_t nsub = rows * G;
  const int64_t sv0 = ((int64_t)blockIdx.x * ET_WARPS + warp) * (RT * 16);
  const uint16_t *xs = X + set * x_set_stride;
  // A = -2 x for the warp's 4 row tiles (rows beyond the end are zero)
  uint32_t a[RT][KS][4];
#pragma unroll
  for (int rt = 0; rt < RT; ++rt) {
    const int64_t ra = sv0 + rt * 16 + g, rb = ra + 8;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k0 = 16 * ks + 2 * t;
      uint32_t v[4] = {0u, 0u, 0u, 0u};
      if (ra < nsub) {
        v[0] = *reinterpret_cast<const uint32_t *>(xs + ra * DS + k0);
        v[2] = *reinterpret_cast<const uint32_t *>(xs + ra * DS + k0 + 8);
      }
      if (rb < nsub) {
        v[1] = *reinterpret_cast<const uint32_t *>(xs + rb * DS + k0);
        v[3] = *reinterpret_cast<const uint32_t *>(xs + rb * DS + k0 + 8);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t neg2 = 0xC000C000u;   // (-2, -2): the same bits in bf16 and fp16
        if (BF16) {
          __nv_bfloat162 p = __hmul2(*reinterpret_cast<__nv_bfloat162 *>(&v[e]),
                                     *reinterpret_cast<const __nv_bfloat162 *>(&neg2));
          a[rt][ks][e] = *reinterpret_cast<uint32_t *>(&p);
        } else {
          __half2 p = __hmul2(*reinterpret_cast<__half2 *>(&v[e]), *reinterpret_cast<const __half2 *>(&neg2));
          a[rt][ks][e] = *reinterpret_cast<uint32_t *>(&p);
        }
      }
    }
  }
  float best[RT][2];
  int bidx[RT][2];
#pragma unroll
  for (int rt = 0; rt < RT; ++rt) {
    best[rt][0] = best[rt][1] = INFINITY;
    bidx[rt][0] = bidx[rt][1] = 0;
  }
  // ldmatrix lanes 0-7: centroids 8j + (lane & 7), chunk 2ks; lanes 8-15: chunk 2ks + 1
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sb)) + (lane & 7) * PITCH +
                         ((lane >> 3) & 1) * 16;
  // the chunk's fp32 centroids, one float4 (centroid cc, quad q) per
  // element e = tid + 256 k; the next chunk's are loaded during this one's MMAs
  constexpr int QPC = DS / 4;                              // quads per centroid
  constexpr int PFN = CN * QPC / (ET_WARPS * 32);          // float4 per thread
  static_assert(PFN * ET_WARPS * 32 == CN * QPC, "chunk split");
  float4 pf[PFN];
  auto load_chunk = [&](int base) {
#pragma unroll
    for (int k = 0; k < PFN; ++k) {
      const int e = threadIdx.x + k * ET_WARPS * 32, cc = e / QPC, q = e % QPC;
      pf[k] = base + cc < m ? __ldg(reinterpret_cast<const float4 *>(cb + (int64_t)(base + cc) * DS) + q)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  load_chunk(0);
  for (int c0 = 0; c0 < m; c0 += CN) {
    __syncthreads();   // the previous chunk is consumed
    // split into hi / mid / lo parts; |c|^2 from the same values (QPC adjacent
    // lanes hold one centroid: partial sums reduced across them)
#pragma unroll
    for (int k = 0; k < PFN; ++k) {
      const int e = threadIdx.x + k * ET_WARPS * 32, cc = e / QPC, q = e % QPC;
      const float x[4] = {pf[k].x, pf[k].y, pf[k].z, pf[k].w};
      uint32_t hi[2], mid[2], lo[2];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const float ah = r16<BF16>(x[2 * p]), bh = r16<BF16>(x[2 * p + 1]);
        const float ar = x[2 * p] - ah, br = x[2 * p + 1] - bh;
        const float am = r16<BF16>(ar), bm = r16<BF16>(br);
        hi[p] = pk16<BF16>(ah, bh);
        mid[p] = pk16<BF16>(am, bm);
        lo[p] = pk16<BF16>(ar - am, br - bm);
      }
      uint8_t *row = sb + cc * PITCH + 8 * q;   // part p at p * DS * 2 bytes
      *reinterpret_cast<uint2 *>(row) = make_uint2(hi[0], hi[1]);
      *reinterpret_cast<uint2 *>(row + DS * 2) = make_uint2(mid[0], mid[1]);
      *reinterpret_cast<uint2 *>(row + DS * 4) = make_uint2(lo[0], lo[1]);
      float nrm = x[0] * x[0];
      nrm = fmaf(x[1], x[1], nrm);
      nrm = fmaf(x[2], x[2], nrm);
      nrm = fmaf(x[3], x[3], nrm);
#pragma unroll
      for (int o = 1; o < QPC; o <<= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      if (q == 0) snorm[cc] = c0 + cc < m ? nrm : INFINITY;
    }
    __syncthreads();
    if (c0 + CN < m) load_chunk(c0 + CN);   // in flight during the MMAs below
    const int cn = min(CN, m - c0);
    for (int j = 0; j < (cn + 7) / 8; ++j) {
      float acc[RT][4];
      const float2 nn = *reinterpret_cast<const float2 *>(&snorm[8 * j + 2 * t]);
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) {
        acc[rt][0] = nn.x;
        acc[rt][1] = nn.y;
        acc[rt][2] = nn.x;
        acc[rt][3] = nn.y;
      }
#pragma unroll
      for (int p = 0; p < 3; ++p) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t b0, b1;
          ldsm2(sbase + j * 8 * PITCH + p * DS * 2 + ks * 32, b0, b1);
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) mma16<BF16>(acc[rt], a[rt][ks], b0, b1);
        }
      }
      const int col = c0 + 8 * j + 2 * t;
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) {   // columns in index order: strict < keeps the lowest
        if (acc[rt][0] < best[rt][0]) { best[rt][0] = acc[rt][0]; bidx[rt][0] = col; }
        if (acc[rt][1] < best[rt][0]) { best[rt][0] = acc[rt][1]; bidx[rt][0] = col + 1; }
        if (acc[rt][2] < best[rt][1]) { best[rt][1] = acc[rt][2]; bidx[rt][1] = col; }
        if (acc[rt][3] < best[rt][1]) { best[rt][1] = acc[rt][3]; bidx[rt][1] = col + 1; }
      }
    }
  }
  // reduce over the 4 lanes of a row: smaller distance, then lower index
  __shared__ uint32_t spk[ET_WARPS][RT * 16];   // 12-bit packing: the warp's codes by sub-vector
#pragma unroll
  for (int rt = 0; rt < RT; ++rt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float b = best[rt][h];
      int bi = bidx[rt][h];
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, b, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < b || (ob == b && oi < bi)) { b = ob; bi = oi; }
      }
      const int64_t sv = sv0 + rt * 16 + g + 8 * h;
      if (code_bytes == 3) {
        if (t == 0) spk[warp][rt * 16 + g + 8 * h] = static_cast<uint32_t>(bi);
        continue;
      }
      if (t == 0 && sv < nsub) {
        const int64_t r = sv / G;
        const int gg = static_cast<int>(sv - r * G);
        store_code_u(codes, set * code_set_stride + (r >> 4) * code_tile_stride + (r & 15) * code_row_stride + gg,
                     code_bytes, bi);
      }
    }
  }
  if (code_bytes == 3) {   // whole rows (G | RT * 16, so the warp's sub-vectors are RT * 16 / G rows,
    __syncwarp();          // up to 64 for d_sub = 32 with G = 2: lanes loop over them)
    for (int rr = lane; rr < RT * 16 / G && sv0 + rr * G < nsub; rr += 32) {
      const int64_t r = (sv0 + rr * G) / G;
      code_put_row(static_cast<uint8_t *>(codes), set * code_set_stride + (r >> 4) * code_tile_stride +
                   (r & 15) * code_row_stride, G, &spk[warp][rr * G], 3);
    }
  }
}

}  // namespace

// Returns ANTKV_EUNSUPPORTED (nothing launched) when the configuration is not
// one of this encoder's; the caller then tries the next encoder.
int launch_encode_tc(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride, int nsets,
                     const float *codebooks, int cb_mod, int m, int d_sub, void *codes, int code_bytes,
                     int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                     const float *d2, cudaStream_t st) {
  static int off = -1;   // ANTKV_NO_TC_ENC=1: the float32 exhaustive encoder instead (A/B timing)
  if (off < 0) {
    const char *e = getenv("ANTKV_NO_TC_ENC");
    off = e && e[0] == '1';
  }
  if (off || d2 != nullptr || m < 1 || (d_sub != 16 && d_sub != 32 && d_sub != 64) || d % d_sub != 0)
    return ANTKV_EUNSUPPORTED;
  if (dtype != ANTKV_BF16 && dtype != ANTKV_F16) return ANTKV_EUNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(X) & 3) || (x_set_stride & 1) || (reinterpret_cast<uintptr_t>(codebooks) & 15))
    return ANTKV_EUNSUPPORTED;
  if (rows == 0 || nsets == 0) return ANTKV_OK;
  const int G = d / d_sub;
  const int64_t per_cta = ET_WARPS * et_rt(d_sub) * 16;
  dim3 grid(ceil_div(rows * G, per_cta), nsets);
  const uint16_t *Xh = reinterpret_cast<const uint16_t *>(X);
#define ET_LAUNCH(BF, DSV)                                                                           \
  vq_encode_tc_kernel<BF, DSV><<<grid, ET_WARPS * 32, 0, st>>>(Xh, rows, G, x_set_stride, codebooks, \
                                                               cb_mod, m, codes, code_bytes,        \
                                                               code_set_stride, code_tile_stride,   \
                                                               code_row_stride)
  const bool bf = dtype == ANTKV_BF16;
  if (d_sub == 16) { if (bf) ET_LAUNCH(true, 16); else ET_LAUNCH(false, 16); }
  else if (d_sub == 32) { if (bf) ET_LAUNCH(true, 32); else ET_LAUNCH(false, 32); }
  else { if (bf) ET_LAUNCH(true, 64); else ET_LAUNCH(false, 64); }
#undef ET_LAUNCH
  ANTKV_LAUNCH_CHECK("vq_encode_tc_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
