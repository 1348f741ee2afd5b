// Tensor-core prefill kernels (d = 128): blocked online-softmax attention with
// the (O, L, M) auxiliaries (attention.py:146-169, _ckernels.pyx:10-88) and
// the Alg. 1 anchor-score column sums (anchors.py:66-87,
// _ckernels.pyx:91-131), on mma.sync m16n8k16.
//
// Numerics.  Anchor sets must match the float64 reference wherever the budget
// boundary margin exceeds ~1e-4 relative and M / L / O must
// meet the reference's own 1e-4 / 1e-5 checks, so every product is formed
// from two-part splits with float32 accumulation (a.b = ah.bh + ah.bl +
// al.bh, ~2^-22 relative for fp16 parts, ~2^-16 for bf16):
//   * S = Qs.Kr^T from fp16 parts.  fp16 has no exponent headroom, so the Q
//     rows of a warp and each 64-row K tile are first scaled by a power of two
//     that puts their largest magnitude in [2^13, 2^14) (the lo parts stay
//     normal; the tensor cores flush fp16 subnormals); the accumulator is
//     scaled back exactly.
//   * P.V from bf16 parts (P <= 1 and V need no range handling in bf16).
// M, L and the AnS sums are float32.

// Inputs are the rotated float32 rows the reference FFI works on: Qs [heads]
// [n_q][128] (pre-scaled by 1/sqrt(d)), Kr / V [kv_heads][n_k][128].
#include "common.cuh"

namespace antkv {

constexpr int PM_WARPS = 4;
constexpr int PM_THREADS = 32 * PM_WARPS;
constexpr int PM_B = 64;   // rows per block (queries or keys)

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t bf2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}
__device__ __forceinline__ void split_bf(float a, float b, uint32_t &hi, uint32_t &lo) {
  const float ah = __bfloat162float(__float2bfloat16_rn(a));
  const float bh = __bfloat162float(__float2bfloat16_rn(b));
  hi = bf2(ah, bh);
  lo = bf2(a - ah, b - bh);
}
// Power of two that maps the magnitude mx into [2^13, 2^14) (1 for mx == 0).
__device__ __forceinline__ float pow2_scale(float mx) {
  if (!(mx > 0.f)) return 1.f;
  int e = (__float_as_int(mx) >> 23) & 0xff;   // biased exponent
  e = e < 14 ? 14 : (e > 266 ? 266 : e);
  return __int_as_float((267 - e) << 23);
}
__device__ __forceinline__ uint32_t hf2(float a, float b) {
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}
// (a, b) -> fp16x2 hi and lo parts (a = hi + lo to ~2^-22 relative)
__device__ __forceinline__ void split_hf(float a, float b, uint32_t &hi, uint32_t &lo) {
  const float ah = __half2float(__float2half_rn(a));
  const float bh = __half2float(__float2half_rn(b));
  hi = hf2(ah, bh);
  lo = hf2(a - ah, b - bh);
}

// Byte offset of (row, 16-byte chunk) in a [64][128] 16-bit tile, chunks
// XOR-swizzled by row & 7 so ldmatrix phases are conflict-free.
__device__ __forceinline__ uint32_t tile_off(int row, int chunk) {
  return row * 256 + ((chunk ^ (row & 7)) << 4);
}

// Cooperative load of rows [r0, r0 + 64) of a [rows][128] float32 matrix
// into hi / lo tiles (zero beyond `rows`): fp16 parts of x * scale (FP16), or
// bf16 parts of x.
template <bool FP16>
__device__ __forceinline__ void load_split_tile(uint8_t *hi, uint8_t *lo, const float *__restrict__ src,
                                                int r0, int rows, float scale) {
  for (int e = threadIdx.x; e < PM_B * 32; e += PM_THREADS) {   // 4-float units
    const int r = e >> 5, c4 = e & 31;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r0 + r < rows) v = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)(r0 + r) * 128) + c4);
    uint32_t h0, l0, h1, l1;
    if (FP16) {
      split_hf(v.x * scale, v.y * scale, h0, l0);
      split_hf(v.z * scale, v.w * scale, h1, l1);
    } else {
      split_bf(v.x, v.y, h0, l0);
      split_bf(v.z, v.w, h1, l1);
    }
    const uint32_t off = tile_off(r, c4 >> 1) + (c4 & 1) * 8;
    *reinterpret_cast<uint2 *>(hi + off) = make_uint2(h0, h1);
    *reinterpret_cast<uint2 *>(lo + off) = make_uint2(l0, l1);
  }
}

// Largest |x| over rows [r0, r0 + 64) of a [rows][128] matrix (block-wide,
// `red` = 4 floats of shared scratch).
__device__ __forceinline__ float tile_absmax(const float *__restrict__ src, int r0, int rows, float *red) {
  float mx = 0.f;
  for (int e = threadIdx.x; e < PM_B * 32; e += PM_THREADS) {
    const int r = e >> 5, c4 = e & 31;
    if (r0 + r < rows) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)(r0 + r) * 128) + c4);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
  mx = warp_max(mx);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  return fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
}

// ---------------------------------------------------------------- FA + aux
// CTA = (head, 64 queries); warp w owns queries 16w..16w+15 (Q fragments in
// registers), loops over 64-key blocks.
__global__ void __launch_bounds__(PM_THREADS)
flash_mma_kernel(const float *__restrict__ Qs, const float *__restrict__ Kr, const float *__restrict__ V,
                 int group, int n_q, int n_k, int causal, float *__restrict__ O,
                 float *__restrict__ Lout, float *__restrict__ Mout) {
  extern __shared__ __align__(128) uint8_t fsm[];   // K hi, K lo, V hi, V lo tiles
  uint8_t *sKh = fsm, *sKl = fsm + PM_B * 256, *sVh = fsm + 2 * PM_B * 256, *sVl = fsm + 3 * PM_B * 256;
  __shared__ float red[4];
  const int h = blockIdx.y, q0 = blockIdx.x * PM_B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const float *Qh = Qs + (int64_t)h * n_q * 128;
  const float *Kh = Kr + (int64_t)(h / group) * n_k * 128;
  const float *Vh = V + (int64_t)(h / group) * n_k * 128;
  const int qa = q0 + 16 * warp + g, qb = qa + 8;   // this lane's two query rows
  // Q fragments (fp16 hi / lo of the warp-scaled rows) for 8 k-steps
  uint32_t qh[8][4], ql[8][4];
  float sQ;
  {
    float2 v[8][4];
    float mx = 0.f;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[s][e] = make_float2(0.f, 0.f);
      if (qa < n_q) {
        v[s][0] = *reinterpret_cast<const float2 *>(Qh + (int64_t)qa * 128 + 16 * s + 2 * t);
        v[s][2] = *reinterpret_cast<const float2 *>(Qh + (int64_t)qa * 128 + 16 * s + 8 + 2 * t);
      }
      if (qb < n_q) {
        v[s][1] = *reinterpret_cast<const float2 *>(Qh + (int64_t)qb * 128 + 16 * s + 2 * t);
        v[s][3] = *reinterpret_cast<const float2 *>(Qh + (int64_t)qb * 128 + 16 * s + 8 + 2 * t);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fmaxf(fabsf(v[s][e].x), fabsf(v[s][e].y)));
    }
    sQ = pow2_scale(warp_max(mx));
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int e = 0; e < 4; ++e) split_hf(v[s][e].x * sQ, v[s][e].y * sQ, qh[s][e], ql[s][e]);
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[i][e] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const float log2e = 1.4426950408889634f;
  const int q_last = min(q0 + PM_B, n_q) - 1;
  // ldmatrix lane addressing
  const int kb_row = (lane & 7) + 8 * (lane >> 4), kb_chunk = (lane >> 3) & 1;   // K (B operand)
  const int vb_row = (lane & 7) + 8 * ((lane >> 3) & 1), vb_chunk = lane >> 4;   // V (B, .trans)
  for (int k0 = 0; k0 < n_k; k0 += PM_B) {
    if (causal && k0 > q_last) break;
    const float sK = pow2_scale(tile_absmax(Kh, k0, n_k, red));   // (synchronises the block)
    load_split_tile<true>(sKh, sKl, Kh, k0, n_k, sK);
    load_split_tile<false>(sVh, sVl, Vh, k0, n_k, 1.f);
    __syncthreads();
    const float unscale = 1.f / (sQ * sK);
    float sc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[i][e] = 0.f;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {   // key n-tiles 2np, 2np+1
        uint32_t bh[4], bl[4];
        const uint32_t off = tile_off(16 * np + kb_row, 2 * s + kb_chunk);
        ldsm4(smem_addr(sKh) + off, bh);
        ldsm4(smem_addr(sKl) + off, bl);
        mma_f16(sc[2 * np], qh[s], bh[0], bh[1]);
        mma_f16(sc[2 * np], qh[s], bl[0], bl[1]);
        mma_f16(sc[2 * np], ql[s], bh[0], bh[1]);
        mma_f16(sc[2 * np + 1], qh[s], bh[2], bh[3]);
        mma_f16(sc[2 * np + 1], qh[s], bl[2], bl[3]);
        mma_f16(sc[2 * np + 1], ql[s], bh[2], bh[3]);
      }
    }
    // mask (causal / tails) and online softmax over this block
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + 8 * i + 2 * t + (e & 1);
        const int qi = (e < 2) ? qa : qb;
        const bool ok = key < n_k && qi < n_q && (!causal || key <= qi);
        sc[i][e] = ok ? sc[i][e] * unscale : -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], sc[i][e]);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float al[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float mn = fmaxf(m[r], mx[r]);
      al[r] = (m[r] == -INFINITY) ? 0.f : exp2f((m[r] - mn) * log2e);
      m[r] = mn;
      l[r] *= al[r];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= al[0];
      o[i][1] *= al[0];
      o[i][2] *= al[1];
      o[i][3] *= al[1];
    }
    // P (bf16 hi / lo A fragments for 4 key k-steps)
    uint32_t ph[4][4], pl[4][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mr = m[e >> 1];
        p[e] = (sc[i][e] == -INFINITY) ? 0.f : exp2f((sc[i][e] - mr) * log2e);
        l[e >> 1] += p[e];
      }
      // n-tile i covers keys 8i..8i+7 = k-step i/2, half i&1
      split_bf(p[0], p[1], ph[i >> 1][(i & 1) * 2 + 0], pl[i >> 1][(i & 1) * 2 + 0]);   // row g
      split_bf(p[2], p[3], ph[i >> 1][(i & 1) * 2 + 1], pl[i >> 1][(i & 1) * 2 + 1]);   // row g+8
    }
    // O += P . V  (bf16 splits: Ph.Vh + Ph.Vl + Pl.Vh)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {   // dim n-tiles 2dp, 2dp+1
        uint32_t vh[4], vl[4];
        const uint32_t off = tile_off(16 * ks + vb_row, 2 * dp + vb_chunk);
        ldsm4_t(smem_addr(sVh) + off, vh);
        ldsm4_t(smem_addr(sVl) + off, vl);
        mma_bf16(o[2 * dp], ph[ks], vh[0], vh[1]);
        mma_bf16(o[2 * dp], ph[ks], vl[0], vl[1]);
        mma_bf16(o[2 * dp], pl[ks], vh[0], vh[1]);
        mma_bf16(o[2 * dp + 1], ph[ks], vh[2], vh[3]);
        mma_bf16(o[2 * dp + 1], ph[ks], vl[2], vl[3]);
        mma_bf16(o[2 * dp + 1], pl[ks], vh[2], vh[3]);
      }
    }
  }
  // finish: L = sum over the row (4 lanes), O / L
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
  const float inv0 = l[0] > 0.f ? 1.f / l[0] : 0.f, inv1 = l[1] > 0.f ? 1.f / l[1] : 0.f;
  float *Oh = O + (int64_t)h * n_q * 128;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (qa < n_q)
      *reinterpret_cast<float2 *>(Oh + (int64_t)qa * 128 + 8 * i + 2 * t) =
          make_float2(o[i][0] * inv0, o[i][1] * inv0);
    if (qb < n_q)
      *reinterpret_cast<float2 *>(Oh + (int64_t)qb * 128 + 8 * i + 2 * t) =
          make_float2(o[i][2] * inv1, o[i][3] * inv1);
  }
  if (t == 0) {
    if (qa < n_q) {
      Lout[(int64_t)h * n_q + qa] = l[0];
      Mout[(int64_t)h * n_q + qa] = m[0];
    }
    if (qb < n_q) {
      Lout[(int64_t)h * n_q + qb] = l[1];
      Mout[(int64_t)h * n_q + qb] = m[1];
    }
  }
}

// ---------------------------------------------------------------- AnS
// CTA = (output head, 64 keys); warp w owns keys 16w..16w+15 as the A operand
// (S^T = K.Q^T), loops over the sum_group query heads and the query blocks
// (from the key block on when causal); per lane the column sums of its two
// keys accumulate over its query columns, reduced over the 4 lanes at the end.
__global__ void __launch_bounds__(PM_THREADS)
ans_mma_kernel(const float *__restrict__ Qs, const float *__restrict__ Kr, const float *__restrict__ Mv,
               const float *__restrict__ Lv, const float *__restrict__ qn, int group, int sum_group,
               int n_q, int n_k, int causal, float *__restrict__ ans_k, float *__restrict__ ans_v) {
  __shared__ __align__(128) uint8_t sQh[PM_B * 256], sQl[PM_B * 256];
  __shared__ float sM[PM_B], sIL[PM_B], sQN[PM_B], red[4];
  const int ho = blockIdx.y, k0 = blockIdx.x * PM_B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ka = k0 + 16 * warp + g, kb = ka + 8;   // this lane's two keys
  const int qb_row = (lane & 7) + 8 * (lane >> 4), qb_chunk = (lane >> 3) & 1;
  const float log2e = 1.4426950408889634f;
  float sv[2] = {0.f, 0.f}, sk[2] = {0.f, 0.f};
  for (int gq = 0; gq < sum_group; ++gq) {
    const int h = ho * sum_group + gq, hk = h / group;
    const float *Qh = Qs + (int64_t)h * n_q * 128;
    const float *Kh = Kr + (int64_t)hk * n_k * 128;
    uint32_t kh[8][4], kl[8][4];
    float sKw;
    {
      float2 v[8][4];
      float mx = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[s][e] = make_float2(0.f, 0.f);
        if (ka < n_k) {
          v[s][0] = *reinterpret_cast<const float2 *>(Kh + (int64_t)ka * 128 + 16 * s + 2 * t);
          v[s][2] = *reinterpret_cast<const float2 *>(Kh + (int64_t)ka * 128 + 16 * s + 8 + 2 * t);
        }
        if (kb < n_k) {
          v[s][1] = *reinterpret_cast<const float2 *>(Kh + (int64_t)kb * 128 + 16 * s + 2 * t);
          v[s][3] = *reinterpret_cast<const float2 *>(Kh + (int64_t)kb * 128 + 16 * s + 8 + 2 * t);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fmaxf(fabsf(v[s][e].x), fabsf(v[s][e].y)));
      }
      sKw = pow2_scale(warp_max(mx));
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int e = 0; e < 4; ++e) split_hf(v[s][e].x * sKw, v[s][e].y * sKw, kh[s][e], kl[s][e]);
    }
    const int qstart = causal ? (k0 / PM_B) * PM_B : 0;
    for (int q0 = qstart; q0 < n_q; q0 += PM_B) {
      const float sQt = pow2_scale(tile_absmax(Qh, q0, n_q, red));   // (synchronises the block)
      load_split_tile<true>(sQh, sQl, Qh, q0, n_q, sQt);
      const float unscale = 1.f / (sKw * sQt);
      for (int i = threadIdx.x; i < PM_B; i += PM_THREADS) {
        const int qi = q0 + i;
        const bool ok = qi < n_q;
        sM[i] = ok ? Mv[(int64_t)h * n_q + qi] : 0.f;
        sIL[i] = ok ? 1.f / Lv[(int64_t)h * n_q + qi] : 0.f;
        sQN[i] = ok ? qn[(int64_t)h * n_q + qi] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int np = 0; np < 4; ++np) {   // query n-tiles 2np, 2np+1
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          uint32_t bh[4], bl[4];
          const uint32_t off = tile_off(16 * np + qb_row, 2 * s + qb_chunk);
          ldsm4(smem_addr(sQh) + off, bh);
          ldsm4(smem_addr(sQl) + off, bl);
          mma_f16(sc[0], kh[s], bh[0], bh[1]);
          mma_f16(sc[0], kh[s], bl[0], bl[1]);
          mma_f16(sc[0], kl[s], bh[0], bh[1]);
          mma_f16(sc[1], kh[s], bh[2], bh[3]);
          mma_f16(sc[1], kh[s], bl[2], bl[3]);
          mma_f16(sc[1], kl[s], bh[2], bh[3]);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int col = 16 * np + 8 * j + 2 * t + (e & 1);   // query within the block
            const int qi = q0 + col;
            const int key = (e < 2) ? ka : kb;
            if (qi < n_q && key < n_k && (!causal || key <= qi)) {
              const float a = exp2f((sc[j][e] * unscale - sM[col]) * log2e) * sIL[col];
              sv[e >> 1] += a;
              sk[e >> 1] = fmaf(a * (1.f - a), sQN[col], sk[e >> 1]);
            }
          }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    sv[r] += __shfl_xor_sync(0xffffffffu, sv[r], 1);
    sv[r] += __shfl_xor_sync(0xffffffffu, sv[r], 2);
    sk[r] += __shfl_xor_sync(0xffffffffu, sk[r], 1);
    sk[r] += __shfl_xor_sync(0xffffffffu, sk[r], 2);
  }
  if (t == 0) {
    if (ka < n_k) {
      ans_v[(int64_t)ho * n_k + ka] = sv[0];
      ans_k[(int64_t)ho * n_k + ka] = sk[0];
    }
    if (kb < n_k) {
      ans_v[(int64_t)ho * n_k + kb] = sv[1];
      ans_k[(int64_t)ho * n_k + kb] = sk[1];
    }
  }
}

int launch_flash_mma(const float *Qs, const float *Kr, const float *V, int heads, int kv_heads,
                     int n_q, int n_k, int d, int dv, int causal, float *O, float *L, float *M,
                     cudaStream_t st) {
  if (d != 128 || dv != 128) return ANTKV_EUNSUPPORTED;
  if (n_q == 0) return ANTKV_OK;
  dim3 grid(ceil_div(n_q, PM_B), heads);
  const int smem = 4 * PM_B * 256;
  cudaFuncSetAttribute(flash_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  flash_mma_kernel<<<grid, PM_THREADS, smem, st>>>(Qs, Kr, V, heads / kv_heads, n_q, n_k, causal, O, L, M);
  ANTKV_LAUNCH_CHECK("flash_mma_kernel");
  return ANTKV_OK;
}

int launch_ans_mma(const float *Qs, const float *Kr, const float *M, const float *L, const float *qn,
                   int heads, int kv_heads, int sum_group, int n_q, int n_k, int d, int causal,
                   float *ans_k, float *ans_v, cudaStream_t st) {
  if (d != 128) return ANTKV_EUNSUPPORTED;
  if (n_k == 0) return ANTKV_OK;
  dim3 grid(ceil_div(n_k, PM_B), heads / sum_group);
  ans_mma_kernel<<<grid, PM_THREADS, 0, st>>>(Qs, Kr, M, L, qn, heads / kv_heads, sum_group, n_q, n_k,
                                              causal, ans_k, ans_v);
  ANTKV_LAUNCH_CHECK("ans_mma_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
