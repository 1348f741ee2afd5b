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
//
// Inputs are the rotated float32 rows the reference FFI works on: Qs [heads]
// [n_q][128] (pre-scaled by 1/sqrt(d)), Kr / V [kv_heads][n_k][128].  The
// operand tiles are split once (presplit_kernel) and streamed by bulk copies
// through two-stage shared-memory pipelines.
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

// ---------------------------------------------------------------- pre-split tiles
// Every K / V / Q tile is split once (presplit_kernel) into the swizzled
// 16-bit layout the MMAs read, [rows/64][hi 16 KB | lo 16 KB] (+ one
// power-of-two scale per fp16 tile); the attention kernels then stream tiles
// with bulk copies through a two-stage shared-memory pipeline instead of
// re-converting every tile in every CTA.
constexpr int PM_TILE = 2 * PM_B * 256;   // hi + lo bytes of one tile

__device__ __forceinline__ void pm_mbar_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void pm_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void pm_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void pm_wait(unsigned long long *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void pm_bulk(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// X [heads][rows][128] fp32 -> tiles [heads][ceil(rows/64)][hi | lo] (fp16 of
// x * scale with scale[heads][tiles] when FP16, else bf16 parts of x).
template <bool FP16>
__global__ void __launch_bounds__(PM_THREADS)
presplit_kernel(const float *__restrict__ X, int rows, uint8_t *__restrict__ tiles, float *__restrict__ scales) {
  __shared__ float red[4];
  const int h = blockIdx.y, tile = blockIdx.x, nt = gridDim.x;
  const float *src = X + (int64_t)h * rows * 128;
  uint8_t *dst = tiles + ((int64_t)h * nt + tile) * PM_TILE;
  float sc = 1.f;
  if (FP16) {
    sc = pow2_scale(tile_absmax(src, tile * PM_B, rows, red));
    if (threadIdx.x == 0) scales[(int64_t)h * nt + tile] = sc;
  }
  for (int e = threadIdx.x; e < PM_B * 32; e += PM_THREADS) {
    const int r = e >> 5, c4 = e & 31, gr = tile * PM_B + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gr < rows) v = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)gr * 128) + c4);
    uint32_t h0, l0, h1, l1;
    if (FP16) {
      split_hf(v.x * sc, v.y * sc, h0, l0);
      split_hf(v.z * sc, v.w * sc, h1, l1);
    } else {
      split_bf(v.x, v.y, h0, l0);
      split_bf(v.z, v.w, h1, l1);
    }
    const uint32_t off = tile_off(r, c4 >> 1) + (c4 & 1) * 8;
    *reinterpret_cast<uint2 *>(dst + off) = make_uint2(h0, h1);
    *reinterpret_cast<uint2 *>(dst + PM_B * 256 + off) = make_uint2(l0, l1);
  }
}

constexpr int PM2_WARPS = 8;
constexpr int PM2_THREADS = 32 * PM2_WARPS;
constexpr int PM2_BQ = 16 * PM2_WARPS;   // 128 queries per CTA

struct Fa2Smem {
  uint8_t k[2][PM_TILE];
  uint8_t v[2][PM_TILE];
  unsigned long long full[2], empty[2];
};

// FA + aux over pre-split K (fp16, scaled) / V (bf16) tiles; CTA = (head,
// 128 queries), 8 warps x 16 rows, two-stage bulk-copy pipeline.
__global__ void __launch_bounds__(PM2_THREADS, 1)
flash_mma2_kernel(const float *__restrict__ Qs, const uint8_t *__restrict__ Kt, const float *__restrict__ Ksc,
                  const uint8_t *__restrict__ Vt, int group, int n_q, int n_k, int causal,
                  float *__restrict__ O, float *__restrict__ Lout, float *__restrict__ Mout) {
  extern __shared__ __align__(128) uint8_t fsm2[];
  Fa2Smem &sm = *reinterpret_cast<Fa2Smem *>(fsm2);
  const int h = blockIdx.y, q0 = blockIdx.x * PM2_BQ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int hk = h / group;
  const int nkt = (n_k + PM_B - 1) / PM_B;
  const int q_last = min(q0 + PM2_BQ, n_q) - 1;
  const int kt_end = causal ? min(nkt, q_last / PM_B + 1) : nkt;
  const uint8_t *Kh = Kt + (int64_t)hk * nkt * PM_TILE;
  const uint8_t *Vh = Vt + (int64_t)hk * nkt * PM_TILE;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      pm_mbar_init(&sm.full[s], 1);
      pm_mbar_init(&sm.empty[s], PM2_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int kt) {
    const int s = kt & 1;
    pm_expect_tx(&sm.full[s], 2 * PM_TILE);
    pm_bulk(sm.k[s], Kh + (int64_t)kt * PM_TILE, PM_TILE, &sm.full[s]);
    pm_bulk(sm.v[s], Vh + (int64_t)kt * PM_TILE, PM_TILE, &sm.full[s]);
  };
  if (threadIdx.x == 0) {
    if (kt_end > 0) issue(0);
    if (kt_end > 1) issue(1);
  }
  const float *Qh = Qs + (int64_t)h * n_q * 128;
  const int qa = q0 + 16 * warp + g, qb = qa + 8;
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
  const int kb_row = (lane & 7) + 8 * (lane >> 4), kb_chunk = (lane >> 3) & 1;
  const int vb_row = (lane & 7) + 8 * ((lane >> 3) & 1), vb_chunk = lane >> 4;
  const int warp_last = min(q0 + 16 * warp + 15, n_q - 1);   // this warp's last query
  for (int kt = 0; kt < kt_end; ++kt) {
    const int s = kt & 1, k0 = kt * PM_B;
    pm_wait(&sm.full[s], (kt >> 1) & 1);
    if (!causal || k0 <= warp_last) {   // (tiles entirely above this warp's rows skip the math)
      const uint32_t kh_a = smem_addr(sm.k[s]), kl_a = kh_a + PM_B * 256;
      const uint32_t vh_a = smem_addr(sm.v[s]), vl_a = vh_a + PM_B * 256;
      const float unscale = 1.f / (sQ * __ldg(Ksc + (int64_t)hk * nkt + kt));
      float sc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[i][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int np = 0; np < 4; ++np) {
          uint32_t bh[4], bl[4];
          const uint32_t off = tile_off(16 * np + kb_row, 2 * ks + kb_chunk);
          ldsm4(kh_a + off, bh);
          ldsm4(kl_a + off, bl);
          mma_f16(sc[2 * np], qh[ks], bh[0], bh[1]);
          mma_f16(sc[2 * np], qh[ks], bl[0], bl[1]);
          mma_f16(sc[2 * np], ql[ks], bh[0], bh[1]);
          mma_f16(sc[2 * np + 1], qh[ks], bh[2], bh[3]);
          mma_f16(sc[2 * np + 1], qh[ks], bl[2], bl[3]);
          mma_f16(sc[2 * np + 1], ql[ks], bh[2], bh[3]);
        }
      }
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
        split_bf(p[0], p[1], ph[i >> 1][(i & 1) * 2 + 0], pl[i >> 1][(i & 1) * 2 + 0]);
        split_bf(p[2], p[3], ph[i >> 1][(i & 1) * 2 + 1], pl[i >> 1][(i & 1) * 2 + 1]);
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
        for (int dp = 0; dp < 8; ++dp) {
          uint32_t vh[4], vl[4];
          const uint32_t off = tile_off(16 * ks + vb_row, 2 * dp + vb_chunk);
          ldsm4_t(vh_a + off, vh);
          ldsm4_t(vl_a + off, vl);
          mma_bf16(o[2 * dp], ph[ks], vh[0], vh[1]);
          mma_bf16(o[2 * dp], ph[ks], vl[0], vl[1]);
          mma_bf16(o[2 * dp], pl[ks], vh[0], vh[1]);
          mma_bf16(o[2 * dp + 1], ph[ks], vh[2], vh[3]);
          mma_bf16(o[2 * dp + 1], ph[ks], vl[2], vl[3]);
          mma_bf16(o[2 * dp + 1], pl[ks], vh[2], vh[3]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) pm_arrive(&sm.empty[s]);
    if (threadIdx.x == 0 && kt + 2 < kt_end) {   // stage s is free once every warp is done
      pm_wait(&sm.empty[s], (kt >> 1) & 1);
      issue(kt + 2);
    }
  }
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
      *reinterpret_cast<float2 *>(Oh + (int64_t)qa * 128 + 8 * i + 2 * t) = make_float2(o[i][0] * inv0, o[i][1] * inv0);
    if (qb < n_q)
      *reinterpret_cast<float2 *>(Oh + (int64_t)qb * 128 + 8 * i + 2 * t) = make_float2(o[i][2] * inv1, o[i][3] * inv1);
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

struct Ans2Smem {
  uint8_t q[2][PM_TILE];
  float row[2][3][PM_B];   // M, 1/L, q_norm of the tile's queries
  unsigned long long full[2], empty[2];
};

// AnS over pre-split Q tiles (fp16, scaled): CTA = (output head, 64 keys),
// 4 warps x 16 keys as the A operand, streaming (query head, query tile)
// items through a two-stage pipeline; rows M / 1/L / |q| staged per item.
__global__ void __launch_bounds__(PM_THREADS)
ans_mma2_kernel(const uint8_t *__restrict__ Qt, const float *__restrict__ Qsc, const float *__restrict__ Kr,
                const float *__restrict__ Mv, const float *__restrict__ Lv, const float *__restrict__ qn,
                int group, int sum_group, int n_q, int n_k, int causal, float *__restrict__ ans_k,
                float *__restrict__ ans_v) {
  extern __shared__ __align__(128) uint8_t asm2[];
  Ans2Smem &sm = *reinterpret_cast<Ans2Smem *>(asm2);
  const int ho = blockIdx.y, kblk = blockIdx.x, k0 = kblk * PM_B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ka = k0 + 16 * warp + g, kb = ka + 8;
  const int nqt = (n_q + PM_B - 1) / PM_B;
  const int qt0 = causal ? kblk : 0;
  const int per_head = max(0, nqt - qt0);
  const int items = per_head * sum_group;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      pm_mbar_init(&sm.full[s], 1);
      pm_mbar_init(&sm.empty[s], PM_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int it) {
    const int s = it & 1, gq = it / per_head, qt = qt0 + it % per_head;
    const int h = ho * sum_group + gq;
    pm_expect_tx(&sm.full[s], PM_TILE);
    pm_bulk(sm.q[s], Qt + ((int64_t)h * nqt + qt) * PM_TILE, PM_TILE, &sm.full[s]);
  };
  auto stage_rows = [&](int it) {   // plain loads (the tail tile may be partial)
    const int s = it & 1, gq = it / per_head, qt = qt0 + it % per_head;
    const int h = ho * sum_group + gq;
    for (int i = threadIdx.x; i < PM_B; i += PM_THREADS) {
      const int qi = qt * PM_B + i;
      const bool ok = qi < n_q;
      sm.row[s][0][i] = ok ? Mv[(int64_t)h * n_q + qi] : 0.f;
      sm.row[s][1][i] = ok ? 1.f / Lv[(int64_t)h * n_q + qi] : 0.f;
      sm.row[s][2][i] = ok ? qn[(int64_t)h * n_q + qi] : 0.f;
    }
  };
  if (threadIdx.x == 0) {
    if (items > 0) issue(0);
    if (items > 1) issue(1);
  }
  const int qb_row = (lane & 7) + 8 * (lane >> 4), qb_chunk = (lane >> 3) & 1;
  const float log2e = 1.4426950408889634f;
  float sv[2] = {0.f, 0.f}, sk[2] = {0.f, 0.f};
  int cur_h = -1;
  uint32_t kh[8][4], kl[8][4];
  float sKw = 1.f;
  for (int it = 0; it < items; ++it) {
    const int s = it & 1, gq = it / per_head, qt = qt0 + it % per_head;
    const int h = ho * sum_group + gq, hk = h / group;
    if (hk != cur_h) {   // key fragments of this warp (fp16 parts, warp scale)
      cur_h = hk;
      const float *Kh = Kr + (int64_t)hk * n_k * 128;
      float2 v[8][4];
      float mx = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[ks][e] = make_float2(0.f, 0.f);
        if (ka < n_k) {
          v[ks][0] = *reinterpret_cast<const float2 *>(Kh + (int64_t)ka * 128 + 16 * ks + 2 * t);
          v[ks][2] = *reinterpret_cast<const float2 *>(Kh + (int64_t)ka * 128 + 16 * ks + 8 + 2 * t);
        }
        if (kb < n_k) {
          v[ks][1] = *reinterpret_cast<const float2 *>(Kh + (int64_t)kb * 128 + 16 * ks + 2 * t);
          v[ks][3] = *reinterpret_cast<const float2 *>(Kh + (int64_t)kb * 128 + 16 * ks + 8 + 2 * t);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fmaxf(fabsf(v[ks][e].x), fabsf(v[ks][e].y)));
      }
      sKw = pow2_scale(warp_max(mx));
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int e = 0; e < 4; ++e) split_hf(v[ks][e].x * sKw, v[ks][e].y * sKw, kh[ks][e], kl[ks][e]);
    }
    stage_rows(it);
    __syncthreads();   // rows of item it visible (stage s is free: see the arrive below)
    pm_wait(&sm.full[s], (it >> 1) & 1);
    const float unscale = 1.f / (sKw * __ldg(Qsc + (int64_t)h * nqt + qt));
    const uint32_t qh_a = smem_addr(sm.q[s]), ql_a = qh_a + PM_B * 256;
    const int q0 = qt * PM_B;
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t bh[4], bl[4];
        const uint32_t off = tile_off(16 * np + qb_row, 2 * ks + qb_chunk);
        ldsm4(qh_a + off, bh);
        ldsm4(ql_a + off, bl);
        mma_f16(sc[0], kh[ks], bh[0], bh[1]);
        mma_f16(sc[0], kh[ks], bl[0], bl[1]);
        mma_f16(sc[0], kl[ks], bh[0], bh[1]);
        mma_f16(sc[1], kh[ks], bh[2], bh[3]);
        mma_f16(sc[1], kh[ks], bl[2], bl[3]);
        mma_f16(sc[1], kl[ks], bh[2], bh[3]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = 16 * np + 8 * j + 2 * t + (e & 1);
          const int qi = q0 + col;
          const int key = (e < 2) ? ka : kb;
          if (qi < n_q && key < n_k && (!causal || key <= qi)) {
            const float a = exp2f((sc[j][e] * unscale - sm.row[s][0][col]) * log2e) * sm.row[s][1][col];
            sv[e >> 1] += a;
            sk[e >> 1] = fmaf(a * (1.f - a), sm.row[s][2][col], sk[e >> 1]);
          }
        }
    }
    __syncwarp();
    if (lane == 0) pm_arrive(&sm.empty[s]);
    if (threadIdx.x == 0 && it + 2 < items) {
      pm_wait(&sm.empty[s], (it >> 1) & 1);
      issue(it + 2);
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
  // pre-split K (fp16, scaled) and V (bf16) tiles, then the pipelined kernel
  const int nkt = ceil_div(n_k, PM_B);
  uint8_t *kt = nullptr, *vt = nullptr;
  float *ksc = nullptr;
  const size_t tb = (size_t)kv_heads * nkt * PM_TILE;
  cudaError_t e = scratch_alloc((void **)&kt, tb, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&vt, tb, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&ksc, sizeof(float) * (size_t)kv_heads * nkt, st);
  if (e != cudaSuccess) return cuda_status(e, "prefill tile scratch");
  presplit_kernel<true><<<dim3(nkt, kv_heads), PM_THREADS, 0, st>>>(Kr, n_k, kt, ksc);
  presplit_kernel<false><<<dim3(nkt, kv_heads), PM_THREADS, 0, st>>>(V, n_k, vt, nullptr);
  const int smem = sizeof(Fa2Smem);
  cudaFuncSetAttribute(flash_mma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(ceil_div(n_q, PM2_BQ), heads);
  flash_mma2_kernel<<<grid, PM2_THREADS, smem, st>>>(Qs, kt, ksc, vt, heads / kv_heads, n_q, n_k, causal,
                                                      O, L, M);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(kt, st);
  cudaFreeAsync(vt, st);
  cudaFreeAsync(ksc, st);
  if (le != cudaSuccess) return cuda_status(le, "flash_mma2_kernel");
  return ANTKV_OK;
}

int launch_ans_mma(const float *Qs, const float *Kr, const float *M, const float *L, const float *qn,
                   int heads, int kv_heads, int sum_group, int n_q, int n_k, int d, int causal,
                   float *ans_k, float *ans_v, cudaStream_t st) {
  if (d != 128) return ANTKV_EUNSUPPORTED;
  if (n_k == 0) return ANTKV_OK;
  const int nqt = ceil_div(n_q, PM_B);
  uint8_t *qt = nullptr;
  float *qsc = nullptr;
  cudaError_t e = scratch_alloc((void **)&qt, (size_t)heads * nqt * PM_TILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&qsc, sizeof(float) * (size_t)heads * nqt, st);
  if (e != cudaSuccess) return cuda_status(e, "anchor-score tile scratch");
  presplit_kernel<true><<<dim3(nqt, heads), PM_THREADS, 0, st>>>(Qs, n_q, qt, qsc);
  dim3 grid(ceil_div(n_k, PM_B), heads / sum_group);
  const int smem = sizeof(Ans2Smem);
  cudaFuncSetAttribute(ans_mma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ans_mma2_kernel<<<grid, PM_THREADS, smem, st>>>(qt, qsc, Kr, M, L, qn, heads / kv_heads, sum_group, n_q, n_k,
                                               causal, ans_k, ans_v);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(qt, st);
  cudaFreeAsync(qsc, st);
  if (le != cudaSuccess) return cuda_status(le, "ans_mma2_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
