// VQ encoder for d = 128, d_sub = 8, m <= 256, bf16 inputs (the 1-bit d8m256
// configuration) on the 5th-generation tensor cores.  Reference: vq.encode_rows
// (vq.py:226-232) -> assign_nearest (_ckernels.pyx:134-163): strict-< argmin
// of the squared distance over the centroids, lowest index on ties.
//
// A tile is 128 sub-vectors (8 tokens x 16 groups; TMEM lane l = token l / 16,
// group l % 16) against all 256 centroids: D[128 x 256] (fp32, TMEM) =
// A[128 x 48] . B[256 x 48]^T, three tcgen05.mma (K = 16 each, bf16 operands
// in 128B-swizzled K-major shared memory, the codebook operand B resident for
// the whole CTA).  With s = 2^-e a per-row power of two:
//   k  0..23  A: -2 s x (three copies)       B: c split hi | mid | lo (bf16,
//                                               24 mantissa bits = the fp32 c)
//   k 24      A: bf16(s |x|^2) (a per-row    B: 1
//             constant: keeps D >= 0)
//   k 25..27  A: s                           B: |c|^2 split hi | mid | lo
//   k 32, 33  A: 1, 1                        B: 2^23, 2^13 (2^24 for c >= m)
// so D = 2^23 + 2^13 + s (|c|^2 - 2 x.c + ~|x|^2), the last MMA adding only
// the exact constant.  D then lies in [2^23, 2^24), where the fp32 bit
// pattern is 0x4B000000 + round(D - 2^23): the bits, times 256, plus the
// column index form an integer key whose minimum is the strict-< argmin with
// the lowest index on ties -- one IMAD and half a 3-input integer min
// (VIMNMX3) per distance, read from TMEM with tcgen05.ld.
//
// Exactness: e is chosen so that the grid step 1/s lies in (3e-7, 6e-7] x
// (|x|^2 + max|c|^2); the distance range 2 (|x|^2 + max|c|^2) then stays
// below 2^23 steps, and two centroids are ordered differently from the
// float64 distances only when their margin is below one step plus the fp32
// accumulation error, i.e. below the 1e-6 (|x|^2 + max|c|^2) of the parity
// rule.
//
// Warp roles (14 warps): 13 bulk-copies the raw input tiles (8 tokens, 2 KB)
// 16 stages ahead; 0-3 build the A tiles from them (warp w the tiles w mod 4,
// a lane four sub-vector rows: 16-byte shared loads, swizzled 16-byte
// stores), 4-11 are the epilogue (warp w reads TMEM lanes 32 (w % 4).. of
// the even (w < 8) or odd tiles, a thread = one sub-vector's 256
// distances), 12 allocates TMEM and its lane 0 issues the MMAs.  Six A stages, two TMEM accumulators (256 columns
// each): the MMAs of tile t + 1 overlap the epilogue of tile t.  Codes leave
// as one 16-byte store per token (the cache's row layout).
#include "common.cuh"

namespace antkv {
namespace {

constexpr int T5_ROWS = 128;                  // sub-vectors per tile
constexpr int T5_TOK = 8;                     // tokens per tile
constexpr int T5_N = 256;                     // centroid columns
constexpr int T5_AS = 6;                      // A stages
constexpr int T5_PROD = 4, T5_EPI = 8;        // warps
constexpr int T5_MMA_WARP = T5_PROD + T5_EPI;
constexpr int T5_LOAD_WARP = T5_MMA_WARP + 1;
constexpr int T5_THREADS = 32 * (T5_LOAD_WARP + 1);
constexpr int T5_XS = 16;                     // raw input stages (2 KB each)
constexpr int T5_XTILE = T5_TOK * 128 * 2;
constexpr int T5_ATILE = T5_ROWS * 128;       // 16 KB
constexpr int T5_BTILE = T5_N * 128;          // 32 KB

struct T5Smem {
  uint8_t b[T5_BTILE];
  uint8_t a[T5_AS][T5_ATILE];
  uint8_t x[T5_XS][T5_XTILE];
  uint8_t ct[T5_EPI][32];
  float part[T5_THREADS / 32];
  unsigned long long afull[T5_AS], aempty[T5_AS], dfull[2], dempty[2], xfull[T5_XS], xempty[T5_XS];
  uint32_t tmem;
  float cbmax;
};

// byte offset of the 16-byte chunk (row, k / 8) in a 128B-swizzled K-major tile
__device__ __forceinline__ uint32_t t5_off(int row, int chunk) {
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint32_t t5_smem(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void t5_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(t5_smem(bar)), "r"(count));
}
__device__ __forceinline__ void t5_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(t5_smem(bar)) : "memory");
}
__device__ __forceinline__ void t5_wait(unsigned long long *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(t5_smem(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// K-major, 128B swizzle, 8-row groups 1024 B apart, sm_100 descriptor version
__device__ __forceinline__ uint64_t t5_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Warp-wide forms (all lanes call with the same operands, one elected lane
// issues): from converged code the operands stay uniform and UTCHMMA needs no
// per-instruction ELECT/BRA.U.ANY waterfall as under lane == 0.
__device__ __forceinline__ void t5_mma_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void t5_commit_w(unsigned long long *bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(t5_smem(bar))
      : "memory");
}
__device__ __forceinline__ void t5_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// tcgen05.wait::ld, then tie the loaded registers to it: their consumers
// cannot be scheduled above the wait
__device__ __forceinline__ void t5_ld_wait(uint32_t (&x)[32], uint32_t (&y)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(x[i]), "+r"(y[i]));
}

__device__ __forceinline__ uint32_t bf16_bits(float x) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(x)));
}
__device__ __forceinline__ uint32_t bf16_pair(float lo, float hi) { return bf16_bits(lo) | (bf16_bits(hi) << 16); }
__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// x = hi + mid + lo exactly (24 mantissa bits in three 8-bit parts)
__device__ __forceinline__ void split3_bf16(float x, float &hi, float &mid, float &lo) {
  hi = bf16_round(x);
  const float r = x - hi;
  mid = bf16_round(r);
  lo = bf16_round(r - mid);
}

// min of the 32 keys (bits * 256 + i)
// (mul == 256 at run time: three in four keys are IMADs on the FMA pipe, the
// rest LEAs on the ALU pipe, which also runs the VIMNMX3 tree)
__device__ __forceinline__ uint32_t chunk_min(const uint32_t (&r)[32], uint32_t mul) {
  uint32_t k[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) k[i] = (i & 3) == 0 ? r[i] * 256u + (uint32_t)i : r[i] * mul + (uint32_t)i;
  uint32_t m[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) m[i] = __vimin3_u32(k[3 * i], k[3 * i + 1], k[3 * i + 2]);
  m[10] = min(k[30], k[31]);
  const uint32_t a = __vimin3_u32(m[0], m[1], m[2]), b = __vimin3_u32(m[3], m[4], m[5]);
  const uint32_t c = __vimin3_u32(m[6], m[7], m[8]), d = min(m[9], m[10]);
  return min(__vimin3_u32(a, b, c), d);
}

__global__ void __launch_bounds__(T5_THREADS, 1)
vq_encode_tc5_kernel(const uint16_t *__restrict__ X, int64_t rows, int64_t x_set_stride,
                     const float *__restrict__ codebooks, int cb_mod, int m, void *__restrict__ codes,
                     int code_bytes, int64_t code_set_stride, int64_t code_tile_stride,
                     int64_t code_row_stride, int64_t tiles_per_cta, int vec_store, uint32_t mul) {
  extern __shared__ __align__(128) unsigned char t5raw[];
  T5Smem &sm = *reinterpret_cast<T5Smem *>(t5raw + ((1024 - (t5_smem(t5raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int set = blockIdx.y;
  const int64_t ntiles = (rows + T5_TOK - 1) / T5_TOK;
  const int64_t tile0 = blockIdx.x * tiles_per_cta;
  const int items = (int)max((int64_t)0, min(tiles_per_cta, ntiles - tile0));
  const float *cb = codebooks + (int64_t)(set % cb_mod) * m * 8;

  if (threadIdx.x == 0) {
    for (int s = 0; s < T5_AS; ++s) {
      t5_init(&sm.afull[s], 32);
      t5_init(&sm.aempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      t5_init(&sm.dfull[s], 1);
      t5_init(&sm.dempty[s], 32 * T5_EPI / 2);
    }
    for (int s = 0; s < T5_XS; ++s) {
      t5_init(&sm.xfull[s], 1);
      t5_init(&sm.xempty[s], 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == T5_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(t5_smem(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // ---- codebook operand (resident): rows c < 256, chunks 0-2 = c hi/mid/lo,
  // 3 = (1, |c|^2 hi/mid/lo), 4 = the constant (2^23, 2^13) or 2^24 past m
  float nmax = 0.f;
  for (int c = threadIdx.x; c < T5_N; c += T5_THREADS) {
    float x[8];
    if (c < m) {
      const float4 p = __ldg(reinterpret_cast<const float4 *>(cb + c * 8));
      const float4 q = __ldg(reinterpret_cast<const float4 *>(cb + c * 8 + 4));
      x[0] = p.x; x[1] = p.y; x[2] = p.z; x[3] = p.w; x[4] = q.x; x[5] = q.y; x[6] = q.z; x[7] = q.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = 0.f;
    }
    float nn = x[0] * x[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) nn = fmaf(x[i], x[i], nn);
    float hi[8], mi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split3_bf16(x[i], hi[i], mi[i], lo[i]);
    float nh, nm, nl;
    split3_bf16(nn, nh, nm, nl);
    uint8_t *row = sm.b;
    *reinterpret_cast<uint4 *>(row + t5_off(c, 0)) =
        make_uint4(bf16_pair(hi[0], hi[1]), bf16_pair(hi[2], hi[3]), bf16_pair(hi[4], hi[5]), bf16_pair(hi[6], hi[7]));
    *reinterpret_cast<uint4 *>(row + t5_off(c, 1)) =
        make_uint4(bf16_pair(mi[0], mi[1]), bf16_pair(mi[2], mi[3]), bf16_pair(mi[4], mi[5]), bf16_pair(mi[6], mi[7]));
    *reinterpret_cast<uint4 *>(row + t5_off(c, 2)) =
        make_uint4(bf16_pair(lo[0], lo[1]), bf16_pair(lo[2], lo[3]), bf16_pair(lo[4], lo[5]), bf16_pair(lo[6], lo[7]));
    *reinterpret_cast<uint4 *>(row + t5_off(c, 3)) =
        c < m ? make_uint4(bf16_pair(1.f, nh), bf16_pair(nm, nl), 0u, 0u) : make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4 *>(row + t5_off(c, 4)) =
        make_uint4(bf16_pair(c < m ? 8388608.f : 16777216.f, 8192.f), 0u, 0u, 0u);
    *reinterpret_cast<uint4 *>(row + t5_off(c, 5)) = make_uint4(0u, 0u, 0u, 0u);
    if (c < m) nmax = fmaxf(nmax, nn);
  }
  // constant chunks of the A stages: 4 = (1, 1, 0...), 5 = 0
  for (int e = threadIdx.x; e < T5_AS * T5_ROWS; e += T5_THREADS) {
    uint8_t *a = sm.a[e / T5_ROWS];
    const int r = e % T5_ROWS;
    *reinterpret_cast<uint4 *>(a + t5_off(r, 4)) = make_uint4(bf16_pair(1.f, 1.f), 0u, 0u, 0u);
    *reinterpret_cast<uint4 *>(a + t5_off(r, 5)) = make_uint4(0u, 0u, 0u, 0u);
  }
  nmax = warp_max(nmax);
  if (lane == 0) sm.part[warp] = nmax;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // operand stores -> tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem;
  if (tmem != 0) __trap();   // 512 columns at one CTA per SM start at column 0 (the MMA warps assume it)

  if (warp < T5_PROD) {
    // ---- A producer: thread = sub-vector row (token r / 16, group r % 16)
    float cbmax = sm.part[0];
#pragma unroll
    for (int i = 1; i < T5_THREADS / 32; ++i) cbmax = fmaxf(cbmax, sm.part[i]);
    // warp w builds the tiles it = w (mod T5_PROD), lane l
    // builds rows l + 32 u (token r / 16, group r % 16)
    for (int it = warp; it < items; it += T5_PROD) {
      const int st = it % T5_AS, xs = it % T5_XS;
      t5_wait(&sm.xfull[xs], (it / T5_XS) & 1);
      uint4 xr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = lane + 32 * u, tl = r >> 4, grp = r & 15;
        const int64_t tok = (tile0 + it) * T5_TOK + tl;
        xr[u] = tok < rows ? *reinterpret_cast<const uint4 *>(&sm.x[xs][(tl * 128 + grp * 8) * 2])
                           : make_uint4(0u, 0u, 0u, 0u);
      }
      __syncwarp();
      t5_arrive(&sm.xempty[xs]);
      uint4 ax[4], an[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float x[8];
        x[0] = __uint_as_float(xr[u].x << 16); x[1] = __uint_as_float(xr[u].x & 0xffff0000u);
        x[2] = __uint_as_float(xr[u].y << 16); x[3] = __uint_as_float(xr[u].y & 0xffff0000u);
        x[4] = __uint_as_float(xr[u].z << 16); x[5] = __uint_as_float(xr[u].z & 0xffff0000u);
        x[6] = __uint_as_float(xr[u].w << 16); x[7] = __uint_as_float(xr[u].w & 0xffff0000u);
        float n2 = x[0] * x[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) n2 = fmaf(x[i], x[i], n2);
        // grid step 2^e in (3e-7, 6e-7] * (|x|^2 + max|c|^2)
        const float tt = 6e-7f * (n2 + cbmax);
        int e = ((__float_as_int(tt) >> 23) & 0xff) - 127;
        e = max(-126, min(126, e));
        const float s = __int_as_float((127 - e) << 23);     // 2^-e
        const float m2s = -2.f * s;
        ax[u] = make_uint4(bf16_pair(x[0] * m2s, x[1] * m2s), bf16_pair(x[2] * m2s, x[3] * m2s),
                           bf16_pair(x[4] * m2s, x[5] * m2s), bf16_pair(x[6] * m2s, x[7] * m2s));
        an[u] = make_uint4(bf16_pair(n2 * s, s), bf16_pair(s, s), 0u, 0u);
      }
      if (it >= T5_AS) t5_wait(&sm.aempty[st], ((it / T5_AS) - 1) & 1);
      uint8_t *a = sm.a[st];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = lane + 32 * u;
        *reinterpret_cast<uint4 *>(a + t5_off(r, 0)) = ax[u];
        *reinterpret_cast<uint4 *>(a + t5_off(r, 1)) = ax[u];
        *reinterpret_cast<uint4 *>(a + t5_off(r, 2)) = ax[u];
        *reinterpret_cast<uint4 *>(a + t5_off(r, 3)) = an[u];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      t5_arrive(&sm.afull[st]);
    }
  } else if (warp == T5_LOAD_WARP) {
    // ---- raw input tiles (8 tokens = 2 KB contiguous) by bulk copy, 16 stages ahead
    if (lane == 0) {
      const uint8_t *xg = reinterpret_cast<const uint8_t *>(X + set * x_set_stride);
      for (int it = 0; it < items; ++it) {
        const int xs = it % T5_XS;
        if (it >= T5_XS) t5_wait(&sm.xempty[xs], ((it / T5_XS) - 1) & 1);
        const int64_t tok0 = (tile0 + it) * T5_TOK;
        const uint32_t bytes = (uint32_t)(min((int64_t)T5_TOK, rows - tok0) * 256);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(t5_smem(&sm.xfull[xs])),
                     "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                t5_smem(sm.x[xs])),
            "l"(xg + tok0 * 256), "r"(bytes), "r"(t5_smem(&sm.xfull[xs]))
            : "memory");
      }
    }
  } else if (warp == T5_MMA_WARP) {
    // ---- MMA issuer: kind::f16, bf16 A/B (bits 7-9, 10-12), fp32 D, K-major,
    // N = 256 (bits 17-22), M = 128 (bits 24-28)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T5_N >> 3) << 17) |
                           ((uint32_t)(T5_ROWS >> 4) << 24);
    const uint32_t bsm = t5_smem(sm.b);
    for (int it = 0; it < items; ++it) {
      const int st = it % T5_AS, buf = it & 1;
      t5_wait(&sm.afull[st], (it / T5_AS) & 1);
      if (it >= 2) t5_wait(&sm.dempty[buf], ((it >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      {
        // 512 columns, one CTA per SM: the allocation starts at column 0
        const uint32_t asm_ = t5_smem(sm.a[st]), d = buf * T5_N;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) t5_mma_w(d, t5_desc(asm_ + 32 * ks), t5_desc(bsm + 32 * ks), idesc, ks > 0);
        t5_commit_w(&sm.aempty[st]);
        t5_commit_w(&sm.dfull[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 (row r of the
    // tile) of every other tile: warps 4-7 the even tiles (accumulator 0),
    // 8-11 the odd ones (accumulator 1); a thread scans all 256 columns
    const int ew = warp - T5_PROD, q = warp & 3, par = ew >> 2;
    const int r = 32 * q + lane;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + par * T5_N;
    uint8_t *ctw = sm.ct[ew];
    for (int it = par; it < items; it += 2) {
      t5_wait(&sm.dfull[par], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t best = 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        uint32_t v0[32], v1[32];
        t5_ld32(tq + 32 * j, v0);
        t5_ld32(tq + 32 * (j + 1), v1);
        t5_ld_wait(v0, v1);
        if (j == 6) {   // the accumulator is in registers: hand it back to the MMAs
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          t5_arrive(&sm.dempty[par]);
        }
        best = min(best, chunk_min(v0, mul) + (uint32_t)(32 * j));
        best = min(best, chunk_min(v1, mul) + (uint32_t)(32 * (j + 1)));
      }
      const int code = (int)(best & 0xffu);
      const int64_t tok = (tile0 + it) * T5_TOK + (r >> 4);
      if (vec_store) {   // lanes 0 / 16 store the 16 codes of tokens 2q / 2q + 1
        ctw[lane] = static_cast<uint8_t>(code);
        __syncwarp();
        if ((lane & 15) == 0 && tok < rows) {
          uint8_t *dst = static_cast<uint8_t *>(codes) + set * code_set_stride + (tok >> 4) * code_tile_stride +
                         (tok & 15) * code_row_stride;
          *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>(&ctw[lane]);
        }
        __syncwarp();
      } else if (tok < rows) {
        const int64_t off = set * code_set_stride + (tok >> 4) * code_tile_stride + (tok & 15) * code_row_stride +
                            (r & 15);
        if (code_bytes == 1) static_cast<uint8_t *>(codes)[off] = static_cast<uint8_t>(code);
        else if (code_bytes == 2) static_cast<uint16_t *>(codes)[off] = static_cast<uint16_t>(code);
        else if (code_bytes == 4) static_cast<int32_t *>(codes)[off] = code;
        else static_cast<int64_t *>(codes)[off] = code;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == T5_MMA_WARP) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------------------
// Long codebooks (d_sub 16 / 32, any m <= 65536: config #3's d32m4096) and
// 4-dim sub-vectors (config #4's d4m256: one distance k-step per block):
// the same integer-key argmin over 128-centroid blocks of the codebook.
//
// A sub-vector row of DSUB dims spans two 128B-swizzled atoms (K = 128):
//   k 0 .. 3 DSUB - 1   A: -2 s x (three copies)     B: c hi | mid | lo
//   k 3 DSUB            A: bf16(s |x|^2)             B: 1
//   k 3 DSUB + 1 .. +3  A: s                         B: |c|^2 hi | mid | lo
//   k-step KD (16 KD, 16 KD + 1)  A: 1, 1            B: 2^23, 2^13 (2^24 past m)
// with KD = ceil((3 DSUB + 4) / 16) distance k-steps (7 for DSUB = 32).  The
// codebook operand is pre-swizzled once per call into a global image of
// 128-centroid blocks (32 KB each, L2-resident) that a loader warp streams
// through a 4-stage ring; a CTA keeps a PAIR of A tiles (2 x 128 sub-vectors)
// resident while every block passes, so each 32 KB block feeds 2 x (KD + 1)
// MMAs (M = 128, N = 128).  TMEM: tile t, buffer u at column 256 t + 128 u
// (two buffers per tile).  Epilogue warps 4-7 reduce tile 0, 8-11 tile 1;
// a thread keeps its sub-vector's best (key, block) over the blocks (strict
// <: the earlier block wins ties, so the lowest index overall).  The grid
// step 1/s lies in (2.5e-7, 5e-7] (|x|^2 + max|c|^2) here: 2 (|x|^2 +
// max|c|^2) stays below 2^23 steps and one step plus the fp32 accumulation
// error of the longer dot products stays inside the parity rule's 1e-6.
constexpr int TL_NB = 128;                      // centroids per block
constexpr int TL_BS = 4;                        // B ring stages
constexpr int TL_ATILE = 128 * 256;             // two atoms x 128 rows
constexpr int TL_BBLK = TL_NB * 256;            // 32 KB
constexpr int TL_PROD = 4, TL_EPI = 8;
constexpr int TL_MMA_WARP = TL_PROD + TL_EPI, TL_LOAD_WARP = TL_MMA_WARP + 1;
constexpr int TL_THREADS = 32 * (TL_LOAD_WARP + 1);

struct TlSmem {
  uint8_t a[2][TL_ATILE];
  uint8_t b[TL_BS][TL_BBLK];
  uint32_t cw[TL_EPI][32];                      // packed-row staging of the epilogue warps
  unsigned long long afull, aempty, bfull[TL_BS], bempty[TL_BS], dfull[2], dempty[2];
  uint32_t tmem;
};

// chunk (16 bytes) c of `row` in a two-atom 128B-swizzled tile of R rows
template <int R>
__device__ __forceinline__ uint32_t tl_off(int row, int c) {
  return (c >> 3) * (R * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4);
}

template <int DSUB>
constexpr int tl_kd() { return (3 * DSUB + 4 + 15) / 16; }

// Codebook image: [codebook][block][two atoms x 128 rows x 128 B]
template <int DSUB>
__global__ void __launch_bounds__(TL_NB)
tl_codebook_image_kernel(const float *__restrict__ codebooks, int m, uint8_t *__restrict__ img, int nblk,
                         float *__restrict__ blkmax) {
  constexpr int KD = tl_kd<DSUB>();
  const int blk = blockIdx.x, cbk = blockIdx.y, r = threadIdx.x;
  const int c = blk * TL_NB + r;
  const float *cb = codebooks + ((int64_t)cbk * m + (c < m ? c : 0)) * DSUB;
  uint8_t *dst = img + ((int64_t)cbk * nblk + blk) * TL_BBLK;
  for (int ch = 0; ch < 16; ++ch) *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, ch)) = make_uint4(0u, 0u, 0u, 0u);
  float nn = 0.f;
  if constexpr (DSUB == 4) {   // one k-step: (hi | mid), (lo | 1, |c|^2 hi / mid / lo)
    float hi[4], mi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float x = c < m ? cb[i] : 0.f;
      nn = fmaf(x, x, nn);
      split3_bf16(x, hi[i], mi[i], lo[i]);
    }
    float nh, nm, nl;
    split3_bf16(nn, nh, nm, nl);
    *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, 0)) =
        make_uint4(bf16_pair(hi[0], hi[1]), bf16_pair(hi[2], hi[3]), bf16_pair(mi[0], mi[1]), bf16_pair(mi[2], mi[3]));
    *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, 1)) =
        c < m ? make_uint4(bf16_pair(lo[0], lo[1]), bf16_pair(lo[2], lo[3]), bf16_pair(1.f, nh), bf16_pair(nm, nl))
              : make_uint4(0u, 0u, 0u, 0u);
  }
  for (int j0 = 0; DSUB >= 8 && j0 < DSUB; j0 += 8) {
    float hi[8], mi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float x = c < m ? cb[j0 + i] : 0.f;
      nn = fmaf(x, x, nn);
      split3_bf16(x, hi[i], mi[i], lo[i]);
    }
    const int ch = j0 / 8;
    *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, ch)) =
        make_uint4(bf16_pair(hi[0], hi[1]), bf16_pair(hi[2], hi[3]), bf16_pair(hi[4], hi[5]), bf16_pair(hi[6], hi[7]));
    *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, ch + DSUB / 8)) =
        make_uint4(bf16_pair(mi[0], mi[1]), bf16_pair(mi[2], mi[3]), bf16_pair(mi[4], mi[5]), bf16_pair(mi[6], mi[7]));
    *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, ch + DSUB / 4)) =
        make_uint4(bf16_pair(lo[0], lo[1]), bf16_pair(lo[2], lo[3]), bf16_pair(lo[4], lo[5]), bf16_pair(lo[6], lo[7]));
  }
  if constexpr (DSUB >= 8) {
    float nh, nm, nl;
    split3_bf16(nn, nh, nm, nl);
    if (c < m)
      *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, 3 * DSUB / 8)) = make_uint4(bf16_pair(1.f, nh), bf16_pair(nm, nl), 0u, 0u);
  }
  // the block's max |c|^2 (the exactness scale is the max over the blocks)
  __shared__ float red[TL_NB / 32];
  float mx = warp_max(c < m ? nn : 0.f);
  if ((r & 31) == 0) red[r >> 5] = mx;
  __syncthreads();
  if (r == 0) {
    for (int i = 1; i < TL_NB / 32; ++i) mx = fmaxf(mx, red[i]);
    blkmax[(int64_t)cbk * nblk + blk] = fmaxf(mx, red[0]);
  }
  *reinterpret_cast<uint4 *>(dst + tl_off<TL_NB>(r, 2 * KD)) =
      make_uint4(bf16_pair(c < m ? 8388608.f : 16777216.f, 8192.f), 0u, 0u, 0u);
}

template <int DSUB>
__global__ void __launch_bounds__(TL_THREADS, 1)
vq_encode_tc5l_kernel(const uint16_t *__restrict__ X, int64_t rows, int64_t x_set_stride,
                      const uint8_t *__restrict__ img, const float *__restrict__ blkmax, int cb_mod, int m,
                      int nblk, void *__restrict__ codes, int code_bytes, int64_t code_set_stride,
                      int64_t code_tile_stride, int64_t code_row_stride, int64_t tiles_per_cta, uint32_t mul) {
  constexpr int G = 128 / DSUB, KD = tl_kd<DSUB>(), NCH = DSUB >= 8 ? DSUB / 8 : 1;
  constexpr int PT = DSUB == 4 ? 2 : 3 * NCH + 1;   // A chunks rewritten per tile (the rest are constant)
  extern __shared__ __align__(128) unsigned char tlraw[];
  TlSmem &sm = *reinterpret_cast<TlSmem *>(tlraw + ((1024 - (t5_smem(tlraw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int set = blockIdx.y;
  // the CTA's tiles [tile0, tile0 + ntl) go in pairs; an odd count ends with a single tile
  const int64_t nsub = rows * G, ntiles = (nsub + 127) / 128;
  const int64_t tile0 = blockIdx.x * tiles_per_cta;
  const int ntl = (int)max((int64_t)0, min(tiles_per_cta, ntiles - tile0));
  const int items = (ntl + 1) / 2;
  const int64_t sv_end = min(nsub, (tile0 + ntl) * 128);   // rows past it: zero, not stored
  const uint8_t *bimg = img + (int64_t)(set % cb_mod) * nblk * TL_BBLK;
  if (threadIdx.x == 0) {
    t5_init(&sm.afull, 32 * TL_PROD);
    t5_init(&sm.aempty, 1);
    for (int s = 0; s < TL_BS; ++s) {
      t5_init(&sm.bfull[s], 1);
      t5_init(&sm.bempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      t5_init(&sm.dfull[s], 1);
      t5_init(&sm.dempty[s], 32 * TL_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == TL_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(t5_smem(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // constant A chunks: zeros between the norm chunk and the magic one, the
  // magic chunk (1, 1, 0...) and the zero tail of the last k-step
  for (int e = threadIdx.x; e < 2 * 128; e += TL_THREADS) {
    uint8_t *a = sm.a[e >> 7];
    const int r = e & 127;
    for (int ch = PT; ch < 16; ++ch)
      *reinterpret_cast<uint4 *>(a + tl_off<128>(r, ch)) =
          ch == 2 * KD ? make_uint4(bf16_pair(1.f, 1.f), 0u, 0u, 0u) : make_uint4(0u, 0u, 0u, 0u);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem;
  if (tmem != 0) __trap();   // 512 columns at one CTA per SM start at column 0 (the MMA warps assume it)

  if (warp < TL_PROD) {
    // ---- A pair producer: thread p builds rows p and p + 128 of the pair
    // (tile p / 128... = tile 0 rows p, tile 1 rows p), the next pair's inputs
    // prefetched into registers while the current pair streams the blocks
    float cbmax = 0.f;
    for (int i = 0; i < nblk; ++i) cbmax = fmaxf(cbmax, __ldg(blkmax + (int64_t)(set % cb_mod) * nblk + i));
    const int r = threadIdx.x;   // 0..127: row of both tiles
    auto load = [&](int it, int t, uint4 (&v)[NCH]) {
      const int64_t sv = (tile0 + 2 * it + t) * 128 + r;
      if (sv < sv_end && DSUB == 4) {   // 8 bytes: x in .x, .y
        const uint2 x2 = __ldg(reinterpret_cast<const uint2 *>(X + set * x_set_stride + (sv / G) * 128 + (sv % G) * DSUB));
        v[0] = make_uint4(x2.x, x2.y, 0u, 0u);
      } else if (sv < sv_end) {
        const uint4 *src = reinterpret_cast<const uint4 *>(X + set * x_set_stride + (sv / G) * 128 + (sv % G) * DSUB);
#pragma unroll
        for (int i = 0; i < NCH; ++i) v[i] = __ldg(src + i);
      } else {
#pragma unroll
        for (int i = 0; i < NCH; ++i) v[i] = make_uint4(0u, 0u, 0u, 0u);
      }
    };
    uint4 nx[2][NCH];
    if (items > 0) { load(0, 0, nx[0]); load(0, 1, nx[1]); }
    for (int it = 0; it < items; ++it) {
      uint4 xv[2][NCH];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int i = 0; i < NCH; ++i) xv[t][i] = nx[t][i];
      if (it + 1 < items) { load(it + 1, 0, nx[0]); load(it + 1, 1, nx[1]); }
      if (it > 0) t5_wait(&sm.aempty, (it - 1) & 1);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        float n2 = 0.f;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t w4[4] = {xv[t][i].x, xv[t][i].y, xv[t][i].z, xv[t][i].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float x0 = __uint_as_float(w4[k] << 16), x1 = __uint_as_float(w4[k] & 0xffff0000u);
            n2 = fmaf(x0, x0, n2);
            n2 = fmaf(x1, x1, n2);
          }
        }
        // grid step 2^e in (2.5e-7, 5e-7] * (|x|^2 + max|c|^2)
        const float tt = 5e-7f * (n2 + cbmax);
        int e = ((__float_as_int(tt) >> 23) & 0xff) - 127;
        e = max(-126, min(126, e));
        const float s = __int_as_float((127 - e) << 23);
        const float m2s = -2.f * s;
        uint8_t *a = sm.a[t];
        if constexpr (DSUB == 4) {   // (x' | x'), (x' | |x|^2 s, s, s, s)
          const uint32_t o0 = bf16_pair(__uint_as_float(xv[t][0].x << 16) * m2s, __uint_as_float(xv[t][0].x & 0xffff0000u) * m2s);
          const uint32_t o1 = bf16_pair(__uint_as_float(xv[t][0].y << 16) * m2s, __uint_as_float(xv[t][0].y & 0xffff0000u) * m2s);
          *reinterpret_cast<uint4 *>(a + tl_off<128>(r, 0)) = make_uint4(o0, o1, o0, o1);
          *reinterpret_cast<uint4 *>(a + tl_off<128>(r, 1)) = make_uint4(o0, o1, bf16_pair(n2 * s, s), bf16_pair(s, s));
          continue;
        }
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t w4[4] = {xv[t][i].x, xv[t][i].y, xv[t][i].z, xv[t][i].w};
          uint32_t o[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o[k] = bf16_pair(__uint_as_float(w4[k] << 16) * m2s, __uint_as_float(w4[k] & 0xffff0000u) * m2s);
          const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<uint4 *>(a + tl_off<128>(r, i)) = ov;
          *reinterpret_cast<uint4 *>(a + tl_off<128>(r, i + NCH)) = ov;
          *reinterpret_cast<uint4 *>(a + tl_off<128>(r, i + 2 * NCH)) = ov;
        }
        *reinterpret_cast<uint4 *>(a + tl_off<128>(r, 3 * NCH)) =
            make_uint4(bf16_pair(n2 * s, s), bf16_pair(s, s), 0u, 0u);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      t5_arrive(&sm.afull);
    }
  } else if (warp == TL_LOAD_WARP) {
    // ---- codebook blocks, every block for every pair, through the B ring
    if (lane == 0) {
      for (int it = 0, k = 0; it < items; ++it) {
        for (int blk = 0; blk < nblk; ++blk, ++k) {
          const int st = k % TL_BS;
          if (k >= TL_BS) t5_wait(&sm.bempty[st], ((k / TL_BS) - 1) & 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(t5_smem(&sm.bfull[st])),
                       "r"(TL_BBLK) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  t5_smem(sm.b[st])),
              "l"(bimg + (int64_t)blk * TL_BBLK), "r"(TL_BBLK), "r"(t5_smem(&sm.bfull[st]))
              : "memory");
        }
      }
    }
  } else if (warp == TL_MMA_WARP) {
    // ---- MMA issuer: kind::f16, bf16 A/B, fp32 D, K-major, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TL_NB >> 3) << 17) | (8u << 24);
    for (int it = 0, k = 0; it < items; ++it) {
      t5_wait(&sm.afull, it & 1);
      for (int blk = 0; blk < nblk; ++blk, ++k) {
        const int st = k % TL_BS, buf = k & 1;
        t5_wait(&sm.bfull[st], (k / TL_BS) & 1);
        if (k >= 2) t5_wait(&sm.dempty[buf], ((k >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        {
          const uint32_t bs = t5_smem(sm.b[st]);
          const int npt = min(2, ntl - 2 * it);   // tiles in this pair
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (t >= npt) break;
            // 512 columns, one CTA per SM: the allocation starts at column 0
            const uint32_t as = t5_smem(sm.a[t]), d = t * 256 + buf * 128;
#pragma unroll
            for (int ks = 0; ks <= KD; ++ks) {
              const uint32_t ao = (ks >> 2) * (128 * 128) + (ks & 3) * 32, bo = (ks >> 2) * (TL_NB * 128) + (ks & 3) * 32;
              t5_mma_w(d, t5_desc(as + ao), t5_desc(bs + bo), idesc, ks > 0);
            }
          }
          t5_commit_w(&sm.bempty[st]);
          if (blk == nblk - 1) t5_commit_w(&sm.aempty);
          t5_commit_w(&sm.dfull[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue: warps 4-7 tile 0, 8-11 tile 1 (lanes 32 (w % 4).. of its
    // accumulators); best (key, block) of the thread's sub-vector over the blocks
    const int ew = warp - TL_PROD, q = warp & 3, t = ew >> 2;
    const int r = 32 * q + lane;
    for (int it = 0, k = 0; it < items; ++it) {
      uint32_t best = 0xffffffffu;
      int bblk = 0;
      const bool live = t < ntl - 2 * it;   // a single last tile: the tile-1 warps only keep the barrier count
      for (int blk = 0; blk < nblk; ++blk, ++k) {
        const int buf = k & 1;
        t5_wait(&sm.dfull[buf], (k >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (!live) {
          t5_arrive(&sm.dempty[buf]);
          continue;
        }
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + t * 256 + buf * 128;
        uint32_t v0[32], v1[32], v2[32], v3[32];
        t5_ld32(tq, v0);
        t5_ld32(tq + 32, v1);
        t5_ld_wait(v0, v1);
        t5_ld32(tq + 64, v2);
        t5_ld32(tq + 96, v3);
        uint32_t bm = min(chunk_min(v0, mul), chunk_min(v1, mul) + 32u);
        t5_ld_wait(v2, v3);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        t5_arrive(&sm.dempty[buf]);
        bm = min(bm, min(chunk_min(v2, mul) + 64u, chunk_min(v3, mul) + 96u));
        if (bm < best) { best = bm; bblk = blk; }   // strict: the earlier block keeps ties
      }
      if (!live) continue;
      const int64_t sv = (tile0 + 2 * it + t) * 128 + r;
      const uint32_t code = (uint32_t)bblk * TL_NB + (best & 0xffu);
      if (code_bytes == 3) {   // whole rows of G codes (G consecutive lanes of this warp)
        sm.cw[ew][lane] = code;
        __syncwarp();
        if (lane % G == 0 && sv < sv_end) {
          const int64_t tok = sv / G;
          code_put_row(static_cast<uint8_t *>(codes), set * code_set_stride + (tok >> 4) * code_tile_stride +
                       (tok & 15) * code_row_stride, G, &sm.cw[ew][lane], 3);
        }
        __syncwarp();
      } else if (sv < sv_end) {
        const int64_t tok = sv / G;
        const int64_t off = set * code_set_stride + (tok >> 4) * code_tile_stride + (tok & 15) * code_row_stride + sv % G;
        if (code_bytes == 1) static_cast<uint8_t *>(codes)[off] = static_cast<uint8_t>(code);
        else if (code_bytes == 2) static_cast<uint16_t *>(codes)[off] = static_cast<uint16_t>(code);
        else if (code_bytes == 4) static_cast<int32_t *>(codes)[off] = (int32_t)code;
        else static_cast<int64_t *>(codes)[off] = code;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == TL_MMA_WARP) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace

// Returns ANTKV_EUNSUPPORTED (nothing launched) outside the configuration
// (d = 128, d_sub = 8, m <= 256, bf16 rows, no distance output); the caller
// then tries the mma.sync encoder.  ANTKV_NO_TC5_ENC=1 disables it (A/B).
int launch_encode_tc5(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride, int nsets,
                      const float *codebooks, int cb_mod, int m, int d_sub, void *codes, int code_bytes,
                      int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                      const float *d2, cudaStream_t st) {
  if (d != 128 || d_sub != 8 || m > 256 || m < 1 || d2 != nullptr || dtype != ANTKV_BF16)
    return ANTKV_EUNSUPPORTED;
  static int off = -1;
  if (off < 0) {
    const char *e = getenv("ANTKV_NO_TC5_ENC");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  if (off) return ANTKV_EUNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (x_set_stride & 7) || d != 128 ||
      (reinterpret_cast<uintptr_t>(codebooks) & 15))
    return ANTKV_EUNSUPPORTED;
  if (rows == 0 || nsets == 0) return ANTKV_OK;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (rows + T5_TOK - 1) / T5_TOK;
  const int64_t cps = nsets >= sms ? 1 : sms / nsets;
  int64_t per = (ntiles + cps - 1) / cps;
  if (per < 4) per = 4;
  dim3 grid((unsigned)((ntiles + per - 1) / per), (unsigned)nsets);
  // one 16-byte store per token: 1-byte codes, 16 per row, 16-byte aligned rows
  const int vec = code_bytes == 1 && code_row_stride == 16 && !(reinterpret_cast<uintptr_t>(codes) & 15) &&
                  !(code_set_stride & 15) && !(code_tile_stride & 15);
  // >= 116 KB: one CTA per SM (each allocates all 512 TMEM columns)
  const size_t smem = max(sizeof(T5Smem) + 1024, (size_t)116 * 1024);
  static bool attr[64] = {};
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaFuncSetAttribute(vq_encode_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  vq_encode_tc5_kernel<<<grid, T5_THREADS, smem, st>>>(
      reinterpret_cast<const uint16_t *>(X), rows, x_set_stride, codebooks, cb_mod, m, codes, code_bytes,
      code_set_stride, code_tile_stride, code_row_stride, per, vec, 256u);
  ANTKV_LAUNCH_CHECK("vq_encode_tc5_kernel");
  return ANTKV_OK;
}

// Long codebooks and 4-dim sub-vectors: d_sub 4 / 16 / 32, any m <= 65536,
// bf16 rows, no distance output (ANTKV_NO_TC5_ENC=1 disables it as well).
int launch_encode_tc5l(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride, int nsets,
                       const float *codebooks, int cb_mod, int m, int d_sub, void *codes, int code_bytes,
                       int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                       const float *d2, cudaStream_t st) {
  if (d != 128 || (d_sub != 4 && d_sub != 16 && d_sub != 32) || m < 1 || m > 65536 || d2 != nullptr ||
      dtype != ANTKV_BF16)
    return ANTKV_EUNSUPPORTED;
  if (code_bytes == 3 && m > 4096) return ANTKV_EUNSUPPORTED;
  static int off = -1;
  if (off < 0) {
    const char *e = getenv("ANTKV_NO_TC5_ENC");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  if (off) return ANTKV_EUNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (x_set_stride & 7) || (reinterpret_cast<uintptr_t>(codebooks) & 15))
    return ANTKV_EUNSUPPORTED;
  if (rows == 0 || nsets == 0) return ANTKV_OK;
  const int G = d / d_sub;
  const int nblk = (m + TL_NB - 1) / TL_NB;
  const int ncb = min(cb_mod, nsets);
  uint8_t *img = nullptr;
  float *blkmax = nullptr;
  cudaError_t e = scratch_alloc((void **)&img, (size_t)ncb * nblk * TL_BBLK, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&blkmax, sizeof(float) * ncb * nblk, st);
  if (e != cudaSuccess) return cuda_status(e, "encoder codebook image");
  if (d_sub == 32) tl_codebook_image_kernel<32><<<dim3(nblk, ncb), TL_NB, 0, st>>>(codebooks, m, img, nblk, blkmax);
  else if (d_sub == 16) tl_codebook_image_kernel<16><<<dim3(nblk, ncb), TL_NB, 0, st>>>(codebooks, m, img, nblk, blkmax);
  else tl_codebook_image_kernel<4><<<dim3(nblk, ncb), TL_NB, 0, st>>>(codebooks, m, img, nblk, blkmax);
  ANTKV_LAUNCH_CHECK("tl_codebook_image_kernel");
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (rows * G + 127) / 128;
  const int64_t cps = nsets >= sms ? 1 : sms / nsets;
  const int64_t per = (ntiles + cps - 1) / cps;
  dim3 grid((unsigned)((ntiles + per - 1) / per), (unsigned)nsets);
  const size_t smem = sizeof(TlSmem) + 1024;
  static bool attr[64] = {};
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaFuncSetAttribute(vq_encode_tc5l_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(vq_encode_tc5l_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(vq_encode_tc5l_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  const uint16_t *Xh = reinterpret_cast<const uint16_t *>(X);
  if (d_sub == 32)
    vq_encode_tc5l_kernel<32><<<grid, TL_THREADS, smem, st>>>(Xh, rows, x_set_stride, img, blkmax, ncb, m, nblk, codes,
                                                             code_bytes, code_set_stride, code_tile_stride,
                                                             code_row_stride, per, 256u);
  else if (d_sub == 16)
    vq_encode_tc5l_kernel<16><<<grid, TL_THREADS, smem, st>>>(Xh, rows, x_set_stride, img, blkmax, ncb, m, nblk, codes,
                                                             code_bytes, code_set_stride, code_tile_stride,
                                                             code_row_stride, per, 256u);
  else
    vq_encode_tc5l_kernel<4><<<grid, TL_THREADS, smem, st>>>(Xh, rows, x_set_stride, img, blkmax, ncb, m, nblk, codes,
                                                            code_bytes, code_set_stride, code_tile_stride,
                                                            code_row_stride, per, 256u);
  ANTKV_LAUNCH_CHECK("vq_encode_tc5l_kernel");
  cudaFreeAsync(img, st);
  cudaFreeAsync(blkmax, st);
  return ANTKV_OK;
}

}  // namespace antkv
