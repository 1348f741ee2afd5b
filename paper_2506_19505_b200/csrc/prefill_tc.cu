// Anchor-score column sums (Alg. 1 second pass, anchors.py:66-87,
// _ckernels.pyx:91-131) on the 5th-generation tensor cores: tcgen05.mma with
// operands in shared memory (bulk-copied, 128B-swizzled K-major tiles) and
// the logit tile accumulated in tensor memory.
//
// Each CTA owns 128 keys of one KV head and walks the query tiles of the
// heads in its group (causal: only tiles at or after its own).  The logit
// tile is computed TRANSPOSED, S^T[128 keys x 128 queries] = K . Q^T, so the
// epilogue thread that owns TMEM lane j owns key j and sums its column of A
// over the queries in registers — no cross-thread reduction:
//   A_ij = exp(S_ij - M_i) / L_i = 2^(S_ij log2e - (M_i log2e + log2 L_i)),
//   ans_v_j += A_ij,  ans_k_j += A_ij (1 - A_ij) ||q_i||.
// Numerics as the mma.sync kernels (prefill_mma.cu): S from two-part fp16
// splits of power-of-two-scaled tiles (Kh.Qh + Kh.Ql + Kl.Qh, float32
// accumulation), scale removed exactly.
//
// Warp roles (2 + 4 TC_EG warps): warp 0 lane 0 issues the bulk copies (K
// tile once, Q tiles with their 1 KB of packed column statistics through a
// 3-stage ring); warp 1 owns the TMEM allocation and issues the 24 MMAs per
// query tile warp-wide (elect.sync); the other warps are the epilogue —
// warps w, w + 4, ... share TMEM lanes 32 (w % 4) .. + 31 and split the 128
// query columns into TC_EG groups.  TMEM: two 128-column logit buffers (the MMAs of tile t + 1
// overlap the exponentials of tile t) and the K tile's fp16 parts (128
// columns), which the epilogue warps copy there once so the MMAs read only
// the Q tile from shared memory (at N = 128 both operands from shared memory
// would saturate its bandwidth).
#include "common.cuh"

namespace antkv {

constexpr int TC_ROWS = 128;                 // keys / queries per tile
constexpr int TC_PART = TC_ROWS * 128 * 2;   // one fp16 part of a tile: 32 KB
constexpr int TC_TILE = 2 * TC_PART;         // hi | lo
#ifndef TC_EG
#define TC_EG 4                               // epilogue column groups per TMEM lane quarter (16 warps: 8.62 -> 8.52 ms at 32K)
#endif
constexpr int TC_WARPS = 2 + 4 * TC_EG;
constexpr int TC_THREADS = 32 * TC_WARPS;
constexpr int TC_EPI = 4 * TC_EG * 32;        // epilogue threads
constexpr int TC_ECH = 4 / TC_EG;             // 32-column chunks per epilogue warp
constexpr uint32_t TC_AH = 256, TC_AL = 320; // TMEM columns of the K tile (A operand): hi, lo

// Byte offset of element (row, k) in one 128B-swizzled K-major part of R
// rows: 64-column atoms of [R rows][128 B], 16-byte chunks XOR-ed with
// row & 7 (8-row groups 1024 B apart).
template <int R = TC_ROWS>
__host__ __device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return (k >> 6) * (R * 128) + row * 128 + ((((k & 63) >> 3) ^ (row & 7)) << 4) + (k & 7) * 2;
}

__device__ __forceinline__ uint32_t tc_smem(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tc_mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void tc_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tc_bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// Shared-memory matrix descriptor: K-major, 128B swizzle, 8-row groups
// 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane (no wait: pair with
// tc_ld_wait before using v)
__device__ __forceinline__ void tc_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
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
__device__ __forceinline__ void tc_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tc_ex2(float x) {   // 2^x, x <= 0 here (-inf -> 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (FFMA2 / FADD2 on sm_100): each lane rounds exactly as
// the scalar instruction would, at half the issue slots.
__device__ __forceinline__ float2 tc_ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mov.b64 rc, {%6,%7};\n"
      " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 tc_fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0,%1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 tc_fsub2(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n"
      " sub.rn.f32x2 rd, ra, rb;\n mov.b64 {%0,%1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// 1 / x for a normal power of two x (the tile scales of tc_pow2_scale): exact
__device__ __forceinline__ float tc_pow2_inv(float x) { return __int_as_float(0x7F000000 - __float_as_int(x)); }

// 32 consecutive 32-bit columns of this thread's TMEM lane <- r[0..31]
__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// Warp-wide forms: every lane executes the call with the same operands, one
// elected lane issues.  Called from converged, warp-uniform code the operands
// stay in uniform registers, so no per-instruction waterfall loop is needed
// around UTCHMMA (the lane == 0 forms get one: ELECT + BRA.U.ANY each).
__device__ __forceinline__ void tc_mma_f16_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit_w(uint32_t bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Power of two that maps the magnitude mx into [2^13, 2^14) (1 for mx == 0).
__device__ __forceinline__ float tc_pow2_scale(float mx) {
  if (!(mx > 0.f)) return 1.f;
  int e = (__float_as_int(mx) >> 23) & 0xff;
  e = e < 14 ? 14 : (e > 266 ? 266 : e);
  return __int_as_float((267 - e) << 23);
}

// X [heads][rows][128] float32 -> [heads][ceil(rows/R)][hi | lo] fp16 parts
// of x * scale in the 128B-swizzled K-major layout, scale [heads][tiles].
template <int R>
__global__ void __launch_bounds__(256)
presplit_sw128_kernel(const float *__restrict__ X, int rows, uint8_t *__restrict__ tiles,
                      float *__restrict__ scales) {
  constexpr int PART = R * 128 * 2;
  __shared__ float red[8];
  const int h = blockIdx.y, tile = blockIdx.x, nt = gridDim.x;
  const float *src = X + (int64_t)h * rows * 128;
  uint8_t *dst = tiles + ((int64_t)h * nt + tile) * (2 * PART);
  float mx = 0.f;
  for (int e = threadIdx.x; e < R * 32; e += 256) {
    const int r = tile * R + (e >> 5);
    if (r < rows) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)r * 128) + (e & 31));
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, red[i]);
  const float sc = tc_pow2_scale(mx);
  if (threadIdx.x == 0) scales[(int64_t)h * nt + tile] = sc;
  // one 16-byte chunk (8 elements) of one row per thread and step
  for (int e = threadIdx.x; e < R * 16; e += 256) {
    const int r = e >> 4, c = e & 15, gr = tile * R + r;
    float x[8];
    if (gr < rows) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)gr * 128 + 8 * c));
      const float4 b = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)gr * 128 + 8 * c + 4));
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = 0.f;
    }
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float p = x[2 * i] * sc, q = x[2 * i + 1] * sc;
      const __half ph = __float2half_rn(p), qh = __float2half_rn(q);
      const __half pl = __float2half_rn(p - __half2float(ph)), ql = __float2half_rn(q - __half2float(qh));
      __half2 hh = __halves2half2(ph, qh), ll = __halves2half2(pl, ql);
      hi[i] = *reinterpret_cast<uint32_t *>(&hh);
      lo[i] = *reinterpret_cast<uint32_t *>(&ll);
    }
    const uint32_t off = sw128_off<R>(r, 8 * c);
    *reinterpret_cast<uint4 *>(dst + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4 *>(dst + PART + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// Per query: c_i = M_i log2e + log2 L_i (+inf beyond n_q) and ||q_i||,
// [heads][nqt * 128] laid out per column pair p as the float4
// (-c_2p, -c_2p+1, |q_2p|, |q_2p+1|): the anchor-score epilogue's packed
// operands, bulk-copied next to each Q tile (1 KB per tile).
__global__ void ans_tc_stats_kernel(const float *__restrict__ M, const float *__restrict__ L,
                                    const float *__restrict__ qn, int heads, int n_q, int padded,
                                    float *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)heads * padded) return;
  const int h = (int)(i / padded), q = (int)(i % padded);
  float c = INFINITY, nq = 0.f;
  if (q < n_q) {
    const int64_t k = (int64_t)h * n_q + q;
    c = M[k] * 1.4426950408889634f + log2f(L[k]);
    nq = qn[k];
  }
  float *o = out + 2 * ((int64_t)h * padded + (q & ~1)) + (q & 1);
  o[0] = -c;
  o[2] = nq;
}

constexpr int TC_QS = 3;      // Q stages; stage 2 first carries the K tile (until it is in TMEM)
struct AnsTcSmem {
  uint8_t q[TC_QS][TC_TILE];  // 1024-aligned (the struct is placed at a 1024 boundary)
  float stat[TC_QS][2 * TC_ROWS];   // the Q stage's column statistics (ans_tc_stats_kernel layout)
  float red[TC_EG - 1][2][TC_ROWS];   // column groups 1.. : (sv, skn) per key
  unsigned long long kbar, aready, qfull[TC_QS], qempty[TC_QS], tfull[2], tempty[2];
  uint32_t tmem;
};

__global__ void __launch_bounds__(TC_THREADS, 1)
ans_tc_kernel(const uint8_t *__restrict__ Qt, const float *__restrict__ Qsc, const uint8_t *__restrict__ Kt,
              const float *__restrict__ Ksc, const float *__restrict__ stats, int group, int sum_group,
              int n_q, int n_k, int causal, float *__restrict__ ans_k, float *__restrict__ ans_v) {
  extern __shared__ uint8_t tc_raw[];
  AnsTcSmem &sm = *reinterpret_cast<AnsTcSmem *>(tc_raw + ((1024 - (tc_smem(tc_raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = blockIdx.x, ho = blockIdx.y;                  // key tile, output head
  const int nqt = (n_q + TC_ROWS - 1) / TC_ROWS, nkt = gridDim.x;
  const int qt0 = causal ? kt : 0;
  const int per_head = nqt - qt0 > 0 ? nqt - qt0 : 0;
  const int items = sum_group * per_head;
  const int hk = (ho * sum_group) / group;                     // KV head of this group
  const int padded = nqt * TC_ROWS;

  if (threadIdx.x == 0) {
    tc_mbar_init(tc_smem(&sm.kbar), 1);
    tc_mbar_init(tc_smem(&sm.aready), TC_EPI);
    for (int s = 0; s < TC_QS; ++s) {
      tc_mbar_init(tc_smem(&sm.qfull[s]), 1);
      tc_mbar_init(tc_smem(&sm.qempty[s]), 1 + TC_EPI / 32);   // the MMAs' commit + each epilogue warp
    }
    for (int s = 0; s < 2; ++s) {
      tc_mbar_init(tc_smem(&sm.tfull[s]), 1);
      tc_mbar_init(tc_smem(&sm.tempty[s]), TC_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc_smem(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  // Producer and MMA warps run their loops warp-wide (aligned barriers stay
  // convergent); lane 0 issues the copies / MMAs.
  if (warp == 0) {                  // ---- bulk-copy producer
    if (items > 0) {
      if (lane == 0) {
        tc_expect_tx(tc_smem(&sm.kbar), TC_TILE);
        tc_bulk(tc_smem(sm.q[TC_QS - 1]), Kt + ((int64_t)hk * nkt + kt) * TC_TILE, TC_TILE, tc_smem(&sm.kbar));
      }
      for (int it = 0; it < items; ++it) {
        const int s = it % TC_QS;
        if (it >= TC_QS) tc_wait(tc_smem(&sm.qempty[s]), ((it / TC_QS) - 1) & 1);
        else if (s == TC_QS - 1) tc_wait(tc_smem(&sm.aready), 0);   // the K tile has left stage 2
        const int h = ho * sum_group + it / per_head, qt = qt0 + it % per_head;
        if (lane == 0) {
          tc_expect_tx(tc_smem(&sm.qfull[s]), TC_TILE + 8 * TC_ROWS);
          tc_bulk(tc_smem(sm.q[s]), Qt + ((int64_t)h * nqt + qt) * TC_TILE, TC_TILE, tc_smem(&sm.qfull[s]));
          tc_bulk(tc_smem(sm.stat[s]), stats + 2 * ((int64_t)h * padded + qt * TC_ROWS), 8 * TC_ROWS,
                  tc_smem(&sm.qfull[s]));
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {           // ---- MMA issuer
    if (items > 0) {
      // kind::f16, fp16 A/B, fp32 D, both K-major, N = 128 (bits 17-22), M = 128 (bits 24-28)
      const uint32_t idesc = (1u << 4) | ((uint32_t)(TC_ROWS >> 3) << 17) | ((uint32_t)(TC_ROWS >> 4) << 24);
      tc_wait(tc_smem(&sm.aready), 0);   // the K tile is in TMEM (columns 256..383)
      // 512 columns on a one-CTA-per-SM kernel: the allocation starts at 0, and
      // a constant keeps the MMA operands uniform (warp-wide elect issue)
      if (tmem != 0) __trap();
      constexpr uint32_t tm = 0;
      for (int it = 0; it < items; ++it) {
        const int s = it % TC_QS, b = it & 1;
        tc_wait(tc_smem(&sm.qfull[s]), (it / TC_QS) & 1);
        if (it >= 2) tc_wait(tc_smem(&sm.tempty[b]), ((it >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t qa = tc_smem(sm.q[s]), d = tm + b * TC_ROWS;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * (TC_ROWS * 128) + (kk & 3) * 32;
          const uint32_t kh = tm + TC_AH + 8 * kk, kl = tm + TC_AL + 8 * kk;
          const uint64_t qh = sw128_desc(qa + off), ql = sw128_desc(qa + TC_PART + off);
          tc_mma_f16_ts_w(d, kh, qh, idesc, kk > 0);
          tc_mma_f16_ts_w(d, kh, ql, idesc, 1);
          tc_mma_f16_ts_w(d, kl, qh, idesc, 1);
        }
        tc_commit_w(tc_smem(&sm.qempty[s]));
        tc_commit_w(tc_smem(&sm.tfull[b]));
        __syncwarp();
      }
    }
  } else {                          // ---- epilogue: 4 TC_EG warps
    const int quarter = warp & 3, cg = (warp - 2) >> 2;     // TMEM lanes, column group
    const int key_local = 32 * quarter + lane;
    const int key = kt * TC_ROWS + key_local;
    if (items > 0) {
      // K tile -> TMEM as the MMA's A operand: lane = key row, column c = the
      // fp16 pair (2c, 2c+1); the four 32-column pieces (part, 64-dim half)
      // are dealt to the column groups
      tc_wait(tc_smem(&sm.kbar), 0);
#pragma unroll
      for (int pc = cg * TC_ECH; pc < (cg + 1) * TC_ECH; ++pc) {
        const int prt = pc >> 1, cb = pc & 1;
        const uint8_t *part = sm.q[TC_QS - 1] + prt * TC_PART;
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {   // 8 chunks of 8 elements = 64 dims
          const uint4 v = *reinterpret_cast<const uint4 *>(part + sw128_off<>(key_local, 64 * cb + 8 * c));
          r[4 * c] = v.x;
          r[4 * c + 1] = v.y;
          r[4 * c + 2] = v.z;
          r[4 * c + 3] = v.w;
        }
        tc_st32(tmem + ((uint32_t)(32 * quarter) << 16) + (prt ? TC_AL : TC_AH) + 32 * cb, r);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      tc_arrive(tc_smem(&sm.aready));
    }
    const float ksc_inv = tc_pow2_inv(__ldg(Ksc + (int64_t)hk * nkt + kt));   // powers of two: exact
    float sv = 0.f, skn = 0.f;   // skn = -(the A(1 - A)|q| sum), accumulated negated (see below)
    // item it = (head gq of the group, query tile qt0 + qi); its column
    // statistics arrive with the Q tile (stage it % TC_QS; no epilogue-wide
    // barrier per item), the next item's scale is loaded one item ahead
    int gq = 0, qi = 0;
    float nqsc = 1.f;
    if (items > 0) nqsc = __ldg(Qsc + (int64_t)(ho * sum_group) * nqt + qt0);
    for (int it = 0; it < items; ++it) {
      const int s = it & 1, sq = it % TC_QS;
      const int qt = qt0 + qi;
      const float u = 1.4426950408889634f * ksc_inv * tc_pow2_inv(nqsc);
      if (++qi == per_head) {
        qi = 0;
        ++gq;
      }
      if (it + 1 < items) nqsc = __ldg(Qsc + (int64_t)(ho * sum_group + gq) * nqt + qt0 + qi);
      tc_wait(tc_smem(&sm.qfull[sq]), (it / TC_QS) & 1);   // long complete: the MMAs of this item waited on it
      tc_wait(tc_smem(&sm.tfull[s]), (it >> 1) & 1);
      tc_fence_after();
      const bool diag = causal && qt == kt;
      // this tile's share (two-level sums over long contexts), columns in
      // packed fp32 pairs: a = 2^(v u - c); tv += a; tkn += (a a - a) |q|,
      // i.e. -(A(1 - A)|q|) — fma(a, a, -a) = -fma(-a, a, a) exactly, so the
      // negated sum is the scalar one with its sign flipped
      float2 tv2 = make_float2(0.f, 0.f), tk2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int cb = 0; cb < TC_ECH; ++cb) {
        const int c0 = 32 * (cg * TC_ECH + cb);
        float v[32];
        tc_ld32(tmem + ((uint32_t)(32 * quarter) << 16) + s * TC_ROWS + c0, v);
        if (diag) {                 // keys after the query are masked (causal): A = 0
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i < key_local) v[i] = -INFINITY;
        }
        const float4 *st4 = reinterpret_cast<const float4 *>(&sm.stat[sq][2 * c0]);
        const float2 uu = make_float2(u, u);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float4 st = st4[i >> 1];   // (-c, -c', |q|, |q'|) of columns c0 + i, c0 + i + 1
          const float2 e = tc_ffma2(make_float2(v[i], v[i + 1]), uu, make_float2(st.x, st.y));
          const float2 a = make_float2(tc_ex2(e.x), tc_ex2(e.y));
          tv2 = tc_fadd2(tv2, a);
          const float2 w = tc_ffma2(a, a, make_float2(-a.x, -a.y));
          tk2 = tc_ffma2(w, make_float2(st.z, st.w), tk2);
        }
      }
      sv += tv2.x + tv2.y;
      skn += tk2.x + tk2.y;
      tc_fence_before();
      tc_arrive(tc_smem(&sm.tempty[s]));
      __syncwarp();
      if (lane == 0) tc_arrive(tc_smem(&sm.qempty[sq]));   // this warp is done with the stage's statistics
    }
    // combine the two column halves of each key
    if (cg > 0) {
      sm.red[cg - 1][0][key_local] = sv;
      sm.red[cg - 1][1][key_local] = skn;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI) : "memory");
    if (cg == 0 && key < n_k) {
#pragma unroll
      for (int gi = 0; gi < TC_EG - 1; ++gi) {
        sv += sm.red[gi][0][key_local];
        skn += sm.red[gi][1][key_local];
      }
      ans_v[(int64_t)ho * n_k + key] = sv;
      ans_k[(int64_t)ho * n_k + key] = -skn;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int launch_ans_tc(const float *Qs, const float *Kr, const float *M, const float *L, const float *qn,
                  int heads, int kv_heads, int sum_group, int n_q, int n_k, int d, int causal,
                  float *ans_k, float *ans_v, cudaStream_t st) {
  if (d != 128) return ANTKV_EUNSUPPORTED;
  if (getenv("ANTKV_NO_TCGEN05")) return ANTKV_EUNSUPPORTED;
  if (n_k == 0) return ANTKV_OK;
  const int nqt = ceil_div(n_q, TC_ROWS), nkt = ceil_div(n_k, TC_ROWS);
  uint8_t *qt = nullptr, *kt = nullptr;
  float *qsc = nullptr, *ksc = nullptr;
  float *stats = nullptr;
  cudaError_t e = scratch_alloc((void **)&qt, (size_t)heads * (nqt ? nqt : 1) * TC_TILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&kt, (size_t)kv_heads * nkt * TC_TILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&qsc, sizeof(float) * (size_t)heads * (nqt ? nqt : 1), st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&ksc, sizeof(float) * (size_t)kv_heads * nkt, st);
  if (e == cudaSuccess)
    e = scratch_alloc((void **)&stats, 2 * sizeof(float) * (size_t)heads * (nqt ? nqt : 1) * TC_ROWS, st);
  if (e != cudaSuccess) return cuda_status(e, "anchor-score tile scratch");
  if (nqt > 0) {
    presplit_sw128_kernel<TC_ROWS><<<dim3(nqt, heads), 256, 0, st>>>(Qs, n_q, qt, qsc);
    const int64_t ns = (int64_t)heads * nqt * TC_ROWS;
    ans_tc_stats_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(M, L, qn, heads, n_q, nqt * TC_ROWS,
                                                                       stats);
  }
  presplit_sw128_kernel<TC_ROWS><<<dim3(nkt, kv_heads), 256, 0, st>>>(Kr, n_k, kt, ksc);
  const int smem = (int)sizeof(AnsTcSmem) + 1024;
  cudaFuncSetAttribute(ans_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ans_tc_kernel<<<dim3(nkt, heads / sum_group), TC_THREADS, smem, st>>>(
      qt, qsc, kt, ksc, stats, heads / kv_heads, sum_group, n_q, n_k, causal, ans_k, ans_v);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(qt, st);
  cudaFreeAsync(kt, st);
  cudaFreeAsync(qsc, st);
  cudaFreeAsync(ksc, st);
  cudaFreeAsync(stats, st);
  if (le != cudaSuccess) return cuda_status(le, "ans_tc_kernel");
  return ANTKV_OK;
}


// ============================================================================
// Flash attention with the (O, L, M) auxiliaries (attention.py:146-169,
// _ckernels.pyx:10-88) on tcgen05, for bf16-exact V (the prefill path with
// bf16 inputs).  CTA = (head, 128 queries): the query tile's fp16 parts live
// in TMEM as the A operand of S = Q.K^T (M = 128 queries, N = 128 keys per
// tile — below N = 128 a tcgen05.mma runs at half rate, measured); each
// softmax thread owns one query row (its TMEM lane), keeps a lazily raised
// reference max (rescale only when a tile's max exceeds it by 2^8, so P <=
// 2^8 keeps exact bf16 parts) and the exact running max for M, and writes
// P's bf16 parts back over its S columns as the A operand of O += P.V
// (N = 128 dims, B = the V^T tile).  Products are the mma.sync kernel's
// two-part splits (S: fp16 parts of power-of-two-scaled tiles, three
// products; P.V: bf16 parts of P against exact bf16 V, two products),
// float32 accumulation in TMEM.
//
// Warps: 0 bulk-copy producer (two rings of two stages: K hi | K lo, 64 KB,
// freed as soon as S(t) completes; V^T, 32 KB, freed by P.V(t)), 1 TMEM owner + MMA issuer, warp-wide
// with elect.sync so the operands stay uniform (S of tile t is issued before P.V of
// tile t - 1 so the tensor core works while the softmax of t - 1 runs), 2-17
// softmax: warps w, w + 4, w + 8, w + 12 own the same 32 rows (TMEM lanes)
// and take 32 key columns each, exchanging quarter-row maxima through shared
// memory (16 softmax warps rather than 8: with two per scheduler the
// exponentials could not keep up with S(t + 1), tensor pipe 62 %).  TMEM
// columns: S/P buffers 0 and 128, O 256..383,
// Q parts 384..511.  Per 16-key step kk the P parts sit at columns 16 kk
// (hi) and 16 kk + 8 (lo) of the buffer, so the 32 columns a softmax chunk
// writes are exactly the S columns it has just read.
constexpr int FT_KR = 128;                   // keys per tile
constexpr int FT_KPART = FT_KR * 128 * 2;    // 32 KB (one fp16 part of a K tile)
constexpr int FT_VTILE = 128 * FT_KR * 2;    // 32 KB (V^T bf16)
constexpr int FT_NS = 2;                     // stages of each ring (K: 64 KB, V^T: 32 KB)
constexpr int FT_SOFT = 16;                  // softmax warps: 4 per TMEM lane quarter, 32 key columns each
constexpr int FT_THREADS = (2 + FT_SOFT) * 32;
constexpr uint32_t FT_O = 256, FT_QH = 384, FT_QL = 448;

struct FlashTcSmem {
  uint8_t k[FT_NS][2 * FT_KPART];   // K hi | K lo, released when S(t) completes
  uint8_t v[FT_NS][FT_VTILE];       // V^T, released when P.V(t) completes
  unsigned long long kfull[FT_NS], kempty[FT_NS], vfull[FT_NS], vempty[FT_NS];
  unsigned long long sfull[2], pfull[2], pvdone[2], qready;
  float xm[2][4][TC_ROWS];   // [buffer][column quarter][row]: quarter-row maxima
  float lx[4][TC_ROWS];      // [column quarter][row]: quarter-row sums at the end
#ifdef FT_TRACE
  uint32_t tr_sready[64], tr_pdone[64], tr_pfirst[64], tr_mwake[64], tr_pvissued[64], tr_sissued[64];
#endif
  uint32_t tmem;
};

// V [heads][rows][128] float32 (bf16-exact) -> [heads][ceil(rows/128)] tiles
// V^T[128 dims][128 keys] bf16, K-major, 128B-swizzled: the B operand of O +=
// P.V.
template <typename T>
__global__ void __launch_bounds__(256)
presplit_vt_kernel(const T *__restrict__ V, int rows, uint8_t *__restrict__ tiles) {
  const int h = blockIdx.y, tile = blockIdx.x, nt = gridDim.x;
  const T *src = V + (int64_t)h * rows * 128;
  uint8_t *dst = tiles + ((int64_t)h * nt + tile) * FT_VTILE;
  // thread -> (dim, chunk of 8 keys); consecutive threads take consecutive dims
  for (int e = threadIdx.x; e < 128 * 16; e += 256) {
    const int dim = e & 127, c = e >> 7;
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k0 = tile * FT_KR + 8 * c + 2 * i;
      const float a = k0 < rows ? (float)src[(int64_t)k0 * 128 + dim] : 0.f;
      const float b = k0 + 1 < rows ? (float)src[(int64_t)(k0 + 1) * 128 + dim] : 0.f;
      const __nv_bfloat162 v2 = __floats2bfloat162_rn(a, b);
      w[i] = *reinterpret_cast<const uint32_t *>(&v2);
    }
    *reinterpret_cast<uint4 *>(dst + sw128_off<128>(dim, 8 * c)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void __launch_bounds__(FT_THREADS, 1)
flash_tc_kernel(const uint8_t *__restrict__ Qt, const float *__restrict__ Qsc, const uint8_t *__restrict__ Kt,
                const float *__restrict__ Ksc, const uint8_t *__restrict__ Vt, int group, int n_q, int n_k,
                int causal, float *__restrict__ O, float *__restrict__ Lout, float *__restrict__ Mout) {
  extern __shared__ uint8_t ft_raw[];
  FlashTcSmem &sm = *reinterpret_cast<FlashTcSmem *>(ft_raw + ((1024 - (tc_smem(ft_raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = gridDim.x, h = blockIdx.y, hk = h / group;
  const int qt = nqt - 1 - blockIdx.x;              // long causal rows first
  const int q0 = qt * TC_ROWS;
  const int nkt = (n_k + FT_KR - 1) / FT_KR;
  const int last = causal ? min(q0 + TC_ROWS, n_q) - 1 : n_k - 1;
  const int T = min(nkt, last / FT_KR + 1);         // key tiles this CTA visits
  if (threadIdx.x == 0) {
    for (int s = 0; s < FT_NS; ++s) {
      tc_mbar_init(tc_smem(&sm.kfull[s]), 1);
      tc_mbar_init(tc_smem(&sm.kempty[s]), 1);
      tc_mbar_init(tc_smem(&sm.vfull[s]), 1);
      tc_mbar_init(tc_smem(&sm.vempty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc_mbar_init(tc_smem(&sm.sfull[b]), 1);
      tc_mbar_init(tc_smem(&sm.pfull[b]), FT_SOFT);   // one arrival per softmax warp
      tc_mbar_init(tc_smem(&sm.pvdone[b]), 1);
    }
    tc_mbar_init(tc_smem(&sm.qready), FT_SOFT);
#ifdef FT_TRACE
    for (int i = 0; i < 64; ++i) { sm.tr_pdone[i] = 0; sm.tr_pfirst[i] = 0xffffffffu; }
#endif
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc_smem(&sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  const uint8_t *Kg = Kt + (int64_t)hk * nkt * (2 * FT_KPART);
  const uint8_t *Vg = Vt + (int64_t)hk * nkt * FT_VTILE;

  if (warp == 0) {                  // ---- producer: K and V^T rings, in tile order
#ifdef FT_EXP_NOLOAD
    if (false)
#endif
    for (int t = 0; t < T; ++t) {
      const int st = t % FT_NS, ph = ((t / FT_NS) - 1) & 1;
      if (t >= FT_NS) tc_wait(tc_smem(&sm.kempty[st]), ph);
      if (lane == 0) {
        const uint32_t bar = tc_smem(&sm.kfull[st]);
        tc_expect_tx(bar, 2 * FT_KPART);
        tc_bulk(tc_smem(sm.k[st]), Kg + (int64_t)t * (2 * FT_KPART), 2 * FT_KPART, bar);
      }
      __syncwarp();
      if (t >= FT_NS) tc_wait(tc_smem(&sm.vempty[st]), ph);
      if (lane == 0) {
        const uint32_t bar = tc_smem(&sm.vfull[st]);
        tc_expect_tx(bar, FT_VTILE);
        tc_bulk(tc_smem(sm.v[st]), Vg + (int64_t)t * FT_VTILE, FT_VTILE, bar);
      }
      __syncwarp();
    }
  } else if (warp == 1) {           // ---- MMA issuer
    const uint32_t idS = (1u << 4) | ((uint32_t)(FT_KR >> 3) << 17) | ((uint32_t)(TC_ROWS >> 4) << 24);
    const uint32_t idPV = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                          ((uint32_t)(TC_ROWS >> 4) << 24);
    // all 512 columns belong to this CTA (one CTA per SM), so the allocation
    // starts at column 0: a constant keeps every MMA operand uniform
    if (tmem != 0) __trap();
    constexpr uint32_t tm = 0;
    tc_wait(tc_smem(&sm.qready), 0);
    for (int t = 0; t <= T; ++t) {
      if (t < T) {                  // S(t) = Q . K_t^T into buffer t & 1
        const int b = t & 1, st = t % FT_NS;
#ifndef FT_EXP_NOLOAD
        tc_wait(tc_smem(&sm.kfull[st]), (t / FT_NS) & 1);
#endif
        // buffer b still holds P(t-2), read by P.V(t-2): that MMA was issued
        // before this one and tcgen05.mma executes in issue order, so no wait
        tc_fence_after();
        {
          const uint32_t kb = tc_smem(sm.k[st]), d = tm + 128 * b;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * (FT_KR * 128) + (kk & 3) * 32;
            const uint64_t kh = sw128_desc(kb + off), kl = sw128_desc(kb + FT_KPART + off);
            tc_mma_f16_ts_w(d, tm + FT_QH + 8 * kk, kh, idS, kk > 0);
            tc_mma_f16_ts_w(d, tm + FT_QH + 8 * kk, kl, idS, 1);
            tc_mma_f16_ts_w(d, tm + FT_QL + 8 * kk, kh, idS, 1);
          }
          tc_commit_w(tc_smem(&sm.kempty[st]));
          tc_commit_w(tc_smem(&sm.sfull[b]));
#ifdef FT_TRACE
          if (lane == 0 && t < 64) sm.tr_sissued[t] = (uint32_t)clock();
#endif
        }
        __syncwarp();
      }
      if (t >= 1) {                 // O += P(t-1) . V_{t-1}
        const int u = t - 1, b = u & 1, st = u % FT_NS;
#ifndef FT_EXP_NOLOAD
        tc_wait(tc_smem(&sm.vfull[st]), (u / FT_NS) & 1);
#endif
        tc_wait(tc_smem(&sm.pfull[b]), (u >> 1) & 1);
        tc_fence_after();
#ifdef FT_TRACE
        if (lane == 0 && u < 64) sm.tr_mwake[u] = (uint32_t)clock();
#endif
        {
          const uint32_t vb = tc_smem(sm.v[st]);
#pragma unroll
          for (int kk = 0; kk < FT_KR / 16; ++kk) {
#ifdef FT_EXP_NOPV
            break;
#endif
            const uint32_t ph = tm + 128 * b + 16 * kk, pl = ph + 8;
            const uint64_t vh = sw128_desc(vb + (kk >> 2) * (128 * 128) + (kk & 3) * 32);
            tc_mma_f16_ts_w(tm + FT_O, ph, vh, idPV, (u > 0 || kk > 0) ? 1u : 0u);
            tc_mma_f16_ts_w(tm + FT_O, pl, vh, idPV, 1);
          }
          tc_commit_w(tc_smem(&sm.vempty[st]));
          tc_commit_w(tc_smem(&sm.pvdone[b]));
#ifdef FT_TRACE
          if (lane == 0 && u < 64) sm.tr_pvissued[u] = (uint32_t)clock();
#endif
        }
        __syncwarp();
      }
    }
  } else {                          // ---- softmax: warps w, w + 4, w + 8, w + 12 share rows, split columns
    const int quarter = warp & 3, cq = (warp - 2) >> 2, row = 32 * quarter + lane, qi = q0 + row;
    const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
    const int bar_id = 1 + quarter;                 // named barrier of the four warps of a row quarter
    {   // Q tile parts -> TMEM (A operand of S): column quarters 0, 1 the hi part, 2, 3 the lo part
      const int part = cq >> 1, cb = cq & 1;
      const uint8_t *qg = Qt + ((int64_t)h * nqt + qt) * TC_TILE + part * TC_PART;
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(qg + sw128_off<>(row, 64 * cb + 8 * c)));
        r[4 * c] = v.x;
        r[4 * c + 1] = v.y;
        r[4 * c + 2] = v.z;
        r[4 * c + 3] = v.w;
      }
      tc_st32(tmem + lane_base + (part ? FT_QL : FT_QH) + 32 * cb, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) tc_arrive(tc_smem(&sm.qready));
    }
    const float qs_inv = tc_pow2_inv(__ldg(Qsc + (int64_t)h * nqt + qt));
    float mref = -INFINITY, mex = -INFINITY, l = 0.f, lc = 0.f;
    float ksc_next = T > 0 ? __ldg(Ksc + (int64_t)hk * nkt) : 1.f;
    for (int t = 0; t < T; ++t) {
      const int b = t & 1, k0 = t * FT_KR + 32 * cq;   // first key of this quarter
      const uint32_t sb = tmem + lane_base + 128 * b + 32 * cq;
      const float u = 1.4426950408889634f * qs_inv * tc_pow2_inv(ksc_next);   // log2 units, exact scales
      if (t + 1 < T) ksc_next = __ldg(Ksc + (int64_t)hk * nkt + t + 1);
      tc_wait(tc_smem(&sm.sfull[b]), (t >> 1) & 1);
      tc_fence_after();
#ifdef FT_TRACE
      if (warp == 2 && lane == 0 && t < 64) sm.tr_sready[t] = (uint32_t)clock();
#endif
#ifdef FT_EXP_NOSOFT
      tc_fence_before();
      __syncwarp();
      if (lane == 0) tc_arrive(tc_smem(&sm.pfull[b]));
      continue;
#endif
      const bool full = (!causal || t * FT_KR + FT_KR - 1 <= q0) && t * FT_KR + FT_KR <= n_k;
      // pass 1: max of this quarter (raw accumulator; u > 0 commutes with max),
      // combined with the other three quarters through shared memory
      float mt;
      uint32_t c0[32];   // this quarter's 32 logits, kept for pass 2
      {
        tc_ld32_nowait(sb, c0);
        tc_ld_wait();
        if (!full) {     // one branch: masked keys become -inf for both passes
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (k0 + i >= n_k || (causal && k0 + i > qi)) c0[i] = 0xff800000u;
        }
        float m8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          m8[j] = fmaxf(fmaxf(__uint_as_float(c0[j]), __uint_as_float(c0[j + 8])),
                        fmaxf(__uint_as_float(c0[j + 16]), __uint_as_float(c0[j + 24])));
        const float pm = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        sm.xm[b][cq][row] = pm;
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        mt = fmaxf(fmaxf(sm.xm[b][0][row], sm.xm[b][1][row]), fmaxf(sm.xm[b][2][row], sm.xm[b][3][row])) * u;
      }
      mex = fmaxf(mex, mt);
      if (__any_sync(0xffffffffu, mt > mref + 8.f)) {   // same decision in the four warps of the rows
        const float mn = fmaxf(mref, mt);
        const float al = mref == -INFINITY ? 0.f : tc_ex2(mref - mn);
        l *= al;
        lc *= al;
        if (t > 0) {        // O holds P.V of earlier tiles: wait for the last one, rescale this quarter
          tc_wait(tc_smem(&sm.pvdone[(t - 1) & 1]), ((t - 1) >> 1) & 1);
          tc_fence_after();
          float ov[32];
          tc_ld32(tmem + lane_base + FT_O + 32 * cq, ov);
          uint32_t r[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(ov[i] * al);
          tc_st32(tmem + lane_base + FT_O + 32 * cq, r);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        mref = mn;
      }
      const float msub = mref == -INFINITY ? 0.f : mref;
      // pass 2: P in bf16 parts over the S columns read in pass 1 (key pairs
      // in packed fp32: FFMA2 for the exponent argument, FADD2 for the sums
      // and the lo residuals)
      float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      {
        const float2 uu = make_float2(u, u), mm = make_float2(-msub, -msub);
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {   // key pair (2i, 2i+1) of this quarter
          const float2 e = tc_ffma2(make_float2(__uint_as_float(c0[2 * i]), __uint_as_float(c0[2 * i + 1])), uu, mm);
          const float2 p = make_float2(tc_ex2(e.x), tc_ex2(e.y));
          ls2[i & 1] = tc_fadd2(ls2[i & 1], p);
          const __nv_bfloat162 hh = __floats2bfloat162_rn(p.x, p.y);
          const float2 r = tc_fsub2(p, __bfloat1622float2(hh));
          const __nv_bfloat162 lo = __floats2bfloat162_rn(r.x, r.y);
          // 16-key step s = i / 8 of this quarter: hi words at 16 s + (i % 8), lo at + 8
          w[16 * (i >> 3) + (i & 7)] = *reinterpret_cast<const uint32_t *>(&hh);
          w[16 * (i >> 3) + 8 + (i & 7)] = *reinterpret_cast<const uint32_t *>(&lo);
        }
        tc_st32(sb, w);
      }
      const float ls = (ls2[0].x + ls2[1].x) + (ls2[0].y + ls2[1].y);
      {   // l += ls, compensated (long contexts add thousands of tile sums)
        const float y = ls - lc, tt = l + y;
        lc = (tt - l) - y;
        l = tt;
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
#ifdef FT_TRACE
      if (lane == 0 && t < 64) {
        const uint32_t c = (uint32_t)clock();
        atomicMax(&sm.tr_pdone[t], c - sm.tr_sready[0]);
        atomicMin(&sm.tr_pfirst[t], c - sm.tr_sready[0]);
      }
#endif
      if (lane == 0) tc_arrive(tc_smem(&sm.pfull[b]));
    }
    // the row's l = the four quarters' sums
    sm.lx[cq][row] = l;
    asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
    const float lrow = (sm.lx[0][row] + sm.lx[1][row]) + (sm.lx[2][row] + sm.lx[3][row]);
    // O / l (this quarter's 32 columns), L relative to the exact max M (natural log)
    if (T > 0) {
      tc_wait(tc_smem(&sm.pvdone[(T - 1) & 1]), ((T - 1) >> 1) & 1);
      tc_fence_after();
    }
    const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
    float *orow = O + ((int64_t)h * n_q + qi) * 128 + 32 * cq;
    {
      float v[32];
      if (T > 0) {
        tc_ld32(tmem + lane_base + FT_O + 32 * cq, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      if (qi < n_q) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4 *>(orow + i) = make_float4(v[i] * inv, v[i + 1] * inv, v[i + 2] * inv, v[i + 3] * inv);
      }
    }
    if (qi < n_q && cq == 0) {
      const bool any = mex > -INFINITY;
      Mout[(int64_t)h * n_q + qi] = any ? mex * 0.6931471805599453f : -INFINITY;
      Lout[(int64_t)h * n_q + qi] = any ? lrow * exp2f(mref - mex) : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef FT_TRACE
  if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 2 && T >= 64) {
    const uint32_t b0 = sm.tr_sready[0];
    double ts = 0, tsf = 0, w1 = 0, iss = 0, sq = 0, per = 0, sw = 0;
    int n = 0;
    for (int t = 8; t < 60; ++t, ++n) {
      const uint32_t sr = sm.tr_sready[t] - b0, pd = sm.tr_pdone[t], pf = sm.tr_pfirst[t];
      ts += (double)(pd - sr);
      tsf += (double)(pf - sr);
      w1 += (double)(sm.tr_mwake[t] - b0 - pd);
      iss += (double)(sm.tr_pvissued[t] - sm.tr_mwake[t]);
      sq += (double)(sm.tr_sready[t + 2] - sm.tr_pvissued[t]);
      per += (double)(sm.tr_sready[t + 1] - sm.tr_sready[t]);
      sw += (double)(sm.tr_sready[t + 1] - b0 - pd);
    }
    for (int t = 20; t < 24; ++t)
      printf("FT_RAW cta %d t %d: S issued %d  S ready %d  P done first %d last %d  mma wake %d  PV issued %d\n",
             blockIdx.x, t, (int)(sm.tr_sissued[t] - sm.tr_sready[20]), (int)(sm.tr_sready[t] - sm.tr_sready[20]),
             (int)(sm.tr_pfirst[t] + b0 - sm.tr_sready[20]), (int)(sm.tr_pdone[t] + b0 - sm.tr_sready[20]),
             (int)(sm.tr_mwake[t] - sm.tr_sready[20]), (int)(sm.tr_pvissued[t] - sm.tr_sready[20]));
    printf("FT_TRACE cta %d: period %.0f  softmax(first/last) %.0f/%.0f  pfull->mma wake %.0f  pv+S issue %.0f  "
           "pv issued->S(t+2) ready %.0f  softmax done->S(t+1) ready %.0f\n",
           blockIdx.x, per / n, tsf / n, ts / n, w1 / n, iss / n, sq / n, sw / n);
  }
#endif
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// v_bf16: every V element is exactly a bf16 (the prefill path's bf16 inputs);
// otherwise the mma.sync kernel (which splits V) runs instead.
int launch_flash_tc(const float *Qs, const float *Kr, const float *V, int heads, int kv_heads, int n_q,
                    int n_k, int d, int dv, int causal, int v_bf16, float *O, float *L, float *M,
                    cudaStream_t st) {
  if (d != 128 || dv != 128 || !v_bf16) return ANTKV_EUNSUPPORTED;
  if (getenv("ANTKV_NO_TCGEN05")) return ANTKV_EUNSUPPORTED;
  if (n_q == 0) return ANTKV_OK;
  const int nqt = ceil_div(n_q, TC_ROWS), nkt = ceil_div(n_k, FT_KR);
  uint8_t *qt = nullptr, *kt = nullptr, *vt = nullptr;
  float *qsc = nullptr, *ksc = nullptr;
  cudaError_t e = scratch_alloc((void **)&qt, (size_t)heads * nqt * TC_TILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&kt, (size_t)kv_heads * nkt * 2 * FT_KPART, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&vt, (size_t)kv_heads * nkt * FT_VTILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&qsc, sizeof(float) * (size_t)heads * nqt, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&ksc, sizeof(float) * (size_t)kv_heads * nkt, st);
  if (e != cudaSuccess) return cuda_status(e, "attention tile scratch");
  presplit_sw128_kernel<TC_ROWS><<<dim3(nqt, heads), 256, 0, st>>>(Qs, n_q, qt, qsc);
  presplit_sw128_kernel<FT_KR><<<dim3(nkt, kv_heads), 256, 0, st>>>(Kr, n_k, kt, ksc);
  presplit_vt_kernel<float><<<dim3(nkt, kv_heads), 256, 0, st>>>(V, n_k, vt);
  const int smem = (int)sizeof(FlashTcSmem) + 1024;
  cudaFuncSetAttribute(flash_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  flash_tc_kernel<<<dim3(nqt, heads), FT_THREADS, smem, st>>>(qt, qsc, kt, ksc, vt, heads / kv_heads, n_q, n_k,
                                                              causal, O, L, M);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(qt, st);
  cudaFreeAsync(kt, st);
  cudaFreeAsync(vt, st);
  cudaFreeAsync(qsc, st);
  cudaFreeAsync(ksc, st);
  if (le != cudaSuccess) return cuda_status(le, "flash_tc_kernel");
  return ANTKV_OK;
}


// ============================================================================
// Fused prefill front end for bf16 inputs: RoPE (float64-reduced angles, as
// rope_rotate_kernel), the 1/sqrt(d) query scale and the fp16 hi/lo split of
// power-of-two-scaled 128-row tiles in one pass from the bf16 rows, plus the
// pre-RoPE query norms; V goes straight to its bf16 V^T tiles.  The attention
// and anchor-score kernels then share the same Q and K tiles.
__global__ void __launch_bounds__(256)
presplit_rope_kernel(const __nv_bfloat16 *__restrict__ X, const int64_t *__restrict__ positions, int heads_per_b,
                     int rows, double theta, float scale, uint8_t *__restrict__ tiles, float *__restrict__ scales,
                     float *__restrict__ norms) {
  constexpr int PER = TC_ROWS * 16 / 256;   // (row, 8-element chunk) items per thread
  __shared__ double freq[64];
  __shared__ float red[8];
  const int h = blockIdx.y, tile = blockIdx.x, nt = gridDim.x;
  const int b = h / heads_per_b;
  const __nv_bfloat16 *src = X + (int64_t)h * rows * 128;
  if (threadIdx.x < 64) freq[threadIdx.x] = rope_freq(theta, threadIdx.x, 128);
  __syncthreads();
  // item e = threadIdx.x + 256 j -> row e / 16, chunk e % 16 (16 lanes per row)
  float y[PER][8];
  float mx = 0.f;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = threadIdx.x + 256 * j, r = e >> 4, c = e & 15, gr = tile * TC_ROWS + r;
    float nrm = 0.f;
    if (gr < rows) {
      const uint4 raw = *reinterpret_cast<const uint4 *>(src + (int64_t)gr * 128 + 8 * c);
      const __nv_bfloat162 *p2 = reinterpret_cast<const __nv_bfloat162 *>(&raw);
      const double pos = (double)positions[(int64_t)b * rows + gr];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 x = __bfloat1622float2(p2[k]);
        nrm = fmaf(x.x, x.x, fmaf(x.y, x.y, nrm));
        float cs, sn;
        rope_cs(pos * freq[4 * c + k], cs, sn);
        y[j][2 * k] = (x.x * cs - x.y * sn) * scale;
        y[j][2 * k + 1] = (x.x * sn + x.y * cs) * scale;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) y[j][k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) mx = fmaxf(mx, fabsf(y[j][k]));
    if (norms) {
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      if (c == 0 && gr < rows) norms[(int64_t)h * rows + gr] = sqrtf(nrm);
    }
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, red[i]);
  const float sc = tc_pow2_scale(mx);
  if (threadIdx.x == 0) scales[(int64_t)h * nt + tile] = sc;
  uint8_t *dst = tiles + ((int64_t)h * nt + tile) * TC_TILE;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = threadIdx.x + 256 * j, r = e >> 4, c = e & 15;
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float p = y[j][2 * k] * sc, q = y[j][2 * k + 1] * sc;
      const __half ph = __float2half_rn(p), qh = __float2half_rn(q);
      const __half pl = __float2half_rn(p - __half2float(ph)), ql = __float2half_rn(q - __half2float(qh));
      __half2 hh = __halves2half2(ph, qh), ll = __halves2half2(pl, ql);
      hi[k] = *reinterpret_cast<uint32_t *>(&hh);
      lo[k] = *reinterpret_cast<uint32_t *>(&ll);
    }
    const uint32_t off = sw128_off<>(r, 8 * c);
    *reinterpret_cast<uint4 *>(dst + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4 *>(dst + TC_PART + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// Causal prefill of bf16 rows, d = 128: (O, M, L, ||q||) and the GQA-summed
// anchor scores from one set of tiles.  B is folded into the head index.
int prefill_tc_fused(const void *Q, const void *K, const void *V, int dtype, const int64_t *positions, int B,
                     int Hq, int Hkv, int n, int d, double theta, float *O, float *M, float *L, float *qn,
                     float *ans_k, float *ans_v, cudaStream_t st) {
  if (d != 128 || dtype != ANTKV_BF16) return ANTKV_EUNSUPPORTED;
  if (getenv("ANTKV_NO_TCGEN05")) return ANTKV_EUNSUPPORTED;
  if ((int64_t)B * n == 0) return ANTKV_OK;
  const int heads = B * Hq, kv_heads = B * Hkv, nt = ceil_div(n, TC_ROWS), group = Hq / Hkv;
  uint8_t *qt = nullptr, *kt = nullptr, *vt = nullptr;
  float *qsc = nullptr, *ksc = nullptr;
  float *stats = nullptr;
  cudaError_t e = scratch_alloc((void **)&qt, (size_t)heads * nt * TC_TILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&kt, (size_t)kv_heads * nt * TC_TILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&vt, (size_t)kv_heads * nt * FT_VTILE, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&qsc, sizeof(float) * (size_t)heads * nt, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&ksc, sizeof(float) * (size_t)kv_heads * nt, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&stats, 2 * sizeof(float) * (size_t)heads * nt * TC_ROWS, st);
  if (e != cudaSuccess) return cuda_status(e, "prefill tile scratch");
  const __nv_bfloat16 *Qb = reinterpret_cast<const __nv_bfloat16 *>(Q);
  const __nv_bfloat16 *Kb = reinterpret_cast<const __nv_bfloat16 *>(K);
  presplit_rope_kernel<<<dim3(nt, heads), 256, 0, st>>>(Qb, positions, Hq, n, theta, 1.f / sqrtf(128.f), qt,
                                                        qsc, qn);
  presplit_rope_kernel<<<dim3(nt, kv_heads), 256, 0, st>>>(Kb, positions, Hkv, n, theta, 1.f, kt, ksc, nullptr);
  presplit_vt_kernel<__nv_bfloat16><<<dim3(nt, kv_heads), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16 *>(V), n, vt);
  const int fsmem = (int)sizeof(FlashTcSmem) + 1024;
  cudaFuncSetAttribute(flash_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  flash_tc_kernel<<<dim3(nt, heads), FT_THREADS, fsmem, st>>>(qt, qsc, kt, ksc, vt, group, n, n, 1, O, L, M);
  const int64_t ns = (int64_t)heads * nt * TC_ROWS;
  ans_tc_stats_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(M, L, qn, heads, n, nt * TC_ROWS, stats);
  const int asmem = (int)sizeof(AnsTcSmem) + 1024;
  cudaFuncSetAttribute(ans_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, asmem);
  ans_tc_kernel<<<dim3(nt, kv_heads), TC_THREADS, asmem, st>>>(qt, qsc, kt, ksc, stats, group, group, n, n, 1,
                                                               ans_k, ans_v);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(qt, st);
  cudaFreeAsync(kt, st);
  cudaFreeAsync(vt, st);
  cudaFreeAsync(qsc, st);
  cudaFreeAsync(ksc, st);
  cudaFreeAsync(stats, st);
  if (le != cudaSuccess) return cuda_status(le, "fused prefill kernels");
  return ANTKV_OK;
}

}  // namespace antkv
