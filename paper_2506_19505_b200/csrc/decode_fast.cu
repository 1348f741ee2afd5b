// sm_100a decode-attention kernel for the 1-bit d8m256 configuration
// (d = 128, d_sub = 8, m <= 256, 4 query heads per KV head, contiguous
// positions).  Reference semantics: cache.py:168-178 (RoPE after
// reconstruction, softmax over the whole cache, A.V).
//
// Per 16-slot tile the score matrix S^T[16 tokens x 8 cols] and the output
// O^T[128 dims x 8 cols] are computed with m16n8k16 tensor-core MMAs whose
// operands come straight from registers:
//   * K_hat / V_hat rows are gathered from a shared-memory fp16 codebook
//     with ldmatrix (one 16-byte centroid row per lane address).  The
//     codebook is replicated 8x across the 16-byte bank groups so the eight
//     row addresses of every ldmatrix phase hit distinct banks.
//   * RoPE: rows 0-7 of a tile are tokens P0..P0+7 (group a), rows 8-15 are
//     P0+8..P0+15 (group b).  Each row is rotated by its offset g (0..7) in
//     its group with per-lane constant fp16 (cos, sin) pairs; the group base
//     rotation is applied to the query instead: columns 0-3 of the MMA carry
//     the 4 query heads in group a's frame R(p_q - P0) q, columns 4-7 in group
//     b's frame R(p_q - P0 - 8) q.  Frames advance by R(-16) per tile in fp32
//     (seeded with float64-reduced angles per warp).
//   * Group a tokens only see columns 0-3 and group b tokens only 4-7 (the
//     other products are masked), giving two independent online-softmax
//     streams that are merged with the CTA merge at the end.
// Code tiles (K codes 256 B + V codes 256 B per tile) are streamed into a
// shared-memory ring with cp.async.bulk (TMA bulk copies) and mbarriers.
// Anchor / window rows (the full-precision pool) are handled by extra CTAs
// on CUDA cores from fp16 pre-rotated K rows.
#include <stdlib.h>

#include "common.cuh"

namespace antkv {

constexpr int FK_WARPS = 4;
constexpr int FK_THREADS = 32 * FK_WARPS;
constexpr int FK_STAGES = 8;
constexpr int FK_TILE_BYTES = 512;                       // K 256 B + V 256 B
constexpr int FK_WARP_STAGE_BYTES = 2 * FK_TILE_BYTES;   // 2 tiles per warp per stage
constexpr int FK_STAGE_BYTES = FK_WARPS * FK_WARP_STAGE_BYTES;
constexpr int FK_MAX_WARP_WORDS = 64;                    // qmask words per warp (2048 slots)

struct __align__(128) FastSmem {
  uint4 cbK[256 * 8];                          // [code][copy] 16 B
  uint4 cbV[256 * 8];
  uint8_t ring[FK_STAGES][FK_STAGE_BYTES];
  uint32_t qm[FK_WARPS][FK_MAX_WARP_WORDS];
  float po[FK_WARPS][4][128];                  // pool-row partials per warp (4 heads)
  float pm[FK_WARPS][4], pl[FK_WARPS][4];
  unsigned long long full[FK_STAGES];
  unsigned long long empty[FK_STAGES];
  unsigned long long cbbar;
  int ticket;
  int upd[4];
};

struct MergeSmem {                             // aliases the ring after the loop
  float o[FK_WARPS][8][128];
  float m[FK_WARPS][8];
  float l[FK_WARPS][8];
};
static_assert(sizeof(MergeSmem) <= sizeof(uint8_t) * FK_STAGES * FK_STAGE_BYTES, "merge scratch");

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                             unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2 *>(&u); }

// (x0, x1) -> (c x0 - s x1, s x0 + c x1) with cs = (c, s), ns = (-s, c)
__device__ __forceinline__ uint32_t rot2(uint32_t x, uint32_t cs, uint32_t ns) {
  __half2 v = u2h(x);
  __half2 r = __hmul2(__high2half2(v), u2h(ns));
  r = __hfma2(__low2half2(v), u2h(cs), r);
  return h2u(r);
}

__device__ __forceinline__ float shfl_max_g(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
  return v;
}
__device__ __forceinline__ float shfl_sum_g(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  return v;
}

// Arguments of one decode step / attention call.
struct StepArgs {
  const void *q;           // [B][Hq][128]
  const void *knew;        // [B][Hkv][128] token appended this step (NULL: attend only)
  const void *vnew;
  int qdtype, kvdtype;
  const int64_t *qpos;     // [B]
  float *out;              // [B][Hq][128]
  float *lse;              // [B][Hq] or NULL
  float *ws_o, *ws_m, *ws_l;
  int *cnt;                // [B*Hkv] CTA tickets, [B] head tickets (self-resetting),
                           // [B*Hkv][4] cache-update plan
  int splits;              // CTAs per (b, head)
  unsigned long long *trace;   // optional per-CTA timeline (ANTKV_TRACE=1)
  int debug_mode;              // ANTKV_DEBUG_MODE: 1 skip pool rows, 2 stop after setup
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ float round_to(int dtype, float x) {
  if (dtype == ANTKV_BF16) return __bfloat162float(__float2bfloat16_rn(x));
  if (dtype == ANTKV_F16) return __half2float(__float2half_rn(x));
  return x;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------------ pool
// Full-precision rows [r0, r1) of the pool (anchors + window) on CUDA cores:
// a warp handles 4 rows per step (32 lanes x 4 dims), all loads of the 4
// rows in flight together.  With `with_new` the token appended this step is
// attended too (the reference appends before attending, cache.py:162-178).
// Results (natural-log units) go to the per-warp pool area of shared memory.
template <typename AfterLoads>
__device__ void pool_rows_part(const antkv_cache_desc &c, const StepArgs &a, FastSmem &sm,
                               double pq, int b, int h, int r0, int r1, bool with_new,
                               AfterLoads after_loads) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bh = (int64_t)b * c.Hkv + h;
  const int n = c.seq_len[b];
  const FastTables *tab = reinterpret_cast<const FastTables *>(c.fast_tables);
  float qv[4][4], qcs[2], qsn[2];
  const float scale = rsqrtf(128.f);
#pragma unroll
  for (int pp = 0; pp < 2; ++pp) rope_cs(pq * tab->omega[2 * lane + pp], qcs[pp], qsn[pp]);
#pragma unroll
  for (int hh = 0; hh < 4; ++hh) {
    const int64_t qb = ((int64_t)b * c.Hq + h * 4 + hh) * 128 + 4 * lane;
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const float x0 = load_elem(a.q, qb + 2 * pp, a.qdtype), x1 = load_elem(a.q, qb + 2 * pp + 1, a.qdtype);
      qv[hh][2 * pp] = (x0 * qcs[pp] - x1 * qsn[pp]) * scale;
      qv[hh][2 * pp + 1] = (x0 * qsn[pp] + x1 * qcs[pp]) * scale;
    }
  }
  float m[4], l[4], acc[4][4];
#pragma unroll
  for (int hh = 0; hh < 4; ++hh) {
    m[hh] = -INFINITY;
    l[hh] = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[hh][e] = 0.f;
  }
  if (with_new && warp == 0) {
    // K rotated in fp32 then rounded to fp16 like every pool K row; V in the pool dtype
    float kk[4], vv[4];
    const int64_t kb = bh * 128 + 4 * lane;
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const float x0 = round_to(c.row_dtype, load_elem(a.knew, kb + 2 * pp, a.kvdtype));
      const float x1 = round_to(c.row_dtype, load_elem(a.knew, kb + 2 * pp + 1, a.kvdtype));
      kk[2 * pp] = __half2float(__float2half_rn(x0 * qcs[pp] - x1 * qsn[pp]));
      kk[2 * pp + 1] = __half2float(__float2half_rn(x0 * qsn[pp] + x1 * qcs[pp]));
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) vv[e] = round_to(c.row_dtype, load_elem(a.vnew, kb + e, a.kvdtype));
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
      m[hh] = warp_sum(qv[hh][0] * kk[0] + qv[hh][1] * kk[1] + qv[hh][2] * kk[2] + qv[hh][3] * kk[3]);
      l[hh] = 1.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[hh][e] = vv[e];
    }
  }
  const __half *krot = reinterpret_cast<const __half *>(c.pool_krot) + bh * c.pool_capacity * 128;
  const int64_t vbase = bh * c.pool_capacity * 2 * 128 + 128;
  constexpr int RB = 10;  // rows per warp per round (all loads in flight together)
  bool first = true;
  for (int rb = r0 + RB * warp; first || rb < r1; rb += RB * FK_WARPS) {
    if (rb >= r1) {   // no rows for this warp: still run the hook once
      after_loads();
      break;
    }
    bool ok[RB];
    uint2 kraw[RB];
    float vv[RB][4];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int r = min(rb + u, r1 - 1);
      const int8_t kind = c.pool_kind[bh * c.pool_capacity + r];
      const int tok = c.pool_tok[bh * c.pool_capacity + r];
      ok[u] = (rb + u < r1) && kind != ANTKV_KIND_FREE && tok >= 0 && tok < n;
      kraw[u] = *reinterpret_cast<const uint2 *>(krot + (int64_t)r * 128 + 4 * lane);
      if (c.row_dtype == ANTKV_F32) {
        const float4 f = *reinterpret_cast<const float4 *>(
            reinterpret_cast<const float *>(c.pool_rows) + vbase + (int64_t)r * 256 + 4 * lane);
        vv[u][0] = f.x; vv[u][1] = f.y; vv[u][2] = f.z; vv[u][3] = f.w;
      } else {
        const uint2 raw = *reinterpret_cast<const uint2 *>(
            reinterpret_cast<const uint16_t *>(c.pool_rows) + vbase + (int64_t)r * 256 + 4 * lane);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint16_t hb = static_cast<uint16_t>((e < 2 ? raw.x : raw.y) >> (16 * (e & 1)));
          vv[u][e] = c.row_dtype == ANTKV_BF16 ? bf16_bits_to_float(hb)
                                               : __half2float(__ushort_as_half(hb));
        }
      }
    }
    if (first) {
      after_loads();   // rows requested: now queue the bulk copies behind them
      first = false;
    }
    float sc[RB][4];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const float2 k01 = __half22float2(u2h(kraw[u].x)), k23 = __half22float2(u2h(kraw[u].y));
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
        sc[u][hh] = qv[hh][0] * k01.x + qv[hh][1] * k01.y + qv[hh][2] * k23.x + qv[hh][3] * k23.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < RB; ++u)
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) sc[u][hh] += __shfl_xor_sync(0xffffffffu, sc[u][hh], o);
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
      float mx = m[hh];
#pragma unroll
      for (int u = 0; u < RB; ++u) if (ok[u]) mx = fmaxf(mx, sc[u][hh]);
      const float al = (m[hh] == mx) ? 1.f : __expf(m[hh] - mx);
      l[hh] *= al;
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[hh][e] *= al;
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const float p = ok[u] ? __expf(sc[u][hh] - mx) : 0.f;
        l[hh] += p;
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[hh][e] = fmaf(p, vv[u][e], acc[hh][e]);
      }
      m[hh] = mx;
    }
  }
#pragma unroll
  for (int hh = 0; hh < 4; ++hh) {
    *reinterpret_cast<float4 *>(&sm.po[warp][hh][4 * lane]) =
        make_float4(acc[hh][0], acc[hh][1], acc[hh][2], acc[hh][3]);
    if (lane == 0) {
      sm.pm[warp][hh] = m[hh];
      sm.pl[warp][hh] = l[hh];
    }
  }
}

// Cache-update plan of this step for head (b, h), prepared early by one CTA
// while the others still read the cache (cache.py:162-166, 180-193):
// the new token's rows go into the next free pool slot (still marked FREE,
// so readers skip it) and, if the window overflows and the anchor budget is
// exhausted, the oldest window row is encoded into its (still masked) code
// slot.  plan = {new slot, evicted slot, action 0 none / 1 promote / 2 encode,
// evicted token}; the last CTA of (b, h) commits it.
__device__ void prepare_update(const antkv_cache_desc &c, const StepArgs &a, FastSmem &sm, int b,
                               int h, int n, double pq) {
  const int64_t bh = (int64_t)b * c.Hkv + h;
  const int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
  const int top = hs[ANTKV_HS_FREE_TOP];
  const int slot_new = top > 0 ? c.free_stack[bh * c.pool_capacity + top - 1] : -1;
  const FastTables *tab = reinterpret_cast<const FastTables *>(c.fast_tables);
  if (slot_new >= 0) {
    const int64_t dst = (bh * c.pool_capacity + slot_new) * 256;
    __half *kr = reinterpret_cast<__half *>(c.pool_krot) + (bh * c.pool_capacity + slot_new) * 128;
    for (int t = threadIdx.x; t < 128; t += blockDim.x) {
      store_elem(c.pool_rows, dst + t, c.row_dtype, load_elem(a.knew, bh * 128 + t, a.kvdtype));
      store_elem(c.pool_rows, dst + 128 + t, c.row_dtype, load_elem(a.vnew, bh * 128 + t, a.kvdtype));
    }
    for (int p = threadIdx.x; p < 64; p += blockDim.x) {
      const float x0 = round_to(c.row_dtype, load_elem(a.knew, bh * 128 + 2 * p, a.kvdtype));
      const float x1 = round_to(c.row_dtype, load_elem(a.knew, bh * 128 + 2 * p + 1, a.kvdtype));
      float cs, sn;
      rope_cs(pq * tab->omega[p], cs, sn);
      kr[2 * p] = __float2half_rn(x0 * cs - x1 * sn);
      kr[2 * p + 1] = __float2half_rn(x0 * sn + x1 * cs);
    }
  }
  int es = -1, action = 0, j = -1;
  if (slot_new >= 0 && hs[ANTKV_HS_WIN_COUNT] + 1 > c.window_size) {
    es = hs[ANTKV_HS_WIN_COUNT] > 0 ? c.win_ring[bh * (c.window_size + 1) + hs[ANTKV_HS_WIN_HEAD]]
                                     : slot_new;
    j = es == slot_new ? n : c.pool_tok[bh * c.pool_capacity + es];
    const int budget = budget_for((int64_t)n + 1 + c.token_offset, c.anchor_count, c.anchor_fraction);
    action = hs[ANTKV_HS_ANCHORS] < budget ? 1 : 2;
  }
  if (action == 2) {
    __syncthreads();   // the new row (if evicted itself) is visible to the block
    // 32 units (kv, group) x 4 threads, each scanning 64 centroids of the fp16
    // shared-memory codebook for a top-4 shortlist, then rescoring it with the
    // float32 centroids: float32 distances, lowest index on ties
    // (_ckernels.pyx:150-162; SURVEY.md §7 hard part 2: shortlist + exact
    // rescore).
    const int64_t row = (bh * c.pool_capacity + es) * 256;
    const int u = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int kv = u >> 4, grp = u & 15;
    float x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = load_elem(c.pool_rows, row + kv * 128 + grp * 8 + e, c.row_dtype);
    const uint4 *cb16 = kv ? sm.cbV : sm.cbK;
    float sd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    int si[4] = {0, 0, 0, 0};
    const int lo_c = part * 64, hi_c = min(c.m, lo_c + 64);
    for (int ci = lo_c; ci < hi_c; ++ci) {
      const uint4 raw = cb16[ci * 8 + (threadIdx.x & 7)];
      const float2 c01 = __half22float2(u2h(raw.x)), c23 = __half22float2(u2h(raw.y));
      const float2 c45 = __half22float2(u2h(raw.z)), c67 = __half22float2(u2h(raw.w));
      float d = 0.f, df;
      df = x[0] - c01.x; d = fmaf(df, df, d);
      df = x[1] - c01.y; d = fmaf(df, df, d);
      df = x[2] - c23.x; d = fmaf(df, df, d);
      df = x[3] - c23.y; d = fmaf(df, df, d);
      df = x[4] - c45.x; d = fmaf(df, df, d);
      df = x[5] - c45.y; d = fmaf(df, df, d);
      df = x[6] - c67.x; d = fmaf(df, df, d);
      df = x[7] - c67.y; d = fmaf(df, df, d);
      if (d < sd[3]) {   // insert into the sorted top-4 (earlier index first on ties)
        sd[3] = d;
        si[3] = ci;
#pragma unroll
        for (int k = 3; k > 0; --k) {
          if (sd[k] < sd[k - 1]) {
            const float td = sd[k]; sd[k] = sd[k - 1]; sd[k - 1] = td;
            const int ti = si[k]; si[k] = si[k - 1]; si[k - 1] = ti;
          }
        }
      }
    }
    const float *cb = (kv ? c.codebook_v : c.codebook_k) + (int64_t)h * c.m * 8;
    float4 cv[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ci = si[k];
      cv[k][0] = __ldg(reinterpret_cast<const float4 *>(cb + ci * 8));
      cv[k][1] = __ldg(reinterpret_cast<const float4 *>(cb + ci * 8 + 4));
    }
    float best = INFINITY;
    int best_i = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (sd[k] == INFINITY) continue;
      float d = 0.f, df;
      df = x[0] - cv[k][0].x; d = fmaf(df, df, d);
      df = x[1] - cv[k][0].y; d = fmaf(df, df, d);
      df = x[2] - cv[k][0].z; d = fmaf(df, df, d);
      df = x[3] - cv[k][0].w; d = fmaf(df, df, d);
      df = x[4] - cv[k][1].x; d = fmaf(df, df, d);
      df = x[5] - cv[k][1].y; d = fmaf(df, df, d);
      df = x[6] - cv[k][1].z; d = fmaf(df, df, d);
      df = x[7] - cv[k][1].w; d = fmaf(df, df, d);
      if (d < best || (d == best && si[k] < best_i)) { best = d; best_i = si[k]; }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
      if (ob < best || (ob == best && oi < best_i)) { best = ob; best_i = oi; }
    }
    if (part == 0)
      c.codes[bh * c.capacity * 32 + code_offset(j, kv, grp, 16)] = static_cast<uint8_t>(best_i);
  }
  if (threadIdx.x == 0) {
    int *plan = a.cnt + (int64_t)c.B * c.Hkv + c.B + bh * 4;
    plan[0] = slot_new;
    plan[1] = es;
    plan[2] = action;
    plan[3] = j;
  }
}

// Commit the plan (last CTA of (b, h), every reader of the head is done).
__device__ void commit_update(const antkv_cache_desc &c, const StepArgs &a, int b, int h, int n) {
  const int64_t bh = (int64_t)b * c.Hkv + h;
  int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
  const int *plan = a.cnt + (int64_t)c.B * c.Hkv + c.B + bh * 4;
  const int slot_new = __ldcg(plan), es = __ldcg(plan + 1), action = __ldcg(plan + 2), j = __ldcg(plan + 3);
  const int W1 = c.window_size + 1;
  int32_t *ring = c.win_ring + bh * W1;
  if (slot_new >= 0) {
    hs[ANTKV_HS_FREE_TOP] -= 1;
    c.pool_tok[bh * c.pool_capacity + slot_new] = n;
    c.pool_kind[bh * c.pool_capacity + slot_new] = ANTKV_KIND_WINDOWED;
    ring[(hs[ANTKV_HS_WIN_HEAD] + hs[ANTKV_HS_WIN_COUNT]) % W1] = slot_new;
    hs[ANTKV_HS_WIN_COUNT] += 1;
    if (slot_new + 1 > hs[ANTKV_HS_POOL_HIGH]) hs[ANTKV_HS_POOL_HIGH] = slot_new + 1;
  }
  if (action != 0) {
    hs[ANTKV_HS_WIN_HEAD] = (hs[ANTKV_HS_WIN_HEAD] + 1) % W1;
    hs[ANTKV_HS_WIN_COUNT] -= 1;
    if (action == 1) {
      c.pool_kind[bh * c.pool_capacity + es] = ANTKV_KIND_ANCHOR;
      hs[ANTKV_HS_ANCHORS] += 1;
    } else {
      atomicOr(&c.qmask[bh * (c.capacity / 32) + j / 32], 1u << (j % 32));
      c.pool_kind[bh * c.pool_capacity + es] = ANTKV_KIND_FREE;
      c.pool_tok[bh * c.pool_capacity + es] = -1;
      c.free_stack[bh * c.pool_capacity + hs[ANTKV_HS_FREE_TOP]] = es;
      hs[ANTKV_HS_FREE_TOP] += 1;
    }
  }
}

// Per-warp streaming state for the code tiles.  A stage holds an even and an
// odd 16-slot tile; both are multiplied with ONE B fragment: columns 0-3 are
// the 4 query heads in the even tile's frame R(p_q - P0) q (lanes 0-15),
// columns 4-7 in the odd tile's frame R(p_q - P0 - 16) q (lanes 16-31).  Row r
// of a tile is rotated by R(r), r = g or g + 8.  Even-tile scores are read
// from columns 0-3 and odd-tile scores from 4-7, so the O^T columns 0-3 / 4-7
// accumulate two independent streams merged at the end.
struct WarpState {
  uint32_t kc[8][8];      // key rotation (cos,sin)/(-sin,cos) for rows g, g+8
  float fx[16], fy[16];   // query frame pairs (log2-scaled)
  float stc[16], sts[16]; // R(-32) per pair
  float mrun[2], lrun[2]; // softmax of this lane's 2 columns (log2 units; lrun per lane)
  float o[8][4];          // O^T accumulators
};

// Code records of one 16-slot tile for this lane: 8 K codes (groups 2s+pk)
// and 8 V codes (groups 2mt+pv), packed 4 per word.
struct TileCodes {
  uint32_t k0, k1, v0, v1;
};

__device__ __forceinline__ TileCodes tile_codes(const uint8_t *tb, int tk, int tv, uint32_t sel_k,
                                                uint32_t sel_v) {
  const uint4 kr = *reinterpret_cast<const uint4 *>(tb + tk * 16);
  const uint4 vr = *reinterpret_cast<const uint4 *>(tb + 256 + tv * 16);
  TileCodes tc;
  tc.k0 = __byte_perm(kr.x, kr.y, sel_k);
  tc.k1 = __byte_perm(kr.z, kr.w, sel_k);
  tc.v0 = __byte_perm(vr.x, vr.y, sel_v);
  tc.v1 = __byte_perm(vr.z, vr.w, sel_v);
  return tc;
}

// Shared-memory address of centroid `byte k of word` in a replicated codebook.
__device__ __forceinline__ uint32_t cb_addr(uint32_t word, int k, uint32_t base) {
  uint32_t code, addr;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(code) : "r"(word), "r"(0x4440 + k));
  asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(code), "r"(base));
  return addr;
}

// S^T = rot(K_hat) . B (8 HMMA in two chains); returns the 4 accumulators.
__device__ __forceinline__ float4 qk_tile(const WarpState &w, const TileCodes &tc,
                                          const uint32_t (&bq)[8][2], uint32_t cbK_base) {
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    uint32_t a[4];
    ldsm_x4(cb_addr(s < 4 ? tc.k0 : tc.k1, s & 3, cbK_base), a);
    a[0] = rot2(a[0], w.kc[s][0], w.kc[s][1]);
    a[1] = rot2(a[1], w.kc[s][2], w.kc[s][3]);
    a[2] = rot2(a[2], w.kc[s][4], w.kc[s][5]);
    a[3] = rot2(a[3], w.kc[s][6], w.kc[s][7]);
    if (s & 1) mma16816(sb, a, bq[s][0], bq[s][1]);
    else mma16816(sa, a, bq[s][0], bq[s][1]);
  }
  return make_float4(sa[0] + sb[0], sa[1] + sb[1], sa[2] + sb[2], sa[3] + sb[3]);
}

// O^T += V_hat^T . P (8 independent HMMA).
__device__ __forceinline__ void pv_tile(WarpState &w, const TileCodes &tc, uint32_t pb0,
                                        uint32_t pb1, uint32_t cbV_base) {
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    uint32_t a[4];
    ldsm_x4_t(cb_addr(mt < 4 ? tc.v0 : tc.v1, mt & 3, cbV_base), a);
    mma16816(w.o[mt], a, pb0, pb1);
  }
}

// One stage = even + odd tile.  `mrow` holds this lane's two row-valid bits
// (row g in bit 0, row g+8 in bit 1) of the tile whose columns it owns.
__device__ __forceinline__ void stage_tiles(WarpState &w, const TileCodes &te, const TileCodes &to,
                                            uint32_t mrow, uint32_t cbK_base, uint32_t cbV_base,
                                            bool lo) {
  uint32_t bq[8][2];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    bq[s][0] = h2u(__floats2half2_rn(w.fx[2 * s], w.fy[2 * s]));
    bq[s][1] = h2u(__floats2half2_rn(w.fx[2 * s + 1], w.fy[2 * s + 1]));
  }
  const float4 se = qk_tile(w, te, bq, cbK_base);
  const float4 so = qk_tile(w, to, bq, cbK_base);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const float x = w.fx[k], y = w.fy[k];
    w.fx[k] = x * w.stc[k] - y * w.sts[k];
    w.fy[k] = x * w.sts[k] + y * w.stc[k];
  }
  // this lane's scores: (row g, col 2t), (row g, 2t+1), (row g+8, 2t), (row g+8, 2t+1)
  const float4 sv = lo ? se : so;
  const bool v0 = mrow & 1u, v1 = mrow & 2u;
  const float s00 = v0 ? sv.x : -INFINITY, s01 = v0 ? sv.y : -INFINITY;
  const float s10 = v1 ? sv.z : -INFINITY, s11 = v1 ? sv.w : -INFINITY;
  // lazily updated reference max (P <= 2^8 keeps fp16 safe); exact max + rescale on raise
  const bool up = fmaxf(s00, s10) > w.mrun[0] + 8.f || fmaxf(s01, s11) > w.mrun[1] + 8.f;
  if (__any_sync(0xffffffffu, up)) {
    const float mn0 = fmaxf(w.mrun[0], shfl_max_g(fmaxf(s00, s10)));
    const float mn1 = fmaxf(w.mrun[1], shfl_max_g(fmaxf(s01, s11)));
    const float a0 = (w.mrun[0] == mn0) ? 1.f : ex2(w.mrun[0] - mn0);
    const float a1 = (w.mrun[1] == mn1) ? 1.f : ex2(w.mrun[1] - mn1);
    w.lrun[0] *= a0;
    w.lrun[1] *= a1;
    w.mrun[0] = mn0;
    w.mrun[1] = mn1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      w.o[i][0] *= a0;
      w.o[i][1] *= a1;
      w.o[i][2] *= a0;
      w.o[i][3] *= a1;
    }
  }
  const float p00 = v0 ? ex2(s00 - w.mrun[0]) : 0.f, p01 = v0 ? ex2(s01 - w.mrun[1]) : 0.f;
  const float p10 = v1 ? ex2(s10 - w.mrun[0]) : 0.f, p11 = v1 ? ex2(s11 - w.mrun[1]) : 0.f;
  w.lrun[0] += p00 + p10;
  w.lrun[1] += p01 + p11;
  const uint32_t x0 = h2u(__floats2half2_rn(p00, p01));   // P[row g][cols 2t, 2t+1]
  const uint32_t x1 = h2u(__floats2half2_rn(p10, p11));   // P[row g+8][...]
  pv_tile(w, te, movm_t(lo ? x0 : 0u), movm_t(lo ? x1 : 0u), cbV_base);
  pv_tile(w, to, movm_t(lo ? 0u : x0), movm_t(lo ? 0u : x1), cbV_base);
}

// ---------------------------------------------------------------- kernel
// Every CTA of (b, h) handles an equal share of the code tiles and of the
// pool rows; the last split also attends the appended token and prepares the
// cache update; the last CTA to finish combines the partials and commits.
__global__ void __launch_bounds__(FK_THREADS, 2)
decode_fast_kernel(antkv_cache_desc c, StepArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  FastSmem &sm = *reinterpret_cast<FastSmem *>(smraw);
  MergeSmem &mg = *reinterpret_cast<MergeSmem *>(&sm.ring[0][0]);
  const int b = blockIdx.z, h = blockIdx.y, split = blockIdx.x;
  const int S = a.splits;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t bh = (int64_t)b * c.Hkv + h;
  const int64_t row0 = ((int64_t)split * c.B + b) * c.Hq + h * 4;
  const double pq = static_cast<double>(a.qpos[b]);
  const int n = c.seq_len[b];
  const bool last_split = split == S - 1;
  unsigned long long tr[8];
  if (a.trace && threadIdx.x == 0) tr[0] = gtimer();

  // ---- code range: tiles [T0, T0 + per_cta), 4 contiguous warp ranges of Tw tiles
  // the last split also prepares the cache update, so it gets half a share
  const int ntiles = (n + 15) >> 4;
  const float shares = (a.knew && S > 1) ? S - 0.5f : (float)S;
  const int per_cta = ((int)ceilf(ntiles / shares) + 2 * FK_WARPS - 1) / (2 * FK_WARPS) * (2 * FK_WARPS);
  const int T0 = split * per_cta;
  const int mine = max(0, min(per_cta, ntiles - T0));           // valid tiles of this CTA
  const int Tw = ((mine + FK_WARPS - 1) / FK_WARPS + 1) & ~1;   // even; tiles per warp
  const int nstages = Tw / 2;
  const int64_t pos0 = c.positions[(int64_t)b * c.capacity];
  const uint8_t *codes = c.codes + bh * c.capacity * 32;   // 32 code bytes per slot
  const uint32_t *qmg = c.qmask + bh * (c.capacity / 32);
  const int cap_tiles = c.capacity / 16;
  const FastTables *tab = reinterpret_cast<const FastTables *>(c.fast_tables);

  if (threadIdx.x == 0) {
    for (int s = 0; s < FK_STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], FK_WARPS);
    }
    mbar_init(&sm.cbbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int st) {
    const int slot = st % FK_STAGES;
    mbar_expect_tx(&sm.full[slot], FK_STAGE_BYTES);
    for (int w = 0; w < FK_WARPS; ++w) {
      int tile = T0 + w * Tw + 2 * st;
      if (tile + 2 > cap_tiles) tile = 0;   // beyond capacity: masked dummy data
      tma_bulk_g2s(&sm.ring[slot][w * FK_WARP_STAGE_BYTES], codes + (int64_t)tile * FK_TILE_BYTES,
                   FK_WARP_STAGE_BYTES, &sm.full[slot]);
    }
  };
  const bool prep = last_split && a.knew;
  // ---- pool rows (anchors + window) of this CTA's share first: their loads
  // are issued before the code-tile bulk copies that follow in the hook
  {
    const int pool_high = c.hstate[bh * ANTKV_HSTATE_WORDS + ANTKV_HS_POOL_HIGH];
    const int per = (pool_high + S - 1) / S;
    const int r0 = min(pool_high, split * per), r1 = min(pool_high, r0 + per);
    pool_rows_part(c, a, sm, pq, b, h, r0, (a.debug_mode & 1) ? r0 : r1, prep, [&]() {
      if (threadIdx.x == 0)
        for (int st = 0; st < min(nstages, FK_STAGES); ++st) issue(st);
    });
  }
  if (a.trace && threadIdx.x == 0) tr[4] = gtimer();
  // ---- replicated fp16 codebooks: row `code` holds the centroid in all 8
  // 16-byte bank groups (copy 0 of the prepared global layout is read)
  if (nstages > 0 || prep) {
    const uint4 *src = reinterpret_cast<const uint4 *>(c.codebook_f16) + (int64_t)h * 4096;
    uint4 vk[2], vv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int code = threadIdx.x + u * FK_THREADS;
      vk[u] = __ldg(src + code * 8);
      vv[u] = __ldg(src + 2048 + code * 8);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int code = threadIdx.x + u * FK_THREADS;
#pragma unroll
      for (int cp = 0; cp < 8; ++cp) {
        sm.cbK[code * 8 + ((cp + threadIdx.x) & 7)] = vk[u];
        sm.cbV[code * 8 + ((cp + threadIdx.x) & 7)] = vv[u];
      }
    }
  }
  __syncthreads();
  if (a.trace && threadIdx.x == 0) tr[5] = gtimer();
  if (a.debug_mode & 2) return;
  for (int i = lane; i < Tw / 2; i += 32) {
    const int word = ((T0 + warp * Tw) >> 1) + i;
    sm.qm[warp][i] = (word * 32 < c.capacity) ? qmg[word] : 0u;
  }
  WarpState w;
  w.mrun[0] = w.mrun[1] = -INFINITY;
  w.lrun[0] = w.lrun[1] = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) w.o[i][e] = 0.f;
  if (nstages > 0) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int pair = 8 * s + 4 * u + t;
        w.kc[s][4 * u] = tab->kc[g][pair][0];
        w.kc[s][4 * u + 1] = tab->kc[g][pair][1];
        w.kc[s][4 * u + 2] = tab->kc[g + 8][pair][0];
        w.kc[s][4 * u + 3] = tab->kc[g + 8][pair][1];
      }
    }
    // query frame: lanes 0-15 head g in the even tile's frame, 16-31 head g-4 in the odd's
    const int head = g & 3;
    const int64_t first_slot = (int64_t)(T0 + warp * Tw) * 16 + (g >= 4 ? 16 : 0);
    const double delta = pq - static_cast<double>(pos0 + first_slot);
    const float scale = rsqrtf(128.f) * 1.4426950408889634f;   // 1/sqrt(d) * log2(e)
    const int64_t qb = ((int64_t)b * c.Hq + h * 4 + head) * 128;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int pair = 8 * s + 4 * u + t, k = 2 * s + u;
        const float x0 = load_elem(a.q, qb + 2 * pair, a.qdtype) * scale;
        const float x1 = load_elem(a.q, qb + 2 * pair + 1, a.qdtype) * scale;
        float cs, sn;
        rope_cs(delta * tab->omega[pair], cs, sn);
        w.fx[k] = x0 * cs - x1 * sn;
        w.fy[k] = x0 * sn + x1 * cs;
        w.stc[k] = tab->step[pair][0];
        w.sts[k] = tab->step[pair][1];
      }
    }
    const uint32_t cbK_base = smem_u32(&sm.cbK[0]) + (lane & 7) * 16;
    const uint32_t cbV_base = smem_u32(&sm.cbV[0]) + (lane & 7) * 16;
    const int tk = (lane & 7) + 8 * ((lane >> 3) & 1);     // K-side token row
    const int tv = (lane & 7) + 8 * (lane >> 4);          // V-side token row
    const uint32_t sel_k = (lane >> 4) ? 0x7531u : 0x6420u;
    const uint32_t sel_v = ((lane >> 3) & 1) ? 0x7531u : 0x6420u;
    const bool lo = t < 2;                                // owns the even tile's columns
    const int rowbit = g + (lo ? 0 : 16);                 // rows g (+8 via >>7 above)
    // the last split (smallest code share) prepares the cache update
    if (prep) prepare_update(c, a, sm, b, h, n, pq);
    if (a.trace && threadIdx.x == 0) tr[1] = gtimer();
    for (int st = 0; st < nstages; ++st) {
      const int slot = st % FK_STAGES;
      mbar_wait(&sm.full[slot], (st / FK_STAGES) & 1);
      const uint8_t *tb = &sm.ring[slot][warp * FK_WARP_STAGE_BYTES];
      const TileCodes te = tile_codes(tb, tk, tv, sel_k, sel_v);
      const TileCodes to = tile_codes(tb + FK_TILE_BYTES, tk, tv, sel_k, sel_v);
      const uint32_t qw = sm.qm[warp][st] >> rowbit;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[slot]);   // codes are in registers
      if (threadIdx.x == 0 && st + FK_STAGES < nstages) {
        mbar_wait(&sm.empty[slot], (st / FK_STAGES) & 1);
        issue(st + FK_STAGES);
      }
      stage_tiles(w, te, to, (qw & 1u) | ((qw >> 7) & 2u), cbK_base, cbV_base, lo);
    }
  }
  if (nstages == 0 && prep) prepare_update(c, a, sm, b, h, n, pq);
  if (a.trace && threadIdx.x == 0) tr[2] = gtimer();
  // ---- merge 4 warps x (2 code streams + pool rows) -> partial (natural log)
  __syncthreads();   // all stages consumed; the ring becomes merge scratch
  const float ln2 = 0.6931471805599453f;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    mg.o[warp][2 * t][16 * mt + g] = w.o[mt][0];
    mg.o[warp][2 * t + 1][16 * mt + g] = w.o[mt][1];
    mg.o[warp][2 * t][16 * mt + g + 8] = w.o[mt][2];
    mg.o[warp][2 * t + 1][16 * mt + g + 8] = w.o[mt][3];
  }
  const float lsum0 = shfl_sum_g(w.lrun[0]), lsum1 = shfl_sum_g(w.lrun[1]);
  if (g == 0) {
    mg.m[warp][2 * t] = w.mrun[0] * ln2;
    mg.m[warp][2 * t + 1] = w.mrun[1] * ln2;
    mg.l[warp][2 * t] = lsum0;
    mg.l[warp][2 * t + 1] = lsum1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 128; i += FK_THREADS) {
    const int hh = i / 128, dim = i % 128;
    float M = -INFINITY;
    for (int ww = 0; ww < FK_WARPS; ++ww)
      M = fmaxf(M, fmaxf(fmaxf(mg.m[ww][hh], mg.m[ww][hh + 4]), sm.pm[ww][hh]));
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int ww = 0; ww < FK_WARPS; ++ww) {
#pragma unroll
        for (int src = 0; src < 3; ++src) {
          const float mv = src < 2 ? mg.m[ww][hh + 4 * src] : sm.pm[ww][hh];
          if (mv == -INFINITY) continue;
          const float f = __expf(mv - M);
          L += f * (src < 2 ? mg.l[ww][hh + 4 * src] : sm.pl[ww][hh]);
          O += f * (src < 2 ? mg.o[ww][hh + 4 * src][dim] : sm.po[ww][hh][dim]);
        }
      }
    }
    a.ws_o[(row0 + hh) * 128 + dim] = O;
    if (dim == 0) {
      a.ws_m[row0 + hh] = M;
      a.ws_l[row0 + hh] = L;
    }
  }

  // ---- ticket: the last CTA of (b, h) combines the partials and commits
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sm.ticket = atomicAdd(&a.cnt[bh], 1);
  __syncthreads();
  if (a.trace && threadIdx.x == 0) {
    tr[3] = gtimer();
    unsigned long long *o = a.trace + 8 * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
    o[0] = smid() | ((unsigned long long)sm.ticket << 32);
    o[1] = tr[0];
    o[2] = tr[1];
    o[3] = tr[2];
    o[4] = tr[3];
    o[5] = 0;
    o[6] = tr[4];
    o[7] = tr[5];
  }
  if (sm.ticket != S - 1) return;
  __threadfence();
  const int64_t rows = (int64_t)c.B * c.Hq;
  float *wts = reinterpret_cast<float *>(&sm.ring[0][0]);   // [S][4] (merge data consumed)
  float *hdr = wts + 4 * S;                                       // [4] M, [4] L
  {
    const int hh = warp;   // warp hh: max / normaliser over splits for head hh
    const int64_t row = (int64_t)b * c.Hq + h * 4 + hh;
    float M = -INFINITY;
    for (int s2 = lane; s2 < S; s2 += 32) M = fmaxf(M, __ldcg(a.ws_m + s2 * rows + row));
    M = warp_max(M);
    float L = 0.f;
    for (int s2 = lane; s2 < S; s2 += 32) {
      const float ms = __ldcg(a.ws_m + s2 * rows + row);
      const float wv = (ms == -INFINITY) ? 0.f : __expf(ms - M);
      wts[s2 * 4 + hh] = wv;
      L += wv * __ldcg(a.ws_l + s2 * rows + row);
    }
    L = warp_sum(L);
    if (lane == 0) {
      hdr[hh] = M;
      hdr[4 + hh] = L;
      if (a.lse) a.lse[row] = M + logf(L);
    }
  }
  __syncthreads();
  {
    // thread = (head warp, 4 consecutive dims); 8 split rows in flight per round
    const int hh = warp, d4 = 4 * lane;
    const int64_t row = (int64_t)b * c.Hq + h * 4 + hh;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < S; s0 += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int s2 = min(s0 + u, S - 1);
        v[u] = __ldcg(reinterpret_cast<const float4 *>(a.ws_o + (s2 * rows + row) * 128 + d4));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float wv = (s0 + u < S) ? wts[(s0 + u) * 4 + hh] : 0.f;
        acc.x = fmaf(wv, v[u].x, acc.x);
        acc.y = fmaf(wv, v[u].y, acc.y);
        acc.z = fmaf(wv, v[u].z, acc.z);
        acc.w = fmaf(wv, v[u].w, acc.w);
      }
    }
    const float inv = 1.f / hdr[4 + hh];
    *reinterpret_cast<float4 *>(a.out + row * 128 + d4) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
  if (threadIdx.x == 0) {
    if (a.knew) commit_update(c, a, b, h, n);
    if (a.trace) a.trace[8 * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) + 5] = gtimer();
    __threadfence();
    a.cnt[bh] = 0;
    if (a.knew) {
      // the last head of sequence b publishes the new length / position
      int *cb = a.cnt + (int64_t)c.B * c.Hkv + b;
      if (atomicAdd(cb, 1) == c.Hkv - 1) {
        c.positions[(int64_t)b * c.capacity + n] = a.qpos[b];
        __threadfence();
        c.seq_len[b] = n + 1;
        *cb = 0;
      }
    }
  }
}

int decode_fast_supported(const antkv_cache_desc &c) {
  return c.d == 128 && c.d_sub == 8 && c.m <= 256 && c.code_bytes == 1 && c.Hq == 4 * c.Hkv &&
         c.codebook_f16 != nullptr && c.pool_krot != nullptr && c.fast_tables != nullptr &&
         c.capacity % 128 == 0;
}

// CTAs per (sequence, head): ~2 resident CTAs per SM in total.
void decode_fast_plan(const antkv_cache_desc &c, int requested, int &code_splits, int &pool_splits) {
  const int bh = c.B * c.Hkv;
  code_splits = requested > 0 ? requested : max(1, (2 * 148) / bh);
  // per-warp qmask staging caps a CTA at 4 warps x 128 tiles (FK_MAX_WARP_WORDS)
  const int cap_tiles = c.capacity / 16;
  const int min_code = (cap_tiles + 503) / 504;
  if (code_splits < min_code) code_splits = min_code;
  pool_splits = 0;
}

static unsigned long long *g_trace = nullptr;
static int g_trace_n = 0;
static unsigned long long *debug_trace_buffer() {
  static int enabled = -1;
  if (enabled < 0) {
    const char *e = getenv("ANTKV_TRACE");
    enabled = e && e[0] == '1';
    if (enabled) {
      g_trace_n = 8 * 65536;
      if (cudaMalloc(&g_trace, sizeof(unsigned long long) * g_trace_n) != cudaSuccess) g_trace = nullptr;
    }
  }
  return g_trace;
}

}  // namespace antkv

// Debug: copy the per-CTA timeline of the last traced fast-decode launch
// (8 words per CTA: smid | ticket << 32, t_start, t_loop, t_pool, t_done,
// t_committed) to host memory.  Returns the number of words copied.
extern "C" int antkv_debug_trace(unsigned long long *host, int max_words) {
  if (!antkv::g_trace) return 0;
  const int n = max_words < antkv::g_trace_n ? max_words : antkv::g_trace_n;
  cudaDeviceSynchronize();
  cudaMemcpy(host, antkv::g_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  return n;
}

namespace antkv {

// One fused launch: attention over the cache (+ the appended token), LSE
// combine of the splits, and (when knew != NULL) append + evict.
int decode_fast_launch(const antkv_cache_desc &c, const void *q, int qdtype, const void *knew,
                       const void *vnew, int kvdtype, const int64_t *qpos, float *out, float *lse,
                       float *ws_o, float *ws_m, float *ws_l, int *cnt, int splits,
                       cudaStream_t st) {
  StepArgs a;
  a.q = q;
  a.knew = knew;
  a.vnew = vnew;
  a.qdtype = qdtype;
  a.kvdtype = kvdtype;
  a.qpos = qpos;
  a.out = out;
  a.lse = lse;
  a.ws_o = ws_o;
  a.ws_m = ws_m;
  a.ws_l = ws_l;
  a.cnt = cnt;
  int cs, ps;
  decode_fast_plan(c, splits, cs, ps);
  a.splits = cs + ps;
  a.trace = debug_trace_buffer();
  {
    static int dm = -1;
    if (dm < 0) {
      const char *e = getenv("ANTKV_DEBUG_MODE");
      dm = e ? atoi(e) : 0;
    }
    a.debug_mode = dm;
  }
  const size_t smem = sizeof(FastSmem);
  cudaFuncSetAttribute(decode_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(a.splits, c.Hkv, c.B);
  decode_fast_kernel<<<grid, FK_THREADS, smem, st>>>(c, a);
  ANTKV_LAUNCH_CHECK("decode_fast_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
