// sm_100a decode-attention kernel for the 1-bit d8m256 configuration
// (d = 128, d_sub = 8, m <= 256, 4 query heads per KV head, contiguous
// positions).  Reference semantics: cache.py:149-194 (append the new token,
// RoPE after reconstruction, softmax over the whole cache, A.V, then evict).
//
// One launch does the whole decode step for every (sequence, KV head):
//   * CTAs: `splits` per (sequence, head), one CTA of 8 warps per SM.  Each
//     CTA owns a contiguous range of 16-slot code tiles (split into 8
//     contiguous warp ranges) and a share of the full-precision pool tiles.
//   * Codebooks: the compact fp16 codebook (8 KB per head, [code][K 8 | V 8])
//     is read with one 32-byte load per thread and replicated in shared
//     memory as [code][K 8 copies | V 8 copies]: a centroid row sits in all
//     eight 16-byte bank groups, so the eight row addresses of an ldmatrix
//     phase (copy = lane & 7) never conflict, and an address is ONE prmt:
//     (code << 8) | lane_offset, with the codebook base folded into the
//     ldmatrix uniform operand.  (A bulk copy of the replicated 64 KB per
//     CTA moved 9.4 MB through L2 per launch, ahead of the cache state.)
//   * Code tiles (K codes 256 B + V codes 256 B per tile) stream through a
//     private 8-stage ring per warp (cp.async.bulk + mbarrier); the warp
//     refills its own slots, so warps never wait on each other.
//   * Per stage (an even and an odd tile) S^T[16 x 8] = rot(K_hat) . B and
//     O^T[128 x 8] += V_hat^T . P with m16n8k16 tensor-core MMAs on register
//     operands.  RoPE: row r of a tile is rotated by R(r) with per-lane fp16
//     (cos, sin) constants; the tile base rotation lives in the query
//     frames: B columns 0-3 hold the 4 query heads in the even tile's frame,
//     columns 4-7 in the odd tile's frame.  Frames advance by R(-32) per
//     stage in packed fp32 (FFMA2), seeded from float64-reduced angles.
//   * Pool tiles (anchors + window: K rotated at its own position and V, in
//     fp16, pre-swizzled) are bulk-copied per warp and multiplied with the
//     query in the absolute frame (no per-row rotation).
//   * Online softmax in log2 units with a lazily raised reference max (P <=
//     2^8 keeps fp16 P exact enough); CTA merge in shared memory; the last
//     CTA of each (sequence, head) (atomic ticket) combines the splits and
//     commits the cache-update plan that one CTA prepared while the others
//     were reading (new row into a free pool slot, oldest window row
//     promoted or encoded).
#include <stdlib.h>

#include "common.cuh"

namespace antkv {

constexpr int FK_WARPS = 8;
constexpr int FK_THREADS = 32 * FK_WARPS;
constexpr int FK_NS = 4;                                 // ring slots per warp
constexpr int FK_TILE_BYTES = 512;                       // K 256 B + V 256 B
constexpr int FK_STAGE_BYTES = 2 * FK_TILE_BYTES;        // even + odd tile
constexpr int FK_SLOT_BYTES = 2 * FK_STAGE_BYTES;        // two stages per ring slot
// The codebook sits at offset 0 of dynamic shared memory, whose shared-window
// address is 0x400 on sm_100 (the 1 KB reserved block; probed once on the
// host, decode_fast_smem_base_ok): gathers use it as an ldmatrix immediate.
constexpr uint32_t FK_SMEM_BASE = 0x400;
// ANTKV_TRACE=1: per-CTA timeline words: 0 smid | ticket << 32, then global
// timer stamps 1 start, 2 barriers ready, 3 prologue loads issued, 4 frames,
// 5 pool wait, 6 pool done, 7 prepare done, 8 loop start, 9 loop end,
// 10 after the tickets, 11 committed (last CTA only), 12 all warps done,
// 13 partial written, 15 combine done (last CTA only).
constexpr int FK_TRACE_WORDS = 16;
constexpr int FK_POOL_TILE_BYTES = 8192;                 // [K|V][16 slots][128] fp16
constexpr int FK_MAX_WARP_WORDS = 64;                    // qmask words per warp (2048 slots)
constexpr int FK_CB_BYTES = 256 * 256;                   // [code][K 128 B | V 128 B]

struct __align__(128) FastSmem {
  uint8_t cb[FK_CB_BYTES];
  uint8_t ring[FK_WARPS][FK_NS][FK_SLOT_BYTES];
  uint8_t pool[FK_WARPS][FK_POOL_TILE_BYTES];
  uint32_t qm[FK_WARPS][FK_MAX_WARP_WORDS];
  float xo[4][128];                          // the appended token's row (prep CTA)
  float xm[4];                               // its scaled logits (log2 units)
  FastTables tab;                            // RoPE constants (bulk copy)
  uint8_t qraw[4 * 128 * 4];                 // the 4 query rows of the head (input dtype)
  float2 qf[4][64];                          // the same, float32 pairs in lane order, scaled
                                             // by log2(e)/sqrt(d)
  float2 ang[2 * FK_WARPS + 1][64];          // (cos, sin) per query frame, pairs in lane order
  unsigned long long full[FK_WARPS][FK_NS];
  unsigned long long pfull[FK_WARPS];
  unsigned long long tbar, qbar;
  unsigned long long t0clk;                  // trace: start clock of the CTA
};

struct MergeSmem {                             // aliases the pool area after the loops
  float o[FK_WARPS][8][128];
  float m[FK_WARPS][8];
  float l[FK_WARPS][8];
};
static_assert(sizeof(MergeSmem) <= sizeof(uint8_t) * FK_WARPS * FK_POOL_TILE_BYTES, "merge scratch");

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
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
// Gathers from the codebook: `off` = (code << 8) | copy offset (| 128 for V).
__device__ __forceinline__ void ldsm_cb(uint32_t off, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4+1024];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(off));
}
__device__ __forceinline__ void ldsm_cb_t(uint32_t off, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4+1024];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(off));
}
static_assert(FK_SMEM_BASE == 1024, "ldsm_cb immediates");
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
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2 *>(&u); }
__device__ __forceinline__ uint32_t pack_h2(float x, float y) { return h2u(__floats2half2_rn(x, y)); }

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
  int *cnt;                // [B*Hkv] CTA tickets, [B] sequence tickets (self-resetting),
                           // [B*Hkv][kPlanWords] cache-update plans
  int splits;              // CTAs per (b, head)
  int early;               // the previous kernel in the stream wrote no state of this
                           // cache: read cache state before griddepcontrol.wait
  int early_q;             // ... and none of q / qpos / the appended rows: then nothing
                           // this launch reads was written by the previous kernel, and
                           // the wait (with the dependents' release) moves to the end of
                           // the streaming loop -- the whole prologue, the pool tiles
                           // and the loop overlap the previous launch's tail
  unsigned long long *trace;   // optional per-CTA timeline (ANTKV_TRACE=1)
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

// ------------------------------------------------------------ cache update
// Plan of this step's cache update for head (b, h), prepared by the last
// split while the other CTAs still read the cache (cache.py:157-166,
// 180-193): the new token's rows go into the next free pool slot (still
// marked FREE, so readers skip it) and, if the window overflows and the
// anchor budget is exhausted, the oldest window row is encoded into its
// (still masked) code slot.  All new state words are computed here, so the
// commit in the last CTA is a batch of independent stores.
// plan: 0 slot_new, 1 evicted slot, 2 action (0 none / 1 promote / 2 encode),
// 3 evicted token, 4 ring position of slot_new, 5..9 new hstate words 0..4,
// 10 free-stack index receiving the evicted slot.
__device__ void prepare_update(const antkv_cache_desc &c, const StepArgs &a, FastSmem &sm, int b,
                               int h, int n, double pq) {
  const int64_t bh = (int64_t)b * c.Hkv + h;
  const int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
  const int A0 = hs[ANTKV_HS_ANCHORS], H0 = hs[ANTKV_HS_WIN_HEAD], C0 = hs[ANTKV_HS_WIN_COUNT];
  const int F0 = hs[ANTKV_HS_FREE_TOP], PH0 = hs[ANTKV_HS_POOL_HIGH];
  const int W1 = c.window_size + 1;
  const int slot_new = F0 > 0 ? c.free_stack[bh * c.pool_capacity + F0 - 1] : -1;
  const FastTables *tab = reinterpret_cast<const FastTables *>(c.fast_tables);
  if (slot_new >= 0) {
    const int64_t dst = (bh * c.pool_capacity + slot_new) * 256;
    __half *pf = reinterpret_cast<__half *>(c.pool_f16) + bh * c.pool_capacity * 256;
    for (int t = threadIdx.x; t < 128; t += blockDim.x) {
      const float vk = load_elem(a.knew, bh * 128 + t, a.kvdtype);
      const float vv = load_elem(a.vnew, bh * 128 + t, a.kvdtype);
      store_elem(c.pool_rows, dst + t, c.row_dtype, vk);
      store_elem(c.pool_rows, dst + 128 + t, c.row_dtype, vv);
      pf[pool_f16_offset(slot_new, 1, t)] = __float2half_rn(round_to(c.row_dtype, vv));
    }
    for (int p = threadIdx.x; p < 64; p += blockDim.x) {
      const float x0 = round_to(c.row_dtype, load_elem(a.knew, bh * 128 + 2 * p, a.kvdtype));
      const float x1 = round_to(c.row_dtype, load_elem(a.knew, bh * 128 + 2 * p + 1, a.kvdtype));
      float cs, sn;
      rope_cs(pq * tab->omega[p], cs, sn);
      pf[pool_f16_offset(slot_new, 0, 2 * p)] = __float2half_rn(x0 * cs - x1 * sn);
      pf[pool_f16_offset(slot_new, 0, 2 * p + 1)] = __float2half_rn(x0 * sn + x1 * cs);
    }
  }
  int F1 = F0, C1 = C0, PH1 = PH0, ring_pos = -1;
  if (slot_new >= 0) {
    F1 = F0 - 1;
    ring_pos = (H0 + C0) % W1;
    C1 = C0 + 1;
    PH1 = max(PH0, slot_new + 1);
  }
  int es = -1, action = 0, j = -1, A1 = A0, H1 = H0, C2 = C1, F2 = F1, push = -1;
  if (slot_new >= 0 && C1 > c.window_size) {
    es = C0 > 0 ? c.win_ring[bh * W1 + H0] : slot_new;
    j = es == slot_new ? n : c.pool_tok[bh * c.pool_capacity + es];
    const int budget = budget_for((int64_t)n + 1 + c.token_offset, c.anchor_count, c.anchor_fraction);
    action = A0 < budget ? 1 : 2;
    H1 = (H0 + 1) % W1;
    C2 = C1 - 1;
    if (action == 1) {
      A1 = A0 + 1;
    } else {
      push = F1;
      F2 = F1 + 1;
    }
  }
  if (action == 2) {
    __syncthreads();   // the new row (if evicted itself) is visible to the block
    // 32 units (kv, group) x 8 threads, each scanning 32 centroids of the
    // fp16 shared-memory codebook for a top-4 shortlist, then rescoring it
    // with the float32 centroids: float32 distances, lowest index on ties
    // (_ckernels.pyx:150-162; SURVEY.md §7 hard part 2: shortlist + exact
    // rescore).
    const int64_t row = (bh * c.pool_capacity + es) * 256;
    const int u = threadIdx.x >> 3, part = threadIdx.x & 7;
    const int kv = u >> 4, grp = u & 15;
    float x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = load_elem(c.pool_rows, row + kv * 128 + grp * 8 + e, c.row_dtype);
    float sd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    int si[4] = {0, 0, 0, 0};
    const int lo_c = part * 32, hi_c = min(c.m, lo_c + 32);
    for (int ci = lo_c; ci < hi_c; ++ci) {
      const uint4 raw =
          *reinterpret_cast<const uint4 *>(&sm.cb[ci * 256 + kv * 128 + (threadIdx.x & 7) * 16]);
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
    for (int o = 1; o < 8; o <<= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
      if (ob < best || (ob == best && oi < best_i)) { best = ob; best_i = oi; }
    }
    if (part == 0)
      c.codes[bh * c.capacity * 32 + code_offset(j, kv, grp, 16)] = static_cast<uint8_t>(best_i);
  }
  if (threadIdx.x == 0) {
    int *plan = a.cnt + (int64_t)c.B * c.Hkv + c.B + bh * kPlanWords;
    plan[0] = slot_new;
    plan[1] = es;
    plan[2] = action;
    plan[3] = j;
    plan[4] = ring_pos;
    plan[5 + ANTKV_HS_ANCHORS] = A1;
    plan[5 + ANTKV_HS_WIN_HEAD] = H1;
    plan[5 + ANTKV_HS_WIN_COUNT] = C2;
    plan[5 + ANTKV_HS_FREE_TOP] = F2;
    plan[5 + ANTKV_HS_POOL_HIGH] = PH1;
    plan[10] = push;
    if (h == 0) c.positions[(int64_t)b * c.capacity + n] = a.qpos[b];   // read by nobody this step
  }
}

// Commit the plan (last CTA of (b, h): every reader of the head is done).
// All values were computed by prepare_update; these are independent stores
// (program order keeps slot_new == evicted slot, window_size == 0, right).
__device__ void commit_update(const antkv_cache_desc &c, const StepArgs &a, int b, int h, int n) {
  const int64_t bh = (int64_t)b * c.Hkv + h;
  const int *plan = a.cnt + (int64_t)c.B * c.Hkv + c.B + bh * kPlanWords;
  int p[11];
#pragma unroll
  for (int i = 0; i < 11; ++i) p[i] = __ldcg(plan + i);
  const int slot_new = p[0], es = p[1], action = p[2], j = p[3];
  int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
  if (slot_new >= 0) {
    c.pool_tok[bh * c.pool_capacity + slot_new] = n;
    c.pool_kind[bh * c.pool_capacity + slot_new] = ANTKV_KIND_WINDOWED;
    c.win_ring[bh * (c.window_size + 1) + p[4]] = slot_new;
  }
  if (action == 1) {
    c.pool_kind[bh * c.pool_capacity + es] = ANTKV_KIND_ANCHOR;
  } else if (action == 2) {
    atomicOr(&c.qmask[bh * (c.capacity / 32) + j / 32], 1u << (j % 32));
    c.pool_kind[bh * c.pool_capacity + es] = ANTKV_KIND_FREE;
    c.pool_tok[bh * c.pool_capacity + es] = -1;
    c.free_stack[bh * c.pool_capacity + p[10]] = es;
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) hs[i] = p[5 + i];
}

// ------------------------------------------------------------ streaming
// Per-warp state.  Lane (g = lane / 4, t = lane % 4) holds, per k-step s,
// the query-frame pairs 8s + t (u = 0) and 8s + 4 + t (u = 1) of column g.
struct WarpState {
  uint32_t kc[8][8];      // key rotation (cos,sin)/(-sin,cos) for rows g, g+8
  float2 fx[8], fy[8];    // frame pairs k = 2s + u, planar: fx[s] = (x_{2s}, x_{2s+1})
  float2 sc[8], ss[8];    // cos / sin of -32 omega for the same pairs
  float mrun[2], lrun[2]; // softmax of this lane's 2 columns (log2 units; lrun per lane)
  float o[8][4];          // O^T accumulators
};

// Per-lane constants of the code-tile addressing.
struct LaneAddr {
  uint32_t lcK, lcV;      // copy offset (lane & 7) * 16 (+128 for V) in byte 0
  uint32_t sK0, sK1;      // prmt selectors: byte 2(s&1) + (lane >> 4) of a K code word -> byte 1
  uint32_t sV0, sV1;      // byte 2(mt&1) + ((lane >> 3) & 1) of a V code word -> byte 1
};

__device__ __forceinline__ uint32_t word_of(const uint4 &v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// S^T = rot(K_hat) . B (8 HMMA in two chains) for one tile whose 16 K codes
// of this lane's ldmatrix row are `kr`.
__device__ __forceinline__ float4 qk_tile(const WarpState &w, const uint4 &kr,
                                          const uint32_t (&bq)[8][2], const LaneAddr &la) {
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    uint32_t a[4];
    ldsm_cb(prmt(word_of(kr, s >> 1), la.lcK, (s & 1) ? la.sK1 : la.sK0), a);
#ifndef FK_EXP_NOROT
    a[0] = rot2(a[0], w.kc[s][0], w.kc[s][1]);
    a[1] = rot2(a[1], w.kc[s][2], w.kc[s][3]);
    a[2] = rot2(a[2], w.kc[s][4], w.kc[s][5]);
    a[3] = rot2(a[3], w.kc[s][6], w.kc[s][7]);
#endif
#ifdef FK_EXP_NOQKMMA
    sa[s & 3] += __uint_as_float((a[0] ^ a[1] ^ a[2] ^ a[3] ^ bq[s][0]) & 0x3fffffffu);
#else
    if (s & 1) mma16816(sb, a, bq[s][0], bq[s][1]);
    else mma16816(sa, a, bq[s][0], bq[s][1]);
#endif
  }
  return make_float4(sa[0] + sb[0], sa[1] + sb[1], sa[2] + sb[2], sa[3] + sb[3]);
}

// O^T += V_hat^T . P (8 independent HMMA).
__device__ __forceinline__ void pv_tile(WarpState &w, const uint4 &vr, uint32_t pb0, uint32_t pb1,
                                        const LaneAddr &la) {
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    uint32_t a[4];
    ldsm_cb_t(prmt(word_of(vr, mt >> 1), la.lcV, (mt & 1) ? la.sV1 : la.sV0), a);
    mma16816(w.o[mt], a, pb0, pb1);
  }
}

// Online softmax of this lane's 4 scores (rows g / g+8, columns 2t / 2t+1;
// `mrow` bit 0 = row g valid, bit 1 = row g+8).  Returns P packed as the
// C-fragment half2 pairs of rows g and g+8.
__device__ __forceinline__ void softmax_p(WarpState &w, const float4 &sv, uint32_t mrow,
                                          uint32_t &x0, uint32_t &x1) {
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
  x0 = pack_h2(p00, p01);   // P[row g][cols 2t, 2t+1]
  x1 = pack_h2(p10, p11);   // P[row g+8][...]
}

// One code stage = even + odd tile.  `mrow` holds this lane's two row-valid
// bits of the tile whose columns it owns.
__device__ __forceinline__ void stage_tiles(WarpState &w, const uint4 &kre, const uint4 &vre,
                                            const uint4 &kro, const uint4 &vro, uint32_t mrow,
                                            const LaneAddr &la, bool lo) {
  uint32_t bq[8][2];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    bq[s][0] = pack_h2(w.fx[s].x, w.fy[s].x);
    bq[s][1] = pack_h2(w.fx[s].y, w.fy[s].y);
  }
  const float4 se = qk_tile(w, kre, bq, la);
  const float4 so = qk_tile(w, kro, bq, la);
#pragma unroll
  for (int s = 0; s < 8; ++s) {   // frames advance by R(-32): packed fp32 complex multiply
    const float2 x = w.fx[s], y = w.fy[s];
    w.fx[s] = __ffma2_rn(make_float2(-y.x, -y.y), w.ss[s], __fmul2_rn(x, w.sc[s]));
    w.fy[s] = __ffma2_rn(y, w.sc[s], __fmul2_rn(x, w.ss[s]));
  }
  uint32_t x0, x1;
  softmax_p(w, lo ? se : so, mrow, x0, x1);
  pv_tile(w, vre, movm_t(lo ? x0 : 0u), movm_t(lo ? x1 : 0u), la);
  pv_tile(w, vro, movm_t(lo ? 0u : x0), movm_t(lo ? 0u : x1), la);
}

// Online softmax over two stages at once (one lazy-max check): sA / sB are
// this lane's scores of stage A / B, mA / mB their row-valid bits.
__device__ __forceinline__ void softmax_p2(WarpState &w, const float4 &sA, uint32_t mA,
                                           const float4 &sB, uint32_t mB, uint32_t (&x)[4]) {
  float v[8];
  v[0] = (mA & 1u) ? sA.x : -INFINITY;
  v[1] = (mA & 1u) ? sA.y : -INFINITY;
  v[2] = (mA & 2u) ? sA.z : -INFINITY;
  v[3] = (mA & 2u) ? sA.w : -INFINITY;
  v[4] = (mB & 1u) ? sB.x : -INFINITY;
  v[5] = (mB & 1u) ? sB.y : -INFINITY;
  v[6] = (mB & 2u) ? sB.z : -INFINITY;
  v[7] = (mB & 2u) ? sB.w : -INFINITY;
  const float c0 = fmaxf(fmaxf(v[0], v[2]), fmaxf(v[4], v[6]));   // column 2t
  const float c1 = fmaxf(fmaxf(v[1], v[3]), fmaxf(v[5], v[7]));   // column 2t+1
  if (__any_sync(0xffffffffu, c0 > w.mrun[0] + 8.f || c1 > w.mrun[1] + 8.f)) {
    const float mn0 = fmaxf(w.mrun[0], shfl_max_g(c0));
    const float mn1 = fmaxf(w.mrun[1], shfl_max_g(c1));
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
  // a column with no valid score yet keeps mrun = -inf: subtract 0 instead
  const float m0 = w.mrun[0] == -INFINITY ? 0.f : w.mrun[0];
  const float m1 = w.mrun[1] == -INFINITY ? 0.f : w.mrun[1];
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = ex2(v[i] - ((i & 1) ? m1 : m0));   // ex2(-inf) = 0
  w.lrun[0] += (p[0] + p[2]) + (p[4] + p[6]);
  w.lrun[1] += (p[1] + p[3]) + (p[5] + p[7]);
  x[0] = pack_h2(p[0], p[1]);   // stage A, row g
  x[1] = pack_h2(p[2], p[3]);   // stage A, row g+8
  x[2] = pack_h2(p[4], p[5]);
  x[3] = pack_h2(p[6], p[7]);
}

__device__ __forceinline__ void advance_frames(WarpState &w) {
#pragma unroll
  for (int s = 0; s < 8; ++s) {   // frames advance by R(-32): packed fp32 complex multiply
    const float2 x = w.fx[s], y = w.fy[s];
    w.fx[s] = __ffma2_rn(make_float2(-y.x, -y.y), w.ss[s], __fmul2_rn(x, w.sc[s]));
    w.fy[s] = __ffma2_rn(y, w.sc[s], __fmul2_rn(x, w.ss[s]));
  }
}

// One ring slot = two stages = tiles 0..3 (stage A: 0 even / 1 odd, stage B:
// 2 / 3).  All QK products first (8 independent HMMA chains), one softmax,
// then all PV products, so each phase is one long basic block.
__device__ __forceinline__ void slot_tiles(WarpState &w, const uint8_t *tb, int tk, int tv,
                                           uint32_t qwA, uint32_t qwB, const LaneAddr &la,
                                           bool lo) {
  const uint4 k0 = *reinterpret_cast<const uint4 *>(tb + 0 * FK_TILE_BYTES + tk * 16);
  const uint4 k1 = *reinterpret_cast<const uint4 *>(tb + 1 * FK_TILE_BYTES + tk * 16);
  const uint4 k2 = *reinterpret_cast<const uint4 *>(tb + 2 * FK_TILE_BYTES + tk * 16);
  const uint4 k3 = *reinterpret_cast<const uint4 *>(tb + 3 * FK_TILE_BYTES + tk * 16);
  float4 sA, sB;
  {
    uint32_t bq[8][2];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      bq[s][0] = pack_h2(w.fx[s].x, w.fy[s].x);
      bq[s][1] = pack_h2(w.fx[s].y, w.fy[s].y);
    }
    const float4 s0 = qk_tile(w, k0, bq, la);
    const float4 s1 = qk_tile(w, k1, bq, la);
    sA = lo ? s0 : s1;
  }
  advance_frames(w);
  {
    uint32_t bq[8][2];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      bq[s][0] = pack_h2(w.fx[s].x, w.fy[s].x);
      bq[s][1] = pack_h2(w.fx[s].y, w.fy[s].y);
    }
    const float4 s2 = qk_tile(w, k2, bq, la);
    const float4 s3 = qk_tile(w, k3, bq, la);
    sB = lo ? s2 : s3;
  }
  advance_frames(w);
  const uint4 v0 = *reinterpret_cast<const uint4 *>(tb + 0 * FK_TILE_BYTES + 256 + tv * 16);
  const uint4 v1 = *reinterpret_cast<const uint4 *>(tb + 1 * FK_TILE_BYTES + 256 + tv * 16);
  const uint4 v2 = *reinterpret_cast<const uint4 *>(tb + 2 * FK_TILE_BYTES + 256 + tv * 16);
  const uint4 v3 = *reinterpret_cast<const uint4 *>(tb + 3 * FK_TILE_BYTES + 256 + tv * 16);
  uint32_t x[4];
  softmax_p2(w, sA, (qwA & 1u) | ((qwA >> 7) & 2u), sB, (qwB & 1u) | ((qwB >> 7) & 2u), x);
#ifndef FK_EXP_NOPV
  pv_tile(w, v0, movm_t(lo ? x[0] : 0u), movm_t(lo ? x[1] : 0u), la);
  pv_tile(w, v1, movm_t(lo ? 0u : x[0]), movm_t(lo ? 0u : x[1]), la);
  pv_tile(w, v2, movm_t(lo ? x[2] : 0u), movm_t(lo ? x[3] : 0u), la);
  pv_tile(w, v3, movm_t(lo ? 0u : x[2]), movm_t(lo ? 0u : x[3]), la);
#else
  w.o[0][0] += __uint_as_float(x[0] ^ x[1] ^ x[2] ^ x[3] ^ v0.x ^ v1.x ^ v2.x ^ v3.x);
#endif
}

// One pool tile (16 full-precision slots) in the absolute frame `bqa`
// (columns 4-7 zero; only the lanes owning columns 0-3 keep scores).
__device__ __forceinline__ void pool_tile(WarpState &w, uint32_t base, const uint32_t (&bqa)[8][2],
                                          uint32_t mrow, bool lo) {
  const int lane = threadIdx.x & 31;
  const int tk = (lane & 7) + 8 * ((lane >> 3) & 1), hk = lane >> 4;
  const int tv = (lane & 7) + 8 * (lane >> 4), pv = (lane >> 3) & 1;
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    uint32_t a[4];
    ldsm_x4(base + tk * 256 + ((((2 * s + hk) ^ (lane & 7))) << 4), a);
    if (s & 1) mma16816(sb, a, bqa[s][0], bqa[s][1]);
    else mma16816(sa, a, bqa[s][0], bqa[s][1]);
  }
  const float4 sv = make_float4(sa[0] + sb[0], sa[1] + sb[1], sa[2] + sb[2], sa[3] + sb[3]);
  uint32_t x0, x1;
  softmax_p(w, sv, lo ? mrow : 0u, x0, x1);
  const uint32_t p0 = movm_t(lo ? x0 : 0u), p1 = movm_t(lo ? x1 : 0u);
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    uint32_t a[4];
    ldsm_x4_t(base + 4096 + tv * 256 + ((((2 * mt + pv) ^ (lane & 7))) << 4), a);
    mma16816(w.o[mt], a, p0, p1);
  }
}

// ---------------------------------------------------------------- kernel
__global__ void __launch_bounds__(FK_THREADS, 1)
decode_fast_kernel(antkv_cache_desc c, StepArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  FastSmem &sm = *reinterpret_cast<FastSmem *>(smraw);
  MergeSmem &mg = *reinterpret_cast<MergeSmem *>(&sm.pool[0][0]);
  // grid (heads, splits, sequences), heads fastest: the CTAs are dispatched
  // split-major, so each head's last split -- the one with the reduced share
  // that also prepares the cache update -- goes out last, onto the SMs the
  // previous launch frees last (its combining CTAs), where the smaller share
  // absorbs the late start
  const int b = blockIdx.z, h = blockIdx.x, split = blockIdx.y;
  const int S = a.splits;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t bh = (int64_t)b * c.Hkv + h;
  const bool last_split = split == S - 1;
  const bool prep = last_split && a.knew;
  unsigned long long tr[FK_TRACE_WORDS];
  // stamps: SM cycle counter (clock64) relative to the start, plus the
  // global timer at the start to align CTAs (globaltimer ticks too coarsely
  // for sub-microsecond phases)
#define FK_TR(i) \
  if (a.trace && threadIdx.x == 0) tr[i] = clock64();
  FK_TR(1);
  unsigned long long g0 = 0;
  if (a.trace && threadIdx.x == 0) g0 = gtimer();

  // ---- prologue.  Phase 0 touches only data no kernel writes during
  // decoding (the prepared codebook and RoPE tables), so with programmatic
  // dependent launch it overlaps the tail of the previous kernel in the
  // stream; griddepcontrol.wait then orders everything else (cache state, q)
  // after that kernel has completed.
  if (threadIdx.x == 0) {
    for (int ww = 0; ww < FK_WARPS; ++ww) {
      for (int s = 0; s < FK_NS; ++s) mbar_init(&sm.full[ww][s], 1);
      mbar_init(&sm.pfull[ww], 1);
    }
    mbar_init(&sm.tbar, 1);
    mbar_init(&sm.qbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // compact fp16 codebook row of code threadIdx.x ([K 8 | V 8] halves, 32 B;
  // immutable while decoding, so read before the wait), replicated into the
  // eight bank groups of sm.cb before the frames' barrier
  const uint4 *cbg = reinterpret_cast<const uint4 *>(c.codebook_f16) + (int64_t)h * (FK_CB_BYTES / 16) +
                     2 * threadIdx.x;
  const uint4 cbk = __ldg(cbg), cbv = __ldg(cbg + 1);
  const int qbytes = 4 * 128 * dtype_size(a.qdtype);
  if (threadIdx.x == 0) {
    mbar_expect_tx(&sm.tbar, sizeof(FastTables));
    tma_bulk_g2s(&sm.tab, c.fast_tables, sizeof(FastTables), &sm.tbar);
    if (a.early_q) {
      mbar_expect_tx(&sm.qbar, qbytes);
      tma_bulk_g2s(sm.qraw, reinterpret_cast<const uint8_t *>(a.q) + ((int64_t)b * c.Hq + h * 4) * (qbytes / 4),
                   qbytes, &sm.qbar);   // rows h*4 .. h*4+3 of sequence b
    }
  }
  // Cache state is read before the wait only when the host knows the
  // previous kernel in the stream did not write this cache (a.early); the
  // loads and the table copy are in flight together.
  if (!a.early) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n = c.seq_len[b];
  const int pool_high = c.hstate[bh * ANTKV_HSTATE_WORDS + ANTKV_HS_POOL_HIGH];
  const int64_t pos0 = c.positions[(int64_t)b * c.capacity];
  int64_t qp = a.early_q ? a.qpos[b] : 0;
  WarpState w;

  // ---- phase 1 (needs n / pool_high): work split, bulk copies of the code
  // and pool tiles, qmask words, pool-tile kinds.  Code tiles: the last
  // split also prepares the cache update, so it gets half a share; each warp
  // streams Tw contiguous tiles.
  const int ntiles = (n + 15) >> 4;
  const float shares = (a.knew && S > 1) ? S - 0.5f : (float)S;
  const int per_cta = ((int)ceilf(ntiles / shares) + 4 * FK_WARPS - 1) / (4 * FK_WARPS) * (4 * FK_WARPS);
  const int T0 = split * per_cta;
  const int mine = max(0, min(per_cta, ntiles - T0));
  const int Tw = ((mine + FK_WARPS - 1) / FK_WARPS + 3) & ~3;   // a multiple of 4 tiles
  const int nstages = Tw / 2;                                    // even
  const int nslots = nstages / 2;
  const int wt0 = T0 + warp * Tw;
  const int cap_tiles = c.capacity / 16;
  const uint8_t *codes = c.codes + bh * c.capacity * 32;   // 32 code bytes per slot
  // pool tiles: an equal share per CTA, one tile per warp per round
  const int ptiles = (pool_high + 15) >> 4;
  const int pper = (ptiles + S - 1) / S;
  const int pt0 = min(ptiles, split * pper), pt1 = min(ptiles, pt0 + pper);
  const uint8_t *pool_g = reinterpret_cast<const uint8_t *>(c.pool_f16) + bh * c.pool_capacity * 512;
  auto issue_code = [&](int it) {   // ring slot it % FK_NS <- tiles wt0 + 4 it .. + 3
    const int slot = it % FK_NS;
    int tile = wt0 + 4 * it;
    if (tile + 4 > cap_tiles) tile = 0;   // beyond capacity: masked dummy data
    mbar_expect_tx(&sm.full[warp][slot], FK_SLOT_BYTES);
    tma_bulk_g2s(&sm.ring[warp][slot][0], codes + (int64_t)tile * FK_TILE_BYTES, FK_SLOT_BYTES,
                 &sm.full[warp][slot]);
  };
  auto issue_pool = [&](int tile) {
    mbar_expect_tx(&sm.pfull[warp], FK_POOL_TILE_BYTES);
    tma_bulk_g2s(&sm.pool[warp][0], pool_g + (int64_t)tile * FK_POOL_TILE_BYTES, FK_POOL_TILE_BYTES,
                 &sm.pfull[warp]);
  };
#ifndef FK_EARLY_SLOTS
#define FK_EARLY_SLOTS 2   // slots 2-3 after the prologue: 33.4 -> 33.2 us (less shared-memory contention while the tables load)
#endif
  constexpr int kEarlySlots = FK_EARLY_SLOTS < FK_NS ? FK_EARLY_SLOTS : FK_NS;
  if (lane == 0) {
    if (pt0 + warp < pt1) issue_pool(pt0 + warp);
    for (int it = 0; it < min(nslots, kEarlySlots); ++it) issue_code(it);
  }
  // key-rotation constants and frame steps into registers (the tables copy
  // was issued first; the code / pool copies above are already in flight)
  mbar_wait(&sm.tbar, 0);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const float4 st = sm.tab.step[s][t];
    w.sc[s] = make_float2(st.x, st.z);
    w.ss[s] = make_float2(st.y, st.w);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint4 k = sm.tab.kc[s][u][t][g];
      w.kc[s][4 * u] = k.x;
      w.kc[s][4 * u + 1] = k.y;
      w.kc[s][4 * u + 2] = k.z;
      w.kc[s][4 * u + 3] = k.w;
    }
  }
  FK_TR(2);
  const int8_t *kinds = c.pool_kind + bh * c.pool_capacity;
  int8_t kd0 = ANTKV_KIND_FREE, kd1 = ANTKV_KIND_FREE;
  if (pt0 + warp < pt1) {
    kd0 = kinds[(pt0 + warp) * 16 + g];
    kd1 = kinds[(pt0 + warp) * 16 + g + 8];
  }
  // qmask words of this warp's range (one word per stage), up to 2 per lane
  const uint32_t *qmg = c.qmask + bh * (c.capacity / 32);
  uint32_t qmv[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = lane + 32 * u, word = (wt0 >> 1) + i;
    qmv[u] = (i < nstages && word * 32 < c.capacity) ? __ldcs(qmg + word) : 0u;
  }
  // (cos, sin) of every query frame of the CTA, cooperatively from
  // integer-reduced angles (frame 2w + e: warp w's even / odd tile frame;
  // frame 16: the absolute frame p_q of the pool rows)
  auto frame_angles = [&]() {
    for (int e = threadIdx.x; e < (2 * FK_WARPS + 1) * 64; e += FK_THREADS) {
      const int f = e >> 6, p = e & 63;
      const int64_t delta = f < 2 * FK_WARPS
          ? qp - (pos0 + (int64_t)(T0 + (f >> 1) * Tw) * 16 + (f & 1) * 16)
          : qp;
      float cs, sn;
      turns_cs(delta, sm.tab.turns[p], cs, sn);
      sm.ang[f][lane_pair_pos(p)] = make_float2(cs, sn);
    }
  };
  if (a.early_q) frame_angles();
  FK_TR(5);
  // inputs produced by earlier kernels (q, positions, the appended rows) are
  // read after the previous kernel completed unless the host vouched for
  // them (early / early_q); only then may the next kernel start (a
  // dependency chain of depth one).  With early_q nothing read here comes
  // from the previous kernel: wait and release after the streaming loop
  // instead (every launch still waits before it completes, so completion
  // keeps implying the predecessor's, and the dependents still launch only
  // after this launch has waited).
  if (!a.early_q) {
    if (a.early) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (!a.early_q) {
    qp = a.qpos[b];
    if (threadIdx.x == 0) {
      mbar_expect_tx(&sm.qbar, qbytes);
      tma_bulk_g2s(sm.qraw, reinterpret_cast<const uint8_t *>(a.q) + ((int64_t)b * c.Hq + h * 4) * (qbytes / 4),
                   qbytes, &sm.qbar);   // rows h*4 .. h*4+3 of sequence b
    }
  }
  FK_TR(3);

  // ---- phase 2: query rows, frames (the angles overlap the query copy)
  if (!a.early_q) frame_angles();
  mbar_wait(&sm.qbar, 0);
  const double pq = static_cast<double>(qp);
  {
    const float sc = rsqrtf(128.f) * 1.4426950408889634f;   // 1/sqrt(d) * log2(e)
    for (int e = threadIdx.x; e < 256; e += FK_THREADS)
      sm.qf[e >> 6][lane_pair_pos(e & 63)] =
          make_float2(load_elem(sm.qraw, 2 * e, a.qdtype) * sc, load_elem(sm.qraw, 2 * e + 1, a.qdtype) * sc);
  }
  {
    static_assert(FK_THREADS == 256, "one codebook row per thread");
    uint8_t *row = sm.cb + threadIdx.x * 256;
#pragma unroll
    for (int i = 0; i < 8; ++i) {   // copy (i + code) & 7 first: the 8 lanes of a phase hit 8 bank groups
      const int cp = (i + threadIdx.x) & 7;
      *reinterpret_cast<uint4 *>(row + cp * 16) = cbk;
      *reinterpret_cast<uint4 *>(row + 128 + cp * 16) = cbv;
    }
  }
  __syncthreads();
  if (kEarlySlots < FK_NS && lane == 0)   // the rest of the ring's first fill
    for (int it = kEarlySlots; it < min(nslots, FK_NS); ++it) issue_code(it);
  FK_TR(14);
  {
    const int fr = 2 * warp + (g >= 4 ? 1 : 0);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const float4 xq = *reinterpret_cast<const float4 *>(&sm.qf[g & 3][(s * 4 + t) * 2]);
      const float4 cf = *reinterpret_cast<const float4 *>(&sm.ang[fr][(s * 4 + t) * 2]);
      // pair u = 0: (xq.x, xq.y) rotated by (cf.x, cf.y); u = 1: (xq.z, xq.w) by (cf.z, cf.w)
      w.fx[s] = make_float2(xq.x * cf.x - xq.y * cf.y, xq.z * cf.z - xq.w * cf.w);
      w.fy[s] = make_float2(xq.x * cf.y + xq.y * cf.x, xq.z * cf.w + xq.w * cf.z);
    }
  }
  w.mrun[0] = w.mrun[1] = -INFINITY;
  w.lrun[0] = w.lrun[1] = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) w.o[i][e] = 0.f;
  FK_TR(4);
  // ---- the appended token (prep CTA, warp 0): attended like a pool row
  if (prep && warp == 0) {
    const int64_t kb = bh * 128 + 4 * lane;
    float kk[4], vv[4], cs[2], sn[2];
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const float2 ca = sm.ang[2 * FK_WARPS][lane_pair_pos(2 * lane + pp)];
      cs[pp] = ca.x;
      sn[pp] = ca.y;
      const float x0 = round_to(c.row_dtype, load_elem(a.knew, kb + 2 * pp, a.kvdtype));
      const float x1 = round_to(c.row_dtype, load_elem(a.knew, kb + 2 * pp + 1, a.kvdtype));
      kk[2 * pp] = __half2float(__float2half_rn(x0 * cs[pp] - x1 * sn[pp]));
      kk[2 * pp + 1] = __half2float(__float2half_rn(x0 * sn[pp] + x1 * cs[pp]));
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      vv[e] = __half2float(__float2half_rn(round_to(c.row_dtype, load_elem(a.vnew, kb + e, a.kvdtype))));
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
      float sdot = 0.f;
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const float2 xq = sm.qf[hh][lane_pair_pos(2 * lane + pp)];
        const float x0 = xq.x, x1 = xq.y;
        sdot += (x0 * cs[pp] - x1 * sn[pp]) * kk[2 * pp] + (x0 * sn[pp] + x1 * cs[pp]) * kk[2 * pp + 1];
      }
      sdot = warp_sum(sdot);
      *reinterpret_cast<float4 *>(&sm.xo[hh][4 * lane]) = make_float4(vv[0], vv[1], vv[2], vv[3]);
      if (lane == 0) sm.xm[hh] = sdot;
    }
  } else if (warp == 0 && lane < 4) {
    sm.xm[lane] = -INFINITY;
  }

  const bool lo = t < 2;   // owns columns 0-3 (even tile / pool)
  // ---- pool tiles (absolute frame: R(p_q) q, columns 4-7 zero)
  if (pt0 + warp < pt1) {
    uint32_t bqa[8][2];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const float4 xq = *reinterpret_cast<const float4 *>(&sm.qf[g & 3][(s * 4 + t) * 2]);
      const float4 ca = *reinterpret_cast<const float4 *>(&sm.ang[2 * FK_WARPS][(s * 4 + t) * 2]);
      bqa[s][0] = g < 4 ? pack_h2(xq.x * ca.x - xq.y * ca.y, xq.x * ca.y + xq.y * ca.x) : 0u;
      bqa[s][1] = g < 4 ? pack_h2(xq.z * ca.z - xq.w * ca.w, xq.z * ca.w + xq.w * ca.z) : 0u;
    }
    int r = 0;
    for (int tile = pt0 + warp; tile < pt1; tile += FK_WARPS, ++r) {
      if (r > 0) {
        kd0 = kinds[tile * 16 + g];
        kd1 = kinds[tile * 16 + g + 8];
      }
      const uint32_t mrow = (kd0 != ANTKV_KIND_FREE ? 1u : 0u) | (kd1 != ANTKV_KIND_FREE ? 2u : 0u);
      mbar_wait(&sm.pfull[warp], r & 1);
      pool_tile(w, smem_u32(&sm.pool[warp][0]), bqa, mrow, lo);
      __syncwarp();
      if (lane == 0 && tile + FK_WARPS < pt1) {
        fence_proxy_async();
        issue_pool(tile + FK_WARPS);
      }
    }
  }
  FK_TR(6);
  if (prep) {
    prepare_update(c, a, sm, b, h, n, pq);
  }
  FK_TR(7);

  // ---- code tiles
  if (nstages > 0) {
    LaneAddr la;
    la.lcK = (lane & 7) * 16;
    la.lcV = la.lcK + 128;
    la.sK0 = 0x5504u | ((0u + (lane >> 4)) << 4);
    la.sK1 = 0x5504u | ((2u + (lane >> 4)) << 4);
    la.sV0 = 0x5504u | ((0u + ((lane >> 3) & 1)) << 4);
    la.sV1 = 0x5504u | ((2u + ((lane >> 3) & 1)) << 4);
    const int tk = (lane & 7) + 8 * ((lane >> 3) & 1);     // K-side token row
    const int tv = (lane & 7) + 8 * (lane >> 4);          // V-side token row
    const int rowbit = g + (lo ? 0 : 16);                 // rows g (+8 via >> 7 below)
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (lane + 32 * u < nstages) sm.qm[warp][lane + 32 * u] = qmv[u];
    __syncwarp();                                         // qm words visible to the warp
    FK_TR(8);
    for (int it = 0; it < nslots; ++it) {
      const int slot = it % FK_NS;
      mbar_wait(&sm.full[warp][slot], (it / FK_NS) & 1);
      const uint32_t qwA = sm.qm[warp][2 * it] >> rowbit, qwB = sm.qm[warp][2 * it + 1] >> rowbit;
#ifdef FK_EXP_STREAM
      {
        const uint4 k0 = *reinterpret_cast<const uint4 *>(&sm.ring[warp][slot][tk * 16]);
        w.o[0][0] += __uint_as_float((k0.x ^ qwA ^ qwB) & 0x3fffffffu) * 1e-30f;
      }
#else
      slot_tiles(w, &sm.ring[warp][slot][0], tk, tv, qwA, qwB, la, lo);
#endif
      __syncwarp();
      if (lane == 0 && it + FK_NS < nslots) {   // every lane has read the slot: refill it
        fence_proxy_async();
        issue_code(it + FK_NS);
      }
    }
  }
  FK_TR(9);
  if (a.early_q) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  // ---- merge 8 warps x 2 streams (+ the appended token) -> partial (natural log)
  __syncthreads();   // pool tiles consumed: the pool area becomes merge scratch
  FK_TR(12);
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
    mg.m[warp][2 * t] = w.mrun[0];
    mg.m[warp][2 * t + 1] = w.mrun[1];
    mg.l[warp][2 * t] = lsum0;
    mg.l[warp][2 * t + 1] = lsum1;
  }
  __syncthreads();
  // per head: max, weights of the 16 streams (+ the appended token), normaliser
  float *mw = reinterpret_cast<float *>(&sm.ring[0][0][0]);   // [4][17] weights, [4] M, [4] L
  if (threadIdx.x < 4) {
    const int hh = threadIdx.x;
    float M = sm.xm[hh];
#pragma unroll
    for (int src = 0; src < 2 * FK_WARPS; ++src) M = fmaxf(M, mg.m[src >> 1][hh + 4 * (src & 1)]);
    float L = 0.f;
#pragma unroll
    for (int src = 0; src < 2 * FK_WARPS; ++src) {
      const float mv = mg.m[src >> 1][hh + 4 * (src & 1)];
      const float f = (mv == -INFINITY) ? 0.f : ex2(mv - M);
      mw[hh * 17 + src] = f;
      L += f * mg.l[src >> 1][hh + 4 * (src & 1)];
    }
    const float fx = (sm.xm[hh] == -INFINITY) ? 0.f : ex2(sm.xm[hh] - M);
    mw[hh * 17 + 16] = fx;
    L += fx;
    mw[68 + hh] = M;
    mw[72 + hh] = L;
  }
  __syncthreads();
  const int64_t rows = (int64_t)c.B * c.Hq;
  const int64_t row0 = ((int64_t)split * c.B + b) * c.Hq + h * 4;
  for (int i = threadIdx.x; i < 4 * 128; i += FK_THREADS) {
    const int hh = i >> 7, dim = i & 127;
    float O = mw[hh * 17 + 16] != 0.f ? mw[hh * 17 + 16] * sm.xo[hh][dim] : 0.f;   // xo unset unless prep
#pragma unroll
    for (int src = 0; src < 2 * FK_WARPS; ++src)
      O = fmaf(mw[hh * 17 + src], mg.o[src >> 1][hh + 4 * (src & 1)][dim], O);
    a.ws_o[(row0 + hh) * 128 + dim] = O;
    if (dim == 0) {
      a.ws_m[row0 + hh] = mw[68 + hh] * ln2;
      a.ws_l[row0 + hh] = mw[72 + hh];
    }
  }

  FK_TR(13);
  // ---- arrivals: the head's last split (the reduced-share CTA that also
  // prepared the cache update, dispatched last) combines and commits; every
  // other CTA releases its partial with a fire-and-forget red.release and
  // exits at once, so the next launch's CTA can take its SM without waiting
  // for a gpu-scope fence round trip (a returned ticket cost ~1-2 us here).
  // The CTA barrier orders every thread's partial stores before thread 0's
  // release (cumulative); the combiner's acquire load of the count orders
  // its reads of the partials after them, and the next barrier passes that
  // on to the CTA.  The combiners are the last CTAs in dispatch order (split
  // major), and the ones waiting hold at most one SM per (b, head) -- never
  // all SMs -- while every other CTA runs to completion, so the CTAs a
  // combiner waits for always get an SM (also when S x B x Hkv exceeds the
  // SM count, e.g. the minimum splits of very long caches).  The last CTA of
  // the heads' combiners publishes the sequence's new length.
  __syncthreads();
  const bool combiner = split == S - 1;
  if (!combiner) {
    if (threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.cnt + bh) : "memory");
  } else if (threadIdx.x == 0) {
    uint32_t seen;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(a.cnt + bh) : "memory");
      if ((int)seen >= S - 1) break;
      __nanosleep(64);
    }
  }
  if (combiner) __syncthreads();
  if (a.trace && threadIdx.x == 0) {
    tr[10] = gtimer();
    unsigned long long *o =
        a.trace + FK_TRACE_WORDS * ((blockIdx.z * gridDim.x + blockIdx.x) * gridDim.y + blockIdx.y);
    o[0] = smid() | ((unsigned long long)split << 32);   // (the split stands in for the old ticket)
    for (int i = 2; i <= 9; ++i) o[i] = tr[i] - tr[1];
    o[10] = tr[10];   // global timer after the arrival (absolute, like o[1])
    tr[12] = clock64();   // ... and the SM clock at the same point (clock calibration)
    o[1] = g0;
    o[11] = 0;
    o[12] = tr[12] - tr[1];
    o[13] = tr[13] - tr[1];
    o[14] = tr[14] - tr[1];
    o[15] = 0;
    sm.t0clk = tr[1];
  }
  if (!combiner) return;
  if (threadIdx.x == 0 && a.knew &&
      atomicAdd(&a.cnt[(int64_t)c.B * c.Hkv + b], 1) == c.Hkv - 1) {
    // the last CTA of every head of sequence b is here, so every CTA of the
    // sequence has read seq_len: publish the appended token
    c.seq_len[b] = n + 1;
    a.cnt[(int64_t)c.B * c.Hkv + b] = 0;
  }
  if (warp < 4) {
    // warp hh combines head hh: lane = 4 dims; the loads of up to 24 splits
    // are in flight together, then a running max across passes
    const int hh = warp, d4 = 4 * lane;
    const int64_t row = (int64_t)b * c.Hq + h * 4 + hh;
    float M = -INFINITY, L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int CH = 24;
    for (int s0 = 0; s0 < S; s0 += CH) {
      float ms[CH], ls[CH];
      float4 v[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int s2 = min(s0 + u, S - 1);
        ms[u] = __ldcg(a.ws_m + s2 * rows + row);
        ls[u] = __ldcg(a.ws_l + s2 * rows + row);
        v[u] = __ldcg(reinterpret_cast<const float4 *>(a.ws_o + (s2 * rows + row) * 128 + d4));
      }
      float mc = M;
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (s0 + u < S) mc = fmaxf(mc, ms[u]);
      if (mc == -INFINITY) continue;
      const float al = (M == -INFINITY) ? 0.f : __expf(M - mc);
      L *= al;
      acc.x *= al; acc.y *= al; acc.z *= al; acc.w *= al;
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const float wv = (s0 + u >= S || ms[u] == -INFINITY) ? 0.f : __expf(ms[u] - mc);
        L = fmaf(wv, ls[u], L);
        acc.x = fmaf(wv, v[u].x, acc.x);
        acc.y = fmaf(wv, v[u].y, acc.y);
        acc.z = fmaf(wv, v[u].z, acc.z);
        acc.w = fmaf(wv, v[u].w, acc.w);
      }
      M = mc;
    }
    const float inv = 1.f / L;
    *reinterpret_cast<float4 *>(a.out + row * 128 + d4) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (lane == 0 && a.lse) a.lse[row] = M + logf(L);
    if (a.trace && threadIdx.x == 0) {
      unsigned long long *o =
          a.trace + FK_TRACE_WORDS * ((blockIdx.z * gridDim.x + blockIdx.x) * gridDim.y + blockIdx.y);
      o[15] = clock64() - sm.t0clk;
    }
  } else if (threadIdx.x == 128) {
    if (a.knew) commit_update(c, a, b, h, n);   // overlaps the combine
    if (a.trace) {
      unsigned long long *o =
          a.trace + FK_TRACE_WORDS * ((blockIdx.z * gridDim.x + blockIdx.x) * gridDim.y + blockIdx.y);
      o[11] = clock64() - sm.t0clk;
    }
    a.cnt[bh] = 0;
  }
}

__global__ void smem_base_probe_kernel(uint32_t *out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  *out = smem_u32(smraw);
}

// The kernel's gathers assume dynamic shared memory starts at 0x400.
int decode_fast_smem_base_ok() {
  static int ok = -1;
  if (ok < 0) {
    uint32_t *d = nullptr, h = 0;
    ok = 0;
    if (cudaMalloc(&d, 4) == cudaSuccess) {
      smem_base_probe_kernel<<<1, 1, 1024>>>(d);
      if (cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost) == cudaSuccess) ok = (h == FK_SMEM_BASE);
      cudaFree(d);
    }
    cudaGetLastError();
  }
  return ok;
}

int decode_fast_supported(const antkv_cache_desc &c) {
  return decode_fast_smem_base_ok() && c.d == 128 && c.d_sub == 8 && c.m <= 256 && c.code_bytes == 1 && c.Hq == 4 * c.Hkv &&
         c.codebook_f16 != nullptr && c.pool_f16 != nullptr && c.fast_tables != nullptr &&
         c.capacity % 128 == 0 && c.pool_capacity % 16 == 0;
}

// CTAs per (sequence, head): one resident CTA per SM in total.
void decode_fast_plan(const antkv_cache_desc &c, int requested, int &code_splits, int &pool_splits) {
  const int bh = c.B * c.Hkv;
  code_splits = requested > 0 ? requested : max(1, 148 / bh);
  // per-warp qmask staging caps a CTA at 8 warps x 128 tiles (FK_MAX_WARP_WORDS)
  // (per_cta <= 1008 tiles once splits >= cap_tiles / 1000 + 1)
  const int min_code = c.capacity / 16 / 1000 + 1;
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
      g_trace_n = FK_TRACE_WORDS * 65536;
      if (cudaMalloc(&g_trace, sizeof(unsigned long long) * g_trace_n) != cudaSuccess) g_trace = nullptr;
    }
  }
  return g_trace;
}

}  // namespace antkv

// Debug: copy the per-CTA timeline of the last traced fast-decode launch
// (FK_TRACE_WORDS = 16 words per CTA, see FK_TRACE_WORDS) to host memory.
// Returns the number of words copied.
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
  if (a.trace) {   // two halves, alternating per launch: the previous launch stays readable
    static unsigned launch_no = 0;
    a.trace += (size_t)(launch_no++ & 1) * FK_TRACE_WORDS * 32768;
  }
  // reads before griddepcontrol.wait only on a stream the caller declared
  // exclusive to this library (antkv_stream_exclusive): then the previous
  // kernel is one of ours, and the state of another cache ...
  a.early = previous_cache_on_stream(st, c.codes) != c.codes && stream_exclusive(st);
  // ... and q / qpos, unless the previous fused launch on this stream (the
  // only kernel that can still be running then) wrote them
  a.early_q = a.early && !overlaps_previous_fast_outputs(st, q, (int64_t)c.B * c.Hq * 128 * dtype_size(qdtype)) &&
              !overlaps_previous_fast_outputs(st, qpos, (int64_t)c.B * sizeof(int64_t)) &&
              (!knew || !overlaps_previous_fast_outputs(st, knew, (int64_t)c.B * c.Hkv * 128 * dtype_size(kvdtype))) &&
              (!vnew || !overlaps_previous_fast_outputs(st, vnew, (int64_t)c.B * c.Hkv * 128 * dtype_size(kvdtype)));
  record_fast_outputs(st, out, (int64_t)c.B * c.Hq * 128 * sizeof(float), lse,
                      lse ? (int64_t)c.B * c.Hq * sizeof(float) : 0);
  const size_t smem = sizeof(FastSmem);
  static bool attr_set[64] = {};   // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaFuncSetAttribute(decode_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  // programmatic dependent launch: the prologue's immutable prefetch overlaps
  // the previous kernel's tail (griddepcontrol.wait orders the rest)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c.Hkv, a.splits, c.B);
  cfg.blockDim = dim3(FK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static int pdl = -1;   // ANTKV_NO_PDL=1 disables programmatic dependent launch (A/B timing)
  if (pdl < 0) {
    const char *e = getenv("ANTKV_NO_PDL");
    pdl = !(e && e[0] == '1');
  }
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, decode_fast_kernel, c, a);
  if (e != cudaSuccess) return cuda_status(e, "decode_fast_kernel");
  ANTKV_LAUNCH_CHECK("decode_fast_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
