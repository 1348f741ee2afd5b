// sm_100a decode attention for every d = 128 code shape that the d8m256
// kernel (decode_fast.cu) does not cover: d_sub 4 / 8 / 16 / 32 / 64, m up
// to 65536 (1- or 2-byte indices, e.g. config #3's 0.375-bit d32m4096 and
// config #4's 2-bit d4m256), GQA groups of 1, 2, 4 or 8 query heads.
// Reference semantics: cache.py:168-178 (RoPE after reconstruction, softmax
// over the whole cache, A.V); the cache update runs before / after this
// launch (antkv_cache_append / antkv_cache_evict, cache.py:157-166,180-193).
//
// A codebook of m = 4096 centroids of 32 dims is 256 KB per head and side,
// larger than shared memory, so centroids are not gathered from shared
// memory as in the d8m256 kernel.  Instead each warp reconstructs 16-token
// tiles into a private shared-memory ring:
//   * code tiles ([K 16 x G | V 16 x G] code units, the cache's own layout)
//     arrive by bulk copy (cp.async.bulk + mbarrier) into a per-warp ring,
//     several tiles per copy;
//   * lane l owns token row l % 16 of side l / 16 (K or V): it reads that
//     row's G codes from the ring and issues one cp.async per 16-byte (8 for
//     d_sub = 4) centroid chunk from the fp16 codebook copy
//     (codebook_f16g [Hkv][2][m][d_sub], L2 / L1 resident) straight into
//     the reconstructed tile [K | V][16][128], chunk-swizzled like the pool
//     tiles so ldmatrix reads are conflict-free;
//   * the tile is consumed two tiles later (three-tile ring): ldmatrix,
//     per-row RoPE R(r) (fp16 constants), S^T = rot(K_hat) . B and
//     O^T += V_hat^T . P with m16n8k16 MMAs, exactly the per-tile math of
//     the pool path of decode_fast.cu.
// The MMA's 8 B columns are (query head c % GQ, tile phase c / GQ): a
// stage of F = 8 / GQ consecutive tiles shares one set of query frames, the
// tile with phase i owning columns [i GQ, (i+1) GQ); frames advance by
// R(-16 F omega) per stage (packed fp32), seeded from integer-reduced angles.
// Pool tiles (anchors + window, K rotated at its own position, fp16 in
// pool_f16) are bulk-copied and attended in the absolute frame.  Each CTA
// writes an (o, m, l) partial; the last CTA of each (sequence, head) (atomic
// ticket) merges the splits.
#include "common.cuh"

namespace antkv {

__global__ void cache_pool_f16_kernel(antkv_cache_desc c);   // cache.cu

namespace {

constexpr int TW = 8;                 // warps per CTA
constexpr int TT = 32 * TW;
constexpr int TNST = 3;               // reconstructed-tile ring depth per warp
constexpr int TSTAGE = 8192;          // [K | V][16 slots][128] fp16
constexpr int TCS = 1024;             // code ring slot bytes
constexpr int TNCS = 3;               // code ring slots per warp

struct __align__(128) TcSmem {
  uint8_t stage[TNST][TW][TSTAGE];   // slot-major: slot 1 of all warps is one 64 KB block
  uint8_t code[TW][TNCS][TCS];
  float2 step[64];                    // (cos, sin) of -16 F omega_p, lane-pair order
  unsigned long long cfull[TW][TNCS];
  unsigned long long pfull[TW];
  float mw[8][TW * 8 + 1];            // merge weights per head and source (+ M, L)
  uint16_t cunp[TW][32 * 8];          // a tile's 12-bit packed codes, unpacked (rows x groups <= 8)
  int ticket;
};

struct TcArgs {
  const void *q;          // [B][Hq][128]
  int qdtype;
  const int64_t *qpos;    // [B]
  float *ws_o, *ws_m, *ws_l;
  float *out, *lse;       // [B][Hq][128], [B][Hq] (lse may be NULL)
  int *cnt;               // [B*Hkv] self-resetting CTA tickets
  int splits;
  int gq;                 // query heads per KV head (1, 2, 4, 8)
};

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mb_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cpa16(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16_cg(uint32_t dst, const void *src) {   // L2 only (no L1 allocation)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movt(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t hu(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
__device__ __forceinline__ __half2 uh(uint32_t u) { return *reinterpret_cast<__half2 *>(&u); }
__device__ __forceinline__ uint32_t pk(float x, float y) { return hu(__floats2half2_rn(x, y)); }
// (x0, x1) -> (c x0 - s x1, s x0 + c x1) with cs = (c, s), ns = (-s, c)
__device__ __forceinline__ uint32_t rot(uint32_t x, uint32_t cs, uint32_t ns) {
  const __half2 v = uh(x);
  __half2 r = __hmul2(__high2half2(v), uh(ns));
  r = __hfma2(__low2half2(v), uh(cs), r);
  return hu(r);
}
__device__ __forceinline__ float e2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gmax(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
  return v;
}
__device__ __forceinline__ float gsum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  return v;
}

// Per-lane streaming state (lane g = lane / 4 owns B column g and rows g,
// g + 8 of each tile; t = lane % 4 its pairs / columns 2t, 2t + 1).
struct Lane {
  uint32_t kc[8][8];      // row rotations R(r omega), rows g, g + 8 (fp16 pairs)
  float2 fx[8], fy[8];    // query frame of column g: pairs 8s + t (.x), 8s + 4 + t (.y)
  uint32_t bq[8][2];      // the same, packed fp16 (the MMA B operand)
  float mrun[2], lrun[2]; // softmax of columns 2t, 2t + 1 (log2 units)
  float o[8][4];          // O^T accumulators
};

// One reconstructed (or pool) tile at shared address `base`: scores of the
// 16 rows against the 8 columns, online softmax of this lane's two columns
// (valid when their phase equals `phase`; rows by `rows` bits g / g + 8),
// then O^T += V^T P.
template <bool ROT>
__device__ __forceinline__ void tile_attend(Lane &w, uint32_t base, const uint32_t (&bq)[8][2], uint32_t rows,
                                            bool c0ok, bool c1ok) {
  const int lane = threadIdx.x & 31;
  const int tk = (lane & 7) + 8 * ((lane >> 3) & 1), hk = lane >> 4;
  const int tv = (lane & 7) + 8 * (lane >> 4), pv = (lane >> 3) & 1;
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    uint32_t a[4];
    ldsm4(base + tk * 256 + ((((2 * s + hk) ^ (lane & 7))) << 4), a);
    if (ROT) {
      a[0] = rot(a[0], w.kc[s][0], w.kc[s][1]);
      a[1] = rot(a[1], w.kc[s][2], w.kc[s][3]);
      a[2] = rot(a[2], w.kc[s][4], w.kc[s][5]);
      a[3] = rot(a[3], w.kc[s][6], w.kc[s][7]);
    }
    if (s & 1) mma(sb, a, bq[s][0], bq[s][1]);
    else mma(sa, a, bq[s][0], bq[s][1]);
  }
  const bool r0 = rows & 1u, r1 = rows & 2u;
  const float s00 = (r0 && c0ok) ? sa[0] + sb[0] : -INFINITY;
  const float s01 = (r0 && c1ok) ? sa[1] + sb[1] : -INFINITY;
  const float s10 = (r1 && c0ok) ? sa[2] + sb[2] : -INFINITY;
  const float s11 = (r1 && c1ok) ? sa[3] + sb[3] : -INFINITY;
  const float c0 = fmaxf(s00, s10), c1 = fmaxf(s01, s11);
  if (__any_sync(0xffffffffu, c0 > w.mrun[0] + 8.f || c1 > w.mrun[1] + 8.f)) {
    const float mn0 = fmaxf(w.mrun[0], gmax(c0));
    const float mn1 = fmaxf(w.mrun[1], gmax(c1));
    const float a0 = (w.mrun[0] == mn0) ? 1.f : e2(w.mrun[0] - mn0);
    const float a1 = (w.mrun[1] == mn1) ? 1.f : e2(w.mrun[1] - mn1);
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
  const float m0 = w.mrun[0] == -INFINITY ? 0.f : w.mrun[0];
  const float m1 = w.mrun[1] == -INFINITY ? 0.f : w.mrun[1];
  const float p00 = e2(s00 - m0), p01 = e2(s01 - m1), p10 = e2(s10 - m0), p11 = e2(s11 - m1);
  w.lrun[0] += p00 + p10;
  w.lrun[1] += p01 + p11;
  const uint32_t b0 = movt(pk(p00, p01)), b1 = movt(pk(p10, p11));
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    uint32_t a[4];
    ldsm4t(base + 4096 + tv * 256 + ((((2 * mt + pv) ^ (lane & 7))) << 4), a);
    mma(w.o[mt], a, b0, b1);
  }
}

// Code unit g of a lane's row (RCB = G * CB bytes held in `cw`).
template <int CB, int NW>
__device__ __forceinline__ uint32_t code_unit(const uint32_t (&cw)[NW], int g) {
  if (CB == 1) return (cw[g >> 2] >> (8 * (g & 3))) & 0xffu;
  return (cw[g >> 1] >> (16 * (g & 1))) & 0xffffu;
}

template <int DSUB, int CB>
__global__ void __launch_bounds__(TT, 1) decode_tc_kernel(antkv_cache_desc c, TcArgs a) {
  constexpr int G = 128 / DSUB;
  // CB = 3: 12-bit indices packed two per three bytes (common.cuh code_get)
  constexpr int RCB = CB == 3 ? G * 3 / 2 : G * CB;   // code bytes of one token row (one side)
  constexpr int NW = RCB >= 4 ? RCB / 4 : 1;          // 32-bit words of them
  constexpr int TILEB = 32 * RCB;                     // code bytes of one 16-slot tile (K + V)
  constexpr int TPS = TCS / TILEB;            // tiles per code ring slot
  static_assert(TPS >= 1, "code tile larger than a ring slot");
  // d_sub = 4 with byte codes (m <= 256): an 8-byte centroid costs a whole
  // L1 wavefront when gathered from global memory, so the codebook is
  // replicated 16x in shared memory (stage slot 1: [side][code][copy][8 B],
  // copy = lane & 15 puts every lane of a half-warp on its own bank pair) and
  // each tile is rebuilt synchronously into stage slot 0 (LDS.64 pairs ->
  // STS.128); pool tiles then go through slot 0 before the loop
  constexpr bool SCB = DSUB == 4 && CB == 1;
  static_assert(!SCB || 2 * 256 * 16 * 8 <= TW * TSTAGE, "replicated codebook exceeds stage slot 1");
  extern __shared__ __align__(128) unsigned char smraw[];
  TcSmem &sm = *reinterpret_cast<TcSmem *>(smraw);
  const int b = blockIdx.z, h = blockIdx.y, split = blockIdx.x;
  const int S = a.splits, GQ = a.gq, F = 8 / GQ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t bh = (int64_t)b * c.Hkv + h;

  if (threadIdx.x == 0) {
    for (int ww = 0; ww < TW; ++ww) {
      for (int s = 0; s < TNCS; ++s) mb_init(&sm.cfull[ww][s], 1);
      mb_init(&sm.pfull[ww], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  const int n = c.seq_len[b];
  const int pool_high = c.hstate[bh * ANTKV_HSTATE_WORDS + ANTKV_HS_POOL_HIGH];
  const int64_t pos0 = c.positions[(int64_t)b * c.capacity];
  const int64_t qp = a.qpos[b];

  // ---- work split: contiguous tile ranges, each warp a multiple of F tiles
  const int ntiles = (n + 15) >> 4;
  const int per_cta0 = (ntiles + S - 1) / S;
  const int Tw = ((per_cta0 + TW - 1) / TW + F - 1) / F * F;
  const int T0 = split * Tw * TW;
  const int wt0 = T0 + warp * Tw;
  const int nt = max(0, min(Tw, ntiles - wt0));
  const int nslots = (nt + TPS - 1) / TPS;
  const uint8_t *codes = c.codes + bh * (int64_t)c.capacity / 16 * TILEB;   // per-head code stream
  auto issue_code = [&](int k) {   // ring slot k % TNCS <- tiles wt0 + k TPS ..
    const int cnt = min(TPS, nt - k * TPS);
    unsigned long long *bar = &sm.cfull[warp][k % TNCS];
    mb_expect_tx(bar, cnt * TILEB);
    bulk_g2s(&sm.code[warp][k % TNCS][0], codes + (int64_t)(wt0 + k * TPS) * TILEB, cnt * TILEB, bar);
  };
  if (lane == 0)
    for (int k = 0; k < min(TNCS, nslots); ++k) issue_code(k);

  // ---- query frames, cooperatively from integer-reduced angles (in the
  // stage area, before any tile lands there): frame f < TW F is warp f / F's
  // phase f % F; frame TW F is the absolute frame p_q of the pool rows
  const FastTables *tab = reinterpret_cast<const FastTables *>(c.fast_tables);
  float2 *ang = reinterpret_cast<float2 *>(&sm.stage[0][0][0]);
  float2 *qf = ang + (TW * 8 + 1) * 64;
  {
    const int nf = TW * F + 1;
    for (int e = threadIdx.x; e < nf * 64; e += TT) {
      const int f = e >> 6, p = e & 63;
      const int64_t delta = f < TW * F ? qp - (pos0 + 16 * (int64_t)(T0 + (f / F) * Tw + (f % F))) : qp;
      float cs, sn;
      turns_cs(delta, tab->turns[p], cs, sn);
      ang[f * 64 + lane_pair_pos(p)] = make_float2(cs, sn);
    }
    const float sc = rsqrtf(128.f) * 1.4426950408889634f;   // 1/sqrt(d) * log2(e)
    const int64_t qrow = (int64_t)b * c.Hq + (int64_t)h * GQ;
    for (int e = threadIdx.x; e < GQ * 64; e += TT)
      qf[(e >> 6) * 64 + lane_pair_pos(e & 63)] =
          make_float2(load_elem(a.q, qrow * 128 + 2 * e, a.qdtype) * sc,
                      load_elem(a.q, qrow * 128 + 2 * e + 1, a.qdtype) * sc);
    if (threadIdx.x < 64) {
      float cs, sn;
      turns_cs(-16 * (int64_t)F, tab->turns[threadIdx.x], cs, sn);
      sm.step[lane_pair_pos(threadIdx.x)] = make_float2(cs, sn);
    }
  }
  __syncthreads();
  Lane w;
  uint32_t bqa[8][2];
  const int hh = g % GQ, phase_g = g / GQ;
  {
    const int fr = warp * F + phase_g;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const float4 xq = *reinterpret_cast<const float4 *>(&qf[hh * 64 + (s * 4 + t) * 2]);
      const float4 cf = *reinterpret_cast<const float4 *>(&ang[fr * 64 + (s * 4 + t) * 2]);
      const float4 ca = *reinterpret_cast<const float4 *>(&ang[TW * F * 64 + (s * 4 + t) * 2]);
      w.fx[s] = make_float2(xq.x * cf.x - xq.y * cf.y, xq.z * cf.z - xq.w * cf.w);
      w.fy[s] = make_float2(xq.x * cf.y + xq.y * cf.x, xq.z * cf.w + xq.w * cf.z);
      w.bq[s][0] = pk(w.fx[s].x, w.fy[s].x);
      w.bq[s][1] = pk(w.fx[s].y, w.fy[s].y);
      bqa[s][0] = g < GQ ? pk(xq.x * ca.x - xq.y * ca.y, xq.x * ca.y + xq.y * ca.x) : 0u;
      bqa[s][1] = g < GQ ? pk(xq.z * ca.z - xq.w * ca.w, xq.z * ca.w + xq.w * ca.z) : 0u;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint4 k = __ldg(&tab->kc[s][u][t][g]);
        w.kc[s][4 * u] = k.x;
        w.kc[s][4 * u + 1] = k.y;
        w.kc[s][4 * u + 2] = k.z;
        w.kc[s][4 * u + 3] = k.w;
      }
    }
  }
  w.mrun[0] = w.mrun[1] = -INFINITY;
  w.lrun[0] = w.lrun[1] = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) w.o[i][e] = 0.f;
  if (SCB) {
    uint2 *cbs = reinterpret_cast<uint2 *>(&sm.stage[1][0][0]);
    const uint2 *src = reinterpret_cast<const uint2 *>(c.codebook_f16g) + (int64_t)h * 2 * c.m;
    for (int e = threadIdx.x; e < 2 * 256 * 16; e += TT) {
      const int side = e >> 12, code = (e >> 4) & 255;
      cbs[e] = code < c.m ? src[side * c.m + code] : make_uint2(0u, 0u);
    }
  }
  __syncthreads();   // frames read: the stage area becomes the tile rings
  if (lane == 0) fence_async();

  // ---- gathers: lane = (side kv = lane / 16, token row r = lane % 16)
  const int kv = lane >> 4, r = lane & 15;
  const uint8_t *cbase = reinterpret_cast<const uint8_t *>(c.codebook_f16g) +
                         ((int64_t)(h * 2 + kv) * c.m) * DSUB * 2;
  const uint32_t *qmg = c.qmask + bh * (c.capacity / 32);
  const uint32_t mmax = static_cast<uint32_t>(c.m - 1);
  auto gather = [&](int j, uint32_t &qword) {
    if (j < nt) {
      const int ks = j / TPS, slot = ks % TNCS;
      mb_wait(&sm.cfull[warp][slot], (ks / TNCS) & 1);
      if (SCB) {
        const int jc = lane & 15, rsel = lane >> 4;
        const uint8_t *cpt = &sm.code[warp][slot][(j % TPS) * TILEB];
        const uint32_t sb = su32(&sm.stage[0][warp][0]);
        const uint32_t cbs = su32(&sm.stage[1][0][0]) + jc * 8;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int kvv = i >> 3, rr = (2 * i + rsel) & 15;
          const uint32_t u = *reinterpret_cast<const uint16_t *>(cpt + kvv * 16 * RCB + rr * RCB + 2 * jc);
          const uint32_t c0 = min(u & 0xffu, mmax), c1 = min(u >> 8, mmax);
          uint32_t x0, x1, x2, x3;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x0), "=r"(x1) : "r"(cbs + ((kvv * 256 + c0) << 7)));
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x2), "=r"(x3) : "r"(cbs + ((kvv * 256 + c1) << 7)));
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sb + kvv * 4096 + rr * 256 + ((jc ^ (rr & 7)) << 4)),
                       "r"(x0), "r"(x1), "r"(x2), "r"(x3) : "memory");
        }
      } else if (DSUB >= 16) {
        // two token rows per instruction, lanes of one centroid adjacent: the
        // 32 chunks of an instruction touch 2 G cache lines (L1 / L2 gathers
        // cost one wavefront per line, not per lane)
        constexpr int CPC = DSUB >= 8 ? DSUB / 8 : 1;   // 16-byte chunks per centroid
        const int jc = lane & 15, rsel = lane >> 4, gq = jc / CPC, within = jc % CPC;
        const uint8_t *cpt = &sm.code[warp][slot][(j % TPS) * TILEB];
        const uint32_t sb = su32(&sm.stage[j % TNST][warp][0]);
        if (CB == 3) {   // lane = row (K rows 0-15, V rows 16-31): unpack it once for the 16 loads below
          static_assert(CB != 3 || DSUB < 16 || G <= 8, "unpack scratch holds 8 groups per row");
          __syncwarp();
#pragma unroll
          for (int gg = 0; gg < G; gg += 2) {
            const uint8_t *p3 = cpt + lane * RCB + 3 * (gg >> 1);
            const uint32_t b0 = p3[0], b1 = p3[1], b2 = p3[2];
            sm.cunp[warp][lane * G + gg] = static_cast<uint16_t>(b0 | ((b1 & 0xfu) << 8));
            sm.cunp[warp][lane * G + gg + 1] = static_cast<uint16_t>((b1 >> 4) | (b2 << 4));
          }
          __syncwarp();
        }
        const uint8_t *cb0 = reinterpret_cast<const uint8_t *>(c.codebook_f16g) +
                             (int64_t)h * 2 * c.m * DSUB * 2 + within * 16;
        const int64_t side = (int64_t)c.m * DSUB * 2;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int kvv = i >> 3, rr = (2 * i + rsel) & 15;
          const uint32_t code =
              min(CB == 3 ? (uint32_t)sm.cunp[warp][(kvv * 16 + rr) * G + gq] : code_get(cpt, (int64_t)(kvv * 16 + rr) * G + gq, CB),
                  mmax);
          // codebooks of m > 256 (2-byte / packed indices) are L2-resident and
          // hardly hit in L1: bypassing it measured 102 -> 92.5 us (d32m4096);
          // m <= 256 codebooks live in L1 (.cg: 94 -> 323 us at d8m256)
          if (CB != 1) cpa16_cg(sb + kvv * 4096 + rr * 256 + ((jc ^ (rr & 7)) << 4), cb0 + kvv * side + (int64_t)code * (DSUB * 2));
          else cpa16(sb + kvv * 4096 + rr * 256 + ((jc ^ (rr & 7)) << 4), cb0 + kvv * side + (int64_t)code * (DSUB * 2));
        }
      } else {
      const uint8_t *cp = &sm.code[warp][slot][(j % TPS) * TILEB + kv * 16 * RCB + r * RCB];
      uint32_t cw[NW];
      if (CB == 3) {
      } else if (RCB >= 16) {
#pragma unroll
        for (int i = 0; i < NW; i += 4) {
          const uint4 v = *reinterpret_cast<const uint4 *>(cp + 4 * i);
          cw[i] = v.x; cw[i + 1] = v.y; cw[i + 2] = v.z; cw[i + 3] = v.w;
        }
      } else if (RCB == 8) {
        const uint2 v = *reinterpret_cast<const uint2 *>(cp);
        cw[0] = v.x; cw[NW - 1] = v.y;
      } else if (RCB == 4) {
        cw[0] = *reinterpret_cast<const uint32_t *>(cp);
      } else {
        cw[0] = *reinterpret_cast<const uint16_t *>(cp);
      }
      const uint32_t dst = su32(&sm.stage[j % TNST][warp][0]) + kv * 4096 + r * 256;
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const uint32_t code = min(CB == 3 ? code_get(cp, gg, 3) : code_unit<CB, NW>(cw, gg), mmax);
        const uint8_t *src = cbase + (int64_t)code * (DSUB * 2);
        if (DSUB >= 8) {
#pragma unroll
          for (int k = 0; k < DSUB / 8; ++k) {
            const int c16 = (gg * DSUB) / 8 + k;
            if (CB != 1) cpa16_cg(dst + ((c16 ^ (r & 7)) << 4), src + 16 * k);
            else cpa16(dst + ((c16 ^ (r & 7)) << 4), src + 16 * k);
          }
        } else {
          const int c16 = (gg * DSUB) >> 3, half = ((gg * DSUB) >> 2) & 1;
          cpa8(dst + ((c16 ^ (r & 7)) << 4) + 8 * half, src);
        }
      }
      }
      const int gt = wt0 + j;
      qword = (__ldg(qmg + (gt >> 1)) >> (16 * (gt & 1))) & 0xffffu;
      if (j % TPS == TPS - 1 || j == nt - 1) {   // the slot's codes are read: refill it
        __syncwarp();
        if (lane == 0 && ks + TNCS < nslots) {
          fence_async();
          issue_code(ks + TNCS);
        }
      }
    }
    cpa_commit();
  };
  static_assert(TNST == 3, "the qmask words below rotate through three registers");
  uint32_t q0 = 0, q1 = 0, q2 = 0;
  if (SCB) {
    for (int k = 0; k < 2 && k < nt; ++k) {
      const int gt = wt0 + k;
      (k ? q1 : q0) = (__ldg(qmg + (gt >> 1)) >> (16 * (gt & 1))) & 0xffffu;
    }
  } else {
    gather(0, q0);
    gather(1, q1);
  }

  // ---- pool tiles (anchors + window) through the warp's third ring slot
  {
    const int ptiles = (pool_high + 15) >> 4;
    const int pper = (ptiles + S - 1) / S;
    const int pt0 = min(ptiles, split * pper), pt1 = min(ptiles, pt0 + pper);
    const uint8_t *pool_g = reinterpret_cast<const uint8_t *>(c.pool_f16) + bh * (int64_t)c.pool_capacity * 512;
    const int8_t *kinds = c.pool_kind + bh * c.pool_capacity;
    const int32_t *ptok = c.pool_tok + bh * c.pool_capacity;
    uint8_t *pbuf = &sm.stage[SCB ? 0 : TNST - 1][warp][0];
    int rnd = 0;
    for (int tile = pt0 + warp; tile < pt1; tile += TW, ++rnd) {
      if (lane == 0) {
        mb_expect_tx(&sm.pfull[warp], TSTAGE);
        bulk_g2s(pbuf, pool_g + (int64_t)tile * TSTAGE, TSTAGE, &sm.pfull[warp]);
      }
      const int s0 = tile * 16 + g, s1 = s0 + 8;
      const bool v0 = kinds[s0] != ANTKV_KIND_FREE && ptok[s0] >= 0 && ptok[s0] < n;
      const bool v1 = kinds[s1] != ANTKV_KIND_FREE && ptok[s1] >= 0 && ptok[s1] < n;
      mb_wait(&sm.pfull[warp], rnd & 1);
      tile_attend<false>(w, su32(pbuf), bqa, (v0 ? 1u : 0u) | (v1 ? 2u : 0u), 2 * t < GQ, 2 * t + 1 < GQ);
      __syncwarp();
      if (lane == 0) fence_async();   // generic reads of the slot before the next bulk write
    }
  }

  // ---- code tiles
  const int ph0 = (2 * t) / GQ, ph1 = (2 * t + 1) / GQ;
  for (int i = 0; i < nt; ++i) {
    const int ph = i % F;
    const uint32_t rows = ((q0 >> g) & 1u) | (((q0 >> (g + 8)) & 1u) << 1);
    if (SCB) {   // synchronous rebuild into slot 0 (q words prefetched two tiles ahead)
      if (i + 2 < nt) {
        const int gt = wt0 + i + 2;
        q2 = (__ldg(qmg + (gt >> 1)) >> (16 * (gt & 1))) & 0xffffu;
      }
      uint32_t unused;
      gather(i, unused);
      __syncwarp();
      tile_attend<true>(w, su32(&sm.stage[0][warp][0]), w.bq, rows, ph0 == ph, ph1 == ph);
    } else {
      gather(i + 2, q2);
      cpa_wait<TNST - 1>();
      __syncwarp();
      tile_attend<true>(w, su32(&sm.stage[i % TNST][warp][0]), w.bq, rows, ph0 == ph, ph1 == ph);
    }
    if (ph == F - 1) {   // next stage: frames advance by R(-16 F omega)
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const float4 st = *reinterpret_cast<const float4 *>(&sm.step[(s * 4 + t) * 2]);
        const float2 sc = make_float2(st.x, st.z), ss = make_float2(st.y, st.w);
        const float2 x = w.fx[s], y = w.fy[s];
        w.fx[s] = __ffma2_rn(make_float2(-y.x, -y.y), ss, __fmul2_rn(x, sc));
        w.fy[s] = __ffma2_rn(y, sc, __fmul2_rn(x, ss));
        w.bq[s][0] = pk(w.fx[s].x, w.fy[s].x);
        w.bq[s][1] = pk(w.fx[s].y, w.fy[s].y);
      }
    }
    __syncwarp();
    q0 = q1;
    q1 = q2;
  }
  cpa_wait<0>();

  // ---- merge 8 warps x 8 columns -> one partial per query head (natural log)
  __syncthreads();
  float *mo = reinterpret_cast<float *>(&sm.stage[0][0][0]);   // [TW][8 cols][128]
  float *mm = mo + TW * 8 * 128;                                  // [TW][8]
  float *ml = mm + TW * 8;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    mo[(warp * 8 + 2 * t) * 128 + 16 * mt + g] = w.o[mt][0];
    mo[(warp * 8 + 2 * t + 1) * 128 + 16 * mt + g] = w.o[mt][1];
    mo[(warp * 8 + 2 * t) * 128 + 16 * mt + g + 8] = w.o[mt][2];
    mo[(warp * 8 + 2 * t + 1) * 128 + 16 * mt + g + 8] = w.o[mt][3];
  }
  const float ls0 = gsum(w.lrun[0]), ls1 = gsum(w.lrun[1]);
  if (g == 0) {
    mm[warp * 8 + 2 * t] = w.mrun[0];
    mm[warp * 8 + 2 * t + 1] = w.mrun[1];
    ml[warp * 8 + 2 * t] = ls0;
    ml[warp * 8 + 2 * t + 1] = ls1;
  }
  __syncthreads();
  const int nsrc = TW * F;   // sources of head x: (warp, column x + GQ f)
  if (threadIdx.x < GQ) {
    const int x = threadIdx.x;
    float M = -INFINITY;
    for (int e = 0; e < nsrc; ++e) M = fmaxf(M, mm[(e / F) * 8 + x + GQ * (e % F)]);
    float L = 0.f;
    for (int e = 0; e < nsrc; ++e) {
      const int src = (e / F) * 8 + x + GQ * (e % F);
      const float f = mm[src] == -INFINITY ? 0.f : e2(mm[src] - M);
      sm.mw[x][e] = f;
      L += f * ml[src];
    }
    const int64_t row = ((int64_t)split * c.B + b) * c.Hq + (int64_t)h * GQ + x;
    a.ws_m[row] = M * 0.6931471805599453f;
    a.ws_l[row] = L;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < GQ * 128; i += TT) {
    const int x = i >> 7, dim = i & 127;
    float O = 0.f;
    for (int e = 0; e < nsrc; ++e)
      O = fmaf(sm.mw[x][e], mo[((e / F) * 8 + x + GQ * (e % F)) * 128 + dim], O);
    a.ws_o[(((int64_t)split * c.B + b) * c.Hq + (int64_t)h * GQ + x) * 128 + dim] = O;
  }

  // ---- the last CTA of (b, h) (atomic ticket) merges the splits' partials
  // barrier + one thread's acq_rel fences around the ticket (see decode_fast.cu)
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    sm.ticket = atomicAdd(&a.cnt[bh], 1);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  if (sm.ticket != S - 1) return;
  if (warp < GQ) {   // warp x: query head h GQ + x, lane: 4 dims; loads of 16 splits in flight
    const int64_t rows = (int64_t)c.B * c.Hq;
    const int64_t row = (int64_t)b * c.Hq + (int64_t)h * GQ + warp;
    const int d4 = 4 * lane;
    float M = -INFINITY, L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int CH = 16;
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
    *reinterpret_cast<float4 *>(a.out + row * 128 + d4) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (lane == 0 && a.lse) a.lse[row] = M + logf(L);
  }
  if (threadIdx.x == 0) a.cnt[bh] = 0;
}

template <int DSUB, int CB>
int launch_tc(const antkv_cache_desc &c, const TcArgs &a, cudaStream_t st) {
  const size_t smem = sizeof(TcSmem);
  static bool attr[64] = {};   // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaFuncSetAttribute(decode_tc_kernel<DSUB, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  decode_tc_kernel<DSUB, CB><<<dim3(a.splits, c.Hkv, c.B), TT, smem, st>>>(c, a);
  ANTKV_LAUNCH_CHECK("decode_tc_kernel");
  return ANTKV_OK;
}

// fp16 codebook copy [Hkv][2][m][d_sub] + (block Hkv * 2) the RoPE tables.
__global__ void cache_prepare_tc_kernel(antkv_cache_desc c) {
  if (blockIdx.x == gridDim.x - 1) {
    fill_fast_tables(reinterpret_cast<FastTables *>(c.fast_tables), c.theta_base);
    return;
  }
  const int h = blockIdx.x / 2, kv = blockIdx.x % 2;
  const float *cb = (kv ? c.codebook_v : c.codebook_k) + (int64_t)h * c.m * c.d_sub;
  __half *dst = reinterpret_cast<__half *>(c.codebook_f16g) + (int64_t)(h * 2 + kv) * c.m * c.d_sub;
  for (int64_t i = threadIdx.x; i < (int64_t)c.m * c.d_sub; i += blockDim.x) dst[i] = __float2half_rn(cb[i]);
}

}  // namespace

int decode_tc_supported(const antkv_cache_desc &c) {
  if (c.d != 128 || c.Hq % c.Hkv != 0) return 0;
  const int gq = c.Hq / c.Hkv;
  if (gq != 1 && gq != 2 && gq != 4 && gq != 8) return 0;
  if (c.d_sub != 4 && c.d_sub != 8 && c.d_sub != 16 && c.d_sub != 32 && c.d_sub != 64) return 0;
  if (code_stream_bytes(128 / c.d_sub, c.code_bytes) > 32) return 0;
  return c.codebook_f16g != nullptr && c.pool_f16 != nullptr && c.fast_tables != nullptr &&
         c.capacity % 32 == 0 && c.pool_capacity % 16 == 0 && c.m >= 1 && c.m <= 65536;
}

int decode_mha_supported(const antkv_cache_desc &c);   // decode_mha.cu
int decode_mha_plan(const antkv_cache_desc &c, int requested);
int decode_mha_launch(const antkv_cache_desc &c, const void *q, int qdtype, const int64_t *qpos, float *ws_o,
                      float *ws_m, float *ws_l, float *out, float *lse, int *cnt, int splits, cudaStream_t st);

int decode_tc_plan(const antkv_cache_desc &c, int requested) {
  if (decode_mha_supported(c)) return decode_mha_plan(c, requested);   // MHA d4m256: CUDA-core kernel
  if (requested > 0) return requested;
  const int bh = c.B * c.Hkv;
  return bh >= 148 ? 1 : 148 / bh;
}

int decode_tc_launch(const antkv_cache_desc &c, const void *q, int qdtype, const int64_t *qpos, float *ws_o,
                     float *ws_m, float *ws_l, float *out, float *lse, int *cnt, int splits, cudaStream_t st) {
  if (decode_mha_supported(c))
    return decode_mha_launch(c, q, qdtype, qpos, ws_o, ws_m, ws_l, out, lse, cnt, splits, st);
  TcArgs a;
  a.out = out;
  a.lse = lse;
  a.cnt = cnt;
  a.q = q;
  a.qdtype = qdtype;
  a.qpos = qpos;
  a.ws_o = ws_o;
  a.ws_m = ws_m;
  a.ws_l = ws_l;
  a.splits = splits;
  a.gq = c.Hq / c.Hkv;
  const int key = c.d_sub * 4 + c.code_bytes;
  switch (key) {
    case 4 * 4 + 1: return launch_tc<4, 1>(c, a, st);
    case 8 * 4 + 1: return launch_tc<8, 1>(c, a, st);
    case 8 * 4 + 2: return launch_tc<8, 2>(c, a, st);
    case 16 * 4 + 1: return launch_tc<16, 1>(c, a, st);
    case 16 * 4 + 2: return launch_tc<16, 2>(c, a, st);
    case 32 * 4 + 1: return launch_tc<32, 1>(c, a, st);
    case 32 * 4 + 2: return launch_tc<32, 2>(c, a, st);
    case 64 * 4 + 1: return launch_tc<64, 1>(c, a, st);
    case 64 * 4 + 2: return launch_tc<64, 2>(c, a, st);
    case 8 * 4 + 3: return launch_tc<8, 3>(c, a, st);
    case 16 * 4 + 3: return launch_tc<16, 3>(c, a, st);
    case 32 * 4 + 3: return launch_tc<32, 3>(c, a, st);
    case 64 * 4 + 3: return launch_tc<64, 3>(c, a, st);
    default:
      set_error("staged tensor-core decode: d_sub=%d code_bytes=%d unsupported", c.d_sub, c.code_bytes);
      return ANTKV_EUNSUPPORTED;
  }
}

}  // namespace antkv

using namespace antkv;

extern "C" int antkv_cache_prepare_tc(const antkv_cache_desc *c, void *stream) {
  ANTKV_REQUIRE(c != nullptr, "null cache descriptor");
  previous_cache_on_stream(as_stream(stream), c->codes);   // this stream now touched c
  ANTKV_REQUIRE(c->d == 128 && c->codebook_f16g && c->fast_tables && c->pool_f16,
                "staged tensor-core path needs d=128 and its fp16 buffers");
  ANTKV_REQUIRE(c->pool_capacity % 16 == 0, "pool_capacity must be a multiple of 16");
  cudaStream_t st = as_stream(stream);
  cache_prepare_tc_kernel<<<c->Hkv * 2 + 1, 256, 0, st>>>(*c);
  ANTKV_LAUNCH_CHECK("cache_prepare_tc_kernel");
  cache_pool_f16_kernel<<<dim3(c->pool_capacity, c->B * c->Hkv), 64, 0, st>>>(*c);
  ANTKV_LAUNCH_CHECK("cache_pool_f16_kernel");
  return ANTKV_OK;
}
