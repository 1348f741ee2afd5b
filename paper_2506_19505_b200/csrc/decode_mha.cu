// sm_100a decode attention for multi-head attention (one query head per KV
// head, e.g. BASELINE config #4's LLaMA-2-7B shapes) with d = 128 and 4-dim
// sub-vectors of at most 256 centroids (the 2-bit d4m256 code).  Reference
// semantics: cache.py:168-178 (RoPE after reconstruction, softmax over the
// whole cache, A.V); the cache update runs around this launch
// (antkv_cache_append / antkv_cache_evict), as for the staged kernel.
//
// With one query per KV head nothing is shared between the MMA columns, so
// this path uses the CUDA cores and spends shared memory only on gathers:
//   * lane g of a warp owns sub-vector group g (dims 4g..4g+3 = RoPE pairs
//     2g, 2g+1) of every token the warp visits; the fp16 codebook sits in
//     shared memory replicated 16x ([side][code][copy][4 dims], copy =
//     lane & 15), so a warp's 32 gathers of one token are one conflict-free
//     LDS.64 (256 B, 2 wavefronts) -- against ~14 wavefronts per token-head
//     for rebuilding tiles for the tensor cores (decode_tc.cu);
//   * the key side needs no rotation: score_j = (R((p_q - p_j) w) q) . k_j
//     (pre-RoPE codes), so each lane rotates only its 2 query pairs, by
//     R(-w) per token (fp32, the Chebyshev recurrence x_{i+1} = 2 cos(w)
//     x_i - x_{i-1}: one FMA per component), re-seeded exactly from
//     integer-reduced angles at every 32-token chunk;
//   * a chunk's 32 x 32 partial dot products are summed by a butterfly
//     transpose-reduce (31 shuffles), leaving token i's score in lane i; the
//     online softmax runs there and P_i is broadcast back for O += P_i V_i;
//   * code tiles stream per warp through a 2-slot ring (cp.async.bulk), 2
//     CTAs of 8 warps per SM; anchor / window rows (pool_f16, K rotated at
//     its own position) are read from global memory against the query in
//     the absolute frame; splits of a (sequence, head) merge in the last CTA
//     (atomic ticket), as in decode_tc.cu.
#include "common.cuh"

namespace antkv {
namespace {

constexpr int HW = 8;                  // warps per CTA
constexpr int HT = 32 * HW;
constexpr int HNS = 2;                 // code ring slots per warp
constexpr int HTILE = 1024;            // d4m256 code tile: [K 16 x 32 | V 16 x 32] bytes
constexpr int HSLOT = 2 * HTILE;       // one 32-token chunk

struct MhaSmem {
  uint2 cbk[256][16];                  // K: [code][copy] 4 fp16 dims (pairs' x | y halves)
  float4 cbv[256][8];                  // V: [code][copy] 4 fp32 dims (no conversion on the FMA pipe)
  uint8_t ring[HW][HNS][HSLOT];
  float mo[HW][128];
  float mm[HW], ml[HW];
  unsigned long long full[HW][HNS];
  int ticket;
};

struct MhaArgs {
  const void *q;          // [B][Hq][128]
  int qdtype;
  const int64_t *qpos;    // [B]
  float *ws_o, *ws_m, *ws_l;
  float *out, *lse;
  int *cnt;
  int splits;
};

__device__ __forceinline__ uint32_t msu32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float mex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float4 h4(uint2 v) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&v.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&v.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float2 h2f(uint32_t v) { return __half22float2(*reinterpret_cast<const __half2 *>(&v)); }

// Butterfly transpose-reduce: on return v[0] of lane l holds the sum over
// the warp's lanes of their v[l].
__device__ __forceinline__ float transpose_sum(float (&v)[32], int lane) {
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool up = lane & k;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const float send = up ? v[i] : v[i + k];
      const float keep = up ? v[i + k] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0];
}

struct MhaLane {
  float2 o01, o23;  // O of dims 4g..4g+3
  float m, l;       // running max (log2 units, warp-uniform), this lane's share of the normaliser
};

// Online softmax over one chunk (lane i: score s of token i, -inf when not
// valid), then O += sum_i P_i V_i with V rows from `vrow(i)`.
template <class VRow>
__device__ __forceinline__ void chunk_softmax_pv(MhaLane &w, float s, int lane, VRow vrow) {
  float cm = s;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
  // (no early exit: cm is warp-uniform but a branch on it would make the
  // shuffles below collective; an all-masked chunk adds zeros)
  if (cm > w.m) {
    const float al = w.m == -INFINITY ? 0.f : mex2(w.m - cm);
    w.l *= al;
    w.o01 = __fmul2_rn(w.o01, make_float2(al, al));
    w.o23 = __fmul2_rn(w.o23, make_float2(al, al));
    w.m = cm;
  }
  const float p = s == -INFINITY ? 0.f : mex2(s - w.m);
  w.l += p;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    const float pi = __shfl_sync(0xffffffffu, p, i);
    const float4 v = vrow(i);
    w.o01 = __ffma2_rn(make_float2(pi, pi), make_float2(v.x, v.y), w.o01);
    w.o23 = __ffma2_rn(make_float2(pi, pi), make_float2(v.z, v.w), w.o23);
  }
}

__global__ void __launch_bounds__(HT, 2) decode_mha_kernel(antkv_cache_desc c, MhaArgs a) {
  extern __shared__ __align__(128) unsigned char mraw[];
  MhaSmem &sm = *reinterpret_cast<MhaSmem *>(mraw);
  const int b = blockIdx.z, h = blockIdx.y, split = blockIdx.x, S = a.splits;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bh = (int64_t)b * c.Hkv + h;

  if (threadIdx.x == 0) {
    for (int ww = 0; ww < HW; ++ww)
      for (int s = 0; s < HNS; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(msu32(&sm.full[ww][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the codebooks: K fp16 ([Hkv][K][m][4]) replicated 16x with its halves as
  // (d0, d2), (d1, d3) = the x and y components of pairs 2g, 2g+1; V fp32
  // (the cache's own codebook) replicated 8x (LDS.128 phases of 8 lanes)
  {
    const uint2 *src = reinterpret_cast<const uint2 *>(c.codebook_f16g) + (int64_t)h * 2 * c.m;
    for (int e = threadIdx.x; e < 256 * 16; e += HT) {
      const int code = e >> 4;
      const uint2 v = code < c.m ? src[code] : make_uint2(0u, 0u);
      (&sm.cbk[0][0])[e] = make_uint2(__byte_perm(v.x, v.y, 0x5410), __byte_perm(v.x, v.y, 0x7632));
    }
    const float4 *srcv = reinterpret_cast<const float4 *>(c.codebook_v + (int64_t)h * c.m * 4);
    for (int e = threadIdx.x; e < 256 * 8; e += HT) {
      const int code = e >> 3;
      (&sm.cbv[0][0])[e] = code < c.m ? __ldg(srcv + code) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __syncthreads();

  const int n = c.seq_len[b];
  const int pool_high = c.hstate[bh * ANTKV_HSTATE_WORDS + ANTKV_HS_POOL_HIGH];
  const int64_t pos0 = c.positions[(int64_t)b * c.capacity];
  const int64_t qp = a.qpos[b];
  const FastTables *tab = reinterpret_cast<const FastTables *>(c.fast_tables);

  // ---- work split: 32-token chunks, contiguous per CTA and per warp
  const int nch = (n + 31) >> 5;
  const int per_cta = (nch + S - 1) / S;
  const int per_warp = (per_cta + HW - 1) / HW;
  const int c0 = min(nch, split * per_cta + warp * per_warp);
  const int c1 = min(nch, min(split * per_cta + per_cta, c0 + per_warp));
  const int nc = max(0, c1 - c0);
  const uint8_t *codes = c.codes + bh * (int64_t)c.capacity * 64;   // 64 code bytes per token (K + V)
  auto issue = [&](int k) {   // ring slot k % HNS <- chunk c0 + k (two 16-token tiles)
    unsigned long long *bar = &sm.full[warp][k % HNS];
    int ch = c0 + k;
    if ((ch + 1) * 32 > c.capacity) ch = 0;   // beyond capacity: masked dummy data
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(msu32(bar)), "r"(HSLOT) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            msu32(&sm.ring[warp][k % HNS][0])),
        "l"(codes + (int64_t)ch * HSLOT), "r"(HSLOT), "r"(msu32(bar))
        : "memory");
  };
  if (lane == 0)
    for (int k = 0; k < min(HNS, nc); ++k) issue(k);

  // ---- lane state: query pairs 2g, 2g+1 (scaled to log2 units), their
  // per-token step R(-w) and the absolute frame R(p_q w) q of the pool rows
  const float sc = rsqrtf(128.f) * 1.4426950408889634f;
  const int64_t qrow = (int64_t)b * c.Hq + h;
  float qx[2], qy[2], cw[2], sw[2], ax[2], ay[2];   // [u]: pair 2g + u
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int p = 2 * lane + u;
    qx[u] = load_elem(a.q, qrow * 128 + 2 * p, a.qdtype) * sc;
    qy[u] = load_elem(a.q, qrow * 128 + 2 * p + 1, a.qdtype) * sc;
    turns_cs(1, tab->turns[p], cw[u], sw[u]);
    float cs, sn;
    turns_cs(qp, tab->turns[p], cs, sn);
    ax[u] = qx[u] * cs - qy[u] * sn;
    ay[u] = qx[u] * sn + qy[u] * cs;
  }
  MhaLane w;
  w.m = -INFINITY;
  w.l = 0.f;
  w.o01 = w.o23 = make_float2(0.f, 0.f);
  const float2 C2 = make_float2(cw[0], cw[1]), S2 = make_float2(sw[0], sw[1]);
  const float2 NS2 = make_float2(-sw[0], -sw[1]);
  const float2 TC2 = make_float2(2.f * cw[0], 2.f * cw[1]);
  const uint32_t *qmg = c.qmask + bh * (c.capacity / 32);
  const int copy = lane & 15;

  // ---- code chunks
  for (int k = 0; k < nc; ++k) {
    const int ch = c0 + k, slot = k % HNS;
    const uint32_t qw = __ldg(qmg + ch);
    float2 FX, FY, PX, PY;   // R((p_q - p_j) w) q at token j (exact at the chunk's first), and at j - 1
    {
      float cs0, sn0, cs1, sn1;
      turns_cs(qp - (pos0 + (int64_t)ch * 32), tab->turns[2 * lane], cs0, sn0);
      turns_cs(qp - (pos0 + (int64_t)ch * 32), tab->turns[2 * lane + 1], cs1, sn1);
      FX = make_float2(qx[0] * cs0 - qy[0] * sn0, qx[1] * cs1 - qy[1] * sn1);
      FY = make_float2(qx[0] * sn0 + qy[0] * cs0, qx[1] * sn1 + qy[1] * cs1);
    }
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            msu32(&sm.full[warp][slot])),
        "r"((uint32_t)((k / HNS) & 1))
        : "memory");
    const uint8_t *tb = &sm.ring[warp][slot][0];
    float ps[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int kc = tb[(i >> 4) * HTILE + (i & 15) * 32 + lane];
      const uint2 kv = sm.cbk[kc][copy];   // (k0, k2), (k1, k3)
      const float2 d = __ffma2_rn(FY, h2f(kv.y), __fmul2_rn(FX, h2f(kv.x)));
      ps[i] = d.x + d.y;
      // next token, R(-w) on both pairs: a rotation by a fixed angle obeys
      // x_{i+1} = 2 cos(w) x_i - x_{i-1} per component (one FMA each after
      // the first step, which rotates exactly)
      if (i == 0) {
        const float2 nx = __ffma2_rn(S2, FY, __fmul2_rn(C2, FX));
        const float2 ny = __ffma2_rn(NS2, FX, __fmul2_rn(C2, FY));
        PX = FX; PY = FY; FX = nx; FY = ny;
      } else {
        const float2 nx = __ffma2_rn(TC2, FX, make_float2(-PX.x, -PX.y));
        const float2 ny = __ffma2_rn(TC2, FY, make_float2(-PY.x, -PY.y));
        PX = FX; PY = FY; FX = nx; FY = ny;
      }
    }
    float s = transpose_sum(ps, lane);
    if (!((qw >> lane) & 1u)) s = -INFINITY;
    chunk_softmax_pv(w, s, lane, [&](int i) {
      const int vc = tb[(i >> 4) * HTILE + 512 + (i & 15) * 32 + lane];
      return sm.cbv[vc][lane & 7];
    });
    __syncwarp();
    if (lane == 0 && k + HNS < nc) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + HNS);
    }
  }

  // ---- pool rows (anchors + window), 16-slot tiles split over CTAs and warps
  {
    const int ptiles = (pool_high + 15) >> 4;
    const int pper = (ptiles + S - 1) / S;
    const int pt0 = min(ptiles, split * pper), pt1 = min(ptiles, pt0 + pper);
    const __half *pf = reinterpret_cast<const __half *>(c.pool_f16) + bh * (int64_t)c.pool_capacity * 256;
    const int8_t *kinds = c.pool_kind + bh * c.pool_capacity;
    const int32_t *ptok = c.pool_tok + bh * c.pool_capacity;
    for (int tile = pt0 + warp; tile < pt1; tile += HW) {
      float ps[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int slot = tile * 16 + i;
        const float4 kv = h4(__ldg(reinterpret_cast<const uint2 *>(pf + pool_f16_offset(slot, 0, 4 * lane))));
        ps[i] = fmaf(ax[0], kv.x, fmaf(ay[0], kv.y, fmaf(ax[1], kv.z, ay[1] * kv.w)));
        ps[i + 16] = 0.f;
      }
      float s = transpose_sum(ps, lane);
      const int slot = tile * 16 + (lane & 15);
      const bool ok = lane < 16 && kinds[slot] != ANTKV_KIND_FREE && ptok[slot] >= 0 && ptok[slot] < n;
      if (!ok) s = -INFINITY;
      chunk_softmax_pv(w, s, lane, [&](int i) {
        const int sl = tile * 16 + (i & 15);
        return i < 16 ? h4(__ldg(reinterpret_cast<const uint2 *>(pf + pool_f16_offset(sl, 1, 4 * lane))))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      });
    }
  }

  // ---- merge the 8 warps -> one partial (natural log), then the splits
  float lsum = w.l;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  *reinterpret_cast<float4 *>(&sm.mo[warp][4 * lane]) = make_float4(w.o01.x, w.o01.y, w.o23.x, w.o23.y);
  if (lane == 0) {
    sm.mm[warp] = w.m;
    sm.ml[warp] = lsum;
  }
  __syncthreads();
  const int64_t rows = (int64_t)c.B * c.Hq;
  const int64_t row = (int64_t)b * c.Hq + h;
  if (threadIdx.x < 128) {
    float M = -INFINITY;
#pragma unroll
    for (int ww = 0; ww < HW; ++ww) M = fmaxf(M, sm.mm[ww]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int ww = 0; ww < HW; ++ww) {
      const float f = sm.mm[ww] == -INFINITY ? 0.f : mex2(sm.mm[ww] - M);
      L = fmaf(f, sm.ml[ww], L);
      O = fmaf(f, sm.mo[ww][threadIdx.x], O);
    }
    a.ws_o[((int64_t)split * rows + row) * 128 + threadIdx.x] = O;
    if (threadIdx.x == 0) {
      a.ws_m[split * rows + row] = M == -INFINITY ? -INFINITY : M * 0.6931471805599453f;
      a.ws_l[split * rows + row] = L;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    sm.ticket = atomicAdd(&a.cnt[bh], 1);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  if (sm.ticket != S - 1) return;
  if (warp == 0) {   // lane: 4 dims; the splits' partials 16 at a time
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
    if (lane == 0) a.cnt[bh] = 0;
  }
}

}  // namespace

int decode_mha_supported(const antkv_cache_desc &c) {
  static int off = -1;   // ANTKV_NO_MHA=1: the staged tensor-core kernel instead (A/B timing)
  if (off < 0) {
    const char *e = getenv("ANTKV_NO_MHA");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  return !off && c.d == 128 && c.Hq == c.Hkv && c.d_sub == 4 && c.code_bytes == 1 && c.m >= 1 && c.m <= 256 &&
         c.codebook_f16g != nullptr && c.pool_f16 != nullptr && c.fast_tables != nullptr &&
         c.capacity % 32 == 0 && c.pool_capacity % 16 == 0;
}

int decode_mha_plan(const antkv_cache_desc &c, int requested) {
  if (requested > 0) return requested;
  const int bh = c.B * c.Hkv;   // two CTAs per SM
  return bh >= 2 * 148 ? 1 : (2 * 148 + bh - 1) / bh;
}

int decode_mha_launch(const antkv_cache_desc &c, const void *q, int qdtype, const int64_t *qpos, float *ws_o,
                      float *ws_m, float *ws_l, float *out, float *lse, int *cnt, int splits, cudaStream_t st) {
  MhaArgs a;
  a.q = q;
  a.qdtype = qdtype;
  a.qpos = qpos;
  a.ws_o = ws_o;
  a.ws_m = ws_m;
  a.ws_l = ws_l;
  a.out = out;
  a.lse = lse;
  a.cnt = cnt;
  a.splits = splits;
  const size_t smem = sizeof(MhaSmem);
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaFuncSetAttribute(decode_mha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  decode_mha_kernel<<<dim3(splits, c.Hkv, c.B), HT, smem, st>>>(c, a);
  ANTKV_LAUNCH_CHECK("decode_mha_kernel");
  return ANTKV_OK;
}

}  // namespace antkv
