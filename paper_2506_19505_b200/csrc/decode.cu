// Decode attention over the quantised cache (cache.py:168-178):
//   out_h = softmax(RoPE(q_h, p_q) . RoPE(K_hat_j, p_j) / sqrt(d)) V_hat
// with K_hat/V_hat reconstructed from codes (quantised slots) or read from
// the bf16 full-precision pool (anchors + window), split-KV partials and a
// log-sum-exp combine.  This file holds the generic float32 kernel (any
// d <= 256, d_sub, m) and the combine; decode_fast.cu holds the sm_100a
// tensor-core kernel for the 1-bit d8m256 configuration.
#include "common.cuh"

namespace antkv {

constexpr int DG_T = 128;  // items per chunk == threads per CTA

__device__ __forceinline__ int load_code_unit(const antkv_cache_desc &c, int64_t off) {
  return static_cast<int>(code_get(c.codes, off, c.code_bytes));
}

int decode_fast_launch(const antkv_cache_desc &c, const void *q, int qdtype, const void *knew,
                       const void *vnew, int kvdtype, const int64_t *qpos, float *out, float *lse,
                       float *ws_o, float *ws_m, float *ws_l, int *cnt, int splits,
                       cudaStream_t st);
int decode_fast_supported(const antkv_cache_desc &c);
int decode_tc_supported(const antkv_cache_desc &c);
int decode_tc_plan(const antkv_cache_desc &c, int requested);
int decode_tc_launch(const antkv_cache_desc &c, const void *q, int qdtype, const int64_t *qpos, float *ws_o,
                     float *ws_m, float *ws_l, float *out, float *lse, int *cnt, int splits, cudaStream_t st);

// Decode kernel choice: the fused d8m256 kernel, the staged tensor-core
// kernel (decode_tc.cu, any other d = 128 code shape) or the generic one.
enum DecodeMode { kGeneric = 0, kFast = 1, kStaged = 2 };
void decode_fast_plan(const antkv_cache_desc &c, int requested, int &code_splits, int &pool_splits);

template <int GQ, bool CB_SMEM>
__global__ void __launch_bounds__(DG_T)
decode_generic_kernel(antkv_cache_desc c, const void *__restrict__ q, int dtype,
                      const int64_t *__restrict__ qpos, float *__restrict__ ws_o,
                      float *__restrict__ ws_m, float *__restrict__ ws_l) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int d = c.d, G = c.groups, dsub = c.d_sub;
  const int b = blockIdx.z, h = blockIdx.y, split = blockIdx.x, splits = gridDim.x;
  const int64_t bh = (int64_t)b * c.Hkv + h;
  double *sFreq = reinterpret_cast<double *>(smraw);                // [d/2]
  float2 *sRot = reinterpret_cast<float2 *>(sFreq + d / 2);         // [d/2][T]: R(t) of thread t
  float *sQ = reinterpret_cast<float *>(sRot + (d / 2) * DG_T);     // [GQ][d] q in the chunk frame
  float *sS = sQ + GQ * d;                                          // [GQ][T]
  float *sRed = sS + GQ * DG_T;                                     // [GQ][4] + [GQ][4]
  int *sSrc = reinterpret_cast<int *>(sRed + 8 * GQ);               // [T] source tag
  int *sVc = sSrc + DG_T;                                           // [T][G] V codes
  float *sCbK = reinterpret_cast<float *>(sVc + DG_T * G);          // [m][dsub]
  float *sCbV = sCbK + (CB_SMEM ? c.m * dsub : 0);
  const float *cbK = CB_SMEM ? sCbK : c.codebook_k + (int64_t)h * c.m * dsub;
  const float *cbV = CB_SMEM ? sCbV : c.codebook_v + (int64_t)h * c.m * dsub;

  for (int i = threadIdx.x; i < d / 2; i += DG_T) sFreq[i] = rope_freq(c.theta_base, i, d);
  __syncthreads();
  // residual rotations: thread t rotates a key t positions after the chunk
  // frame by R(t) (position-independent, so computed once per CTA)
  for (int p = 0; p < d / 2; ++p) {
    float cs, sn;
    rope_cs(static_cast<double>(threadIdx.x) * sFreq[p], cs, sn);
    sRot[p * DG_T + threadIdx.x] = make_float2(cs, sn);
  }
  if (CB_SMEM) {
    const float *gk = c.codebook_k + (int64_t)h * c.m * dsub;
    const float *gv = c.codebook_v + (int64_t)h * c.m * dsub;
    for (int i = threadIdx.x; i < c.m * dsub; i += DG_T) {
      sCbK[i] = gk[i];
      sCbV[i] = gv[i];
    }
  }
  __syncthreads();
  const float scale = rsqrtf(static_cast<float>(d));
  const int64_t pq = qpos[b];
  const int n = c.seq_len[b];
  const int pool_high = c.hstate[bh * ANTKV_HSTATE_WORDS + ANTKV_HS_POOL_HIGH];
  const int total = n + pool_high;
  const int per = (total + splits - 1) / splits;
  const int s0 = split * per, s1 = min(total, s0 + per);
  const int64_t hb = bh * c.capacity * 2 * G;   // code-unit offset of this head
  const uint32_t *qm = c.qmask + bh * (c.capacity / 32);
  const int64_t pool = bh * c.pool_capacity * 2 * d;   // element offset of this head's pool

  float m_run[GQ], l_run[GQ], acc[GQ][2];
#pragma unroll
  for (int hh = 0; hh < GQ; ++hh) {
    m_run[hh] = -INFINITY;
    l_run[hh] = 0.f;
    acc[hh][0] = acc[hh][1] = 0.f;
  }
  __syncthreads();
  for (int c0 = s0; c0 < s1; c0 += DG_T) {
    // ---- chunk frame: positions are relative to pc (the first code slot's
    // position); q is rotated by R(p_q - pc) and a key at pc + t by R(t)
    // from the table, so only keys off that grid (anchors / window rows in
    // the pool, non-contiguous caches) need their own angle
    const int64_t pc = c0 < n ? c.positions[(int64_t)b * c.capacity + c0] : pq;
    __syncthreads();   // the previous chunk's readers of sQ are done
    for (int i = threadIdx.x; i < GQ * (d / 2); i += DG_T) {
      const int hh = i / (d / 2), p = i % (d / 2);
      const int64_t qb = ((int64_t)b * c.Hq + h * GQ + hh) * d;
      const float x0 = load_elem(q, qb + 2 * p, dtype), x1 = load_elem(q, qb + 2 * p + 1, dtype);
      float cs, sn;
      rope_cs(static_cast<double>(pq - pc) * sFreq[p], cs, sn);
      sQ[hh * d + 2 * p] = (x0 * cs - x1 * sn) * scale;
      sQ[hh * d + 2 * p + 1] = (x0 * sn + x1 * cs) * scale;
    }
    __syncthreads();
    // ---- K side: one item per thread
    const int it = c0 + threadIdx.x;
    int src = -1;          // >= 0 code slot, <= -2 pool slot (-2 - s), -1 invalid
    int64_t tok = -1;
    if (it < s1) {
      if (it < n) {
        if (qm[it >> 5] & (1u << (it & 31))) { src = it; tok = it; }
      } else {
        const int s = it - n;
        const int8_t kind = c.pool_kind[bh * c.pool_capacity + s];
        const int t = c.pool_tok[bh * c.pool_capacity + s];
        if (kind != ANTKV_KIND_FREE && t >= 0 && t < n) { src = -2 - s; tok = t; }
      }
    }
    float sc[GQ];
#pragma unroll
    for (int hh = 0; hh < GQ; ++hh) sc[hh] = 0.f;
    if (src != -1) {
      const int64_t rel = c.positions[(int64_t)b * c.capacity + tok] - pc;
      const bool grid = rel == threadIdx.x;          // R(rel) is in the table
      const double drel = static_cast<double>(rel);
      auto pair = [&](int p, float k0, float k1) {
        float cs, sn;
        if (grid) {
          const float2 r = sRot[p * DG_T + threadIdx.x];
          cs = r.x;
          sn = r.y;
        } else {
          rope_cs(drel * sFreq[p], cs, sn);
        }
        const float r0 = k0 * cs - k1 * sn, r1 = k0 * sn + k1 * cs;
#pragma unroll
        for (int hh = 0; hh < GQ; ++hh)
          sc[hh] = fmaf(sQ[hh * d + 2 * p], r0, fmaf(sQ[hh * d + 2 * p + 1], r1, sc[hh]));
      };
      if (src >= 0) {
        // one code per group, its centroid read as pairs (d_sub is even for RoPE pairs
        // that stay inside a group; odd d_sub falls back to element reads)
        for (int g = 0; g < G; ++g) {
          const int code = load_code_unit(c, hb + code_offset(src, 0, g, G));
          const float *cen = cbK + (int64_t)code * dsub;
          if ((dsub & 1) == 0) {
            for (int o = 0; o < dsub; o += 2) {
              const float2 kv = *reinterpret_cast<const float2 *>(cen + o);
              pair((g * dsub + o) >> 1, kv.x, kv.y);
            }
          } else {
            for (int o = 0; o < dsub; ++o) {
              const int e = g * dsub + o;
              if (e & 1) continue;
              const int g1 = (e + 1) / dsub, o1 = (e + 1) % dsub;
              const float k1 = g1 == g ? cen[o + 1]
                                       : cbK[(int64_t)load_code_unit(c, hb + code_offset(src, 0, g1, G)) * dsub + o1];
              pair(e >> 1, cen[o], k1);
            }
          }
          sVc[threadIdx.x * G + g] = load_code_unit(c, hb + code_offset(src, 1, g, G));
        }
      } else {
        const int64_t prow = pool + (int64_t)(-2 - src) * 2 * d;
        for (int p = 0; p < d / 2; ++p)
          pair(p, load_elem(c.pool_rows, prow + 2 * p, c.row_dtype),
               load_elem(c.pool_rows, prow + 2 * p + 1, c.row_dtype));
      }
    }
    sSrc[threadIdx.x] = src;
#pragma unroll
    for (int hh = 0; hh < GQ; ++hh) sS[hh * DG_T + threadIdx.x] = src != -1 ? sc[hh] : -INFINITY;
    __syncthreads();
    // ---- online softmax over the chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int hh = 0; hh < GQ; ++hh) {
      float v = warp_max(sS[hh * DG_T + threadIdx.x]);
      if (lane == 0) sRed[hh * 4 + warp] = v;
    }
    __syncthreads();
    float m_new[GQ], alpha[GQ];
#pragma unroll
    for (int hh = 0; hh < GQ; ++hh) {
      float cm = fmaxf(fmaxf(sRed[hh * 4], sRed[hh * 4 + 1]), fmaxf(sRed[hh * 4 + 2], sRed[hh * 4 + 3]));
      m_new[hh] = fmaxf(m_run[hh], cm);
      alpha[hh] = (m_run[hh] == -INFINITY) ? 0.f : __expf(m_run[hh] - m_new[hh]);
      const float sv = sS[hh * DG_T + threadIdx.x];
      const float p = (sv == -INFINITY) ? 0.f : __expf(sv - m_new[hh]);
      sS[hh * DG_T + threadIdx.x] = p;
      const float ps = warp_sum(p);
      if (lane == 0) sRed[4 * GQ + hh * 4 + warp] = ps;
    }
    __syncthreads();
#pragma unroll
    for (int hh = 0; hh < GQ; ++hh) {
      const float cs = sRed[4 * GQ + hh * 4] + sRed[4 * GQ + hh * 4 + 1] +
                       sRed[4 * GQ + hh * 4 + 2] + sRed[4 * GQ + hh * 4 + 3];
      l_run[hh] = l_run[hh] * alpha[hh] + cs;
      m_run[hh] = m_new[hh];
      acc[hh][0] *= alpha[hh];
      acc[hh][1] *= alpha[hh];
    }
    // ---- V side: one (or two) dims per thread
    const int cnt = min(DG_T, s1 - c0);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int dim = threadIdx.x + half * DG_T;
      if (dim >= d) continue;
      const int g = dim / dsub, o = dim % dsub;
      float a[GQ];
#pragma unroll
      for (int hh = 0; hh < GQ; ++hh) a[hh] = acc[hh][half];
      for (int t = 0; t < cnt; ++t) {
        const int s = sSrc[t];
        if (s == -1) continue;
        float v;
        if (s >= 0) v = cbV[sVc[t * G + g] * dsub + o];
        else v = load_elem(c.pool_rows, pool + (int64_t)(-2 - s) * 2 * d + d + dim, c.row_dtype);
#pragma unroll
        for (int hh = 0; hh < GQ; ++hh) a[hh] = fmaf(sS[hh * DG_T + t], v, a[hh]);
      }
#pragma unroll
      for (int hh = 0; hh < GQ; ++hh) acc[hh][half] = a[hh];
    }
    __syncthreads();
  }
  // ---- partials
#pragma unroll
  for (int hh = 0; hh < GQ; ++hh) {
    const int64_t row = ((int64_t)split * c.B + b) * c.Hq + h * GQ + hh;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int dim = threadIdx.x + half * DG_T;
      if (dim < d) ws_o[row * d + dim] = acc[hh][half];
    }
    if (threadIdx.x == 0) {
      ws_m[row] = m_run[hh];
      ws_l[row] = l_run[hh];
    }
  }
}

// Split-KV combine: unnormalised partial o_s with (m_s, l_s) per split.
// One CTA per output row: warp 0 turns the (m, l) of every split into
// weights in shared memory, then each thread sums its dims over the splits
// with all loads of a batch of 8 splits in flight.
__global__ void decode_combine_kernel(const float *__restrict__ ws_o, const float *__restrict__ ws_m,
                                      const float *__restrict__ ws_l, int splits, int64_t rows,
                                      int d, float *__restrict__ out, float *__restrict__ lse) {
  extern __shared__ float cw[];   // [splits] weights, then M, L
  const int64_t row = blockIdx.x;
  if (threadIdx.x < 32) {
    float M = -INFINITY;
    for (int s = threadIdx.x; s < splits; s += 32) M = fmaxf(M, ws_m[s * rows + row]);
    M = warp_max(M);
    float L = 0.f;
    for (int s = threadIdx.x; s < splits; s += 32) {
      const float ms = ws_m[s * rows + row];
      const float wv = ms == -INFINITY ? 0.f : __expf(ms - M);
      cw[s] = wv;
      L += wv * ws_l[s * rows + row];
    }
    L = warp_sum(L);
    if (threadIdx.x == 0) {
      cw[splits] = M;
      cw[splits + 1] = L;
    }
  }
  __syncthreads();
  const float inv = 1.f / cw[splits + 1];
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float acc = 0.f;
    int s = 0;
    for (; s + 8 <= splits; s += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ws_o[((s + u) * rows + row) * d + t];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fmaf(cw[s + u], v[u], acc);
    }
    for (; s < splits; ++s) acc = fmaf(cw[s], ws_o[(s * rows + row) * d + t], acc);
    out[row * d + t] = acc * inv;
  }
  if (lse && threadIdx.x == 0) lse[row] = cw[splits] + logf(cw[splits + 1]);
}

// Merge of P normalised shard results with their LSE (sequence sharding).
__global__ void lse_combine_kernel(const float *__restrict__ o, const float *__restrict__ lse,
                                   int P, int64_t rows, int d, float *__restrict__ out,
                                   float *__restrict__ lse_out) {
  const int64_t row = blockIdx.x;
  float M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmaxf(M, lse[p * rows + row]);
  float W = 0.f;
  for (int p = 0; p < P; ++p) {
    const float l = lse[p * rows + row];
    if (l != -INFINITY) W += __expf(l - M);
  }
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < P; ++p) {
      const float l = lse[p * rows + row];
      if (l != -INFINITY) acc = fmaf(__expf(l - M), o[(p * rows + row) * d + t], acc);
    }
    out[row * d + t] = acc / W;
  }
  if (lse_out && threadIdx.x == 0) lse_out[row] = M + logf(W);
}

// Generic-path publish: copy the rank's partial rows into each peer's slot of
// the step's buffer half (parity seq & 1), then the last CTA releases the slot
// flags (system scope).  Two halves make reuse race-free by construction: a
// rank publishes step s + 2 only after its merge of s + 1, which waited for
// every peer's publish of s + 1, which each peer issued after its own merge of
// s (stream order) -- so nobody still reads the half that s + 2 overwrites.
__global__ void publish_partial_kernel(const float *__restrict__ out, const float *__restrict__ lse, int d,
                                       PublishArgs pub) {
  const int64_t row = blockIdx.x, prow = (int64_t)pub.rank * pub.rows + row;
  const int64_t half = pub.seq & 1u;
  for (int p = 0; p < pub.n; ++p) {
    float *o = pub.o[p] + half * pub.n * pub.rows * d;
    for (int t = threadIdx.x; t < d; t += blockDim.x) o[prow * d + t] = out[row * d + t];
    if (threadIdx.x == 0) pub.lse[p][half * pub.n * pub.rows + prow] = lse[row];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(pub.cnt, 1) == (int)pub.rows - 1) {
    *pub.cnt = 0;
    __threadfence_system();
    for (int p = 0; p < pub.n; ++p)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pub.flag[p] + half * pub.n + pub.rank),
                   "r"(pub.seq)
                   : "memory");
  }
}

// Waits until every slot's flag of the step's half (parity seq & 1) equals
// `seq` exactly (system-scope acquire), then merges the P partials like
// lse_combine_kernel.  Slots are read through L2
// (__ldcg): peers write them over NVLink every step.
__global__ void lse_merge_wait_kernel(const float *__restrict__ o, const float *__restrict__ lse,
                                      const unsigned *__restrict__ flags, int P, unsigned seq,
                                      int64_t rows, int d, float *__restrict__ out,
                                      float *__restrict__ lse_out) {
  // bounded wait: a peer that never publishes (a dead rank, a mapping that
  // does not reach this GPU) turns into NaN outputs after ~10 s, not a hang
  const int64_t half = seq & 1u;
  o += half * P * rows * d;
  lse += half * P * rows;
  flags += half * P;
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < P) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + threadIdx.x) : "memory");
      if (v != seq) {
        __nanosleep(64);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10000000000ull) {
          timed_out = 1;
          break;
        }
      }
    } while (v != seq);
  }
  __syncthreads();
  if (timed_out) {
    const int64_t row = blockIdx.x;
    for (int t = threadIdx.x; t < d; t += blockDim.x) out[row * d + t] = __int_as_float(0x7fc00000);
    if (lse_out && threadIdx.x == 0) lse_out[row] = __int_as_float(0x7fc00000);
    return;
  }
  const int64_t row = blockIdx.x;
  float M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmaxf(M, __ldcg(lse + p * rows + row));
  float W = 0.f;
  for (int p = 0; p < P; ++p) {
    const float l = __ldcg(lse + p * rows + row);
    if (l != -INFINITY) W += __expf(l - M);
  }
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < P; ++p) {
      const float l = __ldcg(lse + p * rows + row);
      if (l != -INFINITY) acc = fmaf(__expf(l - M), __ldcg(o + (p * rows + row) * d + t), acc);
    }
    out[row * d + t] = acc / W;
  }
  if (lse_out && threadIdx.x == 0) lse_out[row] = M + logf(W);
}

static size_t generic_smem(const antkv_cache_desc &c, int gq, bool cb_smem) {
  size_t s = sizeof(double) * (c.d / 2) + sizeof(float2) * (c.d / 2) * DG_T +
             sizeof(float) * (gq * c.d + gq * DG_T + 8 * gq) + sizeof(int) * (DG_T + DG_T * c.groups);
  if (cb_smem) s += sizeof(float) * 2 * c.m * c.d_sub;
  return s;
}

template <int GQ>
static int launch_generic(const antkv_cache_desc &c, const void *q, int dtype, const int64_t *qpos,
                          float *wo, float *wm, float *wl, int splits, cudaStream_t st) {
  const bool cb_smem = sizeof(float) * 2 * (size_t)c.m * c.d_sub <= 96 * 1024;
  const size_t smem = generic_smem(c, GQ, cb_smem);
  ANTKV_REQUIRE(smem <= 200 * 1024, "decode shared memory %zu too large", smem);
  dim3 grid(splits, c.Hkv, c.B);
  if (cb_smem) {
    cudaFuncSetAttribute(decode_generic_kernel<GQ, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    decode_generic_kernel<GQ, true><<<grid, DG_T, smem, st>>>(c, q, dtype, qpos, wo, wm, wl);
  } else {
    cudaFuncSetAttribute(decode_generic_kernel<GQ, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    decode_generic_kernel<GQ, false><<<grid, DG_T, smem, st>>>(c, q, dtype, qpos, wo, wm, wl);
  }
  ANTKV_LAUNCH_CHECK("decode_generic_kernel");
  return ANTKV_OK;
}

static int auto_splits(const antkv_cache_desc &c) {
  // enough CTAs for ~2 waves on 148 SMs; each split covers >= 256 items
  int64_t items = (int64_t)c.capacity + c.pool_capacity;
  int want = (2 * 148 + c.B * c.Hkv - 1) / (c.B * c.Hkv);
  int maxs = static_cast<int>((items + 255) / 256);
  int s = want < maxs ? want : maxs;
  return s < 1 ? 1 : (s > 1024 ? 1024 : s);
}

// Number of partials a call produces (generic: splits; fast: code + pool CTAs).
static int planned_splits(const antkv_cache_desc &c, int splits, int mode) {
  if (mode == kFast) {
    int cs, ps;
    decode_fast_plan(c, splits, cs, ps);
    return cs + ps;
  }
  if (mode == kStaged) return decode_tc_plan(c, splits);
  return splits > 0 ? splits : auto_splits(c);
}

}  // namespace antkv

using namespace antkv;

// tickets [B*Hkv] + [B], the per-head cache-update plans [B*Hkv][kPlanWords]
// and the publish counter [1] (padded to 4 words)
static int64_t counter_bytes(const antkv_cache_desc &c) {
  return (int64_t)(c.B * c.Hkv + c.B + kPlanWords * c.B * c.Hkv + 4) * 4;   // +4: keeps 16-byte alignment
}

static int64_t partial_bytes(const antkv_cache_desc &c, int used) {
  return (int64_t)used * c.B * c.Hq * (c.d + 2) * (int64_t)sizeof(float);
}

// Workspace = split partials (o, m, l) + self-resetting CTA tickets
// [B*Hkv + B] int32 at the end.  Zero it once before the first call.
extern "C" int64_t antkv_decode_workspace_bytes(const antkv_cache_desc *c, int splits) {
  if (!c) return -1;
  int s = planned_splits(*c, splits, kGeneric);
  if (decode_fast_supported(*c)) s = max(s, planned_splits(*c, splits, kFast));
  if (decode_tc_supported(*c)) s = max(s, planned_splits(*c, splits, kStaged));
  return partial_bytes(*c, s) + counter_bytes(*c) + 256;
}

static int attention_impl(const antkv_cache_desc *c, const void *q, int dtype, const void *knew,
                          const void *vnew, int kvdtype, const int64_t *qpos, float *out,
                          float *lse, void *workspace, int64_t workspace_bytes, int splits,
                          int mode, cudaStream_t st) {
  const int used = planned_splits(*c, splits, mode);
  const int64_t rows = (int64_t)c->B * c->Hq;
  ANTKV_REQUIRE(workspace_bytes >= antkv_decode_workspace_bytes(c, splits), "decode workspace too small");
  float *wo = reinterpret_cast<float *>(workspace);
  float *wm = wo + (int64_t)used * rows * c->d;
  float *wl = wm + (int64_t)used * rows;
  int *cnt = reinterpret_cast<int *>(reinterpret_cast<char *>(workspace) + workspace_bytes -
                                     256 - counter_bytes(*c));
  if (mode != kFast) previous_cache_on_stream(st, c->codes);   // (the fast launch records itself)
  if (mode == kFast)
    return decode_fast_launch(*c, q, dtype, knew, vnew, kvdtype, qpos, out, lse, wo, wm, wl, cnt,
                              splits, st);
  const int gq = c->Hq / c->Hkv;
  int rc;
  if (mode == kStaged)   // one launch: partials + the last CTA's merge
    return decode_tc_launch(*c, q, dtype, qpos, wo, wm, wl, out, lse, cnt, used, st);
  switch (gq) {
    case 1: rc = launch_generic<1>(*c, q, dtype, qpos, wo, wm, wl, used, st); break;
    case 2: rc = launch_generic<2>(*c, q, dtype, qpos, wo, wm, wl, used, st); break;
    case 4: rc = launch_generic<4>(*c, q, dtype, qpos, wo, wm, wl, used, st); break;
    case 8: rc = launch_generic<8>(*c, q, dtype, qpos, wo, wm, wl, used, st); break;
    default:
      set_error("GQA group size %d unsupported (1, 2, 4, 8)", gq);
      return ANTKV_EUNSUPPORTED;
  }
  if (rc) return rc;
  decode_combine_kernel<<<(unsigned)rows, 128, (used + 2) * sizeof(float), st>>>(wo, wm, wl, used, rows, c->d, out, lse);
  ANTKV_LAUNCH_CHECK("decode_combine_kernel");
  return ANTKV_OK;
}

static int check_decode_args(const antkv_cache_desc *c, const void *q, float *out) {
  ANTKV_REQUIRE(c != nullptr && q != nullptr && out != nullptr, "null argument");
  ANTKV_REQUIRE(c->Hq % c->Hkv == 0, "Hq must be a multiple of Hkv");
  ANTKV_REQUIRE(c->d % 2 == 0 && c->d <= 256, "head dimension must be even and <= 256");
  return ANTKV_OK;
}

// The fused kernel bulk-copies the 4 query rows of a head: q must be 16-byte
// aligned (any contiguous tensor is); otherwise the generic kernels run.
static bool fast_ok(const antkv_cache_desc *c, const void *q, int fast) {
  return fast == 1 && decode_fast_supported(*c) && (reinterpret_cast<uintptr_t>(q) & 15) == 0;
}

// fast: 0 generic, 1 best available (fused d8m256, else staged), 2 staged.
static int decode_mode(const antkv_cache_desc *c, const void *q, int fast) {
  if (fast_ok(c, q, fast)) return kFast;
  if (fast >= 1 && decode_tc_supported(*c)) return kStaged;
  return kGeneric;
}

extern "C" int antkv_decode_attention(const antkv_cache_desc *c, const void *q, int dtype,
                                      const int64_t *qpos, float *out, float *lse,
                                      void *workspace, int64_t workspace_bytes, int splits,
                                      int fast, void *stream) {
  int rc = check_decode_args(c, q, out);
  if (rc) return rc;
  return attention_impl(c, q, dtype, nullptr, nullptr, dtype, qpos, out, lse, workspace,
                        workspace_bytes, splits, decode_mode(c, q, fast), as_stream(stream));
}

extern "C" int antkv_decode_step(const antkv_cache_desc *c, const void *q, const void *k,
                                 const void *v, int dtype, const int64_t *qpos, float *out,
                                 float *lse, void *workspace, int64_t workspace_bytes, int splits,
                                 int fast, void *stream) {
  int rc = check_decode_args(c, q, out);
  if (rc) return rc;
  ANTKV_REQUIRE(k != nullptr && v != nullptr, "null k/v");
  cudaStream_t st = as_stream(stream);
  const int mode = decode_mode(c, q, fast);
  if (mode == kFast)   // one fused launch
    return attention_impl(c, q, dtype, k, v, dtype, qpos, out, lse, workspace, workspace_bytes,
                          splits, kFast, st);
  rc = antkv_cache_append(c, k, v, dtype, qpos, stream);
  if (rc) return rc;
  rc = attention_impl(c, q, dtype, nullptr, nullptr, dtype, qpos, out, lse, workspace,
                      workspace_bytes, splits, mode, st);
  if (rc) return rc;
  return antkv_cache_evict(c, stream);
}

extern "C" int antkv_lse_combine(const float *o, const float *lse, int P, int64_t rows, int d,
                                 float *out, float *lse_out, void *stream) {
  ANTKV_REQUIRE(P >= 1 && d >= 1, "bad combine shape");
  if (rows == 0) return ANTKV_OK;
  lse_combine_kernel<<<(unsigned)rows, 128, 0, as_stream(stream)>>>(o, lse, P, rows, d, out, lse_out);
  ANTKV_LAUNCH_CHECK("lse_combine_kernel");
  return ANTKV_OK;
}

// ---------------------------------------------------------------- peer exchange
// The counter for publish completion lives after the plans in the workspace.
static int *publish_counter(const antkv_cache_desc &c, void *workspace, int64_t workspace_bytes) {
  int *cnt = reinterpret_cast<int *>(reinterpret_cast<char *>(workspace) + workspace_bytes - 256 -
                                     counter_bytes(c));
  return cnt + c.B * c.Hkv + c.B + kPlanWords * c.B * c.Hkv;
}

extern "C" int antkv_decode_step_publish(const antkv_cache_desc *c, const void *q, const void *k,
                                         const void *v, int dtype, const int64_t *qpos, float *out,
                                         float *lse, void *workspace, int64_t workspace_bytes,
                                         int splits, int fast, float *const *dst_o,
                                         float *const *dst_lse, unsigned *const *dst_flags, int n_dst,
                                         int rank, unsigned seq, void *stream) {
  int rc = check_decode_args(c, q, out);
  if (rc) return rc;
  ANTKV_REQUIRE(lse != nullptr, "publishing needs lse");
  ANTKV_REQUIRE(n_dst >= 1 && dst_o != nullptr && dst_lse != nullptr && dst_flags != nullptr,
                "publishing needs the destination pointer arrays");
  ANTKV_REQUIRE(rank >= 0, "bad rank");
  ANTKV_REQUIRE(workspace_bytes >= antkv_decode_workspace_bytes(c, splits), "decode workspace too small");
  cudaStream_t st = as_stream(stream);
  PublishArgs pub;
  pub.o = dst_o;
  pub.lse = dst_lse;
  pub.flag = dst_flags;
  pub.n = n_dst;
  pub.rank = rank;
  pub.rows = (int64_t)c->B * c->Hq;
  pub.cnt = publish_counter(*c, workspace, workspace_bytes);
  pub.seq = seq;
  // the step (one fused launch on the fast path), then the partial's rows go
  // to every peer slot and the flags are released (a second, tiny launch: the
  // fused decode kernel is kept exactly as timed)
  const int mode = decode_mode(c, q, fast);
  if (mode == kFast) {
    rc = attention_impl(c, q, dtype, k, v, dtype, qpos, out, lse, workspace, workspace_bytes, splits,
                        kFast, st);
    if (rc) return rc;
  } else {
    if (k) {
      ANTKV_REQUIRE(v != nullptr, "null v");
      rc = antkv_cache_append(c, k, v, dtype, qpos, stream);
      if (rc) return rc;
    }
    rc = attention_impl(c, q, dtype, nullptr, nullptr, dtype, qpos, out, lse, workspace,
                        workspace_bytes, splits, mode, st);
    if (rc) return rc;
    if (k) {
      rc = antkv_cache_evict(c, stream);
      if (rc) return rc;
    }
  }
  publish_partial_kernel<<<(unsigned)pub.rows, 128, 0, st>>>(out, lse, c->d, pub);
  ANTKV_LAUNCH_CHECK("publish_partial_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_lse_merge_wait(const float *o, const float *lse, const unsigned *flags, int P,
                                    unsigned seq, int64_t rows, int d, float *out, float *lse_out,
                                    void *stream) {
  ANTKV_REQUIRE(P >= 1 && P <= 128 && d >= 1, "bad merge shape");
  if (rows == 0) return ANTKV_OK;
  lse_merge_wait_kernel<<<(unsigned)rows, 128, 0, as_stream(stream)>>>(o, lse, flags, P, seq, rows, d,
                                                                       out, lse_out);
  ANTKV_LAUNCH_CHECK("lse_merge_wait_kernel");
  return ANTKV_OK;
}
