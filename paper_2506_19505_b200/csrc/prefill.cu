// Prefill path: RoPE rotation, blocked attention with (O, L, M) auxiliaries,
// Alg. 1 anchor-score column sums, and the reference FFI entry points that
// share these kernels (antkv._ckernels.flash_aux / ans_blocked).
//
// d = 128 runs on the tensor-core kernels of prefill_mma.cu (split-precision
// logits); other head sizes use the float32 CUDA-core tiles below.  The
// anchor scores need S accurate enough that anchor sets match the float64
// oracle wherever the budget-boundary margin allows (SURVEY.md §7 hard
// part 3).
#include "common.cuh"

namespace antkv {

constexpr int FA_BQ = 64;
constexpr int FA_BK = 64;
constexpr int FA_THREADS = 256;
constexpr int FA_DMAX = 128;

// X [rows][d] with rows = B*H*n, positions [B][n] -> out fp32 rotated*scale;
// norms (optional) = L2 norm of the pre-RoPE row.  attention.py:89-106,167.
__global__ void rope_rotate_kernel(const void *__restrict__ X, int dtype,
                                   const int64_t *__restrict__ positions, int H,
                                   int n, int d, double theta, float scale,
                                   float *__restrict__ out, float *__restrict__ norms) {
  int64_t row = blockIdx.x;
  int b = static_cast<int>(row / ((int64_t)H * n));
  int j = static_cast<int>(row % n);
  double pos = positions ? static_cast<double>(positions[(int64_t)b * n + j]) : 0.0;
  const int64_t base = row * d;
  float nrm = 0.f;
  if (!positions) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      float x = load_elem(X, base + i, dtype);
      nrm = fmaf(x, x, nrm);
      out[base + i] = x * scale;
    }
  }
  for (int i = threadIdx.x; positions && i < d / 2; i += blockDim.x) {
    float x0 = load_elem(X, base + 2 * i, dtype);
    float x1 = load_elem(X, base + 2 * i + 1, dtype);
    nrm = fmaf(x0, x0, fmaf(x1, x1, nrm));
    float c, s;
    rope_cs(pos * rope_freq(theta, i, d), c, s);
    out[base + 2 * i] = (x0 * c - x1 * s) * scale;
    out[base + 2 * i + 1] = (x0 * s + x1 * c) * scale;
  }
  if (norms) {
    __shared__ float red[32];
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
      norms[row] = sqrtf(t);
    }
  }
}

// Load a [64][d] fp32 tile (rows r0.., zero beyond nrows) into smem with a
// padded stride (d+1) to break bank conflicts on the column walks.
__device__ __forceinline__ void load_tile(float *dst, const float *__restrict__ src,
                                          int r0, int nrows, int d, int ld) {
  for (int idx = threadIdx.x; idx < 64 * d; idx += blockDim.x) {
    int r = idx / d, c = idx - r * d;
    int gr = r0 + r;
    dst[r * ld + c] = (gr < nrows) ? src[(int64_t)gr * d + c] : 0.f;
  }
}

// One CTA = (query head, 64-query tile).  Online softmax over 64-key tiles
// (kernels/pure.py:13-52 semantics).  Thread (ty, tx): S rows 4ty..4ty+3,
// S cols 4tx..4tx+3; O rows 4ty..+3, O cols tx + 16c.
__global__ void __launch_bounds__(FA_THREADS)
flash_aux_kernel(const float *__restrict__ Qs, const float *__restrict__ Kr,
                 const float *__restrict__ V, int heads, int group, int n_q, int n_k,
                 int d, int dv, int causal, float *__restrict__ O,
                 float *__restrict__ Lout, float *__restrict__ Mout) {
  extern __shared__ float sm[];
  const int ldq = d + 1, ldv = dv + 1;
  float *sQ = sm;
  float *sK = sQ + 64 * ldq;
  float *sV = sK + 64 * ldq;
  float *sP = sV + 64 * ldv;  // [64][65]
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * FA_BQ;
  const int hk = h / group;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float *Qh = Qs + (int64_t)h * n_q * d;
  const float *Kh = Kr + (int64_t)hk * n_k * d;
  const float *Vh = V + (int64_t)hk * n_k * dv;
  load_tile(sQ, Qh, q0, n_q, d, ldq);

  const int ncol = (dv + 15) / 16;  // <= 8
  float acc[4][8];
  float m_run[4], l_run[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m_run[r] = -INFINITY;
    l_run[r] = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
  }
  const int q_last = min(q0 + FA_BQ, n_q) - 1;
  for (int k0 = 0; k0 < n_k; k0 += FA_BK) {
    if (causal && k0 > q_last) break;
    __syncthreads();
    load_tile(sK, Kh, k0, n_k, d, ldq);
    load_tile(sV, Vh, k0, n_k, dv, ldv);
    __syncthreads();
    float s[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) s[r][c] = 0.f;
    for (int t = 0; t < d; ++t) {
      float qv[4], kv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) qv[r] = sQ[(4 * ty + r) * ldq + t];
#pragma unroll
      for (int c = 0; c < 4; ++c) kv[c] = sK[(4 * tx + c) * ldq + t];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) s[r][c] = fmaf(qv[r], kv[c], s[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qi = q0 + 4 * ty + r;
      float rmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int kj = k0 + 4 * tx + c;
        if (kj >= n_k || (causal && kj > qi)) s[r][c] = -INFINITY;
        rmax = fmaxf(rmax, s[r][c]);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      const float m_new = fmaxf(m_run[r], rmax);
      const float alpha = (m_run[r] == -INFINITY) ? 0.f : __expf(m_run[r] - m_new);
      float psum = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float p = (s[r][c] == -INFINITY) ? 0.f : expf(s[r][c] - m_new);
        psum += p;
        sP[(4 * ty + r) * 65 + 4 * tx + c] = p;
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
      l_run[r] = l_run[r] * alpha + psum;
      m_run[r] = m_new;
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] *= alpha;
    }
    __syncthreads();
    const int kcount = min(FA_BK, n_k - k0);
    for (int t = 0; t < kcount; ++t) {
      float pv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pv[r] = sP[(4 * ty + r) * 65 + t];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < ncol) {
          const int col = tx + 16 * c;
          const float vv = (col < dv) ? sV[t * ldv + col] : 0.f;
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[r][c] = fmaf(pv[r], vv, acc[r][c]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = q0 + 4 * ty + r;
    if (qi >= n_q) continue;
    const float inv = 1.f / l_run[r];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = tx + 16 * c;
      if (c < ncol && col < dv) O[((int64_t)h * n_q + qi) * dv + col] = acc[r][c] * inv;
    }
    if (tx == 0) {
      Lout[(int64_t)h * n_q + qi] = l_run[r];
      Mout[(int64_t)h * n_q + qi] = m_run[r];
    }
  }
}

// One CTA = (output head, 64-key tile); loops over query tiles (and, for the
// GQA-summed prefill variant, over the `sum_group` query heads mapping to the
// same output head).  A = exp(S - M_i)/L_i, column sums
// (kernels/pure.py:55-81, Alg. 1 second pass).
__global__ void __launch_bounds__(FA_THREADS)
ans_kernel(const float *__restrict__ Qs, const float *__restrict__ Kr,
           const float *__restrict__ Mv, const float *__restrict__ Lv,
           const float *__restrict__ qn, int group, int sum_group, int n_q, int n_k,
           int d, int causal, float *__restrict__ ans_k, float *__restrict__ ans_v) {
  extern __shared__ float sm[];
  const int ld = d + 1;
  float *sQ = sm;
  float *sK = sQ + 64 * ld;
  float *sRow = sK + 64 * ld;      // [64] M, [64] 1/L, [64] qn
  float *sRed = sRow + 3 * 64;     // [16][64] x2
  const int ho = blockIdx.y;       // output head
  const int k0 = blockIdx.x * FA_BK;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float colk[4] = {0.f, 0.f, 0.f, 0.f}, colv[4] = {0.f, 0.f, 0.f, 0.f};
  for (int gq = 0; gq < sum_group; ++gq) {
    const int h = ho * sum_group + gq;     // query head
    const int hk = h / group;              // key head
    const float *Qh = Qs + (int64_t)h * n_q * d;
    const float *Kh = Kr + (int64_t)hk * n_k * d;
    __syncthreads();
    load_tile(sK, Kh, k0, n_k, d, ld);
    const int qstart = causal ? (k0 / FA_BQ) * FA_BQ : 0;
    for (int q0 = qstart; q0 < n_q; q0 += FA_BQ) {
      __syncthreads();
      load_tile(sQ, Qh, q0, n_q, d, ld);
      for (int i = threadIdx.x; i < 64; i += blockDim.x) {
        const int qi = q0 + i;
        const bool ok = qi < n_q;
        sRow[i] = ok ? Mv[(int64_t)h * n_q + qi] : 0.f;
        sRow[64 + i] = ok ? 1.f / Lv[(int64_t)h * n_q + qi] : 0.f;
        sRow[128 + i] = ok ? qn[(int64_t)h * n_q + qi] : 0.f;
      }
      __syncthreads();
      float s[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) s[r][c] = 0.f;
      for (int t = 0; t < d; ++t) {
        float qv[4], kv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) qv[r] = sQ[(4 * ty + r) * ld + t];
#pragma unroll
        for (int c = 0; c < 4; ++c) kv[c] = sK[(4 * tx + c) * ld + t];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) s[r][c] = fmaf(qv[r], kv[c], s[r][c]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int qi = q0 + 4 * ty + r;
        if (qi >= n_q) continue;
        const float mi = sRow[4 * ty + r], invl = sRow[64 + 4 * ty + r], qni = sRow[128 + 4 * ty + r];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int kj = k0 + 4 * tx + c;
          if (kj >= n_k || (causal && kj > qi)) continue;
          const float a = expf(s[r][c] - mi) * invl;
          colv[c] += a;
          colk[c] = fmaf(a * (1.f - a), qni, colk[c]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    sRed[ty * 64 + 4 * tx + c] = colk[c];
    sRed[1024 + ty * 64 + 4 * tx + c] = colv[c];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 64; c += blockDim.x) {
    const int kj = k0 + c;
    if (kj >= n_k) continue;
    float sk = 0.f, sv = 0.f;
    for (int r = 0; r < 16; ++r) {
      sk += sRed[r * 64 + c];
      sv += sRed[1024 + r * 64 + c];
    }
    ans_k[(int64_t)ho * n_k + kj] = sk;
    ans_v[(int64_t)ho * n_k + kj] = sv;
  }
}

int launch_flash_mma(const float *Qs, const float *Kr, const float *V, int heads, int kv_heads,
                     int n_q, int n_k, int d, int dv, int causal, float *O, float *L, float *M,
                     cudaStream_t st);
int launch_flash_tc(const float *Qs, const float *Kr, const float *V, int heads, int kv_heads, int n_q,
                    int n_k, int d, int dv, int causal, int v_bf16, float *O, float *L, float *M,
                    cudaStream_t st);
int prefill_tc_fused(const void *Q, const void *K, const void *V, int dtype, const int64_t *positions, int B,
                     int Hq, int Hkv, int n, int d, double theta, float *O, float *M, float *L, float *qn,
                     float *ans_k, float *ans_v, cudaStream_t st);
int launch_ans_tc(const float *Qs, const float *Kr, const float *M, const float *L, const float *qn,
                  int heads, int kv_heads, int sum_group, int n_q, int n_k, int d, int causal,
                  float *ans_k, float *ans_v, cudaStream_t st);
int launch_ans_mma(const float *Qs, const float *Kr, const float *M, const float *L, const float *qn,
                   int heads, int kv_heads, int sum_group, int n_q, int n_k, int d, int causal,
                   float *ans_k, float *ans_v, cudaStream_t st);

static int launch_flash(const float *Qs, const float *Kr, const float *V, int heads,
                        int kv_heads, int n_q, int n_k, int d, int dv, int causal,
                        float *O, float *L, float *M, cudaStream_t st, int v_bf16 = 0) {
  ANTKV_REQUIRE(d >= 1 && d <= FA_DMAX && dv >= 1 && dv <= FA_DMAX,
                "head dimension must be in [1, %d]", FA_DMAX);
  ANTKV_REQUIRE(heads >= 1 && kv_heads >= 1 && heads % kv_heads == 0,
                "heads must be a multiple of kv_heads");
  ANTKV_REQUIRE(!causal || n_q == n_k, "causal attention requires matching Q/K token counts");
  if (n_q == 0) return ANTKV_OK;
  ANTKV_REQUIRE(n_k >= 1, "empty key set");
  {  // d = 128: tcgen05 kernel (prefill_tc.cu), else mma.sync (prefill_mma.cu)
    int rc = launch_flash_tc(Qs, Kr, V, heads, kv_heads, n_q, n_k, d, dv, causal, v_bf16, O, L, M, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
    rc = launch_flash_mma(Qs, Kr, V, heads, kv_heads, n_q, n_k, d, dv, causal, O, L, M, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
  }
  size_t smem = sizeof(float) * (64 * (d + 1) * 2 + 64 * (dv + 1) + 64 * 65);
  cudaFuncSetAttribute(flash_aux_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(ceil_div(n_q, FA_BQ), heads);
  flash_aux_kernel<<<grid, FA_THREADS, smem, st>>>(Qs, Kr, V, heads, heads / kv_heads, n_q,
                                                   n_k, d, dv, causal, O, L, M);
  ANTKV_LAUNCH_CHECK("flash_aux_kernel");
  return ANTKV_OK;
}

static int launch_ans(const float *Qs, const float *Kr, const float *M, const float *L,
                      const float *qn, int heads, int kv_heads, int sum_group, int n_q,
                      int n_k, int d, int causal, float *ans_k, float *ans_v,
                      cudaStream_t st) {
  ANTKV_REQUIRE(d >= 1 && d <= FA_DMAX, "head dimension must be in [1, %d]", FA_DMAX);
  ANTKV_REQUIRE(heads >= 1 && kv_heads >= 1 && heads % kv_heads == 0,
                "heads must be a multiple of kv_heads");
  ANTKV_REQUIRE(!causal || n_q == n_k, "causal attention requires matching Q/K token counts");
  if (n_k == 0) return ANTKV_OK;
  {  // d = 128: tcgen05 kernel (prefill_tc.cu), else mma.sync (prefill_mma.cu)
    int rc = launch_ans_tc(Qs, Kr, M, L, qn, heads, kv_heads, sum_group, n_q, n_k, d, causal, ans_k,
                           ans_v, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
    rc = launch_ans_mma(Qs, Kr, M, L, qn, heads, kv_heads, sum_group, n_q, n_k, d, causal,
                                  ans_k, ans_v, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
  }
  size_t smem = sizeof(float) * (64 * (d + 1) * 2 + 3 * 64 + 2 * 16 * 64);
  cudaFuncSetAttribute(ans_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(ceil_div(n_k, FA_BK), heads / sum_group);
  ans_kernel<<<grid, FA_THREADS, smem, st>>>(Qs, Kr, M, L, qn, heads / kv_heads, sum_group,
                                             n_q, n_k, d, causal, ans_k, ans_v);
  ANTKV_LAUNCH_CHECK("ans_kernel");
  return ANTKV_OK;
}

int rope_rotate(const void *X, int dtype, const int64_t *positions, int B, int H, int n,
                int d, double theta, float scale, float *out, float *norms,
                cudaStream_t st) {
  int64_t rows = (int64_t)B * H * n;
  if (rows == 0) return ANTKV_OK;
  int threads = d < 32 ? 32 : (d > 128 ? 128 : ((d + 31) / 32) * 32);
  rope_rotate_kernel<<<(unsigned)rows, threads, 0, st>>>(X, dtype, positions, H, n, d, theta,
                                                         scale, out, norms);
  ANTKV_LAUNCH_CHECK("rope_rotate_kernel");
  return ANTKV_OK;
}

}  // namespace antkv

using namespace antkv;

extern "C" int antkv_flash_aux(const float *Qs, const float *Kr, const float *V, int heads,
                               int kv_heads, int n_q, int n_k, int d, int dv, int block_q,
                               int block_k, int causal, float *O, float *L, float *M,
                               void *stream) {
  ANTKV_REQUIRE(block_q >= 1 && block_k >= 1, "block sizes must be >= 1");
  return launch_flash(Qs, Kr, V, heads, kv_heads, n_q, n_k, d, dv, causal, O, L, M,
                      as_stream(stream));
}

// ---------------------------------------------------------------- finiteness
// Exponent bits all ones = NaN or +-inf.  16-byte loads, grid-stride; one
// atomic per thread that saw any.
__device__ __forceinline__ bool word_nonfinite(uint32_t w, int dtype) {
  if (dtype == ANTKV_F32) return (w & 0x7F800000u) == 0x7F800000u;
  const uint32_t m = dtype == ANTKV_BF16 ? 0x7F80u : 0x7C00u;
  return (w & m) == m || ((w >> 16) & m) == m;
}
__global__ void __launch_bounds__(256) check_finite_kernel(const uint8_t *__restrict__ x, int dtype,
                                                           int64_t bytes, int *__restrict__ flag) {
  bool bad = false;
  const int64_t nvec = bytes >> 4, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(x) + i);
    bad |= word_nonfinite(v.x, dtype) | word_nonfinite(v.y, dtype) | word_nonfinite(v.z, dtype) |
           word_nonfinite(v.w, dtype);
  }
  // tail (< 16 bytes; whole elements, 2- or 4-byte aligned)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int64_t o = nvec << 4; o < bytes; o += (dtype == ANTKV_F32 ? 4 : 2)) {
      const uint32_t w = dtype == ANTKV_F32 ? *reinterpret_cast<const uint32_t *>(x + o)
                                            : *reinterpret_cast<const uint16_t *>(x + o);
      bad |= word_nonfinite(w, dtype);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

extern "C" int antkv_check_finite(const void *X, int dtype, int64_t n, int *flag, void *stream) {
  ANTKV_REQUIRE(dtype == ANTKV_F32 || dtype == ANTKV_BF16 || dtype == ANTKV_F16, "unknown dtype");
  ANTKV_REQUIRE(n >= 0 && flag, "bad arguments");
  ANTKV_REQUIRE((reinterpret_cast<uintptr_t>(X) & 15) == 0, "X must be 16-byte aligned");
  if (n == 0) return ANTKV_OK;
  const int64_t bytes = n * (dtype == ANTKV_F32 ? 4 : 2);
  const int64_t nvec = bytes >> 4;
  const int blocks = (int)std::min<int64_t>(148 * 8, std::max<int64_t>(1, (nvec + 255) / 256));
  check_finite_kernel<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t *>(X), dtype, bytes,
                                                             flag);
  ANTKV_LAUNCH_CHECK("check_finite_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_rope_rotate(const void *X, int dtype, const int64_t *positions, int B,
                                 int H, int n, int d, double theta_base, float scale, float *out,
                                 float *norms, void *stream) {
  ANTKV_REQUIRE(!positions || d % 2 == 0, "head dimension must be even for RoPE");
  ANTKV_REQUIRE(theta_base > 0, "theta_base must be positive");
  return rope_rotate(X, dtype, positions, B, H, n, d, theta_base, scale, out, norms,
                     as_stream(stream));
}

extern "C" int antkv_ans_blocked(const float *Qs, const float *Kr, const float *M,
                                 const float *L, const float *q_norms, int heads,
                                 int kv_heads, int n_q, int n_k, int d, int block_q,
                                 int block_k, int causal, float *ans_k, float *ans_v,
                                 void *stream) {
  ANTKV_REQUIRE(block_q >= 1 && block_k >= 1, "block sizes must be >= 1");
  return launch_ans(Qs, Kr, M, L, q_norms, heads, kv_heads, 1, n_q, n_k, d, causal, ans_k,
                    ans_v, as_stream(stream));
}

// Scratch for the rotated operands is allocated with cudaMallocAsync on the
// caller's stream (stream-ordered, freed at the end of the call's work).
extern "C" int antkv_prefill_attention_block(const void *Q, const void *K, const void *V,
                                             int dtype, const int64_t *q_positions,
                                             const int64_t *k_positions, int B, int Hq, int Hkv,
                                             int n_q, int n_k, int d, double theta_base,
                                             int causal, float *O, float *M, float *L,
                                             float *q_norms, void *stream) {
  ANTKV_REQUIRE_ALIGNED16(Q, "Q");
  ANTKV_REQUIRE_ALIGNED16(K, "K");
  ANTKV_REQUIRE_ALIGNED16(V, "V");
  ANTKV_REQUIRE(d % 2 == 0, "head dimension must be even for RoPE");
  ANTKV_REQUIRE(theta_base > 0, "theta_base must be positive");
  ANTKV_REQUIRE(Hkv >= 1 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  ANTKV_REQUIRE(B >= 0 && n_q >= 0 && n_k >= 0, "negative size");
  ANTKV_REQUIRE(!causal || n_q == n_k, "causal attention requires matching Q/K token counts");
  if ((int64_t)B * n_q == 0) return ANTKV_OK;
  cudaStream_t st = as_stream(stream);
  float *qs = nullptr, *kr = nullptr, *vf = nullptr;
  size_t qbytes = sizeof(float) * (size_t)B * Hq * n_q * d;
  size_t kbytes = sizeof(float) * (size_t)B * Hkv * n_k * d;
  cudaError_t e = scratch_alloc((void **)&qs, qbytes, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&kr, kbytes ? kbytes : 4, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&vf, kbytes ? kbytes : 4, st);
  if (e != cudaSuccess) return cuda_status(e, "prefill scratch");
  int rc = rope_rotate(Q, dtype, q_positions, B, Hq, n_q, d, theta_base, 1.f / sqrtf((float)d),
                       qs, q_norms, st);
  if (rc == ANTKV_OK) rc = rope_rotate(K, dtype, k_positions, B, Hkv, n_k, d, theta_base, 1.f,
                                       kr, nullptr, st);
  if (rc == ANTKV_OK) rc = rope_rotate(V, dtype, nullptr, B, Hkv, n_k, d, theta_base, 1.f, vf,
                                       nullptr, st);
  for (int b = 0; b < B && rc == ANTKV_OK; ++b) {
    rc = launch_flash(qs + (size_t)b * Hq * n_q * d, kr + (size_t)b * Hkv * n_k * d,
                      vf + (size_t)b * Hkv * n_k * d, Hq, Hkv, n_q, n_k, d, d, causal,
                      O + (size_t)b * Hq * n_q * d, L + (size_t)b * Hq * n_q,
                      M + (size_t)b * Hq * n_q, st, dtype == ANTKV_BF16);
  }
  cudaFreeAsync(qs, st);
  cudaFreeAsync(kr, st);
  cudaFreeAsync(vf, st);
  return rc;
}

extern "C" int antkv_prefill_attention(const void *Q, const void *K, const void *V,
                                       int dtype, const int64_t *positions, int B, int Hq,
                                       int Hkv, int n, int d, double theta_base, float *O,
                                       float *M, float *L, float *q_norms, void *stream) {
  return antkv_prefill_attention_block(Q, K, V, dtype, positions, positions, B, Hq, Hkv, n, n,
                                       d, theta_base, 1, O, M, L, q_norms, stream);
}

extern "C" int antkv_prefill_anchor_scores_block(const void *Q, const void *K, int dtype,
                                                 const int64_t *q_positions,
                                                 const int64_t *k_positions, const float *M,
                                                 const float *L, const float *q_norms, int B,
                                                 int Hq, int Hkv, int n_q, int n_k, int d,
                                                 double theta_base, int causal, float *ans_k,
                                                 float *ans_v, void *stream) {
  ANTKV_REQUIRE_ALIGNED16(Q, "Q");
  ANTKV_REQUIRE_ALIGNED16(K, "K");
  ANTKV_REQUIRE(d % 2 == 0, "head dimension must be even for RoPE");
  ANTKV_REQUIRE(theta_base > 0, "theta_base must be positive");
  ANTKV_REQUIRE(Hkv >= 1 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  ANTKV_REQUIRE(B >= 0 && n_q >= 0 && n_k >= 0, "negative size");
  ANTKV_REQUIRE(!causal || n_q == n_k, "causal attention requires matching Q/K token counts");
  if ((int64_t)B * n_k == 0) return ANTKV_OK;
  cudaStream_t st = as_stream(stream);
  if (n_q == 0) {  // no queries: this block contributes nothing
    cudaError_t e = cudaMemsetAsync(ans_k, 0, sizeof(float) * (size_t)B * Hkv * n_k, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ans_v, 0, sizeof(float) * (size_t)B * Hkv * n_k, st);
    return e == cudaSuccess ? ANTKV_OK : cuda_status(e, "anchor-score clear");
  }
  float *qs = nullptr, *kr = nullptr;
  cudaError_t e = scratch_alloc((void **)&qs, sizeof(float) * (size_t)B * Hq * n_q * d, st);
  if (e == cudaSuccess) e = scratch_alloc((void **)&kr, sizeof(float) * (size_t)B * Hkv * n_k * d, st);
  if (e != cudaSuccess) return cuda_status(e, "anchor-score scratch");
  int rc = rope_rotate(Q, dtype, q_positions, B, Hq, n_q, d, theta_base, 1.f / sqrtf((float)d),
                       qs, nullptr, st);
  if (rc == ANTKV_OK) rc = rope_rotate(K, dtype, k_positions, B, Hkv, n_k, d, theta_base, 1.f,
                                       kr, nullptr, st);
  for (int b = 0; b < B && rc == ANTKV_OK; ++b) {
    rc = launch_ans(qs + (size_t)b * Hq * n_q * d, kr + (size_t)b * Hkv * n_k * d,
                    M + (size_t)b * Hq * n_q, L + (size_t)b * Hq * n_q,
                    q_norms + (size_t)b * Hq * n_q, Hq, Hkv, Hq / Hkv, n_q, n_k, d, causal,
                    ans_k + (size_t)b * Hkv * n_k, ans_v + (size_t)b * Hkv * n_k, st);
  }
  cudaFreeAsync(qs, st);
  cudaFreeAsync(kr, st);
  return rc;
}

extern "C" int antkv_prefill_anchor_scores(const void *Q, const void *K, int dtype,
                                           const int64_t *positions, const float *M,
                                           const float *L, const float *q_norms, int B,
                                           int Hq, int Hkv, int n, int d, double theta_base,
                                           float *ans_k, float *ans_v, void *stream) {
  return antkv_prefill_anchor_scores_block(Q, K, dtype, positions, positions, M, L, q_norms, B,
                                           Hq, Hkv, n, n, d, theta_base, 1, ans_k, ans_v, stream);
}

extern "C" int antkv_prefill_attention_scores(const void *Q, const void *K, const void *V, int dtype,
                                              const int64_t *positions, int B, int Hq, int Hkv, int n,
                                              int d, double theta_base, float *O, float *M, float *L,
                                              float *q_norms, float *ans_k, float *ans_v, void *stream) {
  ANTKV_REQUIRE_ALIGNED16(Q, "Q");
  ANTKV_REQUIRE_ALIGNED16(K, "K");
  ANTKV_REQUIRE_ALIGNED16(V, "V");
  ANTKV_REQUIRE(d % 2 == 0, "head dimension must be even for RoPE");
  ANTKV_REQUIRE(theta_base > 0, "theta_base must be positive");
  ANTKV_REQUIRE(Hkv >= 1 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  int rc = prefill_tc_fused(Q, K, V, dtype, positions, B, Hq, Hkv, n, d, theta_base, O, M, L, q_norms,
                            ans_k, ans_v, as_stream(stream));
  if (rc != ANTKV_EUNSUPPORTED) return rc;
  rc = antkv_prefill_attention(Q, K, V, dtype, positions, B, Hq, Hkv, n, d, theta_base, O, M, L, q_norms,
                               stream);
  if (rc != ANTKV_OK) return rc;
  return antkv_prefill_anchor_scores(Q, K, dtype, positions, M, L, q_norms, B, Hq, Hkv, n, d, theta_base,
                                     ans_k, ans_v, stream);
}
