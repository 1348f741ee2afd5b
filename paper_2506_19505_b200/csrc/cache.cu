// Vector quantisation (encode / decode) and the quantised KV-cache state
// machine: build from prefill (cache.py:122-139), append (cache.py:157-166),
// evict with promotion or encoding (cache.py:180-193) and dequantise
// (cache.py:196-211).  All state lives on the device; every call is
// stream-ordered and capturable in a CUDA graph.
#include "common.cuh"

namespace antkv {

constexpr int ENC_THREADS = 256;
constexpr int ENC_CHUNK_FLOATS = 8192;  // 32 KB of centroids per smem stage

// Nearest centroid for one sub-vector held in registers: float32
// sum_t (x_t - c_t)^2 in index order, strict-< argmin (lowest index on ties,
// _ckernels.pyx:150-162).
template <int MAXD>
__device__ __forceinline__ void nearest_update(const float (&x)[MAXD], const float *c, int d_sub,
                                               int cidx, float &best, int &best_i) {
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < MAXD; ++t) {
    if (t < d_sub) {
      float df = x[t] - c[t];
      s = fmaf(df, df, s);
    }
  }
  if (s < best) {
    best = s;
    best_i = cidx;
  }
}

__device__ __forceinline__ void store_code(void *codes, int64_t off_elems, int code_bytes,
                                           int v) {
  if (code_bytes == 1) reinterpret_cast<uint8_t *>(codes)[off_elems] = static_cast<uint8_t>(v);
  else if (code_bytes == 2) reinterpret_cast<uint16_t *>(codes)[off_elems] = static_cast<uint16_t>(v);
  else if (code_bytes == 4) reinterpret_cast<int32_t *>(codes)[off_elems] = v;
  else reinterpret_cast<int64_t *>(codes)[off_elems] = v;
}

__device__ __forceinline__ int load_code(const void *codes, int64_t off_elems, int code_bytes) {
  if (code_bytes == 1) return reinterpret_cast<const uint8_t *>(codes)[off_elems];
  if (code_bytes == 2) return reinterpret_cast<const uint16_t *>(codes)[off_elems];
  if (code_bytes == 4) return reinterpret_cast<const int32_t *>(codes)[off_elems];
  return static_cast<int>(reinterpret_cast<const int64_t *>(codes)[off_elems]);
}

// Bulk encoder.  grid = (ceil(rows*groups / 256), nsets): each set s has its
// own input base (x_set_stride elements), output base (code_set_stride code
// elements) and codebook (set % cb_mod).  Output code for (row r, group g) is
// at codes[s*code_set_stride + (r/16)*code_tile_stride + (r%16)*code_row_stride
// + g] (plain row-major when code_tile_stride == 16*code_row_stride).
template <int MAXD>
__global__ void __launch_bounds__(ENC_THREADS)
vq_encode_kernel(const void *__restrict__ X, int dtype, int64_t rows, int d,
                 int64_t x_set_stride, const float *__restrict__ codebooks, int cb_mod,
                 int m, int d_sub, void *__restrict__ codes, int code_bytes,
                 int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                 float *__restrict__ d2out) {
  __shared__ float sC[ENC_CHUNK_FLOATS];
  const int groups = d / d_sub;
  const int set = blockIdx.y;
  const float *cb = codebooks + (int64_t)(set % cb_mod) * m * d_sub;
  const int64_t item = (int64_t)blockIdx.x * ENC_THREADS + threadIdx.x;
  const bool live = item < rows * groups;
  const int64_t r = live ? item / groups : 0;
  const int g = live ? static_cast<int>(item - r * groups) : 0;
  float x[MAXD];
  const int64_t xbase = set * x_set_stride + r * d + (int64_t)g * d_sub;
#pragma unroll
  for (int t = 0; t < MAXD; ++t) x[t] = (live && t < d_sub) ? load_elem(X, xbase + t, dtype) : 0.f;
  float best = INFINITY;
  int best_i = 0;
  const int chunk = (ENC_CHUNK_FLOATS / d_sub) < m ? (ENC_CHUNK_FLOATS / d_sub) : m;
  for (int c0 = 0; c0 < m; c0 += chunk) {
    const int cn = min(chunk, m - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * d_sub; i += ENC_THREADS) sC[i] = cb[(int64_t)c0 * d_sub + i];
    __syncthreads();
    if (live)
      for (int c = 0; c < cn; ++c) nearest_update<MAXD>(x, sC + c * d_sub, d_sub, c0 + c, best, best_i);
  }
  if (code_bytes == 3) {
    // 12-bit packed rows: lane g == 0 of each row gathers the row's codes
    // (a row's items are consecutive lanes; groups divide 32)
    uint32_t row_codes[32];
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < groups; ++k) row_codes[k] = __shfl_sync(0xffffffffu, (uint32_t)best_i, lane - g + k);
    if (live && g == 0)
      code_put_row(static_cast<uint8_t *>(codes), set * code_set_stride + (r >> 4) * code_tile_stride +
                   (r & 15) * code_row_stride, groups, row_codes, 3);
    if (live && d2out) d2out[set * rows * groups + item] = best;
    return;
  }
  if (live) {
    store_code(codes, set * code_set_stride + (r >> 4) * code_tile_stride + (r & 15) * code_row_stride + g,
               code_bytes, best_i);
    if (d2out) d2out[set * rows * groups + item] = best;
  }
}

int launch_encode_mma(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride,
                      int nsets, const float *codebooks, int cb_mod, int m, int d_sub,
                      void *codes, int code_bytes, int64_t code_set_stride,
                      int64_t code_tile_stride, int64_t code_row_stride, const float *d2,
                      cudaStream_t st);

int launch_encode_tc(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride, int nsets,
                     const float *codebooks, int cb_mod, int m, int d_sub, void *codes, int code_bytes,
                     int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                     const float *d2, cudaStream_t st);

int launch_encode_tc5(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride, int nsets,
                      const float *codebooks, int cb_mod, int m, int d_sub, void *codes, int code_bytes,
                      int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                      const float *d2, cudaStream_t st);

int launch_encode_tc5l(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride, int nsets,
                       const float *codebooks, int cb_mod, int m, int d_sub, void *codes, int code_bytes,
                       int64_t code_set_stride, int64_t code_tile_stride, int64_t code_row_stride,
                       const float *d2, cudaStream_t st);

int launch_encode(const void *X, int dtype, int64_t rows, int d, int64_t x_set_stride,
                  int nsets, const float *codebooks, int cb_mod, int m, int d_sub,
                  void *codes, int code_bytes, int64_t code_set_stride,
                  int64_t code_tile_stride, int64_t code_row_stride, float *d2, cudaStream_t st) {
  // d = 128, d_sub = 8, m <= 256, bf16 inputs: tcgen05 encoder (encode_tc5.cu)
  {
    const int rc = launch_encode_tc5(X, dtype, rows, d, x_set_stride, nsets, codebooks, cb_mod, m, d_sub,
                                     codes, code_bytes, code_set_stride, code_tile_stride, code_row_stride,
                                     d2, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
  }
  // ... fp16 inputs: mma.sync tensor-core encoder (encode_mma.cu)
  {
    const int rc = launch_encode_mma(X, dtype, rows, d, x_set_stride, nsets, codebooks, cb_mod, m,
                                     d_sub, codes, code_bytes, code_set_stride, code_tile_stride,
                                     code_row_stride, d2, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
  }
  // d_sub 16 / 32, any m, bf16 inputs: tcgen05 encoder over codebook blocks (encode_tc5.cu)
  {
    const int rc = launch_encode_tc5l(X, dtype, rows, d, x_set_stride, nsets, codebooks, cb_mod, m, d_sub,
                                      codes, code_bytes, code_set_stride, code_tile_stride, code_row_stride,
                                      d2, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
  }
  // d_sub 16 / 32 / 64, any m, 16-bit inputs: mma.sync tensor-core encoder (encode_tc.cu)
  {
    const int rc = launch_encode_tc(X, dtype, rows, d, x_set_stride, nsets, codebooks, cb_mod, m, d_sub,
                                    codes, code_bytes, code_set_stride, code_tile_stride, code_row_stride,
                                    d2, st);
    if (rc != ANTKV_EUNSUPPORTED) return rc;
  }
  ANTKV_REQUIRE(d_sub >= 1 && d_sub <= 64, "d_sub must be in [1, 64] on the GPU path");
  ANTKV_REQUIRE(d % d_sub == 0, "d=%d not divisible by d_sub=%d", d, d_sub);
  ANTKV_REQUIRE(m >= 1, "empty codebook");
  const int64_t items = rows * (d / d_sub);
  if (items == 0 || nsets == 0) return ANTKV_OK;
  dim3 grid(ceil_div(items, ENC_THREADS), nsets);
#define ENC_LAUNCH(MD)                                                                       \
  vq_encode_kernel<MD><<<grid, ENC_THREADS, 0, st>>>(X, dtype, rows, d, x_set_stride,        \
                                                     codebooks, cb_mod, m, d_sub, codes,     \
                                                     code_bytes, code_set_stride,            \
                                                     code_tile_stride, code_row_stride, d2)
  if (d_sub <= 2) ENC_LAUNCH(2);
  else if (d_sub <= 4) ENC_LAUNCH(4);
  else if (d_sub <= 8) ENC_LAUNCH(8);
  else if (d_sub <= 16) ENC_LAUNCH(16);
  else if (d_sub <= 32) ENC_LAUNCH(32);
  else ENC_LAUNCH(64);
#undef ENC_LAUNCH
  ANTKV_LAUNCH_CHECK("vq_encode_kernel");
  return ANTKV_OK;
}

__global__ void vq_decode_kernel(const void *__restrict__ codes, int code_bytes, int64_t rows,
                                 int groups, const float *__restrict__ cb, int m, int d_sub,
                                 float *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = rows * groups * d_sub;
  if (i >= total) return;
  const int t = static_cast<int>(i % d_sub);
  const int64_t rg = i / d_sub;
  int c = load_code(codes, rg, code_bytes);
  out[i] = (c >= 0 && c < m) ? cb[(int64_t)c * d_sub + t] : NAN;
}

// ------------------------------------------------------------ cache state
__device__ __forceinline__ int64_t bh_index(int b, int h, int H) { return (int64_t)b * H + h; }

// Per (b, head) layout from the sorted anchor list (cache.py:126-139):
// qmask, pool slots (anchors, then the window), free stack, head state.
// One CTA per (b, head); the codes were written by the bulk encoder, the
// pool rows and positions are copied by the launcher's next steps.
__global__ void cache_build_kernel(antkv_cache_desc c, int n, const int32_t *__restrict__ anchors,
                                   int anchor_stride) {
  const int b = blockIdx.x / c.Hkv, h = blockIdx.x % c.Hkv;
  const int64_t bh = bh_index(b, h, c.Hkv);
  const int32_t *anc = anchors + bh * anchor_stride;
  // Every step in parallel: the serial thread-0 loops this replaces ran one
  // dependent global round trip per anchor (~0.5 ms at 128K).
  // a list may end in -1 padding (sequence shards hold different anchor
  // counts per head); the valid prefix is sorted ascending
  constexpr int kWinWords = 64;                 // window-anchor bitmap (windows <= 2048)
  __shared__ int s_na, s_nw;
  __shared__ uint32_t s_winanc[kWinWords];
  const int wstart = n - c.window_size > 0 ? n - c.window_size : 0;
  const int W = n - wstart;                     // windowed-or-anchor tail tokens
  if (threadIdx.x == 0) s_na = 0;
  for (int i = threadIdx.x; i < kWinWords; i += blockDim.x) s_winanc[i] = 0u;
  __syncthreads();
  {
    int cnt = 0;
    for (int k = threadIdx.x; k < anchor_stride; k += blockDim.x) cnt += anc[k] >= 0 ? 1 : 0;
    if (cnt) atomicAdd(&s_na, cnt);
  }
  __syncthreads();
  const int n_anchors = s_na;
  uint32_t *qm = c.qmask + bh * (c.capacity / 32);
  // quantized bit = not anchor and j < n - window
  for (int w = threadIdx.x; w < c.capacity / 32; w += blockDim.x) {
    const int lo = w * 32;
    qm[w] = lo + 32 <= wstart ? 0xffffffffu : (lo >= wstart ? 0u : (1u << (wstart - lo)) - 1u);
  }
  __syncthreads();
  int32_t *ptok = c.pool_tok + bh * c.pool_capacity;
  int8_t *pkind = c.pool_kind + bh * c.pool_capacity;
  // pool: anchors first (ascending), then windowed tokens (ascending)
  for (int a = threadIdx.x; a < n_anchors; a += blockDim.x) {
    const int j = anc[a];
    if (j < wstart) atomicAnd(&qm[j / 32], ~(1u << (j % 32)));
    else if (W <= 32 * kWinWords) atomicOr(&s_winanc[(j - wstart) / 32], 1u << ((j - wstart) % 32));
    ptok[a] = j;
    pkind[a] = ANTKV_KIND_ANCHOR;
  }
  __syncthreads();
  int32_t *ring = c.win_ring + bh * (c.window_size + 1);
  if (threadIdx.x < 32) {           // warp 0: the tail tokens that are not anchors, in order
    const int lane = threadIdx.x;
    int off = 0;
    if (W <= 32 * kWinWords) {
      for (int base = 0; base < W; base += 32) {
        const int i = base + lane;
        const bool keep = i < W && !((s_winanc[i / 32] >> (i % 32)) & 1u);
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          const int pos = off + __popc(m & ((1u << lane) - 1u)), slot = n_anchors + pos;
          ptok[slot] = wstart + i;
          pkind[slot] = ANTKV_KIND_WINDOWED;
          ring[pos] = slot;
        }
        off += __popc(m);
      }
    } else if (lane == 0) {         // windows beyond the bitmap: the serial merge
      int ai = 0;
      for (int j = wstart; j < n; ++j) {
        while (ai < n_anchors && anc[ai] < j) ++ai;
        if (ai < n_anchors && anc[ai] == j) continue;
        ptok[n_anchors + off] = j;
        pkind[n_anchors + off] = ANTKV_KIND_WINDOWED;
        ring[off] = n_anchors + off;
        ++off;
      }
    }
    if (lane == 0) s_nw = off;
  }
  __syncthreads();
  const int nw = s_nw, used = n_anchors + nw;
  int32_t *fs = c.free_stack + bh * c.pool_capacity;
  for (int s2 = used + threadIdx.x; s2 < c.pool_capacity; s2 += blockDim.x) {
    ptok[s2] = -1;
    pkind[s2] = ANTKV_KIND_FREE;
    fs[c.pool_capacity - 1 - s2] = s2;         // the stack pops the lowest free slot first
  }
  if (threadIdx.x == 0) {
    int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
    hs[ANTKV_HS_ANCHORS] = n_anchors;
    hs[ANTKV_HS_WIN_HEAD] = 0;
    hs[ANTKV_HS_WIN_COUNT] = nw;
    hs[ANTKV_HS_FREE_TOP] = c.pool_capacity - used;
    hs[ANTKV_HS_POOL_HIGH] = used;
  }
  // (the rows themselves are copied by cache_pool_rows_kernel, one CTA per
  // pool slot: a loop here over the ~1300 slots of a 128K cache ran one
  // dependent global round trip per row, 1.3 ms)
  // (positions are copied by the launcher: one CTA copying 1 MB of them at
  // 128K took ~0.3 ms)
  if (h == 0 && threadIdx.x == 0) c.seq_len[b] = n;
}

// K / V rows of the used pool slots (after cache_build_kernel): slot = blockIdx.x.
__global__ void cache_pool_rows_kernel(antkv_cache_desc c, const void *__restrict__ K,
                                       const void *__restrict__ V, int dtype, int n) {
  const int slot = blockIdx.x;
  const int64_t bh = blockIdx.y;
  if (slot >= c.hstate[bh * ANTKV_HSTATE_WORDS + ANTKV_HS_POOL_HIGH]) return;
  const int j = c.pool_tok[bh * c.pool_capacity + slot];
  const int64_t src = (bh * n + j) * c.d;
  const int64_t dst = (bh * c.pool_capacity + slot) * 2 * c.d;
  for (int t = threadIdx.x; t < c.d; t += blockDim.x) {
    store_elem(c.pool_rows, dst + t, c.row_dtype, load_elem(K, src + t, dtype));
    store_elem(c.pool_rows, dst + c.d + t, c.row_dtype, load_elem(V, src + t, dtype));
  }
}

// Fast path: fp16 copy of pool row `slot` (K with RoPE applied at `pos`, V)
// in the tiled pool_f16 layout.
__device__ void write_pool_f16(const antkv_cache_desc &c, int64_t bh, int slot, int64_t pos) {
  if (!c.pool_f16) return;
  const int64_t src = (bh * c.pool_capacity + slot) * 2 * c.d;
  __half *dst = reinterpret_cast<__half *>(c.pool_f16) + bh * c.pool_capacity * 2 * c.d;
  for (int i = threadIdx.x; i < c.d / 2; i += blockDim.x) {
    const float x0 = load_elem(c.pool_rows, src + 2 * i, c.row_dtype);
    const float x1 = load_elem(c.pool_rows, src + 2 * i + 1, c.row_dtype);
    float cs, sn;
    rope_cs((double)pos * rope_freq(c.theta_base, i, c.d), cs, sn);
    dst[pool_f16_offset(slot, 0, 2 * i)] = __float2half_rn(x0 * cs - x1 * sn);
    dst[pool_f16_offset(slot, 0, 2 * i + 1)] = __float2half_rn(x0 * sn + x1 * cs);
  }
  for (int i = threadIdx.x; i < c.d; i += blockDim.x)
    dst[pool_f16_offset(slot, 1, i)] = __float2half_rn(load_elem(c.pool_rows, src + c.d + i, c.row_dtype));
}

// Fast path: pool_f16 rows for every live pool slot (after build / load).
__global__ void cache_pool_f16_kernel(antkv_cache_desc c) {
  const int64_t bh = blockIdx.y;
  const int b = static_cast<int>(bh / c.Hkv);
  const int s = blockIdx.x;
  const int tok = c.pool_tok[bh * c.pool_capacity + s];
  if (tok < 0 || c.pool_kind[bh * c.pool_capacity + s] == ANTKV_KIND_FREE) return;
  write_pool_f16(c, bh, s, c.positions[(int64_t)b * c.capacity + tok]);
}

// Append one token per sequence (cache.py:157-166).  One CTA per sequence;
// threads 0..Hkv-1 update the per-head state in parallel, then all threads
// copy the K/V rows of every head and (fast path) write the rotated K rows.
__global__ void cache_append_kernel(antkv_cache_desc c, const void *__restrict__ k,
                                    const void *__restrict__ v, int dtype,
                                    const int64_t *__restrict__ position) {
  const int b = blockIdx.x;
  const int j = c.seq_len[b];
  __shared__ int s_slot[256];
  for (int h = threadIdx.x; h < c.Hkv; h += blockDim.x) {
    const int64_t bh = bh_index(b, h, c.Hkv);
    int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
    const int top = hs[ANTKV_HS_FREE_TOP] - 1;
    const int slot = top >= 0 ? c.free_stack[bh * c.pool_capacity + top] : -1;
    if (slot >= 0) {
      hs[ANTKV_HS_FREE_TOP] = top;
      c.pool_tok[bh * c.pool_capacity + slot] = j;
      c.pool_kind[bh * c.pool_capacity + slot] = ANTKV_KIND_WINDOWED;
      int32_t *ring = c.win_ring + bh * (c.window_size + 1);
      ring[(hs[ANTKV_HS_WIN_HEAD] + hs[ANTKV_HS_WIN_COUNT]) % (c.window_size + 1)] = slot;
      hs[ANTKV_HS_WIN_COUNT] += 1;
      if (slot + 1 > hs[ANTKV_HS_POOL_HIGH]) hs[ANTKV_HS_POOL_HIGH] = slot + 1;
    }
    s_slot[h] = slot;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < c.Hkv * c.d; i += blockDim.x) {
    const int h = i / c.d, t = i % c.d;
    const int slot = s_slot[h];
    if (slot < 0) continue;
    const int64_t bh = bh_index(b, h, c.Hkv);
    const int64_t dst = (bh * c.pool_capacity + slot) * 2 * c.d;
    store_elem(c.pool_rows, dst + t, c.row_dtype, load_elem(k, bh * c.d + t, dtype));
    store_elem(c.pool_rows, dst + c.d + t, c.row_dtype, load_elem(v, bh * c.d + t, dtype));
  }
  if (c.pool_f16) {
    // from the inputs rounded to the pool's dtype (the values just stored):
    // no second round trip through pool_rows
    auto rnd = [&](float x) {
      return c.row_dtype == ANTKV_BF16 ? __bfloat162float(__float2bfloat16_rn(x))
             : c.row_dtype == ANTKV_F16 ? __half2float(__float2half_rn(x)) : x;
    };
    const double pos = static_cast<double>(position[b]);
    for (int i = threadIdx.x; i < c.Hkv * (c.d / 2); i += blockDim.x) {
      const int h = i / (c.d / 2), p = i % (c.d / 2);
      const int slot = s_slot[h];
      if (slot < 0) continue;
      const int64_t bh = bh_index(b, h, c.Hkv);
      const float x0 = rnd(load_elem(k, bh * c.d + 2 * p, dtype));
      const float x1 = rnd(load_elem(k, bh * c.d + 2 * p + 1, dtype));
      float cs, sn;
      const double om = (c.fast_tables && c.d == 128)
                            ? reinterpret_cast<const FastTables *>(c.fast_tables)->omega[p]
                            : rope_freq(c.theta_base, p, c.d);
      rope_cs(pos * om, cs, sn);
      __half *dst = reinterpret_cast<__half *>(c.pool_f16) + bh * c.pool_capacity * 2 * c.d;
      dst[pool_f16_offset(slot, 0, 2 * p)] = __float2half_rn(x0 * cs - x1 * sn);
      dst[pool_f16_offset(slot, 0, 2 * p + 1)] = __float2half_rn(x0 * sn + x1 * cs);
      dst[pool_f16_offset(slot, 1, 2 * p)] = __float2half_rn(rnd(load_elem(v, bh * c.d + 2 * p, dtype)));
      dst[pool_f16_offset(slot, 1, 2 * p + 1)] = __float2half_rn(rnd(load_elem(v, bh * c.d + 2 * p + 1, dtype)));
    }
  }
  // the slot's code bits stay clear (qmask initialised to zero above n)
  if (threadIdx.x == 0) {
    c.positions[(int64_t)b * c.capacity + j] = position[b];
    c.seq_len[b] = j + 1;
  }
}

// Evict (cache.py:180-193) in two launches so the encode of a long-codebook
// row spreads over many SMs: the oldest windowed row beyond window_size is
// promoted to an anchor while the budget allows, otherwise encoded.
// evict_plan() is the decision both launches derive from the unchanged state.
struct EvictPlan {
  int action;   // 0 none, 1 promote, 2 encode
  int slot;     // pool slot of the oldest windowed row
  int j;        // its token
};

__device__ __forceinline__ EvictPlan evict_plan(const antkv_cache_desc &c, int64_t bh, int b) {
  const int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
  EvictPlan p{0, -1, -1};
  if (hs[ANTKV_HS_WIN_COUNT] > c.window_size) {
    p.slot = c.win_ring[bh * (c.window_size + 1) + hs[ANTKV_HS_WIN_HEAD]];
    const int n = c.seq_len[b];
    const int budget = budget_for((int64_t)n + c.token_offset, c.anchor_count, c.anchor_fraction);
    p.action = hs[ANTKV_HS_ANCHORS] < budget ? 1 : 2;
    p.j = c.pool_tok[bh * c.pool_capacity + p.slot];
  }
  return p;
}

// Launch 1: CTA (b*Hkv + h, unit, slice) scans 512 centroids of sub-vector
// `unit` = (kv, group) of the evicted row when the plan says so, and folds
// its minimum into evict_scratch with a 64-bit atomicMin of (distance bits
// << 32 | index): distances are >= 0, so the packed order is the distance
// order with the lower index on ties — the strict-< scan of
// _ckernels.pyx:150-162.  For d_sub = 2^k >= 4 a centroid is read by
// LPC = min(32, d_sub / 4) adjacent lanes (one float4 each per pass, so a
// warp load covers contiguous centroids); float32 distances.
constexpr int kEvictSlice = 512;

__global__ void __launch_bounds__(256)
cache_evict_encode_kernel(antkv_cache_desc c) {
  __shared__ float sx[256];
  __shared__ unsigned long long s_key[8];
  const int b = blockIdx.x / c.Hkv, h = blockIdx.x % c.Hkv;
  const int64_t bh = bh_index(b, h, c.Hkv);
  const EvictPlan p = evict_plan(c, bh, b);
  if (p.action != 2) return;
  const int unit = blockIdx.y, kv = unit / c.groups, g = unit % c.groups;
  const int ds = c.d_sub;
  const int m0 = blockIdx.z * kEvictSlice, m1 = min(c.m, m0 + kEvictSlice);
  const int64_t row = (bh * c.pool_capacity + p.slot) * 2 * c.d + kv * c.d + g * ds;
  for (int i = threadIdx.x; i < ds; i += blockDim.x) sx[i] = load_elem(c.pool_rows, row + i, c.row_dtype);
  __syncthreads();
  const float *cb = (kv ? c.codebook_v : c.codebook_k) + (int64_t)h * c.m * ds;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float best = INFINITY;
  int best_i = 0x7fffffff;
  if (ds >= 4 && (ds & (ds - 1)) == 0) {   // power of two: lanes per centroid divide the warp
    const int lpc = min(32, ds >> 2);
    const int cpw = 32 / lpc;                    // centroids per warp pass
    const int sub = lane % lpc, ci0 = lane / lpc;
    const int nq = ds >> 2;                      // float4s per centroid
    constexpr int U = 4;                         // passes with their loads in flight together
    for (int base = m0 + warp * cpw; base < m1; base += 8 * cpw * U) {
      float part[U];
#pragma unroll
      for (int u = 0; u < U; ++u) part[u] = 0.f;
      for (int q = sub; q < nq; q += lpc) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ci = base + u * 8 * cpw + ci0;
          v[u] = ci < m1 ? __ldg(reinterpret_cast<const float4 *>(cb + (int64_t)ci * ds) + q)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const float x0 = sx[4 * q], x1 = sx[4 * q + 1], x2 = sx[4 * q + 2], x3 = sx[4 * q + 3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float df = x0 - v[u].x; part[u] = fmaf(df, df, part[u]);
          df = x1 - v[u].y; part[u] = fmaf(df, df, part[u]);
          df = x2 - v[u].z; part[u] = fmaf(df, df, part[u]);
          df = x3 - v[u].w; part[u] = fmaf(df, df, part[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        for (int off = lpc >> 1; off > 0; off >>= 1) part[u] += __shfl_down_sync(0xffffffffu, part[u], off, lpc);
        const int ci = base + u * 8 * cpw + ci0;
        if (sub == 0 && ci < m1 && part[u] < best) { best = part[u]; best_i = ci; }
      }
    }
  } else {
    for (int ci = m0 + threadIdx.x; ci < m1; ci += blockDim.x) {
      float s = 0.f;
      for (int t = 0; t < ds; ++t) {
        const float df = sx[t] - cb[(int64_t)ci * ds + t];
        s = fmaf(df, df, s);
      }
      if (s < best) { best = s; best_i = ci; }
    }
  }
  unsigned long long key = best_i == 0x7fffffff
      ? ~0ull : ((unsigned long long)__float_as_uint(best) << 32) | (unsigned)best_i;
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, key, off);
    key = o < key ? o : key;
  }
  if (lane == 0) s_key[warp] = key;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) key = s_key[w] < key ? s_key[w] : key;
    atomicMin(c.evict_scratch + bh * 2 * c.groups + unit, key);
  }
}

// Launch 2: one thread per (b, head) applies the plan to the state words.
__global__ void cache_evict_commit_kernel(antkv_cache_desc c) {
  const int64_t bh = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (bh >= (int64_t)c.B * c.Hkv) return;
  const int b = static_cast<int>(bh / c.Hkv);
  const EvictPlan p = evict_plan(c, bh, b);
  if (p.action == 0) return;
  int32_t *hs = c.hstate + bh * ANTKV_HSTATE_WORDS;
  hs[ANTKV_HS_WIN_HEAD] = (hs[ANTKV_HS_WIN_HEAD] + 1) % (c.window_size + 1);
  hs[ANTKV_HS_WIN_COUNT] -= 1;
  if (p.action == 1) {
    c.pool_kind[bh * c.pool_capacity + p.slot] = ANTKV_KIND_ANCHOR;
    hs[ANTKV_HS_ANCHORS] += 1;
  } else {
    unsigned long long *sk = c.evict_scratch + bh * 2 * c.groups;
    uint32_t row[128];
    for (int kv = 0; kv < 2; ++kv) {   // the encoder's minima -> the code rows; reset the slots
      for (int g = 0; g < c.groups; ++g) {
        row[g] = static_cast<uint32_t>(sk[kv * c.groups + g] & 0xffffffffu);
        sk[kv * c.groups + g] = ~0ull;
      }
      code_put_row(c.codes, bh * c.capacity * 2 * c.groups + code_offset(p.j, kv, 0, c.groups), c.groups, row,
                   c.code_bytes);
    }
    atomicOr(&c.qmask[bh * (c.capacity / 32) + p.j / 32], 1u << (p.j % 32));
    c.pool_kind[bh * c.pool_capacity + p.slot] = ANTKV_KIND_FREE;
    c.pool_tok[bh * c.pool_capacity + p.slot] = -1;
    c.free_stack[bh * c.pool_capacity + hs[ANTKV_HS_FREE_TOP]] = p.slot;
    hs[ANTKV_HS_FREE_TOP] += 1;
  }
}

// Dequantise: codes for quantized slots, pool rows scattered to their tokens.
__global__ void cache_dequant_codes_kernel(antkv_cache_desc c, int n, float *__restrict__ Khat,
                                           float *__restrict__ Vhat) {
  const int64_t bh = blockIdx.y;
  const int h = static_cast<int>(bh % c.Hkv);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * c.d) return;
  const int j = static_cast<int>(i / c.d), t = static_cast<int>(i % c.d);
  const uint32_t bits = c.qmask[bh * (c.capacity / 32) + j / 32];
  float kv = NAN, vv = NAN;
  if (bits & (1u << (j % 32))) {
    const int g = t / c.d_sub, e = t % c.d_sub;
    const int64_t hb = bh * c.capacity * 2 * c.groups;
    const int64_t ok = hb + code_offset(j, 0, g, c.groups), ov = hb + code_offset(j, 1, g, c.groups);
    const int ck = code_get(c.codes, ok, c.code_bytes), cv = code_get(c.codes, ov, c.code_bytes);
    kv = c.codebook_k[((int64_t)h * c.m + ck) * c.d_sub + e];
    vv = c.codebook_v[((int64_t)h * c.m + cv) * c.d_sub + e];
  }
  Khat[(bh * n + j) * c.d + t] = kv;
  Vhat[(bh * n + j) * c.d + t] = vv;
}

__global__ void cache_dequant_pool_kernel(antkv_cache_desc c, int n, float *__restrict__ Khat,
                                          float *__restrict__ Vhat) {
  const int64_t bh = blockIdx.y;
  const int s = blockIdx.x;
  const int j = c.pool_tok[bh * c.pool_capacity + s];
  if (j < 0 || j >= n || c.pool_kind[bh * c.pool_capacity + s] == ANTKV_KIND_FREE) return;
  const int64_t row = (bh * c.pool_capacity + s) * 2 * c.d;
  for (int t = threadIdx.x; t < c.d; t += blockDim.x) {
    Khat[(bh * n + j) * c.d + t] = load_elem(c.pool_rows, row + t, c.row_dtype);
    Vhat[(bh * n + j) * c.d + t] = load_elem(c.pool_rows, row + c.d + t, c.row_dtype);
  }
}

// Fast-path codebook: fp16 [Hkv][256][K 8 | V 8] (zero rows beyond m) at
// the start of each head's 64 KB block (the fused kernel replicates each row
// into the 8 16-byte bank groups of its shared copy).
// Block (Hkv*2) also writes the RoPE constant tables (FastTables).
__global__ void cache_prepare_fast_kernel(antkv_cache_desc c) {
  if (blockIdx.x == gridDim.x - 1) {
    fill_fast_tables(reinterpret_cast<FastTables *>(c.fast_tables), c.theta_base);
    return;
  }
  // compact fp16 rows [code][K 8 | V 8] (32 B) at the start of the head's
  // 64 KB block; decode_fast_kernel replicates them in shared memory
  const int h = blockIdx.x / 2, kv = blockIdx.x % 2;
  const float *cb = (kv ? c.codebook_v : c.codebook_k) + (int64_t)h * c.m * c.d_sub;
  __half *dst = reinterpret_cast<__half *>(c.codebook_f16) + (int64_t)h * 256 * 128 + kv * 8;
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    const int code = i / 8, t = i % 8;
    dst[code * 16 + t] = __float2half_rn(code < c.m ? cb[(int64_t)code * 8 + t] : 0.f);
  }
}

}  // namespace antkv

using namespace antkv;

static int check_desc(const antkv_cache_desc *c) {
  ANTKV_REQUIRE(c != nullptr, "null cache descriptor");
  ANTKV_REQUIRE(c->B >= 1 && c->Hkv >= 1 && c->Hq % c->Hkv == 0, "bad head counts");
  ANTKV_REQUIRE(c->d >= 2 && c->d % 2 == 0 && c->d <= 256, "head dimension must be even and <= 256");
  ANTKV_REQUIRE(c->d_sub >= 1 && c->d % c->d_sub == 0, "d=%d not divisible by d_sub=%d", c->d, c->d_sub);
  ANTKV_REQUIRE(c->groups == c->d / c->d_sub, "groups mismatch");
  ANTKV_REQUIRE(c->code_bytes == (c->index_bits <= 8 ? 1 : 2) ||
                    (c->code_bytes == 3 && c->index_bits <= 12 && c->groups >= 2 && c->groups <= 32 &&
                     (c->groups & (c->groups - 1)) == 0),
                "code_bytes mismatch");
  ANTKV_REQUIRE(c->index_bits <= 16, "index_bits > 16 unsupported");
  ANTKV_REQUIRE(c->row_dtype == ANTKV_BF16 || c->row_dtype == ANTKV_F16 || c->row_dtype == ANTKV_F32,
                "bad row dtype");
  ANTKV_REQUIRE(c->groups <= 128, "more than 128 sub-vectors per row unsupported");
  ANTKV_REQUIRE(c->capacity % 32 == 0 && c->capacity > 0, "capacity must be a positive multiple of 32");
  ANTKV_REQUIRE(c->window_size >= 0 && c->pool_capacity > c->window_size, "pool too small");
  return ANTKV_OK;
}

extern "C" int antkv_assign_nearest(const float *X, const float *C, int64_t n, int m, int d_sub,
                                    int64_t *idx, float *d2, void *stream) {
  return launch_encode(X, ANTKV_F32, n, d_sub, 0, 1, C, 1, m, d_sub, idx, 8, 0, 16, 1, d2,
                       as_stream(stream));
}

extern "C" int antkv_vq_encode(const void *X, int dtype, int64_t rows, int d,
                               const float *codebook, int m, int d_sub, void *codes,
                               int code_bytes, void *stream) {
  ANTKV_REQUIRE(code_bytes == 1 || code_bytes == 2 || code_bytes == 4 || code_bytes == 8,
                "code_bytes must be 1, 2, 4 or 8");
  ANTKV_REQUIRE(code_bytes >= 8 || m <= (1 << (8 * code_bytes)), "codes do not fit");
  ANTKV_REQUIRE_ALIGNED16(X, "X");
  return launch_encode(X, dtype, rows, d, 0, 1, codebook, 1, m, d_sub, codes, code_bytes, 0,
                       16 * (d / d_sub), d / d_sub, nullptr, as_stream(stream));
}

extern "C" int antkv_vq_decode(const void *codes, int code_bytes, int64_t rows, int groups,
                               const float *codebook, int m, int d_sub, float *out,
                               void *stream) {
  int64_t total = rows * groups * d_sub;
  if (total == 0) return ANTKV_OK;
  vq_decode_kernel<<<ceil_div(total, 256), 256, 0, as_stream(stream)>>>(
      codes, code_bytes, rows, groups, codebook, m, d_sub, out);
  ANTKV_LAUNCH_CHECK("vq_decode_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_cache_build(const antkv_cache_desc *c, const void *K, const void *V,
                                 int dtype, const int64_t *positions, int n,
                                 const int32_t *anchors, int n_anchors, void *stream) {
  int rc = check_desc(c);
  if (rc) return rc;
  previous_cache_on_stream(as_stream(stream), c->codes);   // this stream now touched c
  ANTKV_REQUIRE(n >= 0 && n <= c->capacity, "prefill length exceeds capacity");
  ANTKV_REQUIRE_ALIGNED16(K, "K");
  ANTKV_REQUIRE_ALIGNED16(V, "V");
  ANTKV_REQUIRE(n_anchors + c->window_size + 1 <= c->pool_capacity, "pool capacity too small");
  cudaStream_t st = as_stream(stream);
  const int nsets = c->B * c->Hkv;
  const int G = c->groups;
  // tiled layout: set stride = capacity*2G units, tile stride 32G, row stride G;
  // V codes start 16G units into each tile
  rc = launch_encode(K, dtype, n, c->d, (int64_t)n * c->d, nsets, c->codebook_k, c->Hkv, c->m,
                     c->d_sub, c->codes, c->code_bytes, (int64_t)c->capacity * 2 * G, 32 * G, G,
                     nullptr, st);
  if (rc) return rc;
  rc = launch_encode(V, dtype, n, c->d, (int64_t)n * c->d, nsets, c->codebook_v, c->Hkv, c->m,
                     c->d_sub, c->codes + code_stream_bytes(16 * G, c->code_bytes), c->code_bytes,
                     (int64_t)c->capacity * 2 * G, 32 * G, G, nullptr, st);
  if (rc) return rc;
  cache_build_kernel<<<nsets, 256, 0, st>>>(*c, n, anchors, n_anchors);
  ANTKV_LAUNCH_CHECK("cache_build_kernel");
  cache_pool_rows_kernel<<<dim3(c->pool_capacity, nsets), 128, 0, st>>>(*c, K, V, dtype, n);
  ANTKV_LAUNCH_CHECK("cache_pool_rows_kernel");
  if (n > 0) {   // positions [B][n] -> [B][capacity]
    const cudaError_t e = cudaMemcpy2DAsync(c->positions, (size_t)c->capacity * sizeof(int64_t), positions,
                                            (size_t)n * sizeof(int64_t), (size_t)n * sizeof(int64_t), c->B,
                                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "positions copy");
  }
  if (c->pool_f16) {
    cache_pool_f16_kernel<<<dim3(c->pool_capacity, nsets), 64, 0, st>>>(*c);
    ANTKV_LAUNCH_CHECK("cache_pool_f16_kernel");
  }
  return ANTKV_OK;
}

extern "C" int antkv_cache_append(const antkv_cache_desc *c, const void *k, const void *v,
                                  int dtype, const int64_t *position, void *stream) {
  int rc = check_desc(c);
  if (rc) return rc;
  previous_cache_on_stream(as_stream(stream), c->codes);   // this stream now touched c
  ANTKV_REQUIRE(c->Hkv <= 256, "at most 256 KV heads");
  cache_append_kernel<<<c->B, 256, 0, as_stream(stream)>>>(*c, k, v, dtype, position);
  ANTKV_LAUNCH_CHECK("cache_append_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_cache_evict(const antkv_cache_desc *c, void *stream) {
  int rc = check_desc(c);
  if (rc) return rc;
  previous_cache_on_stream(as_stream(stream), c->codes);   // this stream now touched c
  ANTKV_REQUIRE(c->d_sub <= 256, "d_sub > 256 unsupported by the eviction encoder");
  cudaStream_t st = as_stream(stream);
  ANTKV_REQUIRE(c->evict_scratch != nullptr, "evict_scratch not allocated");
  cache_evict_encode_kernel<<<dim3(c->B * c->Hkv, 2 * c->groups, (c->m + kEvictSlice - 1) / kEvictSlice), 256, 0,
                              st>>>(*c);
  ANTKV_LAUNCH_CHECK("cache_evict_encode_kernel");
  const int nbh = c->B * c->Hkv;
  cache_evict_commit_kernel<<<(nbh + 127) / 128, 128, 0, st>>>(*c);
  ANTKV_LAUNCH_CHECK("cache_evict_commit_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_cache_dequantize(const antkv_cache_desc *c, int n, float *Khat, float *Vhat,
                                      void *stream) {
  int rc = check_desc(c);
  if (rc) return rc;
  previous_cache_on_stream(as_stream(stream), c->codes);   // this stream now touched c
  if (n == 0) return ANTKV_OK;
  cudaStream_t st = as_stream(stream);
  dim3 g1(ceil_div((int64_t)n * c->d, 256), c->B * c->Hkv);
  cache_dequant_codes_kernel<<<g1, 256, 0, st>>>(*c, n, Khat, Vhat);
  ANTKV_LAUNCH_CHECK("cache_dequant_codes_kernel");
  dim3 g2(c->pool_capacity, c->B * c->Hkv);
  cache_dequant_pool_kernel<<<g2, 128, 0, st>>>(*c, n, Khat, Vhat);
  ANTKV_LAUNCH_CHECK("cache_dequant_pool_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_cache_prepare_fast(const antkv_cache_desc *c, void *stream) {
  int rc = check_desc(c);
  if (rc) return rc;
  previous_cache_on_stream(as_stream(stream), c->codes);   // this stream now touched c
  ANTKV_REQUIRE(c->d == 128 && c->d_sub == 8 && c->m <= 256 && c->codebook_f16 && c->fast_tables,
                "fast path needs d=128, d_sub=8, m<=256");
  cudaStream_t st = as_stream(stream);
  cache_prepare_fast_kernel<<<c->Hkv * 2 + 1, 256, 0, st>>>(*c);
  ANTKV_LAUNCH_CHECK("cache_prepare_fast_kernel");
  if (c->pool_f16) {
    ANTKV_REQUIRE(c->pool_capacity % 16 == 0, "pool_capacity must be a multiple of 16");
    cache_pool_f16_kernel<<<dim3(c->pool_capacity, c->B * c->Hkv), 64, 0, st>>>(*c);
    ANTKV_LAUNCH_CHECK("cache_pool_f16_kernel");
  }
  return ANTKV_OK;
}
