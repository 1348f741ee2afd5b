// Shared helpers for the AnTKV B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/antkv_b200.h"

namespace antkv {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *where);

// Row / tile inputs are read with 16-byte vector loads and bulk copies.
#define ANTKV_REQUIRE_ALIGNED16(ptr, name) \
  ANTKV_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, name " must be 16-byte aligned")
#define ANTKV_REQUIRE(cond, ...)                                              \
  do {                                                                        \
    if (!(cond)) {                                                            \
      ::antkv::set_error(__VA_ARGS__);                                        \
      return ANTKV_EINVAL;                                                    \
    }                                                                         \
  } while (0)

#define ANTKV_LAUNCH_CHECK(where)                                             \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) return ::antkv::cuda_status(_e, where);            \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// The cache (identified by its codes buffer) touched by the last library
// launch on `st`; records `key` as the new one.  The fused decode kernel reads
// cache state before griddepcontrol.wait only when the previous launch on the
// stream was for another cache.
const void *previous_cache_on_stream(cudaStream_t st, const void *key);
void record_fast_outputs(cudaStream_t st, const void *out, int64_t out_bytes, const void *lse, int64_t lse_bytes);
bool overlaps_previous_fast_outputs(cudaStream_t st, const void *p, int64_t bytes);
bool stream_exclusive(cudaStream_t st);

// Destinations of a sequence shard's partial (o, lse): n receive buffers
// (device arrays of n base pointers, one per peer; this rank's slot is
// `rank`: o [P][rows][d], lse [P][rows], flags [P]) and the release value.
struct PublishArgs {
  float *const *o;
  float *const *lse;
  unsigned *const *flag;
  int n, rank;
  int64_t rows;
  int *cnt;        // device counter of finished heads / rows (self-resetting)
  unsigned seq;
};

// Stream-ordered scratch (cudaMallocAsync from the device's default pool).
// The first call per device raises the pool's release threshold so freed
// scratch stays mapped for the next call instead of being returned to the
// driver at every synchronisation (re-mapping GBs costs milliseconds).
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st);

// ---------------------------------------------------------------- dtypes
__device__ __forceinline__ float load_elem(const void *p, int64_t i, int dtype) {
  if (dtype == ANTKV_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i]);
  if (dtype == ANTKV_F16) return __half2float(reinterpret_cast<const __half *>(p)[i]);
  return reinterpret_cast<const float *>(p)[i];
}

__device__ __forceinline__ void store_elem(void *p, int64_t i, int dtype, float v) {
  if (dtype == ANTKV_BF16) reinterpret_cast<__nv_bfloat16 *>(p)[i] = __float2bfloat16_rn(v);
  else if (dtype == ANTKV_F16) reinterpret_cast<__half *>(p)[i] = __float2half_rn(v);
  else reinterpret_cast<float *>(p)[i] = v;
}

__host__ __device__ inline int dtype_size(int dtype) { return dtype == ANTKV_F32 ? 4 : 2; }

__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

__device__ __forceinline__ uint16_t float_to_bf16_bits(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t *>(&h);
}

// ---------------------------------------------------------------- RoPE
// Frequencies theta^(-2i/d) in float64 (attention.py:84).
__device__ __forceinline__ double rope_freq(double theta, int i, int d) {
  return pow(theta, -2.0 * (double)i / (double)d);
}

// cos/sin of pos*freq, angle formed in float64 and reduced mod 2*pi before a
// float32 sincos (SURVEY.md §7 hard part 4: fp32 angles are off by ~4e-3 rad
// at 128K; this keeps the error near 1e-7 rad).
__device__ __forceinline__ void rope_cs(double angle, float &c, float &s) {
  const double two_pi = 6.283185307179586476925286766559;
  double k = rint(angle * (1.0 / two_pi));
  double r = fma(-k, two_pi, angle);
  r = fma(-k, 2.4492935982947064e-16, r);  // low part of 2*pi
  // |r| <= pi: the hardware approximation is accurate to ~1e-6 absolute here
  __sincosf(static_cast<float>(r), &s, &c);
}

// ---------------------------------------------------------------- ordering
// Order-preserving map float -> uint32 (larger float -> larger key).
__device__ __forceinline__ uint32_t float_order_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Code layout inside one (sequence, head): tiles of 16 slots, each tile
// [K codes 16 x G][V codes 16 x G] in code units (1 or 2 bytes), so the K (or
// V) codes of a tile are one contiguous 16*G-unit block (coalesced / TMA).
__host__ __device__ __forceinline__ int64_t code_offset(int64_t slot, int kv, int g, int G) {
  return (slot >> 4) * (32 * (int64_t)G) + kv * (16 * G) + (slot & 15) * G + g;
}

// Cache code units (antkv_cache_desc::code_bytes): 1 byte, 2 bytes, or 3 =
// 12-bit indices packed two per three bytes (unit u at bits [12u, 12u + 12)
// of the byte stream, little-endian).  Rows hold an even number of groups
// when packed, so every row starts on a byte and is written whole.
__host__ __device__ __forceinline__ int64_t code_stream_bytes(int64_t units, int cb) {
  return cb == 3 ? units * 3 / 2 : units * cb;
}
__device__ __forceinline__ uint32_t code_get(const uint8_t *base, int64_t unit, int cb) {
  if (cb == 1) return base[unit];
  if (cb == 2) return reinterpret_cast<const uint16_t *>(base)[unit];
  const int64_t bit = 12 * unit;
  const uint8_t *p = base + (bit >> 3);
  const uint32_t v = p[0] | ((uint32_t)p[1] << 8);
  return (v >> (bit & 7)) & 0xfffu;
}
// The G codes of one row: units unit0 .. unit0 + G - 1 (unit0 a multiple of G).
__device__ __forceinline__ void code_put_row(uint8_t *base, int64_t unit0, int G, const uint32_t *v, int cb) {
  if (cb == 1) {
    for (int g = 0; g < G; ++g) base[unit0 + g] = static_cast<uint8_t>(v[g]);
  } else if (cb == 2) {
    for (int g = 0; g < G; ++g) reinterpret_cast<uint16_t *>(base)[unit0 + g] = static_cast<uint16_t>(v[g]);
  } else {
    uint8_t *p = base + (12 * unit0 >> 3);
    for (int g = 0; g + 1 < G; g += 2, p += 3) {
      p[0] = static_cast<uint8_t>(v[g]);
      p[1] = static_cast<uint8_t>(((v[g] >> 8) & 0xfu) | ((v[g + 1] & 0xfu) << 4));
      p[2] = static_cast<uint8_t>(v[g + 1] >> 4);
    }
  }
}

// Fast-path pool tile layout (antkv_cache_desc::pool_f16), in halves from the
// (sequence, head) base: 16-slot tiles of [K rotated | V][16 slots][128], the
// 16-byte chunk c of slot r stored at chunk c ^ (r & 7) so the eight row
// addresses of an ldmatrix phase fall into distinct bank groups.
__host__ __device__ __forceinline__ int64_t pool_f16_offset(int slot, int kv, int dim) {
  const int r = slot & 15;
  return (int64_t)(slot >> 4) * 4096 + kv * 2048 + r * 128 + ((((dim >> 3) ^ (r & 7))) << 3) +
         (dim & 7);
}

// Fast-path RoPE constants for d = 128 (antkv_cache_desc::fast_tables).
struct FastTables {
  // fp16x2 {(cos, sin), (-sin, cos)} of r * omega_p for rows r = g and g + 8
  // and pair p = 8 s + 4 u + t, laid out [s][u][t][g] as one 16-byte record
  // {row g: (c,s), (-s,c); row g+8: (c,s), (-s,c)}: the 32 lanes (g = lane / 4,
  // t = lane % 4) of a warp read 512 consecutive bytes with one LDS.128
  uint4 kc[8][2][4][8];
  // cos, sin of -32 * omega_p (frame advance per stage) for pairs p = 8 s + 4 u + t:
  // step[s][t] = (c_{u=0}, s_{u=0}, c_{u=1}, s_{u=1})
  float4 step[8][4];
  double omega[64];        // theta^(-2i/128)
  uint64_t turns[64];      // omega_i / (2 pi) in units of 2^-64 turns
};

// Fills the RoPE constant tables for d = 128 (one block; any blockDim).
__device__ __forceinline__ void fill_fast_tables(FastTables *tab, double theta) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    const double om = rope_freq(theta, i, 128);
    tab->omega[i] = om;
    tab->turns[i] = __double2ull_rn(om * 0.15915494309189535 * 18446744073709551616.0);
    float cs, sn;
    rope_cs(-32.0 * om, cs, sn);
    float *st = reinterpret_cast<float *>(&tab->step[i >> 3][i & 3]) + 2 * ((i >> 2) & 1);
    st[0] = cs;
    st[1] = sn;
    for (int r = 0; r < 16; ++r) {
      rope_cs((double)r * om, cs, sn);
      __half2 a = __floats2half2_rn(cs, sn), b = __floats2half2_rn(-sn, cs);
      uint4 &k = tab->kc[i >> 3][(i >> 2) & 1][i & 3][r & 7];
      (r < 8 ? k.x : k.z) = *reinterpret_cast<uint32_t *>(&a);
      (r < 8 ? k.y : k.w) = *reinterpret_cast<uint32_t *>(&b);
    }
  }
}

// cos/sin of delta * omega for an integer position difference, reduced
// exactly in integer arithmetic: delta * turns mod 2^64 is the fractional
// number of turns (error ~ |delta| * 2^-53 relative turns, < 1e-9 rad).
__device__ __forceinline__ void turns_cs(int64_t delta, uint64_t turns, float &c, float &s) {
  const uint64_t p = static_cast<uint64_t>(delta) * turns;
  const float a = static_cast<float>(static_cast<int64_t>(p)) * 3.4061215800865545e-19f;  // 2pi/2^64
  __sincosf(a, &s, &c);
}
static_assert(sizeof(FastTables) <= 16384, "fast tables");

// Ints per (sequence, head) of the fused decode kernel's cache-update plan
// (decode workspace, after the CTA / sequence tickets).
constexpr int kPlanWords = 12;

// Position of pair p = 8 s + 4 u + t in the fast kernel's lane order
// ((s, t) major, u minor): a lane's two pairs of k-step s are adjacent.
__host__ __device__ __forceinline__ int lane_pair_pos(int p) {
  return ((p >> 3) * 4 + (p & 3)) * 2 + ((p >> 2) & 1);
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// budget_for(n) (cache.py:54-57), evaluated with the same float64 product.
__host__ __device__ inline int budget_for(int64_t n, int anchor_count, double frac) {
  if (anchor_count >= 0) return static_cast<int>(anchor_count < n ? anchor_count : n);
  double b = ceil(frac * static_cast<double>(n));
  if (b < 0) b = 0;
  if (b > static_cast<double>(n)) b = static_cast<double>(n);
  return static_cast<int>(b);
}

}  // namespace antkv
