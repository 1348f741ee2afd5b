// Anchor selection (anchors.py:90-132) on the GPU.
//
// The reference ranks by lexsort((index, -score)) and takes prefixes.  Every
// policy reduces to "top-k SET" queries with ties to the lower index:
//   by_k   = topk(ans_k, B)
//   by_v   = topk(ans_v, B)
//   by_sum = S_K := topk(ans_k, B/2);  S_V := topk(ans_v restricted to the
//            complement of S_K, B - B/2)   (the V fill of anchors.py:112-119
//            walks the V ranking skipping S_K, which is exactly that set);
//            the K top-off (anchors.py:121-126) can never fire once the budget
//            is clipped to n.
// A top-k set is {key > T} plus the lowest-index elements with key == T,
// where T is found by an 8-bit radix select over the order-preserving
// uint32 image of the float scores.  The result is compacted in index order,
// i.e. already sorted (anchors.py:129).  One 1024-thread CTA per (b, head).
#include "common.cuh"

namespace antkv {

constexpr int SEL_THREADS = 1024;

struct SelShared {
  uint32_t hist[256];
  uint32_t scan[SEL_THREADS / 32];
  uint32_t prefix;
  uint32_t want;
  uint32_t total;
};

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total into sh.total.
__device__ uint32_t block_exclusive_scan(uint32_t v, SelShared &sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.scan[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = (lane < SEL_THREADS / 32) ? sh.scan[lane] : 0;
    uint32_t t = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < SEL_THREADS / 32) sh.scan[lane] = t - w;
    if (lane == 31) sh.total = t;
  }
  __syncthreads();
  uint32_t r = sh.scan[warp] + x - v;
  __syncthreads();
  return r;
}

// Select the top-k of `score` (excluding flag bit `excl_bit`), setting
// `set_bit` in flags for the chosen elements.
__device__ void topk_set(const float *__restrict__ score, uint8_t *flags, int n, int k,
                         uint8_t excl_bit, uint8_t set_bit, SelShared &sh) {
  if (k <= 0) return;
  // radix select of the k-th largest key
  uint32_t prefix = 0, mask = 0;
  uint32_t want = k;  // rank (1-based) of the threshold within the prefix class
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += SEL_THREADS) sh.hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += SEL_THREADS) {
      if (flags[i] & excl_bit) continue;
      uint32_t key = float_order_key(score[i]);
      if ((key & mask) == prefix) atomicAdd(&sh.hist[(key >> shift) & 0xFFu], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      int digit = 255;
      for (; digit > 0; --digit) {
        if (acc + sh.hist[digit] >= want) break;
        acc += sh.hist[digit];
      }
      sh.prefix = prefix | (static_cast<uint32_t>(digit) << shift);
      sh.want = want - acc;
    }
    __syncthreads();
    prefix = sh.prefix;
    want = sh.want;
    mask |= 0xFFu << shift;
    __syncthreads();
  }
  // prefix == threshold key T; `want` elements equal to T are needed, taken
  // in index order.  Each thread owns a contiguous index range.
  const int per = (n + SEL_THREADS - 1) / SEL_THREADS;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  uint32_t ties = 0;
  for (int i = lo; i < hi; ++i) {
    if (flags[i] & excl_bit) continue;
    if (float_order_key(score[i]) == prefix) ++ties;
  }
  uint32_t before = block_exclusive_scan(ties, sh);
  for (int i = lo; i < hi; ++i) {
    if (flags[i] & excl_bit) continue;
    uint32_t key = float_order_key(score[i]);
    if (key > prefix) {
      flags[i] |= set_bit;
    } else if (key == prefix) {
      if (before < want) flags[i] |= set_bit;
      ++before;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SEL_THREADS)
select_kernel(const float *__restrict__ ans_k, const float *__restrict__ ans_v, int n,
              int budget, int policy, uint8_t *__restrict__ flags_all,
              int32_t *__restrict__ anchors) {
  __shared__ SelShared sh;
  const int64_t bh = blockIdx.x;
  const float *sk = ans_k + bh * n;
  const float *sv = ans_v + bh * n;
  uint8_t *flags = flags_all + bh * n;
  for (int i = threadIdx.x; i < n; i += SEL_THREADS) flags[i] = 0;
  __syncthreads();
  if (policy == ANTKV_POLICY_BY_K) {
    topk_set(sk, flags, n, budget, 0, 1, sh);
  } else if (policy == ANTKV_POLICY_BY_V) {
    topk_set(sv, flags, n, budget, 0, 1, sh);
  } else {
    topk_set(sk, flags, n, budget / 2, 0, 1, sh);
    topk_set(sv, flags, n, budget - budget / 2, 1, 2, sh);
  }
  // compact chosen indices in ascending order
  const int per = (n + SEL_THREADS - 1) / SEL_THREADS;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  uint32_t cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += flags[i] ? 1u : 0u;
  uint32_t off = block_exclusive_scan(cnt, sh);
  int32_t *out = anchors + bh * budget;
  for (int i = lo; i < hi; ++i)
    if (flags[i]) out[off++] = i;
}

}  // namespace antkv

using namespace antkv;

extern "C" int antkv_select_anchors(const float *ans_k, const float *ans_v, int B, int Hkv,
                                    int n, int budget, int policy, int32_t *anchors,
                                    void *stream) {
  ANTKV_REQUIRE(policy >= 0 && policy <= 2, "unknown policy %d", policy);
  ANTKV_REQUIRE(budget >= 0 && budget <= n, "budget must be clipped to [0, n]");
  if ((int64_t)B * Hkv == 0 || budget == 0) return ANTKV_OK;
  cudaStream_t st = as_stream(stream);
  uint8_t *flags = nullptr;
  cudaError_t e = cudaMallocAsync(&flags, (size_t)B * Hkv * n, st);
  if (e != cudaSuccess) return cuda_status(e, "select scratch");
  select_kernel<<<B * Hkv, SEL_THREADS, 0, st>>>(ans_k, ans_v, n, budget, policy, flags, anchors);
  cudaError_t le = cudaGetLastError();
  cudaFreeAsync(flags, st);
  if (le != cudaSuccess) return cuda_status(le, "select_kernel");
  return ANTKV_OK;
}
