// Weighted k-means (Lloyd) for codebook training, vq.py:141-214 (SURVEY.md
// §8f rank 3), in float64 with the reference's exact operation order so the
// GPU result is the reference's bit for bit:
//
//  * assignment (kernels.assign_nearest, _ckernels.pyx:134-163):
//    s = sum_t (x_t - c_t)^2 accumulated over t in order, each product and
//    sum rounded separately (no FMA contraction: __dmul_rn/__dadd_rn), strict
//    `<` over centroids in index order (ties -> lowest index);
//  * update (vq.py:187-192): per cluster, sum_j w_j * x_j and sum_j w_j over
//    the members in ascending point order (what np.add.at / np.bincount do),
//    then csum / wsum for live clusters.  The rows come in that order from a
//    stable sort of the assignment (gathered once, so each cluster's rows
//    are contiguous); each (cluster, coordinate) sum runs as one sequential
//    chain, which is what makes the rounding identical.
//
// The k-means++ seeding, the empty-cluster repair and the stopping rule stay
// in the host driver (vq.py weighted_kmeans); they are O(m) decisions.
#include "common.cuh"

namespace antkv {

constexpr int KM_THREADS = 256;
constexpr int KM_SMEM_DOUBLES = 6144;  // 48 KB of centroids per chunk

// D > 0: the exact sub-vector length (fully unrolled, vector shared loads);
// D == 0: any d <= MAXD.
template <int D, int MAXD>
__global__ void __launch_bounds__(KM_THREADS)
kmeans_assign_f64_kernel(const double *__restrict__ X, const double *__restrict__ C, int64_t n,
                         int m, int d_rt, int64_t *__restrict__ idx, double *__restrict__ d2) {
  extern __shared__ __align__(16) double sc[];
  const int d = D > 0 ? D : d_rt;
  const int64_t p = (int64_t)blockIdx.x * KM_THREADS + threadIdx.x;
  const bool active = p < n;
  double x[MAXD];
#pragma unroll
  for (int t = 0; t < MAXD; ++t) x[t] = (active && t < d) ? X[p * d + t] : 0.0;
  double best = INFINITY;
  int best_c = 0;
  const int chunk = KM_SMEM_DOUBLES / d;
  for (int c0 = 0; c0 < m; c0 += chunk) {
    const int cn = min(chunk, m - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * d; i += KM_THREADS) sc[i] = C[(int64_t)c0 * d + i];
    __syncthreads();
    if (active) {
      for (int c = 0; c < cn; ++c) {
        const double *cc = sc + c * d;
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < MAXD; ++t) {
          if (t < d) {
            const double diff = __dsub_rn(x[t], cc[t]);
            s = __dadd_rn(s, __dmul_rn(diff, diff));
          }
        }
        if (s < best) {
          best = s;
          best_c = c0 + c;
        }
      }
    }
  }
  if (active) {
    idx[p] = best_c;
    d2[p] = best;
  }
}

// One warp per cluster over the members in sorted order: Xs/ws are X and w
// gathered by the stable sort (row k = k-th member in cluster-then-index
// order), so a cluster's rows are contiguous.  Slot u in [0, d] is
// coordinate u (u < d: the sum of w_j * x_ju) or the weight sum (u == d);
// lane l owns slots l and l + 32.  Members are consumed 32 at a time: the
// next 32 rows are loaded while the current ones run through each slot's
// sequential chain in member order (the reference's rounding sequence).
// d <= 63 (WIDE: d >= 32, two slots per lane).
template <bool WIDE>
struct KmChunk {
  double v0[32], v1[WIDE ? 32 : 1], w;
};

template <bool WIDE>
__device__ __forceinline__ void km_load(KmChunk<WIDE> &ch, const double *__restrict__ Xs,
                                        const double *__restrict__ ws, int64_t k, int cnt, int d,
                                        int lane) {
  ch.w = lane < cnt ? ws[k + lane] : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    ch.v0[i] = (i < cnt && lane < d) ? Xs[(k + i) * d + lane] : 0.0;
    if (WIDE) ch.v1[WIDE ? i : 0] = (i < cnt && lane + 32 < d) ? Xs[(k + i) * d + lane + 32] : 0.0;
  }
}

template <bool WIDE>
__device__ __forceinline__ void km_chain(const KmChunk<WIDE> &ch, int cnt, int d, int lane,
                                         double &s0, double &s1) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const double wi = __shfl_sync(0xffffffffu, ch.w, i);
    if (i < cnt) {
      s0 = __dadd_rn(s0, lane < d ? __dmul_rn(wi, ch.v0[i]) : wi);
      if (WIDE) s1 = __dadd_rn(s1, lane + 32 < d ? __dmul_rn(wi, ch.v1[WIDE ? i : 0]) : wi);
    }
  }
}

template <bool WIDE>
__global__ void __launch_bounds__(256)
kmeans_update_f64_kernel(const int64_t *__restrict__ off, const double *__restrict__ Xs,
                         const double *__restrict__ ws, const double *__restrict__ C_old, int m,
                         int d, double *__restrict__ C_new, double *__restrict__ wsum) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= m) return;
  const int64_t a = off[c], b = off[c + 1];
  double s0 = 0.0, s1 = 0.0;
  KmChunk<WIDE> A, B;
  auto count = [&](int64_t k) { return k >= b ? 0 : (b - k < 32 ? (int)(b - k) : 32); };
  int64_t k = a;
  km_load<WIDE>(A, Xs, ws, k, count(k), d, lane);
  while (k < b) {
    km_load<WIDE>(B, Xs, ws, k + 32, count(k + 32), d, lane);
    km_chain<WIDE>(A, count(k), d, lane, s0, s1);
    k += 32;
    if (k >= b) break;
    km_load<WIDE>(A, Xs, ws, k + 32, count(k + 32), d, lane);
    km_chain<WIDE>(B, count(k), d, lane, s0, s1);
    k += 32;
  }
  // the weight sum is slot d: lane d % 32, register (d < 32 ? s0 : s1)
  const double wt = __shfl_sync(0xffffffffu, d < 32 ? s0 : s1, d & 31);
  const int u0 = lane, u1 = lane + 32;
  if (u0 < d) C_new[(int64_t)c * d + u0] = wt > 0.0 ? __ddiv_rn(s0, wt) : C_old[(int64_t)c * d + u0];
  if (WIDE && u1 < d)
    C_new[(int64_t)c * d + u1] = wt > 0.0 ? __ddiv_rn(s1, wt) : C_old[(int64_t)c * d + u1];
  if (lane == 0) wsum[c] = wt;
}

}  // namespace antkv

using namespace antkv;

extern "C" int antkv_kmeans_assign_f64(const double *X, const double *C, int64_t n, int m, int d,
                                       int64_t *idx, double *d2, void *stream) {
  ANTKV_REQUIRE(n >= 0 && m >= 1 && d >= 1, "bad k-means sizes");
  ANTKV_REQUIRE(d <= 64, "d_sub must be <= 64 for the float64 assignment");
  if (n == 0) return ANTKV_OK;
  cudaStream_t st = as_stream(stream);
  const unsigned grid = (unsigned)((n + KM_THREADS - 1) / KM_THREADS);
  const size_t smem = sizeof(double) * (size_t)(KM_SMEM_DOUBLES / d) * d;
#define KM_LAUNCH(DD, MD)                                                                      \
  kmeans_assign_f64_kernel<DD, MD><<<grid, KM_THREADS, smem, st>>>(X, C, n, m, d, idx, d2);
  switch (d) {
    case 1: KM_LAUNCH(1, 1) break;
    case 2: KM_LAUNCH(2, 2) break;
    case 4: KM_LAUNCH(4, 4) break;
    case 8: KM_LAUNCH(8, 8) break;
    case 16: KM_LAUNCH(16, 16) break;
    case 32: KM_LAUNCH(32, 32) break;
    default:
      if (d <= 8) {
        KM_LAUNCH(0, 8)
      } else if (d <= 16) {
        KM_LAUNCH(0, 16)
      } else if (d <= 32) {
        KM_LAUNCH(0, 32)
      } else {
        KM_LAUNCH(0, 64)
      }
  }
#undef KM_LAUNCH
  ANTKV_LAUNCH_CHECK("kmeans_assign_f64_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_kmeans_update_f64(const int64_t *offsets, const double *Xs,
                                       const double *ws, const double *C_old, int m, int d,
                                       double *C_new, double *wsum, void *stream) {
  ANTKV_REQUIRE(m >= 1 && d >= 1, "bad k-means sizes");
  ANTKV_REQUIRE(d <= 63, "d_sub must be <= 63 for the float64 update");
  cudaStream_t st = as_stream(stream);
  if (d >= 32)
    kmeans_update_f64_kernel<true><<<(unsigned)((m + 7) / 8), 256, 0, st>>>(
        offsets, Xs, ws, C_old, m, d, C_new, wsum);
  else
    kmeans_update_f64_kernel<false><<<(unsigned)((m + 7) / 8), 256, 0, st>>>(
        offsets, Xs, ws, C_old, m, d, C_new, wsum);
  ANTKV_LAUNCH_CHECK("kmeans_update_f64_kernel");
  return ANTKV_OK;
}
