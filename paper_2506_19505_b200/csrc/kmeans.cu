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
//    then csum / wsum for live clusters.  The members come in that order from
//    a stable sort of the assignment; one thread per (cluster, coordinate)
//    runs the sequential sum, which is what makes the rounding identical.
//
// The k-means++ seeding, the empty-cluster repair and the stopping rule stay
// in the host driver (vq.py weighted_kmeans); they are O(m) decisions.
#include "common.cuh"

namespace antkv {

constexpr int KM_THREADS = 256;
constexpr int KM_SMEM_DOUBLES = 6144;  // 48 KB of centroids per chunk

template <int MAXD>
__global__ void __launch_bounds__(KM_THREADS)
kmeans_assign_f64_kernel(const double *__restrict__ X, const double *__restrict__ C, int64_t n,
                         int m, int d, int64_t *__restrict__ idx, double *__restrict__ d2) {
  extern __shared__ double sc[];
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

// Thread (c, t): t < d sums w_j * X[j, t], t == d sums w_j, over the members
// perm[off[c] .. off[c+1]) of cluster c in ascending point order.
__global__ void kmeans_update_f64_kernel(const int64_t *__restrict__ perm,
                                         const int64_t *__restrict__ off,
                                         const double *__restrict__ X,
                                         const double *__restrict__ w,
                                         const double *__restrict__ C_old, int m, int d,
                                         double *__restrict__ C_new, double *__restrict__ wsum) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)m * (d + 1)) return;
  const int c = (int)(gid / (d + 1)), t = (int)(gid % (d + 1));
  const int64_t a = off[c], b = off[c + 1];
  double s = 0.0, ws = 0.0;
  if (t < d) {
    for (int64_t k = a; k < b; ++k) {
      const int64_t j = perm[k];
      s = __dadd_rn(s, __dmul_rn(w[j], X[j * d + t]));
    }
    // wsum is needed for the division: the same sequential sum as t == d
    for (int64_t k = a; k < b; ++k) ws = __dadd_rn(ws, w[perm[k]]);
    C_new[(int64_t)c * d + t] = ws > 0.0 ? __ddiv_rn(s, ws) : C_old[(int64_t)c * d + t];
  } else {
    for (int64_t k = a; k < b; ++k) ws = __dadd_rn(ws, w[perm[k]]);
    wsum[c] = ws;
  }
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
#define KM_LAUNCH(MD)                                                                          \
  kmeans_assign_f64_kernel<MD><<<grid, KM_THREADS, smem, st>>>(X, C, n, m, d, idx, d2);
  if (d <= 8) {
    KM_LAUNCH(8)
  } else if (d <= 16) {
    KM_LAUNCH(16)
  } else if (d <= 32) {
    KM_LAUNCH(32)
  } else {
    KM_LAUNCH(64)
  }
#undef KM_LAUNCH
  ANTKV_LAUNCH_CHECK("kmeans_assign_f64_kernel");
  return ANTKV_OK;
}

extern "C" int antkv_kmeans_update_f64(const int64_t *perm, const int64_t *offsets,
                                       const double *X, const double *w, const double *C_old,
                                       int m, int d, double *C_new, double *wsum, void *stream) {
  ANTKV_REQUIRE(m >= 1 && d >= 1, "bad k-means sizes");
  cudaStream_t st = as_stream(stream);
  const int64_t threads = (int64_t)m * (d + 1);
  kmeans_update_f64_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(
      perm, offsets, X, w, C_old, m, d, C_new, wsum);
  ANTKV_LAUNCH_CHECK("kmeans_update_f64_kernel");
  return ANTKV_OK;
}
