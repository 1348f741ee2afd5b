// Pairwise L1 reductions of the evaluation harness (harness.py:109-235,
// SURVEY.md §8f rank 4), float64:
//
//   out[j] = sum_i W_ij * sum_t | P_ij (X_jt - Y_it) - R_ij (Z_jt - Y_it) |
//
// with W / P / R optional [n_i][n_j] matrices (NULL: W = 1, P = 1, R = 0).
// Two evaluation quantities are this shape:
//  * the K perturbation factor of anchors.k_perturbation_bound
//    (anchors.py:152-186): W = A * ||q_i||, X = V, Y = A V;
//  * the per-token quantisation errors of harness.per_token_errors
//    (harness.py:111-134), which the reference gets from n full attention
//    passes (O(n^3 d)).  Replacing token j's row changes row i of the
//    softmax only through column j, so with a = A_ij, a' = A'_ij (the
//    probability with the quantised key) the output change is exactly
//    (a' (v'_j - o_i) - a (v_j - o_i)) / (1 - a + a'): W = 1 / (1 - A + A'),
//    P = A', R = A, X = V', Z = V, Y = O.  O(n^2 d) in total.
// One CTA owns 32 columns j (one per lane, rows staged in shared memory);
// its 8 warps stride over the rows i; `i_from_j0` skips rows i < j0 (causal
// masks make every term there zero).
#include "common.cuh"

namespace antkv {

constexpr int EV_J = 32;
constexpr int EV_WARPS = 8;

__global__ void __launch_bounds__(EV_WARPS * 32)
eval_pair_l1_kernel(const double *__restrict__ Y, const double *__restrict__ X,
                    const double *__restrict__ Z, const double *__restrict__ W,
                    const double *__restrict__ P, const double *__restrict__ R, int n_i, int n_j,
                    int d, int i_from_j0, double *__restrict__ out) {
  extern __shared__ double evs[];
  const int ld = d + 1;                       // padded rows: lane-strided reads are conflict-free
  double *xs = evs, *zs = evs + EV_J * ld;
  double *red = zs + (Z ? EV_J * ld : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.x * EV_J, j = j0 + lane;
  for (int e = threadIdx.x; e < EV_J * d; e += blockDim.x) {
    const int r = e / d, t = e % d;
    const bool ok = j0 + r < n_j;
    xs[r * ld + t] = ok ? X[(int64_t)(j0 + r) * d + t] : 0.0;
    if (Z) zs[r * ld + t] = ok ? Z[(int64_t)(j0 + r) * d + t] : 0.0;
  }
  __syncthreads();
  double acc = 0.0;
  if (j < n_j) {
    const double *xr = xs + lane * ld, *zr = zs + lane * ld;
    for (int i = (i_from_j0 ? j0 : 0) + warp; i < n_i; i += EV_WARPS) {
      const int64_t ij = (int64_t)i * n_j + j;
      const double w = W ? W[ij] : 1.0;
      const double p = P ? P[ij] : 1.0;
      const double q = (R && Z) ? R[ij] : 0.0;
      if (w == 0.0 || (p == 0.0 && q == 0.0)) continue;
      const double *yr = Y + (int64_t)i * d;
      double s = 0.0;
      if (q == 0.0) {
        for (int t = 0; t < d; ++t) s += fabs(p * (xr[t] - __ldg(yr + t)));
      } else {
        for (int t = 0; t < d; ++t) {
          const double y = __ldg(yr + t);
          s += fabs(p * (xr[t] - y) - q * (zr[t] - y));
        }
      }
      acc += w * s;
    }
  }
  red[warp * EV_J + lane] = acc;
  __syncthreads();
  if (warp == 0 && j < n_j) {
    double s = 0.0;
    for (int w = 0; w < EV_WARPS; ++w) s += red[w * EV_J + lane];
    out[j] = s;
  }
}

}  // namespace antkv

using namespace antkv;

extern "C" int antkv_eval_pair_l1(const double *Y, const double *X, const double *Z,
                                  const double *W, const double *P, const double *R, int n_i,
                                  int n_j, int d, int i_from_j0, double *out, void *stream) {
  ANTKV_REQUIRE(n_i >= 0 && n_j >= 0 && d >= 1 && d <= 256, "bad evaluation sizes");
  if (n_j == 0) return ANTKV_OK;
  cudaStream_t st = as_stream(stream);
  const size_t smem = sizeof(double) * ((size_t)EV_J * (d + 1) * (Z ? 2 : 1) + EV_WARPS * EV_J);
  cudaFuncSetAttribute(eval_pair_l1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  eval_pair_l1_kernel<<<(unsigned)((n_j + EV_J - 1) / EV_J), EV_WARPS * 32, smem, st>>>(
      Y, X, Z, W, P, R, n_i, n_j, d, i_from_j0, out);
  ANTKV_LAUNCH_CHECK("eval_pair_l1_kernel");
  return ANTKV_OK;
}
