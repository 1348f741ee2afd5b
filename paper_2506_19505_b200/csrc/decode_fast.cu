// sm_100a tensor-core decode kernel for d=128, d_sub=8, m<=256 (1-bit d8m256).
#include "common.cuh"

namespace antkv {

int decode_fast_supported(const antkv_cache_desc &c) { return 0; }

int decode_fast_launch(const antkv_cache_desc &c, const void *q, int dtype, const int64_t *qpos,
                       float *ws_o, float *ws_m, float *ws_l, int splits, cudaStream_t st) {
  set_error("fast decode kernel not built");
  return ANTKV_EUNSUPPORTED;
}

}  // namespace antkv
