/*
 * antkv_b200.h — C ABI of the B200-native AnTKV anchor-token sub-bit KV-cache
 * path (libantkv_b200.so, built for sm_100a).
 *
 * Every entry point takes plain device pointers and sizes plus a CUDA stream
 * (as void*, NULL = default stream) and returns an ANTKV_* status code.  No
 * entry point synchronises the stream; outputs are ready when the stream
 * reaches them.  antkv_last_error() returns the message of the last failure
 * on the calling thread.  Invalid arguments (the reference's ValueError)
 * return ANTKV_EINVAL before anything is launched.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/antkv):
 *   antkv_flash_aux        <- kernels.flash_aux      (_ckernels.pyx:10-88,
 *                             kernels/__init__.py:35)
 *   antkv_ans_blocked      <- kernels.ans_blocked    (_ckernels.pyx:91-131,
 *                             kernels/__init__.py:36)
 *   antkv_assign_nearest   <- kernels.assign_nearest (_ckernels.pyx:134-163,
 *                             kernels/__init__.py:37)
 *   antkv_prefill_attention <- attention.flash_attention_aux (attention.py:146-169)
 *                             with RoPE (attention.py:89-106) fused, GQA-batched
 *   antkv_prefill_anchor_scores <- anchors.anchor_scores_blocked (anchors.py:66-87)
 *   antkv_prefill_attention_scores <- both passes of cache.py:100-121 in one call
 *   antkv_prefill_*_block  <- (new) the same two passes per sequence-shard block
 *   antkv_select_anchors   <- anchors.select_anchors  (anchors.py:96-132)
 *   antkv_cache_build      <- QuantizedKVCache.prefill layout step (cache.py:122-139)
 *   antkv_cache_append     <- QuantizedKVCache.decode_step append (cache.py:157-166)
 *   antkv_decode_attention <- QuantizedKVCache.decode_step math (cache.py:168-178)
 *   antkv_cache_evict      <- QuantizedKVCache.decode_step eviction (cache.py:180-193)
 *   antkv_cache_dequantize <- QuantizedKVCache.dequantize (cache.py:196-211)
 *   antkv_vq_encode        <- vq.encode_rows (vq.py:226-232)
 *   antkv_vq_decode        <- vq.decode_rows (vq.py:243-248)
 *   antkv_kmeans_*_f64     <- vq.weighted_kmeans Lloyd step (vq.py:178-197) with
 *                             kernels.assign_nearest (_ckernels.pyx:134-163)
 *   antkv_eval_pair_l1     <- harness.per_token_errors / anchors.k_perturbation_bound
 *                             pair sums (harness.py:111-134, anchors.py:152-186)
 *   antkv_decode_step_publish / antkv_lse_merge_wait / antkv_ipc_* / antkv_p2p_*
 *                          <- (new) peer-memory exchange of sequence-shard partials
 *   antkv_lse_combine      <- (new) split-KV / sequence-shard log-sum-exp merge
 */
#ifndef ANTKV_B200_H
#define ANTKV_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ANTKV_API __attribute__((visibility("default")))
#else
#define ANTKV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ANTKV_OK 0
#define ANTKV_EINVAL 1       /* invalid argument (reference ValueError)      */
#define ANTKV_ECUDA 2        /* CUDA runtime error                           */
#define ANTKV_EUNSUPPORTED 3 /* configuration not supported by this build    */

#define ANTKV_POLICY_BY_K 0
#define ANTKV_POLICY_BY_V 1
#define ANTKV_POLICY_BY_SUM 2

#define ANTKV_KIND_ANCHOR 0
#define ANTKV_KIND_QUANTIZED 1
#define ANTKV_KIND_WINDOWED 2
#define ANTKV_KIND_FREE -1

#define ANTKV_HSTATE_WORDS 8 /* per (sequence, kv head) state words         */
#define ANTKV_HS_ANCHORS 0   /* anchor count                                */
#define ANTKV_HS_WIN_HEAD 1  /* index of the oldest windowed slot in ring   */
#define ANTKV_HS_WIN_COUNT 2 /* number of windowed rows                     */
#define ANTKV_HS_FREE_TOP 3  /* free-stack size                             */
#define ANTKV_HS_POOL_HIGH 4 /* high-water mark of used pool slots          */

/* dtype tags for row inputs */
/* Row / tile arrays handed to the prefill, cache-build and encode entry
 * points (Q, K, V, X) are read with 16-byte vector loads and bulk copies and
 * must start at a 16-byte aligned address (ANTKV_EINVAL otherwise); any
 * freshly allocated device buffer is. */
#define ANTKV_F32 0
#define ANTKV_BF16 1
#define ANTKV_F16 2

ANTKV_API const char *antkv_last_error(void);
ANTKV_API int antkv_version(void);
/* 1 when the running device is sm_100 (B200) and the library kernels load. */
ANTKV_API int antkv_device_check(int device);

/* Declares that, on `stream`, only this library's kernels run between its
 * decode launches (a decode-only layer chain, a CUDA graph of decode steps).
 * Only then may the fused decode kernel, launched with programmatic
 * dependent launch, read the cache state, q and the position before
 * griddepcontrol.wait (its predecessor is then known to be one of ours and
 * to leave them untouched); when none of its inputs (q, the position, the
 * appended k / v rows) is an output of that predecessor, the wait moves
 * behind the streaming loop.  Default off: a foreign kernel writing q (a
 * GEMM, RoPE, a torch copy) may be the predecessor, so everything is read
 * after the wait.  New (no reference counterpart). */
ANTKV_API int antkv_stream_exclusive(void *stream, int exclusive);

/* ------------------------------------------------------------------------
 * Reference FFI (antkv._ckernels).  Batched over `heads` query heads; query
 * head h reads K/V head h / (heads / kv_heads).  Inputs are float32, row
 * major, already RoPE-rotated, Qs pre-scaled by 1/sqrt(d) — exactly the
 * contract of the reference kernels.  Block sizes only change the reference's
 * rounding order; the GPU tiles internally and accepts any block >= 1.
 *   Qs [heads][n_q][d], Kr [kv_heads][n_k][d], V [kv_heads][n_k][dv]
 *   O [heads][n_q][dv], L/M [heads][n_q]
 * causal requires n_q == n_k (attention.py:160-161).
 * ---------------------------------------------------------------------- */
ANTKV_API int antkv_flash_aux(const float *Qs, const float *Kr, const float *V,
                    int heads, int kv_heads, int n_q, int n_k, int d, int dv,
                    int block_q, int block_k, int causal,
                    float *O, float *L, float *M, void *stream);

/* ans_k/ans_v [heads][n_k]: per query head (no GQA summation here). */
ANTKV_API int antkv_ans_blocked(const float *Qs, const float *Kr, const float *M,
                      const float *L, const float *q_norms,
                      int heads, int kv_heads, int n_q, int n_k, int d,
                      int block_q, int block_k, int causal,
                      float *ans_k, float *ans_v, void *stream);

/* X [n][d_sub], C [m][d_sub] float32 -> idx int64 [n], d2 float32 [n].
 * Strict-< argmin over centroids in index order: ties -> lowest index. */
ANTKV_API int antkv_assign_nearest(const float *X, const float *C, int64_t n, int m,
                         int d_sub, int64_t *idx, float *d2, void *stream);

/* ------------------------------------------------------------------------
 * Path kernels.
 * ---------------------------------------------------------------------- */

/* Causal prefill attention with RoPE applied in-kernel (interleaved pairs,
 * fp64-accurate angles), GQA.  Q [B][Hq][n][d], K/V [B][Hkv][n][d] in
 * `dtype`; positions int64 [B][n].  Outputs O float32 [B][Hq][n][d],
 * M/L float32 [B][Hq][n] (scaled-logit max / normaliser at M) and q_norms
 * float32 [B][Hq][n] of the PRE-RoPE queries (attention.py:167). */
ANTKV_API int antkv_prefill_attention(const void *Q, const void *K, const void *V, int dtype,
                            const int64_t *positions, int B, int Hq, int Hkv,
                            int n, int d, double theta_base,
                            float *O, float *M, float *L, float *q_norms,
                            void *stream);

/* Input validation of the prefill (attention.py:59-67 `_check_finite`,
 * called from cache.py:100-140 through attention.flash_attention_with_aux):
 * *flag |= 1 when any of the n elements of X (dtype) is NaN or +-inf.  One
 * HBM pass; the caller zeroes the flags once and reads them back once for
 * Q, K and V together. */
ANTKV_API int antkv_check_finite(const void *X, int dtype, int64_t n, int *flag, void *stream);

/* RoPE (attention.py:89-106): X [B][H][n][d] (dtype) rotated at positions
 * int64 [B][n] (NULL = no rotation), times `scale`, into out float32; norms
 * (optional) float32 [B][H][n] = L2 norm of the un-rotated row. */
ANTKV_API int antkv_rope_rotate(const void *X, int dtype, const int64_t *positions,
                                int B, int H, int n, int d, double theta_base,
                                float scale, float *out, float *norms, void *stream);

/* Anchor scores (Alg. 1 second pass) summed over each KV head's Q group:
 * ans_k/ans_v float32 [B][Hkv][n]. */
ANTKV_API int antkv_prefill_anchor_scores(const void *Q, const void *K, int dtype,
                                const int64_t *positions, const float *M,
                                const float *L, const float *q_norms,
                                int B, int Hq, int Hkv, int n, int d,
                                double theta_base, float *ans_k, float *ans_v,
                                void *stream);

/* Both prefill passes in one call (what QuantizedKVCache.prefill needs):
 * antkv_prefill_attention's outputs plus antkv_prefill_anchor_scores'
 * ans_k/ans_v [B][Hkv][n].  For bf16 rows with d = 128 the two tcgen05
 * kernels share one set of rotated, split Q/K tiles (RoPE fused into the
 * split); other inputs run the two calls. */
ANTKV_API int antkv_prefill_attention_scores(const void *Q, const void *K, const void *V, int dtype,
                            const int64_t *positions, int B, int Hq, int Hkv, int n, int d,
                            double theta_base, float *O, float *M, float *L, float *q_norms,
                            float *ans_k, float *ans_v, void *stream);

/* Sequence-shard blocks of the two prefill passes (context parallelism,
 * SURVEY.md §8e; parallel.py ShardedPrefill).  A query block Q [B][Hq][n_q][d]
 * at q_positions [B][n_q] against a key block K/V [B][Hkv][n_k][d] at
 * k_positions [B][n_k]; `causal` masks key index j > query index i within
 * the block (diagonal blocks only: requires n_q == n_k).  The attention
 * block returns the block-local (O, M, L) that parallel.merge_partial folds
 * together, plus q_norms; the score block returns this block's share of
 * ans_k/ans_v [B][Hkv][n_k] (summed over the query group, overwritten).
 * antkv_prefill_attention / antkv_prefill_anchor_scores are the single-block
 * case. */
ANTKV_API int antkv_prefill_attention_block(const void *Q, const void *K, const void *V,
                            int dtype, const int64_t *q_positions,
                            const int64_t *k_positions, int B, int Hq, int Hkv,
                            int n_q, int n_k, int d, double theta_base, int causal,
                            float *O, float *M, float *L, float *q_norms, void *stream);
ANTKV_API int antkv_prefill_anchor_scores_block(const void *Q, const void *K, int dtype,
                            const int64_t *q_positions, const int64_t *k_positions,
                            const float *M, const float *L, const float *q_norms,
                            int B, int Hq, int Hkv, int n_q, int n_k, int d,
                            double theta_base, int causal, float *ans_k, float *ans_v,
                            void *stream);

/* Top-budget selection per (b, kv head) under `policy`, ties to the lower
 * index, result sorted ascending: anchors int32 [B][Hkv][budget].
 * budget is clipped to [0, n] by the caller (anchors.py:104). */
ANTKV_API int antkv_select_anchors(const float *ans_k, const float *ans_v, int B, int Hkv,
                         int n, int budget, int policy, int32_t *anchors,
                         void *stream);

/* Encode rows: X [rows][d] (dtype) with codebook [m][d_sub] float32 into
 * codes [rows][d/d_sub] of width code_bytes (1, 2, or 8 = int64). */
ANTKV_API int antkv_vq_encode(const void *X, int dtype, int64_t rows, int d,
                    const float *codebook, int m, int d_sub,
                    void *codes, int code_bytes, void *stream);

/* Gather: codes [rows][groups] (code_bytes wide) -> out float32 [rows][groups*d_sub]. */
ANTKV_API int antkv_vq_decode(const void *codes, int code_bytes, int64_t rows, int groups,
                    const float *codebook, int m, int d_sub, float *out,
                    void *stream);

/* Quantized KV cache for B sequences x Hkv heads.  All buffers are device
 * memory owned by the caller; sizes follow the bracketed shapes. */
typedef struct antkv_cache_desc {
  int B, Hq, Hkv, d, d_sub, m, groups, index_bits;
  int code_bytes;      /* 1 when index_bits <= 8; 3 = 12-bit indices packed
                          two per 3 bytes (index_bits <= 12, groups a power
                          of two <= 32); else 2                             */
  int capacity;        /* token slots per sequence                         */
  int pool_capacity;   /* full-precision row slots per (b, kv head)        */
  int window_size;
  int policy;
  int anchor_count;    /* < 0: use anchor_fraction (cache.py:54-57)        */
  int row_dtype;       /* ANTKV_BF16 / ANTKV_F16 / ANTKV_F32: dtype of the
                          full-precision pool rows (the input dtype)        */
  double anchor_fraction;
  double theta_base;
  int64_t token_offset;/* global index of slot 0 (sequence sharding)       */
  uint8_t *codes;      /* [B][Hkv][capacity/16 tiles][K 16 x groups | V 16 x
                          groups] code units (code_bytes wide, or 12-bit
                          packed: a slot's K+V codes take 3*groups bytes)   */
  uint32_t *qmask;     /* [B][Hkv][capacity/32] bit = slot holds codes     */
  void *pool_rows;     /* [B][Hkv][pool_capacity][2][d] (K row, V row)    */
  int32_t *pool_tok;   /* [B][Hkv][pool_capacity] token slot, -1 free      */
  int8_t *pool_kind;   /* [B][Hkv][pool_capacity] ANTKV_KIND_*             */
  int32_t *win_ring;   /* [B][Hkv][window_size+1] pool slots, FIFO          */
  int32_t *free_stack; /* [B][Hkv][pool_capacity]                           */
  int32_t *hstate;     /* [B][Hkv][ANTKV_HSTATE_WORDS]                      */
  int32_t *seq_len;    /* [B] tokens currently held                         */
  int64_t *positions;  /* [B][capacity]                                     */
  const float *codebook_k; /* [Hkv][m][d_sub] float32                       */
  const float *codebook_v;
  uint16_t *codebook_f16;  /* fast path: 64 KB per head; its first 8 KB hold
                              [256 codes][K 8 | V 8] fp16 (the fused kernel
                              replicates each row across the 8 16-byte bank
                              groups of its shared-memory copy)              */
  uint16_t *pool_f16;  /* fast path: fp16 [B][Hkv][pool_capacity/16] tiles of
                          [2 (K rotated at its position, V)][16 slots][128]
                          with the 16-byte chunks of slot r XOR-swizzled by
                          r & 7; pool_capacity is a multiple of 16          */
  void *fast_tables;   /* fast path: 16384-byte RoPE constant tables        */
  uint16_t *codebook_f16g; /* staged tensor-core path (any d = 128 code shape
                              but the d8m256 fast path): fp16 [Hkv][2 (K,V)]
                              [m][d_sub], the float32 codebooks rounded      */
  unsigned long long *evict_scratch; /* [B][Hkv][2*groups] minima of the
                              eviction encoder, (float distance bits << 32) |
                              centroid index; all ones between calls        */
} antkv_cache_desc;

/* Bytes of scratch needed by antkv_decode_attention for `splits` (0 = auto). */
ANTKV_API int64_t antkv_decode_workspace_bytes(const antkv_cache_desc *c, int splits);

/* Populate an EMPTY cache from prefill results (cache.py:122-139):
 * K/V [B][Hkv][n][d] (dtype), positions int64 [B][n], anchors int32
 * [B][Hkv][n_anchors] sorted, optionally ending in -1 padding (per-head
 * counts may differ, e.g. on sequence shards).  Anchors keep full-precision rows, the last
 * window_size non-anchor tokens are windowed, the rest are encoded. */
ANTKV_API int antkv_cache_build(const antkv_cache_desc *c, const void *K, const void *V,
                      int dtype, const int64_t *positions, int n,
                      const int32_t *anchors, int n_anchors, void *stream);

/* Append one token per sequence as WINDOWED (cache.py:157-166):
 * k/v [B][Hkv][d] (dtype), position int64 [B].  seq_len[b] must be < capacity
 * (checked on the host side by the caller's shadow). */
ANTKV_API int antkv_cache_append(const antkv_cache_desc *c, const void *k, const void *v,
                       int dtype, const int64_t *position, void *stream);

/* Decode attention of q [B][Hq][d] (dtype) at positions qpos int64 [B]
 * against the whole cache (anchors + window + codes), RoPE after
 * reconstruction, split-KV with an LSE merge.  Writes out float32
 * [B][Hq][d]; when lse != NULL also writes the log-sum-exp (natural log,
 * scaled logits) float32 [B][Hq] so sequence shards can be merged.
 * fast: 1 = the best sm_100a tensor-core kernel the config allows (the fused
 * d8m256 kernel for d == 128, d_sub == 8, m <= 256, 4 query heads per KV
 * head; else the staged kernel for d == 128, d_sub 4..64, GQA 1/2/4/8),
 * 2 = the staged kernel, 0 = generic fp32 kernel. */
ANTKV_API int antkv_decode_attention(const antkv_cache_desc *c, const void *q, int dtype,
                           const int64_t *qpos, float *out, float *lse,
                           void *workspace, int64_t workspace_bytes, int splits,
                           int fast, void *stream);

/* One full decode step (cache.py:149-194): append (k, v) [B][Hkv][d] as
 * windowed, attend q [B][Hq][d] over the cache (output before eviction),
 * then evict/promote/encode the oldest window row.  With `fast` and a
 * d8m256 cache this is ONE kernel launch (attention + split combine + cache
 * update in the last CTA of every (sequence, head)); otherwise append,
 * attention, combine and evict run as separate kernels.  The workspace
 * (antkv_decode_workspace_bytes) must be zero-filled before its first use;
 * the kernels leave its ticket counters at zero. */
ANTKV_API int antkv_decode_step(const antkv_cache_desc *c, const void *q, const void *k,
                                const void *v, int dtype, const int64_t *qpos, float *out,
                                float *lse, void *workspace, int64_t workspace_bytes,
                                int splits, int fast, void *stream);

/* Evict the oldest windowed row of every (b, head) whose window exceeds
 * window_size: promote to anchor while the budget has headroom, otherwise
 * encode it into the code slots (cache.py:180-193). */
ANTKV_API int antkv_cache_evict(const antkv_cache_desc *c, void *stream);

/* K_hat / V_hat float32 [B][Hkv][n][d], pre-RoPE (cache.py:196-211). */
ANTKV_API int antkv_cache_dequantize(const antkv_cache_desc *c, int n, float *Khat,
                           float *Vhat, void *stream);

/* Merge P partial results: o [P][rows][d] (normalised), lse [P][rows] ->
 * out [rows][d], lse_out [rows] (may be NULL). */
ANTKV_API int antkv_lse_combine(const float *o, const float *lse, int P, int64_t rows,
                      int d, float *out, float *lse_out, void *stream);

/* Codebook training (weighted k-means, vq.py:141-214), float64 with the
 * reference's operation order (bit-identical results).
 * assign: X [n][d], C [m][d] -> idx int64 [n], d2 float64 [n]; sequential
 *   sum over t of (x_t - c_t)^2 without FMA, strict-< argmin (d <= 64).
 * update (d <= 63): Xs [n][d] / ws [n] are X and w in member order (a
 *   stable sort of idx: cluster c owns rows offsets[c] .. offsets[c+1], in
 *   ascending point order); C_new[c] = sum w_j x_j / sum w_j for clusters
 *   with positive weight, else C_old[c]; wsum [m]. */
ANTKV_API int antkv_kmeans_assign_f64(const double *X, const double *C, int64_t n, int m,
                                      int d, int64_t *idx, double *d2, void *stream);
ANTKV_API int antkv_kmeans_update_f64(const int64_t *offsets, const double *Xs,
                                      const double *ws, const double *C_old, int m, int d,
                                      double *C_new, double *wsum, void *stream);

/* Evaluation harness (harness.py:109-235), float64:
 *   out[j] = sum_i W_ij * sum_t |P_ij (X_jt - Y_it) - R_ij (Z_jt - Y_it)|
 * Y [n_i][d], X/Z [n_j][d], W/P/R [n_i][n_j] (NULL: W = 1, P = 1, R = 0;
 * Z NULL drops the R term); i_from_j0 = 1 skips rows i < 32*floor(j/32)
 * (causal masks zero them).  Carries the K perturbation bound
 * (anchors.py:152-186) and the per-token quantisation errors
 * (harness.py:111-134) in O(n^2 d). */
ANTKV_API int antkv_eval_pair_l1(const double *Y, const double *X, const double *Z,
                                 const double *W, const double *P, const double *R, int n_i,
                                 int n_j, int d, int i_from_j0, double *out, void *stream);

/* Sequence-shard exchange over peer memory (replaces the NCCL all-gather of
 * the shards' (o, lse) partials).  Every rank owns receive
 * buffers (antkv_p2p_alloc: o [P][B*Hq][d] | lse [P][B*Hq] | flags [P]
 * uint32, zeroed) and maps its peers' with antkv_ipc_get_handle (64-byte
 * handle) / antkv_ipc_open_handle.
 * antkv_decode_step_publish: antkv_decode_step (k == NULL: attention only)
 *   whose combined partial is then stored into slot `rank` of each of the
 *   n_dst receive buffers (dst_o / dst_lse / dst_flags: DEVICE arrays of
 *   n_dst base pointers) by direct peer stores; then each destination's
 *   flag of that slot is set to `seq` with a system-scope release.  A receive
 *   buffer has two halves selected by seq & 1 (o [2][P][rows][d],
 *   lse [2][P][rows], flags [2][P], P = n_dst): consecutive steps never share
 *   a half, so a rank one step ahead cannot overwrite a slot a slower peer
 *   still merges (it cannot get two steps ahead: its step s + 2 publish is
 *   stream-ordered after its merge of s + 1, which needs every peer's s + 1
 *   publish, issued after that peer's merge of s).  lse must be non-NULL.
 * antkv_lse_merge_wait: waits (system-scope acquire) until flags[seq & 1][p]
 *   equals seq for every p < P, then merges the P partials of that half
 *   (as antkv_lse_combine).  seq advances by one per step and is never 0
 *   (0 is the flags' initial value). */
ANTKV_API int antkv_p2p_alloc(int64_t bytes, void **ptr);
ANTKV_API int antkv_p2p_free(void *ptr);
ANTKV_API int antkv_ipc_get_handle(const void *ptr, void *handle);
ANTKV_API int antkv_ipc_open_handle(const void *handle, void **ptr);
ANTKV_API int antkv_ipc_close_handle(void *ptr);
ANTKV_API int antkv_decode_step_publish(const antkv_cache_desc *c, const void *q, const void *k,
                                        const void *v, int dtype, const int64_t *qpos, float *out,
                                        float *lse, void *workspace, int64_t workspace_bytes,
                                        int splits, int fast, float *const *dst_o,
                                        float *const *dst_lse, unsigned *const *dst_flags,
                                        int n_dst, int rank, unsigned seq, void *stream);
ANTKV_API int antkv_lse_merge_wait(const float *o, const float *lse, const unsigned *flags, int P,
                                   unsigned seq, int64_t rows, int d, float *out, float *lse_out,
                                   void *stream);

/* Debug: per-CTA timeline of the last fast-decode launch when the process
 * runs with ANTKV_TRACE=1 (8 words per CTA); returns words copied. */
ANTKV_API int antkv_debug_trace(unsigned long long *host, int max_words);

/* Build the fast-path fp16 codebooks from codebook_k/v and the rotated
 * pool K rows for the rows currently held. */
ANTKV_API int antkv_cache_prepare_fast(const antkv_cache_desc *c, void *stream);

/* Build the staged tensor-core path's fp16 codebooks (codebook_f16g) and the
 * RoPE tables from codebook_k/v (after the codebooks are set). */
ANTKV_API int antkv_cache_prepare_tc(const antkv_cache_desc *c, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ANTKV_B200_H */
