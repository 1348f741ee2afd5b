"""Seeded synthetic inputs shared by the golden generator and the tests.

Everything is regenerated from a seed (numpy PCG64), so the committed golden
files only hold reference OUTPUTS.  Q/K/V are rounded to bfloat16-exact
values (stored as float32/float64) so that the GPU's bf16 storage of the
full-precision rows is lossless, as SURVEY.md §8(d) prescribes.
"""

import numpy as np


def round_bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def qkv(seed, h_q, h_kv, n, d, heavy=0):
    """Q [h_q, n, d], K/V [h_kv, n, d] bf16-exact float32.  ``heavy`` plants
    that many large-norm early keys per head (harness.py:59-64 pattern)."""
    rng = np.random.default_rng(seed)
    Q = round_bf16(rng.standard_normal((h_q, n, d)))
    K = round_bf16(rng.standard_normal((h_kv, n, d)))
    V = round_bf16(rng.standard_normal((h_kv, n, d)))
    if heavy:
        for h in range(h_kv):
            idx = rng.choice(max(1, n // 2), size=min(heavy, max(1, n // 2)), replace=False)
            K[h, idx] = round_bf16(K[h, idx] * 5.0)
            V[h, idx] = round_bf16(V[h, idx] * 3.0)
    return Q, K, V


def codebooks(seed, h_kv, m, d_sub, scale=1.0):
    """Per-KV-head float32 codebooks [h_kv, m, d_sub] (K and V)."""
    rng = np.random.default_rng(seed + 7919)
    ck = (scale * rng.standard_normal((h_kv, m, d_sub))).astype(np.float32)
    cv = (scale * rng.standard_normal((h_kv, m, d_sub))).astype(np.float32)
    return ck, cv


# name: (seed, n, d, notation, window, frac, count, policy, steps, pos_stride, blocks)
CACHE_CASES = {
    "c1_d8_d4m16": (11, 48, 8, "d4m16", 8, 0.05, None, "by_sum", 12, 1, 16),
    "c2_d128_d8m256": (12, 256, 128, "d8m256", 32, 0.01, None, "by_sum", 64, 1, 64),
    "c3_d64_d32m4096": (13, 128, 64, "d32m4096", 16, 0.02, None, "by_sum", 8, 1, 64),
    "c4_d16_d4m32_byk_stride3": (14, 96, 16, "d4m32", 8, 0.05, 5, "by_k", 16, 3, 16),
    "c5_d32_d2m256_byv": (15, 64, 32, "d2m256", 4, 0.03, None, "by_v", 10, 1, 16),
    "c6_d128_d8m256_all_anchor": (16, 40, 128, "d8m256", 4, 1.0, None, "by_sum", 6, 1, 8),
    "c7_d128_d8m256_no_window": (17, 70, 128, "d8m256", 0, 0.0, None, "by_sum", 6, 1, 32),
}



FA_CASES = {"small": (77, 16, 16, 8, 101), "d128": (200, 128, 64, 64, 102),
            "ragged": (33, 10, 7, 5, 103)}
AN_CASES = {"d8m256": (2000, 256, 8, 201), "d4m16": (500, 16, 4, 202),
            "d32m4096": (64, 4096, 32, 203), "d2m256": (700, 256, 2, 204)}


def fa_inputs(n, d, seed):
    rng = np.random.default_rng(seed)
    return tuple(rng.standard_normal((n, d)) for _ in range(3))


def an_inputs(N, m, ds, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, ds))
    C = rng.standard_normal((m, ds)).astype(np.float32).astype(np.float64)
    return X, C


# weighted k-means cases (vq.py:141-214): name -> (seed, n, d, m, kmeans_seed,
# max_iter, weights kind, init kind)
KM_CASES = {
    "pp_d8m64": (301, 2000, 8, 64, 5, 30, "random", None),
    "init_d4m16": (302, 3000, 4, 16, 0, 50, "ones", "sample"),
    "padded_d3m12": (303, 5, 3, 12, 0, 100, "ones", None),
    "zero_w_d8m32": (304, 500, 8, 32, 1, 40, "zeros30", None),
    "empties_d2m10": (305, 400, 2, 10, 0, 40, "random", "far"),
    "pp_d32m128": (306, 1500, 32, 128, 7, 15, "random", None),
    "single_d1m1": (307, 2, 1, 1, 0, 100, "three_one", None),
}


def km_inputs(name):
    """(X [n, d] float64, w [n], init or None) for a KM_CASES entry."""
    seed, n, d, m, _, _, wk, ik = KM_CASES[name]
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)) * 2.0
    if wk == "ones":
        w = np.ones(n)
    elif wk == "zeros30":
        w = rng.random(n) + 0.01
        w[rng.random(n) < 0.3] = 0.0
    elif wk == "three_one":
        X = np.array([[0.0], [1.0]])
        w = np.array([3.0, 1.0])
    else:
        w = rng.random(n) + 0.01
    init = None
    if ik == "sample":
        init = X[rng.choice(n, size=m, replace=False)].copy()
    elif ik == "far":      # four centroids far from the data: empty clusters
        init = np.concatenate([X[:m - 4], np.full((4, d), 1e3) + np.arange(4)[:, None]])
    return X, w, init


# evaluation grid points (harness.eval_point): name -> (data seed, n, d,
# structure, notation, codebook seed, anchor_fraction, window, policy,
# controls, per-token mode, wiring, decode_steps)
EVAL_CASES = {
    "e1_heavy_d4m16_decode": (401, 96, 16, "heavy_hitter", "d4m16", 411, 0.05, 8, "by_sum", 2,
                              "joint", "decode", 8),
    "e2_clustered_d8m64_konly": (402, 128, 32, "clustered", "d8m64", 412, 0.02, 0, "by_sum", 1,
                                 "k_only", "prefill", 0),
    "e3_gauss_d2m16_vonly_byk": (403, 80, 16, "gaussian", "d2m16", 413, 0.1, 4, "by_k", 0,
                                 "v_only", "prefill", 0),
}


# BASELINE config #1 at its real shape (tests/golden/make_config1_golden.py):
# one LLaMA-3-8B layer, 32 Q / 8 KV heads, d = 128, 2048-token prefill + 128
# decode steps, d8m256, 1 % anchors by_sum, window 32, LLaMA-3 RoPE base.
CONFIG1 = dict(seed=101, Hq=32, Hkv=8, n=2048, steps=128, d=128, heavy=3, frac=0.01, window=32,
               policy="by_sum", theta=5e5, o_stride=64)
