"""Pin the oracle restatement against reference outputs (CPU only).

Golden files come from running the reference package itself
(tests/golden/make_golden.py); oracle/_ref holds the reference's own compiled
Cython kernels built from its sources by oracle/Makefile.
"""
import importlib
import sys
from pathlib import Path

import numpy as np
import pytest

import antkv_oracle as O
from fixtures_gen import (AN_CASES, CACHE_CASES, FA_CASES, KM_CASES, an_inputs, codebooks,
                          fa_inputs, km_inputs, qkv)

GOLD = Path(__file__).resolve().parent / "golden"
KER = np.load(GOLD / "kernels.npz")
REF_DIR = Path(__file__).resolve().parent.parent / "oracle" / "_ref"


def _ref_ckernels():
    if not REF_DIR.exists():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    sys.path.insert(0, str(REF_DIR))
    try:
        return importlib.import_module("antkv_ref._ckernels")
    except ImportError as exc:
        pytest.skip(f"oracle/_ref import failed: {exc}")


@pytest.mark.parametrize("tag", list(FA_CASES))
@pytest.mark.parametrize("causal", [0, 1])
def test_flash_aux_and_ans_match_golden(tag, causal):
    n, d, bq, bk, seed = FA_CASES[tag]
    Q, K, V = fa_inputs(n, d, seed)
    Qs = Q / np.sqrt(d)
    Ob, Lb, Mb = O.flash_aux(Qs, K, V, bq, bk, bool(causal))
    key = f"{tag}_{causal}"
    assert np.abs(Ob - KER[f"fa_O_{key}"]).max() < 1e-12
    assert np.abs(Lb - KER[f"fa_L_{key}"]).max() < 1e-11
    assert np.abs(Mb - KER[f"fa_M_{key}"]).max() < 1e-13
    qn = np.sqrt((Q ** 2).sum(axis=1))
    ak, av = O.ans_blocked(Qs, K, Mb, Lb, qn, bq, bk, bool(causal))
    assert np.abs(ak - KER[f"ans_k_{key}"]).max() < 1e-12
    assert np.abs(av - KER[f"ans_v_{key}"]).max() < 1e-12


@pytest.mark.parametrize("tag", list(AN_CASES))
def test_assign_nearest_matches_golden_and_compiled_reference(tag):
    N, m, ds, seed = AN_CASES[tag]
    X, C = an_inputs(N, m, ds, seed)
    idx, d2 = O.assign_nearest(X, C)
    assert np.array_equal(idx, KER[f"an_idx_{tag}"])
    assert np.abs(d2 - KER[f"an_d2_{tag}"]).max() < 1e-12
    ck = _ref_ckernels()
    ridx, rd2 = ck.assign_nearest(X, C)
    assert np.array_equal(idx, ridx)
    assert np.array_equal(d2, rd2)       # same accumulation order -> bitwise


def test_compiled_reference_flash_and_ans_agree_with_oracle():
    ck = _ref_ckernels()
    n, d, bq, bk, seed = FA_CASES["d128"]
    Q, K, V = fa_inputs(n, d, seed)
    Qs = Q / np.sqrt(d)
    for causal in (False, True):
        Oc, Lc, Mc = ck.flash_aux(Qs, K, V, bq, bk, causal)
        Oo, Lo, Mo = O.flash_aux(Qs, K, V, bq, bk, causal)
        assert np.abs(Oc - Oo).max() < 1e-12 and np.abs(Lc - Lo).max() < 1e-10
        qn = np.sqrt((Q ** 2).sum(axis=1))
        kc, vc = ck.ans_blocked(Qs, K, Mc, Lc, qn, bq, bk, causal)
        ko, vo = O.ans_blocked(Qs, K, Mo, Lo, qn, bq, bk, causal)
        assert np.abs(kc - ko).max() < 1e-11 and np.abs(vc - vo).max() < 1e-11


def test_assign_nearest_tie_breaks_low_index():
    C = np.array([[0.0], [2.0], [0.0], [2.0]])
    idx, d2 = O.assign_nearest(np.array([[1.0]]), C)
    assert idx[0] == 0 and d2[0] == 1.0


def test_select_matches_golden():
    sk, sv = KER["sel_k"], KER["sel_v"]
    for policy in ("by_k", "by_v", "by_sum"):
        for budget in (0, 1, 7, 21, 400, 999, 1000, 5000):
            got = O.select_anchors(sk, sv, budget, policy)
            assert np.array_equal(got, KER[f"sel_{policy}_{budget}"]), (policy, budget)


def test_selection_kats():
    # test_anchors.py:113-147
    s_k = np.array([0.1, 9.0, 3.0, 9.0])
    s_v = np.array([5.0, 0.0, 7.0, 1.0])
    assert list(O.select_anchors(s_k, s_v, 2, "by_k")) == [1, 3]
    assert list(O.select_anchors(s_k, s_v, 2, "by_v")) == [0, 2]
    assert list(O.select_anchors(np.array([0.0, 10.0, 5.0, 1.0]),
                                 np.array([10.0, 9.0, 0.0, 0.0]), 2, "by_sum")) == [0, 1]
    assert list(O.select_anchors(np.ones(4), np.array([1.0, 2.0, 2.0, 2.0]), 2, "by_v")) == [1, 2]


def test_budget_kats():
    # test_cache.py:59-64
    assert O.budget_for(200, 0.01) == 2
    assert O.budget_for(50, 0.01) == 1
    assert O.budget_for(50, 0.01, 7) == 7
    assert O.budget_for(50, 0.01, 99) == 50


def test_pack_roundtrip_kat(rng):
    for bits in (1, 3, 8, 12):
        vals = rng.integers(2 ** bits, size=11)
        packed = O.pack_indices(vals, bits)
        assert len(packed) == (11 * bits + 7) // 8
        assert list(O.unpack_indices(packed, bits, 11)) == list(vals)


def _run_oracle_case(name):
    seed, n, d, notation, window, frac, count, policy, steps, stride, blk = CACHE_CASES[name]
    d_sub, m = (int(x) for x in notation[1:].split("m"))
    Q, K, V = qkv(seed, 1, 1, n + steps, d, heavy=2)
    ck, cv = codebooks(seed, 1, m, d_sub)
    cache = O.OracleCache(ck, cv, anchor_fraction=frac, anchor_count=count,
                          window_size=window, policy=policy, block_q=blk, block_k=blk)
    positions = np.arange(n + steps, dtype=np.int64) * stride
    Op = cache.prefill(Q[:, :n], K[:, :n], V[:, :n], positions[:n])
    outs = [cache.decode_step(Q[:, t], K[:, t], V[:, t], int(positions[t]))
            for t in range(n, n + steps)]
    return cache, Op, np.array(outs), Q


@pytest.mark.parametrize("name", list(CACHE_CASES))
def test_oracle_cache_matches_reference_cache(name):
    """Group size 1: the GQA restatement must equal QuantizedKVCache."""
    g = np.load(GOLD / f"cache_{name}.npz")
    cache, Op, outs, Q = _run_oracle_case(name)
    assert np.abs(Op[0] - g["prefill_O"]).max() < 1e-12
    assert np.array_equal(cache.heads[0].anchor_indices, g["anchors1"])
    kinds = np.array([{"anchor": 0, "quantized": 1, "windowed": 2}[k] for k in cache.heads[0].kinds])
    assert np.array_equal(kinds, g["kinds1"])
    for j, c in cache.heads[0].k_codes.items():
        assert np.array_equal(c, g["kcodes1"][j])
        assert np.array_equal(cache.heads[0].v_codes[j], g["vcodes1"][j])
    assert np.abs(outs[:, 0] - g["decode_out"]).max() < 1e-12
    pay, cbb, eff, fp = cache.memory_report(0)
    assert [pay, cbb, fp] == list(g["mem"]) and eff == g["mem_eff"][0]
    attn = cache.attention_from_cache(Q[:, :cache.token_count])
    assert np.abs(attn[0] - g["attn_from_cache"]).max() < 1e-12


@pytest.mark.parametrize("name", list(KM_CASES))
def test_weighted_kmeans_matches_reference_golden(name):
    """The oracle's weighted k-means reproduces the reference run (compiled
    assign_nearest) bit for bit: centroids, objective trace, iterations."""
    g = np.load(GOLD / "kmeans.npz")
    _, _, _, m, kseed, max_iter, _, _ = KM_CASES[name]
    X, w, init = km_inputs(name)
    C, trace, it, padded = O.weighted_kmeans(X, w, m, kseed, max_iter=max_iter, init_centroids=init)
    assert np.array_equal(C, g[f"{name}_C"])
    assert np.array_equal(np.array(trace), g[f"{name}_trace"])
    assert [it, int(padded)] == g[f"{name}_meta"].tolist()
