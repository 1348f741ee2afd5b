"""Parity at the BASELINE.json configurations' real shapes (GPU, -m gpu).

* config #1 -- one LLaMA-3-8B layer (32 Q / 8 KV heads, d = 128), 2048-token
  prefill + 128 decode steps, d8m256, 1 % anchors: the fused, staged and
  generic decode kernels against the committed oracle golden
  (tests/golden/config1.npz, make_config1_golden.py): prefill output rows,
  anchors per KV head, kinds, prefill codes, all 128 decode outputs, the
  codes of every token evicted during decode, anchors / kinds / memory after.
* config #4 -- LLaMA-2-7B MHA shapes (32 / 32 heads), d4m256 (2 bit),
  batch 16 x 8K context: the whole batch on the GPU, sampled (sequence, head)
  pairs through the single-head oracle (which for MHA is exactly the
  reference, cache.py:100-194).
* config #5 positions -- the tail shard of an 8-way 840K context (tokens at
  positions 735K..840K, token_offset = 735K) through the fused decode kernel.
* 128K prefill (north_star: FA + online AnS + top-k at 128K) -- the anchor
  scores and anchor sets of QuantizedKVCache.prefill at 131072 tokens, 32 Q /
  8 KV heads, against the float64 torch restatement tests/fp64_ans.py (pinned
  to the oracle in the CPU suite, and again here at 2K on the GPU).

Rules (north_star), written in the tests:
  * anchor sets: the GPU's selection is exact on its own float32 scores
    (the oracle's selection rerun on them gives the same set); the scores
    agree with the oracle's within the reference's 1e-4 relative AnS
    tolerance; a token may differ from the oracle's set only if its oracle
    score lies within twice the MEASURED score error of the selection
    boundary.  If the sets differ, the oracle is rerun with the GPU's anchors
    so that every downstream check still runs against the reference
    algorithm.
  * codes: bit-exact except where the float64 distance margin is below
    1e-6 (|x|^2 + max|c|^2).
  * outputs: <= 2e-2 relative for the fp16 tensor-core kernels (fused,
    staged), <= 1e-3 for the float32 generic kernel, per decode step, as
    max|o - o_ref| / max|o_ref| over the step's heads.

Every test appends its observed maxima to gpurun_out/parity_errors.jsonl
(ANTKV_PARITY_LOG overrides) -- the table committed under profiles/.
"""

import json
import os
import time
from pathlib import Path

import numpy as np
import pytest
import torch

import antkv_oracle as O
from fixtures_gen import CONFIG1, codebooks, qkv

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLD = Path(__file__).resolve().parent / "golden"
KIND = {"anchor": 0, "quantized": 1, "windowed": 2}
TOL = {"fused": 2e-2, "staged": 2e-2, "generic": 1e-3}
FAST = {"fused": True, "staged": "staged", "generic": False}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_19505_b200 import _lib
    _lib.load()


def record(test, **vals):
    path = Path(os.environ.get("ANTKV_PARITY_LOG", ROOT / "gpurun_out" / "parity_errors.jsonl"))
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps({"test": test, **vals}) + "\n")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def code_flips(X, C, got, ref):
    """Number of sub-vectors whose code differs; asserts each difference is
    a float32-margin tie (SURVEY.md §8c rule 1)."""
    C = np.asarray(C, np.float64)
    X = np.asarray(X, np.float64).reshape(-1, C.shape[1])
    got = np.asarray(got).reshape(-1)
    ref = np.asarray(ref).reshape(-1)
    bad = np.flatnonzero(got != ref)
    if bad.size:
        scale = (X[bad] ** 2).sum(1) + (C ** 2).sum(1).max()
        dg = ((X[bad] - C[got[bad]]) ** 2).sum(1)
        dr = ((X[bad] - C[ref[bad]]) ** 2).sum(1)
        assert np.all(np.abs(dg - dr) <= 1e-6 * scale), (bad[:5], dg[:5], dr[:5])
    return int(bad.size)


def check_anchor_set(got, ref, sk, sv, gk, gv, budget, policy):
    """Anchor-set rule (module docstring).  Returns (tokens in the ambiguity
    band, tokens that differ, relative score errors)."""
    got = np.asarray(got, np.int64)
    ref = np.asarray(ref, np.int64)
    # the GPU's integer selection is exact on its own scores
    again = O.select_anchors(np.asarray(gk, np.float64), np.asarray(gv, np.float64), budget, policy)
    assert np.array_equal(got, again), "selection not exact on the GPU's own scores"
    errk = float(np.abs(gk - sk).max())
    errv = float(np.abs(gv - sv).max())
    rk, rv = errk / np.abs(sk).max(), errv / np.abs(sv).max()
    assert rk < 1e-4 and rv < 1e-4, (rk, rv)          # test_anchors.py:73-110 tolerance
    band = 0
    diff = set(got.tolist()) ^ set(ref.tolist())
    for s, err in ((sk, errk), (sv, errv)):
        if len(ref):
            b = s[ref].min()
            band += int((np.abs(s - b) <= 2 * err).sum())
    for j in diff:
        ok = any(len(ref) and abs(s[j] - s[ref].min()) <= 2 * err for s, err in ((sk, errk), (sv, errv)))
        assert ok, f"anchor {j} differs beyond twice the measured score error"
    return band, len(diff), rk, rv


# -------------------------------------------------------------- config #1
@pytest.fixture(scope="module")
def config1():
    c = CONFIG1
    Q, K, V = qkv(c["seed"], c["Hq"], c["Hkv"], c["n"] + c["steps"], c["d"], heavy=c["heavy"])
    ck, cv = codebooks(c["seed"], c["Hkv"], 256, 8)
    return Q, K, V, ck, cv, np.load(GOLD / "config1.npz")


@pytest.mark.parametrize("kernel", ["fused", "staged", "generic"])
def test_config1_full_shape_vs_oracle_golden(kernel, config1):
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    Q, K, V, ck, cv, g = config1
    c = CONFIG1
    n, steps, Hkv = c["n"], c["steps"], c["Hkv"]
    vq = VqConfig(8, 256)
    cfg = CacheConfig(vq=vq, anchor_fraction=c["frac"], window_size=c["window"], policy=c["policy"],
                      theta_base=c["theta"])
    cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), fast=FAST[kernel])
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    t0 = time.time()
    Og = cache.prefill(dev(Q[None, :, :n]), dev(K[None, :, :n]), dev(V[None, :, :n]), np.arange(n))
    e_pre = rel(Og[0][:, g["prefill_rows"]].cpu().numpy(), g["prefill_O"])
    assert e_pre < 1e-4
    # ---- anchors per KV head
    gk, gv = (x[0].cpu().numpy().astype(np.float64) for x in cache.last_scores)
    budget = cfg.budget_for(n)
    anchors = [cache.anchor_indices_of(0, h) for h in range(Hkv)]
    band = ndiff = 0
    rk = rv = 0.0
    for h in range(Hkv):
        b_, d_, rk_, rv_ = check_anchor_set(anchors[h], g["anchors0"][h], g["scores_k"][h],
                                            g["scores_v"][h], gk[h], gv[h], budget, c["policy"])
        band, ndiff, rk, rv = band + b_, ndiff + d_, max(rk, rk_), max(rv, rv_)
    forced = ndiff > 0
    if forced:
        # the oracle replays layout, decode and eviction from the GPU's anchors
        ref = O.OracleCache(ck, cv, anchor_fraction=c["frac"], window_size=c["window"],
                            policy=c["policy"], theta_base=c["theta"])
        ref.prefill(None, K[:, :n], V[:, :n], np.arange(n), anchors=anchors)
        want_out = np.array([ref.decode_step(Q[:, t], K[:, t], V[:, t], t) for t in range(n, n + steps)])
        want_kinds0 = None
        want_kinds1 = np.array([[KIND[k] for k in hs.kinds] for hs in ref.heads])
        want_codes = np.zeros_like(g["codes1"])
        for hk, hs in enumerate(ref.heads):
            for j, code in hs.k_codes.items():
                want_codes[hk, j, 0], want_codes[hk, j, 1] = code, hs.v_codes[j]
        want_anchors1 = [hs.anchor_indices for hs in ref.heads]
        want_mem = [ref.memory_report(h)[0] for h in range(Hkv)]
    else:
        want_out = g["decode_out"]
        want_kinds0 = g["kinds0"]
        want_kinds1 = g["kinds1"]
        want_codes = g["codes1"]
        want_anchors1 = [a[a >= 0] for a in g["anchors1"]]
        want_mem = list(g["mem"])
    # ---- layout and prefill codes
    flips0 = 0
    kinds0 = [cache.kinds_array(0, h) for h in range(Hkv)]
    for h in range(Hkv):
        if want_kinds0 is not None:
            assert np.array_equal(kinds0[h], want_kinds0[h])
        arr = cache.codes_array(0, h)
        q = np.flatnonzero(kinds0[h] == KIND["quantized"])
        flips0 += code_flips(K[h, q], ck[h], arr[q, 0], want_codes[h, q, 0])
        flips0 += code_flips(V[h, q], cv[h], arr[q, 1], want_codes[h, q, 1])
    # ---- 128 decode steps
    errs = []
    for i, t in enumerate(range(n, n + steps)):
        o = cache.decode_step(dev(Q[None, :, t]), dev(K[None, :, t]), dev(V[None, :, t]), t)
        errs.append(rel(o[0].cpu().numpy(), want_out[i]))
    assert max(errs) < TOL[kernel], (int(np.argmax(errs)), max(errs))
    # ---- state after decode: anchors (promotions), kinds, evicted-token codes
    flips_ev = evicted = 0
    for h in range(Hkv):
        assert np.array_equal(cache.anchor_indices_of(0, h), want_anchors1[h]), h
        k1 = cache.kinds_array(0, h)
        assert np.array_equal(k1, want_kinds1[h]), h
        arr = cache.codes_array(0, h)
        k0 = np.full(len(k1), -1)
        k0[:n] = kinds0[h]
        ev = np.flatnonzero((k1 == KIND["quantized"]) & (k0 != KIND["quantized"]))
        evicted += len(ev)
        flips_ev += code_flips(K[h, ev], ck[h], arr[ev, 0], want_codes[h, ev, 0])
        flips_ev += code_flips(V[h, ev], cv[h], arr[ev, 1], want_codes[h, ev, 1])
        assert cache.memory_report(0, h).payload_bits == want_mem[h]
    assert evicted > 0
    record(f"config1[{kernel}]", prefill_O_rel=e_pre, ans_k_rel=rk, ans_v_rel=rv,
           anchors_band_tokens=band, anchors_differ=ndiff, oracle_rerun=forced,
           prefill_code_flips=flips0, evicted_tokens=evicted, evicted_code_flips=flips_ev,
           decode_max_rel=max(errs), decode_mean_rel=float(np.mean(errs)), tol=TOL[kernel],
           seconds=time.time() - t0)


# -------------------------------------------------------------- config #4
def test_config4_mha_d4m256_batch16_8k():
    """LLaMA-2-7B MHA shapes, 2-bit d4m256, batch 16 x 8K: GPU prefill and
    decode of the whole batch; 3 sampled (sequence, head) pairs through the
    oracle (single head = the reference algorithm)."""
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    B, H, n, d, steps = 16, 32, 8192, 128, 6
    vq = VqConfig.from_notation("d4m256")
    cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, policy="by_sum", theta_base=1e4)
    ck, cv = codebooks(404, H, 256, 4)
    gen = torch.Generator(device="cuda").manual_seed(404)
    shape = (B, H, n + steps, d)
    Q = torch.randn(shape, device="cuda", generator=gen).to(torch.bfloat16)
    K = torch.randn(shape, device="cuda", generator=gen).to(torch.bfloat16)
    V = torch.randn(shape, device="cuda", generator=gen).to(torch.bfloat16)
    cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), batch=B)
    t0 = time.time()
    Og = cache.prefill(Q[:, :, :n], K[:, :, :n], V[:, :, :n], np.arange(n))
    outs = [cache.decode_step(Q[:, :, t], K[:, :, t], V[:, :, t], t).cpu().numpy()
            for t in range(n, n + steps)]
    t_gpu = time.time() - t0
    gk, gv = (x.cpu().numpy().astype(np.float64) for x in cache.last_scores)
    res = {}
    for b, h in ((0, 0), (7, 13), (15, 31)):
        Qh = Q[b, h].float().cpu().numpy().astype(np.float64)
        Kh = K[b, h].float().cpu().numpy().astype(np.float64)
        Vh = V[b, h].float().cpu().numpy().astype(np.float64)
        ref = O.OracleCache([ck[h]], [cv[h]], anchor_fraction=0.01, window_size=32, policy="by_sum",
                            theta_base=1e4)
        Or = ref.prefill(Qh[None, :n], Kh[None, :n], Vh[None, :n], np.arange(n))
        e_pre = rel(Og[b, h].cpu().numpy(), Or[0])
        assert e_pre < 1e-4
        sk, sv = ref.last_scores
        got = np.asarray(cache.anchor_indices_of(b, h))
        band, ndiff, rk, rv = check_anchor_set(got, ref.heads[0].anchor_indices, sk[0], sv[0], gk[b, h],
                                               gv[b, h], cfg.budget_for(n), "by_sum")
        if ndiff:
            ref = O.OracleCache([ck[h]], [cv[h]], anchor_fraction=0.01, window_size=32, policy="by_sum",
                                theta_base=1e4)
            ref.prefill(None, Kh[None, :n], Vh[None, :n], np.arange(n), anchors=[got])
        errs = []
        for i, t in enumerate(range(n, n + steps)):
            r = ref.decode_step(Qh[None, t], Kh[None, t], Vh[None, t], t)
            errs.append(rel(outs[i][b, h], r[0]))
        assert max(errs) < 2e-2, errs
        # state after the decode steps (the GPU cache has run them all)
        kinds = cache.kinds_array(b, h)
        assert np.array_equal(kinds, [KIND[k] for k in ref.heads[0].kinds])
        assert np.array_equal(cache.anchor_indices_of(b, h), ref.heads[0].anchor_indices)
        arr = cache.codes_array(b, h)
        q = np.flatnonzero(kinds == KIND["quantized"])
        wk = np.array([ref.heads[0].k_codes[j] for j in q])
        wv = np.array([ref.heads[0].v_codes[j] for j in q])
        flips = code_flips(Kh[q], ck[h], arr[q, 0], wk) + code_flips(Vh[q], cv[h], arr[q, 1], wv)
        res[f"b{b}h{h}"] = dict(prefill_O_rel=e_pre, ans_rel=max(rk, rv), band=band, anchors_differ=ndiff,
                                code_flips=flips, decode_max_rel=max(errs))
    record("config4[staged, B16 MHA d4m256 8K]", gpu_seconds=t_gpu, **res)


# ------------------------------------------------ config #5 positions (840K)
def test_config5_tail_shard_positions_735k_840k():
    """The last of 8 sequence shards of an 840K-token context: tokens at
    global positions 735K..840K (token_offset 735K), d8m256, through the
    fused decode kernel (append / attend / evict at position 840K+) vs the
    oracle holding the same rows, codes and anchors at the same positions."""
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    Hq, Hkv, d, steps = 8, 2, 128, 6
    off, n = 735000, 105000
    vq = VqConfig(8, 256)
    rng = np.random.default_rng(840)
    anchors = [np.sort(rng.choice(n - 64, size=n // 100, replace=False)) for _ in range(Hkv)]
    count = n // 100 + 2                          # two promotions, then encodes
    cfg = CacheConfig(vq=vq, anchor_count=count, window_size=32, theta_base=5e5)
    ck, cv = codebooks(840, Hkv, 256, 8)
    gen = torch.Generator(device="cuda").manual_seed(840)
    Q = torch.randn((1, Hq, steps, d), device="cuda", generator=gen).to(torch.bfloat16)
    K = torch.randn((1, Hkv, n + steps, d), device="cuda", generator=gen).to(torch.bfloat16)
    V = torch.randn((1, Hkv, n + steps, d), device="cuda", generator=gen).to(torch.bfloat16)
    pos = torch.arange(off, off + n, device="cuda")[None]
    cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), q_heads=Hq, token_offset=off,
                             capacity=n + 256)
    A = torch.from_numpy(np.stack(anchors).astype(np.int32)).cuda()[None]
    cache.Hq = Hq
    cache.build_from(K[:, :, :n], V[:, :, :n], pos, A)
    Kh = K[0].float().cpu().numpy().astype(np.float64)
    Vh = V[0].float().cpu().numpy().astype(np.float64)
    Qh = Q[0].float().cpu().numpy().astype(np.float64)
    # codes of the GPU cache feed the oracle; a random sample is checked by
    # the margin rule against the oracle's own encoder
    codes, flips = [], 0
    for h in range(Hkv):
        arr = cache.codes_array(0, h)
        codes.append((arr[:, 0], arr[:, 1]))
        kinds = cache.kinds_array(0, h)
        q = np.flatnonzero(kinds == KIND["quantized"])
        smp = np.sort(rng.choice(q, size=2000, replace=False))
        flips += code_flips(Kh[h, smp], ck[h], arr[smp, 0], O.encode_rows(Kh[h, smp], ck[h]))
        flips += code_flips(Vh[h, smp], cv[h], arr[smp, 1], O.encode_rows(Vh[h, smp], cv[h]))
    ref = O.OracleCache(ck, cv, anchor_count=count, window_size=32, theta_base=5e5)
    ref.prefill(None, Kh[:, :n], Vh[:, :n], np.arange(off, off + n), anchors=anchors, codes=codes)
    errs = []
    for s in range(steps):
        p = off + n + s
        o = cache.decode_step(Q[:, :, s], K[:, :, n + s], V[:, :, n + s], p)
        r = ref.decode_step(Qh[:, s], Kh[:, n + s], Vh[:, n + s], p)
        errs.append(rel(o[0].cpu().numpy(), r))
    assert max(errs) < 2e-2, errs
    for h in range(Hkv):
        assert np.array_equal(cache.anchor_indices_of(0, h), ref.heads[h].anchor_indices)
    record("config5[fused, positions 735K-840K]", code_flips_sample=flips, decode_max_rel=max(errs))


def test_prefill_anchors_128k_vs_fp64():
    """QuantizedKVCache.prefill at 131072 tokens (LLaMA-3-8B attention shapes,
    bf16, heavy-hitter keys planted per KV head): the tcgen05 FA + AnS scores
    of every KV head within the reference's 1e-4 relative AnS tolerance of a
    float64 restatement of Alg. 1, and the anchor sets equal except tokens
    within twice the measured score error of the selection boundary
    (anchors.py:66-132, cache.py:100-140).  The restatement itself is
    checked against the oracle at 2K first."""
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from fp64_ans import group_anchor_scores
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    Hq, Hkv, d = 32, 8, 128
    g = Hq // Hkv
    vq = VqConfig(8, 256)
    ck, cv = codebooks(128, Hkv, 256, 8)
    cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=5e5)
    # 2K: fp64 restatement vs the oracle's GQA scores
    Q2, K2, V2 = qkv(1282, Hq, Hkv, 2048, d, heavy=8)
    ref2 = O.OracleCache(ck, cv, anchor_fraction=0.01, window_size=32, theta_base=5e5)
    ref2.prefill(Q2, K2, V2, np.arange(2048))
    for hk in range(Hkv):
        sk, sv = group_anchor_scores(torch.from_numpy(Q2[hk * g:(hk + 1) * g]).cuda(),
                                     torch.from_numpy(K2[hk]).cuda(), torch.arange(2048, device="cuda"),
                                     theta_base=5e5)
        assert rel(sk.cpu().numpy(), ref2.last_scores[0][hk]) < 1e-12
        assert rel(sv.cpu().numpy(), ref2.last_scores[1][hk]) < 1e-12
    # 128K through the GPU prefill
    n = 131072
    gen = torch.Generator(device="cuda").manual_seed(128)
    Q = torch.randn((1, Hq, n, d), device="cuda", generator=gen).to(torch.bfloat16)
    K = torch.randn((1, Hkv, n, d), device="cuda", generator=gen).to(torch.bfloat16)
    V = torch.randn((1, Hkv, n, d), device="cuda", generator=gen).to(torch.bfloat16)
    for h in range(Hkv):   # heavy hitters: 64 early large-norm keys per head
        idx = torch.randperm(n // 2, generator=torch.Generator().manual_seed(h))[:64].cuda()
        K[0, h, idx] = (K[0, h, idx].float() * 5.0).to(torch.bfloat16)
    cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), q_heads=Hq)
    t0 = time.time()
    cache.prefill(Q, K, V, np.arange(n))
    torch.cuda.synchronize()
    gk_all, gv_all = (x[0].double().cpu().numpy() for x in cache.last_scores)
    budget = cfg.budget_for(n)
    pos = torch.arange(n, device="cuda")
    bands, diffs, rks, rvs = [], [], [], []
    for hk in range(Hkv):
        sk, sv = group_anchor_scores(Q[0, hk * g:(hk + 1) * g], K[0, hk], pos, theta_base=5e5)
        sk, sv = sk.cpu().numpy(), sv.cpu().numpy()
        ref_set = O.select_anchors(sk, sv, budget, cfg.policy)
        got = np.asarray(cache.anchor_indices_of(0, hk), np.int64)
        band, diff, rk, rv = check_anchor_set(got, ref_set, sk, sv, gk_all[hk], gv_all[hk], budget, cfg.policy)
        bands.append(band)
        diffs.append(diff)
        rks.append(rk)
        rvs.append(rv)
    record("prefill 128K anchors vs fp64 (32/8 heads, d8m256 cache, 1% anchors)",
           ans_rel_k=max(rks), ans_rel_v=max(rvs), band_tokens=sum(bands), differing=sum(diffs),
           budget_per_head=budget, wall_s=round(time.time() - t0, 1))
