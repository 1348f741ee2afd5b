"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (it needs /root/reference, which does not exist on
the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are regenerated from seeds (tests/fixtures_gen.py); only reference
outputs are stored, in tests/golden/*.npz.  The oracle restatement
(oracle/antkv_oracle.py) is pinned against these files by tests/test_oracle.py
and the CUDA path is checked against them by tests/test_gpu_parity.py.
"""

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import antkv  # noqa: E402  (the reference)
from antkv import (CacheConfig, Codebook, QuantizedKVCache, VqConfig,  # noqa: E402
                   AnchorScores, select_anchors)
from antkv.kernels import pure  # noqa: E402
from antkv.util import pack_indices  # noqa: E402

from fixtures_gen import (AN_CASES, CACHE_CASES, EVAL_CASES, FA_CASES,  # noqa: E402
                          KM_CASES, an_inputs, codebooks, fa_inputs, km_inputs, qkv)

def run_cache_case(name, spec):
    seed, n, d, notation, window, frac, count, policy, steps, stride, blk = spec
    cfg = VqConfig.from_notation(notation)
    Q, K, V = qkv(seed, 1, 1, n + steps, d, heavy=2)
    Q, K, V = Q[0].astype(np.float64), K[0].astype(np.float64), V[0].astype(np.float64)
    ck, cv = codebooks(seed, 1, cfg.m, cfg.d_sub)
    cache = QuantizedKVCache(
        CacheConfig(vq=cfg, anchor_fraction=frac, anchor_count=count,
                    window_size=window, policy=policy, block_q=blk, block_k=blk),
        Codebook(config=cfg, centroids=ck[0]), Codebook(config=cfg, centroids=cv[0]))
    positions = np.arange(n + steps, dtype=np.int64) * stride
    O = cache.prefill(Q[:n], K[:n], V[:n], positions[:n])
    kinds0 = np.array([{"anchor": 0, "quantized": 1, "windowed": 2}[k] for k in cache.kinds])
    anchors0 = cache.anchor_indices.copy()
    kc0 = np.full((n, d // cfg.d_sub), -1, dtype=np.int64)
    vc0 = np.full((n, d // cfg.d_sub), -1, dtype=np.int64)
    for j, c in cache.k_codes.items():
        kc0[j] = c
        vc0[j] = cache.v_codes[j]
    outs = []
    for t in range(n, n + steps):
        outs.append(cache.decode_step(Q[t], K[t], V[t], int(positions[t])))
    kinds1 = np.array([{"anchor": 0, "quantized": 1, "windowed": 2}[k] for k in cache.kinds])
    N = cache.token_count
    kc1 = np.full((N, d // cfg.d_sub), -1, dtype=np.int64)
    vc1 = np.full((N, d // cfg.d_sub), -1, dtype=np.int64)
    for j, c in cache.k_codes.items():
        kc1[j] = c
        vc1[j] = cache.v_codes[j]
    rep = cache.memory_report()
    # packed wire format of the first quantized token (util.py:19-36)
    qj = [j for j, k in enumerate(cache.kinds) if k == "quantized"]
    packed = np.frombuffer(pack_indices(list(cache.k_codes[qj[0]]) + list(cache.v_codes[qj[0]]),
                                        cfg.index_bits), dtype=np.uint8) if qj else np.zeros(0, np.uint8)
    Qp = np.asarray(Q[:N])
    attn = cache.attention_from_cache(Qp)
    return dict(
        prefill_O=O, kinds0=kinds0, anchors0=anchors0, kcodes0=kc0, vcodes0=vc0,
        decode_out=np.array(outs), kinds1=kinds1, anchors1=cache.anchor_indices.copy(),
        kcodes1=kc1, vcodes1=vc1, positions=positions,
        mem=np.array([rep.payload_bits, rep.codebook_bits, rep.fp_baseline_bits]),
        mem_eff=np.array([rep.effective_bits_per_element]),
        packed_first=packed, attn_from_cache=attn,
    )


def kernel_cases():
    rng = np.random.default_rng(2024)
    out = {}
    for tag, (n, d, bq, bk, seed) in FA_CASES.items():
        Q, K, V = fa_inputs(n, d, seed)
        Qs = Q / np.sqrt(d)
        for causal in (False, True):
            O, L, M = pure.flash_aux(Qs, K, V, bq, bk, causal)
            qn = np.sqrt((Q ** 2).sum(axis=1))
            ak, av = pure.ans_blocked(Qs, K, M, L, qn, bq, bk, causal)
            key = f"{tag}_{int(causal)}"
            out[f"fa_O_{key}"] = O
            out[f"fa_L_{key}"] = L
            out[f"fa_M_{key}"] = M
            out[f"ans_k_{key}"] = ak
            out[f"ans_v_{key}"] = av
    for tag, (N, m, ds, seed) in AN_CASES.items():
        X, C = an_inputs(N, m, ds, seed)
        idx, d2 = pure.assign_nearest(X, C)
        out[f"an_idx_{tag}"] = idx
        out[f"an_d2_{tag}"] = d2
    # selection on random and tied scores
    sk = rng.random(1000)
    sv = rng.random(1000)
    sv[::7] = 0.5
    sk[::11] = 0.25
    out["sel_k"] = sk
    out["sel_v"] = sv
    for policy in ("by_k", "by_v", "by_sum"):
        for budget in (0, 1, 7, 21, 400, 999, 1000, 5000):
            sel = select_anchors(AnchorScores(ans_k=sk, ans_v=sv), budget, policy)
            out[f"sel_{policy}_{budget}"] = sel.indices
    return out


def kmeans_cases():
    """weighted_kmeans (vq.py:141-214) with the reference's compiled
    assign_nearest (oracle/_ref, the backend a built reference uses)."""
    sys.path.insert(0, str(HERE.parent.parent / "oracle" / "_ref"))
    import antkv.kernels as K
    import antkv_ref._ckernels as ck
    saved = K.assign_nearest
    K.assign_nearest = ck.assign_nearest
    out = {}
    try:
        for name, (_, _, _, m, kseed, max_iter, _, _) in KM_CASES.items():
            X, w, init = km_inputs(name)
            res = antkv.vq.weighted_kmeans(X, w, m, seed=kseed, max_iter=max_iter,
                                           init_centroids=init)
            out[f"{name}_C"] = res.codebook.centroids
            out[f"{name}_trace"] = np.array(res.objective_trace)
            out[f"{name}_meta"] = np.array([res.n_iter, int(res.padded_init)])
    finally:
        K.assign_nearest = saved
    return out


def eval_cases():
    """harness.eval_point on small grid points, compiled assign_nearest."""
    import json
    sys.path.insert(0, str(HERE.parent.parent / "oracle" / "_ref"))
    import antkv.kernels as K
    import antkv.harness as H
    import antkv.vq as VQ
    import antkv_ref._ckernels as ck
    saved = (K.assign_nearest, VQ.kernels.assign_nearest)
    K.assign_nearest = ck.assign_nearest
    out = {}
    try:
        for name, spec in EVAL_CASES.items():
            (dseed, n, d, structure, notation, cseed, frac, window, policy, controls, mode,
             wiring, steps) = spec
            cfg = VqConfig.from_notation(notation)
            ck_, cv_ = codebooks(cseed, 1, cfg.m, cfg.d_sub)
            data = H.generate_qkv(dseed, n, d, structure)
            rec = H.eval_point(data, Codebook(config=cfg, centroids=ck_[0]),
                               Codebook(config=cfg, centroids=cv_[0]), frac, window_size=window,
                               policy=policy, seed=dseed, controls=controls, per_token_mode=mode,
                               compute_per_token=True, wiring=wiring, decode_steps=steps)
            rec.pop("runtime_ms")
            errs = H.per_token_errors(data["Q"], data["K"], data["V"],
                                      Codebook(config=cfg, centroids=ck_[0]),
                                      Codebook(config=cfg, centroids=cv_[0]),
                                      H.RopeParams(positions=data["positions"]), mode=mode)
            rec["per_token_errors"] = [float(e) for e in errs]
            rec["data_Q_sum"] = float(np.asarray(data["Q"], np.float64).sum())
            out[name] = rec
    finally:
        K.assign_nearest = saved[0]
    (HERE / "eval.json").write_text(json.dumps(out, indent=1))
    return out


def ref_snapshot_case():
    """A snapshot WRITTEN BY THE REFERENCE (QuantizedKVCache.save,
    cache.py:245-284) of cache case c2 after its prefill and 64 decode steps,
    plus the reference's next 16 decode steps from that state: the GPU cache
    must load the directory (cache.py:286-342 format) and continue
    identically (tests/test_gpu_parity.py::test_load_reference_written_snapshot)."""
    import shutil
    name = "c2_d128_d8m256"
    seed, n, d, notation, window, frac, count, policy, steps, stride, blk = CACHE_CASES[name]
    cfg = VqConfig.from_notation(notation)
    more = 16
    Q, K, V = qkv(seed, 1, 1, n + steps + more, d, heavy=2)
    Q, K, V = Q[0].astype(np.float64), K[0].astype(np.float64), V[0].astype(np.float64)
    ck, cv = codebooks(seed, 1, cfg.m, cfg.d_sub)
    cache = QuantizedKVCache(
        CacheConfig(vq=cfg, anchor_fraction=frac, anchor_count=count, window_size=window,
                    policy=policy, block_q=blk, block_k=blk),
        Codebook(config=cfg, centroids=ck[0]), Codebook(config=cfg, centroids=cv[0]))
    cache.prefill(Q[:n], K[:n], V[:n], np.arange(n))
    for t in range(n, n + steps):
        cache.decode_step(Q[t], K[t], V[t], t)
    out_dir = HERE / "ref_snapshot_c2"
    shutil.rmtree(out_dir, ignore_errors=True)
    cache.save(out_dir)
    outs = [cache.decode_step(Q[t], K[t], V[t], t) for t in range(n + steps, n + steps + more)]
    np.savez_compressed(HERE / "ref_snapshot_c2.npz", decode_out=np.array(outs),
                        anchors=cache.anchor_indices.copy(),
                        kinds=np.array([{"anchor": 0, "quantized": 1, "windowed": 2}[k] for k in cache.kinds]))


def main():
    print("reference backend:", antkv.kernels.BACKEND, file=sys.stderr)
    if sys.argv[1:] == ["snapshot"]:
        ref_snapshot_case()
        return
    np.savez_compressed(HERE / "kernels.npz", **kernel_cases())
    np.savez_compressed(HERE / "kmeans.npz", **kmeans_cases())
    eval_cases()
    for name, spec in CACHE_CASES.items():
        res = run_cache_case(name, spec)
        np.savez_compressed(HERE / f"cache_{name}.npz", **res)
        print(name, "anchors", res["anchors0"], "->", res["anchors1"], file=sys.stderr)
    ref_snapshot_case()
    (HERE / "README.md").write_text(
        "Golden fixtures produced by running the reference `antkv` package\n"
        "(`/root/reference/pkg/src`, kernels backend: "
        f"`{antkv.kernels.BACKEND}`) via `make_golden.py`.\n"
        "Inputs are regenerated from the seeds in `make_golden.py` with\n"
        "`tests/fixtures_gen.py`; only reference outputs are stored.\n"
        "`kmeans.npz` runs `weighted_kmeans` with the reference's compiled\n"
        "`assign_nearest` (`oracle/_ref`, built by `make -C oracle`).\n")


if __name__ == "__main__":
    main()
