"""Decode-attention time per layer-step of the three kernels (fused d8m256,
staged tensor-core, generic float32) on BASELINE-shaped caches.

  python tools/staged_bench.py [--configs cfg3,cfg4,...] [--reps 20]

Each config: one layer's cache (random bf16 K/V, random codebooks, 1 %
anchors from the top-k kernel), attention-only launches replayed from a CUDA
graph, CUDA events around the replay.  Prints one JSON line per (config,
kernel) with the algorithmic bytes and the HBM fraction.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

CONFIGS = {
    # name: (notation, batch, Hq, Hkv, ctx)
    "cfg1_128k_d8m256": ("d8m256", 1, 32, 8, 131072),
    "cfg3_128k_d32m4096": ("d32m4096", 1, 32, 8, 131072),
    "cfg4_b16_8k_d4m256_mha": ("d4m256", 16, 32, 32, 8192),
    "d16m4096_128k": ("d16m4096", 1, 32, 8, 131072),
    "d4m256_128k": ("d4m256", 1, 32, 8, 131072),
}


def build(notation, B, Hq, Hkv, n, seed=5):
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    from paper_2506_19505_b200.anchors import select_anchors_device
    vq = VqConfig.from_notation(notation)
    cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=5e5)
    rng = np.random.default_rng(seed)
    ck = rng.standard_normal((Hkv, vq.m, vq.d_sub)).astype(np.float32)
    cv = rng.standard_normal((Hkv, vq.m, vq.d_sub)).astype(np.float32)
    cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), batch=B, q_heads=Hq,
                             capacity=n + 64)
    g = torch.Generator(device="cuda").manual_seed(seed)
    K = torch.randn((B, Hkv, n, 128), device="cuda", generator=g).to(torch.bfloat16)
    V = torch.randn((B, Hkv, n, 128), device="cuda", generator=g).to(torch.bfloat16)
    budget = cfg.budget_for(n)
    sk = torch.rand((B * Hkv, n), device="cuda", generator=g)
    sv = torch.rand((B * Hkv, n), device="cuda", generator=g)
    anchors = select_anchors_device(sk, sv, budget).view(B, Hkv, budget)
    pos = torch.arange(n, device="cuda", dtype=torch.int64)[None].repeat(B, 1)
    cache.build_from(K, V, pos, anchors)
    del K, V
    return cache


def alg_bytes(cache):
    vq = cache.config.vq
    n = cache.token_count
    code_b = 2 * (128 // vq.d_sub) * vq.index_bits / 8.0
    nfp = int((cache.tensors["pool_kind"] >= 0).sum())
    return ((cache.B * cache.Hkv * n - nfp) * code_b + nfp * 2 * 128 * 2
            + cache.B * 2 * cache.Hq * 128 * 2 + cache.Hkv * 2 * vq.m * vq.d_sub * 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(CONFIGS))
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--kernels", default="1,2,0")
    ap.add_argument("--splits", type=int, default=0, help="CTAs per (sequence, head); 0 = the library's plan")
    a = ap.parse_args()
    peak = 6552.3
    try:
        peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json")
                          .read_text())["hbm_gbs"]
    except Exception:  # noqa: BLE001
        pass
    for name in a.configs.split(","):
        notation, B, Hq, Hkv, n = CONFIGS[name]
        cache = build(notation, B, Hq, Hkv, n)
        if a.splits:
            cache.splits = a.splits
        q = torch.randn((B, Hq, 128), device="cuda").to(torch.bfloat16)
        qp = torch.full((B,), n + 3, device="cuda", dtype=torch.int64)
        out = torch.empty((B, Hq, 128), device="cuda", dtype=torch.float32)
        ab = alg_bytes(cache)
        res = {}
        for mode in [int(x) for x in a.kernels.split(",")]:
            if mode == 1 and not (notation == "d8m256" and Hq == 4 * Hkv):
                continue   # mode 1 == staged for every other shape
            reps = a.reps if mode else max(2, a.reps // 10)
            cache.attend_device(q, qp, out, fast=mode)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for _ in range(reps):
                    cache.attend_device(q, qp, out, fast=mode)
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            res[mode] = out.clone()
            gbs = ab / (us * 1e-6) / 1e9
            print(json.dumps({"config": name, "kernel": {0: "generic", 1: "fused", 2: "staged"}[mode],
                              "us_per_layer_step": round(us, 2), "alg_MB": round(ab / 1e6, 2),
                              "GBs": round(gbs, 1), "frac": round(gbs / peak, 4)}), flush=True)
        if 0 in res:
            for m, o in res.items():
                if m:
                    err = ((o - res[0]).abs().max() / res[0].abs().max()).item()
                    print(json.dumps({"config": name, "kernel": m, "rel_err_vs_generic": err}))
        del cache
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
