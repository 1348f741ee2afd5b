"""Prefill timing (FA + aux, AnS, selection, encode/layout) for one layer of
LLaMA-3-8B attention shapes at several context lengths."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig

import os
vq = VqConfig.from_notation(os.environ.get("NOTATION", "d8m256"))
rng = np.random.default_rng(0)
for n in [int(x) for x in (sys.argv[1:] or ["2048", "8192", "32768"])]:
    cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=500000.0)
    ck = rng.standard_normal((8, vq.m, vq.d_sub)).astype(np.float32)
    cv = rng.standard_normal((8, vq.m, vq.d_sub)).astype(np.float32)
    cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), batch=1, q_heads=32)
    Q = torch.randn((1, 32, n, 128), device="cuda").to(torch.bfloat16)
    K = torch.randn((1, 8, n, 128), device="cuda").to(torch.bfloat16)
    V = torch.randn((1, 8, n, 128), device="cuda").to(torch.bfloat16)
    pos = np.arange(n)
    cache.prefill(Q[:, :, :64], K[:, :, :64], V[:, :, :64], pos[:64])   # warm-up
    for rep in range(2):   # the second, warm, run is reported
        cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), batch=1, q_heads=32)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cache.prefill(Q, K, V, pos)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    flops = 6 * 32 * 128 * n * n / 2
    print(f"{vq}: n={n}: prefill {dt * 1e3:.1f} ms, FA+AnS {flops / dt / 1e12:.1f} TFLOP/s effective")
