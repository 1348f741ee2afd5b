import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/oracle')
from fixtures_gen import qkv, codebooks
from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
n = 640
vq = VqConfig.from_notation("d8m256")
cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=10000.0)
B, Hq, Hkv, d, steps = 1, 32, 8, 128, 4
Q, K, V = qkv(21, B * Hq, B * Hkv, n + steps, d, heavy=3)
Q = Q.reshape(B, Hq, n + steps, d); K = K.reshape(B, Hkv, n + steps, d); V = V.reshape(B, Hkv, n + steps, d)
ck, cv = codebooks(21, Hkv, vq.m, vq.d_sub)
cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), batch=B, fast=True)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
cache.prefill(dev(Q[:, :, :n]), dev(K[:, :, :n]), dev(V[:, :, :n]), np.arange(n))
S = 18; rows = B * Hq
for rep in range(6):
    q = dev(Q[:, :, n])
    out = torch.empty((B, Hq, d), device="cuda")
    cache.attend_device(q, torch.tensor([n], device="cuda"), out)
    torch.cuda.synchronize()
    ws = cache._workspace()
    f = ws.view(torch.float32)
    wo = f[: S * rows * d].view(S, rows, d); wm = f[S * rows * d: S * rows * d + S * rows].view(S, rows)
    wl = f[S * rows * d + S * rows: S * rows * d + 2 * S * rows].view(S, rows)
    cnt = ws[-(256 + (8 + 1 + 12 * 8) * 4):].view(torch.int32)[:16].tolist()
    nanh = torch.isnan(out).any(dim=-1)[0].nonzero().flatten().tolist()
    print("rep", rep, "NaN heads", nanh, "cnt", cnt)
    for hq in nanh[:2]:
        m = wm[:, hq].cpu().numpy(); l = wl[:, hq].cpu().numpy(); o = wo[:, hq].cpu().numpy()
        M = np.max(m); wts = np.where(np.isfinite(m), np.exp(m - M), 0)
        ref = (wts[:, None] * o).sum(0) / (wts * l).sum()
        print("  head", hq, "m", np.round(m, 3).tolist())
        print("  l", np.round(l, 2).tolist())
        print("  host combine finite:", np.isfinite(ref).all(), " gpu out sample", out[0, hq, :4].tolist())
