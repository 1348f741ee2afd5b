import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig, _lib
from paper_2506_19505_b200 import cache as C
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
vq = VqConfig.from_notation("d8m256")
cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=500000.0)
rng = np.random.default_rng(3)
cbk = rng.standard_normal((8, vq.m, vq.d_sub)).astype(np.float32)
g = torch.Generator(device="cuda").manual_seed(9)
Q = torch.randn((1, 32, n, 128), device="cuda", generator=g).to(torch.bfloat16)
K = torch.randn((1, 8, n, 128), device="cuda", generator=g).to(torch.bfloat16)
V = torch.randn((1, 8, n, 128), device="cuda", generator=g).to(torch.bfloat16)
# wrap the pieces with timers
marks = []
def tm(name, f):
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); marks.append((name, (time.perf_counter() - t0) * 1e3))
        return r
    return w
orig_call = _lib.call
def call(name, *a):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = orig_call(name, *a)
    torch.cuda.synchronize(); marks.append((name, (time.perf_counter() - t0) * 1e3))
    return r
for it in range(2):
    cache = QuantizedKVCache(cfg, Codebook(vq, cbk), Codebook(vq, cbk), batch=1, q_heads=32)
    marks.clear()
    _lib.call = call
    C.select_anchors_device = tm("select_anchors_device", C.select_anchors_device) if it == 0 else C.select_anchors_device
    cache.build_from = tm("build_from", cache.build_from)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cache.prefill(Q, K, V, np.arange(n))
    torch.cuda.synchronize(); tot = (time.perf_counter() - t0) * 1e3
    _lib.call = orig_call
print("total %.1f ms" % tot)
for m in marks: print("  %-40s %8.2f ms" % m)

if len(sys.argv) > 2 and sys.argv[2] == "cprofile":
    import cProfile, pstats
    cache = QuantizedKVCache(cfg, Codebook(vq, cbk), Codebook(vq, cbk), batch=1, q_heads=32)
    torch.cuda.synchronize()
    pr = cProfile.Profile(); pr.enable()
    cache.prefill(Q, K, V, np.arange(n))
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
