"""Time codebook training (weighted k-means) at the
paper's calibration scale: 128 x 2048 tokens x 16 groups = 4.19M d8
sub-vectors, m = 256 (d8m256), float64.

GPU: paper_2506_19505_b200.weighted_kmeans (antkv_kmeans_assign_f64 +
antkv_kmeans_update_f64), per Lloyd iteration, with the assignment and
update kernels timed alone by CUDA events.  CPU: the reference's compiled
assign_nearest (oracle/_ref) on a 64K-point sample plus the numpy update,
scaled to the full point count (single core, as the reference runs).

    python tools/kmeans_bench.py [--points N] [--iters K]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=128 * 2048 * 16)
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--d", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--cpu-sample", type=int, default=65536)
    a = ap.parse_args()
    from paper_2506_19505_b200 import _lib, weighted_kmeans
    rng = np.random.default_rng(0)
    X = rng.standard_normal((a.points, a.d))
    w = rng.random(a.points) + 0.01
    init = X[rng.choice(a.points, size=a.m, replace=False)].copy()
    weighted_kmeans(X[:100000], w[:100000], a.m, seed=0, max_iter=2, init_centroids=init)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = weighted_kmeans(X, w, a.m, seed=0, max_iter=a.iters, tol=-1.0, init_centroids=init)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0

    # kernels alone
    dev = torch.device("cuda")
    Xd = torch.from_numpy(X).to(dev)
    wd = torch.from_numpy(w).to(dev)
    Cd = torch.from_numpy(init).to(dev)
    idx = torch.empty((a.points,), dtype=torch.int64, device=dev)
    d2 = torch.empty((a.points,), dtype=torch.float64, device=dev)
    st = _lib.stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for _ in range(2):
        _lib.call("antkv_kmeans_assign_f64", _lib.ptr(Xd), _lib.ptr(Cd), a.points, a.m, a.d,
                  _lib.ptr(idx), _lib.ptr(d2), st)
    ev[0].record()
    for _ in range(5):
        _lib.call("antkv_kmeans_assign_f64", _lib.ptr(Xd), _lib.ptr(Cd), a.points, a.m, a.d,
                  _lib.ptr(idx), _lib.ptr(d2), st)
    ev[1].record()
    perm = torch.argsort(idx, stable=True)
    off = torch.zeros((a.m + 1,), dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(torch.bincount(idx, minlength=a.m), 0)
    Cn = torch.empty_like(Cd)
    ws = torch.empty((a.m,), dtype=torch.float64, device=dev)
    Xs = Xd.index_select(0, perm)
    wsr = wd.index_select(0, perm)
    ev[2].record()
    for _ in range(5):
        _lib.call("antkv_kmeans_update_f64", _lib.ptr(off), _lib.ptr(Xs), _lib.ptr(wsr),
                  _lib.ptr(Cd), a.m, a.d, _lib.ptr(Cn), _lib.ptr(ws), st)
    ev[3].record()
    torch.cuda.synchronize()
    assign_ms = ev[0].elapsed_time(ev[1]) / 5
    update_ms = ev[2].elapsed_time(ev[3]) / 5
    flops = 3.0 * a.points * a.m * a.d

    # CPU reference (compiled assign_nearest) on a sample
    cpu = None
    try:
        sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
        import antkv_ref._ckernels as ck
        S = min(a.cpu_sample, a.points)
        t0 = time.perf_counter()
        ridx, rd2 = ck.assign_nearest(X[:S], init)
        t_assign = time.perf_counter() - t0
        t0 = time.perf_counter()
        wsum = np.bincount(ridx, weights=w[:S], minlength=a.m)
        csum = np.zeros((a.m, a.d))
        np.add.at(csum, ridx, w[:S, None] * X[:S])
        t_update = time.perf_counter() - t0
        cpu = {"iter_s_scaled": (t_assign + t_update) * a.points / S, "sample_points": S,
               "cores": 1, "kind": "reference"}
        # parity on the sample: bitwise
        gi, gd = idx[:S].cpu().numpy(), d2[:S].cpu().numpy()
        cpu["assign_bitwise_equal"] = bool(np.array_equal(gi, ridx) and np.array_equal(gd, rd2))
    except Exception as exc:  # oracle/_ref not built
        cpu = {"unavailable": str(exc)}
    out = {
        "workload": f"weighted k-means d{a.d}m{a.m}, {a.points} points, float64",
        "gpu_iter_ms": 1e3 * wall / res.n_iter, "iters": res.n_iter,
        "assign_ms": assign_ms, "update_ms": update_ms,
        "assign_fp64_tflops": flops / assign_ms / 1e9,
        "cpu_reference": cpu,
    }
    if cpu and "iter_s_scaled" in cpu:
        out["speedup_vs_cpu_iter"] = cpu["iter_s_scaled"] / (wall / res.n_iter)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
