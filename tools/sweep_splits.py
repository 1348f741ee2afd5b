"""Time the fast decode kernel (attend-only and full step) on one 128K-token
d8m256 layer for several CTA counts per head.  Usage: python tools/sweep_splits.py"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--ctx", type=int, default=131072)
    p.add_argument("--splits", default="8,16,24,30,33,37,44,55,74")
    p.add_argument("--layers", type=int, default=8)
    a = p.parse_args()
    args = argparse.Namespace(ctx=a.ctx, layers=a.layers, batch=1, notation="d8m256",
                              kernel="fast", splits=0, steps=50, warmup=50)
    caches, _ = bench.build_layers(args, 0, 1, torch)
    q = torch.randn((1, 32, 128), device="cuda").to(torch.bfloat16)
    qp = torch.tensor([a.ctx + 100], device="cuda", dtype=torch.int64)
    out = torch.empty((1, 32, 128), device="cuda")
    for sp in [int(x) for x in a.splits.split(",")]:
        for c in caches:
            c.splits = sp
            c._ws = None
        for c in caches:
            c.attend_device(q, qp, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            for c in caches:
                c.attend_device(q, qp, out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * len(caches))
        print(f"splits/head={sp:3d}  attend {us:7.1f} us  ({38.86e6 / us / 1e3:6.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
