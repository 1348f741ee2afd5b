"""Per-CTA timeline of one fused decode launch (ANTKV_TRACE=1)."""
import argparse
import ctypes
import os
import sys
from pathlib import Path

os.environ["ANTKV_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2506_19505_b200 import _lib  # noqa: E402


def main():
    args = argparse.Namespace(ctx=131072, layers=1, batch=1, notation="d8m256", kernel="fast",
                              splits=0, steps=8, warmup=8)
    caches, _ = bench.build_layers(args, 0, 1, torch)
    c = caches[0]
    q = torch.randn((1, 32, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn((1, 8, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((1, 8, 128), device="cuda").to(torch.bfloat16)
    out = torch.empty((1, 32, 128), device="cuda")
    for i in range(3):
        qp = torch.tensor([131072 + i], device="cuda", dtype=torch.int64)
        c.step_device(q, k, v, qp, out)
        c._n += 1
    torch.cuda.synchronize()
    lib = _lib.load()
    lib.antkv_debug_trace.restype = ctypes.c_int
    buf = (ctypes.c_ulonglong * (8 * 296))()
    lib.antkv_debug_trace(buf, 8 * 296)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(296, 8).astype(np.int64)
    sm = a[:, 0] & 0xffffffff
    ticket = a[:, 0] >> 32
    t0 = a[:, 1].min()
    st, lp, pl, dn, cm = [(a[:, i] - t0) / 1e3 for i in (1, 2, 3, 4, 5)]
    print("CTAs", len(a), "distinct SMs", len(set(sm.tolist())))
    cnt = np.bincount(sm, minlength=148)
    print("CTAs per SM histogram", np.bincount(cnt))
    print(f"start  min {st.min():.1f} max {st.max():.1f} us")
    lp = np.where(lp > 1e6, np.nan, lp); lp = np.where(lp < -1e6, np.nan, lp)
    print(f"loop0  min {np.nanmin(lp):.1f} med {np.nanmedian(lp):.1f} max {np.nanmax(lp):.1f}")
    print(f"loop1  min {pl.min():.1f} med {np.median(pl):.1f} max {pl.max():.1f}")
    print(f"done   min {dn.min():.1f} med {np.median(dn):.1f} max {dn.max():.1f}")
    pdone, cbdone = (a[:, 6] - t0) / 1e3, (a[:, 7] - t0) / 1e3
    print(f"pool done min {pdone.min():.1f} med {np.median(pdone):.1f} max {pdone.max():.1f}")
    print(f"cb done   min {cbdone.min():.1f} med {np.median(cbdone):.1f} max {cbdone.max():.1f}")
    last = a[:, 5] > 0
    print("commit (last CTAs):", np.round(cm[last], 1))
    order = np.argsort(-dn)[:8]
    for i in order:
        print(f"  cta {i:3d} split {i % 37:2d} head {i // 37} sm {sm[i]:3d} start {st[i]:6.1f} loop {lp[i]:6.1f} loopend {pl[i]:6.1f} done {dn[i]:6.1f}")


if __name__ == "__main__":
    main()
