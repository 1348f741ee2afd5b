"""Per-CTA timeline of one fused decode launch (ANTKV_TRACE=1).

Words per CTA (decode_fast.cu FK_TRACE_WORDS): 0 smid | ticket << 32, then
global-timer stamps 1 start, 2 barriers ready, 3 prologue loads issued,
4 frames, 5 pool wait, 6 pool done, 7 prepare done, 8 loop start, 9 loop end,
10 partial written, 11 committed (last CTA of a head only).
"""
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

WORDS = 16
NAMES = {1: "start", 2: "barriers", 3: "loads issued", 14: "angles done", 4: "frames", 5: "pool wait",
         6: "pool done", 7: "prepare done", 8: "loop start", 9: "loop end (w0)",
         12: "all warps done", 13: "partial written", 10: "ticket", 15: "combined", 11: "committed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=1)
    cli = ap.parse_args()
    args = argparse.Namespace(ctx=cli.ctx, layers=1, batch=cli.batch, notation="d8m256", kernel="fast",
                              splits=0, steps=8, warmup=8)
    caches, _ = bench.build_layers(args, 0, 1, torch)
    c = caches[0]
    q = torch.randn((cli.batch, 32, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn((cli.batch, 8, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((cli.batch, 8, 128), device="cuda").to(torch.bfloat16)
    out = torch.empty((cli.batch, 32, 128), device="cuda")
    for i in range(3):
        qp = torch.full((cli.batch,), cli.ctx + i, device="cuda", dtype=torch.int64)
        c.step_device(q, k, v, qp, out)
        c._n += 1
    torch.cuda.synchronize()
    lib = _lib.load()
    nmax = 4096
    buf = (ctypes.c_ulonglong * (WORDS * nmax))()
    lib.antkv_debug_trace(buf, WORDS * nmax)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(nmax, WORDS).astype(np.int64)
    ncta = int(np.count_nonzero(a[:, 1]))
    a = a[:ncta]
    splits = ncta // (8 * cli.batch)
    sm = a[:, 0] & 0xffffffff
    # word 1: global timer at the CTA start (ns); the others: SM cycles since
    # the CTA start (clock64); converted at the SM clock
    mhz = float(os.environ.get("SM_MHZ", "1965"))
    start = (a[:, 1] - a[:, 1].min()) / 1e3
    rel = start[:, None] + a / (mhz)
    rel[:, 1] = start
    print("CTAs", ncta, "distinct SMs", len(set(sm.tolist())), "splits per head", splits)
    for i, name in NAMES.items():
        ok = a[:, i] > 0
        if ok.any():
            col = rel[ok, i]
            print(f"{i:2d} {name:14s} min {col.min():6.1f}  med {np.median(col):6.1f}  max {col.max():6.1f} us")
    order = np.argsort(-rel[:, 10])[:6]
    for i in order:
        print(f"  cta {i:3d} split {i % splits:2d} head {i // splits} sm {sm[i]:3d} " +
              " ".join(f"{rel[i, j]:5.1f}" for j in range(1, 11)))


if __name__ == "__main__":
    main()
