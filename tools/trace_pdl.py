"""Timeline of two consecutive fused decode launches on two different caches
(the CUDA-graph / PDL "early" situation of the bench: layer l then layer
l + 1), ANTKV_TRACE=1.  Prints, on one global-timer axis, when launch B's
CTAs start, pass their wait and start streaming relative to launch A's end."""
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

W = 16


def main():
    args = argparse.Namespace(ctx=131072, layers=2, batch=1, notation="d8m256", kernel="fast",
                              splits=0, steps=8, warmup=8)
    caches, _ = bench.build_layers(args, 0, 1, torch)
    q = torch.randn((1, 32, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn((1, 8, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((1, 8, 128), device="cuda").to(torch.bfloat16)
    out = torch.empty((1, 32, 128), device="cuda")
    graph = "--graph" in sys.argv
    if graph:   # A then B captured once, replayed (the bench's launch mode)
        qp = torch.full((1,), args.ctx, device="cuda", dtype=torch.int64)
        out2 = torch.empty_like(out)
        for c, o in zip(caches, (out, out2)):
            c.attend_device(q, qp, o)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g), _lib.exclusive_stream():
            for c, o in zip(caches, (out, out2)):
                c.attend_device(q, qp, o)
        for _ in range(3):
            g.replay()
    else:
        for i in range(3):
            qp = torch.full((1,), args.ctx + i, device="cuda", dtype=torch.int64)
            for c in caches:
                c.step_device(q, k, v, qp, out)
                c._n += 1
    torch.cuda.synchronize()
    lib = _lib.load()
    n = 2 * W * 32768
    buf = (ctypes.c_ulonglong * n)()
    lib.antkv_debug_trace(buf, n)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 32768, W).astype(np.int64)
    mhz = 1965.0
    # the last launch (B) went to half 1 or 0: B = the one with the later start
    halves = []
    for h in range(2):
        x = a[h][a[h][:, 1] > 0]
        halves.append(x)
    A, B = sorted(halves, key=lambda x: x[:, 1].min())
    t0 = A[:, 1].min()
    def col(x, i):   # absolute us of stamp i (cycles since CTA start, converted)
        return (x[:, 1] - t0) / 1e3 + x[:, i] / mhz
    # SM clock from each CTA's (global timer, clock64) pair at its ticket
    f = (A[:, 12] / ((A[:, 10] - A[:, 1]) / 1e3))
    print(f"A: SM clock from (globaltimer, clock64) at the ticket: med {np.median(f):.0f} MHz "
          f"(min {f.min():.0f}, max {f.max():.0f})")
    mhz = float(np.median(f))   # cycle stamps converted at the measured clock, not the nominal one
    a_end = max(np.max((A[:, 1] - t0) / 1e3 + A[:, 15] / mhz), np.max((A[:, 1] - t0) / 1e3 + A[:, 11] / mhz))
    print(f"A: start {0:.1f}  loop start med {np.median(col(A, 8)):.1f}  loop end med {np.median(col(A, 9)):.1f} "
          f"max {np.max(col(A, 9)):.1f}  partial max {np.max(col(A, 13)):.1f}  A done (combine/commit) {a_end:.1f} us")
    bs = (B[:, 1] - t0) / 1e3
    print(f"B: CTA start min {bs.min():.1f} med {np.median(bs):.1f} max {bs.max():.1f}")
    # per SM: when A's CTA there released its partial vs when B's CTA started
    smA = {int(x[0] & 0xffffffff): (x, i) for i, x in enumerate(A)}
    pairs = []
    for x in B:
        sm = int(x[0] & 0xffffffff)
        if sm in smA:
            ax = smA[sm][0]
            a_part = (ax[1] - t0) / 1e3 + ax[13] / mhz
            a_tick = (ax[10] - t0) / 1e3   # global timer after the ticket / release
            b_start = (x[1] - t0) / 1e3
            pairs.append((a_part, a_tick, b_start, int(ax[0] >> 32)))
    pairs.sort(key=lambda p: p[2])
    print("per SM (A partial, A after ticket, B start, A ticket):")
    for p in pairs[:4] + pairs[len(pairs) // 2:len(pairs) // 2 + 4] + pairs[-4:]:
        print("   %.1f  %.1f  %.1f  %d" % p)
    for i, name in ((2, "state read (pre-wait)"), (5, "before the wait"), (3, "wait passed + q issued"), (14, "angles"), (4, "frames"),
                    (6, "pool done"), (8, "loop start"), (9, "loop end"), (13, "partial")):
        c = col(B, i)
        print(f"B: {name:24s} min {c.min():6.1f} med {np.median(c):6.1f} max {c.max():6.1f} us")


if __name__ == "__main__":
    main()
