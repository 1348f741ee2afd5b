"""Compare the tcgen05 attention kernel with the mma.sync one (O, M, L) and
time both through antkv_prefill_attention: python tools/flash_tc_check.py"""
import os
import subprocess
import sys
import json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def run(n, hq, hkv, seed=0):
    import torch
    from paper_2506_19505_b200 import _lib
    torch.manual_seed(seed)
    B, d = 1, 128
    Q = (torch.randn(B, hq, n, d, device="cuda") * 2).to(torch.bfloat16)
    K = torch.randn(B, hkv, n, d, device="cuda").to(torch.bfloat16)
    K[:, :, 3] *= 6
    V = torch.randn(B, hkv, n, d, device="cuda").to(torch.bfloat16)
    pos = torch.arange(n, device="cuda")[None].contiguous()
    O = torch.empty(B, hq, n, d, device="cuda")
    M = torch.empty(B, hq, n, device="cuda")
    L = torch.empty_like(M)
    qn = torch.empty_like(M)
    st = _lib.stream()
    def once():
        _lib.call("antkv_prefill_attention", _lib.ptr(Q), _lib.ptr(K), _lib.ptr(V), _lib.BF16, _lib.ptr(pos),
                  B, hq, hkv, n, d, 5e5, _lib.ptr(O), _lib.ptr(M), _lib.ptr(L), _lib.ptr(qn), st)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        once()
    e1.record()
    torch.cuda.synchronize()
    return O.cpu().numpy(), M.cpu().numpy(), L.cpu().numpy(), e0.elapsed_time(e1) / 3


if __name__ == "__main__":
    import numpy as np
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        n, hq, hkv = map(int, sys.argv[2:5])
        O, M, L, ms = run(n, hq, hkv)
        np.savez(sys.argv[5], O=O, M=M, L=L, ms=ms)
        sys.exit(0)
    sizes = [(300, 4, 1), (1000, 8, 2), (4096, 32, 8), (32768, 32, 8)]
    if len(sys.argv) > 1:
        sizes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
    for (n, hq, hkv) in sizes:
        outs = {}
        for tag, env in (("tc", {}), ("mma", {"ANTKV_NO_TCGEN05": "1"})):
            f = f"/tmp/fa_{tag}_{n}.npz"
            r = subprocess.run([sys.executable, __file__, "--child", str(n), str(hq), str(hkv), f],
                               env={**os.environ, **env}, timeout=300)
            assert r.returncode == 0, (tag, n)
            outs[tag] = np.load(f)
        a, b = outs["tc"], outs["mma"]
        ro = np.abs(a["O"] - b["O"]).max() / np.abs(b["O"]).max()
        rm = np.abs(a["M"] - b["M"]).max()
        rl = np.abs(a["L"] / b["L"] - 1).max()
        print(json.dumps({"n": n, "O_rel": float(ro), "M_abs": float(rm), "L_rel": float(rl),
                          "finite": bool(np.isfinite(a["O"]).all()),
                          "tc_ms": float(a["ms"]), "mma_ms": float(b["ms"])}))
