"""Compare the tcgen05 anchor-score kernel with the mma.sync one (and time
both) through antkv_prefill_anchor_scores: python tools/ans_tc_check.py [n]."""
import os
import subprocess
import sys
import json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def run(n, hq, hkv, causal_note="causal"):
    import numpy as np
    import torch
    from paper_2506_19505_b200 import _lib
    torch.manual_seed(0)
    B, d = 1, 128
    Q = torch.randn(B, hq, n, d, device="cuda").to(torch.bfloat16)
    K = torch.randn(B, hkv, n, d, device="cuda").to(torch.bfloat16)
    K[:, :, 3] *= 6
    V = torch.randn(B, hkv, n, d, device="cuda").to(torch.bfloat16)
    pos = torch.arange(n, device="cuda")[None].contiguous()
    O = torch.empty(B, hq, n, d, device="cuda")
    M = torch.empty(B, hq, n, device="cuda")
    L = torch.empty_like(M)
    qn = torch.empty_like(M)
    st = _lib.stream()
    _lib.call("antkv_prefill_attention", _lib.ptr(Q), _lib.ptr(K), _lib.ptr(V), _lib.BF16, _lib.ptr(pos),
              B, hq, hkv, n, d, 5e5, _lib.ptr(O), _lib.ptr(M), _lib.ptr(L), _lib.ptr(qn), st)
    ak = torch.empty(B, hkv, n, device="cuda")
    av = torch.empty_like(ak)
    def once():
        _lib.call("antkv_prefill_anchor_scores", _lib.ptr(Q), _lib.ptr(K), _lib.BF16, _lib.ptr(pos),
                  _lib.ptr(M), _lib.ptr(L), _lib.ptr(qn), B, hq, hkv, n, d, 5e5, _lib.ptr(ak),
                  _lib.ptr(av), st)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        once()
    e1.record()
    torch.cuda.synchronize()
    return ak.cpu().numpy(), av.cpu().numpy(), e0.elapsed_time(e1) / 3


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        n, hq, hkv = map(int, sys.argv[2:5])
        import numpy as np
        ak, av, ms = run(n, hq, hkv)
        np.savez(sys.argv[5], ak=ak, av=av, ms=ms)
        sys.exit(0)
    import numpy as np
    for (n, hq, hkv) in [(300, 4, 1), (1000, 8, 2), (4096, 32, 8), (32768, 32, 8)]:
        outs = {}
        for tag, env in (("tc", {}), ("mma", {"ANTKV_NO_TCGEN05": "1"})):
            f = f"/tmp/ans_{tag}_{n}.npz"
            r = subprocess.run([sys.executable, __file__, "--child", str(n), str(hq), str(hkv), f],
                               env={**os.environ, **env}, timeout=300)
            assert r.returncode == 0, (tag, n)
            outs[tag] = np.load(f)
        a, b = outs["tc"], outs["mma"]
        rk = np.abs(a["ak"] - b["ak"]).max() / np.abs(b["ak"]).max()
        rv = np.abs(a["av"] - b["av"]).max() / np.abs(b["av"]).max()
        print(json.dumps({"n": n, "hq": hq, "hkv": hkv, "rel_k": float(rk), "rel_v": float(rv),
                          "tc_ms": float(a["ms"]), "mma_ms": float(b["ms"])}))
