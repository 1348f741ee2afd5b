"""Per-kernel launch list of a few decode steps on one cache (run under
ncu --metrics gpu__time_duration.sum): which launches make up a step."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from staged_bench import CONFIGS, build  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3_128k_d32m4096"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    notation, B, Hq, Hkv, n = CONFIGS[name]
    cache = build(notation, B, Hq, Hkv, n)
    q = torch.randn((B, Hq, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn((B, Hkv, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((B, Hkv, 128), device="cuda").to(torch.bfloat16)
    out = torch.empty((B, Hq, 128), device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("steps")
    for s in range(steps):
        qp = torch.full((B,), n + s, device="cuda", dtype=torch.int64)
        cache.step_device(q, k, v, qp, out)
        cache._n += 1
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("ok")


if __name__ == "__main__":
    main()
