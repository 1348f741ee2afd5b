"""Time harness.eval_point on the GPU at growing
context lengths: d = 128, d8m256, heavy-hitter data, 1% anchors, window 32,
per-token errors (joint) and one random control.  The reference's numpy
eval_point is O(n^3 d) through per_token_errors (measured on this image's
CPU: 1.9 s at n = 256, 11.2 s at n = 512).

    python tools/eval_bench.py [n ...]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_2506_19505_b200 import Codebook, VqConfig
    from paper_2506_19505_b200.harness import eval_point, generate_qkv
    sizes = [int(x) for x in sys.argv[1:]] or [512, 2048, 8192, 16384]
    cfg = VqConfig.from_notation("d8m256")
    rng = np.random.default_rng(0)
    cb = Codebook(cfg, rng.standard_normal((256, 8)).astype(np.float32))
    warm = generate_qkv(1, 256, 128, "heavy_hitter")
    eval_point(warm, cb, cb, 0.01, window_size=32, controls=1)
    for n in sizes:
        data = generate_qkv(5, n, 128, "heavy_hitter")
        torch.cuda.synchronize()
        t = time.perf_counter()
        rec = eval_point(data, cb, cb, 0.01, window_size=32, compute_per_token=True, controls=1)
        torch.cuda.synchronize()
        print(json.dumps({"n": n, "eval_point_s": time.perf_counter() - t,
                          "spearman": rec["ans_rank_agreement"]["spearman"],
                          "attention_l1_error": rec["attention_l1_error"]}))


if __name__ == "__main__":
    main()
