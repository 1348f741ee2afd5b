"""Encode throughput only (bench.encode_throughput) for the code shapes given
as arguments (default d8m256 d32m4096 d16m4096), for quick iterations and
A/B runs (ANTKV_NO_TC_ENC=1: the float32 exhaustive encoder)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_2506_19505_b200 import _lib, VqConfig
_lib.load()
for name in sys.argv[1:] or ["d8m256", "d32m4096", "d16m4096"]:
    vq = VqConfig.from_notation(name)
    n = 131072 if vq.m <= 256 else 32768
    for _ in range(2):
        r = bench.encode_throughput(torch, n=n, vq_m=vq.m, d_sub=vq.d_sub)
    print(name, r)
