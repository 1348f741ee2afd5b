"""Encode throughput only (bench.encode_throughput), for quick iterations."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_2506_19505_b200 import _lib
_lib.load()
for _ in range(2):
    print(bench.encode_throughput(torch))
