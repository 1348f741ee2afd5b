"""One d8m256 encode launch set (bench.encode_throughput shape) for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_2506_19505_b200 import _lib, VqConfig
_lib.load()
vq = VqConfig.from_notation(sys.argv[1] if len(sys.argv) > 1 else "d8m256")
bench.encode_throughput(torch, n=131072 if vq.m <= 256 else 32768, reps=1, vq_m=vq.m, d_sub=vq.d_sub)
torch.cuda.synchronize()
