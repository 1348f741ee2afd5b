"""Per-phase timing of AnTKVLlama.prefill at 32K (CUDA events per layer):
dense GEMMs vs QuantizedKVCache.prefill, to attribute the prefill time."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2506_19505_b200.llama import AnTKVLlama, LlamaConfig, _rms

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = LlamaConfig(layers=layers)
model = AnTKVLlama(cfg, batch=1, capacity=ctx + 256)
toks = torch.randint(0, cfg.vocab, (1, ctx), device="cuda")
x = model.embed[toks]
pos = np.arange(ctx)
for li, L in enumerate(model.layers):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    q, k, v = model._split(_rms(x, L["n1"]) @ L["wqkv"].t(), ctx)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    ev[1].record()
    o = L["cache"].prefill(q, k, v, pos)
    ev[2].record()
    o = o.transpose(1, 2).reshape(1, ctx, -1).to(torch.bfloat16)
    x = x + o @ L["wo"].t()
    x = model._mlp(L, x)
    ev[3].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"layer {li}: qkv {ev[0].elapsed_time(ev[1]):.1f} ms  cache.prefill "
          f"{ev[1].elapsed_time(ev[2]):.1f} ms  o+mlp {ev[2].elapsed_time(ev[3]):.1f} ms  wall {wall*1e3:.1f} ms")
