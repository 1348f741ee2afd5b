"""BASELINE config #2: LLaMA-3-8B shapes (random init), batch 1, a long
synthetic context prefilled through AnTKV, then CUDA-graph decode steps.
Reports prefill time, decode tokens/s and the attention share of a step."""
import argparse
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2506_19505_b200.llama import AnTKVLlama, LlamaConfig

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--notation", default="d8m256")
args = ap.parse_args()
cfg = LlamaConfig(layers=args.layers, notation=args.notation)
model = AnTKVLlama(cfg, batch=1, capacity=args.ctx + args.steps + 256)
g = torch.Generator(device="cuda").manual_seed(0)
toks = torch.randint(0, cfg.vocab, (1, args.ctx), device="cuda", generator=g)
torch.cuda.synchronize()
t0 = time.perf_counter()
logits = model.prefill(toks)
torch.cuda.synchronize()
t_cold = time.perf_counter() - t0
model.reset()                       # the same prompt again: warm allocator, cuBLAS, kernels
t0 = time.perf_counter()
logits = model.prefill(toks)
torch.cuda.synchronize()
t_prefill = time.perf_counter() - t0
tok = logits.argmax(-1)
qpos = torch.full((1,), model.pos, dtype=torch.int64, device="cuda")
logits = model.decode_device(tok, qpos)         # warm-up (eager)
model.advance(1)
qpos.add_(1)
graph = torch.cuda.CUDAGraph()
tok_st = logits.argmax(-1)
with torch.cuda.graph(graph):
    out = model.decode_device(tok_st, qpos)
    tok_st.copy_(out.argmax(-1))
    qpos.add_(1)
for _ in range(3):
    graph.replay()
model.advance(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    graph.replay()
e1.record()
torch.cuda.synchronize()
model.advance(args.steps)
ms = e0.elapsed_time(e1) / args.steps
# attention share: the 32 fused decode kernels alone
caches = [L["cache"] for L in model.layers]
q = torch.randn((1, cfg.q_heads, 128), device="cuda").to(torch.bfloat16)
o = torch.empty((1, cfg.q_heads, 128), device="cuda")
for c in caches:
    c.attend_device(q, qpos, o)
torch.cuda.synchronize()
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
for _ in range(10):
    for c in caches:
        c.attend_device(q, qpos, o)
a1.record()
torch.cuda.synchronize()
att_ms = a0.elapsed_time(a1) / 10
print(f"ctx {args.ctx} x {args.layers} layers: prefill {t_prefill:.2f} s (cold first call {t_cold:.2f} s), decode {ms:.3f} ms/token "
      f"({1e3 / ms:.1f} tok/s), attention {att_ms:.3f} ms/token ({att_ms / ms:.0%})")
