import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2506_19505_b200.llama import AnTKVLlama, LlamaConfig, _rms
ctx = 32768
cfg = LlamaConfig(layers=3)
model = AnTKVLlama(cfg, batch=1, capacity=ctx + 256)
toks = torch.randint(0, cfg.vocab, (1, ctx), device="cuda")
x = model.embed[toks]
pos = np.arange(ctx)
def layer(L, x):
    q, k, v = model._split(_rms(x, L["n1"]) @ L["wqkv"].t(), ctx)
    o = L["cache"].prefill(q.contiguous(), k.contiguous(), v.contiguous(), pos)
    o = o.transpose(1, 2).reshape(1, ctx, -1).to(torch.bfloat16)
    return model._mlp(L, x + o @ L["wo"].t())
x = layer(model.layers[0], x)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for L in model.layers[1:]:
        x = layer(L, x)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=14))
