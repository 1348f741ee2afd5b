"""A LLaMA-style decoder that serves its attention from AnTKV caches.

SURVEY.md §8(f) rank 1: the workload the path serves.  The dense parts
(projections, SwiGLU MLP, norms, embedding / LM head) are plain torch bf16
GEMMs (cuBLAS); every attention layer is a QuantizedKVCache: prefill runs the
full-precision FA + AnS + anchor selection + encode (and returns the
full-precision output, as the reference's prefill does, cache.py:100-140),
decode appends / attends / evicts through `step_device` -- one fused kernel
per layer on the d8m256 path.  Weights are random (no checkpoints offline);
shapes default to LLaMA-3-8B (BASELINE config #2).
"""

from dataclasses import dataclass

import numpy as np
import torch

from .cache import CacheConfig, QuantizedKVCache
from .vq import Codebook, VqConfig

__all__ = ["LlamaConfig", "AnTKVLlama"]


@dataclass
class LlamaConfig:
    layers: int = 32
    hidden: int = 4096
    q_heads: int = 32
    kv_heads: int = 8
    head_dim: int = 128
    ffn: int = 14336
    vocab: int = 128256
    theta: float = 500000.0
    notation: str = "d8m256"
    anchor_fraction: float = 0.01
    window: int = 32


def _rms(x, w, eps=1e-5):
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


class AnTKVLlama:
    """Random-init decoder; batch B sequences of equal length."""

    def __init__(self, cfg: LlamaConfig, batch=1, capacity=None, seed=0, device="cuda"):
        self.cfg = cfg
        self.B = batch
        g = torch.Generator(device=device).manual_seed(seed)
        H, D = cfg.hidden, cfg.head_dim

        def w(*shape, scale=None):
            s = scale if scale is not None else shape[-1] ** -0.5
            return (torch.randn(shape, device=device, generator=g) * s).to(torch.bfloat16)

        self.embed = w(cfg.vocab, H, scale=1.0)
        self.lm_head = w(cfg.vocab, H)
        self.norm = torch.ones(H, device=device, dtype=torch.bfloat16)
        self.layers = []
        vq = VqConfig.from_notation(cfg.notation)
        rng = np.random.default_rng(seed)
        for _ in range(cfg.layers):
            ck = rng.standard_normal((cfg.kv_heads, vq.m, vq.d_sub)).astype(np.float32)
            cv = rng.standard_normal((cfg.kv_heads, vq.m, vq.d_sub)).astype(np.float32)
            self._cache_args = (vq, batch, capacity)
            cache = self._new_cache(Codebook(vq, ck), Codebook(vq, cv))
            self.layers.append({
                "wqkv": w((cfg.q_heads + 2 * cfg.kv_heads) * D, H),
                "wo": w(H, cfg.q_heads * D),
                "w13": w(2 * cfg.ffn, H),
                "w2": w(H, cfg.ffn),
                "n1": torch.ones(H, device=device, dtype=torch.bfloat16),
                "n2": torch.ones(H, device=device, dtype=torch.bfloat16),
                "cache": cache,
            })
        self.pos = 0
        self._out = torch.empty((batch, cfg.q_heads, D), dtype=torch.float32, device=device)

    def _new_cache(self, cbk, cbv):
        cfg = self.cfg
        vq, batch, capacity = self._cache_args
        return QuantizedKVCache(
            CacheConfig(vq=vq, anchor_fraction=cfg.anchor_fraction, window_size=cfg.window,
                        theta_base=cfg.theta),
            cbk, cbv, batch=batch, q_heads=cfg.q_heads, kv_heads=cfg.kv_heads, capacity=capacity)

    def reset(self):
        """Empty every layer's cache (same codebooks), position 0: the next
        prefill starts a new sequence with warm allocators and libraries."""
        for L in self.layers:
            c = L["cache"]
            L["cache"] = self._new_cache(c.codebook_k, c.codebook_v)
        self.pos = 0

    def _split(self, qkv, n):
        c = self.cfg
        D = c.head_dim
        q, k, v = qkv.split([c.q_heads * D, c.kv_heads * D, c.kv_heads * D], dim=-1)
        # [B, n, heads*D] -> [B, heads, n, D]
        return (q.view(self.B, n, c.q_heads, D).transpose(1, 2),
                k.view(self.B, n, c.kv_heads, D).transpose(1, 2),
                v.view(self.B, n, c.kv_heads, D).transpose(1, 2))

    def _mlp(self, L, x):
        h = _rms(x, L["n2"])
        gu = h @ L["w13"].t()
        gate, up = gu.chunk(2, dim=-1)
        return x + (torch.nn.functional.silu(gate) * up) @ L["w2"].t()

    @torch.no_grad()
    def prefill(self, tokens):
        """tokens int64 [B, n] -> logits [B, vocab] of the last position."""
        B, n = tokens.shape
        x = self.embed[tokens]                                   # [B, n, H]
        positions = np.arange(self.pos, self.pos + n)
        for L in self.layers:
            q, k, v = self._split(_rms(x, L["n1"]) @ L["wqkv"].t(), n)
            o = L["cache"].prefill(q.contiguous(), k.contiguous(), v.contiguous(), positions)
            o = o.transpose(1, 2).reshape(B, n, -1).to(torch.bfloat16)
            x = x + o @ L["wo"].t()
            x = self._mlp(L, x)
        self.pos += n
        return (_rms(x[:, -1], self.norm) @ self.lm_head.t()).float()

    @torch.no_grad()
    def decode_device(self, token, qpos):
        """One decode step, no host synchronisation (CUDA-graph capturable):
        token int64 [B], qpos int64 [B] device tensors -> logits [B, vocab]."""
        c = self.cfg
        x = self.embed[token]                                    # [B, H]
        for L in self.layers:
            qkv = _rms(x, L["n1"]) @ L["wqkv"].t()
            q, k, v = self._split(qkv[:, None], 1)
            L["cache"].step_device(q[:, :, 0].contiguous(), k[:, :, 0].contiguous(),
                                   v[:, :, 0].contiguous(), qpos, self._out)
            x = x + self._out.reshape(self.B, -1).to(torch.bfloat16) @ L["wo"].t()
            x = self._mlp(L, x)
        return (_rms(x, self.norm) @ self.lm_head.t()).float()

    def advance(self, steps=1):
        """Host bookkeeping after `steps` device decode steps."""
        for L in self.layers:
            L["cache"]._n += steps
        self.pos += steps

    @torch.no_grad()
    def decode(self, token):
        qpos = torch.full((self.B,), self.pos, dtype=torch.int64, device=token.device)
        for L in self.layers:
            L["cache"]._ensure_capacity(L["cache"].token_count + 2)
        logits = self.decode_device(token, qpos)
        self.advance(1)
        return logits
