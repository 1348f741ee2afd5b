"""Float64 torch restatement of the prefill anchor scores (Alg. 1 of the
paper, anchors.py:66-87 with the causal FA statistics of attention.py:146-169)
for long contexts -- test infrastructure only, like oracle/.

For query block [q0, q1) every causal key [0, q1) is in one S block, so the
row max M_i and normaliser L_i are exact (no online rescaling) and the
attention probabilities A_ij = exp(S_ij - M_i) / L_i give, summed over the
query heads of a KV group (the oracle's GQA restatement,
oracle/antkv_oracle.py OracleCache.prefill):
    ans_v_j = sum_i A_ij,   ans_k_j = sum_i A_ij (1 - A_ij) ||q_i||
with ||q_i|| of the pre-RoPE query (attention.py:167).  Runs on any torch
device; pinned against the numpy oracle in tests/test_host_cpu.py."""

import math

import torch


def rope64(X, positions, theta_base):
    """Interleaved-pair RoPE in float64 (attention.py:82-106; oracle apply_rope)."""
    n, d = X.shape
    freqs = theta_base ** (-2.0 * torch.arange(d // 2, dtype=torch.float64, device=X.device) / d)
    ang = positions.to(torch.float64)[:, None] * freqs[None, :]
    c, s = torch.cos(ang), torch.sin(ang)
    x0, x1 = X[:, 0::2], X[:, 1::2]
    out = torch.empty_like(X)
    out[:, 0::2] = x0 * c - x1 * s
    out[:, 1::2] = x0 * s + x1 * c
    return out


def group_anchor_scores(Qg, K, positions, theta_base=10000.0, block=2048):
    """Qg [g, n, d] (the query heads of one KV head), K [n, d]: float64
    (ans_k, ans_v) [n] summed over the group, causal."""
    Qg = Qg.to(torch.float64)
    K = K.to(torch.float64)
    g, n, d = Qg.shape
    Kr = rope64(K, positions, theta_base)
    ans_k = torch.zeros(n, dtype=torch.float64, device=K.device)
    ans_v = torch.zeros_like(ans_k)
    for h in range(g):
        qn = torch.sqrt((Qg[h] ** 2).sum(1))
        Qs = rope64(Qg[h], positions, theta_base) / math.sqrt(d)
        for q0 in range(0, n, block):
            q1 = min(q0 + block, n)
            S = Qs[q0:q1] @ Kr[:q1].T
            mask = torch.arange(q1, device=K.device)[None, :] > torch.arange(q0, q1, device=K.device)[:, None]
            S.masked_fill_(mask, -math.inf)
            M = S.max(dim=1, keepdim=True).values
            S.sub_(M).exp_()
            L = S.sum(dim=1, keepdim=True)
            S.div_(L)                                   # A
            ans_v[:q1] += S.sum(0)
            S.mul_(1.0 - S).mul_(qn[q0:q1, None])       # A (1 - A) ||q||
            ans_k[:q1] += S.sum(0)
            del S
    return ans_k, ans_v
