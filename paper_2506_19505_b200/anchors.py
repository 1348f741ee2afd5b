"""Anchor scores and selection, mirroring antkv.anchors (anchors.py:32-132).

anchor_scores_blocked reconstructs A = exp(S - M)/L blockwise on the GPU
(antkv_ans_blocked); select_anchors runs the radix top-k selection kernel
(antkv_select_anchors) with the reference's policies and tie rule."""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import as_cuda, back
from .attention import AttentionAux, _check, rope_device

__all__ = ["AnchorScores", "AnchorSelection", "POLICIES", "anchor_scores", "anchor_scores_blocked",
           "select_anchors", "select_anchors_device"]

POLICIES = ("by_k", "by_v", "by_sum")


@dataclass
class AnchorScores:
    ans_k: object
    ans_v: object


@dataclass
class AnchorSelection:
    indices: np.ndarray
    budget: int
    policy: str


def anchor_scores(A, q_norms):
    """Direct double-sum scores from a materialised attention matrix
    (anchors.py:53-63): ans_v = sum_i A_ij, ans_k = sum_i A_ij (1 - A_ij) |q_i|.
    The oracle of anchor_scores_blocked; float64 on the device."""
    from .attention import _dev64, _out
    At, was_np = _dev64(A, "A")
    qn = torch.as_tensor(np.asarray(q_norms, dtype=np.float64) if not isinstance(q_norms, torch.Tensor)
                         else q_norms).to(device=At.device, dtype=torch.float64)
    if qn.shape != (At.shape[0],):
        raise ValueError("q_norms length must match the query count")
    return AnchorScores(ans_k=_out((At * (1.0 - At) * qn[:, None]).sum(dim=0), was_np),
                        ans_v=_out(At.sum(dim=0), was_np))


def anchor_scores_blocked(Q, K, V, aux: AttentionAux, block_q, block_k, rope=None,
                          causal=False):
    """Blockwise AnS from the attention auxiliaries (anchors.py:66-87)."""
    Qt, was_np = _check(Q, "Q")
    Kt, _ = _check(K, "K")
    H, n_q, d = Qt.shape
    Hk, n_k, _ = Kt.shape
    M, _ = as_cuda(aux.M, torch.float32)
    L, _ = as_cuda(aux.L, torch.float32)
    qn, _ = as_cuda(aux.q_norms, torch.float32)
    if M.numel() != H * n_q or L.numel() != H * n_q:
        raise ValueError("aux statistics do not match the query count")
    if block_q < 1 or block_k < 1:
        raise ValueError("block sizes must be >= 1")
    if causal and n_q != n_k:
        raise ValueError("causal attention requires matching Q/K token counts")
    pos = rope.positions if rope is not None else None
    theta = rope.theta_base if rope is not None else 10000.0
    Qs, _ = rope_device(Qt, pos, theta, 1.0 / np.sqrt(d))
    Kr, _ = rope_device(Kt, pos, theta, 1.0)
    ak = torch.empty((H, n_k), dtype=torch.float32, device=Qt.device)
    av = torch.empty((H, n_k), dtype=torch.float32, device=Qt.device)
    # temporaries stay bound until the launch is enqueued (the caching
    # allocator could otherwise hand their memory to the next allocation)
    M, L, qn = M.contiguous(), L.contiguous(), qn.contiguous()
    _lib.call("antkv_ans_blocked", _lib.ptr(Qs), _lib.ptr(Kr), _lib.ptr(M),
              _lib.ptr(L), _lib.ptr(qn), H, Hk, n_q, n_k, d,
              int(block_q), int(block_k), int(bool(causal)), _lib.ptr(ak), _lib.ptr(av),
              _lib.stream())
    single = was_np or (isinstance(Q, torch.Tensor) and Q.ndim == 2)
    if single:
        ak, av = ak[0], av[0]
    return AnchorScores(ans_k=back(ak, was_np), ans_v=back(av, was_np))


def select_anchors_device(ans_k, ans_v, budget, policy="by_sum"):
    """ans_k/ans_v float32 CUDA [R, n] -> int32 [R, budget] sorted indices."""
    R, n = ans_k.shape
    out = torch.empty((R, budget), dtype=torch.int32, device=ans_k.device)
    if budget > 0:
        ans_k, ans_v = ans_k.contiguous(), ans_v.contiguous()
        _lib.call("antkv_select_anchors", _lib.ptr(ans_k), _lib.ptr(ans_v),
                  1, R, n, int(budget), _lib.POLICY[policy], _lib.ptr(out), _lib.stream())
    return out


def select_anchors(scores: AnchorScores, budget, policy="by_sum"):
    """Top-budget tokens under the policy, ties to the lower index
    (anchors.py:96-132).  Scores are compared in float32 on the GPU."""
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy!r}")
    k, was_np = as_cuda(scores.ans_k, torch.float32)
    v, _ = as_cuda(scores.ans_v, torch.float32)
    n = k.shape[-1]
    budget = int(np.clip(budget, 0, n))
    single = k.ndim == 1
    k2 = k.reshape(-1, n)
    v2 = v.reshape(-1, n)
    idx = select_anchors_device(k2, v2, budget, policy).to(torch.int64)
    if single:
        idx = idx[0]
    return AnchorSelection(indices=idx.cpu().numpy() if was_np or single else idx,
                           budget=budget, policy=policy)
