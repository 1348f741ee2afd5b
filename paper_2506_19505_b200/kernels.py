"""Drop-in replacement for the reference's compiled kernel module.

The reference picks ``antkv._ckernels`` at import time
(kernels/__init__.py:19-37).  This module exposes the same three functions
with the same signatures, float64 numpy in and out, computed on the GPU by
libantkv_b200.so: attention and anchor scores in float32 arithmetic,
assign_nearest in float64 with the compiled backend's operation order
(bit-identical to _ckernels.assign_nearest for d_sub <= 64).  Installing it as ``antkv._ckernels``
 routes the reference's flash_attention_aux,
anchor_scores_blocked, encode_rows and weighted_kmeans through the B200.
"""

import numpy as np
import torch

from . import _lib

__all__ = ["flash_aux", "ans_blocked", "assign_nearest", "BACKEND"]

BACKEND = "b200"


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def flash_aux(Qs, Kr, V, block_q, block_k, causal):
    """(O, L, M) of blocked attention over pre-rotated, pre-scaled inputs
    (_ckernels.pyx:10-88)."""
    Qd, Kd, Vd = _dev(Qs), _dev(Kr), _dev(V)
    n_q, d = Qd.shape
    n_k, dv = Vd.shape
    O = torch.empty((n_q, dv), dtype=torch.float32, device=Qd.device)
    L = torch.empty((n_q,), dtype=torch.float32, device=Qd.device)
    M = torch.empty((n_q,), dtype=torch.float32, device=Qd.device)
    _lib.call("antkv_flash_aux", _lib.ptr(Qd), _lib.ptr(Kd), _lib.ptr(Vd), 1, 1, n_q, n_k, d, dv,
              int(block_q), int(block_k), int(bool(causal)), _lib.ptr(O), _lib.ptr(L), _lib.ptr(M),
              _lib.stream())
    return (O.cpu().numpy().astype(np.float64), L.cpu().numpy().astype(np.float64),
            M.cpu().numpy().astype(np.float64))


def ans_blocked(Qs, Kr, M, L, q_norms, block_q, block_k, causal):
    """Blocked anchor-score column sums (_ckernels.pyx:91-131)."""
    Qd, Kd = _dev(Qs), _dev(Kr)
    Md, Ld, qd = _dev(M), _dev(L), _dev(q_norms)
    n_q, d = Qd.shape
    n_k = Kd.shape[0]
    ak = torch.empty((n_k,), dtype=torch.float32, device=Qd.device)
    av = torch.empty((n_k,), dtype=torch.float32, device=Qd.device)
    _lib.call("antkv_ans_blocked", _lib.ptr(Qd), _lib.ptr(Kd), _lib.ptr(Md), _lib.ptr(Ld),
              _lib.ptr(qd), 1, 1, n_q, n_k, d, int(block_q), int(block_k), int(bool(causal)),
              _lib.ptr(ak), _lib.ptr(av), _lib.stream())
    return ak.cpu().numpy().astype(np.float64), av.cpu().numpy().astype(np.float64)


def assign_nearest(X, C):
    """Nearest centroid, lowest index on ties (_ckernels.pyx:134-163):
    float64, the same per-coordinate accumulation order, no FMA."""
    Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).cuda()
    Cd = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float64)).cuda()
    n, d_sub = Xd.shape
    m = Cd.shape[0]
    idx = torch.empty((n,), dtype=torch.int64, device=Xd.device)
    if d_sub > 64:       # float32 kernel beyond the float64 kernel's register budget
        d2 = torch.empty((n,), dtype=torch.float32, device=Xd.device)
        Xf, Cf = Xd.float(), Cd.float()
        _lib.call("antkv_assign_nearest", _lib.ptr(Xf), _lib.ptr(Cf), n, m, d_sub,
                  _lib.ptr(idx), _lib.ptr(d2), _lib.stream())
        return idx.cpu().numpy(), d2.cpu().numpy().astype(np.float64)
    d2 = torch.empty((n,), dtype=torch.float64, device=Xd.device)
    _lib.call("antkv_kmeans_assign_f64", _lib.ptr(Xd), _lib.ptr(Cd), n, m, d_sub, _lib.ptr(idx),
              _lib.ptr(d2), _lib.stream())
    return idx.cpu().numpy(), d2.cpu().numpy()
