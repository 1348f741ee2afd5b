"""RoPE and blocked attention with auxiliaries, mirroring antkv.attention.

The arithmetic runs on the GPU (antkv_rope_rotate / antkv_flash_aux).  The
public functions accept the reference's single-head numpy matrices (n, d)
and return numpy; torch CUDA tensors of shape [H, n, d] (GQA: K/V may have
fewer heads) are also accepted and returned as tensors.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import as_cuda, back
from .errors import NumericalError

__all__ = ["RopeParams", "AttentionAux", "apply_rope", "flash_attention_aux", "rope_device",
           "softmax_rows", "attention_scores", "attention_exact"]


@dataclass(frozen=True)
class RopeParams:
    """Per-token positions and frequency base (attention.py:28-43)."""

    positions: np.ndarray
    theta_base: float = 10000.0

    def __post_init__(self):
        pos = self.positions
        if isinstance(pos, torch.Tensor):
            pos = pos.detach().cpu().numpy()
        pos = np.asarray(pos, dtype=np.int64)
        object.__setattr__(self, "positions", pos)
        if self.theta_base <= 0:
            raise ValueError("theta_base must be positive")
        if pos.ndim != 1:
            raise ValueError("positions must be a 1-d array")
        if np.any(pos < 0):
            raise ValueError("positions must be nonnegative")


@dataclass
class AttentionAux:
    """O plus (L, M, q_norms) for post-hoc anchor scoring (attention.py:46-56)."""

    O: object
    L: object
    M: object
    q_norms: object
    block_q: int = field(default=0)
    block_k: int = field(default=0)


def _check(X, name, d_even=False):
    """attention.py:59-67 on host or device data."""
    t, was_np = as_cuda(X)
    if t.ndim not in (2, 3):
        raise ValueError(f"{name} must be 2-d (or [H, n, d]), got shape {tuple(t.shape)}")
    if not bool(torch.isfinite(t).all()):
        raise NumericalError(f"non-finite values in {name}")
    if d_even and t.shape[-1] % 2 != 0:
        raise ValueError(f"{name} head dimension must be even for RoPE")
    if t.dtype not in (torch.float32, torch.bfloat16, torch.float16):
        t = t.float()
    return (t if t.ndim == 3 else t[None]).contiguous(), was_np


def rope_device(X3, positions, theta_base, scale=1.0, want_norms=False):
    """[H, n, d] -> float32 rotated*scale (+ pre-RoPE row norms)."""
    H, n, d = X3.shape
    out = torch.empty((H, n, d), dtype=torch.float32, device=X3.device)
    norms = torch.empty((H, n), dtype=torch.float32, device=X3.device) if want_norms else None
    pos = None
    if positions is not None:
        p = np.asarray(positions, dtype=np.int64)
        if len(p) < n:
            raise ValueError("positions shorter than token count")
        pos = torch.from_numpy(np.ascontiguousarray(p[:n])).to(X3.device)
    # positions are shared across heads: treat heads as the batch axis with H=1
    # rows each by repeating positions per head
    if pos is not None:
        pos = pos.repeat(H)
    _lib.call("antkv_rope_rotate", _lib.ptr(X3), _lib.dtype_tag(X3), _lib.ptr(pos), H, 1, n, d,
              float(theta_base), float(scale), _lib.ptr(out), _lib.ptr(norms), _lib.stream())
    return out, norms


def apply_rope(X, params: RopeParams, sign=1.0):
    """Rotate pairs (2i, 2i+1) of row t by positions[t]*theta^(-2i/d)
    (attention.py:89-106).  sign=-1 gives the adjoint."""
    t, was_np = _check(X, "X", d_even=True)
    pos = params.positions if sign >= 0 else -params.positions
    if sign < 0:
        # negative positions are allowed here only as the adjoint rotation
        pos = np.asarray(pos, dtype=np.int64)
    out, _ = rope_device(t, pos, params.theta_base)
    return back(out if np.ndim(X) == 3 else out[0], was_np)


def flash_attention_aux(Q, K, V, block_q, block_k, rope=None, causal=False):
    """Blocked attention returning (O, L, M, q_norms) (attention.py:146-169).

    GPU float32 tiles; block sizes are validated but only change the
    reference's rounding order."""
    Qt, was_np = _check(Q, "Q")
    Kt, _ = _check(K, "K")
    Vt, _ = _check(V, "V")
    if Qt.shape[-1] != Kt.shape[-1]:
        raise ValueError("Q and K head dimensions differ")
    if Kt.shape[-2] != Vt.shape[-2]:
        raise ValueError("K and V token counts differ")
    if causal and Qt.shape[-2] != Kt.shape[-2]:
        raise ValueError("causal attention requires matching Q/K token counts")
    if block_q < 1 or block_k < 1:
        raise ValueError("block sizes must be >= 1")
    H, n_q, d = Qt.shape
    Hk, n_k, _ = Kt.shape
    if H % Hk or Vt.shape[0] != Hk:
        raise ValueError("query heads must be a multiple of key heads")
    pos = rope.positions if rope is not None else None
    theta = rope.theta_base if rope is not None else 10000.0
    if rope is not None and d % 2:
        raise ValueError("Q head dimension must be even for RoPE")
    Qs, qn = rope_device(Qt, pos, theta, 1.0 / np.sqrt(d), want_norms=True)
    Kr, _ = rope_device(Kt, pos, theta, 1.0)
    Vf = Vt.float().contiguous()
    dv = Vf.shape[-1]
    O = torch.empty((H, n_q, dv), dtype=torch.float32, device=Qt.device)
    L = torch.empty((H, n_q), dtype=torch.float32, device=Qt.device)
    M = torch.empty((H, n_q), dtype=torch.float32, device=Qt.device)
    _lib.call("antkv_flash_aux", _lib.ptr(Qs), _lib.ptr(Kr), _lib.ptr(Vf), H, Hk, n_q, n_k, d, dv,
              int(block_q), int(block_k), int(bool(causal)), _lib.ptr(O), _lib.ptr(L), _lib.ptr(M),
              _lib.stream())
    single = was_np or (isinstance(Q, torch.Tensor) and Q.ndim == 2)
    sq = (lambda x: x[0]) if single else (lambda x: x)
    return AttentionAux(O=back(sq(O), was_np), L=back(sq(L), was_np), M=back(sq(M), was_np),
                        q_norms=back(sq(qn), was_np), block_q=block_q, block_k=block_k)


# ---------------------------------------------------------------- exact oracles
# The reference's unblocked float64 attention (attention.py:70-79, 121-143),
# the correctness oracle of every blocked and quantized path.  Computed on the
# device in float64 (torch CUDA tensors; there is no CPU path); numpy in,
# numpy out as in the reference, CUDA tensors in, tensors out.

def _dev64(X, name, d_even=False):
    """attention.py:59-67 (_check_matrix) on the device: float64, 2-d,
    finite, even head dimension for RoPE."""
    was_np = not isinstance(X, torch.Tensor)
    if was_np:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(X, dtype=np.float64)))
    else:
        t = X.detach()
    _lib.load()
    t = t.to(device="cuda", dtype=torch.float64)
    if t.ndim != 2:
        raise ValueError(f"{name} must be 2-d, got shape {tuple(t.shape)}")
    if not bool(torch.isfinite(t).all()):
        raise NumericalError(f"non-finite values in {name}")
    if d_even and t.shape[1] % 2 != 0:
        raise ValueError(f"{name} head dimension must be even for RoPE")
    return t, was_np


def _out(t, was_np):
    return t.cpu().numpy() if was_np else t


def _softmax64(M, causal):
    if causal:
        n_q, n_k = M.shape
        mask = torch.arange(n_k, device=M.device)[None, :] > torch.arange(n_q, device=M.device)[:, None]
        M = M.masked_fill(mask, float("-inf"))
    P = torch.exp(M - M.max(dim=1, keepdim=True).values)
    return P / P.sum(dim=1, keepdim=True)


def softmax_rows(M, causal=False):
    """Row softmax with per-row max subtraction; causal masks j > i
    (attention.py:70-79)."""
    t, was_np = _dev64(M, "logits")
    return _out(_softmax64(t, causal), was_np)


def _rope64(X, params: RopeParams):
    """attention.py:82-106 in float64 on the device (angles pos * freq formed
    in float64, as _rope_trig does)."""
    n, d = X.shape
    if len(params.positions) < n:
        raise ValueError("positions shorter than token count")
    freqs = params.theta_base ** (-2.0 * np.arange(d // 2) / d)
    ang = torch.from_numpy(params.positions[:n, None].astype(np.float64) * freqs[None, :]).to(X.device)
    c, s = torch.cos(ang), torch.sin(ang)
    x0, x1 = X[:, 0::2], X[:, 1::2]
    out = torch.empty_like(X)
    out[:, 0::2] = x0 * c - x1 * s
    out[:, 1::2] = x0 * s + x1 * c
    return out


def _scores64(Q, K, rope, causal):
    if Q.shape[1] != K.shape[1]:
        raise ValueError("Q and K head dimensions differ")
    if causal and Q.shape[0] != K.shape[0]:
        raise ValueError("causal attention requires matching Q/K token counts")
    if rope is not None:
        if Q.shape[1] % 2:
            raise ValueError("Q head dimension must be even for RoPE")
        Q, K = _rope64(Q, rope), _rope64(K, rope)
    return _softmax64((Q @ K.T) / np.sqrt(Q.shape[1]), causal)


def attention_scores(Q, K, rope=None, causal=False):
    """Softmax(Q~ K~^T / sqrt(d)), optionally RoPE-rotated and causal
    (attention.py:121-131)."""
    Qt, was_np = _dev64(Q, "Q")
    Kt, _ = _dev64(K, "K")
    return _out(_scores64(Qt, Kt, rope, causal), was_np)


def attention_exact(Q, K, V, rope=None, causal=False):
    """Attn(Q, K, V) = Softmax(Q~ K~^T / sqrt(d)) V, unblocked
    (attention.py:134-143)."""
    Vt, _ = _dev64(V, "V")
    Kt, _ = _dev64(K, "K")
    if Vt.shape[0] != Kt.shape[0]:
        raise ValueError("K and V token counts differ")
    Qt, was_np = _dev64(Q, "Q")
    return _out(_scores64(Qt, Kt, rope, causal) @ Vt, was_np)
