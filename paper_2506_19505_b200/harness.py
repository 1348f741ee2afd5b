"""Evaluation at scale: the reference's quantisation-error study
(harness.py:35-253) on the GPU.

``eval_point`` runs the prefill path of a QuantizedKVCache and records, as
the reference does, the attention error of the quantised cache, the V and K
perturbation bounds (anchors.py:135-186), the first-order residual
(anchors.py:189-207), the AnS rank agreement with per-token errors, random
anchor controls and the decode-wiring error.  Everything dense runs in
float64 on the device (cuBLAS products, elementwise softmax); the two
pairwise L1 reductions run in antkv_eval_pair_l1, and per-token errors use
the exact single-column softmax update, O(n^2 d) instead of the
reference's n attention passes (O(n^3 d)), so a 16K-token point takes
seconds.  Quantised rows come from the float64 assignment kernel
(antkv_kmeans_assign_f64, the compiled backend's order), so codes match the
reference bit for bit.
"""

import math
import time

import numpy as np
import torch

from . import _lib
from .cache import CacheConfig, QuantizedKVCache
from .errors import NumericalError
from .util import stream_rng
from .vq import bits_per_element

__all__ = ["generate_qkv", "quantized_reconstruction", "per_token_errors", "eval_point",
           "STRUCTURES", "EVAL_SCHEMA_VERSION"]

EVAL_SCHEMA_VERSION = 1
STRUCTURES = ("gaussian", "clustered", "heavy_hitter")


def generate_qkv(seed, n, d, structure="gaussian", planted=None, clusters=8, cluster_d_sub=8):
    """Deterministic synthetic (Q, K, V, positions) for one head, the
    reference's generator (harness.py:35-72; host numpy, same streams)."""
    if structure not in STRUCTURES:
        raise ValueError(f"unknown structure {structure!r}")
    rng = stream_rng(seed, f"gen:{structure}:{n}:{d}")
    Q = rng.standard_normal((n, d))
    K = rng.standard_normal((n, d))
    V = rng.standard_normal((n, d))
    planted_idx = []
    if structure == "clustered":
        groups = d // cluster_d_sub
        centers = 4.0 * rng.standard_normal((clusters, cluster_d_sub))
        for X in (K, V):
            choice = rng.integers(clusters, size=(n, groups))
            X[:] = (centers[choice] + 0.05 * rng.standard_normal((n, groups, cluster_d_sub))
                    ).reshape(n, d)
    elif structure == "heavy_hitter":
        count = planted if planted is not None else max(1, n // 100)
        planted_idx = list(range(1, 1 + 2 * count, 2))[:count]
        for j in planted_idx:
            K[j] *= 5.0
            V[j] *= 3.0
    return {"Q": Q.astype(np.float32), "K": K.astype(np.float32), "V": V.astype(np.float32),
            "positions": np.arange(n, dtype=np.int64), "planted": planted_idx}


# ------------------------------------------------------------------ float64
def _dev64(x):
    if isinstance(x, torch.Tensor):
        return x.detach().to("cuda", torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


class _Rope:
    """cos/sin tables of attention._rope_trig (attention.py:82-86), evaluated
    on the host exactly as the reference does, applied on the device."""

    def __init__(self, positions, d, theta_base=10000.0):
        half = d // 2
        freqs = theta_base ** (-2.0 * np.arange(half) / d)
        ang = np.asarray(positions, dtype=np.int64)[:, None].astype(np.float64) * freqs[None, :]
        self.cos = torch.from_numpy(np.cos(ang)).cuda()
        self.sin = torch.from_numpy(np.sin(ang)).cuda()

    def __call__(self, X):
        x0, x1 = X[:, 0::2], X[:, 1::2]
        n = X.shape[0]
        c, s = self.cos[:n], self.sin[:n]
        out = torch.empty_like(X)
        out[:, 0::2] = x0 * c - x1 * s
        out[:, 1::2] = x0 * s + x1 * c
        return out


def _softmax_rows(M, causal):
    if causal:
        n_q, n_k = M.shape
        mask = torch.arange(n_k, device=M.device)[None, :] > torch.arange(n_q, device=M.device)[:, None]
        M = M.masked_fill(mask, -math.inf)
    m = M.max(dim=1, keepdim=True).values
    P = torch.exp(M - m)
    return P / P.sum(dim=1, keepdim=True)


def _scores(Qr, Kr, causal):
    return _softmax_rows((Qr @ Kr.T) / math.sqrt(Qr.shape[1]), causal)


def _pair_l1(Y, X, Z=None, W=None, P=None, R=None, causal=False):
    n_i, d = Y.shape
    n_j = X.shape[0]
    out = torch.empty((n_j,), dtype=torch.float64, device=Y.device)
    keep = [t.contiguous() if t is not None else None for t in (Y, X, Z, W, P, R)]
    _lib.call("antkv_eval_pair_l1", *[_lib.ptr(t) for t in keep], n_i, n_j, d, int(causal),
              _lib.ptr(out), _lib.stream())
    return out


def _quantize64(X, codebook):
    """decode(encode(X)) with the float64 nearest-centroid kernel."""
    C = codebook.centroids
    if C.ndim == 3:
        C = C[0]
    Cd = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float64)).cuda()
    n, d = X.shape
    m, ds = Cd.shape
    sub = X.reshape(-1, ds).contiguous()
    idx = torch.empty((sub.shape[0],), dtype=torch.int64, device=X.device)
    d2 = torch.empty((sub.shape[0],), dtype=torch.float64, device=X.device)
    _lib.call("antkv_kmeans_assign_f64", _lib.ptr(sub), _lib.ptr(Cd), sub.shape[0], m, ds,
              _lib.ptr(idx), _lib.ptr(d2), _lib.stream())
    # decode_rows returns float32 centroids (vq.py:243-248)
    return Cd.float().double()[idx].reshape(n, d)


def quantized_reconstruction(K, V, codebook_k, codebook_v, protected):
    """(K_hat, V_hat) with every unprotected token quantised
    (harness.py:84-101).  float64 device tensors."""
    Kd, Vd = _dev64(K), _dev64(V)
    Kh, Vh = _quantize64(Kd, codebook_k), _quantize64(Vd, codebook_v)
    prot = torch.as_tensor(sorted(int(j) for j in protected), dtype=torch.int64, device=Kd.device)
    if prot.numel():
        Kh[prot] = Kd[prot]
        Vh[prot] = Vd[prot]
    return Kh, Vh


def _attention(Qr, Kr, V, causal=True):
    return _scores(Qr, Kr, causal) @ V


def per_token_errors(Q, K, V, codebook_k, codebook_v, rope, causal=True, mode="joint"):
    """L1 attention-output error from quantising one token at a time
    (harness.py:111-134): errors[j] = ||Attn with row j quantised - Attn||_1.

    Exact single-column update instead of n attention passes: with A the
    base probabilities, A' those with token j's quantised key, o_i the base
    output, the change of row i is (A'_ij (v'_j - o_i) - A_ij (v_j - o_i))
    / (1 - A_ij + A'_ij)."""
    if mode not in ("joint", "k_only", "v_only"):
        raise ValueError(f"unknown per-token mode {mode!r}")
    Qd, Kd, Vd = _dev64(Q), _dev64(K), _dev64(V)
    n, d = Kd.shape
    R = rope if isinstance(rope, _Rope) else _Rope(rope.positions, d, rope.theta_base)
    Qr, Kr = R(Qd), R(Kd)
    Kq = _quantize64(Kd, codebook_k) if mode != "v_only" else Kd
    Vq = _quantize64(Vd, codebook_v) if mode != "k_only" else Vd
    logits = (Qr @ Kr.T) / math.sqrt(d)
    if causal:
        mask = torch.arange(n, device=Qd.device)[None, :] > torch.arange(n, device=Qd.device)[:, None]
        logits = logits.masked_fill(mask, -math.inf)
    m = logits.max(dim=1, keepdim=True).values
    E = torch.exp(logits - m)
    Zs = E.sum(dim=1, keepdim=True)
    A = E / Zs
    O = A @ Vd
    if mode == "v_only":
        Ap = A
    else:
        # the quantised key only changes column j's logit: diag of Qr Kq_r^T
        lq = (Qr @ R(Kq).T) / math.sqrt(d)
        if causal:
            lq = lq.masked_fill(mask, -math.inf)
        Ap = torch.exp(lq - m) / Zs
    Wt = 1.0 / (1.0 - A + Ap)
    return _pair_l1(O, Vq, Vd, Wt, Ap, A, causal=causal).cpu().numpy()


def _rank_agreement(errors, scores, frac=0.01):
    from scipy import stats
    rho = float(stats.spearmanr(errors, scores).statistic)
    n = len(errors)
    k = max(1, math.ceil(frac * n))
    top_err = set(np.argsort(-errors, kind="stable")[:k])
    top_score = set(np.argsort(-scores, kind="stable")[:k])
    return {"spearman": rho, "topk_overlap": len(top_err & top_score) / k, "topk": k}


def _protected_set(n, anchors, window_size):
    prot = set(int(j) for j in anchors)
    prot.update(range(max(0, n - window_size), n))
    return prot


def eval_point(data, codebook_k, codebook_v, anchor_fraction, window_size=0, policy="by_sum",
               seed=0, controls=0, per_token_mode="joint", compute_per_token=True,
               wiring="prefill", decode_steps=32):
    """One evaluation grid point (harness.py:137-235) on the GPU; same
    record keys and meaning."""
    t0 = time.perf_counter()
    Qh = np.asarray(data["Q"], dtype=np.float64)
    Kh = np.asarray(data["K"], dtype=np.float64)
    Vh = np.asarray(data["V"], dtype=np.float64)
    positions = np.asarray(data["positions"], dtype=np.int64)
    n, d = Kh.shape
    R = _Rope(positions, d)
    config = CacheConfig(vq=codebook_k.config, anchor_fraction=anchor_fraction,
                         window_size=window_size, policy=policy)
    cache = QuantizedKVCache(config, codebook_k, codebook_v, fast=False)
    cache.prefill(Qh, Kh, Vh, positions)
    Q, K, V = _dev64(Qh), _dev64(Kh), _dev64(Vh)
    Qr, Kr = R(Q), R(K)
    A = _scores(Qr, Kr, causal=True)
    exact = A @ V
    Kc, Vc = cache.dequantize()
    Kc, Vc = _dev64(Kc), _dev64(Vc)
    approx = _attention(Qr, R(Kc), Vc)                      # cache.attention_from_cache
    err = float((approx - exact).abs().sum())
    dK, dV = Kc - K, Vc - V
    v_bound = float((A.abs().sum(dim=0) * dV.abs().sum(dim=1)).sum())
    q_norms = torch.sqrt((Q ** 2).sum(dim=1))
    factor = _pair_l1(exact, V, W=A * q_norms[:, None], causal=True)
    k_bound = float((factor * dK.abs().sum(dim=1)).sum())
    dKr = R(dK)
    X = (Qr @ dKr.T) / math.sqrt(d)
    Y = X - (A * X).sum(dim=1, keepdim=True)
    fo = (A * Y) @ V
    exact_k_delta = _attention(Qr, R(K + dK), V) - exact
    denom = max(float(exact_k_delta.abs().sum()), 1e-300)
    fo_residual = float((exact_k_delta - fo).abs().sum()) / denom
    ans_v = A.sum(dim=0)
    ans_k = (A * (1.0 - A) * q_norms[:, None]).sum(dim=0)
    record = {
        "vq": codebook_k.config.notation,
        "bits_per_element": float(bits_per_element(codebook_k.config)),
        "anchor_fraction": anchor_fraction,
        "window_size": window_size,
        "policy": policy,
        "seed": seed,
        "n": n,
        "d": d,
        "wiring": wiring,
        "attention_l1_error": err,
        "v_bound": v_bound,
        "k_bound": k_bound,
        "first_order_residual": fo_residual,
    }
    for name, val in record.items():
        if isinstance(val, float) and not math.isfinite(val):
            raise NumericalError(f"non-finite value for {name}")
    if compute_per_token:
        errors = per_token_errors(Qh, Kh, Vh, codebook_k, codebook_v, R, mode=per_token_mode)
        ak, av = ans_k.cpu().numpy(), ans_v.cpu().numpy()
        ranking = ak if per_token_mode == "k_only" else av if per_token_mode == "v_only" else ak + av
        record["ans_rank_agreement"] = _rank_agreement(errors, ranking)
        record["per_token_mode"] = per_token_mode
    if controls > 0:
        budget = config.budget_for(n)
        rng = stream_rng(seed, "controls")
        ctl = []
        for _ in range(controls):
            anchors = rng.choice(n, size=budget, replace=False)
            Kq, Vq = quantized_reconstruction(K, V, codebook_k, codebook_v,
                                              _protected_set(n, anchors, window_size))
            ctl.append(float((_attention(Qr, R(Kq), Vq) - exact).abs().sum()))
        record["random_control"] = {"trials": controls, "mean": float(np.mean(ctl)), "errors": ctl}
    if wiring == "decode":
        steps = min(decode_steps, n - 1)
        split = n - steps
        dc = QuantizedKVCache(config, codebook_k, codebook_v, fast=False)
        dc.prefill(Qh[:split], Kh[:split], Vh[:split], positions[:split])
        total = 0.0
        ex = exact.cpu().numpy()
        for t in range(split, n):
            out = dc.decode_step(Qh[t], Kh[t], Vh[t], int(positions[t]))
            total += float(np.abs(np.asarray(out, dtype=np.float64) - ex[t]).sum())
        record["decode_l1_error"] = total
    record["runtime_ms"] = (time.perf_counter() - t0) * 1e3
    return record
