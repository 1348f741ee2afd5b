"""GPU-resident quantised KV cache, mirroring antkv.cache (cache.py:31-342).

One object holds B sequences x H_kv heads.  All per-token state lives in
device memory (layout: DESIGN.md §3); prefill, decode_step and eviction are
stream-ordered GPU work with no host synchronisation, so a decode step can be
captured in a CUDA graph.  The reference's single-head numpy API is kept:
``prefill(Q, K, V, positions)`` with (n, d) matrices returns a numpy (n, d)
output and ``decode_step(q, k, v, position)`` with (d,) vectors returns a
numpy (d,) output.  Batched GQA calls take torch tensors
Q [B, Hq, n, d], K/V [B, Hkv, n, d] and q [B, Hq, d], k/v [B, Hkv, d].

GQA semantics (the reference is single-head): each KV head keeps
its own anchors, chosen from anchor scores summed over the Q heads of its
group (exact for MHA, where it is the reference).
"""

import ctypes
import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._tensors import as_cuda
from .anchors import POLICIES, select_anchors_device
from .attention import rope_device
from .errors import FormatError
from .util import pack_indices, unpack_indices
from .vq import Codebook, VqConfig, load_codebook, save_codebook

__all__ = ["CacheConfig", "MemoryReport", "QuantizedKVCache"]

KIND_ANCHOR = "anchor"
KIND_QUANTIZED = "quantized"
KIND_WINDOWED = "windowed"
FORMAT_VERSION = 1


@dataclass(frozen=True)
class CacheConfig:
    """cache.py:31-57.  anchor_count, when set, overrides anchor_fraction."""

    vq: VqConfig
    anchor_fraction: float = 0.01
    anchor_count: int = None
    window_size: int = 32
    policy: str = "by_sum"
    theta_base: float = 10000.0
    block_q: int = 64
    block_k: int = 64

    def __post_init__(self):
        if not 0.0 <= self.anchor_fraction <= 1.0:
            raise ValueError("anchor_fraction must be in [0, 1]")
        if self.window_size < 0:
            raise ValueError("window_size must be >= 0")
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}")

    def budget_for(self, n):
        if self.anchor_count is not None:
            return int(np.clip(self.anchor_count, 0, n))
        return int(np.clip(math.ceil(self.anchor_fraction * n), 0, n))


@dataclass
class MemoryReport:
    payload_bits: int
    codebook_bits: int
    effective_bits_per_element: float
    fp_baseline_bits: int


_FAST_TABLES = {}


def _shared_fast_tables(dev, theta):
    """RoPE constant tables of the fast decode kernel.  They depend only on
    theta (d = 128), so every cache of the process shares one copy, which
    stays L2-resident across the layers of a decode step."""
    key = (dev.index, theta)
    if key not in _FAST_TABLES:
        _FAST_TABLES[key] = torch.zeros((16384,), dtype=torch.uint8, device=dev)
    return _FAST_TABLES[key]


def _round_up(x, m):
    return (x + m - 1) // m * m


def _code_kind(vq, groups):
    """Code unit of the device layout (antkv_cache_desc::code_bytes): 1 byte
    for m <= 256, 3 = 12-bit indices packed two per three bytes (m <= 4096,
    a power-of-two number of groups <= 32: config #3's 0.375-bit d32m4096
    really takes 0.375 bit per element), else 2 bytes."""
    if vq.index_bits <= 8:
        return 1
    if vq.index_bits <= 12 and 2 <= groups <= 32 and groups & (groups - 1) == 0:
        return 3
    return 2


def _slot_code_bytes(kind, groups):
    return 3 * groups if kind == 3 else 2 * groups * kind


def unpack_units(raw, kind):
    """uint8 code stream -> code units (uint16) for a device code kind."""
    raw = np.asarray(raw, dtype=np.uint8).reshape(-1)
    if kind == 1:
        return raw.astype(np.uint16)
    if kind == 2:
        return raw.view(np.uint16)
    t = raw.reshape(-1, 3).astype(np.uint16)
    out = np.empty((t.shape[0], 2), dtype=np.uint16)
    out[:, 0] = t[:, 0] | ((t[:, 1] & 0xF) << 8)
    out[:, 1] = (t[:, 1] >> 4) | (t[:, 2] << 4)
    return out.reshape(-1)


def pack_units(units, kind):
    """code units -> uint8 code stream for a device code kind."""
    u = np.asarray(units).reshape(-1)
    if kind == 1:
        return u.astype(np.uint8)
    if kind == 2:
        return u.astype(np.uint16).view(np.uint8)
    u = u.astype(np.uint16).reshape(-1, 2)
    out = np.empty((u.shape[0], 3), dtype=np.uint8)
    out[:, 0] = u[:, 0] & 0xFF
    out[:, 1] = ((u[:, 0] >> 8) & 0xF) | ((u[:, 1] & 0xF) << 4)
    out[:, 2] = u[:, 1] >> 4
    return out.reshape(-1)


class QuantizedKVCache:
    """Anchor rows + sub-vector codes + a full-precision recent window, on
    the GPU (cache.py:68-98)."""

    def __init__(self, config: CacheConfig, codebook_k: Codebook, codebook_v: Codebook,
                 *, batch=1, kv_heads=None, q_heads=None, capacity=None, fast=True,
                 splits=0, token_offset=0):
        if codebook_k is None or codebook_v is None:
            raise ValueError("both codebooks are required")
        if codebook_k.config != codebook_v.config:
            raise ValueError("K and V codebooks must share one VqConfig")
        if codebook_k.config != config.vq:
            raise ValueError("codebook config does not match cache config")
        self.config = config
        self.codebook_k = codebook_k
        self.codebook_v = codebook_v
        self.B = int(batch)
        self.Hkv = kv_heads
        self.Hq = q_heads
        self.d = None
        # 0: generic kernels; 1 (True): the best tensor-core kernel the shape
        # allows (fused d8m256, else the staged kernel); "staged" / 2: staged
        self.fast = 2 if fast in ("staged", 2) else int(bool(fast))
        self.row_dtype = None    # dtype of the full-precision pool rows = input dtype
        self.splits = int(splits)
        self._capacity_hint = capacity
        self.token_offset = int(token_offset)   # global index of slot 0 (sequence shards)
        self._single = False
        self._n = 0
        self._last_pos = None
        self._t = None          # device tensors
        self._contiguous = True
        self._desc = None
        self._pool_min_anchors = 0

    # ------------------------------------------------------------ layout
    @property
    def token_count(self):
        return self._n

    @property
    def capacity(self):
        return self._desc.capacity if self._desc is not None else 0

    def _pool_capacity(self, cap):
        # anchors (the budget of the whole sequence when this cache is a
        # sequence shard starting at token_offset; at least the anchors it was
        # built with) + window + the appended row; a multiple of 16: the fast
        # decode kernel streams the pool in 16-slot tiles
        anchors = max(self.config.budget_for(cap + self.token_offset), self._pool_min_anchors)
        return _round_up(anchors + self.config.window_size + 2, 16)

    def _alloc(self, cap):
        """(Re)allocate device state for `cap` token slots, keeping contents."""
        cfg = self.config.vq
        dev = torch.device("cuda", torch.cuda.current_device())
        B, H, d = self.B, self.Hkv, self.d
        G = d // cfg.d_sub
        kind = _code_kind(cfg, G)
        P = self._pool_capacity(cap)
        W = self.config.window_size
        old = self._t
        t = {
            "codes": torch.zeros((B, H, cap, _slot_code_bytes(kind, G)), dtype=torch.uint8, device=dev),
            "qmask": torch.zeros((B, H, cap // 32), dtype=torch.int32, device=dev),
            "pool_rows": torch.zeros((B, H, P, 2, d), dtype=self.row_dtype or torch.bfloat16,
                                     device=dev),
            "pool_tok": torch.full((B, H, P), -1, dtype=torch.int32, device=dev),
            "pool_kind": torch.full((B, H, P), -1, dtype=torch.int8, device=dev),
            "win_ring": torch.zeros((B, H, W + 1), dtype=torch.int32, device=dev),
            "free_stack": torch.zeros((B, H, P), dtype=torch.int32, device=dev),
            "hstate": torch.zeros((B, H, _lib.HSTATE_WORDS), dtype=torch.int32, device=dev),
            "seq_len": torch.zeros((B,), dtype=torch.int32, device=dev),
            "positions": torch.zeros((B, cap), dtype=torch.int64, device=dev),
            "evict_scratch": torch.full((B, H, 2 * G), -1, dtype=torch.int64, device=dev),
            "cb_k": self.codebook_k.device_tensor(H),
            "cb_v": self.codebook_v.device_tensor(H),
        }
        use_fast = bool(self.fast) and d == 128 and cfg.d_sub == 8 and cfg.m <= 256
        use_tc = (bool(self.fast) and d == 128 and cfg.d_sub in (4, 8, 16, 32, 64)
                  and _slot_code_bytes(kind, G) // 2 <= 32)
        if use_fast:
            t["cb_f16"] = torch.zeros((H, 256, 2, 64), dtype=torch.float16, device=dev)
        if use_tc:
            t["cb_f16g"] = torch.zeros((H, 2, cfg.m, cfg.d_sub), dtype=torch.float16, device=dev)
        if use_fast or use_tc:
            t["fast_tables"] = _shared_fast_tables(dev, float(self.config.theta_base))
            t["pool_f16"] = torch.zeros((B, H, P, 2, d), dtype=torch.float16, device=dev)
        if old is not None:
            oc = old["positions"].shape[1]
            oP = old["pool_tok"].shape[2]
            t["codes"][:, :, :oc] = old["codes"]
            t["qmask"][:, :, :oc // 32] = old["qmask"]
            t["positions"][:, :oc] = old["positions"]
            t["pool_rows"][:, :, :oP] = old["pool_rows"]
            t["pool_tok"][:, :, :oP] = old["pool_tok"]
            t["pool_kind"][:, :, :oP] = old["pool_kind"]
            t["win_ring"].copy_(old["win_ring"])
            t["seq_len"].copy_(old["seq_len"])
            t["hstate"].copy_(old["hstate"])
            # free stack: old free slots plus the new pool slots
            top = old["hstate"][:, :, _lib.HS_FREE_TOP]
            fs = old["free_stack"]
            newslots = torch.arange(P - 1, oP - 1, -1, dtype=torch.int32, device=dev)
            for b in range(B):
                for h in range(H):
                    k = int(top[b, h])
                    merged = torch.cat([newslots, fs[b, h, :k]])
                    t["free_stack"][b, h, :merged.numel()] = merged
                    t["hstate"][b, h, _lib.HS_FREE_TOP] = merged.numel()
            if "pool_f16" in t and "pool_f16" in old:
                t["pool_f16"][:, :, :oP] = old["pool_f16"]   # whole 16-slot tiles
        self._t = t
        self._desc = self._make_desc(cap, P, t)
        self._ws = None
        if use_fast:
            _lib.call("antkv_cache_prepare_fast", ctypes.byref(self._desc), _lib.stream())
        if use_tc:
            _lib.call("antkv_cache_prepare_tc", ctypes.byref(self._desc), _lib.stream())

    def _make_desc(self, cap, P, t):
        cfg = self.config.vq
        D = _lib.CacheDesc()
        D.B, D.Hq, D.Hkv, D.d = self.B, self.Hq, self.Hkv, self.d
        D.d_sub, D.m, D.groups, D.index_bits = cfg.d_sub, cfg.m, self.d // cfg.d_sub, cfg.index_bits
        D.code_bytes = _code_kind(cfg, self.d // cfg.d_sub)
        D.capacity, D.pool_capacity, D.window_size = cap, P, self.config.window_size
        D.policy = _lib.POLICY[self.config.policy]
        D.anchor_count = -1 if self.config.anchor_count is None else int(self.config.anchor_count)
        D.anchor_fraction = float(self.config.anchor_fraction)
        D.theta_base = float(self.config.theta_base)
        D.token_offset = self.token_offset
        D.row_dtype = _lib.dtype_tag(t["pool_rows"])
        for f, k in (("codes", "codes"), ("qmask", "qmask"), ("pool_rows", "pool_rows"),
                     ("pool_tok", "pool_tok"), ("pool_kind", "pool_kind"), ("win_ring", "win_ring"),
                     ("free_stack", "free_stack"), ("hstate", "hstate"), ("seq_len", "seq_len"),
                     ("positions", "positions"), ("codebook_k", "cb_k"), ("codebook_v", "cb_v"),
                     ("codebook_f16", "cb_f16"), ("pool_f16", "pool_f16"),
                     ("fast_tables", "fast_tables"), ("codebook_f16g", "cb_f16g"), ("evict_scratch", "evict_scratch")):
            setattr(D, f, t[k].data_ptr() if k in t else None)
        return D

    def _ensure_capacity(self, need):
        if self._desc is not None and need <= self._desc.capacity:
            return
        cap = max(need, self._capacity_hint or 0, 2 * (self._desc.capacity if self._desc else 0))
        self._alloc(_round_up(max(cap, 128), 128))

    @property
    def desc(self):
        return self._desc

    @property
    def tensors(self):
        return self._t

    # ----------------------------------------------------------- inputs
    def _shape_inputs(self, Q, K, V):
        Qt, was_np = as_cuda(Q)
        Kt, _ = as_cuda(K)
        Vt, _ = as_cuda(V)
        if Qt.ndim == 2:                    # reference single-head (n, d)
            single = True
            Qt, Kt, Vt = Qt[None, None], Kt[None, None], Vt[None, None]
        elif Qt.ndim == 4:
            single = False
        else:
            raise ValueError("expected (n, d) or [B, H, n, d] inputs")
        return Qt, Kt, Vt, single, was_np

    def _row_dtype(self, t):
        """Contiguous rows in a kernel dtype at a 16-byte aligned address (the
        kernels read rows with vector loads and bulk copies)."""
        if t.dtype not in (torch.float32, torch.bfloat16, torch.float16):
            t = t.float()
        t = t.contiguous()
        return t if t.data_ptr() % 16 == 0 else t.clone()

    # ----------------------------------------------------------- prefill
    def prefill(self, Q, K, V, positions):
        """FA+aux -> AnS -> selection -> layout (cache.py:100-140).  Returns
        the full-precision prefill attention output."""
        if self._n:
            raise ValueError("prefill on a non-empty cache")
        Qt, Kt, Vt, single, was_np = self._shape_inputs(Q, K, V)
        B, Hq, n, d = Qt.shape
        _, Hkv, _, _ = Kt.shape
        if d % self.config.vq.d_sub != 0:
            raise ValueError("head dimension incompatible with codebook")
        if d % 2:
            raise ValueError("head dimension must be even for RoPE")
        if Hq % Hkv:
            raise ValueError("query heads must be a multiple of KV heads")
        if B != self.B:
            raise ValueError(f"cache was created for batch {self.B}")
        # the three checks of attention.py:59-67: one HBM pass each on the GPU
        # (antkv_check_finite), one host synchronisation for all three
        flags = torch.zeros(3, dtype=torch.int32, device=Qt.device)
        for i, X in enumerate((Qt, Kt, Vt)):
            if (X.is_contiguous() and X.data_ptr() % 16 == 0
                    and X.dtype in (torch.float32, torch.bfloat16, torch.float16)):
                _lib.call("antkv_check_finite", _lib.ptr(X), _lib.dtype_tag(X), X.numel(),
                          _lib.ptr(flags[i:]), _lib.stream())
            else:
                flags[i] = (~torch.isfinite(X)).any().to(torch.int32)
        bad = flags.cpu()
        if bool(bad.any()):
            from .errors import NumericalError
            name = ("Q", "K", "V")[int(bad.nonzero()[0, 0])]
            raise NumericalError(f"non-finite values in {name}")
        self._single = single
        self.Hq, self.Hkv, self.d = Hq, Hkv, d
        pos_np = np.array(positions.detach().cpu().numpy() if isinstance(positions, torch.Tensor)
                          else positions, dtype=np.int64)
        if pos_np.ndim == 1:
            pos_np = np.repeat(pos_np[None], B, axis=0)
        if pos_np.shape != (B, n):
            raise ValueError("positions must have one entry per token")
        if np.any(pos_np < 0):
            raise ValueError("positions must be nonnegative")
        dev = Qt.device
        pos = torch.from_numpy(np.ascontiguousarray(pos_np)).to(dev)
        Qc, Kc, Vc = self._row_dtype(Qt), self._row_dtype(Kt), self._row_dtype(Vt)
        dt = _lib.dtype_tag(Qc)
        if _lib.dtype_tag(Kc) != dt or _lib.dtype_tag(Vc) != dt:
            Qc, Kc, Vc = Qc.float(), Kc.float(), Vc.float()
            dt = _lib.F32
        O = torch.empty((B, Hq, n, d), dtype=torch.float32, device=dev)
        M = torch.empty((B, Hq, n), dtype=torch.float32, device=dev)
        L = torch.empty_like(M)
        qn = torch.empty_like(M)
        th = float(self.config.theta_base)
        st = _lib.stream()
        ans_k = torch.empty((B, Hkv, n), dtype=torch.float32, device=dev)
        ans_v = torch.empty_like(ans_k)
        # FA + aux and AnS (cache.py:100-121) in one call: bf16 d = 128 rows
        # share one set of RoPE'd, split tiles between the two tcgen05 kernels
        _lib.call("antkv_prefill_attention_scores", _lib.ptr(Qc), _lib.ptr(Kc), _lib.ptr(Vc), dt,
                  _lib.ptr(pos), B, Hq, Hkv, n, d, th, _lib.ptr(O), _lib.ptr(M), _lib.ptr(L),
                  _lib.ptr(qn), _lib.ptr(ans_k), _lib.ptr(ans_v), st)
        self.last_scores = (ans_k, ans_v)
        budget = self.config.budget_for(n)
        anchors = select_anchors_device(ans_k.view(B * Hkv, n), ans_v.view(B * Hkv, n), budget,
                                        self.config.policy).view(B, Hkv, budget)
        self.build_from(Kc, Vc, pos, anchors)
        self._last_pos = pos_np[:, -1].copy() if n else None
        if single:
            return O[0, 0].cpu().numpy().astype(np.float64) if was_np else O[0, 0]
        return O

    def build_from(self, K, V, positions, anchors):
        """Lay out an empty cache from K/V [B, Hkv, n, d], positions [B, n]
        (device int64) and sorted anchors int32 [B, Hkv, A] (cache.py:122-139).
        Also the entry point for caches whose anchors come from elsewhere
        (synthetic benchmarks, sequence shards)."""
        B, Hkv, n, d = K.shape
        if self.Hkv is None:
            self.Hkv = Hkv
        if self.Hq is None:
            self.Hq = Hkv
        self.d = d
        self._pool_min_anchors = max(self._pool_min_anchors, int(anchors.shape[-1]))
        K = self._row_dtype(K)
        V = self._row_dtype(V.to(K.dtype))
        if self.row_dtype is None:
            self.row_dtype = K.dtype
        self._ensure_capacity(n + 1)
        positions, anchors = positions.contiguous(), anchors.contiguous()
        _lib.call("antkv_cache_build", ctypes.byref(self._desc), _lib.ptr(K), _lib.ptr(V),
                  _lib.dtype_tag(K), _lib.ptr(positions), n,
                  _lib.ptr(anchors), int(anchors.shape[-1]), _lib.stream())
        self._n = n
        if n:
            pos_h = positions.cpu().numpy()
            self._last_pos = pos_h[:, -1].copy()
            # the tensor-core decode kernel needs position(slot) = position(0) + slot
            self._contiguous = bool(np.all(pos_h == pos_h[:, :1] + np.arange(n)[None, :]))

    # ------------------------------------------------------------ decode
    def _workspace(self):
        if self._ws is None:
            nbytes = _lib.load().antkv_decode_workspace_bytes(ctypes.byref(self._desc), self.splits)
            # zero-filled once: the kernels keep its ticket counters at zero
            self._ws = torch.zeros((int(nbytes),), dtype=torch.uint8,
                                   device=self._t["codes"].device)
        return self._ws

    def _use_fast(self, fast):
        """Kernel mode for the ABI's `fast` argument (0 generic, 1 best, 2
        staged); the tensor-core kernels need contiguous positions."""
        f = self.fast if fast is None else (2 if fast == "staged" else int(fast))
        return f if self._contiguous else 0

    def step_device(self, q, k, v, qpos, out, lse=None, fast=None):
        """One decode step on device tensors, no host synchronisation:
        append (k, v) as windowed, attend q over the cache, evict
        (antkv_decode_step: a single fused kernel on the d8m256 fast path).
        q [B, Hq, d], k/v [B, Hkv, d] (one dtype: bf16/fp16/fp32), qpos int64
        [B], out float32 [B, Hq, d].  The caller maintains capacity."""
        ws = self._workspace()
        lib = _lib.load(check_device=False)
        _lib.check(lib.antkv_decode_step(ctypes.byref(self._desc), _lib.ptr(q), _lib.ptr(k),
                                         _lib.ptr(v), _lib.dtype_tag(q), _lib.ptr(qpos),
                                         _lib.ptr(out), _lib.ptr(lse), _lib.ptr(ws), ws.numel(),
                                         self.splits, int(self._use_fast(fast)), _lib.stream()))

    def step_publish(self, q, k, v, qpos, out, lse, exchange, fast=None):
        """step_device (k is None: attention only) whose partial (out, lse)
        is also written into this rank's slot of every receive buffer of the
        PeerExchange, then flagged (antkv_decode_step_publish)."""
        ws = self._workspace()
        lib = _lib.load(check_device=False)
        seq = exchange.seq
        _lib.check(lib.antkv_decode_step_publish(
            ctypes.byref(self._desc), _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), _lib.dtype_tag(q),
            _lib.ptr(qpos), _lib.ptr(out), _lib.ptr(lse), _lib.ptr(ws), ws.numel(), self.splits,
            int(self._use_fast(fast)), _lib.ptr(exchange.dst_o), _lib.ptr(exchange.dst_lse),
            _lib.ptr(exchange.dst_flags), exchange.n_dst, exchange.rank, seq, _lib.stream()))

    def attend_device(self, q, qpos, out, lse=None, fast=None):
        """Attention only (no append/evict): used by sequence shards."""
        ws = self._workspace()
        _lib.call("antkv_decode_attention", ctypes.byref(self._desc), _lib.ptr(q),
                  _lib.dtype_tag(q), _lib.ptr(qpos), _lib.ptr(out), _lib.ptr(lse), _lib.ptr(ws),
                  ws.numel(), self.splits, int(self._use_fast(fast)), _lib.stream())

    def decode_step(self, q_new, k_new, v_new, position):
        """Append one token, attend, then evict (cache.py:149-194)."""
        pos = np.asarray(position.detach().cpu().numpy() if isinstance(position, torch.Tensor)
                         else position, dtype=np.int64).reshape(-1)
        if pos.size == 1 and self.B > 1:
            pos = np.repeat(pos, self.B)
        if self._last_pos is not None and np.any(pos <= self._last_pos):
            raise ValueError("position must exceed all existing positions")
        if self._last_pos is not None and np.any(pos != self._last_pos + 1):
            self._contiguous = False
        qt, was_np = as_cuda(q_new)
        kt, _ = as_cuda(k_new)
        vt, _ = as_cuda(v_new)
        single = qt.ndim == 1
        if single:
            qt, kt, vt = qt[None, None], kt[None, None], vt[None, None]
        if self._t is None or self._n == 0 and self.d is None:
            self._start_empty(qt, kt, single)
        self._ensure_capacity(self._n + 2)
        qt, kt, vt = self._row_dtype(qt), self._row_dtype(kt), self._row_dtype(vt.to(kt.dtype))
        qt = qt.to(kt.dtype)
        qp = torch.from_numpy(pos).to(qt.device)
        out = torch.empty((self.B, self.Hq, self.d), dtype=torch.float32, device=qt.device)
        self.step_device(qt, kt, vt, qp, out)
        self._n += 1
        self._last_pos = pos.copy()
        if single:
            return out[0, 0].cpu().numpy().astype(np.float64) if was_np else out[0, 0]
        return out

    def _start_empty(self, qt, kt, single):
        """decode_step on a cache that was never prefilled: the reference
        accepts it and takes d from the first token (cache.py:155-166); the
        shapes come from q [B, Hq, d] / k [B, Hkv, d]."""
        B, Hq, d = qt.shape
        Hkv = kt.shape[1]
        if B != self.B:
            raise ValueError(f"cache was created for batch {self.B}")
        if Hq % Hkv:
            raise ValueError("query heads must be a multiple of KV heads")
        if d % self.config.vq.d_sub != 0:
            raise ValueError("head dimension incompatible with codebook")
        self._single = single
        self.Hq, self.Hkv = Hq, Hkv
        dt = kt.dtype if kt.dtype in (torch.float32, torch.bfloat16, torch.float16) else torch.float32
        dev = kt.device
        empty = torch.empty((B, Hkv, 0, d), dtype=dt, device=dev)
        self.build_from(empty, empty, torch.empty((B, 0), dtype=torch.int64, device=dev),
                        torch.empty((B, Hkv, 0), dtype=torch.int32, device=dev))

    # ------------------------------------------------------- inspection
    def dequantize(self):
        """(K_hat, V_hat) float32 pre-RoPE (cache.py:196-211)."""
        n = self._n
        if n == 0:
            raise ValueError("cache is empty")
        dev = self._t["codes"].device
        Kh = torch.empty((self.B, self.Hkv, n, self.d), dtype=torch.float32, device=dev)
        Vh = torch.empty_like(Kh)
        _lib.call("antkv_cache_dequantize", ctypes.byref(self._desc), n, _lib.ptr(Kh),
                  _lib.ptr(Vh), _lib.stream())
        if self._single:
            return Kh[0, 0].cpu().numpy(), Vh[0, 0].cpu().numpy()
        return Kh, Vh

    def attention_from_cache(self, Q):
        """Causal attention of Q over the dequantised cache with RoPE at the
        stored positions (cache.py:213-223), on the GPU blocked kernel."""
        Qt, was_np = as_cuda(Q)
        single = Qt.ndim == 2
        if single:
            Qt = Qt[None, None]
        Kh, Vh = self.dequantize()
        if self._single:
            Kh, Vh = torch.from_numpy(Kh).cuda()[None, None], torch.from_numpy(Vh).cuda()[None, None]
        B, Hq, n, d = Qt.shape
        pos = self._t["positions"][:, :n]
        outs = []
        for b in range(B):
            p = pos[b].cpu().numpy()
            Qs, _ = rope_device(Qt[b].float().contiguous(), p, self.config.theta_base, 1.0 / math.sqrt(d))
            Kr, _ = rope_device(Kh[b].contiguous(), p, self.config.theta_base, 1.0)
            O = torch.empty((Hq, n, d), dtype=torch.float32, device=Qt.device)
            L = torch.empty((Hq, n), dtype=torch.float32, device=Qt.device)
            M = torch.empty_like(L)
            Vb = Vh[b].contiguous()
            _lib.call("antkv_flash_aux", _lib.ptr(Qs), _lib.ptr(Kr), _lib.ptr(Vb),
                      Hq, self.Hkv, n, n, d, d, 64, 64, 1, _lib.ptr(O), _lib.ptr(L), _lib.ptr(M),
                      _lib.stream())
            outs.append(O)
        O = torch.stack(outs)
        if single:
            return O[0, 0].cpu().numpy().astype(np.float64) if was_np else O[0, 0]
        return O

    def _host(self, key, b, h):
        """One (sequence, head) slice of a state tensor, on the host."""
        return self._t[key][b, h].cpu().numpy()

    def kinds_array(self, b=0, h=0):
        """Per-token kinds of (sequence b, KV head h) as int8 (KIND_ANCHOR /
        KIND_QUANTIZED / KIND_WINDOWED): one copy of the qmask and pool
        bookkeeping of that head, no per-token Python loop."""
        n = self._n
        kinds = np.full(n, _lib.KIND_QUANTIZED, dtype=np.int8)
        qm = self._host("qmask", b, h).view(np.uint32)
        bits = np.unpackbits(qm.view(np.uint8), bitorder="little")[:n].astype(bool)
        tok = self._host("pool_tok", b, h).astype(np.int64)
        kd = self._host("pool_kind", b, h).astype(np.int64)
        live = (tok >= 0) & (tok < n) & (kd != _lib.KIND_FREE)
        kinds[tok[live]] = np.where(kd[live] == _lib.KIND_ANCHOR, _lib.KIND_ANCHOR,
                                    _lib.KIND_WINDOWED).astype(np.int8)
        orphan = (kinds == _lib.KIND_QUANTIZED) & ~bits
        if orphan.any():
            raise RuntimeError(f"token {int(np.flatnonzero(orphan)[0])} has neither codes nor a "
                               "full-precision row")
        return kinds

    def kinds_of(self, b=0, h=0):
        """Per-token kind strings for (sequence b, KV head h)."""
        names = {_lib.KIND_ANCHOR: KIND_ANCHOR, _lib.KIND_QUANTIZED: KIND_QUANTIZED,
                 _lib.KIND_WINDOWED: KIND_WINDOWED}
        return [names[int(k)] for k in self.kinds_array(b, h)]

    @property
    def kinds(self):
        return self.kinds_of(0, 0)

    def anchor_indices_of(self, b=0, h=0):
        tok = self._host("pool_tok", b, h)
        kind = self._host("pool_kind", b, h)
        return np.sort(tok[(kind == _lib.KIND_ANCHOR) & (tok >= 0)].astype(np.int64))

    @property
    def anchor_indices(self):
        return self.anchor_indices_of(0, 0)

    def codes_array(self, b=0, h=0):
        """int64 [n, 2, groups] code indices (K, V) of every slot of
        (sequence b, KV head h); rows of non-quantized tokens hold stale
        values (see kinds_array)."""
        G = self.d // self.config.vq.d_sub
        raw = self._host("codes", b, h).reshape(-1)
        cap = self._t["codes"].shape[2]
        units = unpack_units(raw, _code_kind(self.config.vq, G))
        # tiled layout [tile][kv][16 slots][G] (common.cuh code_offset)
        arr = units.reshape(cap // 16, 2, 16, G).transpose(0, 2, 1, 3).reshape(cap, 2, G)
        return arr[:self._n].astype(np.int64)

    def codes_of(self, b=0, h=0):
        """(k_codes, v_codes) dicts {token: int64[groups]} for quantized tokens."""
        arr = self.codes_array(b, h)
        q = np.flatnonzero(self.kinds_array(b, h) == _lib.KIND_QUANTIZED)
        return {int(j): arr[j, 0] for j in q}, {int(j): arr[j, 1] for j in q}

    @property
    def positions(self):
        return [int(p) for p in self._t["positions"][0, :self._n].cpu()]

    def memory_report(self, b=0, h=0):
        """cache.py:225-243 semantics (full-precision rows counted as 2*d*32
        bits, as the reference stores them; on the GPU they are bf16)."""
        if self._n == 0:
            raise ValueError("cache is empty")
        nq = int((self.kinds_array(b, h) == _lib.KIND_QUANTIZED).sum())
        bits = self.config.vq.index_bits
        groups = self.d // self.config.vq.d_sub
        payload = nq * 2 * groups * bits + (self._n - nq) * 2 * self.d * 32
        denom = 2 * self._n * self.d
        return MemoryReport(payload_bits=payload,
                            codebook_bits=2 * self.config.vq.m * self.config.vq.d_sub * 32,
                            effective_bits_per_element=payload / denom,
                            fp_baseline_bits=denom * 32)

    def device_bytes(self):
        """Bytes of device memory held by the cache state."""
        return sum(t.numel() * t.element_size() for t in self._t.values())

    # ---------------------------------------------------------- snapshot
    def save(self, out_dir):
        """Reference snapshot format (cache.py:245-284) for a single-head
        cache; multi-head caches write one sub-directory per (b, head)."""
        out_dir = Path(out_dir)
        if self.B * self.Hkv > 1:
            for b in range(self.B):
                for h in range(self.Hkv):
                    self._save_one(out_dir / f"seq{b}_head{h}", b, h)
            (out_dir / "layout.json").write_text(json.dumps(
                {"B": self.B, "Hkv": self.Hkv, "Hq": self.Hq}) + "\n")
            return out_dir
        return self._save_one(out_dir, 0, 0)

    def _save_one(self, out_dir, b, h):
        out_dir.mkdir(parents=True, exist_ok=True)
        bits = self.config.vq.index_bits
        kinds = self.kinds_of(b, h)
        kc, vc = self.codes_of(b, h)
        tok = self._host("pool_tok", b, h)
        rows_bf = self._t["pool_rows"][b, h].float().cpu().numpy()
        slot_of = {int(tok[s]): s for s in range(len(tok)) if tok[s] >= 0}
        rows = bytearray()
        codes = bytearray()
        for j, kind in enumerate(kinds):
            if kind == KIND_QUANTIZED:
                codes.extend(pack_indices(list(kc[j]) + list(vc[j]), bits))
            else:
                s = slot_of[j]
                rows.extend(np.ascontiguousarray(rows_bf[s, 0], dtype="<f4").tobytes())
                rows.extend(np.ascontiguousarray(rows_bf[s, 1], dtype="<f4").tobytes())
        c = self.config
        manifest = {
            "format_version": FORMAT_VERSION,
            "config": {"vq": c.vq.notation, "anchor_fraction": c.anchor_fraction,
                       "anchor_count": c.anchor_count, "window_size": c.window_size,
                       "policy": c.policy, "theta_base": c.theta_base, "block_q": c.block_q,
                       "block_k": c.block_k},
            "n": self._n,
            "d": self.d,
            "positions": [int(p) for p in self._t["positions"][b, :self._n].cpu()],
            "kinds": kinds,
            "anchor_indices": [int(j) for j in self.anchor_indices_of(b, h)],
        }
        (out_dir / "manifest.json").write_text(json.dumps(manifest, indent=2) + "\n")
        (out_dir / "rows.bin").write_bytes(bytes(rows))
        (out_dir / "codes.bin").write_bytes(bytes(codes))
        ck = Codebook(self.codebook_k.config, self._t["cb_k"][h].cpu().numpy())
        cv = Codebook(self.codebook_v.config, self._t["cb_v"][h].cpu().numpy())
        save_codebook(ck, out_dir / "codebook_k.json")
        save_codebook(cv, out_dir / "codebook_v.json")
        return out_dir

    @classmethod
    def load(cls, in_dir, **kw):
        """Read a reference snapshot (cache.py:286-342) into a GPU cache."""
        in_dir = Path(in_dir)
        try:
            manifest = json.loads((in_dir / "manifest.json").read_text())
        except (OSError, json.JSONDecodeError) as exc:
            raise FormatError(f"cannot read cache manifest: {exc}") from exc
        if manifest.get("format_version") != FORMAT_VERSION:
            raise FormatError("unsupported cache format_version")
        cd = manifest["config"]
        config = CacheConfig(vq=VqConfig.from_notation(cd["vq"]),
                             anchor_fraction=cd["anchor_fraction"], anchor_count=cd["anchor_count"],
                             window_size=cd["window_size"], policy=cd["policy"],
                             theta_base=cd["theta_base"], block_q=cd["block_q"],
                             block_k=cd["block_k"])
        cbk = load_codebook(in_dir / "codebook_k.json")
        cbv = load_codebook(in_dir / "codebook_v.json")
        cache = cls(config, cbk, cbv, **kw)
        d, n = manifest["d"], manifest["n"]
        kinds = list(manifest["kinds"])
        groups = d // config.vq.d_sub
        bits = config.vq.index_bits
        token_bytes = (2 * groups * bits + 7) // 8
        rows = (in_dir / "rows.bin").read_bytes()
        codes = (in_dir / "codes.bin").read_bytes()
        K = np.zeros((n, d), dtype=np.float32)
        V = np.zeros((n, d), dtype=np.float32)
        kcodes = np.zeros((n, groups), dtype=np.int64)
        vcodes = np.zeros((n, groups), dtype=np.int64)
        r_off = c_off = 0
        for j, kind in enumerate(kinds):
            if kind == KIND_QUANTIZED:
                chunk = codes[c_off:c_off + token_bytes]
                if len(chunk) != token_bytes:
                    raise FormatError("truncated code section")
                both = unpack_indices(chunk, bits, 2 * groups)
                kcodes[j], vcodes[j] = both[:groups], both[groups:]
                c_off += token_bytes
            else:
                if r_off + 8 * d > len(rows):
                    raise FormatError("truncated row section")
                K[j] = np.frombuffer(rows, dtype="<f4", count=d, offset=r_off)
                V[j] = np.frombuffer(rows, dtype="<f4", count=d, offset=r_off + 4 * d)
                r_off += 8 * d
        if r_off != len(rows) or c_off != len(codes):
            raise FormatError("trailing bytes in cache binary sections")
        cache._restore(kinds, manifest["positions"], manifest["anchor_indices"], K, V,
                       kcodes, vcodes, d)
        return cache

    def _restore(self, kinds, positions, anchors, K, V, kcodes, vcodes, d):
        """Install an explicit single-head state (snapshot load)."""
        self._single = True
        self.B, self.Hkv, self.Hq, self.d = 1, 1, self.Hq or 1, d
        self.row_dtype = torch.float32          # the snapshot stores float32 rows
        n = len(kinds)
        self._ensure_capacity(n + 1)
        t = self._t
        G = d // self.config.vq.d_sub
        kind = _code_kind(self.config.vq, G)
        cap = t["codes"].shape[2]
        rec = np.zeros((cap, 2, G), dtype=np.uint16)
        rec[:n, 0], rec[:n, 1] = kcodes, vcodes
        tiled = rec.reshape(cap // 16, 16, 2, G).transpose(0, 2, 1, 3).reshape(-1)
        t["codes"][0, 0] = torch.from_numpy(pack_units(tiled, kind).reshape(cap, -1)).cuda()
        qbits = np.zeros(t["qmask"].shape[-1] * 32, dtype=np.uint8)
        P = t["pool_tok"].shape[-1]
        ptok = np.full(P, -1, np.int32)
        pkind = np.full(P, -1, np.int8)
        ring = []
        s = 0
        for j, kind in enumerate(kinds):
            if kind == KIND_QUANTIZED:
                qbits[j] = 1
            else:
                ptok[s] = j
                pkind[s] = _lib.KIND_ANCHOR if kind == KIND_ANCHOR else _lib.KIND_WINDOWED
                if kind == KIND_WINDOWED:
                    ring.append(s)
                t["pool_rows"][0, 0, s, 0] = torch.from_numpy(K[j]).to(t["pool_rows"].dtype)
                t["pool_rows"][0, 0, s, 1] = torch.from_numpy(V[j]).to(t["pool_rows"].dtype)
                s += 1
        t["qmask"][0, 0] = torch.from_numpy(np.packbits(qbits, bitorder="little").view(np.int32).copy()).cuda()
        t["pool_tok"][0, 0] = torch.from_numpy(ptok).cuda()
        t["pool_kind"][0, 0] = torch.from_numpy(pkind).cuda()
        W = self.config.window_size
        t["win_ring"][0, 0, :len(ring)] = torch.tensor(ring, dtype=torch.int32)
        free = list(range(P - 1, s - 1, -1))
        t["free_stack"][0, 0, :len(free)] = torch.tensor(free, dtype=torch.int32)
        t["hstate"][0, 0] = torch.tensor([sum(k == KIND_ANCHOR for k in kinds), 0, len(ring),
                                          len(free), s, 0, 0, 0], dtype=torch.int32)
        t["seq_len"][0] = n
        t["positions"][0, :n] = torch.tensor(positions, dtype=torch.int64)
        self._n = n
        self._last_pos = np.asarray([positions[-1]], dtype=np.int64) if n else None
        self._contiguous = bool(n == 0 or np.all(np.asarray(positions) == positions[0] + np.arange(n)))
        if "cb_f16" in t:
            _lib.call("antkv_cache_prepare_fast", ctypes.byref(self._desc), _lib.stream())
        if "cb_f16g" in t:
            _lib.call("antkv_cache_prepare_tc", ctypes.byref(self._desc), _lib.stream())
