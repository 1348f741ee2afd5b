"""ctypes binding of libantkv_b200.so (the C ABI in include/antkv_b200.h).

There is no CPU fallback: if the shared library is missing, or the device is
not an sm_100 part, every entry point raises.  Tensors cross the boundary as
raw device pointers; streams as the current torch CUDA stream handle.
"""

import ctypes
import os
from pathlib import Path

import torch

from .errors import UnsupportedError

# ANTKV_LIB overrides the library path (kernel experiments); there is no fallback
LIB_PATH = Path(os.environ.get("ANTKV_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libantkv_b200.so")

OK, EINVAL, ECUDA, EUNSUPPORTED = 0, 1, 2, 3
F32, BF16, F16 = 0, 1, 2
POLICY = {"by_k": 0, "by_v": 1, "by_sum": 2}
KIND_ANCHOR, KIND_QUANTIZED, KIND_WINDOWED, KIND_FREE = 0, 1, 2, -1
HSTATE_WORDS = 8
HS_ANCHORS, HS_WIN_HEAD, HS_WIN_COUNT, HS_FREE_TOP, HS_POOL_HIGH = 0, 1, 2, 3, 4

_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double
_f = ctypes.c_float


class CacheDesc(ctypes.Structure):
    """Mirror of antkv_cache_desc (include/antkv_b200.h)."""

    _fields_ = [
        ("B", _i), ("Hq", _i), ("Hkv", _i), ("d", _i), ("d_sub", _i), ("m", _i),
        ("groups", _i), ("index_bits", _i), ("code_bytes", _i), ("capacity", _i),
        ("pool_capacity", _i), ("window_size", _i), ("policy", _i), ("anchor_count", _i),
        ("row_dtype", _i), ("anchor_fraction", _d), ("theta_base", _d), ("token_offset", _i64),
        ("codes", _vp), ("qmask", _vp), ("pool_rows", _vp), ("pool_tok", _vp),
        ("pool_kind", _vp), ("win_ring", _vp), ("free_stack", _vp), ("hstate", _vp),
        ("seq_len", _vp), ("positions", _vp), ("codebook_k", _vp), ("codebook_v", _vp),
        ("codebook_f16", _vp), ("pool_f16", _vp), ("fast_tables", _vp),
        ("codebook_f16g", _vp), ("evict_scratch", _vp),
    ]


_SIGS = {
    "antkv_last_error": (ctypes.c_char_p, []),
    "antkv_version": (_i, []),
    "antkv_stream_exclusive": (_i, [_vp, _i]),
    "antkv_device_check": (_i, [_i]),
    "antkv_flash_aux": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "antkv_ans_blocked": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "antkv_assign_nearest": (_i, [_vp, _vp, _i64, _i, _i, _vp, _vp, _vp]),
    "antkv_rope_rotate": (_i, [_vp, _i, _vp, _i, _i, _i, _i, _d, _f, _vp, _vp, _vp]),
    "antkv_check_finite": (_i, [_vp, _i, _i64, _vp, _vp]),
    "antkv_prefill_attention": (_i, [_vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _d, _vp, _vp, _vp, _vp, _vp]),
    "antkv_prefill_anchor_scores": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _d, _vp, _vp, _vp]),
    "antkv_kmeans_assign_f64": (_i, [_vp, _vp, _i64, _i, _i, _vp, _vp, _vp]),
    "antkv_kmeans_update_f64": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp]),
    "antkv_eval_pair_l1": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "antkv_prefill_attention_scores": (_i, [_vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _d, _vp, _vp, _vp,
                                            _vp, _vp, _vp, _vp]),
    "antkv_p2p_alloc": (_i, [_i64, _vp]),
    "antkv_p2p_free": (_i, [_vp]),
    "antkv_ipc_get_handle": (_i, [_vp, _vp]),
    "antkv_ipc_open_handle": (_i, [_vp, _vp]),
    "antkv_ipc_close_handle": (_i, [_vp]),
    "antkv_decode_step_publish": (_i, [ctypes.POINTER(CacheDesc), _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i64, _i, _i, _vp, _vp,
                                       _vp, _i, _i, ctypes.c_uint32, _vp]),
    "antkv_lse_merge_wait": (_i, [_vp, _vp, _vp, _i, ctypes.c_uint32, _i64, _i, _vp, _vp, _vp]),
    "antkv_prefill_attention_block": (_i, [_vp, _vp, _vp, _i, _vp, _vp, _i, _i, _i, _i, _i, _i, _d, _i,
                                           _vp, _vp, _vp, _vp, _vp]),
    "antkv_prefill_anchor_scores_block": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                                               _i, _d, _i, _vp, _vp, _vp]),
    "antkv_select_anchors": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "antkv_vq_encode": (_i, [_vp, _i, _i64, _i, _vp, _i, _i, _vp, _i, _vp]),
    "antkv_vq_decode": (_i, [_vp, _i, _i64, _i, _vp, _i, _i, _vp, _vp]),
    "antkv_decode_workspace_bytes": (_i64, [ctypes.POINTER(CacheDesc), _i]),
    "antkv_cache_build": (_i, [ctypes.POINTER(CacheDesc), _vp, _vp, _i, _vp, _i, _vp, _i, _vp]),
    "antkv_cache_append": (_i, [ctypes.POINTER(CacheDesc), _vp, _vp, _i, _vp, _vp]),
    "antkv_decode_attention": (_i, [ctypes.POINTER(CacheDesc), _vp, _i, _vp, _vp, _vp, _vp, _i64, _i, _i, _vp]),
    "antkv_cache_evict": (_i, [ctypes.POINTER(CacheDesc), _vp]),
    "antkv_decode_step": (_i, [ctypes.POINTER(CacheDesc), _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i64, _i, _i, _vp]),
    "antkv_cache_dequantize": (_i, [ctypes.POINTER(CacheDesc), _i, _vp, _vp, _vp]),
    "antkv_lse_combine": (_i, [_vp, _vp, _i, _i64, _i, _vp, _vp, _vp]),
    "antkv_cache_prepare_fast": (_i, [ctypes.POINTER(CacheDesc), _vp]),
    "antkv_cache_prepare_tc": (_i, [ctypes.POINTER(CacheDesc), _vp]),
    "antkv_debug_trace": (_i, [_vp, _i]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(check_device=True):
    """Load the library (once).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2506_19505_b200/csrc`")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if check_device:
        _require_device()
    return _lib


_device_ok = {}


def _require_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_19505_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU path")
    dev = torch.cuda.current_device()
    if dev not in _device_ok:
        ok = _lib.antkv_device_check(dev)
        if not ok:
            raise RuntimeError("antkv_device_check failed: " + _lib.antkv_last_error().decode())
        _device_ok[dev] = True


def check(rc):
    if rc == OK:
        return
    msg = _lib.antkv_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EUNSUPPORTED:
        raise UnsupportedError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def call(name, *args):
    lib = load()
    check(getattr(lib, name)(*args))


def stream():
    return _vp(torch.cuda.current_stream().cuda_stream)


class exclusive_stream:
    """Context manager: declare the current stream exclusive to this
    library's launches (antkv_stream_exclusive) -- e.g. while capturing a
    graph of decode steps -- so the fused decode kernel may read its inputs
    before griddepcontrol.wait.  Only for chains with no foreign kernels."""

    def __enter__(self):
        self._s = stream()
        check(load().antkv_stream_exclusive(self._s, 1))
        return self

    def __exit__(self, *exc):
        check(load(check_device=False).antkv_stream_exclusive(self._s, 0))
        return False


def ptr(t):
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return _vp(t.data_ptr())


def dtype_tag(t):
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float16:
        return F16
    raise ValueError(f"unsupported dtype {t.dtype}")
