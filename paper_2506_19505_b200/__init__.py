"""B200-native AnTKV anchor-token sub-bit KV-cache path (arXiv 2506.19505).

Drop-in for the reference ``antkv`` package's hot path: codebook objects,
anchor scoring and selection, the quantised KV cache (prefill / decode_step /
dequantize / attention_from_cache / snapshot) and the three reference kernels
(``kernels`` = an ``antkv._ckernels`` replacement).  Everything computes on
sm_100a through libantkv_b200.so; there is no CPU fallback.
"""

from .errors import FormatError, NumericalError, UnsupportedError
from .vq import (Codebook, KMeansResult, VqConfig, bits_per_element, decode_rows, decode_token,
                 encode_rows, encode_token, load_codebook, save_codebook, weighted_kmeans)
from .attention import (AttentionAux, RopeParams, apply_rope, attention_exact, attention_scores,
                        flash_attention_aux, softmax_rows)
from .anchors import AnchorScores, AnchorSelection, anchor_scores, anchor_scores_blocked, select_anchors
from .cache import CacheConfig, MemoryReport, QuantizedKVCache
from . import kernels

__version__ = "0.1.0"

__all__ = [
    "AnchorScores", "AnchorSelection", "AttentionAux", "CacheConfig", "Codebook", "FormatError",
    "MemoryReport", "NumericalError", "QuantizedKVCache", "RopeParams", "UnsupportedError",
    "VqConfig", "anchor_scores_blocked", "apply_rope", "bits_per_element", "decode_rows",
    "decode_token", "encode_rows", "encode_token", "flash_attention_aux", "kernels",
    "load_codebook", "save_codebook", "select_anchors", "KMeansResult", "weighted_kmeans",
    "anchor_scores", "attention_exact", "attention_scores", "softmax_rows",
]
