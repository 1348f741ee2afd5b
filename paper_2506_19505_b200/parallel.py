"""Sequence (context) sharding of the quantised cache across GPUs.

Rank r owns a contiguous token range of every sequence: its codes, anchors
and (on the last rank) the full-precision window that receives appended
tokens.  A decode step runs the local split-KV kernel on every rank, producing
a normalised partial output and its log-sum-exp, all-gathers the partials
(NCCL over NVLink; ~Hq*(d+1)*4 bytes per rank per layer-step) and merges them
with the LSE combine kernel.  This is the only exchange on the decode path
(SURVEY.md §5, §8e).
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["shard_ranges", "gather_partials", "lse_merge", "ShardedDecoder"]


def shard_ranges(n, world):
    """Contiguous [start, stop) token ranges, sizes differing by at most one."""
    base, extra = divmod(n, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def gather_partials(o, lse, group=None):
    """All-gather (o [rows, d], lse [rows]) -> ([P, rows, d], [P, rows])."""
    world = dist.get_world_size(group)
    o = o.contiguous()
    lse = lse.contiguous()
    # concatenated along dim 0 (the form every backend accepts), then viewed
    o_all = torch.empty((world * o.shape[0],) + tuple(o.shape[1:]), dtype=o.dtype, device=o.device)
    l_all = torch.empty((world * lse.shape[0],) + tuple(lse.shape[1:]), dtype=lse.dtype,
                        device=lse.device)
    dist.all_gather_into_tensor(o_all, o, group=group)
    dist.all_gather_into_tensor(l_all, lse, group=group)
    return o_all.view((world,) + tuple(o.shape)), l_all.view((world,) + tuple(lse.shape))


def lse_merge(o_all, lse_all, out=None, lse_out=None):
    """Merge P normalised partials: out = sum_p w_p o_p, w_p ∝ exp(lse_p)
    (antkv_lse_combine).  GPU only."""
    P, rows, d = o_all.shape[0], int(np.prod(o_all.shape[1:-1])), o_all.shape[-1]
    if out is None:
        out = torch.empty(o_all.shape[1:], dtype=torch.float32, device=o_all.device)
    _lib.call("antkv_lse_combine", _lib.ptr(o_all.contiguous()), _lib.ptr(lse_all.contiguous()),
              P, rows, d, _lib.ptr(out), _lib.ptr(lse_out), _lib.stream())
    return out


class ShardedDecoder:
    """Decode driver for one rank's shard.

    ``cache`` holds this rank's token range (its ``desc.token_offset`` is the
    global index of its first slot).  Only the tail rank (``is_tail``) appends
    and evicts; every rank attends.  ``combine`` defaults to the GPU LSE merge;
    tests may pass another merge to exercise the collective on CPU/gloo."""

    def __init__(self, cache, is_tail, group=None, combine=None):
        self.cache = cache
        self.is_tail = is_tail
        self.group = group
        self.combine = combine or lse_merge

    def step(self, q, k, v, qpos, out_local, lse_local):
        """q [B, Hq, d], k/v [B, Hkv, d] (only used on the tail), qpos [B].
        The tail shard appends, attends and evicts in one fused launch
        (antkv_decode_step with the log-sum-exp output); the others attend."""
        c = self.cache
        if self.is_tail:
            c.step_device(q, k, v, qpos, out_local, lse_local)
            c._n += 1
        else:
            c.attend_device(q, qpos, out_local, lse_local)
        o_all, l_all = gather_partials(out_local, lse_local, self.group)
        return self.combine(o_all, l_all)
