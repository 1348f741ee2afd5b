"""numpy <-> CUDA tensor plumbing for the reference-shaped (numpy) API."""

import numpy as np
import torch


def as_cuda(x, dtype=None):
    """Return (CUDA tensor, was_numpy).  numpy float64 becomes float32."""
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
        if dtype is not None:
            t = t.to(dtype)
        return t, False
    a = np.asarray(x)
    if a.dtype == np.float64:
        a = a.astype(np.float32)
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if dtype is not None:
        t = t.to(dtype)
    return t, True


def back(t, was_numpy, np_dtype=None):
    if not was_numpy:
        return t
    a = t.detach().cpu().numpy()
    if np_dtype is not None:
        a = a.astype(np_dtype)
    elif a.dtype == np.float32:
        a = a.astype(np.float64)
    return a
