"""Device plumbing: torch is used only as the allocator / stream provider.

Residue buffers are torch int64 CUDA tensors reinterpreted as uint64 by the
native library (all residues are < 2^62, so the signed view is also exact).
"""

from __future__ import annotations

import numpy as np

from . import _lib

try:
    import torch
except Exception:  # pragma: no cover - torch is part of the image
    torch = None


def require_cuda():
    """Fail loudly when the GPU path cannot run (there is no CPU fallback)."""
    if torch is None or not torch.cuda.is_available():
        raise _lib.FcnUnavailable("a CUDA device is required: this package has no CPU fallback")
    _lib.load()


def current_device() -> int:
    require_cuda()
    return torch.cuda.current_device()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def empty(shape, device=None):
    require_cuda()
    return torch.empty(tuple(shape), dtype=torch.int64, device=device if device is not None else "cuda")


def zeros(shape, device=None):
    require_cuda()
    return torch.zeros(tuple(shape), dtype=torch.int64, device=device if device is not None else "cuda")


def to_device(arr, device=None):
    """numpy uint64/int64 array -> contiguous int64 CUDA tensor (bit-identical)."""
    require_cuda()
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype != np.int64:
        a = a.astype(np.int64)
    return torch.from_numpy(a).to(device if device is not None else "cuda", non_blocking=False)


def to_host(t) -> np.ndarray:
    """CUDA tensor -> numpy uint64 (bit-identical)."""
    return t.detach().contiguous().cpu().numpy().view(np.uint64)


def ptr(t) -> int:
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("device buffers passed to libfcn must be contiguous")
    return t.data_ptr()
