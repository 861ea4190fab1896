"""Device-memory plumbing: residues live in CUDA ``torch.int64`` tensors that
are bit-reinterpreted as uint64 by the kernels.  Host inputs (numpy uint64 or
CPU tensors) are copied in and results copied back, so the drop-in API keeps
the reference's value semantics for host callers."""

from __future__ import annotations

import numpy as np
import torch

from .errors import ConfigError, RingMpcError

_DEVICE = None


def device() -> torch.device:
    global _DEVICE
    if _DEVICE is None:
        if not torch.cuda.is_available():
            raise RingMpcError("no CUDA device: this package runs its protocol only on the GPU")
        _DEVICE = torch.device("cuda", torch.cuda.current_device())
        bind_thread()
    return _DEVICE


def bind_thread() -> None:
    """Point the library's own CUDA runtime at this thread's device (torch's current device): the
    library links the runtime statically, so its per-thread current device is not torch's."""
    from . import _lib

    _lib.call("hb_set_device", torch.cuda.current_device())


def is_device(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def to_device(a, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """uint64 residues as a contiguous CUDA int64 tensor (no copy if already there)."""
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.uint64:
            a = a.view(torch.int64)
        if a.dtype != torch.int64:
            raise ConfigError(f"share tensors must hold 64-bit words, got {a.dtype}")
        if a.is_cuda:
            return a.contiguous()
        return a.contiguous().to(device(), non_blocking=a.is_pinned())
    arr = np.asarray(a)
    if arr.dtype != np.uint64:
        raise ConfigError("share data must be uint64 residues")
    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.int64))
    return t.to(device())


def to_host(t: torch.Tensor, like) -> object:
    """Return `t` in the caller's representation (numpy for numpy inputs)."""
    if isinstance(like, torch.Tensor):
        if like.is_cuda:
            return t
        if like.is_pinned():
            out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            out.copy_(t, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return out
        return t.cpu()
    return t.cpu().numpy().view(np.uint64)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def words(nbytes: int) -> torch.Tensor:
    return torch.empty(max(nbytes // 8, 1), dtype=torch.int64, device=device())


def stream_handle(s: torch.cuda.Stream | None = None) -> int:
    s = s or torch.cuda.current_stream()
    return s.cuda_stream
