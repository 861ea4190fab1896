"""Secret-share tensor types and local (communication-free) share algebra.

Same conventions as the reference (sharing.py:1-10, 88-173): party 0 holds
x + r and party 1 holds -r (or x ^ r / r); public constants land on party 0
only; tensors carry their ring width and mixing widths is a ConfigError.

``data`` is either a numpy uint64 array (host, as in the reference) or a
CUDA int64 tensor read as uint64 (device).  Protocol calls accept both and
return the caller's representation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib, ring
from .errors import ConfigError
from .ring import BitWindow

PARTIES = (0, 1)


def _check_party(party: int) -> None:
    if party not in PARTIES:
        raise ConfigError(f"party must be 0 or 1, got {party}")


def _check_data(data, what: str) -> None:
    if isinstance(data, torch.Tensor):
        if data.dtype not in (torch.int64, torch.uint64):
            raise ConfigError(f"{what} data must be 64-bit words, got {data.dtype}")
    elif not (isinstance(data, np.ndarray) and data.dtype == np.uint64):
        raise ConfigError(f"{what} data must be uint64 residues")


class _Share:
    party: int
    width: int
    data: object

    def __post_init__(self) -> None:
        _check_party(self.party)
        ring.mask_of(self.width)
        _check_data(self.data, type(self).__name__)

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.data.shape)

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape)) if len(self.shape) else 1

    @property
    def on_device(self) -> bool:
        return _dev.is_device(self.data)

    def with_data(self, data, width: int | None = None):
        return type(self)(self.party, self.width if width is None else width, data)

    def cuda(self):
        return self.with_data(_dev.to_device(self.data))

    def numpy(self) -> np.ndarray:
        if isinstance(self.data, torch.Tensor):
            return self.data.detach().cpu().numpy().view(np.uint64)
        return self.data


@dataclass
class ArithShareTensor(_Share):
    """One party's additive share on Z/2^width (sharing.py:29-52)."""

    party: int
    width: int
    data: object

    __post_init__ = _Share.__post_init__


@dataclass
class BinShareTensor(_Share):
    """One party's XOR share of width-bit words (sharing.py:55-78)."""

    party: int
    width: int
    data: object

    __post_init__ = _Share.__post_init__


def _check_pair(a, b) -> None:
    if a.width != b.width:
        raise ConfigError(f"width mismatch: {a.width} vs {b.width}")
    if a.shape != b.shape:
        raise ConfigError(f"shape mismatch: {a.shape} vs {b.shape}")


def _mask_t(t: torch.Tensor, width: int) -> torch.Tensor:
    if width == 64:
        return t
    return torch.bitwise_and(t, (1 << width) - 1)


def _const_like(c, a):
    """Public constant as residues broadcast to a's shape, in a's representation."""
    arr = ring.to_unsigned(np.broadcast_to(np.asarray(c), a.shape), a.width)
    if a.on_device:
        return torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).to(a.data.device)
    return arr


# ------------------------------------------------------------ split / reconstruct (host prep)
def share_arith(secret: np.ndarray, width: int, rng: np.random.Generator):
    """(x + r, -r) with r from rng.bytes (sharing.py:88-96)."""
    secret = ring.to_unsigned(secret, width)
    r = ring.random_residues(rng, secret.size, width).reshape(secret.shape)
    return (ArithShareTensor(0, width, ring.add_mod(secret, r, width)),
            ArithShareTensor(1, width, ring.neg_mod(r, width)))


def share_binary(secret: np.ndarray, width: int, rng: np.random.Generator):
    secret = ring.to_unsigned(secret, width)
    r = ring.random_residues(rng, secret.size, width).reshape(secret.shape)
    return BinShareTensor(0, width, secret ^ r), BinShareTensor(1, width, r)


def reconstruct_arith(s0: ArithShareTensor, s1: ArithShareTensor) -> np.ndarray:
    _check_pair(s0, s1)
    return ring.add_mod(s0.numpy(), s1.numpy(), s0.width)


def reconstruct_binary(s0: BinShareTensor, s1: BinShareTensor) -> np.ndarray:
    _check_pair(s0, s1)
    return s0.numpy() ^ s1.numpy()


# ------------------------------------------------------------ local algebra
def _same_party(a, b, verb):
    _check_pair(a, b)
    if a.party != b.party:
        raise ConfigError(f"cannot {verb} shares held by different parties")


def add_shares(a: ArithShareTensor, b: ArithShareTensor) -> ArithShareTensor:
    _same_party(a, b, "add")
    if a.on_device:
        return a.with_data(_mask_t(a.data + _dev.to_device(b.data), a.width))
    return a.with_data(ring.add_mod(a.data, b.numpy(), a.width))


def sub_shares(a: ArithShareTensor, b: ArithShareTensor) -> ArithShareTensor:
    _same_party(a, b, "subtract")
    if a.on_device:
        return a.with_data(_mask_t(a.data - _dev.to_device(b.data), a.width))
    return a.with_data(ring.sub_mod(a.data, b.numpy(), a.width))


def neg_shares(a: ArithShareTensor) -> ArithShareTensor:
    if a.on_device:
        return a.with_data(_mask_t(-a.data, a.width))
    return a.with_data(ring.neg_mod(a.data, a.width))


def add_public(a: ArithShareTensor, c) -> ArithShareTensor:
    if a.party != 0:
        return a
    cv = _const_like(c, a)
    if a.on_device:
        return a.with_data(_mask_t(a.data + cv, a.width))
    return a.with_data(ring.add_mod(a.data, cv, a.width))


def mul_public(a: ArithShareTensor, c) -> ArithShareTensor:
    cv = _const_like(c, a)
    if a.on_device:
        return a.with_data(_mask_t(a.data * cv, a.width))
    return a.with_data(ring.mul_mod(a.data, cv, a.width))


def xor_shares(a: BinShareTensor, b: BinShareTensor) -> BinShareTensor:
    _same_party(a, b, "xor")
    if a.on_device:
        return a.with_data(torch.bitwise_xor(a.data, _dev.to_device(b.data)))
    return a.with_data(a.data ^ b.numpy())


def xor_public(a: BinShareTensor, c) -> BinShareTensor:
    if a.party != 0:
        return a
    cv = _const_like(c, a)
    if a.on_device:
        return a.with_data(torch.bitwise_xor(a.data, cv))
    return a.with_data(a.data ^ cv)


def slice_shares(s: ArithShareTensor, window: BitWindow) -> ArithShareTensor:
    """Keep bits m..k-1 locally, on the (k-m)-bit ring (sharing.py:165-173), on the GPU."""
    window.check_fits(s.width)
    x = _dev.to_device(s.data)
    out = torch.empty_like(x)
    _lib.call("hb_ewise", _lib.EW["SLICE"], s.party, window.width, x.numel(), window.m, x.data_ptr(), None,
              out.data_ptr(), None, _dev.stream_handle())
    return ArithShareTensor(s.party, window.width, _dev.to_host(out, s.data))
