"""The windowed sign decision evaluated in the clear, on the GPU.

``drelu_from_shares`` is the arithmetic the protocol evaluates under encryption
(ringmpc simulator.py:33-44): slice both shares of an explicit split, add on the
(k-m)-bit ring, keep iff the top bit is clear.  ``sim_relu`` is the simulator's
windowed ReLU on floats (simulator.py:47-54) -- encode, split with the caller's
generator (same draws as the reference), decide on the GPU.  They are the inner
loop of the offline window search and of protocol-vs-simulator agreement checks.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib, ring, sharing
from .ring import BitWindow, FixedPointConfig


def drelu_from_shares(s0, s1, width: int, window: BitWindow):
    """1 where the window's sign bit of (s0 + s1) is clear (simulator.py:33-44)."""
    window.check_fits(width)
    a, b = _dev.to_device(s0).reshape(-1), _dev.to_device(s1).reshape(-1)
    out = torch.empty_like(a)
    _lib.call("hb_ewise", _lib.EW["DRELU_SHARES"], 0, window.width, a.numel(), window.m, a.data_ptr(), b.data_ptr(),
              out.data_ptr(), None, _dev.stream_handle())
    return _dev.to_host(out.reshape(tuple(np.shape(s0))), s0)


def sim_relu(x_f: np.ndarray, window: BitWindow, cfg: FixedPointConfig, rng: np.random.Generator) -> np.ndarray:
    """Windowed ReLU on floats: encode, split, slice, keep-or-zero (simulator.py:47-54)."""
    e = ring.encode_array(x_f, cfg)
    s0, s1 = sharing.share_arith(e, cfg.ring_bits, rng)
    keep = drelu_from_shares(s0.data, s1.data, cfg.ring_bits, window)
    return np.asarray(x_f, dtype=np.float64) * keep.astype(np.float64)
