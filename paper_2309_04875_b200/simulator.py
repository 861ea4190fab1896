"""The windowed sign decision evaluated in the clear, on the GPU -- the offline window search's
inner loop, for models the reference cannot express (ResNets, ``nn.Residual``).

``drelu_from_shares`` is the arithmetic the protocol evaluates under encryption
(ringmpc simulator.py:33-44): slice both shares of an explicit split, add on the
(k-m)-bit ring, keep iff the top bit is clear.  ``sim_relu`` is the simulator's
windowed ReLU on floats (simulator.py:47-54): encode, split, decide, keep-or-zero --
one fused CUDA kernel (``hb_sim_relu``) that regenerates the split's randomness from the
caller's numpy generator state on the device (PCG64 jump-ahead: the same draws as
``rng.bytes``), so the output is bit-identical to the reference.  ``sim_forward``,
``plain_forward``, ``collect_drelu_decisions`` and ``collect_activation_ranges`` follow
simulator.py:57-174 with the float pipeline on the GPU in float64 (library conv/matmul --
this is the offline search, not the online path; float summation order differs from
numpy's im2col matmul, so logits agree to ~1e-12 relative, and the ReLU decisions are
exact given equal pre-activations).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib, ring, sharing
from .errors import ConfigError, EncodeRangeError
from .ring import BitWindow, FixedPointConfig


@dataclass
class SimConfig:
    """Windows per ReLU group plus the split seed (simulator.py:25-30)."""

    fxp: FixedPointConfig
    windows: list = field(default_factory=list)
    seed: int = 0


def drelu_from_shares(s0, s1, width: int, window: BitWindow):
    """1 where the window's sign bit of (s0 + s1) is clear (simulator.py:33-44)."""
    window.check_fits(width)
    a, b = _dev.to_device(s0).reshape(-1), _dev.to_device(s1).reshape(-1)
    out = torch.empty_like(a)
    _lib.call("hb_ewise", _lib.EW["DRELU_SHARES"], 0, window.width, a.numel(), window.m, a.data_ptr(), b.data_ptr(),
              out.data_ptr(), None, _dev.stream_handle())
    return _dev.to_host(out.reshape(tuple(np.shape(s0))), s0)


def _sim_relu_dev(x: torch.Tensor, window: BitWindow, cfg: FixedPointConfig, rng: np.random.Generator) -> torch.Tensor:
    """Device float64 x -> x * keep; consumes x.numel() 64-bit draws of `rng` (as share_arith does)."""
    window.check_fits(cfg.ring_bits)
    x = x.contiguous().to(torch.float64)
    n = x.numel()
    st = rng.bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    out = torch.empty_like(x)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    m64 = (1 << 64) - 1
    _lib.call("hb_sim_relu", x.data_ptr(), n, cfg.frac_bits, cfg.ring_bits, window.k, window.m, s & m64, s >> 64,
              inc & m64, inc >> 64, out.data_ptr(), err.data_ptr(), _dev.stream_handle())
    rng.bit_generator.advance(n)  # the generator moves past the split, as rng.bytes(8 n) would
    if int(err.item()):
        raise EncodeRangeError(f"input exceeds the signed range of a {cfg.ring_bits}-bit ring")
    return out


def sim_relu(x_f, window: BitWindow, cfg: FixedPointConfig, rng: np.random.Generator):
    """Windowed ReLU on floats: encode, split, slice, keep-or-zero (simulator.py:47-54)."""
    on_host = not isinstance(x_f, torch.Tensor)
    x = torch.from_numpy(np.ascontiguousarray(x_f, dtype=np.float64)).to(_dev.device()) if on_host else x_f
    out = _sim_relu_dev(x, window, cfg, rng)
    return out.cpu().numpy() if on_host else out


def exact_relu(x: torch.Tensor, cfg: FixedPointConfig) -> torch.Tensor:
    """Keep x where encode(x) is non-negative (simulator.py:85-93): x * (rounded >= 0)."""
    s = x * float(cfg.scale)
    r = torch.copysign(torch.floor(torch.abs(s) + 0.5), s)
    if bool((torch.abs(r) >= float(1 << (cfg.ring_bits - 1))).any()):
        raise EncodeRangeError(f"input exceeds the signed range of a {cfg.ring_bits}-bit ring")
    return x * (r >= 0).to(torch.float64)


def _float_forward(model, x_f, relu_hook) -> torch.Tensor:
    """Float64 pipeline on the GPU; relu_hook(layer_path, group_id, pre_activation) -> post.
    layer_path is (i,) for top-level layer i, as the reference indexes (simulator.py:57-82), and
    (i, 0, j) / (i, 1, j) for layer j of Residual i's body / shortcut."""
    import torch.nn.functional as F

    from .nn import AvgPool, Conv2d, Flatten, Linear, Relu, Residual

    def w(name):
        return torch.from_numpy(np.asarray(model.weights[name], dtype=np.float64)).to(_dev.device())

    def run(layers, cur, prefix):
        for i, L in enumerate(layers):
            idx = prefix + (i,)
            if isinstance(L, Linear):
                cur = cur @ w(L.weight).T + w(L.bias)[None, :]
            elif isinstance(L, Conv2d):
                cur = F.conv2d(cur, w(L.weight), w(L.bias), L.stride, L.pad)
            elif isinstance(L, AvgPool):
                cur = F.avg_pool2d(cur, (L.kh, L.kw), L.stride)
            elif isinstance(L, Relu):
                cur = relu_hook(idx, L.group_id, cur)
            elif isinstance(L, Flatten):
                cur = cur.reshape(cur.shape[0], -1)
            elif isinstance(L, Residual):
                cur = run(L.body, cur, idx + (0,)) + run(L.shortcut, cur, idx + (1,))
            else:
                raise ConfigError(f"unknown layer kind {L!r}")
        return cur

    x = torch.from_numpy(np.asarray(x_f, dtype=np.float64)).to(_dev.device())
    return run(model.layers, x, ())


def plain_forward(model, x_f) -> np.ndarray:
    """Float forward with exact (full-window) ReLU decisions (simulator.py:96-98)."""
    return _float_forward(model, x_f, lambda i, g, a: exact_relu(a, model.fixed_point)).cpu().numpy()


def _split_rng(seed: int, layer_path: tuple) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed, *layer_path]))


def sim_forward(model, x_f, labels, cfg: SimConfig):
    """Forward with windowed ReLU decisions -> (logits, accuracy) (simulator.py:101-124); the
    split of layer i is seeded by (cfg.seed, i) so a configuration always sees the same splits."""
    if len(cfg.windows) != model.n_groups:
        raise ConfigError(f"sim config has {len(cfg.windows)} windows, model needs {model.n_groups}")

    def hook(layer_index, group_id, act):
        window = cfg.windows[group_id]
        if window is None:
            return act
        return _sim_relu_dev(act, window, cfg.fxp, _split_rng(cfg.seed, layer_index))

    logits = _float_forward(model, x_f, hook).cpu().numpy()
    accuracy = float("nan")
    if labels is not None:
        accuracy = float(np.mean(np.argmax(logits, axis=1) == np.asarray(labels)))
    return logits, accuracy


def collect_drelu_decisions(model, x_f, cfg: SimConfig):
    """sim_forward plus each ReLU layer's keep mask (simulator.py:127-144)."""
    masks = []

    def hook(layer_index, group_id, act):
        window = cfg.windows[group_id]
        if window is None:
            masks.append(np.ones(tuple(act.shape), dtype=bool))
            return act
        out = _sim_relu_dev(act, window, cfg.fxp, _split_rng(cfg.seed, layer_index))
        masks.append((out != 0.0).cpu().numpy())
        return out

    logits = _float_forward(model, x_f, hook).cpu().numpy()
    return logits, masks


def collect_activation_ranges(model, x_f, cfg: FixedPointConfig | None = None) -> dict:
    """Smallest k per ReLU group holding every encoded pre-activation seen (simulator.py:147-174)."""
    cfg = cfg or model.fixed_point
    extremes: dict = {}

    def hook(layer_index, group_id, act):
        s = act * float(cfg.scale)
        r = torch.copysign(torch.floor(torch.abs(s) + 0.5), s)
        lo, hi = int(r.min().item()), int(r.max().item())
        if group_id in extremes:
            plo, phi = extremes[group_id]
            extremes[group_id] = (min(lo, plo), max(hi, phi))
        else:
            extremes[group_id] = (lo, hi)
        return exact_relu(act, cfg)

    _float_forward(model, x_f, hook)

    def bits_for(value: int) -> int:
        return value.bit_length() + 1 if value >= 0 else (-value - 1).bit_length() + 1

    return {g: min(max(2, bits_for(lo), bits_for(hi)), cfg.ring_bits) for g, (lo, hi) in extremes.items()}


__all__ = ["SimConfig", "drelu_from_shares", "sim_relu", "exact_relu", "plain_forward", "sim_forward",
           "collect_drelu_decisions", "collect_activation_ranges"]
_ = (ring, sharing)
