"""Fixed-point layers over shares and the model-level private-inference entry.

Same layer vocabulary, manifest JSON and semantics as the reference
(ringmpc nn.py:33-174, 198-325) -- Linear, Conv2d, AvgPool, Relu, Flatten --
plus ``Residual`` (out = body(x) + shortcut(x)), which ResNets need and the
reference lacks.  Every layer runs on the GPU:

* Linear / Conv2d: ring-exact (X W^T) mod 2^64 on the int8 tensor cores, by
  byte limbs: the share as 8 unsigned byte limbs, the encoded weight as J
  balanced signed byte limbs (once per model); limb products with the same
  byte shift accumulate in the same TMEM columns and the epilogue folds them
  mod 2^64 together with the local truncation, the party-0 bias and an
  optional fused residual add.  The path is the hand-written tcgen05 kernel:
  hb_limbs_nhwc (NHWC limb planes) + hb_conv_limbs_tma (TMA-fed implicit GEMM)
  for every ResNet geometry, small-K convs (the 3-channel stem) through
  hb_im2col_planes on the same kernel, and the fused-gather tcgen05 kernel
  hb_conv_limbs_tc for shapes neither TMA form tiles.  HB_RING_GEMM=cublaslt
  (im2col + torch._int_mm + combine) is a cross-check only, as is J > 3.
  Bit-identical to the reference's uint64 numpy matmul (nn.py:214-243).
* AvgPool: hb_avgpool (window sum, * encode(1/kk), truncation; nn.py:246-259).
* Relu: ``protocol.relu`` (one party, any endpoint) or, for both parties on one
  GPU, ``protocol.relu_pair`` (model_forward_pair / run_local_forward).
"""

from __future__ import annotations

import collections
import json
import os
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _dev, _lib, dealer, protocol, ring, sharing, transport
from .errors import ConfigError, DataFormatError
from .protocol import ProtocolSession
from .ring import BitWindow, FixedPointConfig
from .sharing import ArithShareTensor


# ------------------------------------------------------------------ layer vocabulary (nn.py:33-74)
@dataclass(frozen=True)
class Linear:
    in_features: int
    out_features: int
    weight: str
    bias: str
    kind: str = field(default="linear", init=False)


@dataclass(frozen=True)
class Conv2d:
    in_channels: int
    out_channels: int
    kh: int
    kw: int
    stride: int
    pad: int
    weight: str
    bias: str
    kind: str = field(default="conv2d", init=False)


@dataclass(frozen=True)
class AvgPool:
    kh: int
    kw: int
    stride: int
    kind: str = field(default="avgpool", init=False)


@dataclass(frozen=True)
class Relu:
    group_id: int
    kind: str = field(default="relu", init=False)


@dataclass(frozen=True)
class Flatten:
    kind: str = field(default="flatten", init=False)


@dataclass(frozen=True)
class Residual:
    """out = body(x) + shortcut(x) (empty shortcut = identity); a local add of shares."""

    body: tuple
    shortcut: tuple = ()
    kind: str = field(default="residual", init=False)


def _walk(layers):
    for L in layers:
        yield L
        if isinstance(L, Residual):
            yield from _walk(L.body)
            yield from _walk(L.shortcut)


def _out_shape(layers, cur):
    for L in layers:
        cur = _layer_shape(L, cur)
    return cur


def _layer_shape(L, cur):
    if isinstance(L, Linear):
        if cur != (L.in_features,):
            raise ConfigError(f"linear layer expects ({L.in_features},), got {cur}")
        return (L.out_features,)
    if isinstance(L, Conv2d):
        if len(cur) != 3 or cur[0] != L.in_channels:
            raise ConfigError(f"conv layer expects ({L.in_channels}, H, W), got {cur}")
        _, h, w = cur
        return (L.out_channels, (h + 2 * L.pad - L.kh) // L.stride + 1, (w + 2 * L.pad - L.kw) // L.stride + 1)
    if isinstance(L, AvgPool):
        if len(cur) != 3:
            raise ConfigError(f"avgpool expects (C, H, W), got {cur}")
        c, h, w = cur
        return (c, (h - L.kh) // L.stride + 1, (w - L.kw) // L.stride + 1)
    if isinstance(L, Flatten):
        return (int(np.prod(cur)),)
    if isinstance(L, Residual):
        a, b = _out_shape(L.body, cur), _out_shape(L.shortcut, cur)
        if a != b:
            raise ConfigError(f"residual branches disagree: {a} vs {b}")
        return a
    return cur  # Relu


@dataclass
class ModelSpec:
    """Layers + public float32 weights (nn.py:77-145)."""

    fixed_point: FixedPointConfig
    input_shape: tuple
    layers: list
    weights: dict

    def __post_init__(self) -> None:
        groups = [L.group_id for L in _walk(self.layers) if isinstance(L, Relu)]
        if sorted(set(groups)) != list(range(len(set(groups)))):
            raise ConfigError(f"relu group ids must cover 0..G-1, got {groups}")
        for L in _walk(self.layers):
            if isinstance(L, Linear):
                self._expect(L.weight, (L.out_features, L.in_features))
                self._expect(L.bias, (L.out_features,))
            elif isinstance(L, Conv2d):
                self._expect(L.weight, (L.out_channels, L.in_channels, L.kh, L.kw))
                self._expect(L.bias, (L.out_channels,))
        self.activation_shapes()

    def _expect(self, name, shape):
        if name not in self.weights:
            raise ConfigError(f"missing weight blob {name!r}")
        if tuple(self.weights[name].shape) != tuple(shape):
            raise ConfigError(f"blob {name!r} has shape {self.weights[name].shape}, expected {shape}")

    @property
    def n_groups(self) -> int:
        return len({L.group_id for L in _walk(self.layers) if isinstance(L, Relu)})

    def activation_shapes(self) -> list:
        shapes, cur = [tuple(self.input_shape)], tuple(self.input_shape)
        for L in self.layers:
            cur = _layer_shape(L, cur)
            shapes.append(cur)
        return shapes

    def relu_sites(self):
        """(group_id, per-sample element count) of every ReLU, in execution order."""
        out = []

        def visit(layers, cur):
            for L in layers:
                if isinstance(L, Relu):
                    out.append((L.group_id, int(np.prod(cur))))
                elif isinstance(L, Residual):
                    visit(L.body, cur)
                    visit(L.shortcut, cur)
                cur = _layer_shape(L, cur)

        visit(self.layers, tuple(self.input_shape))
        return out

    def relu_group_sizes(self) -> dict:
        sizes = {}
        for g, c in self.relu_sites():
            sizes[g] = sizes.get(g, 0) + c
        return sizes


@dataclass
class ReluConfig:
    """Per-group window or None (identity) (nn.py:148-174)."""

    windows: list

    @classmethod
    def full(cls, model: ModelSpec) -> "ReluConfig":
        return cls([BitWindow(model.fixed_point.ring_bits, 0)] * model.n_groups)

    def window_for(self, group_id: int):
        if not 0 <= group_id < len(self.windows):
            raise ConfigError(f"no window configured for relu group {group_id}")
        return self.windows[group_id]

    def to_json(self) -> dict:
        return {"groups": [w.to_json() if w is not None else "identity" for w in self.windows]}

    @classmethod
    def from_json(cls, obj: dict) -> "ReluConfig":
        return cls([None if e == "identity" else BitWindow.from_json(e) for e in obj["groups"]])


# ------------------------------------------------------------------ ring GEMM (int8 limbs)
@dataclass
class _LimbWeight:
    """Encoded weight W [N, K] as J balanced byte limbs, ready for the int8 GEMM."""

    n: int
    k: int
    kp: int
    np_: int
    j: int
    bt: torch.Tensor      # int8 [J*Np, Kp]  (row j*Np + n = limb j of W[n, :])
    colsum: torch.Tensor  # int32 [J, Np]
    bias: torch.Tensor    # uint64 (int64) [Np] encoded bias
    wl_tc: torch.Tensor | None = None  # int8 tiles for hb_conv_limbs_tc (None: not eligible)
    kp_tc: int = 0
    nt: int = 0
    wl_tma: torch.Tensor | None = None  # int8 tiles for hb_conv_limbs_tma, K order (ki, kj, c)
    nt_tma: int = 0                     # its N tile: 128 (two shift passes) when n >= 128
    wl_i2c: torch.Tensor | None = None  # small-K convs: im2col-plane tiles (K = C*kh*kw <= 64 padded to 64)


def _balanced_limbs(w: np.ndarray):
    """W = sum_j l_j 256^j with l_j in [-128, 127]; returns the list of limbs."""
    rem = w.astype(np.int64).copy()
    limbs = []
    while np.any(rem != 0) or not limbs:
        l = ((rem + 128) & 255) - 128
        limbs.append(l.astype(np.int8))
        rem = (rem - l) >> 8
        if len(limbs) > 8:
            raise ConfigError("weight limbs do not terminate")
    return limbs


def _prep_weight(weight: np.ndarray, bias: np.ndarray, cfg: FixedPointConfig) -> _LimbWeight:
    """Encode W once, split it into balanced byte limbs, lay the limbs out for both GEMM paths:
    bt (cuBLASLt) and wl_tc (tcgen05 kernel, UMMA tiles), both in the reference im2col patch
    order c*kh*kw + ki*kw + kj (nn.py:177-195)."""
    w = np.asarray(weight)
    n = w.shape[0]
    w_enc = ring.to_signed(ring.encode_array(w.reshape(n, -1).astype(np.float64), cfg), 64)
    k = w_enc.shape[1]
    kp, np_ = -(-k // 16) * 16, -(-n // 8) * 8
    limbs = _balanced_limbs(w_enc)
    j = len(limbs)
    bt = np.zeros((j, np_, kp), dtype=np.int8)
    for jj, l in enumerate(limbs):
        bt[jj, :n, :k] = l
    colsum = bt.astype(np.int32).sum(axis=2, dtype=np.int32)  # the kernel reads int32
    b = np.zeros(np_, dtype=np.uint64)
    b[:n] = ring.encode_array(np.asarray(bias, dtype=np.float64), cfg)
    dev = _dev.device()
    lw = _LimbWeight(n, k, kp, np_, j, torch.from_numpy(bt.reshape(j * np_, kp)).to(dev),
                     torch.from_numpy(colsum).to(dev), torch.from_numpy(b.view(np.int64)).to(dev))
    if j <= 3 and k <= 21900:
        lw.nt = 64 if n >= 64 else (32 if n > 16 else 16)
        lw.kp_tc = -(-k // 64) * 64
        lw.wl_tc = torch.from_numpy(_tc_tiles(limbs, n, k, lw.nt, lw.kp_tc)).to(dev)
        c = w.shape[1]
        if c % TMA_KB == 0:  # TMA path: TMA_KB-channel K blocks, tap-major K order
            if w.ndim == 4:
                kh, kw = w.shape[2], w.shape[3]
                limbs_t = [l.reshape(n, c, kh, kw).transpose(0, 2, 3, 1).reshape(n, k) for l in limbs]
            else:
                limbs_t = limbs
            # two shift passes (N tile 128) pay off when the K loop is long enough to amortise the
            # second TMEM drain per tile; short-K convs (ResNet 1x1s) stay on one pass at N tile 64
            lw.nt_tma = 128 if n >= 128 and _TMA_WIDE and k >= _TMA_WIDE_MIN_K else lw.nt
            lw.wl_tma = torch.from_numpy(_tc_tiles(limbs_t, n, k, lw.nt_tma, k, TMA_KB)).to(dev)
        elif w.ndim == 4 and k <= TMA_KB:  # small K: 1x1 conv over the im2col planes (reference K order)
            lw.nt_tma = 128 if n >= 128 and _TMA_WIDE else lw.nt
            lw.wl_i2c = torch.from_numpy(_tc_tiles(limbs, n, k, lw.nt_tma, TMA_KB, TMA_KB)).to(dev)
    return lw


def _tc_tiles(limbs, n, k, nt, kp, kb=64):
    """Weight limbs in a tensor-core kernel's order [n tile][k block of kb bytes][limb][row][kb B],
    each [rows x kb B] tile in the UMMA K-major swizzled layout of that row width: 16-byte chunk c
    of row r stored at chunk c ^ sw(r), sw = (r >> 1) & 3 (SWIZZLE_64B, hb_ring_tc.cu canon()) or
    (r >> 2) & 1 (SWIZZLE_32B, hb_conv_tma.cu)."""
    j = len(limbs)
    ntiles = -(-n // nt)
    full = np.zeros((j, ntiles * nt, kp), dtype=np.int8)
    for jj, l in enumerate(limbs):
        full[jj, :n, :k] = l
    nch = kb // 16
    t = full.reshape(j, ntiles, nt, kp // kb, nch, 16)                # j, tile, row, kb, chunk, e
    rows = np.arange(nt)
    sw = (rows >> 1) & 3 if kb == 64 else (rows >> 2) & 1
    src_chunk = np.arange(nch)[None, :] ^ sw[:, None]                  # stored chunk s holds chunk s ^ sw(r)
    t = t[:, :, rows[:, None], :, src_chunk, :]                       # -> (row, s, j, tile, kb, e)
    return np.ascontiguousarray(t.transpose(3, 4, 2, 0, 1, 5)).reshape(-1)  # tile, kb, j, row, s, e


TMA_KB = 64  # channel bytes per stage of hb_conv_limbs_tma (hb_conv_tma.cu TKB)
_TMA_WIDE = os.environ.get("HB_TMA_NT", "128") != "64"  # N tile 128 (two passes) for n >= 128
_TMA_WIDE_MIN_K = int(os.environ.get("HB_TMA_WIDE_MIN_K", "512"))


_WCACHE: dict = {}


def _weight(weight, bias, cfg) -> _LimbWeight:
    """Limb form of a layer's weight, prepared once per weight array (public data)."""
    key = (id(weight), id(bias), cfg)
    hit = _WCACHE.get(key)
    if hit is None or hit[0] is not weight or hit[1] is not bias:
        hit = (weight, bias, _prep_weight(weight, bias, cfg))
        _WCACHE[key] = hit
    return hit[2]


# "tc": hand-written tcgen05 (TMA implicit GEMM where eligible, else the fused gather kernel);
# "tcgather": always the gather kernel; "cublaslt": im2col + torch._int_mm + combine
RING_GEMM = os.environ.get("HB_RING_GEMM", "tc")


def _use_tc(lw: _LimbWeight) -> bool:
    return RING_GEMM in ("tc", "tcgather") and lw.wl_tc is not None


_PLANES: "collections.OrderedDict" = collections.OrderedDict()


def _limb_planes(x_nchw: torch.Tensor, stream) -> torch.Tensor:
    """NHWC byte-limb planes of a share (hb_limbs_nhwc), cached for the few most recent inputs so a
    residual block's body conv and shortcut conv (same input) split it once.  The cache holds the
    input tensor itself (its memory cannot be recycled while cached) and its version counter."""
    key = id(x_nchw)
    hit = _PLANES.get(key)
    if hit is not None and hit[0] is x_nchw and hit[1] == x_nchw._version:
        _PLANES.move_to_end(key)
        return hit[2]
    b, c, h, w = x_nchw.shape
    planes = torch.empty(8 * b * h * w * c, dtype=torch.uint8, device=x_nchw.device)
    _lib.call("hb_limbs_nhwc", x_nchw.data_ptr(), b, c, h, w, planes.data_ptr(), stream)
    _PLANES[key] = (x_nchw, x_nchw._version, planes)
    while len(_PLANES) > 4:
        _PLANES.popitem(last=False)
    return planes


def _tma_box(oh: int, ow: int):
    """The 128-pixel (batch, oh, ow) output box hb_tma_conv_box picks, as (bb, bh, bw), or None when
    the output geometry does not tile (hb_conv_tma.cu:573-591)."""
    if ow >= 128:
        return (1, 1, 128) if ow % 128 == 0 else None
    if 128 % ow:
        return None
    rows = 128 // ow
    if oh >= rows:
        return (1, rows, ow) if oh % rows == 0 else None
    return (rows // oh, oh, ow) if rows % oh == 0 else None


def _tma_box_ok(oh: int, ow: int, stride: int = 1) -> bool:
    """Mirror of every geometry check hb_tma_conv makes before encoding its tensor maps: the box
    tiles the output, and the input window it reads (box extent x conv stride) is at most 256 per
    dimension (hb_conv_tma.cu box check); the traversal stride is at most 8 and the output width at
    most 256 (hb_conv_limbs_tma's checks, hb_api.cu)."""
    box = _tma_box(oh, ow)
    return (box is not None and stride <= 8 and ow <= 256 and box[2] * stride <= 256
            and box[1] * stride <= 256)


def _tma_ok(x_nchw: torch.Tensor, geom, lw: _LimbWeight) -> bool:
    b, c, h, w = x_nchw.shape
    kh, kw, stride, pad = geom
    oh, ow = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    return (RING_GEMM == "tc" and lw.wl_tma is not None and c % TMA_KB == 0 and b > 0
            and _tma_box_ok(oh, ow, stride))


def _gemm_tc(x_nchw: torch.Tensor, geom, lw: _LimbWeight, party: int, frac: int,
             residual: torch.Tensor | None = None) -> torch.Tensor:
    """tcgen05 ring conv: NCHW share in, NCHW [b, n, oh, ow] share out.  TMA-fed implicit GEMM over
    NHWC limb planes (hb_limbs_nhwc + hb_conv_limbs_tma) when the layer qualifies, else the fused
    gather kernel (hb_conv_limbs_tc)."""
    b, c, h, w = x_nchw.shape
    kh, kw, stride, pad = geom
    oh, ow = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    out = torch.empty((b, lw.n, oh, ow), dtype=torch.int64, device=x_nchw.device)
    if _tma_ok(x_nchw, geom, lw):
        s = _dev.stream_handle()
        planes = _limb_planes(x_nchw, s)
        if residual is not None and residual.shape != out.shape:
            raise ConfigError(f"residual shape {tuple(residual.shape)} != conv output {tuple(out.shape)}")
        _lib.call("hb_conv_limbs_tma", planes.data_ptr(), b, c, h, w, kh, kw, stride, pad, lw.wl_tma.data_ptr(),
                  lw.n, lw.j, lw.nt_tma, party, frac, lw.bias.data_ptr() if party == 0 else None,
                  None if residual is None else residual.contiguous().data_ptr(), out.data_ptr(), s)
        return out
    if RING_GEMM == "tc" and lw.wl_i2c is not None and b > 0 and _tma_box_ok(oh, ow) and residual is None:
        s = _dev.stream_handle()
        planes = torch.empty(8 * b * oh * ow * TMA_KB, dtype=torch.uint8, device=x_nchw.device)
        _lib.call("hb_im2col_planes", x_nchw.data_ptr(), b, c, h, w, kh, kw, stride, pad, planes.data_ptr(), s)
        _lib.call("hb_conv_limbs_tma", planes.data_ptr(), b, TMA_KB, oh, ow, 1, 1, 1, 0, lw.wl_i2c.data_ptr(), lw.n,
                  lw.j, lw.nt_tma, party, frac, lw.bias.data_ptr() if party == 0 else None, None, out.data_ptr(), s)
        return out
    if residual is not None:
        raise ConfigError("residual fusion needs the TMA conv path")
    _lib.call("hb_conv_limbs_tc", x_nchw.data_ptr(), b, c, h, w, kh, kw, stride, pad, lw.wl_tc.data_ptr(), lw.n, lw.j,
              lw.kp_tc, lw.nt, party, frac, lw.bias.data_ptr() if party == 0 else None, out.data_ptr(),
              _dev.stream_handle())
    return out


def _gemm_cublaslt(x_nchw: torch.Tensor, geom, lw: _LimbWeight, party: int, frac: int, layout: int) -> torch.Tensor:
    """im2col + limb split kernel, one cuBLASLt int8 GEMM over all limb pairs, combine kernel.
    layout 1: NCHW [b, n, oh, ow] out (conv); 0: [b, n] (linear)."""
    b, c, h, w = x_nchw.shape
    kh, kw, stride, pad = geom
    oh, ow = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    m = b * oh * ow
    s = _dev.stream_handle()
    a = torch.empty((8 * m, lw.kp), dtype=torch.int8, device=x_nchw.device)
    _lib.call("hb_im2col_limbs", x_nchw.data_ptr(), b, c, h, w, kh, kw, stride, pad, lw.kp, a.data_ptr(), s)
    if 8 * m <= 16:  # the int8 GEMM needs more than 16 rows; padded rows are ignored
        a = torch.cat([a, torch.zeros((24 - 8 * m, lw.kp), dtype=torch.int8, device=a.device)])
    prod = torch._int_mm(a, lw.bt.t())  # [8m(+pad), J*Np] int32 -- tensor cores
    out = torch.empty(m * lw.n, dtype=torch.int64, device=x_nchw.device)
    _lib.call("hb_limb_combine", prod.data_ptr(), m, lw.n, lw.np_, lw.j, lw.colsum.data_ptr(), party, frac,
              lw.bias.data_ptr() if party == 0 else None, layout, oh * ow, out.data_ptr(), s)
    return out.view(b, lw.n, oh, ow) if layout == 1 else out.view(b, lw.n)


def _to_layout(d: torch.Tensor, have: str, want: str) -> torch.Tensor:
    if have == want or d.dim() != 4:
        return d
    if want == "nhwc":
        return d.permute(0, 2, 3, 1).contiguous()
    return d.permute(0, 3, 1, 2).contiguous()


def _conv_dev(d, lay, L: Conv2d, lw, party, frac, residual=None):
    """Conv on a device share in layout `lay`; returns (output, its layout).  `residual` (NCHW, the
    output's shape) is added in the TMA kernel's epilogue (callers check _conv_fusable first)."""
    geom = (L.kh, L.kw, L.stride, L.pad)
    d = _to_layout(d, lay, "nchw")
    if _use_tc(lw):
        return _gemm_tc(d, geom, lw, party, frac, residual), "nchw"
    return _gemm_cublaslt(d, geom, lw, party, frac, 1), "nchw"


# both parties' convs of a layer in one launch (hb_conv_limbs_tma_pair) in model_forward_pair;
# HB_CONV_PAIR=0 launches them one by one
CONV_PAIR = os.environ.get("HB_CONV_PAIR", "1") != "0"


def _conv_pair_dev(ds, lay, L: Conv2d, lw, parties, frac, residuals=None):
    """Both parties' TMA convs of one layer in ONE launch; None when the layer does not qualify
    (then the caller runs _conv_dev per party).  Same shares as two _conv_dev calls."""
    if not (CONV_PAIR and len(ds) == 2 and tuple(parties) == (0, 1) and _use_tc(lw)):
        return None
    geom = (L.kh, L.kw, L.stride, L.pad)
    xs = [_to_layout(d, lay, "nchw") for d in ds]
    if xs[0].shape != xs[1].shape or not _tma_ok(xs[0], geom, lw):
        return None
    b, c, h, w = xs[0].shape
    oh, ow = (h + 2 * L.pad - L.kh) // L.stride + 1, (w + 2 * L.pad - L.kw) // L.stride + 1
    outs = [torch.empty((b, lw.n, oh, ow), dtype=torch.int64, device=xs[0].device) for _ in xs]
    if residuals is not None and any(r.shape != outs[0].shape for r in residuals):
        return None
    s = _dev.stream_handle()
    planes = [_limb_planes(x, s) for x in xs]
    res = [None, None] if residuals is None else [r.contiguous().data_ptr() for r in residuals]
    _lib.call("hb_conv_limbs_tma_pair", planes[0].data_ptr(), planes[1].data_ptr(), b, c, h, w, L.kh, L.kw, L.stride,
              L.pad, lw.wl_tma.data_ptr(), lw.n, lw.j, lw.nt_tma, frac, lw.bias.data_ptr(), res[0], res[1],
              outs[0].data_ptr(), outs[1].data_ptr(), s)
    return outs


def _linear_dev(d, lw, party, frac):
    b, k = d.shape
    if _use_tc(lw):
        return _gemm_tc(d.reshape(b, k, 1, 1), (1, 1, 1, 0), lw, party, frac).view(b, lw.n)
    return _gemm_cublaslt(d.reshape(b, k, 1, 1), (1, 1, 1, 0), lw, party, frac, 0)


def _avgpool_dev(d, lay, L: AvgPool, party, cfg):
    inv = ring.encode_fixed(1.0 / (L.kh * L.kw), cfg).value
    s = _dev.stream_handle()
    if lay == "nhwc":
        b, h, w, c = d.shape
        oh, ow = (h - L.kh) // L.stride + 1, (w - L.kw) // L.stride + 1
        out = torch.empty((b, oh, ow, c), dtype=torch.int64, device=d.device)
        _lib.call("hb_avgpool_nhwc", d.data_ptr(), b, h, w, c, L.kh, L.kw, L.stride, inv, party, cfg.frac_bits,
                  out.data_ptr(), s)
        return out
    b, c, h, w = d.shape
    oh, ow = (h - L.kh) // L.stride + 1, (w - L.kw) // L.stride + 1
    out = torch.empty((b, c, oh, ow), dtype=torch.int64, device=d.device)
    _lib.call("hb_avgpool", d.data_ptr(), b * c, h, w, L.kh, L.kw, L.stride, inv, party, cfg.frac_bits,
              out.data_ptr(), s)
    return out


def _check_ring(x, cfg):
    if x.width != 64 or cfg.ring_bits != 64:
        raise ConfigError("GPU ring layers run on Z/2^64 shares (FixedPointConfig(ring_bits=64))")


def truncate_local(x: ArithShareTensor, cfg: FixedPointConfig) -> ArithShareTensor:
    """Local SecureML truncation (nn.py:198-211), on the GPU."""
    _check_ring(x, cfg)
    xd = _dev.to_device(x.data).reshape(-1)
    out = torch.empty_like(xd)
    # the avgpool kernel with a 1x1 window and inv = 1 is exactly the truncation
    _lib.call("hb_avgpool", xd.data_ptr(), xd.numel(), 1, 1, 1, 1, 1, 1, x.party, cfg.frac_bits, out.data_ptr(),
              _dev.stream_handle())
    return ArithShareTensor(x.party, x.width, _dev.to_host(out.reshape(x.shape), x.data))


def linear_forward(session: ProtocolSession, x: ArithShareTensor, weight, bias) -> ArithShareTensor:
    """x @ W^T + b with public fixed-point weights; no communication (nn.py:214-224)."""
    cfg = session.fxp
    _check_ring(x, cfg)
    if len(x.shape) != 2 or x.shape[1] != weight.shape[1]:
        raise ConfigError(f"linear expects [batch, {weight.shape[1]}], got {x.shape}")
    out = _linear_dev(_dev.to_device(x.data), _weight(weight, bias, cfg), x.party, cfg.frac_bits)
    return ArithShareTensor(x.party, 64, _dev.to_host(out, x.data))


def conv2d_forward(session: ProtocolSession, x: ArithShareTensor, layer: Conv2d, weight, bias) -> ArithShareTensor:
    """Convolution on NCHW shares (nn.py:227-243): fused tcgen05 kernel (NHWC inside) or
    im2col + cuBLASLt limb GEMM."""
    cfg = session.fxp
    _check_ring(x, cfg)
    if len(x.shape) != 4 or x.shape[1] != layer.in_channels:
        raise ConfigError(f"conv expects [batch, {layer.in_channels}, H, W], got {x.shape}")
    out, lay = _conv_dev(_dev.to_device(x.data), "nchw", layer, _weight(weight, bias, cfg), x.party, cfg.frac_bits)
    return ArithShareTensor(x.party, 64, _dev.to_host(_to_layout(out, lay, "nchw"), x.data))


def avgpool_forward(session: ProtocolSession, x: ArithShareTensor, layer: AvgPool) -> ArithShareTensor:
    """Window sum, * encode(1/kk), truncation (nn.py:246-259)."""
    cfg = session.fxp
    _check_ring(x, cfg)
    if len(x.shape) != 4:
        raise ConfigError(f"avgpool expects [batch, C, H, W], got {x.shape}")
    out = _avgpool_dev(_dev.to_device(x.data), "nchw", layer, x.party, cfg)
    return ArithShareTensor(x.party, 64, _dev.to_host(out, x.data))


def relu_forward(session: ProtocolSession, x: ArithShareTensor, window) -> ArithShareTensor:
    """Windowed ReLU; None is the identity with no rounds (nn.py:262-268)."""
    return x if window is None else protocol.relu(session, x, window)


def _add_dev(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(a)
    _lib.call("hb_add_shares", a.data_ptr(), b.contiguous().data_ptr(), a.numel(), out.data_ptr(),
              _dev.stream_handle())
    return out


def _has_relu(layers) -> bool:
    return any(isinstance(L, Relu) or (isinstance(L, Residual) and (_has_relu(L.body) or _has_relu(L.shortcut)))
               for L in layers)


def _conv_out_shape(d: torch.Tensor, L: Conv2d):
    b, _, h, w = d.shape
    return torch.Size((b, L.out_channels, (h + 2 * L.pad - L.kh) // L.stride + 1, (w + 2 * L.pad - L.kw) // L.stride + 1))


def _meter_delta(ep, before):
    after = ep.meter.snapshot()
    return sum(after[t][0] - before[t][0] for t in after), sum(after[t][1] - before[t][1] for t in after)


def _run_model(sessions, datas, model: ModelSpec, relu_cfg: ReluConfig, layer_meter, layer_times=None):
    """Run the layers for one party (model_forward) or both parties on this GPU
    (model_forward_pair).  Shares stay on the device between layers, in NCHW: the
    ReLU consumes triples in element order, so keeping the reference's element order
    is what makes the per-party shares (and the truncation after them) bit-exact.

    layer_times (a list, optional): every layer's device time, from CUDA events recorded on the
    current stream around its launches -- {"layer", "kind", "ms"} per layer at every nesting level
    (a Residual's entry includes its body's and shortcut's).  The per-round analogue of the
    reference's wall_ms (cli.py:172-178) for the fused path, whose rounds run inside one kernel.
    Not usable under CUDA-graph capture."""
    if len(relu_cfg.windows) != model.n_groups:
        raise ConfigError(f"relu config has {len(relu_cfg.windows)} groups, model needs {model.n_groups}")
    cfg = model.fixed_point
    parties = [s.party for s in sessions]

    pending = []

    def run(layers, ds, lay, prefix):
        for i, L in enumerate(layers):
            before = [s.endpoint.meter.snapshot() for s in sessions]
            if layer_times is not None:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            if isinstance(L, Relu):
                win = relu_cfg.window_for(L.group_id)
                if win is not None:
                    shares = [ArithShareTensor(p, 64, d) for p, d in zip(parties, ds)]
                    if len(sessions) == 2:
                        out = protocol.relu_pair(tuple(sessions), shares[0], shares[1], win)
                    else:
                        out = [protocol.relu(sessions[0], shares[0], win)]
                    ds = [o.data for o in out]
            elif isinstance(L, Residual):
                last = L.body[-1] if L.body else None
                if (layer_meter is None and isinstance(last, Conv2d) and RING_GEMM == "tc"
                        and not _has_relu(L.shortcut)):
                    # shortcut first (no ReLU: it opens nothing and draws no triples, so triple order
                    # and meters are unchanged), then the body with add_shares fused into its last conv
                    h, lh = run(L.shortcut, ds, lay, f"{prefix}{i}.short.")
                    a, la = run(L.body[:-1], ds, lay, f"{prefix}{i}.body.")
                    a = [_to_layout(d, la, "nchw") for d in a]
                    h = [_to_layout(y, lh, "nchw") for y in h]
                    lw = _weight(model.weights[last.weight], model.weights[last.bias], cfg)
                    geom = (last.kh, last.kw, last.stride, last.pad)
                    pair = _conv_pair_dev(a, "nchw", last, lw, parties, cfg.frac_bits, h)
                    if pair is not None:
                        ds = pair
                    elif _use_tc(lw) and _tma_ok(a[0], geom, lw) and all(
                            y.shape == _conv_out_shape(d, last) for d, y in zip(a, h)):
                        ds = [_conv_dev(d, "nchw", last, lw, p, cfg.frac_bits, y)[0] for d, p, y in zip(a, parties, h)]
                    else:
                        ds = [_add_dev(_conv_dev(d, "nchw", last, lw, p, cfg.frac_bits)[0], y)
                              for d, p, y in zip(a, parties, h)]
                    lay = "nchw"
                else:
                    a, la = run(L.body, ds, lay, f"{prefix}{i}.body.")
                    h, lh = run(L.shortcut, ds, lay, f"{prefix}{i}.short.")
                    ds = [_add_dev(x, _to_layout(y, lh, la)) for x, y in zip(a, h)]
                    lay = la
            elif isinstance(L, Conv2d):
                lw = _weight(model.weights[L.weight], model.weights[L.bias], cfg)
                pair = _conv_pair_dev(ds, lay, L, lw, parties, cfg.frac_bits)
                if pair is not None:
                    ds, lay = pair, "nchw"
                else:
                    res = [_conv_dev(d, lay, L, lw, p, cfg.frac_bits) for d, p in zip(ds, parties)]
                    ds, lay = [r[0] for r in res], res[0][1]
            elif isinstance(L, Linear):
                lw = _weight(model.weights[L.weight], model.weights[L.bias], cfg)
                ds = [_linear_dev(d, lw, p, cfg.frac_bits) for d, p in zip(ds, parties)]
            elif isinstance(L, AvgPool):
                ds = [_avgpool_dev(d, lay, L, p, cfg) for d, p in zip(ds, parties)]
            elif isinstance(L, Flatten):
                ds = [_to_layout(d, lay, "nchw").reshape(d.shape[0], -1) for d in ds]
                lay = "flat"
            else:
                raise ConfigError(f"unknown layer kind {L!r}")
            if layer_meter is not None:
                for p, (s, bef) in enumerate(zip(sessions, before)):
                    nb, nr = _meter_delta(s.endpoint, bef)
                    layer_meter[p].append({"layer": f"{prefix}{i}:{L.kind}", "bytes": nb, "rounds": nr})
            if layer_times is not None:
                ev1 = torch.cuda.Event(enable_timing=True)
                ev1.record()
                pending.append((f"{prefix}{i}", L.kind, ev0, ev1))
        return ds, lay

    try:
        ds, lay = run(model.layers, datas, "nchw" if datas[0].dim() == 4 else "flat", "")
    finally:
        _PLANES.clear()  # the limb-plane cache only serves convs sharing an input within one forward
    out = [_to_layout(d, lay, "nchw") for d in ds]
    if layer_times is not None:
        torch.cuda.synchronize()
        layer_times.extend({"layer": name, "kind": kind, "ms": a.elapsed_time(b)} for name, kind, a, b in pending)
    return out


def model_forward(session: ProtocolSession, x: ArithShareTensor, model: ModelSpec, relu_cfg: ReluConfig,
                  layer_meter: list | None = None) -> ArithShareTensor:
    """One party runs every layer (nn.py:271-307); shares stay on the GPU between layers."""
    (out,) = _run_model([session], [_dev.to_device(x.data)], model, relu_cfg,
                        None if layer_meter is None else (layer_meter,))
    return ArithShareTensor(x.party, x.width, _dev.to_host(out, x.data))


def model_forward_pair(sessions, x0: ArithShareTensor, x1: ArithShareTensor, model: ModelSpec,
                       relu_cfg: ReluConfig, layer_meter: tuple | None = None, layer_times: list | None = None):
    """Both parties on this GPU: local layers per party, every ReLU through the fused
    pair kernel (protocol.relu_pair).  Same shares and meters as two model_forward threads.
    layer_times: see _run_model (per-layer device time from CUDA events)."""
    o0, o1 = _run_model(list(sessions), [_dev.to_device(x0.data), _dev.to_device(x1.data)], model, relu_cfg,
                        layer_meter, layer_times)
    return (ArithShareTensor(0, x0.width, _dev.to_host(o0, x0.data)),
            ArithShareTensor(1, x1.width, _dev.to_host(o1, x1.data)))


def triple_requirements(model: ModelSpec, relu_cfg: ReluConfig, batch: int) -> dict:
    """(kind, width) -> count for one forward pass (nn.py:310-325)."""
    need = {}
    for g, count in model.relu_sites():
        win = relu_cfg.window_for(g)
        if win is None:
            continue
        for key, num in protocol.relu_triple_cost(count * batch, win.width, model.fixed_point.ring_bits).items():
            need[key] = need.get(key, 0) + num
    return need


# ------------------------------------------------------------------ model-level entry (cli.py:159-180)
_INPUT_STREAM = 0x1289


def _seed_rng(seed: int, *scope: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed, *scope]))


def _triple_seed(seed: int, kind: str, width: int) -> int:
    code = 1 if kind == dealer.ARITH else 2
    return int(np.random.SeedSequence([seed, 0x7337, code, width]).generate_state(1)[0])


def build_stores(model: ModelSpec, relu_cfg: ReluConfig, batch: int, seed: int):
    """Both parties' stores dealt from the run seed, as the reference CLI does (cli.py:40-58)."""
    stores = (dealer.TripleStore(0), dealer.TripleStore(1))
    for (kind, width), count in sorted(triple_requirements(model, relu_cfg, batch).items()):
        gen = dealer.gen_arith_triples if kind == dealer.ARITH else dealer.gen_bool_triples
        b = gen(count, width, _triple_seed(seed, kind, width))
        for st in stores:
            st.add_batch(b)
    return stores


def run_local_forward(model: ModelSpec, relu_cfg: ReluConfig, x_f, seed: int, pair: bool = True,
                      layer_logs: bool = True):
    """Both parties in process -> (logits, (meter0, meter1), layer_logs, wall_ms) (cli.py:159-180).

    pair=True runs the parties time-sliced on this GPU (fused ReLU kernel);
    pair=False runs two party threads over a LocalEndpoint, as the reference does.
    layer_logs=False skips the per-layer meter log (empty logs), which lets the runner fuse a
    residual block's add into its last conv."""
    cfg = model.fixed_point
    enc = ring.encode_array(x_f, cfg)
    s0, s1 = sharing.share_arith(enc, cfg.ring_bits, _seed_rng(seed, _INPUT_STREAM))
    stores = build_stores(model, relu_cfg, x_f.shape[0], seed)
    ep0, ep1 = transport.local_pair()
    sessions = (ProtocolSession(ep0, stores[0], cfg), ProtocolSession(ep1, stores[1], cfg))
    logs: tuple = ([], [])
    lg = logs if layer_logs else (None, None)
    torch.cuda.synchronize()
    start = time.perf_counter()
    if pair:
        o0, o1 = model_forward_pair(sessions, s0, s1, model, relu_cfg, lg if layer_logs else None)
    else:
        o0, o1 = transport.run_parties(lambda: model_forward(sessions[0], s0, model, relu_cfg, lg[0]),
                                       lambda: model_forward(sessions[1], s1, model, relu_cfg, lg[1]),
                                       endpoints=(ep0, ep1))
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - start) * 1e3
    logits = ring.decode_array(sharing.reconstruct_arith(o0, o1), cfg)
    return logits, (ep0.meter, ep1.meter), logs, wall_ms


# ------------------------------------------------------------------ manifest I/O (nn.py:372-455)
def _layer_to_json(L) -> dict:
    out = {"kind": L.kind}
    for k, v in L.__dict__.items():
        if k == "kind":
            continue
        out[k] = [_layer_to_json(c) for c in v] if k in ("body", "shortcut") else v
    return out


def _layer_from_json(obj: dict):
    kinds = {"linear": Linear, "conv2d": Conv2d, "avgpool": AvgPool, "relu": Relu, "flatten": Flatten,
             "residual": Residual}
    try:
        cls = kinds[obj["kind"]]
        kw = {k: v for k, v in obj.items() if k != "kind"}
        if cls is Residual:
            kw = {k: tuple(_layer_from_json(c) for c in kw.get(k, ())) for k in ("body", "shortcut")}
        return cls(**kw)
    except (KeyError, TypeError) as exc:
        raise DataFormatError(f"bad layer entry {obj!r}: {exc}") from exc


def save_model(model: ModelSpec, out_dir) -> None:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    blobs = {}
    for name, arr in model.weights.items():
        fname = name.replace(".", "_") + ".bin"
        (out / fname).write_bytes(np.asarray(arr, dtype="<f4").tobytes())
        blobs[name] = fname
    manifest = {"fixed_point": model.fixed_point.to_json(), "input_shape": list(model.input_shape),
                "layers": [_layer_to_json(L) for L in model.layers], "blobs": blobs}
    (out / "manifest.json").write_text(json.dumps(manifest, indent=2))


def load_model(path) -> ModelSpec:
    p = Path(path)
    if p.is_dir():
        p = p / "manifest.json"
    try:
        man = json.loads(p.read_text())
        fxp = FixedPointConfig.from_json(man["fixed_point"])
        layers = [_layer_from_json(o) for o in man["layers"]]
        shapes = {}
        for L in _walk(layers):
            if isinstance(L, Linear):
                shapes[L.weight], shapes[L.bias] = (L.out_features, L.in_features), (L.out_features,)
            elif isinstance(L, Conv2d):
                shapes[L.weight] = (L.out_channels, L.in_channels, L.kh, L.kw)
                shapes[L.bias] = (L.out_channels,)
        weights = {}
        for name, fname in man["blobs"].items():
            raw = np.frombuffer((p.parent / fname).read_bytes(), dtype="<f4")
            weights[name] = raw.reshape(shapes.get(name, raw.shape)).astype(np.float32)
        return ModelSpec(fxp, tuple(man["input_shape"]), layers, weights)
    except (OSError, KeyError, TypeError, ValueError) as exc:
        raise DataFormatError(f"{p}: malformed model: {exc}") from exc
