"""Two-party kernels of the reduced-ring ReLU: Beaver MUL/AND, Kogge-Stone A2B,
single-bit B2A, windowed DReLU and ReLU -- every step on the GPU.

Same functions, arguments, rounds, tags and triple consumption as the
reference (ringmpc protocol.py:45-213).  Three execution paths:

* ``relu`` / ``drelu`` (one party, any endpoint): the staged CUDA driver,
  ``hb_relu_round`` once per round with the endpoint's exchange in between.
  Openings cross the endpoint in the exact reference wire layout.
* ``relu_pair`` (both parties on this GPU): ``hb_relu_pair`` runs the whole
  protocol for both parties in one launch, the wire held in shared memory.
* ``beaver_*`` / ``circuit_add`` / ``a2b`` / ``b2a_bit``: stage kernels, so
  each protocol stage is usable and testable on its own.

Inputs may be host (numpy uint64) or device (CUDA int64) shares; results come
back in the caller's representation.
"""

from __future__ import annotations

import ctypes
import functools

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .dealer import ARITH, BOOL, TripleStore
from .errors import ConfigError
from .ring import BitWindow, FixedPointConfig
from .sharing import ArithShareTensor, BinShareTensor
from .transport import TAG_B2A, TAG_CIRCUIT, TAG_MULT, TAG_OTHER, Endpoint, packed_nbytes


@dataclass
class ProtocolSession:
    """One party's context: link, correlated randomness, encoding (protocol.py:45-59)."""

    endpoint: Endpoint
    triples: TripleStore
    fxp: FixedPointConfig = field(default_factory=FixedPointConfig)

    @property
    def party(self) -> int:
        return self.endpoint.party

    def __post_init__(self) -> None:
        if self.triples.party != self.endpoint.party:
            raise ConfigError("triple store and endpoint belong to different parties")


def prefix_levels(width: int) -> int:
    """Kogge-Stone depth max(1, ceil(log2 w)) (protocol.py:108-110)."""
    return max(1, math.ceil(math.log2(width)))


def relu_triple_cost(count: int, window_width: int, ring_width: int) -> dict:
    """Triples one ReLU consumes (protocol.py:202-213)."""
    return {(BOOL, window_width): count * (1 + 2 * prefix_levels(window_width)), (ARITH, ring_width): 2 * count}


# ------------------------------------------------------------------ helpers
def _flat(data) -> torch.Tensor:
    return _dev.to_device(data).reshape(-1)


def _wrap(cls, party, width, flat: torch.Tensor, like, shape):
    out = flat.reshape(shape)
    return cls(party, width, _dev.to_host(out, like))


def _stream() -> int:
    return _dev.stream_handle()


def _ew(op: str, party: int, w: int, n: int, a, b=None, p: int = 0, out_len: int | None = None, two=False):
    out = torch.empty(out_len if out_len is not None else n, dtype=torch.int64, device=_dev.device())
    out2 = torch.empty(n, dtype=torch.int64, device=_dev.device()) if two else None
    _lib.call("hb_ewise", _lib.EW[op], party, w, n, p, _dev.ptr(a), _dev.ptr(b), out.data_ptr(), _dev.ptr(out2),
              _stream())
    return (out, out2) if two else out


def _beaver(session: ProtocolSession, kind: int, w: int, xd: torch.Tensor, yd: torch.Tensor) -> torch.Tensor:
    """One Beaver opening on flat device operands; returns z (flat device)."""
    n = xd.numel()
    view = session.triples.draw(ARITH if kind else BOOL, w, n)
    tmp = torch.empty(2 * n, dtype=torch.int64, device=xd.device)
    payload = torch.empty(packed_nbytes(2 * n, w) // 8, dtype=torch.int64, device=xd.device)
    _lib.call("hb_beaver_open", kind, w, n, xd.data_ptr(), yd.data_ptr(), view.abi(), tmp.data_ptr(),
              payload.data_ptr(), _stream())
    peer = session.endpoint.exchange(payload)
    z = torch.empty(n, dtype=torch.int64, device=xd.device)
    _lib.call("hb_beaver_close", kind, session.party, w, n, xd.data_ptr(), yd.data_ptr(), view.abi(),
              peer.data_ptr(), z.data_ptr(), _stream())
    return z


def _check_pair(x, y, what):
    if x.width != y.width or x.shape != y.shape:
        raise ConfigError(f"{what} operands must share width and shape")


# ------------------------------------------------------------------ stage operations
def beaver_mul(session: ProtocolSession, x: ArithShareTensor, y: ArithShareTensor) -> ArithShareTensor:
    """z = c + E b + F a (+ E F on party 0), one round (protocol.py:75-89)."""
    _check_pair(x, y, "beaver_mul")
    z = _beaver(session, 1, x.width, _flat(x.data), _flat(y.data))
    return _wrap(ArithShareTensor, x.party, x.width, z, x.data, x.shape)


def beaver_and(session: ProtocolSession, x: BinShareTensor, y: BinShareTensor) -> BinShareTensor:
    """Bitwise AND of XOR-shared words, one round (protocol.py:92-105)."""
    _check_pair(x, y, "beaver_and")
    z = _beaver(session, 0, x.width, _flat(x.data), _flat(y.data))
    return _wrap(BinShareTensor, x.party, x.width, z, x.data, x.shape)


def _adder(session: ProtocolSession, w: int, ud: torch.Tensor, vd: torch.Tensor) -> torch.Tensor:
    n = ud.numel()
    party = session.party
    p0 = _ew("XOR", party, w, n, ud, vd)
    with session.endpoint.tag(TAG_OTHER):
        g = _beaver(session, 0, w, ud, vd)
    p = p0
    with session.endpoint.tag(TAG_CIRCUIT):
        for level in range(prefix_levels(w)):
            lhs = _ew("STACK2", party, w, n, p, out_len=2 * n)
            rhs = _ew("KS_RHS", party, w, n, g, p, p=level, out_len=2 * n)
            both = _beaver(session, 0, w, lhs, rhs)
            g, p = _ew("KS_UPDATE", party, w, n, g, both, two=True)
    return _ew("KS_FINISH", party, w, n, p0, g)


def circuit_add(session: ProtocolSession, a: BinShareTensor, b: BinShareTensor) -> BinShareTensor:
    """Kogge-Stone adder on XOR shares: 1 + ceil(log2 w) rounds (protocol.py:113-143)."""
    if a.width != b.width or a.shape != b.shape:
        raise ConfigError("circuit_add operands must share width and shape")
    out = _adder(session, a.width, _flat(a.data), _flat(b.data))
    return _wrap(BinShareTensor, a.party, a.width, out, a.data, a.shape)


def a2b(session: ProtocolSession, x: ArithShareTensor) -> BinShareTensor:
    """Arithmetic-to-binary via the adder on (own share, zeros) (protocol.py:146-157)."""
    xd = _flat(x.data)
    n, w = xd.numel(), x.width
    u = _ew("OWNER", x.party, w, n, xd, p=0)
    v = _ew("OWNER", x.party, w, n, xd, p=1)
    out = _adder(session, w, u, v)
    return _wrap(BinShareTensor, x.party, w, out, x.data, x.shape)


def b2a_bit(session: ProtocolSession, b: BinShareTensor, out_width: int) -> ArithShareTensor:
    """Lift an XOR-shared bit to Z/2^N: b0 + b1 - 2 b0 b1 (protocol.py:160-176)."""
    bd = _flat(b.data)
    flag = _lib.ctypes.c_int(0)
    _lib.call("hb_any_above_one", bd.data_ptr(), bd.numel(), _lib.ctypes.byref(flag), _stream())
    if flag.value:
        raise ConfigError("b2a_bit expects 0/1 words")
    n = bd.numel()
    with session.endpoint.tag(TAG_B2A):
        u = _ew("OWNER", b.party, out_width, n, bd, p=0)
        v = _ew("OWNER", b.party, out_width, n, bd, p=1)
        t = _beaver(session, 1, out_width, u, v)
        lifted = _ew("B2A_LIFT", b.party, out_width, n, bd, t)
    return _wrap(ArithShareTensor, b.party, out_width, lifted, b.data, b.shape)


# ------------------------------------------------------------------ fused ReLU paths
def _relu_staged(session: ProtocolSession, x: ArithShareTensor, window: BitWindow, drelu_only: bool):
    window.check_fits(x.width)
    N, k, m, w = x.width, window.k, window.m, window.width
    xd = _flat(x.data)
    n = xd.numel()
    levels = prefix_levels(w)
    need_a = n if drelu_only else 2 * n
    session.triples.check({(BOOL, w): n * (1 + 2 * levels), (ARITH, N): need_a})
    bv = session.triples.draw(BOOL, w, n * (1 + 2 * levels))
    av = session.triples.draw(ARITH, N, need_a)
    lib = _lib.load()
    y = torch.empty(n, dtype=torch.int64, device=xd.device)
    ws = torch.empty(max(lib.hb_relu_workspace_bytes(k, m, n) // 8, 1), dtype=torch.int64, device=xd.device)
    rounds = lib.hb_relu_rounds(k, m, int(drelu_only))
    peer = None
    for r in range(rounds + 1):
        own = None
        if r < rounds:
            own = torch.empty(lib.hb_relu_round_bytes(N, k, m, n, r) // 8, dtype=torch.int64, device=xd.device)
        _lib.check(lib.hb_relu_round(session.party, N, k, m, n, r, xd.data_ptr(), y.data_ptr(), bv.abi(), av.abi(),
                                     ws.data_ptr(), _dev.ptr(peer), _dev.ptr(own), int(drelu_only), _stream()))
        if r < rounds:
            with session.endpoint.tag(_lib.TAG_BY_CODE[lib.hb_relu_round_tag(k, m, r)]):
                peer = session.endpoint.exchange(own)
    return _wrap(ArithShareTensor, x.party, N, y, x.data, x.shape)


def drelu(session: ProtocolSession, x: ArithShareTensor, window: BitWindow) -> ArithShareTensor:
    """Shared indicator of x >= 0 on the window [m, k) (protocol.py:179-192)."""
    if session.endpoint.p2p is not None and x.width == 64:
        return relu_p2p(session, x, window, session.endpoint.p2p, drelu_only=True)
    return _relu_staged(session, x, window, drelu_only=True)


def relu(session: ProtocolSession, x: ArithShareTensor, window: BitWindow) -> ArithShareTensor:
    """x * DReLU(x[k:m]), the multiply metered as Mult (protocol.py:195-199)."""
    if session.endpoint.p2p is not None and x.width == 64:
        return relu_p2p(session, x, window, session.endpoint.p2p, drelu_only=False)
    return _relu_staged(session, x, window, drelu_only=False)


def relu_p2p_pair(sessions, x0: ArithShareTensor, x1: ArithShareTensor, window: BitWindow, links,
                  drelu_only: bool = False, sys_scope: bool = False):
    """Both parties' NVLink party kernels in one launch on this GPU (hb_relu_p2p_pair), the openings
    going through each other's receive buffers (`links` = transport.local_p2p_pair()) exactly as
    relu_p2p does across two GPUs.  Same shares / triples / meter as relu_pair and relu.
    sys_scope: run the system-scope flag protocol of the cross-GPU kernel (measurement) instead of
    the gpu scope both parties share on one device."""
    s0, s1 = sessions
    l0, l1 = links
    if (s0.party, s1.party) != (0, 1) or (x0.party, x1.party) != (0, 1):
        raise ConfigError("relu_p2p_pair expects (party 0, party 1) sessions and shares")
    if x0.width != x1.width or x0.shape != x1.shape:
        raise ConfigError("relu_p2p_pair shares must agree in width and shape")
    if x0.width != 64:
        raise ConfigError("the NVLink party kernel runs on Z/2^64 shares (other rings: the staged path)")
    window.check_fits(x0.width)
    N, k, m, w = x0.width, window.k, window.m, window.width
    a0, a1 = _flat(x0.data), _flat(x1.data)
    n = a0.numel()
    levels = prefix_levels(w)
    need = {(BOOL, w): n * (1 + 2 * levels), (ARITH, N): (1 if drelu_only else 2) * n}
    s0.triples.check(need)
    s1.triples.check(need)
    views = [(s.triples.draw(BOOL, w, need[(BOOL, w)]), s.triples.draw(ARITH, N, need[(ARITH, N)])) for s in sessions]
    trace = _relu_trace(n, k, m, N, bool(drelu_only))
    for s in sessions:
        s.endpoint.meter.record_rounds(trace)
    lib = _lib.load()
    ntiles = ctypes.c_int64(0)
    nbytes = lib.hb_relu_p2p_bytes(k, m, n, int(drelu_only), ctypes.byref(ntiles))
    l0.check()
    l0.ensure(nbytes, ntiles.value)
    y0 = torch.empty(n, dtype=torch.int64, device=a0.device)
    y1 = torch.empty(n, dtype=torch.int64, device=a0.device)
    wc = l0.wire_counter
    cur = torch.cuda.current_stream()  # once: the query costs more host time than a small layer's kernel
    # flag sequence and receive-region parity come from the links' device state (graph-capturable)
    _lib.check(lib.hb_relu_p2p_pair_dev(N, k, m, n, a0.data_ptr(), a1.data_ptr(), y0.data_ptr(), y1.data_ptr(),
                                        views[0][0].abi(), views[1][0].abi(), views[0][1].abi(), views[1][1].abi(),
                                        l0.recv, l1.recv, l0.flags, l1.flags, l0.state.data_ptr(),
                                        l1.state.data_ptr(), l0.cap_bytes, l0.max_ctas, l1.max_ctas, int(sys_scope),
                                        l0.timeout_s, l0.err.data_ptr(), int(drelu_only),
                                        None if wc is None else wc.data_ptr(), cur.cuda_stream))
    l0.after_launch(cur)
    return (_wrap(ArithShareTensor, 0, N, y0, x0.data, x0.shape), _wrap(ArithShareTensor, 1, N, y1, x1.data, x1.shape))


def relu_p2p(session: ProtocolSession, x: ArithShareTensor, window: BitWindow, link, drelu_only: bool = False,
             stream=None, out: torch.Tensor | None = None) -> ArithShareTensor:
    """One party's ReLU / DReLU in one launch of the NVLink party kernel (hb_relu_p2p): every
    round's opening goes tile by tile into the peer's receive buffer (`link`, a transport.PeerLink)
    instead of a per-round Endpoint.exchange.  Same output shares, triple consumption and meter
    trace as relu() over any endpoint; both parties must call it for the same layers in order.
    `out` (int64, n elements) avoids an allocation between two parties' launches on one device."""
    window.check_fits(x.width)
    if x.width != 64:
        raise ConfigError("the NVLink party kernel runs on Z/2^64 shares (other rings: the staged path)")
    N, k, m, w = x.width, window.k, window.m, window.width
    xd = _flat(x.data)
    n = xd.numel()
    levels = prefix_levels(w)
    need_a = n if drelu_only else 2 * n
    session.triples.check({(BOOL, w): n * (1 + 2 * levels), (ARITH, N): need_a})
    bv = session.triples.draw(BOOL, w, n * (1 + 2 * levels))
    av = session.triples.draw(ARITH, N, need_a)
    lib = _lib.load()
    ntiles = ctypes.c_int64(0)
    nbytes = lib.hb_relu_p2p_bytes(k, m, n, int(drelu_only), ctypes.byref(ntiles))
    link.check()
    link.ensure(nbytes, ntiles.value)
    session.endpoint.meter.record_rounds(_relu_trace(n, k, m, N, bool(drelu_only)))
    y = torch.empty(n, dtype=torch.int64, device=xd.device) if out is None else out.reshape(-1)
    if y.numel() != n or y.dtype != torch.int64 or not y.is_cuda:
        raise ConfigError("relu_p2p out must be a CUDA int64 tensor of the input's size")
    launch_stream = torch.cuda.current_stream() if stream is None else stream
    st = launch_stream.cuda_stream
    wc = link.wire_counter
    # flag sequence and receive-region parity from the link's device state (graph-capturable)
    _lib.check(lib.hb_relu_p2p_dev(session.party, N, k, m, n, xd.data_ptr(), y.data_ptr(), bv.abi(), av.abi(),
                                   link.recv, link.flags, link.peer_recv, link.peer_flags, link.state.data_ptr(),
                                   link.cap_bytes, link.grid, link.timeout_s, link.err.data_ptr(), int(drelu_only),
                                   None if wc is None else wc.data_ptr(), st))
    link.after_launch(launch_stream)
    return _wrap(ArithShareTensor, x.party, N, y, x.data, x.shape)


def relu_trace(n: int, window: BitWindow, ring_bits: int, drelu_only: bool = False) -> list:
    """(tag, bytes) of every round, as the reference meter records them."""
    return list(_relu_trace(n, window.k, window.m, ring_bits, bool(drelu_only)))


@functools.lru_cache(maxsize=4096)
def _relu_trace(n: int, k: int, m: int, ring_bits: int, drelu_only: bool) -> tuple:
    lib = _lib.load()
    return tuple((_lib.TAG_BY_CODE[lib.hb_relu_round_tag(k, m, r)], int(lib.hb_relu_round_bytes(ring_bits, k, m, n, r)))
                 for r in range(lib.hb_relu_rounds(k, m, int(drelu_only))))


def relu_pair(sessions, x0: ArithShareTensor, x1: ArithShareTensor, window: BitWindow,
              drelu_only: bool = False):
    """Both parties' ReLU (or DReLU) on this GPU in one fused launch.

    Equivalent to ``run_parties(relu(s0, x0, w), relu(s1, x1, w))`` -- same
    output shares, same triple consumption, same meter trace -- with the two
    parties time-sliced inside one kernel and the openings exchanged through
    shared memory (hb_relu_pair)."""
    s0, s1 = sessions
    if (s0.party, s1.party) != (0, 1) or (x0.party, x1.party) != (0, 1):
        raise ConfigError("relu_pair expects (party 0, party 1) sessions and shares")
    if x0.width != x1.width or x0.shape != x1.shape:
        raise ConfigError("relu_pair shares must agree in width and shape")
    window.check_fits(x0.width)
    N, w = x0.width, window.width
    host_pipeline = all(isinstance(x.data, torch.Tensor) and not x.data.is_cuda and x.data.is_pinned()
                        for x in (x0, x1)) and x0.numel > (1 << 22)
    if host_pipeline:
        a0 = a1 = None
        n = x0.numel
    else:
        a0, a1 = _flat(x0.data), _flat(x1.data)
        n = a0.numel()
    levels = prefix_levels(w)
    need = {(BOOL, w): n * (1 + 2 * levels), (ARITH, N): (1 if drelu_only else 2) * n}
    s0.triples.check(need)
    s1.triples.check(need)
    views = [(s.triples.draw(BOOL, w, need[(BOOL, w)]), s.triples.draw(ARITH, N, need[(ARITH, N)])) for s in (s0, s1)]
    trace = _relu_trace(n, window.k, window.m, N, bool(drelu_only))
    for s in (s0, s1):
        s.endpoint.meter.record_rounds(trace)
    if host_pipeline:
        return _relu_pair_pinned(N, window, n, x0, x1, views, drelu_only)
    y0 = torch.empty(n, dtype=torch.int64, device=a0.device)
    y1 = torch.empty(n, dtype=torch.int64, device=a0.device)
    _lib.call("hb_relu_pair", N, window.k, window.m, n, a0.data_ptr(), a1.data_ptr(), y0.data_ptr(), y1.data_ptr(),
              views[0][0].abi(), views[1][0].abi(), views[0][1].abi(), views[1][1].abi(), int(drelu_only), _stream())
    return (_wrap(ArithShareTensor, 0, N, y0, x0.data, x0.shape), _wrap(ArithShareTensor, 1, N, y1, x1.data, x1.shape))


_PIPE_CHUNK = int(os.environ.get("HB_PIPE_CHUNK", str(1 << 21)))  # elements per pinned-pipeline chunk (2^19..2^22 measured: 2^21 best)


def _relu_pair_pinned(N, window, n, x0, x1, views, drelu_only, chunk=None):
    """Pinned host shares in/out: hb_relu_pair_host pipelines host-to-device copies, the fused
    kernel on element ranges and device-to-host copies over three native streams joined per chunk
    by events (chunks ramped at both ends), so both PCIe directions and the kernel overlap.  Same
    kernel, same triples, same shares as the one-shot path."""
    dev = _dev.device()
    h0, h1 = x0.data.reshape(-1), x1.data.reshape(-1)
    o = torch.empty((2, n), dtype=torch.int64, pin_memory=True)  # one allocation: one two-row D2H per chunk
    o0, o1 = o[0], o[1]
    scratch = torch.empty(4 * n, dtype=torch.int64, device=dev)
    _lib.call("hb_relu_pair_host", N, window.k, window.m, n, h0.data_ptr(), h1.data_ptr(), o0.data_ptr(),
              o1.data_ptr(), views[0][0].abi(), views[1][0].abi(), views[0][1].abi(), views[1][1].abi(),
              int(drelu_only), int(chunk or _PIPE_CHUNK), scratch.data_ptr(), _stream())
    return (ArithShareTensor(0, N, o0.reshape(x0.shape)), ArithShareTensor(1, N, o1.reshape(x1.shape)))
