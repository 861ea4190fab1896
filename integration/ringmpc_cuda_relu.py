"""ringmpc/cuda_relu.py -- the ctypes stub a ringmpc maintainer adds to run ONE party's ReLU on the GPU.

Drop-in for `ringmpc.protocol.relu` (protocol.py:195-199) over the reference's own `Endpoint`
(LocalEndpoint / TcpEndpoint, transport.py:119-268) and its numpy `TripleStore`
(dealer.py:120-163): it binds `libhbrelu.so`'s `hb_relu` (include/hb_relu.h) and hands the library
an EXCHANGE callback that moves each round's payload through `Endpoint.exchange` under the
round's meter tag -- so a GPU party interoperates byte for byte with a CPU party, and the meter
records exactly what the reference records.

This file is the stub INTEGRATION.md documents; tests/test_gpu_integration.py imports it and runs
it unmodified against the CPU restatement of the reference party (oracle/hb_oracle.py).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
from cuda.bindings import runtime as cudart

from ringmpc import dealer, protocol
from ringmpc.errors import ConfigError, RingMpcError, TransportError, TripleExhaustedError

LIB = os.environ.get("HB_RELU_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                "paper_2309_04875_b200", "lib", "libhbrelu.so"))
lib = ctypes.CDLL(LIB)


class hb_triples_t(ctypes.Structure):
    _fields_ = [("a", ctypes.c_void_p), ("b", ctypes.c_void_p), ("c", ctypes.c_void_p),
                ("cursor", ctypes.c_int64), ("capacity", ctypes.c_int64), ("width", ctypes.c_int32)]


EXCHANGE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
lib.hb_relu.restype = ctypes.c_int
lib.hb_relu.argtypes = [ctypes.c_int] * 4 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                        hb_triples_t, hb_triples_t, ctypes.c_void_p, ctypes.c_int, EXCHANGE,
                        ctypes.c_void_p, ctypes.c_void_p]
lib.hb_pack.restype = ctypes.c_int
lib.hb_pack.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
lib.hb_relu_callback_workspace_bytes.restype = ctypes.c_size_t
lib.hb_relu_callback_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
lib.hb_last_error.restype = ctypes.c_char_p
TAG_NAMES = {0: "Circuit", 1: "Mult", 2: "B2A", 3: "Other"}
ERRORS = {2: ConfigError, 3: TransportError, 5: TripleExhaustedError}


def _d2h(dev_ptr: int, nbytes: int) -> bytes:
    """Device payload -> host bytes (hb_relu synchronises its stream before each callback)."""
    host = np.empty(nbytes, dtype=np.uint8)
    if nbytes:
        (err,) = cudart.cudaMemcpy(host.ctypes.data, dev_ptr, nbytes, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        if err != cudart.cudaError_t.cudaSuccess:
            raise TransportError(f"cudaMemcpy D2H: {err}")
    return host.tobytes()


def _h2d(dev_ptr: int, blob: bytes) -> None:
    host = np.frombuffer(blob, dtype=np.uint8)
    if len(blob):
        (err,) = cudart.cudaMemcpy(dev_ptr, host.ctypes.data, len(blob), cudart.cudaMemcpyKind.cudaMemcpyHostToDevice)
        if err != cudart.cudaError_t.cudaSuccess:
            raise TransportError(f"cudaMemcpy H2D: {err}")


def _device_stream(store, kind, width):
    """One (kind, width) TripleStore stream in HBM; bool streams packed at `width` bits (the wire layout)."""
    s = store._streams[(kind, width)]
    arrs = [torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda() for a in (s.a, s.b, s.c)]
    if kind == dealer.BOOL:
        packed = []
        for t in arrs:
            out = torch.zeros(max((t.numel() * width + 63) // 64, 1), dtype=torch.int64, device="cuda")
            rc = lib.hb_pack(t.data_ptr(), t.numel(), width, out.data_ptr(), None)
            if rc:
                raise ERRORS.get(rc, RingMpcError)(lib.hb_last_error().decode())
            packed.append(out)
        arrs = packed
    torch.cuda.synchronize()
    return arrs, s


def relu(session, x, window):
    """protocol.relu (protocol.py:195-199) for this session's party on the GPU: same output share,
    same rounds / tags / payload bytes on session.endpoint, same triple consumption."""
    window.check_fits(x.width)
    n, N, w = x.numel, x.width, window.width
    need = protocol.relu_triple_cost(n, w, N)
    (ba, bs), (aa, as_) = (_device_stream(session.triples, dealer.BOOL, w),
                           _device_stream(session.triples, dealer.ARITH, N))
    bt = hb_triples_t(ba[0].data_ptr(), ba[1].data_ptr(), ba[2].data_ptr(), bs.cursor, bs.a.size, w)
    at = hb_triples_t(aa[0].data_ptr(), aa[1].data_ptr(), aa[2].data_ptr(), as_.cursor, as_.a.size, N)
    xd = torch.from_numpy(np.ascontiguousarray(x.data).reshape(-1).view(np.int64)).cuda()
    yd = torch.empty_like(xd)
    ws = torch.empty(lib.hb_relu_callback_workspace_bytes(N, window.k, window.m, n) // 8 + 1,
                     dtype=torch.int64, device="cuda")
    failure = []

    @EXCHANGE
    def exchange(user, tag, send, recv, nbytes, stream):
        try:
            mine = _d2h(send, nbytes)                                  # this round's opening
            with session.endpoint.tag(TAG_NAMES[tag]):
                theirs = session.endpoint.exchange(mine)               # reference transport, metered
            if len(theirs) != nbytes:
                failure.append(TransportError(f"peer sent {len(theirs)} bytes, expected {nbytes}"))
                return 1
            _h2d(recv, theirs)                                         # the peer's opening
            return 0
        except Exception as exc:  # noqa: BLE001 -- surfaced after hb_relu returns
            failure.append(exc)
            return 1

    torch.cuda.synchronize()
    rc = lib.hb_relu(x.party, N, window.k, window.m, n, xd.data_ptr(), yd.data_ptr(), bt, at,
                     ws.data_ptr(), 0, exchange, None, None)
    if failure:
        raise failure[0]
    if rc:
        raise ERRORS.get(rc, RingMpcError)(lib.hb_last_error().decode())
    bs.cursor += need[(dealer.BOOL, w)]
    as_.cursor += need[(dealer.ARITH, N)]
    return type(x)(x.party, N, yd.cpu().numpy().view(np.uint64).reshape(np.shape(x.data)))
