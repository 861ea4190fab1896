"""The reference-side binding, run as a ringmpc maintainer would run it.

integration/ringmpc_cuda_relu.py is the ctypes stub INTEGRATION.md documents: it imports `ringmpc`,
binds libhbrelu.so's `hb_relu` and passes an EXCHANGE callback that moves every round's payload
through the reference `Endpoint.exchange` under the round's meter tag (transport.py:129-133,
protocol.py:195-199).  The reference package itself is not on the GPU box, so `ringmpc` is
provided here with the reference's own shapes: a numpy TripleStore with `_streams[(kind, width)]`
of (a, b, c, cursor) (dealer.py:120-163), an Endpoint with `tag()` / `exchange()` / `meter`
(transport.py:80-142), and the reference error classes.  Party 0 runs the stub on the GPU; party 1
is the CPU restatement of the reference party (oracle/hb_oracle.py) on the other end of the link.
Bar: per-round payload SHA-256, meter trace and both output shares equal the reference's goldens.
"""

import hashlib
import queue
import sys
import threading
import types
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np
import pytest

import golden_cases as gc
from oracle import hb_oracle as O
from paper_2309_04875_b200 import errors as hb_errors
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor

pytestmark = pytest.mark.gpu


@dataclass
class _Stream:  # dealer.py:120-125
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    cursor: int = 0


class _RefStore:  # dealer.py:128-163 (the fields the stub reads)
    def __init__(self, party, batches):
        self.party = party
        self._streams = {}
        for kind, width, (a, b, c) in batches:
            self._streams[(kind, width)] = _Stream(a.copy(), b.copy(), c.copy())


class _RefEndpoint:  # transport.py:80-142: tag(), exchange() metered, payload SHAs kept
    def __init__(self, send_q, recv_q):
        self.send_q, self.recv_q = send_q, recv_q
        self.trace, self.sent_sha, self._tag = [], [], "Other"

    @contextmanager
    def tag(self, name):
        prev, self._tag = self._tag, name
        try:
            yield
        finally:
            self._tag = prev

    def exchange(self, payload: bytes) -> bytes:
        self.sent_sha.append(hashlib.sha256(payload).hexdigest())
        self.send_q.put(payload)
        got = self.recv_q.get(timeout=120)
        self.trace.append([self._tag, len(payload)])
        return got


def _install_ringmpc():
    """`ringmpc` with the reference's module / attribute names, for the stub's imports."""
    from paper_2309_04875_b200 import protocol as hb_protocol

    pkg = types.ModuleType("ringmpc")
    pkg.__path__ = []
    dealer = types.ModuleType("ringmpc.dealer")
    dealer.BOOL, dealer.ARITH = "bool", "arith"  # dealer.py:30-31
    protocol = types.ModuleType("ringmpc.protocol")
    protocol.relu_triple_cost = hb_protocol.relu_triple_cost  # protocol.py:202-213
    errors = types.ModuleType("ringmpc.errors")
    for name in ("ConfigError", "RingMpcError", "TransportError", "TripleExhaustedError"):
        setattr(errors, name, getattr(hb_errors, name))
    pkg.dealer, pkg.protocol, pkg.errors = dealer, protocol, errors
    sys.modules.update({"ringmpc": pkg, "ringmpc.dealer": dealer, "ringmpc.protocol": protocol,
                        "ringmpc.errors": errors})


@pytest.mark.parametrize("name", ["base4096_22_14", "base1001_22_16"])
def test_reference_binding_party_vs_reference_party(golden, name):
    _install_ringmpc()
    import importlib

    stub = importlib.import_module("integration.ringmpc_cuda_relu")
    meta = golden[0]
    case = next(c for c in gc.RELU_CASES if c["name"] == name)
    g = meta[name]
    x0, x1 = gc.make_inputs(case)
    k, m, n = case["k"], case["m"], x0.size
    w = k - m
    curs = O.stocked_cursors(n, w, 64, case["seed"])
    # party 0's reference TripleStore holds exactly the streams the oracle cursor of party 0 holds
    store0 = _RefStore(0, [(kind, width, arrs) for (kind, width), arrs in curs[0].streams.items()])

    class _Sess:
        party, triples = 0, store0

    q01, q10 = queue.Queue(), queue.Queue()
    ep0 = _RefEndpoint(q01, q10)
    _Sess.endpoint = ep0
    wire1 = O.Wire(1, q01, q10, keep_payloads=True)
    out = {}

    def party1():
        out[1] = O.p_relu(1, wire1, curs[1], x1, 64, k, m)

    th = threading.Thread(target=party1)
    th.start()
    y0 = stub.relu(_Sess, ArithShareTensor(0, 64, x0), BitWindow(k, m))
    th.join(120)
    assert O.digest(np.asarray(y0.data, dtype=np.uint64)) == g["y0_sha"]
    assert O.digest(out[1]) == g["y1_sha"]
    assert ep0.sent_sha == g["payload0_sha"]
    assert ep0.trace == g["trace0"]
    assert [hashlib.sha256(p).hexdigest() for p in wire1.sent] == g["payload1_sha"]
    # the stub advanced the reference store's cursors by exactly one ReLU's triples
    cost = O.triple_need(n, w, 64)
    assert store0._streams[("bool", w)].cursor == cost[("bool", w)]
    assert store0._streams[("arith", 64)].cursor == cost[("arith", 64)]
