"""Session stocking for the GPU tests -- the same seeds as the reference
tests/conftest.py:26-61 (bool triples seed 2*seed+1, arith 2*seed+2)."""

from __future__ import annotations

import hashlib
import queue

import numpy as np
import torch

from paper_2309_04875_b200 import dealer, protocol, transport
from paper_2309_04875_b200.protocol import ProtocolSession
from paper_2309_04875_b200.ring import FixedPointConfig


class RecordingEndpoint(transport.LocalEndpoint):
    """LocalEndpoint that keeps a SHA-256 of every payload it sends."""

    def __init__(self, *a):
        super().__init__(*a)
        self.sent_sha = []

    def exchange(self, payload):
        blob = payload.cpu().numpy().tobytes() if isinstance(payload, torch.Tensor) else bytes(payload)
        self.sent_sha.append(hashlib.sha256(blob).hexdigest())
        return super().exchange(payload)


def rec_pair():
    q01, q10 = queue.Queue(), queue.Queue()
    return RecordingEndpoint(0, q10, q01), RecordingEndpoint(1, q01, q10)


def make_sessions(bool_width=0, bool_count=0, arith_width=0, arith_count=0, seed=0, record=False):
    ep0, ep1 = rec_pair() if record else transport.local_pair()
    batches = []
    if bool_count:
        batches.append(dealer.gen_bool_triples(bool_count, bool_width, seed=seed * 2 + 1))
    if arith_count:
        batches.append(dealer.gen_arith_triples(arith_count, arith_width, seed=seed * 2 + 2))
    out = []
    for party, ep in ((0, ep0), (1, ep1)):
        st = dealer.TripleStore(party)
        for b in batches:
            st.add_batch(b)
        out.append(ProtocolSession(ep, st, FixedPointConfig()))
    return out[0], out[1], (ep0, ep1)


def stocked_sessions_for_relu(count, window_width, ring_width, seed=0, record=False):
    need = protocol.relu_triple_cost(count, window_width, ring_width)
    return make_sessions(window_width, need[(dealer.BOOL, window_width)], ring_width,
                         need[(dealer.ARITH, ring_width)], seed, record)


def sha(a) -> str:
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy().view(np.uint64)
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1), dtype="<u8")
                          .tobytes()).hexdigest()
