#!/usr/bin/env python
"""Does a ring conv (tensor / L2-ingress bound) overlap with a pair ReLU (HBM bound) when they run on
two streams?  ResNet18 layer1 shapes at batch 256: both parties' 64->64 3x3 conv, and the pair ReLU
over 256 x 64 x 32 x 32 = 2^24 elements.  Prints alone / concurrent times (CUDA events)."""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04875_b200 import dealer, nn, protocol, transport  # noqa: E402
from paper_2309_04875_b200.protocol import ProtocolSession  # noqa: E402
from paper_2309_04875_b200.ring import BitWindow, FixedPointConfig  # noqa: E402
from paper_2309_04875_b200.sharing import ArithShareTensor  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    b = int(os.environ.get("B", "256"))
    cfg = FixedPointConfig(64, 16)
    rng = np.random.default_rng(0)
    wt = rng.normal(0, 0.06, (64, 64, 3, 3)).astype(np.float32)
    lw = nn._weight(wt, np.zeros(64, np.float32), cfg)
    geom = (3, 3, 1, 1)
    xs = [torch.randint(-2**62, 2**62, (b, 64, 32, 32), dtype=torch.int64, device=dev) for _ in range(2)]
    n = b * 64 * 32 * 32
    win = BitWindow(22, 14)
    eps = transport.local_pair()
    stores = (dealer.TripleStore(0), dealer.TripleStore(1))
    for kind, width, cnt in ((dealer.BOOL, 8, n * 7 * 12), (dealer.ARITH, 64, 2 * n * 12)):
        dealer.stock_on_device(stores, (0, 1), kind, width, cnt, seed=3 + width)
    sess = (ProtocolSession(eps[0], stores[0]), ProtocolSession(eps[1], stores[1]))
    r0 = ArithShareTensor(0, 64, xs[0].reshape(-1))
    r1 = ArithShareTensor(1, 64, xs[1].reshape(-1))
    s_conv, s_relu = torch.cuda.Stream(), torch.cuda.Stream()

    def conv():
        for p in (0, 1):
            nn._PLANES.clear()
            nn._gemm_tc(xs[p], geom, lw, p, 16)

    def relu():
        protocol.relu_pair(sess, r0, r1, win)

    def timed(fn_list, reps=5):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record(torch.cuda.current_stream())
        evs = []
        for _ in range(reps):
            for s, fn in fn_list:
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    fn()
                e = torch.cuda.Event()
                e.record(s)
                evs.append(e)
        for e in evs:
            torch.cuda.current_stream().wait_event(e)
        z.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        return a.elapsed_time(z) / reps

    for _ in range(2):
        conv(), relu()
        for st in stores:
            st.rewind(dealer.BOOL, 8)
            st.rewind(dealer.ARITH, 64)
    out = {}
    out["conv_ms"] = timed([(s_conv, conv)])
    out["relu_ms"] = timed([(s_relu, relu)])
    for st in stores:
        st.rewind(dealer.BOOL, 8)
        st.rewind(dealer.ARITH, 64)
    out["both_ms"] = timed([(s_conv, conv), (s_relu, relu)])
    out["serial_sum_ms"] = out["conv_ms"] + out["relu_ms"]
    out["batch"] = b
    print(json.dumps(out))


if __name__ == "__main__":
    main()
