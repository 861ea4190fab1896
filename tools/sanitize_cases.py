#!/usr/bin/env python
"""Small workloads for compute-sanitizer (racecheck / memcheck / synccheck) on the library's kernels.

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py pair
  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py p2p
  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py conv

Each case runs a few launches at sizes the sanitizer finishes in seconds (partial last tiles
included) and checks the result against the CPU oracle, so a run that 'passes' also computed the
right shares.  Exit code 0 = results correct (the sanitizer's own summary is the race / memory
verdict).
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import golden_cases as gc  # noqa: E402
from hb_helpers import stocked_sessions_for_relu  # noqa: E402
from oracle import hb_oracle as O  # noqa: E402
from paper_2309_04875_b200 import protocol, transport  # noqa: E402
from paper_2309_04875_b200.ring import BitWindow  # noqa: E402
from paper_2309_04875_b200.sharing import ArithShareTensor  # noqa: E402


def _relu_case(n, k, m, seed, run):
    x0, x1 = gc.baseline_inputs(n, seed=seed)
    curs = O.stocked_cursors(n, k - m, 64, seed=seed)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=seed)
    t0 = ArithShareTensor(0, 64, torch.from_numpy(x0.view(np.int64)).cuda())
    t1 = ArithShareTensor(1, 64, torch.from_numpy(x1.view(np.int64)).cuda())
    r0, r1 = run((s0, s1), t0, t1, BitWindow(k, m))
    torch.cuda.synchronize()
    ok = (np.array_equal(r0.data.cpu().numpy().view(np.uint64), y0o)
          and np.array_equal(r1.data.cpu().numpy().view(np.uint64), y1o))
    print(f"  n={n} window=({k},{m}): {'bit-exact' if ok else 'MISMATCH'}")
    return ok


def case_pair():
    """k_relu_pair: the shared-memory double-buffered wire (racecheck target)."""
    return all(_relu_case(n, k, m, 11, protocol.relu_pair)
               for n, (k, m) in ((4096 + 37, (22, 14)), (3000, (64, 0)), (2500, (22, 16)), (5000, (29, 7))))


def case_p2p():
    """k_relu_p2p (both parties in one launch): remote stores, flags, receive regions."""
    links = transport.local_p2p_pair()
    links[0].timeout_s = 60.0

    def run(sessions, t0, t1, win):
        out = protocol.relu_p2p_pair(sessions, t0, t1, win, links)
        links[0].check(sync=True)
        return out

    # several layers on the same links: buffer growth and launch-to-launch reuse of the regions
    return all(_relu_case(n, k, m, 13 + i, run)
               for i, (n, (k, m)) in enumerate(((20000 + 5, (22, 14)), (9000, (64, 0)), (30000, (27, 22)),
                                                 (7000, (22, 16)))))


def case_conv():
    """k_conv_tma (+ limb planes): TMA / mbarrier pipeline, TMEM epilogue, fused residual."""
    from oracle import hb_oracle_nn as ON
    from paper_2309_04875_b200 import nn
    from paper_2309_04875_b200.ring import FixedPointConfig

    class _Sess:
        fxp = FixedPointConfig(64, 16)

    rng = np.random.default_rng(3)
    ok = True
    for (b, c, h, oc, kk, stride, pad) in ((2, 64, 8, 64, 3, 1, 1), (2, 128, 8, 256, 3, 2, 1), (2, 64, 8, 128, 1, 2, 0),
                                           (2, 3, 8, 64, 3, 1, 1)):
        x = np.frombuffer(rng.bytes(8 * b * c * h * h), dtype="<u8").copy().reshape(b, c, h, h)
        wt = rng.normal(0, 0.05, size=(oc, c, kk, kk))
        bias = rng.normal(0, 0.05, size=oc)
        layer = nn.Conv2d(c, oc, kk, kk, stride, pad, weight="w", bias="b")
        for party in (0, 1):
            got = nn.conv2d_forward(_Sess, ArithShareTensor(party, 64, x), layer, wt, bias)
            want = ON.conv2d(x, party, c, oc, kk, kk, stride, pad, wt, bias)
            this = np.array_equal(np.asarray(got.data).view(np.uint64), want)
            print(f"  conv b={b} c={c} h={h} oc={oc} k={kk} s={stride} party {party}: "
                  f"{'bit-exact' if this else 'MISMATCH'}")
            ok &= this
        if c % 64 == 0:  # both parties' convs of the layer in one launch (model_forward_pair's path)
            x1 = np.frombuffer(rng.bytes(8 * b * c * h * h), dtype="<u8").copy().reshape(b, c, h, h)
            lw = nn._weight(wt, bias, FixedPointConfig())
            outs = nn._conv_pair_dev([torch.from_numpy(v.view(np.int64)).cuda() for v in (x, x1)], "nchw", layer, lw,
                                     (0, 1), 16)
            for party, v in enumerate((x, x1)):
                want = ON.conv2d(v, party, c, oc, kk, kk, stride, pad, wt, bias)
                this = np.array_equal(outs[party].cpu().numpy().view(np.uint64), want)
                print(f"  paired conv b={b} c={c} h={h} oc={oc} k={kk} s={stride} party {party}: "
                      f"{'bit-exact' if this else 'MISMATCH'}")
                ok &= this
    return ok


if __name__ == "__main__":
    torch.cuda.set_device(0)
    name = sys.argv[1]
    print(f"[sanitize] case {name}")
    ok = {"pair": case_pair, "p2p": case_p2p, "conv": case_conv}[name]()
    sys.exit(0 if ok else 1)
