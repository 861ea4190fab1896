#!/usr/bin/env python
"""Host cost of one relu_p2p_pair call (small layer): wall time per call and a cProfile breakdown."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2309_04875_b200 import dealer, protocol, transport  # noqa: E402
from paper_2309_04875_b200.protocol import ProtocolSession  # noqa: E402
from paper_2309_04875_b200.ring import BitWindow  # noqa: E402
from paper_2309_04875_b200.sharing import ArithShareTensor  # noqa: E402

n, k, m, reps = 1 << 14, 22, 14, 400
L = protocol.prefix_levels(k - m)
eps = transport.local_pair()
stores = (dealer.TripleStore(0), dealer.TripleStore(1))
dealer.stock_on_device(stores, (0, 1), dealer.BOOL, k - m, n * (1 + 2 * L) * (reps + 10), seed=1)
dealer.stock_on_device(stores, (0, 1), dealer.ARITH, 64, 2 * n * (reps + 10), seed=2)
sess = (ProtocolSession(eps[0], stores[0]), ProtocolSession(eps[1], stores[1]))
x = [torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda") for _ in range(2)]
links = transport.local_p2p_pair()
win = BitWindow(k, m)


def call():
    return protocol.relu_p2p_pair(sess, ArithShareTensor(0, 64, x[0]), ArithShareTensor(1, 64, x[1]), win, links)


for _ in range(5):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    call()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / 100:.1f} us/call, wall incl. GPU {1e6 * (t2 - t0) / 100:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    call()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
