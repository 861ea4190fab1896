"""Host overhead of one relu_pair call at small n (cProfile)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_2309_04875_b200 import dealer, protocol, transport
from paper_2309_04875_b200.protocol import ProtocolSession
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor
n, w = 1 << 16, 8
eps = transport.local_pair()
stores = (dealer.TripleStore(0), dealer.TripleStore(1))
reps = 400
dealer.stock_on_device(stores, (0, 1), "bool", w, n * 7 * reps, seed=1, exact=False)
dealer.stock_on_device(stores, (0, 1), "arith", 64, n * 2 * reps, seed=2, exact=False)
ss = (ProtocolSession(eps[0], stores[0]), ProtocolSession(eps[1], stores[1]))
x0 = ArithShareTensor(0, 64, torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda"))
x1 = ArithShareTensor(1, 64, torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda"))
win = BitWindow(22, 14)
for _ in range(20): protocol.relu_pair(ss, x0, x1, win)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): protocol.relu_pair(ss, x0, x1, win)
torch.cuda.synchronize()
print("per call us", (time.perf_counter() - t) / 200 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(100): protocol.relu_pair(ss, x0, x1, win)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
