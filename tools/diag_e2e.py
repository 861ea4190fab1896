"""PCIe ceiling and e2e variants for the pinned-host relu_pair path (diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
from paper_2309_04875_b200 import dealer, protocol, transport
from paper_2309_04875_b200.protocol import ProtocolSession
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor

n = 1 << 24
dev = torch.device("cuda", 0)
h = torch.empty(n, dtype=torch.int64, pin_memory=True); d = torch.empty(n, dtype=torch.int64, device=dev)
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    print(f"{name}: {8 * n / dt / 1e9:.1f} GB/s")
x0, x1 = bench.device_inputs(n, 64, 1, dev)
h0, h1 = x0.cpu().pin_memory(), x1.cpu().pin_memory()
eps = transport.local_pair(); stores = (dealer.TripleStore(0), dealer.TripleStore(1))
bench.stock_sets(stores, (0, 1), n, 8, 64, 3, 20, 4, 3)
S = (ProtocolSession(eps[0], stores[0]), ProtocolSession(eps[1], stores[1]))
win = BitWindow(22, 14)
def step(a0, a1, chunk=None):
    for st in stores:
        if st.remaining("bool", 8) < 7 * n:
            st.rewind("bool", 8); st.rewind("arith", 64)
    if chunk:
        protocol._relu_pair_pinned.__defaults__ = (chunk,)
    return protocol.relu_pair(S, ArithShareTensor(0, 64, a0), ArithShareTensor(1, 64, a1), win)
for chunk in (1 << 20, 1 << 21, 1 << 22, 1 << 23):
    step(h0, h1, chunk); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): step(h0, h1, chunk)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    print(f"pipelined chunk=2^{chunk.bit_length()-1}: {dt*1e3:.2f} ms/step -> {n/dt:.3e} elem/s")
