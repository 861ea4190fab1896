import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import golden_cases as gc
from hb_helpers import stocked_sessions_for_relu
from paper_2309_04875_b200 import protocol, transport
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor
sync_each = sys.argv[1] == "1"
links = transport.local_p2p_pair(max_ctas=64)
links[0].timeout_s = links[1].timeout_s = 5.0
st = [torch.cuda.Stream(), torch.cuda.Stream()]
layers = [((1 << 20), (22, 20)), ((1 << 21), (64, 0)), (25088, (22, 14)), (802816, (22, 14)), ((1 << 20) + 3, (22, 20)), ((1 << 21), (64, 0))][:int(sys.argv[2]) if len(sys.argv) > 2 else 6]
sess = [stocked_sessions_for_relu(n, k - m, 64, seed=40 + i)[:2] for i, (n, (k, m)) in enumerate(layers)]
ins = [gc.baseline_inputs(n, seed=50 + i) for i, (n, _) in enumerate(layers)]
dev_in = [(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda()) for a, b in ins]
import ctypes
from paper_2309_04875_b200 import _lib
def lb(n, km):
    nt = ctypes.c_int64(0); return _lib.load().hb_relu_p2p_bytes(km[0], km[1], n, 0, ctypes.byref(nt)), nt.value
sizes = [lb(n, km) for n, km in layers]
links[0].ensure(max(b for b, _ in sizes), max(t for _, t in sizes))
torch.cuda.synchronize()
print("after ensure", links[0].state.tolist(), links[1].state.tolist(), links[0].cap_bytes, flush=True)
ybuf = [[torch.empty(n, dtype=torch.int64, device="cuda") for _ in (0, 1)] for n, _ in layers]
torch.cuda.synchronize()
for i, (n, (k, m)) in enumerate(layers):
    for p in (0, 1):
        with torch.cuda.stream(st[p]):
            protocol.relu_p2p(sess[i][p], ArithShareTensor(p, 64, dev_in[i][p]), BitWindow(k, m), links[p], stream=st[p], out=ybuf[i][p])
    if sync_each:
        torch.cuda.synchronize()
        print(i, links[0].state.tolist(), links[1].state.tolist(), int(links[0].err.item()), flush=True)
torch.cuda.synchronize()
print("end", links[0].state.tolist(), links[1].state.tolist(), int(links[0].err.item()), int(links[1].err.item()))
