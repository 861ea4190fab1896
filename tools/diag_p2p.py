"""Debug the local two-stream P2P kernel: tiles per CTA vs grid."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import golden_cases as gc
from hb_helpers import stocked_sessions_for_relu
from paper_2309_04875_b200 import protocol, transport
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor
from test_gpu_p2p import _p2p_pair

def run(logn, k, m, max_ctas, timeout=5.0):
    n = (1 << logn) + 37
    x0, x1 = gc.baseline_inputs(n, seed=logn)
    s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=logn)
    t0 = ArithShareTensor(0, 64, torch.from_numpy(x0.view(np.int64)).cuda())
    t1 = ArithShareTensor(1, 64, torch.from_numpy(x1.view(np.int64)).cuda())
    links = transport.local_p2p_pair(max_ctas)
    for lk in links: lk.timeout_s = timeout
    t = time.time()
    try:
        r0, r1 = _p2p_pair(s0, s1, t0, t1, BitWindow(k, m), links)
        s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=logn)
        q0, q1 = protocol.relu_pair((s0, s1), t0, t1, BitWindow(k, m))
        ok = torch.equal(r0.data, q0.data) and torch.equal(r1.data, q1.data)
    except Exception as e:
        ok = repr(e)[:60]
    print(f"logn={logn} w={k-m} max_ctas={max_ctas}: {ok}  {time.time()-t:.2f}s", flush=True)

for mc in (-1,):
    run(16, 22, 14, mc)
for mc in (-1, 64):
    run(20, 22, 14, mc)
for logn in (22, 24): run(logn, 22, 14, -1); run(logn, 64, 0, -1)
