"""Time one ResNet18 layer1 conv (batch 512) through hb_conv_limbs_tc (debug aid)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_04875_b200 import nn, _lib, _dev
from paper_2309_04875_b200.ring import FixedPointConfig
b, c, h, w, n = 512, 64, 32, 32, 64
rng = np.random.default_rng(0)
W = (rng.normal(0, np.sqrt(2 / 576), (n, c, 3, 3))).astype(np.float32); B = np.zeros(n, np.float32)
lw = nn._weight(W, B, FixedPointConfig())
x = torch.randint(-2**62, 2**62, (b, c, h, w), dtype=torch.int64, device="cuda")
L = nn.Conv2d(c, n, 3, 3, 1, 1, "w", "b")
for _ in range(2): nn._gemm_tc(x, (3, 3, 1, 1), lw, 0, 16)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): nn._gemm_tc(x, (3, 3, 1, 1), lw, 0, 16)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
macs = b * h * w * c * 9 * n * (lw.j * 8 - lw.j * (lw.j - 1) // 2)
print(f"dbg={os.environ.get('HB_TC_DEBUG','0')} J={lw.j}: {ms:.3f} ms  ({macs / ms / 1e9:.1f} TMAC/s int8)")
if int(os.environ.get("HB_TC_DEBUG", "0")) & 4:
    import ctypes
    lib = _lib.load()
    buf = np.zeros(4096 * 8 * 4, dtype=np.int64)
    nn_ = lib.hb_debug_conv_stamps(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
    st = buf[:nn_].reshape(-1, 8)
    d = np.diff(st[:, :6], axis=1)
    print("mean cycles: setup %.0f  mainloop(prod) %.0f  wait_done %.0f  epilogue %.0f  teardown %.0f" % tuple(d.mean(0)))
    tot = st[:, 5] - st[:, 0]
    print("per-CTA total mean %.0f cycles; CTAs %d" % (tot.mean(), len(st)))
    # gap between consecutive CTAs on the same SM
    gaps = []
    for sm in np.unique(st[:, 6]):
        s = st[st[:, 6] == sm]; s = s[np.argsort(s[:, 0])]
        gaps += list(s[1:, 0] - s[:-1, 5])
    print("mean gap between CTAs on an SM: %.0f cycles" % np.mean(gaps))
