"""One ResNet layer shape through the TMA conv path (for ncu): python tools/diag_tma1.py b c h n k stride pad"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_04875_b200 import nn
from paper_2309_04875_b200.ring import FixedPointConfig
b, c, h, n, k, st, pad = map(int, sys.argv[1:8])
rng = np.random.default_rng(0)
W = rng.normal(0, np.sqrt(2 / (c * k * k)), (n, c, k, k)).astype(np.float32)
lw = nn._weight(W, np.zeros(n, np.float32), FixedPointConfig())
x = torch.randint(-2**62, 2**62, (b, c, h, h), dtype=torch.int64, device="cuda")
for _ in range(3):
    nn._PLANES.clear()
    nn._gemm_tc(x, (k, k, st, pad), lw, 0, 16)
torch.cuda.synchronize()
import os
if int(os.environ.get("HB_TC_DEBUG", "0")) & 4:
    import ctypes
    from paper_2309_04875_b200 import _lib
    lib = _lib.load()
    lib.hb_debug_tma_stamps.restype = ctypes.c_int
    buf = np.zeros(1024 * 8, dtype=np.int64)
    lib.hb_debug_tma_stamps(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
    st = buf.reshape(-1, 8)[:148]
    print("MMA warp per CTA (mean clk): total %.0f  wait tmem-empty %.0f  wait full %.0f  issue %.0f  stages %.0f units %.0f"
          "  | epilogue warp0: tmem read %.0f  wait tfull %.0f" % tuple(st[:, :8].mean(0)))
