"""TMA conv with / without the fused residual add, and the unfused add kernel, per ResNet shape."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_04875_b200 import nn
from paper_2309_04875_b200.ring import FixedPointConfig

def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

rng = np.random.default_rng(0)
for (b, c, h, n) in [(512, 64, 32, 64), (512, 128, 16, 128), (512, 512, 4, 512)]:
    W = rng.normal(0, np.sqrt(2 / (c * 9)), (n, c, 3, 3)).astype(np.float32)
    lw = nn._weight(W, np.zeros(n, np.float32), FixedPointConfig())
    x = torch.randint(-2**62, 2**62, (b, c, h, h), dtype=torch.int64, device="cuda")
    r = torch.randint(-2**62, 2**62, (b, n, h, h), dtype=torch.int64, device="cuda")
    g = (3, 3, 1, 1)
    y0 = nn._add_dev(nn._gemm_tc(x, g, lw, 0, 16), r)
    y1 = nn._gemm_tc(x, g, lw, 0, 16, r)
    t_plain = t(lambda: nn._gemm_tc(x, g, lw, 0, 16))
    t_fused = t(lambda: nn._gemm_tc(x, g, lw, 0, 16, r))
    t_add = t(lambda: nn._add_dev(y0, r))
    print(f"b{b} c{c} {h}x{h} n{n}: equal={torch.equal(y0, y1)} conv {t_plain:.3f} ms  conv+res {t_fused:.3f} ms  add {t_add:.3f} ms")
