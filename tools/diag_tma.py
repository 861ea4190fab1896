"""TMA implicit-GEMM ring conv vs the gather kernel: bit-equality and timing per ResNet layer shape."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_04875_b200 import nn
from paper_2309_04875_b200.ring import FixedPointConfig

SHAPES = [  # (b, c, h, w, n, k, stride, pad)
    (512, 64, 32, 32, 64, 3, 1, 1), (512, 64, 32, 32, 128, 3, 2, 1), (512, 64, 32, 32, 128, 1, 2, 0),
    (512, 128, 16, 16, 128, 3, 1, 1), (512, 256, 8, 8, 256, 3, 1, 1), (512, 512, 4, 4, 512, 3, 1, 1),
    (512, 512, 1, 1, 10, 1, 1, 0), (3, 64, 5, 8, 20, 3, 1, 1), (130, 128, 4, 4, 70, 3, 1, 1),
    (64, 128, 8, 8, 200, 3, 1, 1), (64, 64, 16, 16, 136, 3, 2, 1), (96, 256, 4, 4, 384, 3, 1, 1, 8.0),
    (33, 192, 8, 8, 128, 1, 1, 0, 8.0),
]
rng = np.random.default_rng(0)
for shp in SHAPES:
    (b, c, h, w, n, k, st, pad), scale = shp[:8], (shp[8] if len(shp) > 8 else 1.0)
    W = (scale * rng.normal(0, np.sqrt(2 / (c * k * k)), (n, c, k, k))).astype(np.float32)
    if k == 1 and h == 1:
        W = W.reshape(n, c)
    B = rng.normal(0, 0.1, n).astype(np.float32)
    lw = nn._weight(W, B, FixedPointConfig())
    x = torch.randint(-2**62, 2**62, (b, c, h, w), dtype=torch.int64, device="cuda")
    res = {}
    for mode in ("tcgather", "tc"):
        nn.RING_GEMM = mode
        for party in (0, 1):
            res[(mode, party)] = nn._gemm_tc(x, (k, k, st, pad), lw, party, 16)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            nn._gemm_tc(x, (k, k, st, pad), lw, 0, 16)
        e0.record()
        for _ in range(5):
            nn._gemm_tc(x, (k, k, st, pad), lw, 0, 16)
        e1.record(); torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / 5
    oh = (h + 2 * pad - k) // st + 1
    macs = b * oh * oh * c * k * k * n * (lw.j * 8 - lw.j * (lw.j - 1) // 2)
    same = all(torch.equal(res[("tc", p)], res[("tcgather", p)]) for p in (0, 1))
    print(f"b{b} c{c} {h}x{w} n{n} k{k} s{st} J={lw.j} tma={lw.wl_tma is not None}: equal={same} "
          f"gather {res['tcgather']:.3f} ms  tma {res['tc']:.3f} ms  ({macs / res['tc'] / 1e9:.0f} TMAC/s)")
