"""Both parties' convs of one ResNet18 b512 layer in one launch (for ncu):
python tools/diag_conv_pair.py b c h n k stride pad"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04875_b200 import nn  # noqa: E402
from paper_2309_04875_b200.ring import FixedPointConfig  # noqa: E402

b, c, h, n, k, st, pad = map(int, sys.argv[1:8])
rng = np.random.default_rng(0)
W = rng.normal(0, np.sqrt(2 / (c * k * k)), (n, c, k, k)).astype(np.float32)
lw = nn._weight(W, np.zeros(n, np.float32), FixedPointConfig())
layer = nn.Conv2d(c, n, k, k, st, pad, weight="w", bias="b")
xs = [torch.randint(-2**62, 2**62, (b, c, h, h), dtype=torch.int64, device="cuda") for _ in range(2)]
for _ in range(4):
    nn._PLANES.clear()
    out = nn._conv_pair_dev(xs, "nchw", layer, lw, (0, 1), 16)
    assert out is not None
torch.cuda.synchronize()
