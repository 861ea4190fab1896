"""Stage-by-stage check of the int8-limb ring GEMM against numpy (debug aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import golden_cases as gc
from oracle import hb_oracle_nn as ON
from paper_2309_04875_b200 import nn, ring, _lib, _dev
from paper_2309_04875_b200.ring import FixedPointConfig

case = gc.NN_CASES[0]; ins = gc.make_nn_inputs(case)
x, w, b = ins["x0"], ins["w"], ins["b"]
cfg = FixedPointConfig()
lw = nn._weight(w, b, cfg)
m, k = x.shape
xd = _dev.to_device(x)
a = torch.empty((8 * m, lw.kp), dtype=torch.int8, device="cuda")
_lib.call("hb_im2col_limbs", xd.data_ptr(), m, k, 1, 1, 1, 1, 1, 0, lw.kp, a.data_ptr(), _dev.stream_handle())
ah = a.cpu().numpy()
want_a = np.zeros((8, m, lw.kp), dtype=np.int8)
for i in range(8):
    want_a[i, :, :k] = (((x >> np.uint64(8 * i)) & np.uint64(255)).astype(np.int64) - 128).astype(np.int8)
print("im2col limbs ok:", np.array_equal(ah.reshape(8, m, lw.kp)[:, :, :k], want_a[:, :, :k]))
p = torch._int_mm(a, lw.bt.t())
pw = (a.int().cpu() @ lw.bt.int().cpu().t())
print("int_mm ok:", torch.equal(p.cpu(), pw), p.shape, p.stride(), lw.bt.t().stride())
p2 = torch._int_mm(a, lw.bt.t().contiguous())
print("int_mm (row-major mat2) ok:", torch.equal(p2.cpu(), pw))
out = torch.empty(m * lw.n, dtype=torch.int64, device="cuda")
_lib.call("hb_limb_combine", pw.cuda().data_ptr(), m, lw.n, lw.np_, lw.j, lw.colsum.data_ptr(), 0, 16,
          lw.bias.data_ptr(), 0, 1, out.data_ptr(), _dev.stream_handle())
print("combine(exact P) ok:", np.array_equal(out.cpu().numpy().view(np.uint64).reshape(m, lw.n), ON.linear(x, 0, w, b)))
