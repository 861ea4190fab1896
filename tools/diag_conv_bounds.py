#!/usr/bin/env python
"""Time the TMA ring conv alone (limb planes made once, outside the timed region) for the ResNet18
b512 layer shapes.  Run it with HB_TC_DEBUG = 0 (normal), 1 (no MMAs: the TMA load stream alone),
2 (no loads: MMAs + epilogue on stale shared memory) to bound the kernel; 4 adds the per-CTA
phase stamps (MMA warp: waits on TMEM-empty / full barriers, issue time).

    HB_TC_DEBUG=1 python tools/diag_conv_bounds.py
"""

import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04875_b200 import _dev, _lib, nn  # noqa: E402
from paper_2309_04875_b200.ring import FixedPointConfig  # noqa: E402

SHAPES = {  # name: (b, c, h, n, k, stride, pad)
    "l1_3x3": (512, 64, 32, 64, 3, 1, 1),
    "l2_3x3s2": (512, 64, 32, 128, 3, 2, 1),
    "l2_3x3": (512, 128, 16, 128, 3, 1, 1),
    "l2_1x1s2": (512, 64, 32, 128, 1, 2, 0),
    "l3_3x3": (512, 256, 8, 256, 3, 1, 1),
    "l4_3x3": (512, 512, 4, 512, 3, 1, 1),
}


def main():
    dbg = int(os.environ.get("HB_TC_DEBUG", "0"))
    rng = np.random.default_rng(0)
    out = {"dbg": dbg}
    for name, (b, c, h, n, k, st, pad) in SHAPES.items():
        w = rng.normal(0, np.sqrt(2 / (c * k * k)), (n, c, k, k)).astype(np.float32)
        lw = nn._weight(w, np.zeros(n, np.float32), FixedPointConfig())
        x = torch.randint(-2**62, 2**62, (b, c, h, h), dtype=torch.int64, device="cuda")
        s = _dev.stream_handle()
        planes = nn._limb_planes(x, s)
        oh = (h + 2 * pad - k) // st + 1
        y = torch.empty((b, n, oh, oh), dtype=torch.int64, device="cuda")

        def conv():
            _lib.call("hb_conv_limbs_tma", planes.data_ptr(), b, c, h, h, k, k, st, pad, lw.wl_tma.data_ptr(), lw.n,
                      lw.j, lw.nt_tma, 0, 16, lw.bias.data_ptr(), None, y.data_ptr(), s)

        for _ in range(3):
            conv()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            conv()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        macs = b * oh * oh * n * c * k * k
        limb_products = 15 if lw.j == 2 else 8 * lw.j
        rec = {"ms": ms, "nt": lw.nt_tma, "J": lw.j, "int8_Tops": 2 * macs * limb_products / ms / 1e9}
        if dbg & 4:
            lib = _lib.load()
            lib.hb_debug_tma_stamps.restype = ctypes.c_int
            buf = np.zeros(1024 * 8, dtype=np.int64)
            lib.hb_debug_tma_stamps(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
            stp = buf.reshape(-1, 8)[:148].mean(0)
            rec["stamps_clk"] = dict(zip(["total", "wait_tmem_empty", "wait_full", "issue", "stages", "units",
                                          "epi_tmem_read", "epi_wait_tfull"], [round(float(v)) for v in stp]))
        out[name] = rec
        nn._PLANES.clear()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
