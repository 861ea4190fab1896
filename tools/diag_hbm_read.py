#!/usr/bin/env python
"""HBM streaming rates on this B200 for the mixes a read-heavy kernel like the pair ReLU sees (77 B
read + 8 B written per element and party): torch sum (read only), copy (1:1), add (2 reads : 1 write).
Best of 10, CUDA events, 4 GiB operands."""
import json

import torch


def best_s(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


n = 1 << 29  # 4 GiB of int64
x = torch.ones(n, dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
m = n // 3
res = {"read_only_sum_GBps": 8 * n / best_s(lambda: x.sum()) / 1e9,
       "copy_GBps": 16 * n / best_s(lambda: y.copy_(x)) / 1e9,
       "read2_write1_GBps": 24 * m / best_s(lambda: torch.add(x[:m], x[m:2 * m], out=y[:m])) / 1e9}
print(json.dumps(res))
