#!/bin/bash
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn50_launches.csv python bench.py --workload resnet50 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
python tools/launch_breakdown.py gpurun_out/rn50_launches.csv
python - <<'PY'
import torch, time
n = 1 << 26
h = torch.empty(n, dtype=torch.int64, pin_memory=True); d = torch.empty(n, dtype=torch.int64, device="cuda")
h2 = torch.empty(n, dtype=torch.int64, pin_memory=True); d2 = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); a = time.perf_counter() - t
t = time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); b = time.perf_counter() - t
t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c = time.perf_counter() - t
print(f"PCIe: H2D {8*n/a/1e9:.1f} GB/s, D2H {8*n/b/1e9:.1f} GB/s, both at once {2*8*n/c/1e9:.1f} GB/s total")
PY
