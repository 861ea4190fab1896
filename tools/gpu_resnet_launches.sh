#!/bin/bash
# Per-kernel launch list of one ResNet18 b512 forward (cold, serialised) -> gpurun_out/rn18_launches.csv
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_launches.csv \
  python bench.py --workload resnet18 --steps 1 --warmup 1 > gpurun_out/rn18_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/rn18_ncu.log
timeout 600 python bench.py --workload resnet50 --steps 3 --warmup 2 > gpurun_out/rn50.json 2> gpurun_out/rn50_err.log; echo "rn50 rc=$?"
tail -3 gpurun_out/rn50_err.log; cat gpurun_out/rn50.json
