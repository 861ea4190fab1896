#!/bin/bash
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_launches3.csv python bench.py --workload resnet18 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
python tools/launch_breakdown.py gpurun_out/rn18_launches3.csv
