#!/bin/bash
timeout 900 python bench.py --workload resnet50 --steps 3 --warmup 2 > gpurun_out/rn50.json 2> gpurun_out/rn50_err.log; echo "rn50 rc=$?"
tail -3 gpurun_out/rn50_err.log; cat gpurun_out/rn50.json
