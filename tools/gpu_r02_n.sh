#!/bin/bash
mkdir -p gpurun_out
for g in "" "--no-model-graph"; do timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 $g > gpurun_out/rn18_g.json 2> gpurun_out/rn18_g_err.log; echo "rn18 $g rc=$?"; tail -2 gpurun_out/rn18_g_err.log; python -c "import json;d=json.load(open('gpurun_out/rn18_g.json'));print(d['value'],d['ms_per_step'],d['config']['cuda_graph'],d['logits_check'])"; done
timeout 600 python bench.py --workload resnet50 --steps 3 --warmup 2 > gpurun_out/rn50_g.json 2> gpurun_out/rn50_g_err.log; echo "rn50 rc=$?"; tail -2 gpurun_out/rn50_g_err.log; python -c "import json;d=json.load(open('gpurun_out/rn50_g.json'));print(d['value'],d['ms_per_step'],d['config']['cuda_graph'],d['logits_check'])"
