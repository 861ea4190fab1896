#!/bin/bash
# micro-batch lanes for the pair ResNet forward: parity suite + ResNet18 b512 at 1/2/3/4 lanes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_tests.log
for l in 1 2 4; do
  HB_LANES=$l timeout 300 python bench.py --workload resnet18 --steps 5 --warmup 3 > gpurun_out/rn18_lanes$l.json 2> gpurun_out/rn18_lanes${l}_err.log; echo "lanes=$l rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/rn18_lanes$l.json'));print(d['value'],d['ms_per_step'],d['config']['workload'],d['logits_check'])"
done
HB_LANES=2 timeout 300 python bench.py --workload resnet18 --relu-config uniform --steps 5 --warmup 3 > gpurun_out/rn18_lanes2_uniform.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/rn18_lanes2_uniform.json'));print(d['value'],d['ms_per_step'],d['config']['workload'],d['logits_check'])"
