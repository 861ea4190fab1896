#!/bin/bash
# ReLU -> limb planes fusion: parity, ResNet18 b512 with / without, e2e pipeline chunk sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nn.py -q -p no:cacheprovider -x > gpurun_out/gpu_tests_nn.log 2>&1; echo "pytest nn rc=$?"
tail -3 gpurun_out/gpu_tests_nn.log
for pl in 1 0; do
  HB_PLANES_FROM_RELU=$pl timeout 300 python bench.py --workload resnet18 --steps 5 --warmup 3 > gpurun_out/rn18_planes$pl.json 2> gpurun_out/rn18_planes${pl}_err.log; echo "planes=$pl rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/rn18_planes$pl.json'));print(d['value'],d['ms_per_step'],d['logits_check'])"
done
for c in 19 20 21 22; do
  HB_PIPE_CHUNK=$((1<<c)) timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-resnet > gpurun_out/e2e_c$c.json 2> gpurun_out/e2e_c${c}_err.log
  python -c "import json;d=json.load(open('gpurun_out/e2e_c$c.json'));print('chunk 2^$c', d['e2e']['value'])"; grep "per-step" gpurun_out/e2e_c${c}_err.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_launches.csv python bench.py --workload resnet18 --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py launches gpurun_out/rn18_launches.csv 2>/dev/null | head -14
