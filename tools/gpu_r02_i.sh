#!/bin/bash
# both parties' convs in one launch: parity + ResNet18 b512 with / without + conv bounds
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nn.py -q -p no:cacheprovider -x > gpurun_out/gpu_tests_nn.log 2>&1; echo "pytest nn rc=$?"
tail -3 gpurun_out/gpu_tests_nn.log
for cp in 1 0; do
  HB_CONV_PAIR=$cp timeout 300 python bench.py --workload resnet18 --steps 5 --warmup 3 > gpurun_out/rn18_cp$cp.json 2> gpurun_out/rn18_cp${cp}_err.log; echo "conv pair=$cp rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/rn18_cp$cp.json'));print(d['value'],d['ms_per_step'],d['logits_check'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_launches.csv python bench.py --workload resnet18 --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py launches gpurun_out/rn18_launches.csv 2>/dev/null | head -14
