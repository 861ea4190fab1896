#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
for km in "64 0" "32 0" "22 6" "22 14" "22 16"; do set -- $km
  timeout 300 python bench.py --path p2p --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_w$(( $1 - $2 )).json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2p_w$(( $1 - $2 )).json'));print('p2p w=$(( $1 - $2 ))', d['value'], round(d['roofline']['frac'],3), d['correct'])"
done
timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 > gpurun_out/rn18.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/rn18.json'));print('rn18', d['value'], d['ms_per_step'])"
