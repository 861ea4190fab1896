#!/bin/bash
# retuned P2P constants: full GPU suite, P2P width sweep, ResNet50 window search + bench
mkdir -p gpurun_out/configs
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
for km in "64 0" "32 0" "22 6" "22 14" "22 16"; do set -- $km
  timeout 300 python bench.py --path p2p --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_w$(( $1 - $2 )).json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2p_w$(( $1 - $2 )).json'));print('p2p w=$(( $1 - $2 ))', d['value'], round(d['roofline']['frac'],3), d['correct'])"
done
timeout 1500 python tools/search_resnet.py resnet50 --eco-only --n 32 --out-dir gpurun_out/configs > gpurun_out/search_rn50.log 2>&1; echo "search rn50 rc=$?"; tail -2 gpurun_out/search_rn50.log
cp gpurun_out/configs/resnet50_windows_w8.json configs/ 2>/dev/null
timeout 600 python bench.py --workload resnet50 --steps 3 --warmup 2 > gpurun_out/rn50.json 2> gpurun_out/rn50_err.log; echo "rn50 rc=$?"; python -c "import json;d=json.load(open('gpurun_out/rn50.json'));print(d['value'],d['ms_per_step'],d['config']['workload'],d['logits_check'])"
