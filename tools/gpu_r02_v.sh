#!/bin/bash
# round-2 re-entry check: full GPU suite, smoke, default bench line, reference arm, N=2 self-launch (gloo, one GPU)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline']['frac'],d['roofline']['traffic'],d['e2e']['value'],d['resnet18']['value'],d['cpu_baseline']['value'],d['clocks'])"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_ref.json'));print('ref', d['value'], d['cpu_baseline']['cores'])"
timeout 600 python bench.py --gpus 2 --backend gloo --logn 20 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2_err.log; echo "bench n2 rc=$?"; tail -c 600 gpurun_out/bench_n2.json
