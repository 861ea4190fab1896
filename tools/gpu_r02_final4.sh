#!/bin/bash
# closing pass after the pair-kernel register budget change: GPU suite, smoke, bench line, pair sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline']['frac'],d['roofline']['traffic'],d['e2e']['value'],d['resnet18']['value'],d['cpu_baseline']['value'],d['clocks'])"
timeout 900 python bench.py --sweep gpurun_out/sweep_r02b.json --steps 20 --no-resnet > /dev/null 2> gpurun_out/sweep_r02b.err; echo "sweep rc=$?"
