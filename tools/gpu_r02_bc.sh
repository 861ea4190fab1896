#!/bin/bash
# 64-thread pair-kernel CTAs: full GPU suite, bench line, ncu of the timed kernel, pair sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_pair -s 3 -c 1 -o gpurun_out/prof_pair_w8_r02c python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu pair rc=$?"
ncu -i gpurun_out/prof_pair_w8_r02c.ncu-rep --page raw --csv > gpurun_out/ncu_raw_pair_w8_r02.csv 2>/dev/null; rm -f gpurun_out/prof_pair_w8_r02c.ncu-rep
timeout 1200 python bench.py --sweep gpurun_out/sweep_r02.json --steps 20 --no-resnet > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline']['frac'],d['roofline']['kernel'],d['e2e']['value'],d['resnet18']['value'])"
