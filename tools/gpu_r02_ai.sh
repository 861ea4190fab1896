#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_p2p -s 3 -c 1 -o gpurun_out/prof_p2p_w8_r02b python bench.py --path p2p --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu p2p rc=$?"
ncu -i gpurun_out/prof_p2p_w8_r02b.ncu-rep --page raw --csv > gpurun_out/prof_p2p_w8_r02b_raw.csv 2>/dev/null
rm -f gpurun_out/prof_p2p_w8_r02b.ncu-rep
