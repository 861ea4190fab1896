#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['resnet18']['value'],d['desk_cnn']['gpu_samples_per_s'],d['clocks'])"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; head -c 400 gpurun_out/bench_ref.json; echo
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_p2p -s 3 -c 1 -o gpurun_out/prof_p2p_w8_r02b python bench.py --path p2p --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu p2p rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_p2p -s 3 -c 1 -o gpurun_out/prof_p2p_w64_r02b python bench.py --path p2p --k 64 --m 0 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu p2p64 rc=$?"
