#!/bin/bash
# round-2 results pass: bench line, ResNet50, P2P width sweep, pair-kernel sweep, ResNet18 launch list
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline'],d['e2e']['value'],d['resnet18']['value'],d['clocks'])"
timeout 600 python bench.py --workload resnet50 --steps 3 --warmup 2 > gpurun_out/bench_rn50.json 2> gpurun_out/bench_rn50_err.log; echo "rn50 rc=$?"; head -c 600 gpurun_out/bench_rn50.json; echo
for km in "64 0" "32 0" "22 6" "22 14" "22 16"; do set -- $km
  timeout 300 python bench.py --path p2p --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_w$(( $1 - $2 )).json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2p_w$(( $1 - $2 )).json'));print('p2p w=$(( $1 - $2 ))', d['value'], round(d['roofline']['frac'],3), d['correct'])"
done
timeout 1200 python bench.py --sweep gpurun_out/sweep_r02.json --steps 20 --no-resnet > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_launches.csv python bench.py --workload resnet18 --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
