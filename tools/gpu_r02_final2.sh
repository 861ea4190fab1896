#!/bin/bash
# round-2 closing pass: full GPU suite, smoke, default bench line, reference arm, NVLink party kernel
# 2^24 lines and the graph-replayed (n, w) sweep at both flag scopes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline']['frac'],d['roofline']['traffic'],d['e2e']['value'],d['resnet18']['value'],d['cpu_baseline']['value'],d['clocks'])"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_ref.json'));print('ref', d['value'], d['cpu_baseline']['cores'])"
for km in "64 0" "32 0" "22 6" "22 14" "22 16"; do set -- $km
  timeout 300 python bench.py --path p2p --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_w$(( $1 - $2 )).json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2p_w$(( $1 - $2 )).json'));print('p2p gpu w=$(( $1 - $2 ))', '%.3e' % d['value'], round(d['roofline']['frac'],3), d['correct'])"
done
bash tools/gpu_p2p_graph_sweep.sh
