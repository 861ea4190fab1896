#!/bin/bash
# Round 2 (re-entry) first GPU pass: full GPU parity suite, smoke, the default bench line,
# the NVLink party-kernel harness at w=8/64, --set full captures of both timed ReLU kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"; cat gpurun_out/bench_n1.json | head -c 3000; echo
for km in "22 14" "64 0"; do set -- $km
  timeout 300 python bench.py --path p2p --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_w$(( $1 - $2 )).json 2> gpurun_out/p2p_err_w$(( $1 - $2 )).log; echo "p2p w=$(( $1 - $2 )) rc=$?"
  head -c 1500 gpurun_out/p2p_w$(( $1 - $2 )).json; echo
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_pair -s 3 -c 1 -o gpurun_out/prof_pair_w8_r02 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu pair rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_p2p -s 3 -c 1 -o gpurun_out/prof_p2p_w8_r02 python bench.py --path p2p --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu p2p rc=$?"
