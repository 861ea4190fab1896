#!/bin/bash
# Round-2 first GPU pass: parity suite, --set full captures of the timed ReLU kernels (fused pair at
# the bench config, both-party P2P harness), the P2P harness bench line, compute-sanitizer runs.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --path p2p --steps 20 --no-cpu-baseline --no-resnet > gpurun_out/p2p_pair.json 2> gpurun_out/p2p_pair_err.log; echo "p2p bench rc=$?"
cat gpurun_out/p2p_pair.json
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_pair -s 3 -c 1 -o gpurun_out/prof_pair_w8_r02 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu pair rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_relu_p2p -s 3 -c 1 -o gpurun_out/prof_p2p_w8_r02 python bench.py --path p2p --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo "ncu p2p rc=$?"
for c in pair:racecheck pair:memcheck p2p:memcheck p2p:racecheck conv:memcheck conv:racecheck; do
  case=${c%%:*}; tool=${c##*:}
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $case > gpurun_out/sanitize_${case}_${tool}.log 2>&1
  echo "sanitize $case $tool rc=$?"; tail -2 gpurun_out/sanitize_${case}_${tool}.log
done
