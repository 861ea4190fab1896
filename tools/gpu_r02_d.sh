#!/bin/bash
# Round 2 second pass: the P2P smem fix (odd widths), the bench line with model-level baselines, the
# ResNet18 window search, multi-rank bench self-launch on one GPU (gloo), compute-sanitizer runs.
mkdir -p gpurun_out/configs
timeout 900 python -m pytest tests/test_gpu_p2p.py -q -p no:cacheprovider > gpurun_out/gpu_tests_p2p.log 2>&1; echo "pytest p2p rc=$?"
tail -3 gpurun_out/gpu_tests_p2p.log
timeout 1200 python tools/search_resnet.py resnet18 --out-dir gpurun_out/configs > gpurun_out/search_rn18.log 2>&1; echo "search rc=$?"; tail -3 gpurun_out/search_rn18.log
timeout 300 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --multi-path p2p > gpurun_out/multi2_p2p.json 2> gpurun_out/multi2_p2p_err.log; echo "multi2 p2p rc=$?"; head -c 1200 gpurun_out/multi2_p2p.json; echo
timeout 300 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --multi-path nccl > gpurun_out/multi2_nccl.json 2> gpurun_out/multi2_nccl_err.log; echo "multi2 nccl rc=$?"; head -c 1200 gpurun_out/multi2_nccl.json; echo
timeout 600 python bench.py --gpus 2 --backend gloo --workload resnet18 --batch 4096 --steps 2 --warmup 3 --resnet-triple-gb 40 > gpurun_out/multi2_rn18.json 2> gpurun_out/multi2_rn18_err.log; echo "multi2 rn18 rc=$?"; head -c 1500 gpurun_out/multi2_rn18.json; echo
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1_err.log; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['roofline']['frac'],d['desk_cnn'],d['resnet18'])"
for c in pair:racecheck pair:memcheck p2p:memcheck p2p:racecheck conv:memcheck conv:racecheck; do
  case=${c%%:*}; tool=${c##*:}
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $case > gpurun_out/sanitize_${case}_${tool}.log 2>&1
  echo "sanitize $case $tool rc=$?"; tail -2 gpurun_out/sanitize_${case}_${tool}.log
done
timeout 300 python tools/diag_overlap.py > gpurun_out/overlap.json 2> gpurun_out/overlap_err.log; echo "overlap rc=$?"; cat gpurun_out/overlap.json; tail -3 gpurun_out/overlap_err.log
