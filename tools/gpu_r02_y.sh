#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python bench.py --gpus 2 --backend gloo --steps 3 --warmup 3 --logn 20 > gpurun_out/multi2.json 2> gpurun_out/multi2_err.log; echo "multi2 rc=$?"; head -c 400 gpurun_out/multi2.json; echo
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
