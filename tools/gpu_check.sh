#!/bin/bash
# Full GPU check: parity tests, default bench line, and the bench stderr tail.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench_err.log; echo "bench rc=$?"
tail -5 gpurun_out/bench_err.log
cat gpurun_out/bench.json
