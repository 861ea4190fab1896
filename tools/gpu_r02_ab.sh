#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_integration.py -q -p no:cacheprovider > gpurun_out/gpu_tests_p2p.log 2>&1; echo "pytest p2p rc=$?"; tail -2 gpurun_out/gpu_tests_p2p.log
for scope in gpu sys; do for km in "64 0" "32 0" "22 6" "22 14" "22 16"; do set -- $km
  timeout 300 python bench.py --path p2p --p2p-scope $scope --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_${scope}_w$(( $1 - $2 )).json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2p_${scope}_w$(( $1 - $2 )).json'));print('p2p $scope w=$(( $1 - $2 ))', d['value'], round(d['roofline']['frac'],3), d['correct'])"
done; done
