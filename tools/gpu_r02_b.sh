#!/bin/bash
# Round 2, second pass: the rewritten NVLink party kernel (exact w-bit wire, cooperative grid,
# alternating receive regions, gpu/sys scope), the new parity tests, the window search for ResNet18.
mkdir -p gpurun_out/configs
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gpu_tests.log
for scope in gpu sys; do for km in "22 14" "64 0"; do set -- $km
  timeout 300 python bench.py --path p2p --p2p-scope $scope --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet > gpurun_out/p2p_${scope}_w$(( $1 - $2 )).json 2> gpurun_out/p2p_${scope}_err.log; echo "p2p $scope w=$(( $1 - $2 )) rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/p2p_${scope}_w$(( $1 - $2 )).json'));print(d['value'], d['roofline']['frac'], d['correct'])"
done; done
timeout 900 python tools/search_resnet.py resnet18 --out-dir gpurun_out/configs > gpurun_out/search_rn18.log 2>&1; echo "search rc=$?"; tail -3 gpurun_out/search_rn18.log
