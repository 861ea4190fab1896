#!/bin/bash
# NVLink party kernel: parity suite + 2^24 bench lines at w = 64 / 32 / 16 / 8 / 6 (gpu scope)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -q -p no:cacheprovider 2>&1 | tail -2
for km in "64 0" "32 0" "22 6" "22 14" "22 16"; do set -- $km
  timeout 300 python bench.py --path p2p --k $1 --m $2 --steps 20 --no-cpu-baseline --no-resnet --no-e2e > gpurun_out/p2p_w$(( $1 - $2 )).json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2p_w$(( $1 - $2 )).json'));print('p2p gpu w=$(( $1 - $2 ))', '%.3e' % d['value'], round(d['roofline']['frac'],3), d['correct'])"
done
