#!/bin/bash
# conv quick check: layer1 timing, conv parity tests, resnet18 bench
for d in 0 4; do HB_TC_DEBUG=$d timeout 300 python tools/diag_conv.py; done
timeout 900 python -m pytest tests/test_gpu_nn.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python bench.py --workload resnet18 --steps 5 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rn18', d['value'], d['ms_per_step'])"
