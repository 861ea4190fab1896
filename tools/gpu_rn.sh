#!/bin/bash
# ResNet18 (and optionally ResNet50) bench lines + GPU nn parity tests
timeout 900 python -m pytest tests/test_gpu_nn.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
timeout 600 python bench.py --workload resnet18 --steps 5 --warmup 2 2>/dev/null > gpurun_out/rn18.json; python -c "import json; d=json.load(open('gpurun_out/rn18.json')); print('rn18', d['value'], d['ms_per_step'])"
