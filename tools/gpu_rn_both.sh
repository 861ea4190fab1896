#!/bin/bash
for mk in 512 0 1024; do
  echo "HB_TMA_WIDE_MIN_K=$mk"
  HB_TMA_WIDE_MIN_K=$mk timeout 600 python bench.py --workload resnet18 --steps 5 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' rn18', d['value'], d['ms_per_step'])"
  HB_TMA_WIDE_MIN_K=$mk timeout 600 python bench.py --workload resnet50 --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' rn50', d['value'], d['ms_per_step'])"
done
