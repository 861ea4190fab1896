#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nn.py -q -p no:cacheprovider -k "lanes or run_local or wide" 2>&1 | tail -1
for l in 1 2 4; do for g in 148 120; do
  HB_LANES=$l HB_TMA_GRID=$g timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 > gpurun_out/rn18_l${l}_g$g.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rn18_l${l}_g$g.json'));print('lanes=$l grid=$g', round(d['value']), round(d['ms_per_step'],3), d['logits_check']['max_abs_diff_vs_plain_forward'])"
done; done
