#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nn.py -q -p no:cacheprovider -x -k "nhwc or permute or run_local or wide or residual" 2>&1 | tail -3
for o in "" "--no-nhwc"; do
  timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 $o > gpurun_out/rn18.json 2> gpurun_out/rn18_err.log; echo "rc=$?"; tail -2 gpurun_out/rn18_err.log | cut -c1-300
  python -c "import json;d=json.load(open('gpurun_out/rn18.json'));print('$o', round(d['value']), round(d['ms_per_step'],3), d['config']['activation_layout'][:4], d['logits_check']['max_abs_diff_vs_plain_forward'])"
done
