#!/bin/bash
# 4-pass double-buffered N_T=128 conv: parity + bounds vs 2-pass
mkdir -p gpurun_out
HB_TMA_PASSES=4 timeout 900 python -m pytest tests/test_gpu_nn.py -q -p no:cacheprovider -x -k "conv or resnet or residual" > gpurun_out/gpu_tests_p4.log 2>&1; echo "pytest p4 rc=$?"; tail -2 gpurun_out/gpu_tests_p4.log
for p in 2 4; do HB_TMA_PASSES=$p HB_TC_DEBUG=4 timeout 300 python tools/diag_conv_bounds.py > gpurun_out/conv_p$p.json 2>/dev/null; echo "passes=$p"; python -c "
import json;d=json.load(open('gpurun_out/conv_p$p.json'))
for k,v in d.items():
    if k!='dbg': print(k, round(v['ms'],4), v['nt'], v.get('stamps_clk'))"; done
for p in 2 4; do HB_TMA_PASSES=$p timeout 300 python bench.py --workload resnet18 --steps 5 --warmup 3 > gpurun_out/rn18_p$p.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/rn18_p$p.json'));print('passes=$p rn18', d['value'], d['ms_per_step'])"; done
