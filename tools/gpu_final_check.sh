#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 1500 python bench.py --sweep gpurun_out/sweep_r01.json --steps 20 --no-resnet > gpurun_out/sweep_stdout.log 2> gpurun_out/sweep_err.log; echo sweep rc=$?
python -c "
import json
rows=json.load(open('gpurun_out/sweep_r01.json'))
for r in rows: print(r['logn'], r['w'], r['cuda_graph'], '%.3e'%r['elems_per_s'], '%.4f'%r['ms_per_step'], '%.2f'%r['hbm_frac'], r['correct'])
"
