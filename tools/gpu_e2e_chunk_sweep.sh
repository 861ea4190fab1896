#!/bin/bash
# e2e (pinned host shares in/out) vs pipeline chunk size and one- vs two-row copies (HB_PIPE_2D=0/1)
mkdir -p gpurun_out
for c in ${CHUNKS:-19 20 21 22}; do for d2 in ${TWOD:-1}; do
  HB_PIPE_2D=$d2 HB_PIPE_CHUNK=$((1<<c)) timeout 300 python bench.py --steps 10 --warmup 3 --no-resnet --no-cpu-baseline > gpurun_out/e2e_c${c}_2d$d2.json 2>gpurun_out/e2e_c${c}_2d$d2.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_c${c}_2d$d2.json'));print('chunk 2^$c two-row=$d2', d['e2e']['value'], d['correct'])"
  grep "per-step" gpurun_out/e2e_c${c}_2d$d2.err
done; done
