#!/bin/bash
# A/B of the default library against alternative builds paper_2309_04875_b200/lib_<variant>/libhbrelu.so
# (same box, alternating): the bench line at 2^24 and graph-replayed 2^20 / 2^16 layers.
# usage: bash tools/gpu_ab_lib.sh <variant> [<variant> ...]
mkdir -p gpurun_out; cp paper_2309_04875_b200/lib/libhbrelu.so /tmp/libhbrelu_base.so
for rep in 1 2; do for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/libhbrelu_base.so paper_2309_04875_b200/lib/libhbrelu.so
  else cp paper_2309_04875_b200/lib_$v/libhbrelu.so paper_2309_04875_b200/lib/libhbrelu.so; fi
  for logn in 24 20 16; do
    timeout 300 python bench.py --logn $logn --steps 20 --no-e2e --no-cpu-baseline --no-resnet $( [ $logn -le 22 ] && echo --graph ) > gpurun_out/ab_${v}_$logn.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$logn.json'));print('$v', $logn, '%.4e' % d['value'], round(d['roofline']['frac'],4), d['correct'])"
  done
done; done
cp /tmp/libhbrelu_base.so paper_2309_04875_b200/lib/libhbrelu.so
