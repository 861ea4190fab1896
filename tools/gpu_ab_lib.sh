#!/bin/bash
# A/B of the default library against paper_2309_04875_b200/lib_cs (same box, alternating): bench line value
mkdir -p gpurun_out; cp paper_2309_04875_b200/lib/libhbrelu.so /tmp/libhbrelu_base.so
for rep in 1 2; do for v in base cs; do
  if [ $v = cs ]; then cp paper_2309_04875_b200/lib_cs/libhbrelu.so paper_2309_04875_b200/lib/libhbrelu.so; else cp /tmp/libhbrelu_base.so paper_2309_04875_b200/lib/libhbrelu.so; fi
  for logn in 24 20 16; do
    timeout 300 python bench.py --logn $logn --steps 20 --no-e2e --no-cpu-baseline --no-resnet $( [ $logn -le 22 ] && echo --graph ) > gpurun_out/ab_${v}_$logn.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$logn.json'));print('$v', $logn, '%.4e' % d['value'], round(d['roofline']['frac'],4), d['correct'])"
  done
done; done
cp /tmp/libhbrelu_base.so paper_2309_04875_b200/lib/libhbrelu.so
