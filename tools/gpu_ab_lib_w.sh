#!/bin/bash
# A/B of the default library against lib_<variant> at 2^24 for given windows "k:m" (same box, alternating)
# usage: bash tools/gpu_ab_lib_w.sh <variant> <k:m> [<k:m> ...]
v=$1; shift
mkdir -p gpurun_out; cp paper_2309_04875_b200/lib/libhbrelu.so /tmp/libhbrelu_base.so
for rep in 1 2; do for lib in base $v; do
  if [ $lib = base ]; then cp /tmp/libhbrelu_base.so paper_2309_04875_b200/lib/libhbrelu.so
  else cp paper_2309_04875_b200/lib_$lib/libhbrelu.so paper_2309_04875_b200/lib/libhbrelu.so; fi
  for km in "$@"; do k=${km%%:*}; m=${km##*:}
    timeout 300 python bench.py --k $k --m $m --steps 20 --no-e2e --no-cpu-baseline --no-resnet > gpurun_out/abw_${lib}_$k_$m.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abw_${lib}_$k_$m.json'));print('$lib', 'w=$(( k - m ))', '%.4e' % d['value'], round(d['roofline']['frac'],4), d['correct'])"
  done
done; done
cp /tmp/libhbrelu_base.so paper_2309_04875_b200/lib/libhbrelu.so
