#!/bin/bash
# A/B of two builds of the NVLink party kernel (tools/micro/p2pab_<old|new>_w<W>), same box, alternating
for rep in 1 2; do for w in 8 64; do for sys in 0 1; do for v in old new; do
  echo "$v w=$w sys=$sys $(timeout 120 ./tools/micro/p2pab_${v}_w$w 24 20 0 $sys | grep '^{' | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("%.3e" % d["elems_per_s"])')"
done; done; done; done
