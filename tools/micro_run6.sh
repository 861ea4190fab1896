#!/bin/bash
# NVLink party kernel at SYSTEM-scope flags (what two GPUs use): groups per thread C x CTAs per SM, w=8
cd tools/micro
for c in 4 8 16; do for mb in 3 4 5; do for sys in 1 0; do
  echo "C=$c minb=$mb sys=$sys $(timeout 60 ./p2p_bench_sys_w8_b${mb}_c${c} 24 10 0 $sys | grep '^{')"
done; done; done
