#!/bin/bash
# NVLink party kernel: 7 / 8 CTAs per SM
cd tools/micro
for w in 6 8 16 32; do for mb in 7 8; do
  r=$(timeout 60 ./p2p_bench_rp0_w${w}_b${mb} 24 10 0 0 | grep '^{')
  echo "w=$w minb=$mb $r"
done; done
