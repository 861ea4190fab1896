#!/bin/bash
# P2P party kernel variants (both parties on one GPU, gpu-scope flags): width x L2 prefetch x min CTAs/SM x groups/thread
cd tools/micro
for w in 6 16 32; do for pf in 0 1; do for mb in 3 4 5 6; do for c in 4 8; do
  r=$(timeout 60 ./p2p_bench_w${w}_pf${pf}_b${mb}_c${c} 24 10 0 0 | grep '^{')
  echo "w=$w pf=$pf minb=$mb C=$c $r"
done; done; done; done
