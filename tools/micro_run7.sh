#!/bin/bash
# NVLink party kernel: CTAs per SM x flag scope (sys = the two-GPU protocol), per width
cd tools/micro
for w in 8 16 32 64; do for mb in 4 5 6 7 8; do for sys in 1 0; do
  echo "w=$w minb=$mb sys=$sys $(timeout 60 ./p2p_bench_m_w${w}_b${mb} 24 10 0 $sys | grep '^{')"
done; done; done
