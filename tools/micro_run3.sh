#!/bin/bash
# NVLink party kernel: next-level inputs loaded into registers before each exchange (HB_P2P_REGPF) vs not
cd tools/micro
for w in 6 8 16 32; do for mb in 4 5 6; do for rp in 0 1; do
  r=$(timeout 60 ./p2p_bench_rp${rp}_w${w}_b${mb} 24 10 0 0 | grep '^{')
  echo "w=$w minb=$mb regpf=$rp $r"
done; done; done
