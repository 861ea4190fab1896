#!/bin/bash
# NVLink party kernel, byte-granular direct stores to the peer (HB_P2P_BYTEDIRECT) vs shared-memory
# staging for widths whose packed group is not whole 32-bit words: w=6 +3 %, w=5 +2 %, w=22 -18 %
cd tools/micro
for w in 6 5 22; do for bd in 0 1; do echo "w=$w bytedirect=$bd $(./p2p_bench_bd${bd}_w$w 24 10 0 0 | grep "^{")"; done; done
