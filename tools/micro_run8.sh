#!/bin/bash
# NVLink party kernel: threads per CTA (one release per tile-round per CTA) x CTAs per SM, both flag scopes
cd tools/micro
for b in p2p_bench_tp*; do for sys in 1 0; do echo "$b sys=$sys $(timeout 60 ./$b 24 10 0 $sys | grep '^{')"; done; done
