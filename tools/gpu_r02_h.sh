#!/bin/bash
# ring conv bounds: normal / no-MMA / no-load timings, phase stamps, ncu --set full of layer1 + layer3
mkdir -p gpurun_out
for d in 0 1 2 4; do HB_TC_DEBUG=$d timeout 300 python tools/diag_conv_bounds.py > gpurun_out/conv_bounds_d$d.json 2> gpurun_out/conv_bounds_err.log; echo "dbg=$d rc=$?"; cat gpurun_out/conv_bounds_d$d.json; echo; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_conv_l1_r02 python tools/diag_tma1.py 512 64 32 64 3 1 1 > /dev/null 2>&1; echo "ncu l1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_conv_l3_r02 python tools/diag_tma1.py 512 256 8 256 3 1 1 > /dev/null 2>&1; echo "ncu l3 rc=$?"
