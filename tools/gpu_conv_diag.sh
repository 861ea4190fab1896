#!/bin/bash
# Layer1 conv timing under the HB_TC_DEBUG switches (0 normal, 1 no MMA, 2 no gathers, 3 neither, 4 stamps)
for d in 0 1 2 3 4; do HB_TC_DEBUG=$d timeout 300 python tools/diag_conv.py; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 2 -c 1 -o gpurun_out/prof_conv_l1 python tools/diag_conv.py > gpurun_out/ncu_conv_l1.log 2>&1; echo "ncu rc=$?"
