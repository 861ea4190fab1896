#!/bin/bash
# usage: gpu_ncu1.sh name "args for diag_tma1.py"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/$1 python tools/diag_tma1.py $2 > /dev/null 2>&1; echo rc=$?
