#!/bin/bash
timeout 600 python tools/diag_tma.py 2>&1 | tail -12
HB_TC_DEBUG=1 timeout 600 python tools/diag_tma.py 2>&1 | tail -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_tma_l1b python tools/diag_tma1.py 512 64 32 64 3 1 1 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_tma_l4b python tools/diag_tma1.py 512 512 4 512 3 1 1 > /dev/null 2>&1; echo rc=$?
