#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_tma_l1 python tools/diag_tma1.py 512 64 32 64 3 1 1 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_tma_l4 python tools/diag_tma1.py 512 512 4 512 3 1 1 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_limbs_nhwc -s 2 -c 1 -o gpurun_out/prof_limbs_l1 python tools/diag_tma1.py 512 64 32 64 3 1 1 > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_launches2.csv python bench.py --workload resnet18 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
