#!/bin/bash
# Round-1 evidence for profiles/: ReLU launch list, ResNet18 launch list, --set full of the conv kernels.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_r01.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-resnet > /dev/null 2>&1; echo relu-launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_rn18_r01.csv python bench.py --workload resnet18 --steps 1 --warmup 1 > /dev/null 2>&1; echo rn18-launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_conv_tma_l1_r01 python tools/diag_tma1.py 512 64 32 64 3 1 1 > /dev/null 2>&1; echo l1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_conv_tma_l4_r01 python tools/diag_tma1.py 512 512 4 512 3 1 1 > /dev/null 2>&1; echo l4 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_limbs_nhwc -s 2 -c 1 -o gpurun_out/prof_limbs_r01 python tools/diag_tma1.py 512 64 32 64 3 1 1 > /dev/null 2>&1; echo limbs rc=$?
