timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rn18_b512_launches.csv python bench.py --workload resnet18 --batch 512 --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/rn18_b512_launches.csv 2>/dev/null | head -14
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 2 -c 1 -o gpurun_out/prof_conv_ws python bench.py --workload resnet18 --batch 512 --steps 1 --warmup 0 > /dev/null 2>&1
ls gpurun_out | grep prof_conv_ws
