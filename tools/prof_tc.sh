timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/rn18_tc_launches.csv python bench.py --workload resnet18 --steps 1 --warmup 0 --batch 128 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 2 -c 1 -o gpurun_out/prof_conv_tc python bench.py --workload resnet18 --steps 1 --warmup 0 --batch 128 > /dev/null 2>&1
ls -la gpurun_out/
