set -x
timeout 400 python bench.py 2>gpurun_out/bench3_err.log > gpurun_out/bench3.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_r01.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_relu_pair -s 3 -c 1 -o gpurun_out/prof_pair_w8_r01 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 2 --logn 20 --backend gloo > gpurun_out/multi_gloo.json 2>gpurun_out/multi_gloo_err.log
tail -3 gpurun_out/multi_gloo_err.log
cat gpurun_out/multi_gloo.json
