#!/bin/bash
# P2P party kernel: N=1 two-stream bench (both parties on one device), and the N=2 code path as
# two ranks on the one GPU (gloo group for the IPC handle exchange; kernels time-slice).
timeout 600 python bench.py --path p2p --steps 20 --no-cpu-baseline --no-resnet > gpurun_out/bench_p2p.json 2> gpurun_out/bench_p2p_err.log; echo "p2p rc=$?"; tail -2 gpurun_out/bench_p2p_err.log
python -c "import json; d=json.load(open('gpurun_out/bench_p2p.json')); print(d['value'], d['roofline']['frac'], d['correct'])"
for n in 20 24; do timeout 600 python bench.py --path p2p --logn $n --k 64 --m 0 --steps 10 --no-cpu-baseline --no-resnet 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('w64 logn', $n, d['value'], d['roofline']['frac'], d['correct'])"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 1 --logn 18 --backend gloo > gpurun_out/multi_p2p.json 2> gpurun_out/multi_p2p_err.log; echo "multi rc=$?"; tail -3 gpurun_out/multi_p2p_err.log; cat gpurun_out/multi_p2p.json
