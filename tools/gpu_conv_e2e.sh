timeout 300 python -m pytest tests/test_gpu_nn.py -q -x -p no:cacheprovider 2>&1 | tail -2
for impl in tc cublaslt; do
  HB_RING_GEMM=$impl timeout 300 python bench.py --workload resnet18 --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$impl', round(d['value']), 'samples/s', round(d['ms_per_step'],2), 'ms')"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-resnet 2>gpurun_out/b6_err.log > gpurun_out/bench6.json; grep e2e gpurun_out/b6_err.log
python -c "import json; d=json.load(open('gpurun_out/bench6.json')); print(d['value'], d['e2e']['value'])"
