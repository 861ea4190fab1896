timeout 300 python -m pytest tests/test_gpu_nn.py -q -x -p no:cacheprovider 2>&1 | tail -15
for impl in tc cublaslt; do
  HB_RING_GEMM=$impl timeout 300 python bench.py --workload resnet18 --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$impl', round(d['value']), 'samples/s', round(d['ms_per_step'],2), 'ms')"
done
