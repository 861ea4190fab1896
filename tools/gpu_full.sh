timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>gpurun_out/b5_err.log > gpurun_out/bench5.json; tail -2 gpurun_out/b5_err.log
python -c "import json; d=json.load(open('gpurun_out/bench5.json')); print(d['value'], d['roofline']['frac'], d['e2e'], d['resnet18']['value'])"
