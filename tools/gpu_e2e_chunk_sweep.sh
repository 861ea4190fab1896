mkdir -p gpurun_out
for c in ${CHUNKS:-19 20 21 22}; do
  HB_PIPE_CHUNK=$((1<<c)) timeout 300 python bench.py --steps 10 --warmup 3 --no-resnet --no-cpu-baseline > gpurun_out/e2e_c$c.json 2>gpurun_out/e2e_c$c.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_c$c.json'));print('chunk 2^$c', d['e2e']['value'], d['correct'])"
  grep "per-step" gpurun_out/e2e_c$c.err
done
