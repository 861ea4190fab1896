# A/B the fused pair kernel variants on the default workload and a width sweep
for lib in "" "paper_2309_04875_b200/lib/exp_tp32/libhbrelu.so" "paper_2309_04875_b200/lib/exp_tp64m6/libhbrelu.so"; do
  for kk in "22 14" "64 0" "22 16"; do set -- $kk
    HB_LIB_PATH=$lib timeout 200 python bench.py --steps 20 --warmup 3 --k $1 --m $2 --no-e2e --no-cpu-baseline --triple-gb 24 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lib=${lib:-default}', d['config']['window'], round(d['value']/1e9,2), 'Gelem/s', round(d['roofline']['frac'],3), d['correct'])"
  done
done
