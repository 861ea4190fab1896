#!/bin/bash
# NVLink party kernel (both parties on one GPU) over the (n, w) sweep at both flag scopes, layers up to
# 2^22 replayed as one CUDA graph (device-resident flag sequence)
mkdir -p gpurun_out
for scope in gpu sys; do
  timeout 1500 python bench.py --path p2p --p2p-scope $scope --sweep gpurun_out/sweep_p2p_graph_$scope.json --steps 20 --no-resnet > /dev/null 2> gpurun_out/sweep_p2p_graph_$scope.err
  echo "scope $scope rc=$?"
done
python - <<'PY'
import json
for scope in ("gpu", "sys"):
    try:
        rows = json.load(open(f"gpurun_out/sweep_p2p_graph_{scope}.json"))
    except Exception as e:
        print(scope, "missing", e); continue
    for r in rows:
        print(scope, r["logn"], r["w"], f'{r["elems_per_s"]:.3e}', round(r["frac_vs_survey_H"], 3), r["correct"], r["cuda_graph"])
PY
