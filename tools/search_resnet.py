#!/usr/bin/env python
"""Per-group (k, m) windows for the ResNet private-inference benchmarks, chosen by the window search
(paper_2309_04875_b200/search.py = ringmpc search.py:159-334) over the GPU simulator.

Validation set: synthetic inputs of the benchmark shape; labels = the exact (full-window) model's
argmax, so "accuracy" is agreement with the unreduced network (random-init weights: there is no
dataset or checkpoint here).  Writes configs/<model>_windows_{eco,budget}.json (ReluConfig JSON +
accuracy, baseline, bits fraction, search trace) and configs/<model>_windows_w8.json, the benchmark's
8-bit windows: per group k from the lossless eco search (the window's top bit covers the group's
activation range, Theorem 1) and m = k - 8.  With random-init weights the exact model's argmax is
nearly constant, so the budget search's accuracy criterion cannot tell windows apart (it keeps the
smallest m or drops whole groups); the eco search's k does not depend on the labels.

    python tools/search_resnet.py resnet18 [--n 64] [--budget 1/8] [--widths 0,6,8]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2309_04875_b200 import models, search, simulator  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("model", choices=["resnet18", "resnet50"])
    p.add_argument("--n", type=int, default=64)
    p.add_argument("--budget", default="1/8")
    p.add_argument("--widths", default="0,6,8")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out-dir", default=os.path.join(ROOT, "configs"))
    p.add_argument("--eco-only", action="store_true", help="skip the budget search")
    a = p.parse_args()
    model = models.resnet18_cifar(0) if a.model == "resnet18" else models.resnet50(0)
    shape = (3, 32, 32) if a.model == "resnet18" else (3, 64, 64)
    x_val = np.random.default_rng(2024).uniform(0.0, 1.0, (a.n,) + shape)
    labels = np.argmax(simulator.plain_forward(model, x_val), axis=1)
    ranges = simulator.collect_activation_ranges(model, x_val)
    print(f"[search] {a.model}: activation ranges (bits) per group {ranges}", flush=True)
    out_dir = a.out_dir
    os.makedirs(out_dir, exist_ok=True)
    t = time.time()
    eco = search.search_eco(model, x_val, labels, seed=a.seed)
    print(f"[search] eco {time.time() - t:.1f}s {json.dumps(eco.to_json())}", flush=True)
    eco.save(os.path.join(out_dir, f"{a.model}_windows_eco.json"))
    w8 = {"groups": [{"k": w.k, "m": max(0, w.k - 8)} for w in eco.windows],
          "search": {"kind": "search_eco k per group, m = k - 8", "seed": a.seed,
                     "validation": f"{a.n} synthetic uniform[0,1) inputs of shape {shape}",
                     "activation_ranges": {str(g): v for g, v in ranges.items()}}}
    with open(os.path.join(out_dir, f"{a.model}_windows_w8.json"), "w") as fh:
        json.dump(w8, fh, indent=2)
    if a.eco_only:
        return
    t = time.time()
    widths = tuple(int(w) for w in a.widths.split(","))
    bud = search.search_budget(model, x_val, labels, a.budget, candidate_widths=widths, seed=a.seed)
    print(f"[search] budget {a.budget} {time.time() - t:.1f}s {json.dumps(bud.to_json())}", flush=True)
    res = bud.to_json()
    res["search"] = {"kind": "search_budget", "budget": a.budget, "candidate_widths": list(widths), "seed": a.seed,
                     "validation": f"{a.n} synthetic uniform[0,1) inputs of shape {shape}, labels = exact model argmax",
                     "activation_ranges": {str(g): v for g, v in ranges.items()}}
    with open(os.path.join(out_dir, f"{a.model}_windows_budget.json"), "w") as fh:
        json.dump(res, fh, indent=2)


if __name__ == "__main__":
    main()
