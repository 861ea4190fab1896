#!/usr/bin/env python
"""Summarise ncu captures for profiles/.

  python tools/ncu_summary.py full  <report.ncu-rep> <key> [--out profiles/ncu_summary.json]
      key metrics of the (first) kernel in a `--set full` capture; merged into the
      JSON under `key` (bench.py reads `dram_bytes_per_launch` from it as `traffic`).
  python tools/ncu_summary.py launches <launches.csv>
      per-kernel share of device time from a `--metrics gpu__time_duration.sum` list.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEEP = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "lts__t_bytes.sum",
    "l1tex__t_bytes.sum",
    "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
]


def _num(v: str) -> float:
    return float(v.replace(",", ""))


def _scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
            "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1.0)


def full(report: str, key: str, out: str = "profiles/ncu_summary.json") -> dict:
    if report.endswith(".csv"):  # a `--page raw --csv` export made next to the capture
        with open(report) as fh:
            txt = fh.read()
    else:
        txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, val = rows[0], rows[1], rows[2]
    m = {}
    for i, h in enumerate(hdr):
        if h in KEEP:
            try:
                m[h] = {"value": _num(val[i]), "unit": units[i]}
            except ValueError:
                m[h] = {"value": val[i], "unit": units[i]}
        if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                if _num(val[i]) > 0.1:
                    m.setdefault("stalls", {})[h.split("stalled_")[1].split("_per_issue")[0]] = round(_num(val[i]), 2)
            except ValueError:
                pass
    name = val[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    rd = m["dram__bytes_read.sum"]["value"] * _scale(m["dram__bytes_read.sum"]["unit"])
    wr = m["dram__bytes_write.sum"]["value"] * _scale(m["dram__bytes_write.sum"]["unit"])
    dur = m["gpu__time_duration.sum"]["value"] * _scale(m["gpu__time_duration.sum"]["unit"])
    summ = {"kernel": name, "report": report, "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
            "dram_write_bytes": wr, "duration_s_cold": dur, "dram_GBps_cold": (rd + wr) / dur / 1e9, "metrics": m}
    try:
        with open(out) as fh:
            allm = json.load(fh)
    except (OSError, ValueError):
        allm = {}
    allm[key] = summ
    with open(out, "w") as fh:
        json.dump(allm, fh, indent=1, sort_keys=True)
    return summ


def launches(path: str) -> list:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if r[mi] == "gpu__time_duration.sum":
            k = r[ki].split("(")[0]
            tot[k] += _num(r[vi]) * _scale(r[ui])
            cnt[k] += 1
    s = sum(tot.values())
    return [(k, cnt[k], t, t / s) for k, t in sorted(tot.items(), key=lambda x: -x[1])]


if __name__ == "__main__":
    if sys.argv[1] == "full":
        r = full(sys.argv[2], sys.argv[3], *(sys.argv[4:5]))
        print(json.dumps({k: v for k, v in r.items() if k != "metrics"}, indent=1))
        print(json.dumps(r["metrics"].get("stalls", {}), indent=1))
    else:
        for k, c, t, f in launches(sys.argv[2]):
            print(f"{f * 100:6.2f}%  {t * 1e3:10.3f} ms  {c:5d}x  {k}")
