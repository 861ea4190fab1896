"""Group an ncu launch list (gpu__time_duration) of one bench forward by kernel: python tools/launch_breakdown.py csv [marker]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[[i for i, r in enumerate(rows) if r and r[0] == "ID"][0]]
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
seq = [(d["Kernel Name"], float(d["Metric Value"]) / 1e3) for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
marker = sys.argv[2] if len(sys.argv) > 2 else "conv"
idx = [i for i, s in enumerate(seq) if marker in s[0]]
fw = seq[idx[len(idx) // 2]:]  # last forward (the bench ran warmup + 1 step)
agg = collections.defaultdict(lambda: [0, 0.0])
for n, t in fw:
    k = n.split("(")[0][:50]
    agg[k][0] += 1
    agg[k][1] += t
tot = sum(t for _, t in fw)
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}% {c:4d}  {k}")
print(f"total {tot / 1e3:.3f} ms")
