"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals over
the last `per_step` launches (one step) and each kernel's share of that step."""
import csv, sys, collections

path = sys.argv[1]
per_step = int(sys.argv[2]) if len(sys.argv) > 2 else 34
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
step = data[-per_step:]
agg = collections.OrderedDict()
for d in step:
    n = d["Kernel Name"].split("(")[0][:56]
    agg.setdefault(n, []).append(float(d["Metric Value"]) / 1000.0)
tot = sum(sum(v) for v in agg.values())
print(f"{len(data)} launches captured; last {per_step} = one step; serialised kernel time {tot:.1f} us")
for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{n:56s} n={len(v):2d} total {sum(v):8.1f} us  share {sum(v)/tot:6.1%}  ({', '.join(f'{x:.1f}' for x in v)})")
