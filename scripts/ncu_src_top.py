"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur); continue
    if r and r[0] == "Address":
        cur["h"] = r; continue
    if cur is not None and r:
        cur["rows"].append(r)
for b in blocks:
    h = b["h"]; si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source")
    def f(x):
        try: return float(x)
        except ValueError: return 0.0
    tot = sum(f(r[si]) for r in b["rows"])
    print("==", b["name"][:100], "samples", tot)
    for r in sorted(b["rows"], key=lambda r: -f(r[si]))[:n]:
        print(f"{f(r[si]):8.0f} {100*f(r[si])/max(tot,1):5.1f}%  {r[0]}  {r[src][:100]}")
