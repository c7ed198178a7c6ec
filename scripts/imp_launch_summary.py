"""Per-kernel device time of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    n = r[4].split("(")[0][-48:]
    v, u = float(r[-1].replace(",", "")), r[-2]
    tot[n] += v / 1000 if u == "ns" else (v if u == "us" else v * 1000)
    cnt[n] += 1
print(f"launches {len(rows) // steps} per step, device time {sum(tot.values()) / steps / 1000:.1f} ms per step")
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{v / steps:10.0f} us {cnt[n] // steps:6d}  {n}")
