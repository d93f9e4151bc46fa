"""Per-kernel share of GPU time from an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/launch_summary.py profiles/r02/launches_r02g.csv > profiles/r02/launches_r02g_summary.txt
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ci = {h: i for i, h in enumerate(hdr)}
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[ci["Metric Name"]] != "gpu__time_duration.sum":
        continue
    unit = r[ci["Metric Unit"]]
    v = float(r[ci["Metric Value"]].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[unit]
    tot[r[ci["Kernel Name"]]] += v
    cnt[r[ci["Kernel Name"]]] += 1
all_us = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{cnt[k]:5d} {v / cnt[k]:12.1f} us/launch {100 * v / all_us:6.2f}%  {k[:110]}")
