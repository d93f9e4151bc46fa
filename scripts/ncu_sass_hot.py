"""Summarise an ncu --page source --csv (SASS view) export: warp-stall samples by instruction
and by stall reason, hottest instructions first (tuning helper)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
by_reason = Counter()
lines = []
for r in rows[2:]:
    try:
        v = float(r[ci["Warp Stall Sampling (All Samples)"]])
    except (ValueError, IndexError):
        continue
    tot += v
    rs = {h: float(r[ci[h]]) for h in stalls if r[ci[h]] not in ("", "0")}
    by_reason.update(rs)
    lines.append((v, r[ci["Address"]][-5:], r[ci["Source"]].strip()[:60], rs))
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in by_reason.most_common(10)))
lines.sort(key=lambda x: -x[0])
for v, a, s, rs in lines[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    top = ", ".join(f"{k[6:]} {x / v * 100:.0f}%" for k, x in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
    print(f"{v / tot * 100:5.1f}% {a} {s:60s} {top}")
