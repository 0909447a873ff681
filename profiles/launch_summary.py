"""Per-kernel totals and shares from an ncu --csv launch list (gpu__time_duration.sum)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r[ui]]
    tot[r[ki]] += float(r[vi].replace(",", "")) * scale
    cnt[r[ki]] += 1
s = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{k:60s} launches={cnt[k]} total_ms={tot[k]:.3f} per_launch_ms={tot[k]/cnt[k]:.3f} share={100*tot[k]/s:.1f}%")
