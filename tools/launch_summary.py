"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    name = re.sub(r"\(.*", "", r[4]).replace("void ", "")
    tot[name] += float(r[14]) / 1000.0
    cnt[name] += 1
allt = sum(tot.values())
print(f"{len(rows)} launches, {allt / 1000:.2f} ms of kernel time (cold-cache, serialised under ncu)\n")
print("| kernel | launches | total ms | share | avg us |")
print("|---|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| `{k}` | {cnt[k]} | {tot[k] / 1000:.3f} | {tot[k] / allt:.3f} | {tot[k] / cnt[k]:.1f} |")
