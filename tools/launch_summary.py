"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launch_summary.py launches.csv [top] [kernel-prefix ...]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tot, cnt, seq = defaultdict(float), defaultdict(int), defaultdict(list)
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", "")) / 1e6
    except ValueError:
        continue
    name = r[ki].split("(")[0]
    tot[name] += v
    cnt[name] += 1
    seq[name].append(v)
T = sum(tot.values())
print(f"total serialized kernel time {T:.2f} ms over {sum(cnt.values())} launches")
print("# ms_total  share  launches  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:9.3f} {100 * v / T:5.1f}% {cnt[k]:6d}  {k}")
for pre in sys.argv[3:]:
    for k in seq:
        if k.startswith(pre):
            print(k, [round(x, 2) for x in seq[k]])
