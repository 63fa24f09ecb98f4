"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into
per-kernel shares (cold-cache serialised times: compare shares, not
absolutes).  usage: summarize_launches.py launches.csv [header-line ...]"""
import csv, re, sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14]
rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]  # skip the program's own output
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r[ki]).replace("void ", "").strip()
    tot[name] += float(r[vi].replace(",", "")) / 1e6  # ns -> ms
    cnt[name] += 1
T = sum(tot.values())
for h in sys.argv[2:]:
    print("# " + h)
print(f"# total {T:.2f} ms over {sum(cnt.values())} launches\n")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100 * v / T:6.2f}%  {v:9.3f} ms  {cnt[k]:5d}x  {k[:150]}")
