"""Summaries of an ncu report (development aid): key throughput metrics, stall
reasons, and an opcode histogram of the executed SASS with stall samples."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "launch__registers_per_thread"]
for k in keys:
    if k in h:
        print(f"{k:75s} {v[h.index(k)]} {r[1][h.index(k)]}")
st = [(float(v[i]), n) for i, n in enumerate(h) if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued")]
tot = sum(x for x, _ in st)
print("stall samples:", ", ".join(f"{n.split('stalled_')[1]} {x/tot*100:.0f}%" for x, n in sorted(st, reverse=True)[:10]))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]; rows = rows[2:]
    iS, iE, iW = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[iE]) for x in rows); totw = sum(int(x[iW]) for x in rows)
    c, s = Counter(), Counter()
    for x in rows:
        t = x[iS].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += int(x[iE]); s[op] += int(x[iW])
    print("warp instrs", tot)
    for op, n in c.most_common(22):
        print(f"  {op:10s} {n/tot*100:5.1f}% instr  {s[op]/totw*100:5.1f}% stall samples")
