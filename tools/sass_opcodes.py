"""Per-kernel SASS opcode counts of the product library (the instructions
that prove tcgen05 / TMA / hardware FP4 conversion are on the path):
UTCOMMA / UTCHMMA (tcgen05.mma), UTCCP (tcgen05.cp), LDTM / STTM (tcgen05.ld /
st), UTMALDG (TMA tensor loads), UBLKCP (bulk copies), F2FP.*E2M1 / E4M3
(hardware FP4 / FP8 converters), LDG.*256 (256-bit loads), FFMA2 / FMUL2
(packed FP32).  usage: python tools/sass_opcodes.py [objdir]"""
import collections, glob, os, re, subprocess, sys

objdir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_2603_08713_b200", "_lib")
KEYS = ["UTCOMMA", "UTCHMMA", "UTCQMMA", "UTCCP", "LDTM", "STTM", "UTMALDG", "UBLKCP", "F2FP.SATFINITE.E2M1",
        "F2FP.SATFINITE.E4M3", "LDG.E.NA.ENL2.256", "LDG.E.256", "FFMA2", "FMUL2", "SYNCS.ARRIVE", "DFMA"]
for obj in sorted(glob.glob(os.path.join(objdir, "*.o"))):
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, counts = None, collections.defaultdict(collections.Counter)
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        if fn and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            ins = line.split("*/", 1)[1].strip()
            ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
            for k in KEYS:
                if ins.startswith(k):
                    counts[fn][k] += 1
    if not counts:
        continue
    print(f"## {os.path.basename(obj)}")
    for f, c in counts.items():
        dem = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*$", "", dem)
        print(f"  {dem[:110]}")
        print("     " + ", ".join(f"{k} {v}" for k, v in sorted(c.items())))
