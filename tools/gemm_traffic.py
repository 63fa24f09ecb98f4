"""Assemble profiles/gemm_traffic.json from an `ncu --set full` report of the
four MBS-H layer GEMMs (tools/profile_layers.py): DRAM bytes and duration per
launch next to the algorithmic bytes.  usage: gemm_traffic.py report.ncu-rep"""
import csv, json, subprocess, sys

LAYERS = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
M = 4096
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
recs = []
for r, (name, n, k) in zip(rows[2:], LAYERS):
    dur = float(r[col["gpu__time_duration.sum"]])
    unit = rows[1][col["gpu__time_duration.sum"]]
    us = dur / 1000.0 if unit == "nsecond" or unit == "ns" else dur
    rd = float(r[col["dram__bytes_read.sum"]]) * (1e6 if rows[1][col["dram__bytes_read.sum"]] == "Mbyte" else 1.0)
    wr_u = rows[1][col["dram__bytes_write.sum"]]
    wr = float(r[col["dram__bytes_write.sum"]]) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9}.get(wr_u, 1.0)
    if rows[1][col["dram__bytes_read.sum"]] == "Gbyte":
        rd = float(r[col["dram__bytes_read.sum"]]) * 1e9
    alg = (M + n) * k * (0.5 + 1 / 16) + (M + n) * ((k + 127) // 128) * 4 + M * n * 2
    recs.append({"layer": name, "shape": [M, n, k], "ncu_us": round(us, 1), "dram_bytes": rd + wr,
                 "algorithmic_bytes": float(alg), "tflops_ncu": round(2 * M * n * k / (us * 1e-6) / 1e12, 1)})
mean = lambda key: sum(x[key] for x in recs) / len(recs)
print(json.dumps({"mbs_h_bytes_per_launch": mean("dram_bytes"), "algorithmic_bytes_per_launch": mean("algorithmic_bytes"),
                  "layers": recs,
                  "source": "ncu --set full, second launch of each bench layer GEMM (tools/profile_layers.py), "
                            "dram__bytes_read.sum + dram__bytes_write.sum",
                  "note": "per launch, averaged over the 4 Llama-3-8B layer launches (M=4096) like bench.py's achieved; "
                          "algorithmic = FP4 codes + block-16 scales + f32 sigma per macro for A and B + bf16 C"},
                 indent=1))
