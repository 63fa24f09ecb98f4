"""Golden outputs of the reference CLI (src/cli.py) for tests/test_cli.py.

Runs the reference `python -m mxq.cli` (imported from /root/reference in the
build container only) on a fixed list of command lines and records exit code,
stdout and the sha256 of every file it writes.  The GPU box uses the committed
tests/golden/cli/cli_golden.json.  usage: python tests/golden/make_golden_cli.py
"""
import hashlib, json, os, subprocess, sys, tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (name, argv, files-written) -- {d} is the scratch directory
CASES = [
    ("gen_a", ["gen", "--dist", "gaussian-outliers", "--shape", "64x256", "--seed", "3", "--out", "{d}/a.mxt"], ["a.mxt"]),
    ("gen_b", ["gen", "--dist", "student-t", "--shape", "48x256", "--seed", "5", "--out", "{d}/b.mxt"], ["b.mxt"]),
    ("quant_mbs_s", ["quantize", "--in", "{d}/a.mxt", "--scheme", "mbs-s", "--out", "{d}/a_mbs_s.mxq"], ["a_mbs_s.mxq"]),
    ("quant_mbs_d", ["quantize", "--in", "{d}/b.mxt", "--scheme", "mbs-d", "--out", "{d}/b_mbs_d.mxq"], ["b_mbs_d.mxq"]),
    ("quant_nvfp4", ["quantize", "--in", "{d}/a.mxt", "--scheme", "nvfp4", "--out", "{d}/a_nv.mxq"], ["a_nv.mxq"]),
    ("quant_ocp32", ["quantize", "--in", "{d}/a.mxt", "--scheme", "ocp32", "--out", "{d}/a_ocp.mxq"], ["a_ocp.mxq"]),
    ("dequant_mbs_s", ["dequantize", "--in", "{d}/a_mbs_s.mxq", "--out", "{d}/a_deq.mxt"], ["a_deq.mxt"]),
    ("qsnr_gen_csv", ["qsnr", "--scheme", "mbs-d", "--dist", "student-t", "--shape", "64x256", "--n", "2",
                      "--format", "csv"], []),
    ("qsnr_ref_json", ["qsnr", "--ref", "{d}/a.mxt", "--scheme", "mx16-oas", "--format", "json"], []),
    ("qsnr_lut_csv", ["qsnr", "--scheme", "mbs-d", "--mbs-mode", "lut", "--dist", "gaussian", "--shape", "32x256",
                      "--format", "csv"], []),
    ("sweep_csv", ["sweep", "--schemes", "mx16,mbs-s", "--macro-sizes", "64,128", "--n", "2", "--shape", "32x256",
                   "--format", "csv"], []),
    ("gemm_verify", ["gemm", "--a", "{d}/a.mxt", "--b", "{d}/b.mxt", "--scheme-a", "mbs-s", "--scheme-b", "mbs-d",
                     "--verify", "--out", "{d}/c.mxt"], ["c.mxt"]),
    ("roofline_json", ["roofline", "--format", "json"], []),
    ("roofline_csv", ["roofline", "--tm", "256", "--tn", "128", "--tk", "256", "--format", "csv"], []),
    ("lut_json", ["lut-dump", "--format", "json"], []),
    ("usage_error", ["qsnr", "--format", "csv"], []),
    ("data_error", ["gemm", "--a", "{d}/a.mxt", "--b", "{d}/a_deq_missing.mxt", "--scheme-a", "mx16",
                    "--scheme-b", "mx16"], []),
]


def run(cli_module, pythonpath, d):
    out = {}
    for name, argv, files in CASES:
        args = [a.replace("{d}", d) for a in argv]
        env = dict(os.environ, PYTHONPATH=pythonpath)
        r = subprocess.run([sys.executable, "-m", cli_module, *args], capture_output=True, text=True, env=env)
        rec = {"rc": r.returncode, "stdout": r.stdout if name not in ("lut_json",) else
               hashlib.sha256(r.stdout.encode()).hexdigest()}
        for f in files:
            p = os.path.join(d, f)
            rec[f] = hashlib.sha256(open(p, "rb").read()).hexdigest() if os.path.exists(p) else None
        out[name] = rec
    return out


if __name__ == "__main__":
    with tempfile.TemporaryDirectory() as d:
        res = run("mxq.cli", REF, d)
    json.dump(res, open(os.path.join(HERE, "cli", "cli_golden.json"), "w"), indent=1, sort_keys=True)
    print({k: v["rc"] for k, v in res.items()})
