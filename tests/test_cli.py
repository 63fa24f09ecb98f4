"""The GPU-backed CLI (paper_2603_08713_b200/cli.py) against the reference
CLI's recorded outputs (tests/golden/cli/cli_golden.json, written by
tests/golden/make_golden_cli.py from src/cli.py): exit codes, stdout of the
machine-readable formats, and the bytes of every container file written."""

import hashlib
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden_cli import CASES  # noqa: E402

from paper_2603_08713_b200 import cli  # noqa: E402

GOLDEN = json.load(open(os.path.join(HERE, "golden", "cli", "cli_golden.json")))
HOST_ONLY = ("gen_a", "gen_b", "roofline_json", "roofline_csv", "lut_json", "usage_error")
ORDER = [name for name, _, _ in CASES]


def _run(name, d, capsys):
    argv, files = next((a, f) for n, a, f in CASES if n == name)
    args = [x.replace("{d}", str(d)) for x in argv]
    try:
        rc = cli.main(args)
    except SystemExit as e:  # argparse usage errors exit from parse_args
        rc = e.code
    out = capsys.readouterr().out
    got = {"rc": rc, "stdout": out if name != "lut_json" else hashlib.sha256(out.encode()).hexdigest()}
    for f in files:
        p = os.path.join(str(d), f)
        got[f] = hashlib.sha256(open(p, "rb").read()).hexdigest() if os.path.exists(p) else None
    return got


@pytest.mark.parametrize("name", HOST_ONLY)
def test_cli_host_commands_match_reference(name, tmp_path, capsys):
    assert _run(name, tmp_path, capsys) == GOLDEN[name], name


@pytest.mark.gpu
def test_cli_pipeline_matches_reference(tmp_path, capsys):
    """Every recorded command in order (later ones read earlier outputs)."""
    for name in ORDER:
        assert _run(name, tmp_path, capsys) == GOLDEN[name], name


@pytest.mark.gpu
def test_cli_gemm_fast_reports_divergence(tmp_path, capsys):
    for name in ("gen_a", "gen_b"):
        _run(name, tmp_path, capsys)
    rc = cli.main(["gemm", "--a", f"{tmp_path}/a.mxt", "--b", f"{tmp_path}/b.mxt", "--scheme-a", "mbs-s",
                   "--scheme-b", "mbs-d", "--fast"])
    assert rc == 0 and capsys.readouterr().out.startswith("shape: 64x48")
