"""C1 over seeds 0..7 (SURVEY section 8 d, config 1: "seeds 0..7"): QSNR dB,
flush rate and a sha256 of every quantized field for the six variants of the
4096x4096 gaussian+outlier tensor (bf16 RNE), computed by the REAL reference
package (``/root/reference/pkg/src/mxq``, src/metrics.py:127-182, 210-261)
in the build container and committed as ``qsnr_seeds.json`` (the reference
does not travel to the GPU box).  bench.py's C1 block and
tests/test_gpu_quantize.py::test_config1_all_seeds compare against it.

Run:  python tests/golden/make_qsnr_seeds.py   (needs /root/reference; ~6 min,
most of it the reference's MBS-D search)."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mxq import (  # noqa: E402  (the reference)
    GeneratorSpec, SchemeConfig, Variant, dequantize_tensor, flush_to_zero_rate, generate_tensor,
    qsnr_tensor, quantize_tensor,
)

sys.path.insert(0, HERE)
from make_golden import bf16, q_fields  # noqa: E402

SEEDS = range(8)


def mean_db(out) -> dict:
    """The reference's mean_qsnr: a running sum of the per-seed dB values over
    seeds 0..7, divided by n (src/metrics.py:228-246)."""
    res = {}
    for v in Variant:
        acc = 0.0
        for s in SEEDS:
            acc += out["seeds"][str(s)][v.value]["qsnr_db"]
        res[v.value] = acc / len(SEEDS)
    return res


def main() -> None:
    out = {"shape": [4096, 4096], "generator": "gaussian_with_outliers", "dtype": "bf16 RNE", "seeds": {}}
    for s in SEEDS:
        t = bf16(generate_tensor(GeneratorSpec("gaussian_with_outliers", (4096, 4096), seed=s)))
        row = {"sha256_bf16": hashlib.sha256(t.tobytes()).hexdigest()}
        for v in Variant:
            q = quantize_tensor(t, SchemeConfig(v))
            r = qsnr_tensor(t, dequantize_tensor(q))
            h = hashlib.sha256()
            for f, arr in sorted(q_fields(q).items()):
                h.update(f.encode())
                h.update(np.ascontiguousarray(arr).tobytes())
            row[v.value] = {"qsnr_db": r.qsnr_db, "flush": flush_to_zero_rate(t, q), "sha256": h.hexdigest()}
        out["seeds"][str(s)] = row
        print(s, {v: round(row[v]["qsnr_db"], 4) for v in row if v != "sha256_bf16"}, flush=True)
    out["mean_qsnr_db"] = mean_db(out)
    with open(os.path.join(HERE, "qsnr_seeds.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
