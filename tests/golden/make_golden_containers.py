"""MXQ1 / MXT1 container fixtures written by the REAL reference
(``/root/reference/pkg/src/mxq/tensorio.py``) for tests/test_tensorio.py.

For each variant, a small tensor (the reference's own test shapes and seeds,
tests/test_tensorio.py:131-251, plus a 2-macro MBS case) is quantized with the
reference and saved with its ``save_quant``; the f32 input is saved with its
``save_tensor``.  The GPU tests quantize the same input on the device, save it
with ``paper_2603_08713_b200.tensorio.save_quant`` and require the file to be
byte-identical; the CPU tests parse these files with the pure-host reader.

Run:  python tests/golden/make_golden_containers.py   (needs /root/reference)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "containers")
sys.path.insert(0, "/root/reference/pkg/src")

from mxq import SchemeConfig, Variant, quantize_tensor  # noqa: E402
from mxq.tensorio import save_quant, save_tensor  # noqa: E402

CASES = [
    ("t4_6x256", lambda: np.random.Generator(np.random.PCG64(301)).standard_t(4, (6, 256)).astype(np.float32)),
    ("partial_3x208", lambda: np.random.Generator(np.random.PCG64(305)).standard_normal((3, 208)).astype(np.float32)),
    ("outliers_5x384", lambda: (np.random.Generator(np.random.PCG64(306)).standard_normal((5, 384))
                                * np.where(np.random.Generator(np.random.PCG64(307)).random((5, 384)) < 0.02,
                                           100.0, 1.0)).astype(np.float32)),
]

meta = {}
os.makedirs(HERE, exist_ok=True)
for name, gen in CASES:
    t = gen()
    save_tensor(t, os.path.join(HERE, f"{name}.mxt"))
    for v in Variant:
        if name == "partial_3x208" and v is Variant.OCP32:
            continue  # 208 is not a multiple of 32
        q = quantize_tensor(t, SchemeConfig(v))
        fn = f"{name}.{v.value}.mxq"
        save_quant(q, os.path.join(HERE, fn))
        meta[fn] = {"input": f"{name}.mxt", "variant": v.value, "bytes": os.path.getsize(os.path.join(HERE, fn))}
json.dump(meta, open(os.path.join(HERE, "index.json"), "w"), indent=1, sort_keys=True)
print(len(meta), "containers")
