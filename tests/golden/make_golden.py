"""Generate the golden fixtures under tests/golden/ by running the REAL
reference package (``/root/reference/pkg/src/mxq``) in the build container.

The reference is pure Python + numpy and cannot travel to the GPU box, so its
outputs are committed here as small ``.npz`` files.  The oracle
(``oracle/mxq_oracle.py``) is pinned against them by
``tests/test_oracle_golden.py`` and the CUDA path by ``tests/test_gpu_*.py``.

Run:  python tests/golden/make_golden.py   (needs /root/reference; ~1 min,
plus ~40 s for the 4096x4096 MBS-D config-1 QSNR row).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import mxq  # noqa: E402  (the reference)
from mxq import (  # noqa: E402
    CandidateSet, GeneratorSpec, SchemeConfig, TileConfig, Variant,
    dequantize_tensor, flush_to_zero_rate, generate_tensor, matmul_quantized,
    qsnr_tensor, quantize_tensor,
)
from mxq.formats import encode_e2m1_array, encode_e4m3_array  # noqa: E402


def bf16(t):
    u = np.ascontiguousarray(t, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def tensors():
    rng = np.random.Generator(np.random.PCG64(9001))
    out = {
        "t4_48x384": generate_tensor(GeneratorSpec("student_t", (48, 384), seed=71)),
        "gwo_32x256": generate_tensor(GeneratorSpec("gaussian_with_outliers", (32, 256), seed=72)),
        "gauss_6x208": rng.standard_normal((6, 208)).astype(np.float32),
        "gauss_5x2880": rng.standard_normal((5, 2880)).astype(np.float32),
        "tiny_8x64": (rng.standard_normal((8, 64)) * 2.0 ** -135).astype(np.float32),
        "subn_mix_8x64": (rng.standard_normal((8, 64)) * np.exp2(rng.integers(-149, -110, (8, 1)))).astype(np.float32),
        "huge_8x64": (rng.standard_normal((8, 64)) * 2.0 ** 120).astype(np.float32),
        "zeros_4x64": np.zeros((4, 64), np.float32),
        "bf16_gwo_64x512": bf16(generate_tensor(GeneratorSpec("gaussian_with_outliers", (64, 512), seed=0))),
        "wide_exp_16x512": (rng.standard_normal((16, 512)) * np.exp2(rng.integers(-30, 30, (16, 32))).repeat(16, 1)).astype(np.float32),
    }
    grid = np.array([0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    vals = rng.choice(np.concatenate([grid, -grid]), size=(8, 128))
    out["grid_8x128"] = (vals * np.exp2(rng.integers(-8, 8, (8, 8))).repeat(16, 1)).astype(np.float32)
    # saturation-window / OAS trigger sweep: block maxima in (3, 3.5] and 1.75*2^k
    sw = np.zeros((64, 16), np.float32)
    sw[:, 0] = np.float32(3.0 + 0.5 * np.arange(1, 65) / 64.0)
    sw[:, 1] = rng.uniform(-3, 3, 64).astype(np.float32)
    out["oas_window_64x16"] = sw
    return out


def q_fields(q):
    d = {"codes": q.codes}
    for f in ("block_scales", "e4m3_scales", "mbs_mantissas"):
        v = getattr(q, f)
        if v is not None:
            d[f] = v
    if q.tensor_scale is not None:
        d["tensor_scale"] = np.array([q.tensor_scale], np.float64)
    return d


def main():
    arrays = {}
    meta = {"reference": "/root/reference/pkg/src/mxq", "numpy": np.__version__, "cases": []}

    # ---- codecs ---------------------------------------------------------
    rng = np.random.Generator(np.random.PCG64(11))
    e2 = np.concatenate([
        np.array([0.0, -0.0, 0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, -2.5, -0.25, 6.6, -100.0,
                  -0.1, 6.0, 7.0, 5.999, 0.2499, 0.2501, 4.5, 3.0, 1e-30, -1e-30]),
        np.nextafter(np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0]), 0),
        np.nextafter(np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0]), 10),
        rng.uniform(-7.0, 7.0, 20000),
    ])
    arrays["codec/e2m1_in"] = e2
    arrays["codec/e2m1_out"] = encode_e2m1_array(e2, saturate=True)
    tab = mxq.formats.E4M3_TABLE
    fin = tab[np.isfinite(tab)]
    mids = (np.sort(np.unique(np.abs(fin)))[:-1] + np.sort(np.unique(np.abs(fin)))[1:]) / 2
    e4 = np.concatenate([fin, mids, -mids, np.array([500.0, 448.0, 1e-9, 0.0, -0.0]),
                         rng.uniform(0, 460, 20000), np.exp2(rng.uniform(-12, 9, 20000))])
    arrays["codec/e4m3_in"] = e4
    arrays["codec/e4m3_out"] = encode_e4m3_array(e4)
    arrays["codec/e4m3_table"] = tab

    # ---- quantizers ---------------------------------------------------------
    ts = tensors()
    configs = [(v.value, SchemeConfig(v)) for v in Variant]
    configs += [
        ("mbs_d_cand3", SchemeConfig(Variant.MBS_D, candidates=CandidateSet((0, 37, 200)), augment_static=False)),
        ("mbs_d_noaug", SchemeConfig(Variant.MBS_D, augment_static=False)),
        ("mbs_s_m64", SchemeConfig(Variant.MBS_S, macro_size=64)),
        ("mbs_d_m256", SchemeConfig(Variant.MBS_D, macro_size=256)),
        ("mbs_d_m512", SchemeConfig(Variant.MBS_D, macro_size=512)),
        ("mbs_d_m32", SchemeConfig(Variant.MBS_D, macro_size=32)),
        ("mbs_d_lut", SchemeConfig(Variant.MBS_D, mbs_mode="lut")),
    ]
    for tname, t in ts.items():
        arrays[f"in/{tname}"] = t
        for cname, cfg in configs:
            bs = cfg.block_size
            if t.shape[1] % bs:
                continue
            q = quantize_tensor(t, cfg)
            key = f"q/{tname}/{cname}"
            for f, v in q_fields(q).items():
                arrays[f"{key}/{f}"] = v
            deq = dequantize_tensor(q)
            arrays[f"{key}/deq"] = deq
            rec = {"tensor": tname, "config": cname, "flush": flush_to_zero_rate(t, q)}
            if np.any(t != 0):
                r = qsnr_tensor(t, deq)
                rec.update(qsnr_db=r.qsnr_db, mse=r.mse, signal=r.signal_power)
            meta["cases"].append(rec)

    # ---- GEMM (tests/test_gemm.py:73-93 pairs, plus MBS-H) -------------------
    g = np.random.Generator(np.random.PCG64(103))
    a = g.standard_t(4, (33, 384)).astype(np.float32)
    b = g.standard_normal((29, 384)).astype(np.float32)
    arrays["gemm/a"] = a
    arrays["gemm/b"] = b
    pairs = [("mx16", "mx16"), ("ocp32", "mx16_oas"), ("mbs_s", "mbs_d"), ("mbs_d", "nvfp4"),
             ("nvfp4", "ocp32"), ("mx16_oas", "mbs_s"), ("ocp32", "ocp32"), ("nvfp4", "nvfp4")]
    for va, vb in pairs:
        aq = quantize_tensor(a, SchemeConfig(Variant(va)))
        bq = quantize_tensor(b, SchemeConfig(Variant(vb)))
        arrays[f"gemm/{va}x{vb}"] = matmul_quantized(aq, bq, TileConfig(16, 8, 128))
    meta["gemm_pairs"] = [f"{x}x{y}" for x, y in pairs]

    # ---- config-1 (4096x4096 gaussian+outliers, bf16 RNE), seed 0 -----------
    t1 = bf16(generate_tensor(GeneratorSpec("gaussian_with_outliers", (4096, 4096), seed=0)))
    meta["config1_sha256_bf16"] = hashlib.sha256(t1.tobytes()).hexdigest()
    c1 = {}
    for v in Variant:
        q = quantize_tensor(t1, SchemeConfig(v))
        r = qsnr_tensor(t1, dequantize_tensor(q))
        h = hashlib.sha256()
        for f, arr in sorted(q_fields(q).items()):
            h.update(f.encode())
            h.update(np.ascontiguousarray(arr).tobytes())
        c1[v.value] = {"qsnr_db": r.qsnr_db, "mse": r.mse, "signal": r.signal_power,
                       "flush": flush_to_zero_rate(t1, q), "sha256": h.hexdigest()}
        print(v.value, c1[v.value]["qsnr_db"], flush=True)
    meta["config1"] = c1

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
