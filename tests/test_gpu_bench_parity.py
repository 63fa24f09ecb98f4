"""GPU parity at the BENCHMARKED configurations, and the reference's
acceptance criterion C7 re-run on GPU outputs.

* The exact bench step (bench.py: BASELINE configs[1], the four Llama-3-8B
  linear layers at M = 4096, activations quantized per step, resident
  weights) for all four arms -- MBS-H (MBS_S x MBS_D), OCP32, MX16_OAS,
  NVFP4 -- with f32 and bf16 output.  The operands are the GPU quantizer's
  output (bit-exact to the oracle: test_gpu_quantize.py), dequantized by the
  ORACLE (oracle/mxq_oracle.py: src/quantize.py:728-746) and multiplied in f64
  on the host; a 256-row sample of every product (first and last 128-row
  block, so the first and the last persistent tiles of every column) is
  compared against all N columns under the GEMM tolerance stated in
  DESIGN.md section 4 (rel-Frobenius <= 1e-5, |dC_ij| <= 2^-16 (|A||B|^T)_ij).
* k_gemm_tc with more tiles than clusters (2048 x 4096 x 1024: 256 tiles over
  74 clusters), every plain pair and NVFP4 x NVFP4: the persistent
  accumulator reuse and the NVFP4 tensor-scale epilogue.
* C7 (/root/reference/pkg/tests/test_acceptance.py:187-214): every variant
  pair over random shapes -- bit-exact for exact=True (the reference's own
  criterion), within the tolerance on the tcgen05 path.
"""

import numpy as np
import pytest
import torch

from oracle import mxq_oracle as O

pytestmark = pytest.mark.gpu

import paper_2603_08713_b200 as M  # noqa: E402

LAYERS = (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336))
M_TOK = 4096
ARMS = {"mbs_h": ("mbs_s", "mbs_d"), "ocp32": ("ocp32", "ocp32"), "mx16_oas": ("mx16_oas", "mx16_oas"),
        "nvfp4": ("nvfp4", "nvfp4")}


def oracle_view(q, rows=None) -> O.OracleQ:
    """The GPU QuantizedTensor's arrays (optionally a row subset) as an
    OracleQ, so the oracle dequantizes exactly the operands the kernel read."""
    sel = (lambda t: t.cpu().numpy()) if rows is None else (lambda t: t[rows].cpu().numpy())
    n_rows = q.shape[0] if rows is None else len(rows)
    ts = q.tensor_scale
    if isinstance(ts, torch.Tensor):
        ts = float(ts.item())
    return O.OracleQ(q.variant.value, (n_rows, q.shape[1]), q.block_size, q.macro_size, sel(q.codes),
                     None if q.block_scales is None else sel(q.block_scales),
                     None if q.e4m3_scales is None else sel(q.e4m3_scales),
                     None if q.mbs_mantissas is None else sel(q.mbs_mantissas), ts)


def check_tol(c, want, bound, tag):
    c = np.asarray(c, dtype=np.float64)
    rel = np.linalg.norm(c - want) / max(np.linalg.norm(want), 1e-300)
    assert rel <= 1e-5, (tag, rel)
    excess = np.abs(c - want) - 2.0 ** -16 * bound
    assert np.all(excess <= 0), (tag, float(excess.max()), np.unravel_index(np.argmax(excess), excess.shape))


def bench_inputs(dev, k, n, seed):
    """Bench-step operands: student-t dof 4 activations (bf16), N(0, 0.02)
    random-init weights (bf16) -- bench.py's own generator."""
    import bench
    g = torch.Generator(device=dev).manual_seed(seed)
    a = bench.synth_activation(torch, dev, M_TOK, k, g)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    return a, w


@pytest.mark.parametrize("arm", list(ARMS))
def test_bench_step_matches_oracle(arm):
    va, vw = ARMS[arm]
    dev = torch.device("cuda", 0)
    rows = np.r_[0:128, M_TOK - 128:M_TOK]
    for li, (name, n, k) in enumerate(LAYERS):
        a, w = bench_inputs(dev, k, n, 77 + li)
        wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant(vw)))
        # the bench step: per-step activation quantization without a sync, the
        # GEMM into a preallocated output
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)), check=False)
        c32 = torch.empty(M_TOK, n, device=dev, dtype=torch.float32)
        cbf = torch.empty(M_TOK, n, device=dev, dtype=torch.bfloat16)
        M.matmul_quantized(aq, wq, out=c32, out_dtype=torch.float32, check=False)
        M.matmul_quantized(aq, wq, out=cbf, out_dtype=torch.bfloat16, check=False)
        torch.cuda.synchronize()
        da = O.dequantize(oracle_view(aq, rows)).astype(np.float64)
        db = O.dequantize(oracle_view(wq)).astype(np.float64)
        want = da @ db.T
        bound = np.abs(da) @ np.abs(db).T
        got = c32.cpu().numpy()
        check_tol(got[rows], want, bound, (arm, name))
        # bf16 output = RN(f32 output), on the whole product
        assert torch.equal(cbf, c32.to(torch.bfloat16)), (arm, name)
        del da, db, want, bound


@pytest.mark.parametrize("va,vb", [("ocp32", "ocp32"), ("mx16", "mx16"), ("mx16_oas", "mx16_oas"),
                                   ("ocp32", "mx16_oas"), ("mx16", "mx16_oas"), ("nvfp4", "nvfp4")])
def test_plain_gemm_persistent_multi_tile(va, vb):
    """256 output tiles over 74 clusters: each CTA reuses its accumulator over
    several tiles (and the NVFP4 epilogue scales every one of them)."""
    rng = np.random.Generator(np.random.PCG64(2024))
    m, n, k = 2048, 4096, 1024
    a = rng.standard_t(4, (m, k)).astype(np.float32)
    b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
    bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant(vb)))
    assert M.tc_supported(aq, bq)
    c = M.matmul_quantized(aq, bq).cpu().numpy()
    da = O.dequantize(O.quantize(a, va)).astype(np.float64)
    db = O.dequantize(O.quantize(b, vb)).astype(np.float64)
    check_tol(c, da @ db.T, np.abs(da) @ np.abs(db).T, (va, vb))
    cb = M.matmul_quantized(aq, bq, out_dtype=torch.bfloat16)
    assert torch.equal(cb, torch.from_numpy(c).cuda().to(torch.bfloat16))


def test_criterion_07_all_pairs_on_gpu():
    """C7 on GPU outputs: all 36 variant pairs over 20 random shapes (the
    reference's K choices 16 / 128 / 256 / 384 / 1024, M, N in 1..40).  The
    exact path must be bit-identical to dequantize-then-matmul_reference; the
    default path (tensor cores for all 36 pairs where the scale formats allow)
    within the GEMM tolerance."""
    rng = np.random.Generator(np.random.PCG64(77))
    k_choices = (16, 128, 256, 384, 1024)
    n_exact = n_tc = 0
    for shape_i in range(20):
        k = k_choices[shape_i % len(k_choices)]
        m = int(rng.integers(1, 41))
        n = int(rng.integers(1, 41))
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        b = rng.standard_normal((n, k)).astype(np.float32)
        variants = [v for v in O.VARIANTS if not (v == "ocp32" and k % 32)]
        qa = {v: M.quantize_tensor(a, M.SchemeConfig(M.Variant(v))) for v in variants}
        qb = {v: M.quantize_tensor(b, M.SchemeConfig(M.Variant(v))) for v in variants}
        da = {v: O.dequantize(O.quantize(a, v)) for v in variants}
        db = {v: O.dequantize(O.quantize(b, v)) for v in variants}
        for va in variants:
            for vb in variants:
                want = O.matmul_ref(da[va], db[vb])
                got = M.matmul_quantized(qa[va], qb[vb], exact=True).cpu().numpy()
                assert np.array_equal(got, want), ("exact", va, vb, m, n, k)
                n_exact += 1
                # the default path: tcgen05 for every same-format pair and for
                # UE8M0 x NVFP4 pairs whose E8M0 span fits UE4M3, else exact
                c = M.matmul_quantized(qa[va], qb[vb]).cpu().numpy()
                w64 = da[va].astype(np.float64) @ db[vb].astype(np.float64).T
                bound = np.abs(da[va]).astype(np.float64) @ np.abs(db[vb]).astype(np.float64).T
                check_tol(c, w64, bound, ("default", va, vb, m, n, k))
                n_tc += 1
    assert n_exact >= 20 * 25 and n_tc == n_exact


def test_out_argument_is_validated():
    """ADVICE: `out=` must match the result exactly (shape, dtype, device,
    unit column stride); a mismatch raises instead of writing out of bounds."""
    rng = np.random.Generator(np.random.PCG64(3))
    a = rng.standard_normal((64, 256)).astype(np.float32)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S))
    bq = M.quantize_tensor(a[:32], M.SchemeConfig(M.Variant.MBS_D))
    with pytest.raises(ValueError):
        M.matmul_quantized(aq, bq, out=torch.empty(64, 32, device="cuda", dtype=torch.bfloat16))  # dtype
    with pytest.raises(ValueError):
        M.matmul_quantized(aq, bq, out=torch.empty(64, 31, device="cuda"))  # shape
    with pytest.raises(ValueError):
        M.matmul_quantized(aq, bq, out=torch.empty(32, 64, device="cuda").t())  # column stride
    out = torch.empty(64, 32, device="cuda")
    assert M.matmul_quantized(aq, bq, out=out) is out
    ex = torch.empty(64, 32, device="cuda")
    assert M.matmul_quantized(aq, bq, exact=True, out=ex) is ex  # exact path fills `out` too
    assert torch.allclose(out, ex, rtol=1e-5, atol=1e-5)


def test_corrupt_scale_codes_raise_on_tc_path():
    """src/quantize.py:228-241: an E8M0 255 / E4M3 NaN scale byte is a
    ValueError in matmul_quantized, on the tcgen05 path too."""
    import dataclasses

    rng = np.random.Generator(np.random.PCG64(4))
    a = rng.standard_normal((64, 256)).astype(np.float32)
    q = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MX16_OAS))
    bad = q.block_scales.clone()
    bad[3, 2] = 255
    qb = dataclasses.replace(q, block_scales=bad)
    with pytest.raises(ValueError, match="E8M0 code 255"):
        M.matmul_quantized(qb, q)
    n = M.quantize_tensor(a, M.SchemeConfig(M.Variant.NVFP4))
    e = n.e4m3_scales.clone()
    e[0, 0] = 0x7F
    with pytest.raises(ValueError, match="E4M3 NaN"):
        M.matmul_quantized(dataclasses.replace(n, e4m3_scales=e), n)


def test_grouped_plain_pairs_are_block_correct():
    """ADVICE (high): OCP32 x OCP32 groups must not be run with a block-16
    scale layout read as block-32; they take the per-expert path."""
    rng = np.random.Generator(np.random.PCG64(8))
    aqs, bqs, refs = [], [], []
    for t in (3, 17):
        a = rng.standard_normal((t, 512)).astype(np.float32)
        b = (rng.standard_normal((384, 512)) * 0.02).astype(np.float32)
        aqs.append(M.quantize_tensor(a, M.SchemeConfig(M.Variant.OCP32)))
        bqs.append(M.quantize_tensor(b, M.SchemeConfig(M.Variant.OCP32)))
        da = O.dequantize(O.quantize(a, "ocp32")).astype(np.float64)
        db = O.dequantize(O.quantize(b, "ocp32")).astype(np.float64)
        refs.append((da @ db.T, np.abs(da) @ np.abs(db).T))
    for c, (want, bound) in zip(M.matmul_quantized_grouped(aqs, bqs), refs):
        check_tol(c.cpu().numpy(), want, bound, "grouped-ocp32")


@pytest.mark.parametrize("macro", [192, 512])
def test_mbs_gemm_macros_beyond_256(macro):
    """Macro sizes that are multiples of the 64-K MMA step but straddle the
    kernel's 256-K stages now run on the tcgen05 MBS kernel (partial last
    macro at K = 2880)."""
    rng = np.random.Generator(np.random.PCG64(90 + macro))
    for (m, n, k) in [(300, 640, 2048), (130, 384, 2880)]:
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S, macro_size=macro))
        bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant.MBS_D, macro_size=macro))
        assert M.tc_supported(aq, bq)
        tk = macro * (1 if 2048 % macro == 0 else 1)
        c = M.matmul_quantized(aq, bq, M.TileConfig(t_k=tk)).cpu().numpy()
        da = O.dequantize(O.quantize(a, "mbs_s", macro_size=macro)).astype(np.float64)
        db = O.dequantize(O.quantize(b, "mbs_d", macro_size=macro)).astype(np.float64)
        check_tol(c, da @ db.T, np.abs(da) @ np.abs(db).T, ("macro", macro, m, n, k))
