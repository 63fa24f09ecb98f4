"""GPU parity of the tcgen05 block-scaled GEMM against the reference
dequantise-then-f64-matmul.

Tolerance: relative Frobenius error <= 1e-5 AND
per element |dC_ij| <= 2^-16 * (|A| |B|^T)_ij, where A, B are the
reference-dequantised operands.  The tensor core accumulates FP4 products in
f32 (and the MBS sigma is applied per 128-K chunk in f32), so bit-exactness
is not expected; any scale-index / sigma / layout bug shows up as O(1e-2).
"""

import numpy as np
import pytest
import torch

from oracle import mxq_oracle as O

pytestmark = pytest.mark.gpu

import paper_2603_08713_b200 as M  # noqa: E402

PAIRS = [("mx16", "mx16"), ("mx16_oas", "mx16_oas"), ("ocp32", "ocp32"), ("mbs_s", "mbs_d"),
         ("mbs_s", "mx16_oas"), ("mx16_oas", "mbs_d"), ("ocp32", "mx16"), ("nvfp4", "nvfp4"), ("mbs_d", "mbs_d")]
SHAPES = [(128, 256, 256), (256, 512, 1024), (200, 300, 2880), (33, 29, 384), (1, 128, 4096), (384, 256, 512)]


def _ref(a, b, va, vb):
    qa, qb = O.quantize(a, va), O.quantize(b, vb)
    da, db = O.dequantize(qa).astype(np.float64), O.dequantize(qb).astype(np.float64)
    return da @ db.T, np.abs(da) @ np.abs(db).T


def _check(c, want, bound, tag):
    c = c.astype(np.float64)
    rel = np.linalg.norm(c - want) / max(np.linalg.norm(want), 1e-300)
    assert rel <= 1e-5, (tag, rel)
    excess = np.abs(c - want) - 2.0 ** -16 * bound
    assert np.all(excess <= 0), (tag, float(excess.max()), np.unravel_index(np.argmax(excess), excess.shape))


@pytest.mark.parametrize("va,vb", PAIRS)
def test_tc_gemm_matches_reference(va, vb):
    rng = np.random.Generator(np.random.PCG64(103))
    for (m, n, k) in SHAPES:
        if (va == "ocp32" or vb == "ocp32") and k % 32:
            continue
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
        bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant(vb)))
        assert M.tc_supported(aq, bq)
        c = M.matmul_quantized(aq, bq).cpu().numpy()
        want, bound = _ref(a, b, va, vb)
        _check(c, want, bound, (va, vb, m, n, k))
        c2 = M.matmul_quantized(aq, bq).cpu().numpy()
        assert np.array_equal(c, c2), "non-deterministic"
        cb = M.matmul_quantized(aq, bq, out_dtype=torch.bfloat16).float().cpu().numpy()
        assert np.array_equal(cb, torch.from_numpy(c).to(torch.bfloat16).float().numpy())


def test_tc_gemm_llama_shape_mbs_h():
    """One Llama-3-8B O-proj sized MBS-H product (A MBS_S x W MBS_D)."""
    rng = np.random.Generator(np.random.PCG64(5))
    a = rng.standard_t(4, (512, 4096)).astype(np.float32)
    w = (rng.standard_normal((1024, 4096)) * 0.02).astype(np.float32)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S))
    wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant.MBS_D))
    c = M.matmul_quantized(aq, wq).cpu().numpy()
    want, bound = _ref(a, w, "mbs_s", "mbs_d")
    _check(c, want, bound, "llama")


@pytest.mark.parametrize("va,vb", [("mbs_d", "nvfp4"), ("nvfp4", "ocp32"), ("mx16_oas", "nvfp4"), ("nvfp4", "mbs_s")])
def test_mixed_scale_types(va, vb):
    """UE8M0 x NVFP4 pairs (/root/reference/pkg/tests/test_gemm.py:73-80): on
    the tensor cores when the UE8M0 operand's exponents span <= 17 (scales
    re-expressed exactly as UE4M3 powers of two, 2^off folded into s_t) --
    within the GEMM tolerance; exact=True stays bit-identical to the
    reference; a wide exponent span falls back to the exact kernel."""
    rng = np.random.Generator(np.random.PCG64(9))
    for (m, n, k) in [(40, 24, 256), (300, 640, 2048), (130, 384, 2880)]:
        if "ocp32" in (va, vb) and k % 32:
            continue
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
        bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant(vb)))
        assert not M.tc_supported(aq, bq)
        c = M.matmul_quantized(aq, bq).cpu().numpy()
        want, bound = _ref(a, b, va, vb)
        _check(c, want, bound, (va, vb, m, n, k))
        ex = M.matmul_quantized(aq, bq, exact=True).cpu().numpy()
        assert np.array_equal(ex, O.matmul_quantized(O.quantize(a, va), O.quantize(b, vb)))
        cb = M.matmul_quantized(aq, bq, out_dtype=torch.bfloat16).float().cpu().numpy()
        assert np.array_equal(cb, torch.from_numpy(c).to(torch.bfloat16).float().numpy())
    # exponent span > 17 (block maxima from 1e-6 to 1e3): the exact kernel
    a = rng.standard_normal((64, 256)).astype(np.float32) * np.logspace(-6, 3, 64, dtype=np.float32)[:, None]
    b = rng.standard_normal((32, 256)).astype(np.float32)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MX16_OAS))
    bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant.NVFP4))
    c = M.matmul_quantized(aq, bq).cpu().numpy()
    assert np.array_equal(c, O.matmul_quantized(O.quantize(a, "mx16_oas"), O.quantize(b, "nvfp4")))


def test_tk_validation_like_reference():
    rng = np.random.Generator(np.random.PCG64(106))
    a = rng.standard_normal((8, 256)).astype(np.float32)
    q16 = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MX16))
    qm = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_D))
    with pytest.raises(ValueError):
        M.matmul_quantized(q16, q16, M.TileConfig(8, 8, 24))
    with pytest.raises(ValueError):
        M.matmul_quantized(qm, qm, M.TileConfig(8, 8, 64))
    M.matmul_quantized(qm, qm, M.TileConfig(8, 8, 256))


@pytest.mark.parametrize("macro", [64, 128, 256, 512])
def test_tc_gemm_mbs_macro_sizes(macro):
    """The 192-column MBS kernel at macros 64 / 128 / 256 / 512 (512: chunks
    straddle the 256-K stages); partial last macro at K = 2880."""
    rng = np.random.Generator(np.random.PCG64(11 + macro))
    for (m, n, k) in [(200, 500, 1024), (130, 384, 2880)]:
        a = rng.standard_t(4, (m, k)).astype(np.float32)
        b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S, macro_size=macro))
        bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant.MBS_D, macro_size=macro))
        c = M.matmul_quantized(aq, bq, M.TileConfig(t_k=max(macro, 128))).cpu().numpy()
        qa = O.quantize(a, "mbs_s", macro_size=macro)
        qb = O.quantize(b, "mbs_d", macro_size=macro)
        da, db = O.dequantize(qa).astype(np.float64), O.dequantize(qb).astype(np.float64)
        _check(c, da @ db.T, np.abs(da) @ np.abs(db).T, ("macro", macro, m, n, k))


@pytest.mark.parametrize("va,vb", [("mbs_s", "mbs_d"), ("mbs_s", "mx16_oas"), ("ocp32", "mbs_d")])
def test_tc_gemm_mbs_persistent_tiles(va, vb):
    """More tiles than CTAs: each CTA runs several 128x192 tiles back to back
    (TMEM buffer / SF buffer / sigma ring phases carried across tiles)."""
    rng = np.random.Generator(np.random.PCG64(21))
    m, n, k = 2048, 3072, 384
    a = rng.standard_t(4, (m, k)).astype(np.float32)
    b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
    bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant(vb)))
    c = M.matmul_quantized(aq, bq).cpu().numpy()
    want, bound = _ref(a, b, va, vb)
    _check(c, want, bound, (va, vb, "persistent"))
    cb = M.matmul_quantized(aq, bq, out_dtype=torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(cb, torch.from_numpy(c).to(torch.bfloat16).float().numpy())


@pytest.mark.parametrize("m", [1, 8, 33, 64, 128])
def test_tc_gemm_mbs_small_m_split_k(m):
    """GPT-OSS expert shapes (config 5): M <= 64 runs swap-AB (weights on the
    MMA's M side, tokens on N = 16/32/64, transposed stores), K = 2880 split
    across CTAs at stage boundaries (f32 partials summed in a fixed order); the
    last macro is 64 wide.  Same tolerance as every tcgen05 product,
    deterministic."""
    rng = np.random.Generator(np.random.PCG64(31 + m))
    for n in (5760, 2880):
        a = rng.standard_t(4, (m, 2880)).astype(np.float32)
        b = (rng.standard_normal((n, 2880)) * 0.02).astype(np.float32)
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S))
        bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant.MBS_D))
        c = M.matmul_quantized(aq, bq).cpu().numpy()
        want, bound = _ref(a, b, "mbs_s", "mbs_d")
        _check(c, want, bound, ("small-m", m, n))
        assert np.array_equal(c, M.matmul_quantized(aq, bq).cpu().numpy())
        cb = M.matmul_quantized(aq, bq, out_dtype=torch.bfloat16).float().cpu().numpy()
        assert np.array_equal(cb, torch.from_numpy(c).to(torch.bfloat16).float().numpy())


@pytest.mark.parametrize("macro", [64, 256])
def test_tc_gemm_mbs_swap_ab_macro_sizes(macro):
    """Swap-AB decode path with the other macro widths the kernel takes."""
    rng = np.random.Generator(np.random.PCG64(71 + macro))
    m, n, k = 5, 1280, 2048
    a = rng.standard_t(4, (m, k)).astype(np.float32)
    b = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S, macro_size=macro))
    bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant.MBS_D, macro_size=macro))
    c = M.matmul_quantized(aq, bq, M.TileConfig(t_k=max(macro, 128))).cpu().numpy()
    qa, qb = O.quantize(a, "mbs_s", macro_size=macro), O.quantize(b, "mbs_d", macro_size=macro)
    da, db = O.dequantize(qa).astype(np.float64), O.dequantize(qb).astype(np.float64)
    _check(c, da @ db.T, np.abs(da) @ np.abs(db).T, ("swap-macro", macro))


# ---------------------------------------------------------------------------
# activation quantization fused into the MBS GEMM launch.
# The fused result must be bit-identical to quantize_tensor + matmul_quantized.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,k,macro,wv,out_dtype", [
    (256, 768, 1024, 128, "mbs_d", torch.float32),
    (200, 1280, 2880, 128, "mbs_d", torch.bfloat16),   # partial row block, partial last macro (64) and stage
    (1000, 1536, 4096, 64, "mbs_s", torch.float32),
    (384, 576, 2048, 256, "mbs_d", torch.bfloat16),
    (130, 640, 1024, 128, "mx16_oas", torch.float32),  # non-MBS weight side
    (48, 1024, 1024, 128, "mbs_d", torch.float32),     # decode size: two launches (swap-AB GEMM)
])
def test_quantize_matmul_fused_matches_two_step(m, n, k, macro, wv, out_dtype):
    g = torch.Generator(device="cuda").manual_seed(1000 + m + k)
    a = (torch.randn(m, k, device="cuda", generator=g) * 3).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    wvar = M.Variant(wv)
    wcfg = M.SchemeConfig(wvar, macro_size=macro) if wvar in (M.Variant.MBS_S, M.Variant.MBS_D) else M.SchemeConfig(wvar)
    wq = M.quantize_tensor(w, wcfg)
    acfg = M.SchemeConfig(M.Variant.MBS_S, macro_size=macro)
    tile = M.TileConfig(t_k=max(macro, 128))
    c_f, aq_f = M.quantize_matmul(a, wq, acfg, tile, out_dtype=out_dtype, fused=True)
    aq_2 = M.quantize_tensor(a, acfg)
    c_2 = M.matmul_quantized(aq_2, wq, tile, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert aq_f == aq_2
    assert torch.equal(aq_f._cache["sig_t"][:, :m], aq_2._cache["sig_t"][:, :m])
    assert torch.equal(c_f, c_2)


def test_quantize_matmul_fused_repeated_and_nonfinite():
    """Back-to-back fused launches (ready flags reset per launch) and the
    non-finite check of the fused quantizer."""
    g = torch.Generator(device="cuda").manual_seed(5)
    w = (torch.randn(1536, 2048, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant.MBS_D))
    xs = [torch.randn(512, 2048, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3)]
    ref = [M.matmul_quantized(M.quantize_tensor(x, M.SchemeConfig(M.Variant.MBS_S)), wq) for x in xs]
    for _ in range(2):
        for x, r in zip(xs, ref):
            c, _ = M.quantize_matmul(x, wq, fused=True)
            assert torch.equal(c, r)
    bad = xs[0].clone()
    bad[300, 7] = float("nan")
    with pytest.raises(ValueError):
        M.quantize_matmul(bad, wq, fused=True)


# ---------------------------------------------------------------------------
# Grouped expert GEMMs (config 5): one launch per 64 experts of the swap-AB
# MBS kernel, each group against the dequantize-then-f64 reference.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("toks,n,k,wv,av,out_dtype", [
    ([1, 5, 16, 3], 640, 2880, "mbs_d", "mbs_s", torch.float32),      # K = 2880: short last macro and stage
    ([33, 64, 17], 384, 1024, "mbs_d", "mbs_s", torch.bfloat16),
    ([8] * 70, 256, 512, "mbs_d", "mbs_s", torch.float32),            # 70 groups: two launches
    ([2, 9], 512, 1024, "mx16_oas", "mbs_s", torch.float32),          # non-MBS weights
    ([100, 128, 65], 640, 2880, "mbs_d", "mbs_s", torch.float32),     # direct form (65-128 tokens)
    ([128] * 3, 384, 1024, "mbs_d", "mbs_s", torch.bfloat16),
    ([4, 4], 512, 1024, "nvfp4", "nvfp4", torch.float32),             # grouped NVFP4 (UE4M3, swap-AB)
    ([1, 8, 32, 64], 1280, 2880, "nvfp4", "nvfp4", torch.bfloat16),   # GPT-OSS K, decode sizes
    ([100, 128], 640, 2880, "nvfp4", "nvfp4", torch.float32),         # grouped NVFP4, direct form
])
def test_grouped_expert_gemm_matches_reference(toks, n, k, wv, av, out_dtype):
    g = torch.Generator(device="cuda").manual_seed(11 + len(toks) + n)
    aqs, bqs = [], []
    for t in toks:
        a = torch.distributions.StudentT(4.0).sample((t, k)).to("cuda") if t % 2 else torch.randn(t, k, device="cuda", generator=g)
        w = torch.randn(n, k, device="cuda", generator=g) * 0.02
        aqs.append(M.quantize_tensor(a.to(torch.bfloat16), M.SchemeConfig(M.Variant(av))))
        bqs.append(M.quantize_tensor(w.to(torch.bfloat16), M.SchemeConfig(M.Variant(wv))))
    cs = M.matmul_quantized_grouped(aqs, bqs, out_dtype=out_dtype)
    torch.cuda.synchronize()
    for i, (aq, bq, c) in enumerate(zip(aqs, bqs, cs)):
        da, db = M.dequantize_tensor(aq).double(), M.dequantize_tensor(bq).double()
        want, bound = (da @ db.T).cpu().numpy(), (da.abs() @ db.abs().T).cpu().numpy()
        got = c.float().cpu().numpy()
        if out_dtype == torch.float32:
            _check(got, want, bound, ("grouped", i, toks[i]))
        else:
            single = M.matmul_quantized(aq, bq, out_dtype=torch.float32).cpu().numpy()
            _check(single, want, bound, ("single", i))
            assert np.allclose(got, single, rtol=2 ** -7, atol=1e-6 * np.abs(single).max()), i


def test_quantize_matmul_fused_not_co_resident():
    """The fused launch must not rely on all of its CTAs being co-resident
    (ADVICE: MPS limits, green contexts, a concurrent kernel holding SMs).
    MXQ_FUSED_OVERSUBSCRIBE=4 launches 4x more CTAs than fit on the GPU;
    the quantization slices are claimed by running CTAs only, so the launch
    completes and matches the two-call result bit for bit.  (Subprocess: the
    hook is read once per process; a hang fails through the timeout.)"""
    import os
    import subprocess
    import sys

    code = (
        "import torch, paper_2603_08713_b200 as M\n"
        "g = torch.Generator(device='cuda').manual_seed(3)\n"
        "a = torch.randn(1024, 2048, device='cuda', generator=g).to(torch.bfloat16)\n"
        "w = (torch.randn(2304, 2048, device='cuda', generator=g) * 0.02).to(torch.bfloat16)\n"
        "wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant.MBS_D))\n"
        "c, aq = M.quantize_matmul(a, wq, fused=True)\n"
        "c2 = M.matmul_quantized(M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S)), wq)\n"
        "torch.cuda.synchronize()\n"
        "assert torch.equal(c, c2)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MXQ_FUSED_OVERSUBSCRIBE="4", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
