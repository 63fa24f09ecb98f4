"""Acceptance gates re-run on GPU outputs ("C2, C3, C4, C5, C7,
C9 ... with GPU outputs").  Each test draws its inputs exactly like the
reference gate (same PCG64 seeds and generator calls,
/root/reference/pkg/tests/test_acceptance.py), quantizes / dequantizes /
evaluates on the B200 through the product API, and applies the gate's
condition.  C5 and C7 live in test_gpu_quantize.py / test_gpu_bench_parity.py;
C12 (launch / partition invariance) in test_gpu_quantize.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2603_08713_b200 as m
    return m


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_c2_range_invariants(M):
    """alpha / D of every block lands in the variant's window
    (test_acceptance.py:81-99): OCP32 (4, 8], MX16 (3, 6], OAS (3.5, 7]."""
    import torch
    rng = np.random.Generator(np.random.PCG64(22))
    windows = {}
    for width, variant, lo, hi in ((32, M.Variant.OCP32, 4.0, 8.0), (16, M.Variant.MX16, 3.0, 6.0),
                                   (16, M.Variant.MX16_OAS, 3.5, 7.0)):
        t = (rng.standard_normal((10_000, width)) * np.exp2(rng.integers(-30, 30, (10_000, 1)))).astype(np.float32)
        q = M.quantize_tensor(_cuda(t), M.SchemeConfig(variant))
        alpha = torch.from_numpy(np.max(np.abs(t.astype(np.float64)), axis=1)).cuda()
        s = alpha / q.block_dequant_values()[:, 0]
        windows[variant.value] = int((~((s > lo) & (s <= hi))).sum())
    assert windows == {"ocp32": 0, "mx16": 0, "mx16_oas": 0}, windows


def test_c3_oas_dominance(M):
    """OAS never loses to plain MX16 element-wise, and matches it inside the
    (3, 3.5] saturation window to the ulp (test_acceptance.py:102-125)."""
    rng = np.random.Generator(np.random.PCG64(33))
    t = (rng.standard_normal((10_000, 16)) * np.exp2(rng.integers(-20, 21, (10_000, 1)))).astype(np.float32)
    tc = _cuda(t)
    x64 = tc.double()
    d_plain = M.dequantize_tensor(M.quantize_tensor(tc, M.SchemeConfig(M.Variant.MX16))).double()
    d_oas = M.dequantize_tensor(M.quantize_tensor(tc, M.SchemeConfig(M.Variant.MX16_OAS))).double()
    dominance = int(((d_oas - x64).abs() > (d_plain - x64).abs()).sum())

    u = np.float32(3.0 + 0.5 * np.arange(1, 1001) / 1000.0)
    sweep = np.zeros((1000, 16), dtype=np.float32)
    sweep[:, 0] = u
    sc = _cuda(sweep)
    dp = M.dequantize_tensor(M.quantize_tensor(sc, M.SchemeConfig(M.Variant.MX16)))[:, 0].cpu().numpy()
    do = M.dequantize_tensor(M.quantize_tensor(sc, M.SchemeConfig(M.Variant.MX16_OAS)))[:, 0].cpu().numpy()
    x = u.astype(np.float64)
    e_p = np.abs(dp.astype(np.float64) - x) / x
    e_o = np.abs(do.astype(np.float64) - x) / x
    window = int(np.count_nonzero(np.abs(e_p - e_o) > np.spacing(np.maximum(e_p, e_o))))
    assert (dominance, window) == (0, 0)


def test_c4_flush_monotonicity(M):
    """Block-16 never flushes more nonzeros to zero than block-32 on the
    gaussian+outlier tensors (test_acceptance.py:128-145)."""
    violations = 0
    for i in range(100):
        t = M.generate_tensor(M.GeneratorSpec("gaussian_with_outliers", (256, 1024), seed=4000 + i))
        tc = _cuda(t)
        nz = tc != 0
        f16 = (M.quantize_tensor(tc, M.SchemeConfig(M.Variant.MX16)).unpack_codes() & 7) == 0
        f32 = (M.quantize_tensor(tc, M.SchemeConfig(M.Variant.OCP32)).unpack_codes() & 7) == 0
        if int((f16 & nz).sum()) > int((f32 & nz).sum()):
            violations += 1
    assert violations == 0


def test_c9_scheme_ordering(M):
    """Per tensor OCP32 <= MX16 <= OAS <= MBS_S in QSNR, and MBS_S <= MBS_D on
    the mean, over 100 student-t tensors (test_acceptance.py:223-246); QSNR
    from the GPU evaluator (bit-identical to the reference's)."""
    order = (M.Variant.OCP32, M.Variant.MX16, M.Variant.MX16_OAS, M.Variant.MBS_S, M.Variant.MBS_D, M.Variant.NVFP4)
    sums = {v: 0.0 for v in order}
    per_tensor = 0
    for i in range(100):
        t = M.generate_tensor(M.GeneratorSpec("student_t", (256, 1024), seed=9000 + i, dof=4.0))
        tc = _cuda(t)
        db = {}
        for v in order:
            rep, _ = M.qsnr_quantized(tc, M.quantize_tensor(tc, M.SchemeConfig(v)))
            db[v] = rep.qsnr_db
            sums[v] += db[v]
        if not (db[order[0]] <= db[order[1]] <= db[order[2]] <= db[order[3]]):
            per_tensor += 1
    means = {v: s / 100 for v, s in sums.items()}
    assert per_tensor == 0
    assert means[M.Variant.MX16_OAS] <= means[M.Variant.MBS_S] <= means[M.Variant.MBS_D]


def test_c10_device_mantissa_accuracy(M):
    """The MBS-S mantissa byte the device quantizer stores is the top 8
    mantissa bits of 6/alpha in f32 (src/quantize.py:369-380) and meets C10's
    bound (test_acceptance.py:249-259): 1 + m8/256 within 1/256 of the
    significand it encodes.  One 128-element macro per row whose |max| is a
    lognormal draw (the gate's distribution)."""
    rng = np.random.Generator(np.random.PCG64(1010))
    alphas = rng.lognormal(0.0, 3.0, 4096).astype(np.float32)
    t = np.zeros((4096, 128), dtype=np.float32)
    t[:, 0] = alphas
    q = M.quantize_tensor(_cuda(t), M.SchemeConfig(M.Variant.MBS_S))
    got = q.mbs_mantissas[:, 0].cpu().numpy()
    ratio = (np.float32(6.0) / alphas).astype(np.float32)
    want = np.array([M.extract_mantissa8(float(r)).m8 for r in ratio])
    assert np.array_equal(got.astype(np.int64), want.astype(np.int64))
    sig = np.frexp(ratio.astype(np.float64))[0] * 2.0
    factor = 1.0 + got.astype(np.float64) / 256.0
    assert np.max((sig - factor) / sig) <= 1.0 / 256.0
