"""CPU tests of the C-ABI library: it loads, exports every symbol the header
declares, and its host-compiled arithmetic header (the same code the sm_100a
kernels run) matches the reference / oracle bit-for-bit.  No GPU needed."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import mxq_oracle as O
from paper_2603_08713_b200 import _lib
from paper_2603_08713_b200 import formats as F
from paper_2603_08713_b200 import quantize as Q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mxq200.h")).read()
    names = set(re.findall(r"\b(mxq_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    L = _lib.lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    # and every declared function has a ctypes signature in the binding
    assert names <= set(_lib.SIGNATURES), sorted(names - set(_lib.SIGNATURES))
    assert L.mxq_version() >= 100


def test_e2m1_codec_matches_golden(golden):
    assert np.array_equal(F.encode_e2m1_array(golden["codec/e2m1_in"], saturate=True), golden["codec/e2m1_out"])
    # scalar API, tie table from tests/test_formats.py:76-103
    cases = {0.25: 0, 0.75: 2, 1.25: 2, 1.75: 4, 2.5: 4, 3.5: 6, 5.0: 6, -2.5: 12, -0.25: 0, -0.0: 0, -0.1: 0}
    for v, code in cases.items():
        assert F.encode_e2m1(v).code == code, v
    assert F.encode_e2m1(6.6, saturate=True).value == 6.0
    assert F.encode_e2m1(-100.0, saturate=True).value == -6.0
    with pytest.raises(ValueError):
        F.encode_e2m1(6.6)
    with pytest.raises(ValueError):
        F.encode_e2m1(float("nan"))
    with pytest.raises(ValueError):
        F.encode_e2m1_array(np.array([7.0]))


def test_e4m3_codec_matches_golden(golden):
    assert np.array_equal(F.encode_e4m3_array(golden["codec/e4m3_in"]), golden["codec/e4m3_out"])
    assert np.array_equal(F.E4M3_TABLE, golden["codec/e4m3_table"], equal_nan=True)
    assert F.decode_e4m3(F.E4M3Value(0x7E)) == 448.0
    assert F.decode_e4m3(F.encode_e4m3(500.0)) == 448.0
    with pytest.raises(ValueError):
        F.decode_e4m3(F.E4M3Value(0x7F))


def test_e8m0_floor_and_mantissa8():
    for b in range(255):
        assert F.e8m0_floor(F.E8M0Scale(b).value).biased_exponent == b
    s = F.e8m0_floor(2.0 ** -130)
    assert s.clamped and s.biased_exponent == 0
    s = F.e8m0_floor(2.0 ** 200)
    assert s.clamped and s.biased_exponent == 254
    assert F.extract_mantissa8(1.0).m8 == 0
    assert F.extract_mantissa8(1.5).m8 == 128
    assert F.extract_mantissa8(6.0 / 4.4).m8 == 93
    with pytest.raises(ValueError):
        F.extract_mantissa8(-1.0)


def test_closed_form_e8m0_matches_reference_formula():
    """The kernels' integer E8M0 selection against the
    reference's frexp formula on 2M f32 maxima incl. subnormals."""
    rng = np.random.Generator(np.random.PCG64(5))
    bits = rng.integers(1, 0x7F800000, 2_000_000, dtype=np.int64).astype(np.uint32)
    a = bits.view(np.float32)
    a = np.concatenate([a, np.float32([1.5, 1.75, 3.0, 3.5, 6.0, 7.0, 8.0, 1e-45, 2.0 ** -126, 3.4e38])])
    a = np.ascontiguousarray(a)
    L = _lib.lib()
    for kind, want in ((0, O.scale_exp_ocp(a)), (1, O.scale_exp_16(a, False)), (2, O.scale_exp_16(a, True))):
        got = np.empty(a.size, np.uint8)
        L.mxq_host_e8m0_closed_form(a.ctypes.data, a.size, kind, got.ctypes.data)
        assert np.array_equal(got, want), kind


def test_block_scale_kats():
    """tests/test_quantize.py:39-96 frozen examples."""
    pad = lambda v, n=16: np.concatenate([np.asarray(v, float), np.zeros(n - len(v))])
    assert Q.block_scale_ocp(pad([7.6], 32)).value == 1.0
    assert Q.block_scale_ocp(pad([8.0], 32)).value == 2.0
    assert Q.block_scale_ocp(pad([3.4], 32)).biased_exponent == 126
    assert Q.block_scale_16(pad([3.4])).value == 1.0
    assert Q.block_scale_16(pad([3.4]), oas=True).value == 0.5
    assert Q.block_scale_16(pad([3.6]), oas=True).value == 1.0
    assert Q.block_scale_16(np.zeros(16)).value == 1.0
    s = Q.block_scale_16(pad([2.0 ** -140]))
    assert s.clamped and s.biased_exponent == 0
    s = Q.block_scale_16(pad([2.0 ** 130]))
    assert s.clamped and s.biased_exponent == 254
    with pytest.raises(ValueError):
        Q.block_scale_16(np.zeros(32))
    with pytest.raises(ValueError):
        Q.block_scale_ocp(pad([np.nan], 32))


def test_static_mantissa_and_quantize_block():
    assert Q.mbs_static_mantissa(6.0).m8 == 0
    assert Q.mbs_static_mantissa(4.0).m8 == 128
    assert Q.mbs_static_mantissa(4.4).m8 == 93
    assert Q.mbs_static_mantissa(0.0).m8 == 0
    with pytest.raises(ValueError):
        Q.mbs_static_mantissa(-1.0)
    rng = np.random.Generator(np.random.PCG64(3))
    al = rng.uniform(1e-3, 1e3, 5000)
    want = O.static_m8(al)
    got = np.array([Q.mbs_static_mantissa(float(x)).m8 for x in al])
    assert np.array_equal(got, want)
    codes = Q.quantize_block(np.array([3.4, 0.2] + [0.0] * 14), sf=2.0)
    assert F.E2M1_GRID[codes[0] & 7] == 6.0 and F.E2M1_GRID[codes[1] & 7] == 0.5
    codes = Q.quantize_block(np.array([4.4, 1.0] + [0.0] * 14), sf=1.0, factor=F.Mantissa8(93))
    assert codes[0] & 7 == 7


def test_dequant_element_exhaustive():
    """Every (code, E8M0 byte, m8): the kernels' element formula (f32 division
    inside the normal window, f64 outside) equals the reference's
    f32(f64(g*D)/f64(f)) (src/quantize.py:409-423)."""
    L = _lib.lib()
    codes = np.arange(16)
    g = F.decode_e2m1_array(codes)
    for b in list(range(0, 12)) + list(range(120, 136)) + list(range(244, 255)):
        d = np.ldexp(1.0, b - 127)
        for m8 in range(256):
            want = (g * d / (1.0 + m8 / 256.0)).astype(np.float32)
            got = np.array([L.mxq_host_dequant_element(3, int(c), b, m8, 1.0) for c in codes], np.float32)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (b, m8)
        want = (g * d).astype(np.float32)
        got = np.array([L.mxq_host_dequant_element(1, int(c), b, 0, 1.0) for c in codes], np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), b


def test_dequant_fast_window_division_identity():
    """The fast path's f32 division equals the reference's f64 division for
    every grid value and every m8 at one D; power-of-two scaling carries it
    to the whole window [4, 250] (vectorised over all 7x256 quotients)."""
    g = F.E2M1_GRID[1:]
    f32 = (1.0 + np.arange(256) / 256.0).astype(np.float32)
    q32 = (g[:, None].astype(np.float32) / f32[None, :]).astype(np.float32)
    q64 = (g[:, None] / (1.0 + np.arange(256)[None, :] / 256.0)).astype(np.float32)
    assert np.array_equal(q32, q64)


def test_host_mbs_choose_matches_oracle(golden):
    rng = np.random.Generator(np.random.PCG64(17))
    cands = Q.default_candidates()
    macros = np.concatenate([rng.standard_normal((150, 128)), rng.standard_t(4, (150, 128))]).astype(np.float32)
    want = O.choose_exact(macros, cands.mantissas, True)
    want_noaug = O.choose_exact(macros, cands.mantissas, False)
    for i in range(macros.shape[0]):
        assert Q._choose(macros[i], cands, True, None).m8 == want[i]
        assert Q.mbs_dynamic_exact(macros[i], cands).m8 == want_noaug[i]
    # custom candidates (tests/test_quantize.py:184-189)
    c3 = Q.CandidateSet((0, 37, 200))
    assert Q.mbs_dynamic_exact(macros[0], c3).m8 == O.choose_exact(macros[:1], (0, 37, 200), False)[0]
    # trivial macros
    assert Q.mbs_dynamic_exact(np.zeros(128), cands).m8 == 0
    with pytest.raises(ValueError):
        Q.mbs_dynamic_exact(np.zeros(120), cands)


def test_host_lut_choose_matches_oracle():
    rng = np.random.Generator(np.random.PCG64(23))
    cands = Q.default_candidates()
    lut = Q.build_error_lut(cands)
    assert np.array_equal(lut.entries, O.build_lut(cands.mantissas))
    macros = rng.standard_normal((200, 128)).astype(np.float32)
    want = O.choose_lut(macros, lut.entries, cands.mantissas)
    got = np.array([Q.mbs_dynamic_lut(m, lut, cands).m8 for m in macros])
    assert np.array_equal(got, want)
    with pytest.raises(ValueError):
        Q.mbs_dynamic_lut(np.zeros(128), lut, Q.CandidateSet(tuple(range(0, 64, 4))))


def test_scheme_config_validation():
    with pytest.raises(ValueError):
        Q.SchemeConfig(Q.Variant.OCP32, block_size=16)
    with pytest.raises(ValueError):
        Q.SchemeConfig(Q.Variant.MX16, macro_size=24)
    with pytest.raises(ValueError):
        Q.SchemeConfig(Q.Variant.MBS_D, mbs_mode="fast")
    assert Q.SchemeConfig(Q.Variant.OCP32).block_size == 32
    assert Q.macro_segments(208, 128) == [(0, 128), (128, 208)]
    with pytest.raises(ValueError):
        Q.CandidateSet((16, 32))


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        Q.quantize_tensor(np.ones((4, 16), np.float32), Q.SchemeConfig(Q.Variant.MX16))
