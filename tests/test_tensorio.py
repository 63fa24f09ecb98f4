"""MXQ1 / MXT1 containers, mirroring the reference's
tests/test_tensorio.py:40-251 plus byte-identity against files written by the
reference itself (tests/golden/containers, make_golden_containers.py).

CPU: the pure-host reader against the reference-written files and the
oracle, header rejections with the reference's cases, MXT1 round trip,
atomic overwrite.  GPU: quantize on the device -> save_quant is
byte-identical to the reference's file; load_quant of the reference's file
equals the device quantization and feeds the tcgen05 GEMM.
"""

import json
import os
import shutil
import struct

import numpy as np
import pytest

from paper_2603_08713_b200 import tensorio as tio

CDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "containers")
INDEX = json.load(open(os.path.join(CDIR, "index.json")))


def make_envelope(magic, header, payload):
    hb = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    return magic + struct.pack("<I", len(hb)) + hb + payload


def parse_envelope(blob):
    (hlen,) = struct.unpack("<I", blob[4:8])
    return blob[:4], json.loads(blob[8:8 + hlen].decode()), blob[8 + hlen:]


# ---------------------------------------------------------------------------
# CPU
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("fn", sorted(INDEX))
def test_reference_file_parses_and_matches_oracle(fn):
    """The host reader decodes the reference's file, and its sections equal the
    oracle's quantization of the stored input (both pinned to the reference)."""
    from oracle import mxq_oracle as O
    h = tio.read_quant_host(os.path.join(CDIR, fn))
    x = tio.load_tensor(os.path.join(CDIR, INDEX[fn]["input"]), device="cpu")
    q = O.quantize(x, INDEX[fn]["variant"])
    assert h["variant"] == q.variant and tuple(h["shape"]) == tuple(q.shape)
    assert h["block_size"] == q.block_size and h["macro_size"] == q.macro_size
    assert np.array_equal(h["codes"], q.codes)
    for k in ("block_scales", "e4m3_scales", "mbs_mantissas"):
        a, b = h[k], getattr(q, k)
        assert (a is None) == (b is None), k
        if a is not None:
            assert np.array_equal(a, b), k
    assert h["tensor_scale"] == q.tensor_scale


def test_section_arithmetic_and_bits_per_element():
    # src/tensorio.py section order; reference tests :143-186
    for fn, meta in INDEX.items():
        blob = open(os.path.join(CDIR, fn), "rb").read()
        magic, header, payload = parse_envelope(blob)
        assert magic == b"MXQ1"
        f = tio.parse_quant_header(header)
        assert sum(tio.quant_section_sizes(f)) == len(payload)
        rows, cols = header["shape"]
        n = len(payload) - (8 if header["has_tensor_scale"] else 0)
        if header["has_mbs"] and cols % 128 == 0:
            assert n * 8 / (rows * cols) == 4.5625
        elif not header["has_mbs"]:
            assert n * 8 / (rows * cols) == (4.25 if header["variant"] == "ocp32" else 4.5)


def test_quant_header_rejections(tmp_path):
    # the reference's cases, tests/test_tensorio.py:202-237
    good = os.path.join(CDIR, "t4_6x256.mx16.mxq")
    _, header, payload = parse_envelope(open(good, "rb").read())

    def reject(name, mh=None, mp=None, magic=b"MXQ1"):
        h = dict(header)
        h.update(mh or {})
        p = mp(payload) if mp else payload
        path = str(tmp_path / name)
        open(path, "wb").write(make_envelope(magic, h, p))
        with pytest.raises(ValueError):
            tio.read_quant_host(path)

    reject("mbs_flag.mxq", {"has_mbs": True})
    reject("ts_flag.mxq", {"has_tensor_scale": True})
    reject("block.mxq", {"block_size": 32})
    reject("variant.mxq", {"variant": "fp8"})
    reject("shape.mxq", {"shape": [6, 40]})
    reject("macro.mxq", {"macro_size": 0})
    reject("missing.mxq", {"variant": None})
    reject("short.mxq", mp=lambda p: p[:-1])
    reject("long.mxq", mp=lambda p: p + b"\0")
    reject("magic.mxq", magic=b"MXT1")
    trunc = str(tmp_path / "trunc.mxq")
    open(trunc, "wb").write(open(good, "rb").read()[:6])
    with pytest.raises(ValueError):
        tio.read_quant_host(trunc)
    bad_json = str(tmp_path / "json.mxq")
    open(bad_json, "wb").write(b"MXQ1" + struct.pack("<I", 3) + b"{x}" + payload)
    with pytest.raises(ValueError):
        tio.read_quant_host(bad_json)


def test_tensor_round_trip_and_layout(tmp_path):
    # reference tests :40-65
    path = str(tmp_path / "t.mxt")
    t = np.array([[-0.0, 1.0, 1e-42, 3.4e38], [2.0 ** -126, -6.0, 0.1, -1e-30]], dtype=np.float32)
    tio.save_tensor(t, path)
    back = tio.load_tensor(path, device="cpu")
    assert back.dtype == np.float32 and np.array_equal(back.view(np.uint32), t.view(np.uint32))
    magic, header, payload = parse_envelope(open(path, "rb").read())
    assert magic == b"MXT1" and header == {"dtype": "f32", "shape": [2, 4], "layout": "row-major"}
    assert len(payload) == 32
    # the reference wrote the fixture inputs: same bytes from our writer
    for fn in ("t4_6x256.mxt", "partial_3x208.mxt"):
        x = tio.load_tensor(os.path.join(CDIR, fn), device="cpu")
        p2 = str(tmp_path / fn)
        tio.save_tensor(x, p2)
        assert open(p2, "rb").read() == open(os.path.join(CDIR, fn), "rb").read()


def test_tensor_rejections_and_non_finite(tmp_path):
    # reference tests :68-112
    path = str(tmp_path / "t.mxt")
    tio.save_tensor(np.ones((2, 4), np.float32), path)
    blob = open(path, "rb").read()
    cases = {"bad_magic.mxt": b"XXXX" + blob[4:], "trunc.mxt": blob[:6], "short.mxt": blob[:-4],
             "dtype.mxt": make_envelope(b"MXT1", {"dtype": "f64", "shape": [2, 4], "layout": "row-major"},
                                        blob[-32:]),
             "shape.mxt": make_envelope(b"MXT1", {"dtype": "f32", "shape": [2, 0], "layout": "row-major"}, b"")}
    for name, data in cases.items():
        p = str(tmp_path / name)
        open(p, "wb").write(data)
        with pytest.raises(ValueError):
            tio.load_tensor(p, device="cpu")
    with pytest.raises(ValueError):
        tio.save_tensor(np.ones(4, np.float32), path)
    nan = str(tmp_path / "nan.mxt")
    t = np.array([[1.0, np.nan, np.inf, -1.0]], np.float32)
    tio.save_tensor(t, nan)
    with pytest.raises(ValueError):
        tio.load_tensor(nan, device="cpu")
    back = tio.load_tensor(nan, allow_non_finite=True, device="cpu")
    assert np.array_equal(back.view(np.uint32), t.view(np.uint32))


def test_atomic_overwrite(tmp_path):
    # reference tests :115-127
    path = str(tmp_path / "t.mxt")
    tio.save_tensor(np.full((2, 4), 1.0, np.float32), path)
    tio.save_tensor(np.full((2, 4), 2.0, np.float32), path)
    assert np.array_equal(tio.load_tensor(path, device="cpu"), np.full((2, 4), 2.0, np.float32))
    assert os.listdir(tmp_path) == ["t.mxt"]


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("fn", sorted(INDEX))
def test_gpu_save_is_byte_identical_to_reference(fn, tmp_path):
    import paper_2603_08713_b200 as M
    x = tio.load_tensor(os.path.join(CDIR, INDEX[fn]["input"]))  # CUDA f32
    q = M.quantize_tensor(x, M.SchemeConfig(M.Variant(INDEX[fn]["variant"])))
    out = str(tmp_path / fn)
    tio.save_quant(q, out)
    assert open(out, "rb").read() == open(os.path.join(CDIR, fn), "rb").read()
    back = tio.load_quant(os.path.join(CDIR, fn))
    assert back == q
    assert os.listdir(tmp_path) == [fn]


@pytest.mark.gpu
def test_gpu_loaded_weights_feed_the_gemm(tmp_path):
    """Offline-quantized weights (C3 flow): quantize -> save -> load in a
    fresh QuantizedTensor (tcgen05 layout rebuilt on the device) -> GEMM
    equals the GEMM on the in-memory weights, bit for bit."""
    import torch
    import paper_2603_08713_b200 as M
    g = torch.Generator(device="cuda").manual_seed(5)
    w = torch.randn(384, 512, device="cuda", generator=g) * 0.02
    a = torch.randn(200, 512, device="cuda", generator=g)
    for va, vw in (("mbs_s", "mbs_d"), ("mx16_oas", "mx16_oas"), ("ocp32", "ocp32"), ("nvfp4", "nvfp4")):
        wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant(vw)))
        path = str(tmp_path / f"w.{vw}.mxq")
        tio.save_quant(wq, path)
        for eager in (False, True):
            wl = tio.load_quant(path, gemm_layout=eager)
            assert wl == wq
            aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
            c0 = M.matmul_quantized(aq, wq)
            c1 = M.matmul_quantized(aq, wl)
            assert torch.equal(c0, c1), (va, vw, eager)


# ---------------------------------------------------------------------------
# MXG1 sidecar (tcgen05 operand layout export)
# ---------------------------------------------------------------------------
def _layout_header(**kw):
    h = {"layout": tio.LAYOUT_NAME, "version": tio.LAYOUT_VERSION, "variant": "mbs_d", "shape": [300, 2880],
         "block_size": 16, "macro_size": 128, "sf_blocks": [16], "mxq1_crc32": 1234}
    h.update(kw)
    return h


_F = {"variant": "mbs_d", "rows": 300, "cols": 2880, "block_size": 16, "macro_size": 128, "has_mbs": True,
      "has_tensor_scale": False}


def test_layout_header_sections():
    secs = tio.parse_layout_header(_layout_header(), _F, 1234)
    # SF atoms: rows padded to 256 (512), K padded to 256 elements (3072) / 16; sigma^T: 23 macros x 512 f32
    assert secs == [("sf16", 512 * 192), ("sig_t", 23 * 512 * 4)]
    f32 = dict(_F, variant="ocp32", block_size=32, macro_size=32, has_mbs=False)
    secs = tio.parse_layout_header(_layout_header(variant="ocp32", block_size=32, macro_size=32, sf_blocks=[32, 16]),
                                   f32, None)
    assert secs == [("sf32", 512 * 96), ("sf16", 512 * 192)]


@pytest.mark.parametrize("kw, msg", [
    ({"shape": [301, 2880]}, "stale export"),
    ({"variant": "mbs_s"}, "stale export"),
    ({"macro_size": 256}, "stale export"),
    ({"mxq1_crc32": 99}, "CRC-32"),
    ({"version": 2}, "unsupported layout"),
    ({"layout": "other"}, "unsupported layout"),
    ({"sf_blocks": [32]}, "OCP32 container"),
    ({"sf_blocks": [16, 16]}, "invalid sf_blocks"),
    ({"sf_blocks": "x"}, "malformed layout header"),
])
def test_layout_header_rejects(kw, msg):
    with pytest.raises(ValueError, match=msg):
        tio.parse_layout_header(_layout_header(**kw), _F, 1234)


@pytest.mark.gpu
def test_gpu_layout_sidecar_round_trip(tmp_path):
    """save_quant(gemm_layout=True) exports the SF atoms (and sigma^T) next to
    a byte-unchanged MXQ1 file; load_quant uploads them without a rebuild,
    bit-identical to a fresh build, and the GEMM on the loaded weights equals
    the in-memory one.  A sidecar left over from another tensor is refused."""
    import torch
    import paper_2603_08713_b200 as M
    g = torch.Generator(device="cuda").manual_seed(9)
    w = torch.randn(300, 2880, device="cuda", generator=g) * 0.02
    a = torch.randn(64, 2880, device="cuda", generator=g)
    for va, vw in (("mbs_s", "mbs_d"), ("nvfp4", "nvfp4"), ("ocp32", "ocp32"), ("mx16_oas", "mx16_oas")):
        wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant(vw)))
        p0, p1 = str(tmp_path / f"{vw}.plain.mxq"), str(tmp_path / f"{vw}.mxq")
        tio.save_quant(wq, p0)
        tio.save_quant(wq, p1, gemm_layout=True)
        assert open(p0, "rb").read() == open(p1, "rb").read()  # the container is unchanged
        assert os.path.exists(tio.layout_path(p1)) and not os.path.exists(tio.layout_path(p0))
        wl = tio.load_quant(p1)
        sb = wq.block_size
        assert ("mma", sb) in wl._cache and (vw != "mbs_d" or "sig_t" in wl._cache)
        fresh = tio.load_quant(p0, gemm_layout=True)
        assert torch.equal(wl._cache[("mma", sb)], fresh._cache[("mma", sb)])
        if vw == "mbs_d":
            assert torch.equal(wl._cache["sig_t"], fresh._cache["sig_t"])
        aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
        assert torch.equal(M.matmul_quantized(aq, wq), M.matmul_quantized(aq, wl)), vw
    # stale: another tool (e.g. the reference) rewrote the container, the
    # MBS-D sidecar stayed
    other = M.quantize_tensor(w * 2, M.SchemeConfig(M.Variant.MBS_D))
    tio.save_quant(other, str(tmp_path / "other.mxq"))
    shutil.copyfile(str(tmp_path / "other.mxq"), str(tmp_path / "mbs_d.mxq"))
    with pytest.raises(ValueError, match="stale export"):
        tio.load_quant(str(tmp_path / "mbs_d.mxq"))
    # our own save without gemm_layout drops the sidecar it invalidates
    tio.save_quant(other, str(tmp_path / "mbs_d.mxq"))
    assert not os.path.exists(tio.layout_path(str(tmp_path / "mbs_d.mxq")))
    assert tio.load_quant(str(tmp_path / "mbs_d.mxq")) == other
