"""MXT1 / MXQ1 containers from and to GPU buffers.

Same on-disk format as the reference (src/tensorio.py:1-215): a 4-byte magic,
a little-endian uint32 header length, the canonical JSON header
(``sort_keys``, no whitespace), then raw little-endian sections in a fixed
order; writes are atomic (temp file + rename).  Files written here are
byte-identical to the reference's for bit-identical tensors, and files the
reference writes load here bit-exactly (tests/test_tensorio.py).

B200 side: all sections of a file are staged through ONE pinned host buffer
with asynchronous copies on the caller's stream and a single synchronisation,
so a save is one D2H of exactly the payload bytes and a load is one file read
plus one H2D per section.  The tcgen05 scale-factor layout is not stored (the
format is the reference's); ``load_quant`` leaves it to be rebuilt on the
device on first GEMM use (``mxq_build_gemm_layout``), or eagerly with
``gemm_layout=True``.

Header validation and error messages follow the reference line by line
(src/tensorio.py:64-74, :87-120, :152-215), as pure-host functions
(``parse_quant_header``, ``read_quant_host``) that run without a GPU.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile
from typing import Optional

import numpy as np

__all__ = [
    "TENSOR_MAGIC", "QUANT_MAGIC", "save_tensor", "load_tensor", "save_quant", "load_quant",
    "parse_quant_header", "read_quant_host", "quant_section_sizes",
]

TENSOR_MAGIC = b"MXT1"
QUANT_MAGIC = b"MXQ1"
_MBS = ("mbs_s", "mbs_d")
_VARIANTS = ("ocp32", "mx16", "mx16_oas", "mbs_s", "mbs_d", "nvfp4")  # Variant values, src/quantize.py:70-76


# ---------------------------------------------------------------------------
# Envelope (host)
# ---------------------------------------------------------------------------
def _header_bytes(header: dict) -> bytes:
    return json.dumps(header, sort_keys=True, separators=(",", ":")).encode()


def _atomic_write_parts(path: str, parts) -> None:
    """Write byte-like parts to ``path`` via a temp file in the same directory
    and an atomic rename (src/tensorio.py:38-50): readers never see a partial
    file and no temp file survives an error."""
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".tmp-", suffix=".part")
    try:
        with os.fdopen(fd, "wb") as fh:
            for p in parts:
                fh.write(p)
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise


def _read_header(fh, path: str, magic: bytes) -> tuple[dict, int]:
    """Magic + header of an open container; returns (header, payload length)
    (src/tensorio.py:58-70)."""
    fh.seek(0, os.SEEK_END)
    size = fh.tell()
    fh.seek(0)
    head = fh.read(8)
    if len(head) < 8 or head[:4] != magic:
        raise ValueError(f"{path}: bad magic, expected {magic.decode()}")
    (header_len,) = struct.unpack("<I", head[4:8])
    if 8 + header_len > size:
        raise ValueError(f"{path}: truncated header")
    raw = fh.read(header_len)
    try:
        header = json.loads(raw.decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise ValueError(f"{path}: malformed header: {exc}") from exc
    return header, size - 8 - header_len


# ---------------------------------------------------------------------------
# MXQ1 header logic (host, reference src/tensorio.py:152-190)
# ---------------------------------------------------------------------------
def parse_quant_header(header: dict, path: str = "<mxq1>") -> dict:
    """Validate an MXQ1 header exactly like the reference's ``load_quant``;
    returns the normalised fields (variant value, rows, cols, block_size,
    macro_size, has_mbs, has_tensor_scale)."""
    try:
        variant = header["variant"]
        if variant not in _VARIANTS:
            raise ValueError(f"{variant!r} is not a valid Variant")
        rows, cols = (int(d) for d in header["shape"])
        block_size = int(header["block_size"])
        macro_size = int(header["macro_size"])
        has_mbs = bool(header["has_mbs"])
        has_tensor_scale = bool(header["has_tensor_scale"])
    except (KeyError, ValueError, TypeError) as exc:
        raise ValueError(f"{path}: malformed header: {exc}") from exc
    expected_bs = 32 if variant == "ocp32" else 16
    if block_size != expected_bs:
        raise ValueError(f"{path}: variant {variant} cannot have block_size {block_size}")
    if rows <= 0 or cols <= 0 or cols % block_size != 0:
        raise ValueError(f"{path}: invalid shape {rows}x{cols} for block_size {block_size}")
    if macro_size <= 0 or macro_size % expected_bs != 0:
        raise ValueError(f"{path}: invalid macro_size {macro_size}")
    if has_mbs != (variant in _MBS):
        raise ValueError(f"{path}: mantissa section inconsistent with variant {variant}")
    if has_tensor_scale != (variant == "nvfp4"):
        raise ValueError(f"{path}: tensor-scale section inconsistent with variant {variant}")
    return {"variant": variant, "rows": rows, "cols": cols, "block_size": block_size,
            "macro_size": macro_size, "has_mbs": has_mbs, "has_tensor_scale": has_tensor_scale}


def quant_section_sizes(f: dict) -> tuple[int, int, int, int]:
    """(codes, scales, mantissas, tensor scale) byte counts, in file order."""
    rows, cols = f["rows"], f["cols"]
    n_macros = -(-cols // f["macro_size"])
    return (rows * (cols // 2), rows * (cols // f["block_size"]),
            rows * n_macros if f["has_mbs"] else 0, 8 if f["has_tensor_scale"] else 0)


def _open_quant(path: str):
    fh = open(path, "rb")
    try:
        header, plen = _read_header(fh, path, QUANT_MAGIC)
        f = parse_quant_header(header, path)
        sizes = quant_section_sizes(f)
        if plen != sum(sizes):
            raise ValueError(f"{path}: payload length {plen} != expected {sum(sizes)}")
    except BaseException:
        fh.close()
        raise
    return fh, f, sizes


def read_quant_host(path: str) -> dict:
    """The sections of an MXQ1 file as numpy arrays (no GPU needed): keys of
    ``QuantizedTensor.to_host()``."""
    fh, f, sizes = _open_quant(path)
    with fh:
        payload = np.frombuffer(fh.read(), dtype=np.uint8)
    rows, cols = f["rows"], f["cols"]
    o = np.cumsum((0,) + sizes)
    codes = payload[o[0]:o[1]].reshape(rows, cols // 2).copy()
    scales = payload[o[1]:o[2]].reshape(rows, cols // f["block_size"]).copy()
    mant = payload[o[2]:o[3]].reshape(rows, -1).copy() if f["has_mbs"] else None
    ts = struct.unpack("<d", payload[o[3]:o[4]].tobytes())[0] if f["has_tensor_scale"] else None
    nv = f["variant"] == "nvfp4"
    return {"variant": f["variant"], "shape": (rows, cols), "block_size": f["block_size"],
            "macro_size": f["macro_size"], "codes": codes, "block_scales": None if nv else scales,
            "e4m3_scales": scales if nv else None, "mbs_mantissas": mant, "tensor_scale": ts}


# ---------------------------------------------------------------------------
# Device paths
# ---------------------------------------------------------------------------
def _pinned(nbytes: int):
    import torch
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)[:nbytes]


def save_quant(q, path: str) -> None:
    """Write a QuantizedTensor (CUDA buffers) as an MXQ1 container, atomically
    (src/tensorio.py:125-149).  One pinned staging buffer, one D2H per
    section on the current stream, one synchronisation."""
    import torch
    rows, cols = q.shape
    has_mbs = q.mbs_mantissas is not None
    has_ts = q.tensor_scale is not None
    header = {"variant": q.variant.value, "shape": [int(rows), int(cols)], "block_size": int(q.block_size),
              "macro_size": int(q.macro_size), "has_mbs": has_mbs, "has_tensor_scale": has_ts}
    scales = q.e4m3_scales if q.variant.value == "nvfp4" else q.block_scales
    f = {"rows": rows, "cols": cols, "block_size": q.block_size, "macro_size": q.macro_size,
         "has_mbs": has_mbs, "has_tensor_scale": has_ts}
    sizes = quant_section_sizes(f)
    buf = _pinned(sum(sizes))
    off = 0
    for t, n in ((q.codes, sizes[0]), (scales, sizes[1]), (q.mbs_mantissas if has_mbs else None, sizes[2])):
        if t is not None and n:
            buf[off:off + n].view(t.shape).copy_(t, non_blocking=True)
        off += n
    torch.cuda.current_stream().synchronize()
    if has_ts:
        buf[off:off + 8].numpy()[:] = np.frombuffer(struct.pack("<d", float(q.tensor_scale)), dtype=np.uint8)
    hb = _header_bytes(header)
    _atomic_write_parts(path, (QUANT_MAGIC, struct.pack("<I", len(hb)), hb, memoryview(buf.numpy())))


def load_quant(path: str, device=None, gemm_layout: bool = False):
    """Read an MXQ1 container into a QuantizedTensor in CUDA memory,
    bit-exactly (src/tensorio.py:152-215; same ValueErrors).  The payload is
    read straight into a pinned buffer and copied to the device section by
    section.  ``gemm_layout=True`` also builds the tcgen05 operand layouts
    now instead of on first GEMM use."""
    import torch
    from . import _lib
    from .quantize import QuantizedTensor, Variant
    dev = torch.device(device) if device is not None else _lib.require_device()
    fh, f, sizes = _open_quant(path)
    buf = _pinned(sum(sizes))
    with fh:
        if fh.readinto(memoryview(buf.numpy())) != sum(sizes):
            raise ValueError(f"{path}: payload length mismatch while reading")
    rows, cols = f["rows"], f["cols"]
    o = np.cumsum((0,) + sizes)
    up = lambda a, b, shape: buf[a:b].view(shape).to(dev, non_blocking=True)
    codes = up(o[0], o[1], (rows, cols // 2))
    scales = up(o[1], o[2], (rows, cols // f["block_size"]))
    mant = up(o[2], o[3], (rows, sizes[2] // rows)) if f["has_mbs"] else None
    ts = struct.unpack("<d", buf[o[3]:o[4]].numpy().tobytes())[0] if f["has_tensor_scale"] else None
    nv = f["variant"] == "nvfp4"
    q = QuantizedTensor(variant=Variant(f["variant"]), shape=(rows, cols), block_size=f["block_size"],
                        macro_size=f["macro_size"], codes=codes, block_scales=None if nv else scales,
                        e4m3_scales=scales if nv else None, mbs_mantissas=mant, tensor_scale=ts)
    q._cache["staging"] = buf  # keep the pinned source alive until the copies ran
    if gemm_layout:
        q.gemm_qt()
    torch.cuda.current_stream().synchronize()
    q._cache.pop("staging", None)
    return q


def save_tensor(t, path: str) -> None:
    """Write a 2-D float32 tensor (CUDA tensor or array) as MXT1, atomically
    (src/tensorio.py:73-83)."""
    import torch
    if isinstance(t, torch.Tensor):
        if t.dim() != 2:
            raise ValueError(f"expected a 2-D tensor, got shape {tuple(t.shape)}")
        rows, cols = t.shape
        buf = _pinned(rows * cols * 4)
        buf.view(torch.float32).view(rows, cols).copy_(t.to(torch.float32), non_blocking=True)
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        payload = memoryview(buf.numpy())
    else:
        arr = np.ascontiguousarray(t, dtype=np.float32)
        if arr.ndim != 2:
            raise ValueError(f"expected a 2-D tensor, got shape {arr.shape}")
        rows, cols = arr.shape
        payload = arr.astype("<f4").tobytes()
    header = {"dtype": "f32", "shape": [int(rows), int(cols)], "layout": "row-major"}
    hb = _header_bytes(header)
    _atomic_write_parts(path, (TENSOR_MAGIC, struct.pack("<I", len(hb)), hb, payload))


def _tensor_header(fh, path: str) -> tuple[int, int]:
    header, plen = _read_header(fh, path, TENSOR_MAGIC)
    if header.get("dtype") != "f32" or header.get("layout") != "row-major":
        raise ValueError(f"{path}: unsupported dtype/layout in header: {header}")
    shape = header.get("shape")
    if (not isinstance(shape, list) or len(shape) != 2
            or not all(isinstance(d, int) and d > 0 for d in shape)):
        raise ValueError(f"{path}: bad shape in header: {shape}")
    rows, cols = shape
    if plen != rows * cols * 4:
        raise ValueError(f"{path}: payload length {plen} != expected {rows * cols * 4}")
    return rows, cols


def load_tensor(path: str, allow_non_finite: bool = False, device=None):
    """Read an MXT1 container (src/tensorio.py:86-120).  With ``device=None``
    and a GPU present the result is a CUDA float32 tensor (finiteness checked
    on the device); ``device="cpu"`` returns a numpy float32 array."""
    with open(path, "rb") as fh:
        rows, cols = _tensor_header(fh, path)
        if device is not None and str(device) == "cpu":
            arr = np.frombuffer(fh.read(), dtype="<f4").reshape(rows, cols).astype(np.float32)
            if not allow_non_finite and not np.all(np.isfinite(arr)):
                raise ValueError(f"{path}: payload contains non-finite values")
            return arr
        import torch
        from . import _lib
        dev = torch.device(device) if device is not None else _lib.require_device()
        buf = _pinned(rows * cols * 4)
        fh.readinto(memoryview(buf.numpy()))
    out = buf.view(torch.float32).view(rows, cols).to(dev, non_blocking=True)
    if not allow_non_finite and not bool(torch.isfinite(out).all()):
        raise ValueError(f"{path}: payload contains non-finite values")
    return out
