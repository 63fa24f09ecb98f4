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
plus one H2D per section.

The tcgen05 operand layout (scale-factor atoms of 128 rows x 4 blocks, and
the transposed f32 sigma^T of MBS tensors) is exported to a SIDECAR file,
``<path>.mxg`` (magic ``MXG1``, same envelope), never into the MXQ1 file, so
MXQ1 stays byte-identical to the reference's.  ``save_quant(...,
gemm_layout=True)`` writes both; ``load_quant`` uploads a sidecar that
matches the container (shape, variant, sizes and the CRC-32 of the MXQ1
payload) straight into the operand cache, so serving skips the on-device
rebuild (``mxq_build_gemm_layout``); without a sidecar the layout is rebuilt
on first GEMM use, or eagerly with ``gemm_layout=True``.  A sidecar that does
not match its container raises ``ValueError`` (stale export).

Header validation and error messages follow the reference line by line
(src/tensorio.py:64-74, :87-120, :152-215), as pure-host functions
(``parse_quant_header``, ``read_quant_host``) that run without a GPU.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile
import zlib
from typing import Optional

import numpy as np

__all__ = [
    "TENSOR_MAGIC", "QUANT_MAGIC", "LAYOUT_MAGIC", "save_tensor", "load_tensor", "save_quant", "load_quant",
    "save_gemm_layout", "parse_quant_header", "parse_layout_header", "read_quant_host", "quant_section_sizes",
    "layout_path",
]

TENSOR_MAGIC = b"MXT1"
QUANT_MAGIC = b"MXQ1"
LAYOUT_MAGIC = b"MXG1"
LAYOUT_NAME = "tcgen05-sf-atom-128x4"  # csrc/layout.cu: 128-row x 4-block atoms, 512 B, rows padded to 256
LAYOUT_VERSION = 1
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
# MXG1 sidecar: the tcgen05 operand layout (host logic)
# ---------------------------------------------------------------------------
def layout_path(path: str) -> str:
    """Sidecar path of an MXQ1 container."""
    return path + ".mxg"


def _layout_geometry(f: dict, sf_block: int) -> tuple[int, int]:
    """(rows_pad, kpad) of the SF-atom layout for `sf_block` (quantize.py
    gemm_qt): rows padded to 256, K padded to 256 elements."""
    rows_pad = -(-f["rows"] // 256) * 256
    return rows_pad, (-(-f["cols"] // 256) * 256) // sf_block


def layout_sections(f: dict, sf_blocks) -> list[tuple[str, int]]:
    """(name, bytes) of an MXG1 payload, in file order: one SF-atom array per
    scale block size, then sigma^T (n_macros x rows_pad f32) for MBS."""
    out = []
    for sb in sf_blocks:
        rows_pad, kpad = _layout_geometry(f, sb)
        out.append((f"sf{sb}", rows_pad * kpad))
    if f["has_mbs"]:
        rows_pad, _ = _layout_geometry(f, 16)
        out.append(("sig_t", -(-f["cols"] // f["macro_size"]) * rows_pad * 4))
    return out


def parse_layout_header(header: dict, f: dict, crc: Optional[int], path: str = "<mxg1>") -> list[tuple[str, int]]:
    """Validate an MXG1 header against its container's normalised MXQ1 fields
    `f` (and the MXQ1 payload's CRC-32 when given); returns the sections."""
    try:
        name = header["layout"]
        version = int(header["version"])
        fields = {k: header[k] for k in ("variant", "block_size", "macro_size")}
        shape = [int(d) for d in header["shape"]]
        sf_blocks = [int(b) for b in header["sf_blocks"]]
        hcrc = int(header["mxq1_crc32"])
    except (KeyError, ValueError, TypeError) as exc:
        raise ValueError(f"{path}: malformed layout header: {exc}") from exc
    if name != LAYOUT_NAME or version != LAYOUT_VERSION:
        raise ValueError(f"{path}: unsupported layout {name!r} v{version}")
    if (shape != [f["rows"], f["cols"]] or fields["variant"] != f["variant"]
            or int(fields["block_size"]) != f["block_size"] or int(fields["macro_size"]) != f["macro_size"]):
        raise ValueError(f"{path}: layout does not match its container (stale export)")
    if not sf_blocks or any(b not in (16, 32) for b in sf_blocks) or len(set(sf_blocks)) != len(sf_blocks):
        raise ValueError(f"{path}: invalid sf_blocks {sf_blocks}")
    if 32 in sf_blocks and f["block_size"] != 32:
        raise ValueError(f"{path}: 32-element SF atoms need an OCP32 container")
    if crc is not None and hcrc != crc:
        raise ValueError(f"{path}: layout does not match its container (payload CRC-32 differs: stale export)")
    return layout_sections(f, sf_blocks)


# ---------------------------------------------------------------------------
# Device paths
# ---------------------------------------------------------------------------
def _pinned(nbytes: int):
    import torch
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)[:nbytes]


def save_quant(q, path: str, gemm_layout: bool = False) -> None:
    """Write a QuantizedTensor (CUDA buffers) as an MXQ1 container, atomically
    (src/tensorio.py:125-149).  One pinned staging buffer, one D2H per
    section on the current stream, one synchronisation.  ``gemm_layout=True``
    also exports the tcgen05 operand layout to the ``.mxg`` sidecar; without
    it, a sidecar left from an earlier save of `path` is removed."""
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
    if gemm_layout:
        save_gemm_layout(q, path, crc=zlib.crc32(memoryview(buf.numpy())))
    elif os.path.exists(layout_path(path)):
        os.unlink(layout_path(path))  # (it described the container just replaced)


def save_gemm_layout(q, path: str, sf_blocks=None, crc: Optional[int] = None) -> str:
    """Export `q`'s tcgen05 operand layout (built on the device if it is not
    cached yet) to the MXG1 sidecar of the MXQ1 container at `path`, which
    must already hold `q` (its payload CRC-32 binds the two).  `sf_blocks`:
    the SF-atom block sizes to store (default: the tensor's own; OCP32 may
    add 16 for pairs with block-16 partners).  Returns the sidecar path."""
    import torch
    if crc is None:
        fh, _, _ = _open_quant(path)  # (positioned at the payload)
        with fh:
            crc = zlib.crc32(fh.read())
    rows, cols = q.shape
    sf_blocks = list(sf_blocks) if sf_blocks else [int(q.block_size)]
    f = {"variant": q.variant.value, "rows": rows, "cols": cols, "block_size": int(q.block_size),
         "macro_size": int(q.macro_size), "has_mbs": q.mbs_mantissas is not None}
    secs = layout_sections(f, sf_blocks)
    header = {"layout": LAYOUT_NAME, "version": LAYOUT_VERSION, "variant": f["variant"], "shape": [rows, cols],
              "block_size": f["block_size"], "macro_size": f["macro_size"], "sf_blocks": sf_blocks,
              "mxq1_crc32": int(crc)}
    parse_layout_header(header, f, crc)  # (self-check)
    srcs = []
    for sb in sf_blocks:
        q.gemm_qt(sb)
        srcs.append(q._cache[("mma", sb)])
    if f["has_mbs"]:
        srcs.append(q._cache["sig_t"])
    buf = _pinned(sum(n for _, n in secs))
    off = 0
    for t, (_, n) in zip(srcs, secs):
        assert t.numel() * t.element_size() == n
        buf[off:off + n].copy_(t.reshape(-1).view(torch.uint8), non_blocking=True)
        off += n
    torch.cuda.current_stream().synchronize()
    hb = _header_bytes(header)
    out = layout_path(path)
    _atomic_write_parts(out, (LAYOUT_MAGIC, struct.pack("<I", len(hb)), hb, memoryview(buf.numpy())))
    return out


def _load_layout(q, path: str, f: dict, crc: int, dev) -> bool:
    """Upload a matching MXG1 sidecar into q's operand cache; False when
    there is none.  Raises ValueError for a sidecar that does not match."""
    import torch
    lp = layout_path(path)
    if not os.path.exists(lp):
        return False
    with open(lp, "rb") as fh:
        header, plen = _read_header(fh, lp, LAYOUT_MAGIC)
        secs = parse_layout_header(header, f, crc, lp)
        total = sum(n for _, n in secs)
        if plen != total:
            raise ValueError(f"{lp}: payload length {plen} != expected {total}")
        buf = _pinned(total)
        if fh.readinto(memoryview(buf.numpy())) != total:
            raise ValueError(f"{lp}: payload length mismatch while reading")
    off = 0
    for name, n in secs:
        t = buf[off:off + n].to(dev, non_blocking=True)
        off += n
        if name == "sig_t":
            rows_pad, _ = _layout_geometry(f, 16)
            q._cache["sig_t"] = t.view(torch.float32).view(-1, rows_pad)
        else:
            q._cache[("mma", int(name[2:]))] = t
    q._cache["staging_mxg"] = buf
    return True


def load_quant(path: str, device=None, gemm_layout: bool = False):
    """Read an MXQ1 container into a QuantizedTensor in CUDA memory,
    bit-exactly (src/tensorio.py:152-215; same ValueErrors).  The payload is
    read straight into a pinned buffer and copied to the device section by
    section.  A matching ``.mxg`` sidecar is uploaded as the tcgen05 operand
    layout (no rebuild); ``gemm_layout=True`` builds whatever the sidecar did
    not provide now instead of on first GEMM use."""
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
    if os.path.exists(layout_path(path)):
        _load_layout(q, path, f, zlib.crc32(memoryview(buf.numpy())), dev)
    if gemm_layout:
        q.gemm_qt()
    torch.cuda.current_stream().synchronize()
    q._cache.pop("staging", None)
    q._cache.pop("staging_mxg", None)
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
