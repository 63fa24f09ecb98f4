"""Scalar number formats: E2M1, E8M0, E4M3, Mantissa8.

Drop-in for the reference's ``mxq.formats`` (src/formats.py).  The encoders
are served by the C-ABI's host-compiled copy of the kernels' arithmetic
header (``csrc/mxq_arith.cuh``), so the per-element / per-block API and the
CUDA quantizers share one implementation of every rounding rule.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = [
    "E2M1_GRID", "E2M1_MIDPOINTS", "E2M1_MAX", "E4M3_MAX", "Fp4Code", "E8M0Scale", "E4M3Value",
    "Mantissa8", "encode_e2m1", "decode_e2m1", "encode_e2m1_array", "decode_e2m1_array",
    "e8m0_floor", "encode_e4m3", "encode_e4m3_array", "decode_e4m3", "extract_mantissa8",
    "E4M3_TABLE",
]

# Representable E2M1 magnitudes by 3-bit index, and the decision boundaries
# between them (src/formats.py:46-56).
E2M1_GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
E2M1_MIDPOINTS = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
E2M1_MAX = 6.0
E8M0_BIAS = 127
E8M0_INVALID = 255
E4M3_MAX = 448.0


def _e4m3_table() -> np.ndarray:
    """Decode of all 256 E4M3 bytes (1/4/3, bias 7, subnormals, 0x7F/0xFF NaN)."""
    t = np.empty(256)
    for c in range(256):
        e, m = (c >> 3) & 15, c & 7
        if e == 0:
            v = m / 512.0
        elif e == 15 and m == 7:
            v = math.nan
        else:
            v = math.ldexp(8 + m, e - 10)
        t[c] = -v if c & 0x80 else v
    return t


E4M3_TABLE = _e4m3_table()


@dataclass(frozen=True)
class Fp4Code:
    """A 4-bit E2M1 code: bit 3 sign, bits 2..0 magnitude index."""

    code: int

    def __post_init__(self) -> None:
        if not 0 <= self.code <= 15:
            raise ValueError(f"4-bit code out of range: {self.code}")

    @property
    def sign(self) -> int:
        return self.code >> 3

    @property
    def magnitude_index(self) -> int:
        return self.code & 7

    @property
    def value(self) -> float:
        m = float(E2M1_GRID[self.code & 7])
        return -m if self.code & 8 else m


@dataclass(frozen=True)
class E8M0Scale:
    """Power-of-two scale 2**(biased_exponent - 127); 255 is reserved."""

    biased_exponent: int
    clamped: bool = False

    def __post_init__(self) -> None:
        if not 0 <= self.biased_exponent <= 254:
            raise ValueError(f"biased exponent out of range or reserved: {self.biased_exponent}")

    @property
    def exponent(self) -> int:
        return self.biased_exponent - E8M0_BIAS

    @property
    def value(self) -> float:
        return math.ldexp(1.0, self.exponent)


@dataclass(frozen=True)
class E4M3Value:
    """An E4M3 byte (max finite 448)."""

    byte: int

    def __post_init__(self) -> None:
        if not 0 <= self.byte <= 255:
            raise ValueError(f"byte out of range: {self.byte}")

    @property
    def value(self) -> float:
        return decode_e4m3(self)


@dataclass(frozen=True)
class Mantissa8:
    """8-bit mantissa fraction; the factor is 1 + m8/256."""

    m8: int

    def __post_init__(self) -> None:
        if not 0 <= self.m8 <= 255:
            raise ValueError(f"mantissa byte out of range: {self.m8}")

    @property
    def factor(self) -> float:
        return 1.0 + self.m8 / 256.0


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def encode_e2m1_array(values, saturate: bool = False) -> np.ndarray:
    """Nearest E2M1 codes, ties to the even magnitude index; -0 and negative
    flushes give code 0 (src/formats.py:185-200)."""
    v = _f64(values)
    out = np.empty(v.shape, dtype=np.uint8)
    rc = _lib.lib().mxq_host_encode_e2m1(v.ctypes.data, v.size, int(bool(saturate)), out.ctypes.data)
    if rc == _lib.ERR_NONFINITE:
        raise ValueError("cannot encode non-finite values")
    if rc == _lib.ERR_RANGE:
        raise ValueError("magnitude exceeds 6.0 and saturate=False")
    _lib.check(rc, "encode_e2m1")
    return out


def encode_e2m1(value: float, saturate: bool = False) -> Fp4Code:
    """Scalar encode (src/formats.py:154-177)."""
    if not math.isfinite(value):
        raise ValueError(f"cannot encode non-finite value: {value}")
    if abs(value) > E2M1_MAX and not saturate:
        raise ValueError(f"magnitude {abs(value)} exceeds 6.0 and saturate=False")
    return Fp4Code(int(encode_e2m1_array(np.array([value]), saturate=True)[0]))


def decode_e2m1(code: Fp4Code) -> float:
    return code.value


def decode_e2m1_array(codes) -> np.ndarray:
    """uint8 codes -> float64 grid values (src/formats.py:203-207)."""
    c = np.asarray(codes).astype(np.int64)
    mag = E2M1_GRID[c & 7]
    return np.where(c & 8, -mag, mag)


def e8m0_floor(x: float) -> E8M0Scale:
    """Largest power of two <= x, exponent clamped to [-127, 127]
    (src/formats.py:210-227)."""
    b, c = ctypes.c_uint8(), ctypes.c_int32()
    rc = _lib.lib().mxq_host_e8m0_floor(float(x), ctypes.byref(b), ctypes.byref(c))
    if rc:
        raise ValueError(f"e8m0_floor requires a positive finite input, got {x}")
    return E8M0Scale(b.value, clamped=bool(c.value))


def encode_e4m3_array(values) -> np.ndarray:
    """Nearest finite E4M3 (RNE, clamp 448, -0 -> +0) (src/formats.py:278-292)."""
    v = _f64(values)
    out = np.empty(v.shape, dtype=np.uint8)
    rc = _lib.lib().mxq_host_encode_e4m3(v.ctypes.data, v.size, out.ctypes.data)
    if rc == _lib.ERR_NONFINITE:
        raise ValueError("cannot encode non-finite values")
    _lib.check(rc, "encode_e4m3")
    return out


def encode_e4m3(value: float) -> E4M3Value:
    if not math.isfinite(value):
        raise ValueError(f"cannot encode non-finite value: {value}")
    return E4M3Value(int(encode_e4m3_array(np.array([value]))[0]))


def decode_e4m3(code: E4M3Value) -> float:
    v = float(E4M3_TABLE[code.byte])
    if math.isnan(v):
        raise ValueError(f"code 0x{code.byte:02X} is the E4M3 NaN encoding")
    return v


def extract_mantissa8(sf: float) -> Mantissa8:
    """Top 8 fraction bits of f32(sf) (src/formats.py:303-316)."""
    m = ctypes.c_uint8()
    if not (math.isfinite(sf) and sf > 0):
        raise ValueError(f"extract_mantissa8 requires a positive finite input, got {sf}")
    if abs(sf) > 3.4028234663852886e38:
        raise OverflowError("float too large to pack with f format")
    rc = _lib.lib().mxq_host_extract_mantissa8(float(sf), ctypes.byref(m))
    _lib.check(rc, "extract_mantissa8")
    return Mantissa8(m.value)
