"""ctypes binding of the C-ABI library (include/mxq200.h).

The library is built in-tree (``paper_2603_08713_b200/_lib/libmxq200.so``,
see ``build.py``).  There is no fallback: if the library is missing or the
process has no B200, the product entry points raise instead of computing
anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MXQ_LIB_PATH") or os.path.join(_HERE, "_lib", "libmxq200.so")  # (override: development A/B builds)

MXQ_F32, MXQ_BF16 = 0, 1
ERR_INVALID, ERR_NONFINITE, ERR_UNSUPPORTED, ERR_RANGE = -1, -2, -3, -4
ST_NONFINITE, ST_BAD_E8M0, ST_BAD_E4M3, ST_OVERFLOW = 1, 2, 4, 8

VARIANT_CODE = {"ocp32": 0, "mx16": 1, "mx16_oas": 2, "mbs_s": 3, "mbs_d": 4, "nvfp4": 5}


class QT(ctypes.Structure):
    """Mirror of ``mxq_qtensor`` (include/mxq200.h)."""

    _fields_ = [
        ("variant", ctypes.c_int32), ("block_size", ctypes.c_int32),
        ("macro_size", ctypes.c_int32), ("sf_format", ctypes.c_int32),
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("codes", ctypes.c_void_p), ("codes_ld", ctypes.c_int64),
        ("scales", ctypes.c_void_p), ("scales_ld", ctypes.c_int64),
        ("scales_mma", ctypes.c_void_p), ("sf_kpad", ctypes.c_int64),
        ("mant", ctypes.c_void_p), ("mant_ld", ctypes.c_int64),
        ("sig_t", ctypes.c_void_p), ("sig_t_ld", ctypes.c_int64),
        ("tensor_scale", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_I32, _I64, _U32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
_PQT = ctypes.POINTER(QT)

SIGNATURES = {
    "mxq_version": (ctypes.c_int, []),
    "mxq_last_error": (ctypes.c_char_p, []),
    "mxq_device_ok": (ctypes.c_int, []),
    "mxq_debug_set_trace": (None, [_P]),
    "mxq_quantize": (ctypes.c_int, [_P, _I32, _I64, _PQT, _I32, _P, _I32, _I32, _P, _P]),
    "mxq_quantize_mbs_lut": (ctypes.c_int, [_P, _I32, _I64, _PQT, _P, _I32, _P, _P, _P]),
    "mxq_dequantize": (ctypes.c_int, [_PQT, _P, _I64, _P, _P]),
    "mxq_qsnr_workspace_bytes": (_I64, [_I64]),
    "mxq_qsnr": (ctypes.c_int, [_P, _I32, _I64, _PQT, _P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "mxq_gemm": (ctypes.c_int, [_PQT, _PQT, _P, _I32, _I64, _P, _P]),
    "mxq_quantize_gemm": (ctypes.c_int, [_P, _I32, _I64, _PQT, _PQT, _P, _I32, _I64, _P, _P]),
    "mxq_gemm_grouped": (ctypes.c_int, [_PQT, _PQT, _I32, _P, _I32, _I64, _P, _P]),
    "mxq_gemm_exact": (ctypes.c_int, [_PQT, _PQT, _P, _I64, _P, _P]),
    "mxq_matmul_reference": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _P]),
    "mxq_build_gemm_layout": (ctypes.c_int, [_PQT, _I32, _P]),
    "mxq_host_encode_e2m1": (ctypes.c_int, [_P, _I64, _I32, _P]),
    "mxq_host_encode_e4m3": (ctypes.c_int, [_P, _I64, _P]),
    "mxq_host_e8m0_floor": (ctypes.c_int, [ctypes.c_double, _P, _P]),
    "mxq_host_extract_mantissa8": (ctypes.c_int, [ctypes.c_double, _P]),
    "mxq_host_block_scale": (ctypes.c_int, [_P, _I64, _I32, _P, _P]),
    "mxq_host_static_m8": (ctypes.c_int, [ctypes.c_double, _P]),
    "mxq_host_e8m0_closed_form": (ctypes.c_int, [_P, _I64, _I32, _P]),
    "mxq_host_dequant_element": (ctypes.c_float, [_I32, _U32, _U32, _U32, ctypes.c_double]),
    "mxq_host_mbs_choose": (ctypes.c_int, [_P, _I64, _P, _I32, _I32, _P, _P]),
}

_lib = None
_lock = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load (once) the in-tree C-ABI library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is missing: run `python -m paper_2603_08713_b200.build` "
                    "(or __graft_entry__.build()); there is no CPU fallback")
            l = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(l, name)
                fn.restype = res
                fn.argtypes = args
            _lib = l
    return _lib


def last_error() -> str:
    return lib().mxq_last_error().decode()


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if rc == 0:
        return
    msg = last_error()
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg}")


_device_ok = False
_devices: dict = {}


def require_device() -> torch.device:
    """The CUDA device the product path runs on (fails loudly without one).
    The availability check and the library load run once per process."""
    global _device_ok
    if not _device_ok:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_08713_b200 needs a CUDA B200; no CUDA device is visible")
        lib()
        _device_ok = True
    idx = torch.cuda.current_device()
    d = _devices.get(idx)
    if d is None:
        d = _devices[idx] = torch.device("cuda", idx)
    return d


def stream_handle() -> int:
    """cudaStream_t of the current stream (torch's internal accessor: the
    public torch.cuda.current_stream() costs ~10 us of Python per call)."""
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def status_message(bits: int) -> str | None:
    """The reference's error text for device status bits."""
    if bits & ST_NONFINITE:
        return "tensor contains non-finite elements"           # src/quantize.py:581-582
    if bits & ST_OVERFLOW:
        return "cannot encode non-finite values"               # src/formats.py:196-197
    if bits & ST_BAD_E8M0:
        return "corrupt block scale: E8M0 code 255 is reserved"  # src/quantize.py:239-240
    if bits & ST_BAD_E4M3:
        return "corrupt block scale: E4M3 NaN code"            # src/quantize.py:235-236
    if bits:
        return f"device status 0x{bits:x}"
    return None


def raise_on_status(status: torch.Tensor) -> None:
    bits = int(status[0].item()) & 0xFFFFFFFF
    msg = status_message(bits)
    if msg:
        raise ValueError(msg)
