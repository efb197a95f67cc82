"""ctypes binding of libcmb200.so (declared in include/cmb200.h).

There is deliberately no CPU fallback: if the shared library is missing or
cannot reach a CUDA device, every entry point raises ``DeviceError``.
ctypes releases the GIL for the duration of each foreign call, so long GPU
calls do not block other Python threads (the reference's numpy kernels had
the same property, pkg/binding/src/crossmap_binding/__init__.py:7-9).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (CrossmapError, DeviceError, ParameterError, SeriesTooShortError,
                     ZeroVarianceError)

# CMB_LIB names an alternative build of the same library (A/B timing of two builds).
LIB_PATH = Path(os.environ.get("CMB_LIB") or Path(__file__).resolve().parent / "libcmb200.so")
LIB_VERSION = 100  # 0.1.0

_i32, _i64, _dbl, _vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
_P = C.c_void_p  # every array travels as a raw pointer

_SIGNATURES = {
    "cmb_version": ([], C.c_int),
    "cmb_last_error": ([], C.c_char_p),
    "cmb_device_count": ([_P], C.c_int),
    "cmb_diagnostics": ([C.c_int, _P, C.c_int], C.c_int),
    "cmb_shutdown": ([], C.c_int),
    "cmb_pairwise_distances": ([C.c_int, _P, _i64, C.c_int, C.c_int, _P], C.c_int),
    "cmb_partial_sort_topk": ([C.c_int, _P, _i64, C.c_int, _P, _P], C.c_int),
    "cmb_normalize_weights": ([C.c_int, _P, _i64, C.c_int, _P], C.c_int),
    "cmb_knn_table": ([C.c_int, _P, _i64, C.c_int, C.c_int, C.c_int, _P, _P, _P], C.c_int),
    "cmb_pearson": ([C.c_int, _P, _P, _i64, _P], C.c_int),
    "cmb_lookup": ([C.c_int, _P, _P, _i64, C.c_int, C.c_int, _P, _i64, _i64, _P, _P], C.c_int),
    "cmb_simplex": ([C.c_int, _P, _i64, C.c_int, C.c_int, C.c_int, _P], C.c_int),
    "cmb_edim": ([C.c_int, _P, _i64, _i64, C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),
    "cmb_xmap": ([C.c_int, _P, _i64, _i64, _P, C.c_int, _P, C.c_int, _P], C.c_int),
    "cmb_xmap64": ([C.c_int, _P, _i64, _i64, _P, C.c_int, _P, C.c_int, _P], C.c_int),
    "cmb_xmap_predict": ([C.c_int, _P, _i64, _i64, _P, C.c_int, _P, _P, _i64, _P, C.c_int, _P, _P], C.c_int),
    "cmb_xmap_dev": ([C.c_int, _P, _i64, _i64, _i64, _P, C.c_int, _i64, _i64, _P, _i64, _P, _P],
                     C.c_int),
    "cmb_nccl_unique_id": ([_P], C.c_int),
    "cmb_nccl_init_rank": ([C.c_int, _P, C.c_int, C.c_int], C.c_int),
    "cmb_nccl_info": ([C.c_int, _P, _P, _P], C.c_int),
    "cmb_nccl_destroy": ([C.c_int], C.c_int),
    "cmb_xmap_rank": ([C.c_int, _P, _i64, _i64, _P, C.c_int, _P, _P, _P], C.c_int),
    "cmb_xmap_multi": ([_P, C.c_int, _P, _i64, _i64, _P, C.c_int, _P, _P], C.c_int),
    "cmb_edim_dev": ([C.c_int, _P, _i64, _i64, _i64, C.c_int, C.c_int, C.c_int, _P, _P, _P],
                     C.c_int),
    "cmb_ccm_convergence": ([C.c_int, _P, _i64, _i64, C.c_int, C.c_int, _P, _P, _i64, _P, C.c_int,
                             C.c_int, _P, _P], C.c_int),
    "cmb_format_skill_csv": ([C.c_int, _P, C.c_int, C.c_int, _i64, _i64, _i64, _i64, _P, _P, _P, _i64,
                              _P], C.c_int),
    "cmb_csv_header": ([_P, _i64, _P, _i64, _P, _i64, _P, _P], C.c_int),
    "cmb_csv_body": ([_P, _i64, C.c_int, _i64, _P, _i64, _P, _P, _i64, _P, _P, _i64, _P, _i64, _P, _P, _i64,
                      _P], C.c_int),
}

EXPORTS = tuple(_SIGNATURES)

_ERRORS = {
    -1: ParameterError,
    -2: SeriesTooShortError,
    -3: ZeroVarianceError,
    -10: DeviceError,
    -11: DeviceError,
    -12: DeviceError,
}

_lock = threading.Lock()
_lib = None


def load(path: Path | str | None = None):
    """Load (once) and return the CDLL; raise DeviceError if it is absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"{p.name} is not built ({p}); run `python -m paper_2105_12301_b200.build_native` "
                "-- there is no CPU fallback")
        try:
            lib = C.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - broken build
            raise DeviceError(f"cannot load {p}: {exc}") from None
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.cmb_version() != LIB_VERSION:
            raise DeviceError(f"{p.name} version {lib.cmb_version()} != {LIB_VERSION}")
        if path is None:
            _lib = lib
        return lib


def device() -> int:
    """CUDA device used by the single-device API (env CMB_DEVICE, default 0)."""
    return int(os.environ.get("CMB_DEVICE", "0"))


def check(code: int) -> None:
    if code == 0:
        return
    msg = (load().cmb_last_error() or b"").decode(errors="replace")
    raise _ERRORS.get(code, CrossmapError)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(a: np.ndarray | None):
    """Raw pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags.c_contiguous, "arrays crossing the C ABI must be C-contiguous"
    return a.ctypes.data


def diagnostics(dev: int | None = None) -> dict:
    """Counters since the previous call: kNN rows re-selected by the exact fp64 fallback."""
    out = np.zeros(8, dtype=np.int64)
    call("cmb_diagnostics", device() if dev is None else dev, ptr(out), 8)
    return {"exact_fallback_rows": int(out[0]), "rows_checked": int(out[1]),
            "kernel_launches": int(out[2])}


def device_count() -> int:
    n = np.zeros(1, dtype=np.int32)
    check(load().cmb_device_count(ptr(n)))
    return int(n[0])


_MADV_HUGEPAGE = 14
_HUGE = 2 << 20


def host_empty(shape, dtype) -> np.ndarray:
    """np.empty for large result arrays, backed by transparent huge pages where the
    kernel allows it (madvise mode): an N x N float32 cross map at N = 53,053 is
    2.8 M 4 KB page faults on first touch, 5.5 k with 2 MB pages."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    if n < (64 << 20):
        return np.empty(shape, dtype)
    raw = np.empty(n + _HUGE, dtype=np.uint8)
    off = (-raw.ctypes.data) % _HUGE
    buf = raw[off:off + n]
    try:
        libc = C.CDLL(None, use_errno=True)
        libc.madvise(C.c_void_p(buf.ctypes.data), C.c_size_t(n - n % _HUGE), _MADV_HUGEPAGE)
    except (OSError, AttributeError):  # pragma: no cover - platform without madvise
        pass
    return buf.view(dtype).reshape(shape)
