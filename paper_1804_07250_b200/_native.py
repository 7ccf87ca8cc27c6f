"""ctypes binding of libtsb.so (the C ABI in include/tsb.h).

The library is built in-tree (``_lib/libtsb.so``) by :func:`build`.  There is
no CPU fallback: if the library or an sm_100 device is missing, every call
raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import glob
import os
import subprocess
import threading

import numpy as np

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libtsb.so")
CSRC = os.path.join(HERE, "csrc")
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
]

_lib = None
_lock = threading.Lock()
_device = int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("TSB_DEVICE") is None else int(
    os.environ["TSB_DEVICE"])

(OK, E_VALUE, E_INCONSISTENT, E_CAPACITY, E_CUDA, E_NODEVICE, E_CONVERGENCE, E_DOMAIN, E_UNTILEABLE,
 E_INFEASIBLE) = range(10)
_EXC = {
    E_VALUE: ValueError,
    E_INCONSISTENT: errors.InconsistencyError,
    E_CAPACITY: errors.CapacityError,
    E_CUDA: RuntimeError,
    E_NODEVICE: RuntimeError,
    E_CONVERGENCE: errors.ConvergenceCapExceeded,
    E_DOMAIN: errors.DomainError,
    E_UNTILEABLE: errors.UntileableDomain,
    E_INFEASIBLE: errors.InfeasibleBoundary,
}


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def build(verbose: bool = False) -> str:
    """Compile libtsb.so for sm_100a with nvcc (works without a GPU)."""
    os.makedirs(LIB_DIR, exist_ok=True)
    cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB_PATH, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True, cwd=HERE)
    return LIB_PATH


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "tsb.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


_vp = ctypes.c_void_p
_i = ctypes.c_int
_u64 = ctypes.c_uint64

_SIGS = {
    "tsb_last_error": (ctypes.c_char_p, []),
    "tsb_abi_version": (_i, []),
    "tsb_device_info": (_i, [_i, _vp, _vp, _vp, _vp]),
    "tsb_grid_components": (_i, [_i, _vp, _i, _i, _vp]),
    "tsb_tri_check": (_i, [_i, _vp, _vp, _i, _i, _vp, _vp]),
    "tsb_uniform_grid": (_i, [_i, _u64, _i, _i, _u64, _i, _vp]),
    "tsb_domino_create": (_i, [_i, _i, _i, _vp, _vp]),
    "tsb_domino_destroy": (_i, [_vp]),
    "tsb_domino_create_window": (_i, [_i, _i, _i, _i, _vp, _vp]),
    "tsb_domino_upload_rows": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_download_rows": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_set_stream": (_i, [_vp, _vp]),
    "tsb_domino_set_p_up": (_i, [_vp, _vp]),
    "tsb_domino_set_p_up_parity": (_i, [_vp, ctypes.c_double, ctypes.c_double]),
    "tsb_domino_upload": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_download": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_walk": (_i, [_vp, _i, _i, _vp, _u64, _u64]),
    "tsb_domino_sweep": (_i, [_vp, _i, _i, _vp, _u64, _i]),
    "tsb_domino_sync": (_i, [_vp]),
    "tsb_domino_set_window": (_i, [_vp, _i, _i]),
    "tsb_domino_set_collapse": (_i, [_vp, _i]),
    "tsb_domino_row_bytes": (_i, [_vp, _vp]),
    "tsb_domino_get_rows": (_i, [_vp, _i, _i, _i, _vp]),
    "tsb_domino_set_rows": (_i, [_vp, _i, _i, _i, _vp]),
    "tsb_domino_walk_host": (_i, [_i, _vp, _i, _i, _vp, _vp, _vp, _u64]),
    "tsb_domino_heights": (_i, [_vp, _i, _i, _i, _vp]),
    "tsb_domino_extremal": (_i, [_vp, _i, _i, _i, _i]),
    "tsb_domino_coalesced": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_orientation_add": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_height_sum_add": (_i, [_vp, _i, _i, _i, _i, _vp]),
    "tsb_domino_serialize": (_i, [_vp, _i, _vp, ctypes.c_size_t, _vp]),
    "tsb_sv_serialize": (_i, [_vp, _i, _vp, ctypes.c_size_t, _vp]),
    "tsb_loz_serialize": (_i, [_vp, _i, _vp, ctypes.c_size_t, _vp]),
    "tsb_domino_strip_init": (_i, [_vp, _i, _i, _i, _vp]),
    "tsb_domino_strip_connect": (_i, [_vp, _vp, _vp]),
    "tsb_domino_strip_connect_local": (_i, [_vp, _vp, _vp]),
    "tsb_domino_strip_walk": (_i, [_vp, _u64, _u64, _u64]),
    "tsb_domino_strip_seed": (_i, [_vp, _u64]),
    "tsb_domino_strip_step": (_i, [_vp, _u64, _u64, _i]),
    "tsb_domino_strip_status": (_i, [_vp, _vp, _vp]),
    "tsb_domino_strip_close": (_i, [_vp]),
    "tsb_sv_observe_add": (_i, [_vp, _i, _i, _i, _vp]),
    "tsb_sv_height_sum_add": (_i, [_vp, _i, _i, _vp]),
    "tsb_domino_replicate": (_i, [_vp, _i, _i, _i, _i]),
    "tsb_domino_cftp": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp]),
    "tsb_sv_create": (_i, [_i, _i, _i, _vp]),
    "tsb_sv_destroy": (_i, [_vp]),
    "tsb_sv_set_stream": (_i, [_vp, _vp]),
    "tsb_sv_set_p_high": (_i, [_vp, _vp]),
    "tsb_sv_upload": (_i, [_vp, _i, _i, _vp]),
    "tsb_sv_download": (_i, [_vp, _i, _i, _vp]),
    "tsb_sv_walk": (_i, [_vp, _i, _i, _vp, _u64, _u64]),
    "tsb_sv_sweep": (_i, [_vp, _i, _i, _vp, _u64, _i]),
    "tsb_sv_sync": (_i, [_vp]),
    "tsb_sv_set_collapse": (_i, [_vp, _i]),
    "tsb_sv_extremal": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "tsb_sv_coalesced": (_i, [_vp, _i, _i, _vp]),
    "tsb_sv_replicate": (_i, [_vp, _i, _i, _i, _i]),
    "tsb_sv_cftp": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp]),
    "tsb_loz_create": (_i, [_i, _i, _i, _i, _vp, _vp, _vp]),
    "tsb_loz_destroy": (_i, [_vp]),
    "tsb_loz_set_stream": (_i, [_vp, _vp]),
    "tsb_loz_set_p_up": (_i, [_vp, _vp]),
    "tsb_loz_upload": (_i, [_vp, _i, _i, _vp]),
    "tsb_loz_download": (_i, [_vp, _i, _i, _vp]),
    "tsb_loz_walk": (_i, [_vp, _i, _i, _vp, _u64, _u64]),
    "tsb_loz_sweep": (_i, [_vp, _i, _i, _vp, _u64, _i]),
    "tsb_loz_sync": (_i, [_vp]),
    "tsb_loz_set_collapse": (_i, [_vp, _i]),
    "tsb_loz_heights": (_i, [_vp, _i, _i, _i, _vp]),
    "tsb_loz_height_sum_add": (_i, [_vp, _i, _i, _i, _i, _vp]),
    "tsb_loz_extremal": (_i, [_vp, _i, _i, _i, _i]),
    "tsb_loz_coalesced": (_i, [_vp, _i, _i, _vp]),
    "tsb_loz_replicate": (_i, [_vp, _i, _i, _i, _i]),
    "tsb_loz_cftp": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp]),
}


PROGRESS_FN = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p)


def declared_symbols() -> list[str]:
    """Every entry point include/tsb.h declares (parsed from the header)."""
    import re

    text = open(os.path.join(ROOT, "include", "tsb.h")).read()
    return sorted(set(re.findall(r"\b(tsb_[a-z0-9_]+)\s*\(", text)))


def lib() -> ctypes.CDLL:
    """Load libtsb.so (building it first if sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("TSB_LIB")  # A/B experiments: load another build of the same ABI
            if path is None and _stale():
                try:
                    build()
                except (OSError, subprocess.CalledProcessError) as exc:
                    if not os.path.exists(LIB_PATH):
                        raise RuntimeError(f"libtsb.so is missing and could not be built: {exc}")
            L = ctypes.CDLL(path or LIB_PATH)
            for name, (res, args) in _SIGS.items():
                if path is not None and not hasattr(L, name):
                    continue  # an older A/B build may lack newer entry points
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().tsb_last_error().decode(errors="replace")
    raise _EXC.get(rc, RuntimeError)(msg)


def device() -> int:
    return _device


def set_device(d: int) -> None:
    global _device
    _device = int(d)


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def u64(x: int) -> int:
    return int(x) & 0xFFFFFFFFFFFFFFFF


_has_device = None


def has_device() -> bool:
    """True when libtsb loads and sees an sm_100 device (no exception)."""
    global _has_device
    if _has_device is None:
        try:
            sm = ctypes.c_int()
            major = ctypes.c_int()
            _has_device = lib().tsb_device_info(0, ctypes.byref(sm), ctypes.byref(major), None, None) == OK \
                and major.value == 10
        except Exception:
            _has_device = False
    return _has_device
