"""ctypes binding of the C ABI in include/hankelfft_b200.h.

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``)
as ``paper_1401_6238_b200/libhankelfft_b200.so``.  There is no fallback: if the
library or a CUDA device is missing every product raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HK_OK = 0
HK_EINVAL = -1
HK_ECUDA = -2
HK_ENOMEM = -3
HK_EUNSUPPORTED = -4

HK_C128 = 0
HK_F64 = 1
HK_SPEC = 2
HK_C64 = 3
HK_F32 = 4

LIB_NAME = "libhankelfft_b200.so"
LIB_PATH = os.environ.get("HK_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)


class Operand(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("batch_stride", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None
_lock = threading.Lock()

_SIGS = {
    "hk_version": (ctypes.c_int, []),
    "hk_last_error": (ctypes.c_char_p, []),
    "hk_plan_create_hankel": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]),
    "hk_plan_create_block": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                            ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(ctypes.c_int64)]),
    "hk_plan_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "hk_plan_fft_len": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int]),
    "hk_plan_spectrum_len": (ctypes.c_int64, [ctypes.c_void_p]),
    "hk_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int64]),
    "hk_spectrum": (ctypes.c_int, [ctypes.c_void_p, Operand, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]),
    "hk_tvp_partial": (ctypes.c_int, [ctypes.c_void_p, Operand, ctypes.POINTER(Operand),
                                      ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "hk_tvp_partial_host": (ctypes.c_int, [ctypes.c_void_p, Operand, ctypes.c_void_p,
                                           ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                           ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]),
    "hk_tvp_full": (ctypes.c_int, [ctypes.c_void_p, Operand, ctypes.POINTER(Operand),
                                   ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]),
    "hk_vector_spectra": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_void_p]),
    "hk_times_matrices_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p,
                                                            ctypes.POINTER(ctypes.c_int64),
                                                            ctypes.c_int, ctypes.c_int64]),
    "hk_times_matrices": (ctypes.c_int, [ctypes.c_void_p, Operand,
                                         ctypes.POINTER(ctypes.c_void_p),
                                         ctypes.POINTER(ctypes.c_int64),
                                         ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                                         ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def load_library(path: str = LIB_PATH):
    """Load the C-ABI library (no CUDA device needed just to load it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{LIB_NAME} is not built ({path}); run `make` or "
                    "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no CPU "
                    "fallback for the Hankel product path")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == HK_OK:
        return
    msg = load_library().hk_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == HK_EINVAL:
        raise ValueError(text)
    if rc == HK_EUNSUPPORTED:
        raise NotImplementedError(text)
    raise RuntimeError(f"hankelfft_b200 error {rc}: {text}")


def i64_array(values):
    arr = (ctypes.c_int64 * len(values))(*[int(v) for v in values])
    return arr


class Plan:
    """Owning wrapper of an ``hk_plan*`` (immutable, bound to one device)."""

    def __init__(self, handle, device: int, kind: str, key):
        self.handle = handle
        self.device = device
        self.kind = kind
        self.key = key
        lib = load_library()
        self.fft_lens = []
        lvl = 0
        while True:
            L = lib.hk_plan_fft_len(handle, lvl)
            if L < 0:
                break
            self.fft_lens.append(int(L))
            lvl += 1
        self.spectrum_len = int(lib.hk_plan_spectrum_len(handle))
        # > 0 for two-level (workspace-backed) plans
        self.workspace_per_item = int(lib.hk_workspace_bytes(handle, 1))

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.hk_plan_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass
        self.handle = None


_plans: dict = {}
_plans_lock = threading.Lock()


def hankel_plan(shape, device: int, fft_len: int = 0) -> Plan:
    """Cached plan per (device, shape, fft_len)."""
    key = ("hankel", device, tuple(int(n) for n in shape), int(fft_len))
    with _plans_lock:
        p = _plans.get(key)
        if p is not None:
            return p
        lib = load_library()
        h = ctypes.c_void_p()
        sizes = i64_array(shape)
        check(lib.hk_plan_create_hankel(ctypes.byref(h), len(shape), sizes, int(fft_len)),
              "hk_plan_create_hankel")
        p = Plan(h, device, "hankel", key)
        _plans[key] = p
        return p


def block_plan(order, level_shapes, device: int, fft_lens=None) -> Plan:
    key = ("block", device, int(order), tuple(tuple(int(n) for n in lv) for lv in level_shapes),
           None if fft_lens is None else tuple(int(x) for x in fft_lens))
    with _plans_lock:
        p = _plans.get(key)
        if p is not None:
            return p
        lib = load_library()
        h = ctypes.c_void_p()
        flat = [n for lv in level_shapes for n in lv]
        fl = None if fft_lens is None else i64_array(fft_lens)
        check(lib.hk_plan_create_block(ctypes.byref(h), int(order), len(level_shapes),
                                       i64_array(flat), fl), "hk_plan_create_block")
        p = Plan(h, device, "block", key)
        _plans[key] = p
        return p
