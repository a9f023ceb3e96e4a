"""ctypes binding of libchp.so (include/chp.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or ``make
-C paper_2304_14074_b200/csrc``).  There is deliberately no CPU fallback:
``lib()`` raises if the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CHP_LIB: alternative build of the same library (kernel-variant A/B timing only)
LIB_PATH = os.environ.get("CHP_LIB") or os.path.join(_HERE, "libchp.so")

CHP_LINEAR_A, CHP_LINEAR_B, CHP_NONLINEAR_EYRE, CHP_NN_LINEAR_A = 0, 1, 2, 3
SYS_OK, SYS_NEWTON, SYS_NONFINITE, SYS_SINGULAR, SYS_CG, SYS_NN = 0, 1, 2, 3, 4, 5

# Exported symbols, one per declaration in include/chp.h.
EXPORTS = (
    "chp_version", "chp_status_str", "chp_ctx_create", "chp_ctx_destroy", "chp_last_error",
    "chp_sysinfo_reset", "chp_propagate", "chp_coarse_sweep", "chp_max_abs_diff",
    "chp_debug_trace", "chp_nn_propagate", "chp_propagate_hist", "chp_field_stats", "chp_probe_dfma",
    "chp_coarse_sweep_hop", "chp_hop_wait", "chp_hop_take", "chp_mem_alloc", "chp_mem_free",
    "chp_ipc_export", "chp_ipc_open", "chp_ipc_close",
)


class ChpGrid(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("m", C.c_int), ("pitch", C.c_int),
                ("h", C.c_double), ("hd", C.c_double), ("c1", C.c_double),
                ("s_main", C.c_double), ("s_edge", C.c_double), ("s_off1", C.c_double),
                ("s_off2", C.c_double)]


class ChpSpec(C.Structure):
    _fields_ = [("scheme", C.c_int), ("newton_max_iter", C.c_int), ("dt", C.c_double),
                ("eps", C.c_double), ("b", C.c_double), ("newton_tol", C.c_double),
                ("cg_tol", C.c_double), ("cg_max_iter", C.c_int), ("pad_", C.c_int)]


class ChpNNParams(C.Structure):
    _fields_ = [("n_subdomains", C.c_int), ("max_iter", C.c_int), ("warm_start", C.c_int),
                ("pad_", C.c_int), ("theta", C.c_double), ("tol", C.c_double),
                ("h2", C.c_double)]


class ChpHop(C.Structure):
    """include/chp.h chp_hop: the fused boundary hand-off of the sharded coarse chain."""
    _fields_ = [("peer_u", C.c_void_p), ("peer_stride", C.c_longlong),
                ("peer_changed", C.c_void_p), ("peer_flag", C.c_void_p),
                ("seq", C.c_uint), ("pad_", C.c_uint)]


class ChpSysInfo(C.Structure):
    _fields_ = [("status", C.c_int), ("fail_iter", C.c_int), ("fail_resid", C.c_double),
                ("newton_steps", C.c_longlong), ("newton_total", C.c_longlong),
                ("newton_max", C.c_int), ("cg_max", C.c_int), ("newton_maxres", C.c_double),
                ("cg_total", C.c_longlong)]


SYSINFO_DTYPE = np.dtype([("status", np.int32), ("fail_iter", np.int32),
                          ("fail_resid", np.float64), ("newton_steps", np.int64),
                          ("newton_total", np.int64), ("newton_max", np.int32),
                          ("cg_max", np.int32), ("newton_maxres", np.float64),
                          ("cg_total", np.int64)])
assert SYSINFO_DTYPE.itemsize == C.sizeof(ChpSysInfo) == 56

_lock = threading.RLock()
_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libchp.so and declare every entry point (no device work)."""
    if not os.path.exists(path):
        raise RuntimeError(
            f"libchp.so not found at {path}: build it with `python -c 'import "
            f"__graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    L = C.CDLL(path)
    vp, i, ll, d = C.c_void_p, C.c_int, C.c_longlong, C.c_double
    L.chp_version.restype = C.c_char_p
    L.chp_status_str.restype = C.c_char_p
    L.chp_status_str.argtypes = [i]
    L.chp_ctx_create.argtypes = [i, C.POINTER(vp)]
    L.chp_ctx_destroy.argtypes = [vp]
    L.chp_last_error.restype = C.c_char_p
    L.chp_last_error.argtypes = [vp]
    L.chp_sysinfo_reset.argtypes = [vp, vp, i, vp]
    L.chp_propagate.argtypes = [vp, C.POINTER(ChpGrid), C.POINTER(ChpSpec), i, i, vp, ll, vp,
                                ll, vp, vp, vp]
    L.chp_coarse_sweep.argtypes = [vp, C.POINTER(ChpGrid), C.POINTER(ChpSpec), i, i, i, i, i,
                                   vp, vp, vp, ll, ll, vp, vp, vp, vp]
    L.chp_coarse_sweep_hop.argtypes = [vp, C.POINTER(ChpGrid), C.POINTER(ChpSpec), i, i, i, i, i,
                                       vp, vp, vp, ll, ll, vp, vp, vp, C.POINTER(ChpHop), vp]
    L.chp_hop_wait.argtypes = [vp, vp, C.c_uint, vp]
    L.chp_hop_take.argtypes = [vp, C.POINTER(ChpGrid), i, vp, ll, vp, vp, ll, vp, ll, vp, C.c_uint, vp]
    L.chp_mem_alloc.argtypes = [vp, ll, C.POINTER(vp)]
    L.chp_mem_free.argtypes = [vp, vp]
    L.chp_ipc_export.argtypes = [vp, vp, C.c_char_p]
    L.chp_ipc_open.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
    L.chp_ipc_close.argtypes = [vp, vp]
    L.chp_max_abs_diff.argtypes = [vp, C.POINTER(ChpGrid), i, vp, ll, vp, ll, vp, vp]
    L.chp_debug_trace.argtypes = [vp, i]
    L.chp_field_stats.argtypes = [vp, C.POINTER(ChpGrid), i, vp, ll, vp, vp]
    L.chp_probe_dfma.argtypes = [vp, i, i, vp, vp]
    L.chp_propagate_hist.argtypes = [vp, C.POINTER(ChpGrid), C.POINTER(ChpSpec), i, i, vp, ll,
                                     vp, ll, vp, vp, vp, i, vp]
    L.chp_nn_propagate.argtypes = [vp, C.POINTER(ChpGrid), C.POINTER(ChpNNParams), d, d, i, i,
                                   vp, ll, vp, ll, vp, vp, vp, vp, vp]
    for name in EXPORTS:
        if name not in ("chp_version", "chp_status_str", "chp_last_error"):
            getattr(L, name).restype = C.c_int
    return L


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            _lib = load_library()
        return _lib


class NativeError(RuntimeError):
    pass


class Context:
    """One chp_ctx per CUDA device (the factor-cache owner)."""

    _by_device: dict = {}

    def __init__(self, device: int):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2304_14074_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        self.L = lib()
        h = C.c_void_p()
        with torch.cuda.device(device):
            st = self.L.chp_ctx_create(device, C.byref(h))
        if st != 0:
            raise NativeError(f"chp_ctx_create failed: {self.L.chp_status_str(st).decode()}")
        self.h = h

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        import torch
        if device is None:
            device = torch.cuda.current_device()
        with _lock:
            ctx = cls._by_device.get(device)
            if ctx is None:
                ctx = cls(device)
                cls._by_device[device] = ctx
        return ctx

    def check(self, st: int, what: str):
        if st != 0:
            msg = self.L.chp_last_error(self.h).decode()
            if st == 1:
                raise ValueError(f"{what}: {msg}")
            raise NativeError(f"{what}: {self.L.chp_status_str(st).decode()}: {msg}")

    def close(self):
        if self.h:
            self.L.chp_ctx_destroy(self.h)
            self.h = None


def stream_ptr(stream=None, device=None) -> C.c_void_p:
    """The given stream, or the current stream of ``device`` (a torch device, an
    index or None for the current device): the native entry points run on the
    context's device, so the default stream must be that device's."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())
