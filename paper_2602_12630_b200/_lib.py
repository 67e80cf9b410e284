"""ctypes binding of libtcb200.so (include/tc_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every compute
call raises.  Status codes map onto the exception types the reference raises
(field.py:41-42, mvpoly.py:30-57, backend.py:26-27, 319-333).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TC_LIB", os.path.join(HERE, "libtcb200.so"))   # TC_LIB: A/B builds

TC_OK = 0
TC_ERR_VALUE, TC_ERR_INDEX, TC_ERR_ZERO_DIVISION, TC_ERR_BACKEND, TC_ERR_OVERFLOW = 1, 2, 3, 4, 5
TC_ERR_CUDA, TC_ERR_MEMORY, TC_ERR_ARGUMENT = 10, 11, 12

DTYPE_F16, DTYPE_BF16, DTYPE_F32, DTYPE_F64, DTYPE_FP_LIMBS = 1, 2, 3, 4, 16
SRS_MONOMIAL, SRS_LAGRANGE, SRS_SUBGRID = 1, 2, 4
ROUTE_AUTO, ROUTE_MONOMIAL, ROUTE_LAGRANGE = 0, 1, 2


class BackendError(RuntimeError):
    """Same role as tensorcommit.backend.BackendError (backend.py:26-27)."""


_EXC = {
    TC_ERR_VALUE: ValueError,
    TC_ERR_INDEX: IndexError,
    TC_ERR_ZERO_DIVISION: ZeroDivisionError,
    TC_ERR_BACKEND: BackendError,
    TC_ERR_OVERFLOW: OverflowError,
    TC_ERR_CUDA: RuntimeError,
    TC_ERR_MEMORY: MemoryError,
    TC_ERR_ARGUMENT: ValueError,
}

_P = C.c_void_p
_U8P = C.POINTER(C.c_uint8)
_U32P = C.POINTER(C.c_uint32)

# (name, restype, argtypes)
_SIGS = [
    ("tc_abi_version", C.c_int, []),
    ("tc_ctx_create", C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    ("tc_ctx_destroy", C.c_int, [_P]),
    ("tc_ctx_set_stream", C.c_int, [_P, _P]),
    ("tc_ctx_set_pipelined", C.c_int, [_P, C.c_int]),
    ("tc_ctx_synchronize", C.c_int, [_P]),
    ("tc_ctx_last_error", C.c_char_p, [_P]),
    ("tc_ctx_launch_count", C.c_uint64, [_P]),
    ("tc_ctx_set_profiling", C.c_int, [_P, C.c_int]),
    ("tc_ctx_kernel_stats", C.c_int, [_P, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_double)]),
    ("tc_ctx_check_guards", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("tc_srs_generate", C.c_int, [_P, _U32P, C.c_int, C.c_char_p, C.c_int, C.POINTER(_P)]),
    ("tc_srs_load", C.c_int, [_P, _U32P, C.c_int, C.c_char_p, C.c_char_p, C.POINTER(_P)]),
    ("tc_srs_derive_lagrange", C.c_int, [_P, _P]),
    ("tc_srs_export", C.c_int, [_P, _P, C.c_int, C.c_uint64, C.c_uint64, _P]),
    ("tc_srs_export_axis", C.c_int, [_P, _P]),
    ("tc_srs_has", C.c_int, [_P, C.c_int]),
    ("tc_srs_size", C.c_uint64, [_P]),
    ("tc_srs_prepare", C.c_int, [_P, _P, C.c_int, C.c_int]),
    ("tc_srs_table_bytes", C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("tc_srs_destroy", C.c_int, [_P]),
    ("tc_quantize", C.c_int, [_P, _P, C.c_int, C.c_uint64, C.c_int, _P]),
    ("tc_interpolate", C.c_int, [_P, _P, _U32P, C.c_int]),
    ("tc_evaluate", C.c_int, [_P, _P, _U32P, C.c_int, C.c_char_p, _P]),
    ("tc_open_quotients", C.c_int, [_P, _P, _U32P, C.c_int, C.c_char_p, _P, _P]),
    ("tc_msm", C.c_int, [_P, _P, C.c_int, _P, C.c_uint64, _P]),
    ("tc_commit", C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_commit_batch", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_commit_batch_host", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_commit_stream", C.c_int, [_P, _P, C.POINTER(_P), C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_commit_stream_reset", C.c_int, [_P]),
    ("tc_open", C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_char_p, C.c_int, _P, _P]),
    ("tc_open_batch", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int, _P, _P]),
    ("tc_open_slices", C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_uint32, C.c_uint32, _P]),
    ("tc_open_batch_sliced", C.c_int, [_P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_char_p, _P, _P]),
    ("tc_terkle_build", C.c_int, [_P, _P, C.c_char_p, C.c_uint64, _P, C.POINTER(C.c_uint64)]),
    ("tc_commit_tree", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P,
                                 C.POINTER(C.c_uint64), _P, C.POINTER(C.c_uint64)]),
    ("tc_commit_tree_launch", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_commit_stream_tree_launch", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_commit_tree_finish", C.c_int, [_P, _P, _P, C.POINTER(C.c_uint64), _P, C.POINTER(C.c_uint64)]),
    ("tc_commit_stream_tree", C.c_int, [_P, _P, C.POINTER(_P), C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int,
                                        _P, _P, _P, C.POINTER(C.c_uint64), _P, C.POINTER(C.c_uint64)]),
    ("tc_commit_points_launch", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("tc_tree_from_points_launch", C.c_int, [_P, _P, _P, _P, C.c_uint64, C.c_int]),
    ("tc_pairing", C.c_int, [C.c_char_p, C.c_char_p, _P]),
    ("tc_verify_host", C.c_int, [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_int)]),
    ("tc_host_hash_point", C.c_int, [C.c_char_p, C.c_int, _P]),
    ("tc_host_field_inv", C.c_int, [C.c_int, C.c_int, _U32P, _U32P]),
    ("tc_host_hash_to_scalar", C.c_int, [C.c_char_p, C.c_uint32, C.c_char_p, C.c_uint32, _P]),
    ("tc_host_fq_mul", C.c_int, [_U32P, _U32P, _U32P]),
    ("tc_host_fp_mul", C.c_int, [_U32P, _U32P, _U32P]),
    ("tc_host_g_mul", C.c_int, [C.c_char_p, _P]),
    ("tc_debug_field", C.c_int, [_P, C.c_int, _P, _P, _P, C.c_uint64]),
    ("tc_measure_imad_peak", C.c_int, [_P, C.POINTER(C.c_double)]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None
_lib_lock = threading.Lock()


def lib():
    """The loaded library (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
                L = C.CDLL(LIB_PATH)
                for name, res, args in _SIGS:
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(status: int, ctx=None, what: str = ""):
    if status == TC_OK:
        return
    msg = ""
    if ctx is not None:
        raw = lib().tc_ctx_last_error(ctx)
        msg = raw.decode() if raw else ""
    exc = _EXC.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what and msg else (msg or what or f"tc status {status}"))


class Context:
    """One library context per CUDA device, re-bound to torch's current stream per call."""

    _by_device: dict = {}
    _guard = threading.Lock()

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2602_12630_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        self.lock = threading.RLock()
        h = _P()
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream(device).cuda_stream
            check(lib().tc_ctx_create(device, stream, C.byref(h)), None, "tc_ctx_create")
        self.handle = h

    _pipeline: dict = {}

    @classmethod
    def pipeline(cls, device: int, k: int) -> "Context":
        """Context k (0, 1, ...) of the forward pipeline on `device` for the calling thread:
        its own CUDA stream (kept bound), its own scratch, the device's SRSs shared."""
        import torch

        key = (device, k, threading.get_ident())
        with cls._guard:
            ctx = cls._pipeline.get(key)
            if ctx is None:
                ctx = cls(device)
                # high priority: this context's count / scatter / accumulation; each forward's
                # latency-bound tail goes to a low-priority stream (tc_ctx_set_pipelined)
                ctx.fixed_stream = torch.cuda.Stream(device, priority=-1)
                lib().tc_ctx_set_stream(ctx.handle, ctx.fixed_stream.cuda_stream)
                lib().tc_ctx_set_pipelined(ctx.handle, 1)
                cls._pipeline[key] = ctx
        return ctx

    @classmethod
    def get(cls, device=None) -> "Context":
        import torch

        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        with cls._guard:
            ctx = cls._by_device.get(device)
            if ctx is None:
                ctx = cls(device)
                cls._by_device[device] = ctx
        return ctx

    fixed_stream = None

    def bind_stream(self):
        import torch

        if self.fixed_stream is not None:
            lib().tc_ctx_set_stream(self.handle, self.fixed_stream.cuda_stream)
            return

        s = torch.cuda.current_stream(self.device).cuda_stream
        lib().tc_ctx_set_stream(self.handle, s)

    def check(self, status, what=""):
        check(status, self.handle, what)

    @property
    def launches(self) -> int:
        return int(lib().tc_ctx_launch_count(self.handle))

    def set_profiling(self, on: bool):
        self.check(lib().tc_ctx_set_profiling(self.handle, 1 if on else 0), "set_profiling")

    def kernel_stats(self, name: str):
        ms, n, units = C.c_double(), C.c_uint64(), C.c_double()
        self.check(lib().tc_ctx_kernel_stats(self.handle, name.encode(), C.byref(ms), C.byref(n), C.byref(units)))
        return {"ms": ms.value, "launches": int(n.value), "units": units.value}
