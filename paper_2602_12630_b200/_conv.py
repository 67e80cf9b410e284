"""Moving field tensors between Python ints / numpy / torch and the device limb layout
(canonical little-endian 6 x u32 per element, include/tc_b200.h)."""
from __future__ import annotations

import numpy as np

from . import _lib
from .curve import P

LIMBS = 6

_FLOAT_DTYPES = None


_DEVICES = {}   # device argument -> torch.device (parsing a device string per call is not free)


def _float_codes():
    global _FLOAT_DTYPES
    if _FLOAT_DTYPES is None:
        import torch

        _FLOAT_DTYPES = {
            torch.float16: _lib.DTYPE_F16,
            torch.bfloat16: _lib.DTYPE_BF16,
            torch.float32: _lib.DTYPE_F32,
            torch.float64: _lib.DTYPE_F64,
        }
    return _FLOAT_DTYPES


def ints_to_limbs_np(values) -> np.ndarray:
    """Python ints (any sign) -> (n, 6) uint32 canonical residues mod p."""
    vals = [int(v) % P for v in values]
    buf = b"".join(v.to_bytes(4 * LIMBS, "little") for v in vals)
    return np.frombuffer(buf, dtype=np.uint32).reshape(len(vals), LIMBS)


def limbs_to_ints(arr) -> list:
    """(n, 6) limb array (numpy or torch, any device) -> list of Python ints."""
    try:
        import torch

        if isinstance(arr, torch.Tensor):
            arr = arr.detach().to("cpu").contiguous().numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(arr).view(np.uint32).reshape(-1, LIMBS)
    raw = a.tobytes()
    w = 4 * LIMBS
    return [int.from_bytes(raw[i * w:(i + 1) * w], "little") for i in range(a.shape[0])]


def empty_limbs(n: int, device):
    import torch

    return torch.empty((n, LIMBS), dtype=torch.int32, device=device)


def limbs_to_device(arr_np: np.ndarray, device):
    import torch

    return torch.from_numpy(np.array(arr_np, copy=True).view(np.int32)).to(device)


def device_input(T, n: int, device):
    """Resolve a tensor argument into (device pointer, dtype code, keep-alive object).

    Accepted: torch tensors (floating -> quantised on the device; integer -> residues
    mod p), numpy arrays, or any sequence of Python ints (the reference's field tensors).
    Objects exposing ``.limbs`` (FieldTensor) pass their device limbs through.
    """
    import torch

    if isinstance(T, torch.Tensor):
        codes = _float_codes()
        if T.dtype in codes and T.numel() == n and T.is_contiguous():
            dev = _DEVICES.get(device)
            if dev is None:
                dev = _DEVICES[device] = torch.device(device) if isinstance(device, str) else device
            if T.device == dev:
                # already resident and dense (the per-forward hot path): no .to() dispatch
                return T.data_ptr(), codes[T.dtype], T
    if hasattr(T, "limbs") and isinstance(getattr(T, "limbs"), torch.Tensor):
        lt = T.limbs
        if lt.shape[0] != n:
            raise ValueError("tensor size does not match grid shape")
        lt = lt.to(device).contiguous()
        return lt.data_ptr(), _lib.DTYPE_FP_LIMBS, lt
    if isinstance(T, np.ndarray):
        if T.dtype.kind == "f":
            T = torch.from_numpy(np.ascontiguousarray(T))
        else:
            T = [int(v) for v in T.reshape(-1).tolist()]
    if isinstance(T, torch.Tensor):
        if T.numel() != n:
            raise ValueError("tensor size does not match grid shape")
        codes = _float_codes()
        if T.dtype in codes:
            t = T.detach().to(device).contiguous()
            return t.data_ptr(), codes[T.dtype], t
        T = [int(v) for v in T.detach().reshape(-1).cpu().tolist()]
    vals = list(T)
    if len(vals) != n:
        raise ValueError("tensor size does not match grid shape")
    lt = limbs_to_device(ints_to_limbs_np(vals), device)
    return lt.data_ptr(), _lib.DTYPE_FP_LIMBS, lt
