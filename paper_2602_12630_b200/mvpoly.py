"""Dense multivariate polynomials in lexicographic layout, GPU-backed.

Drop-in for the hot-path subset of tensorcommit.mvpoly:
  check_shape / lex_strides / lex_index  (mvpoly.py:27-59)
  MultiPoly, Grid, default_grid           (mvpoly.py:67-133)
  interpolate_lagrange                    (mvpoly.py:233-247)  -> K2 on the device
  evaluate                                (mvpoly.py:140-161)  -> device Horner
  open_quotients                          (mvpoly.py:521-534)  -> K4 on the device
Only the default grid (nodes 1..d_j) and the production scalar field are supported on the
device — exactly what the prover uses; other domains / grids raise ValueError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _conv, _lib
from .curve import P, encode_scalar

MAX_COEFFS = 1 << 26


def check_shape(shape) -> int:
    if len(shape) == 0:
        raise ValueError("shape needs at least one axis")
    total = 1
    for d in shape:
        if d < 1:
            raise ValueError(f"axis degree bound must be >= 1, got {d}")
        total *= d
    if total > MAX_COEFFS:
        raise ValueError(f"coefficient array of {total} entries exceeds limit")
    return total


def lex_strides(shape):
    st = [1] * len(shape)
    for j in range(len(shape) - 2, -1, -1):
        st[j] = st[j + 1] * shape[j + 1]
    return tuple(st)


def lex_index(idx, shape) -> int:
    if len(idx) != len(shape):
        raise ValueError("index arity does not match shape")
    off = 0
    for i, d in zip(idx, shape):
        if not 0 <= i < d:
            raise IndexError(f"index {idx} out of bounds for shape {shape}")
        off = off * d + i
    return off


@dataclass(frozen=True)
class MultiPoly:
    shape: tuple
    coeffs: tuple

    def __post_init__(self):
        n = check_shape(self.shape)
        if len(self.coeffs) != n:
            raise ValueError(f"expected {n} coefficients for shape {self.shape}, got {len(self.coeffs)}")

    @property
    def arity(self) -> int:
        return len(self.shape)

    def coeff(self, idx):
        return self.coeffs[lex_index(idx, self.shape)]


@dataclass(frozen=True)
class Grid:
    axes: tuple

    def __post_init__(self):
        if len(self.axes) == 0:
            raise ValueError("grid needs at least one axis")
        for nodes in self.axes:
            if len(set(nodes)) != len(nodes):
                raise ValueError("repeated node on a grid axis")

    @property
    def shape(self) -> tuple:
        return tuple(len(a) for a in self.axes)

    def point(self, idx) -> tuple:
        return tuple(self.axes[j][i] for j, i in enumerate(idx))


def default_grid(dom, shape) -> Grid:
    """Axis j uses nodes 1..d_j (mvpoly.py:130-133)."""
    check_shape(shape)
    return Grid(tuple(tuple(range(1, d + 1)) for d in shape))


def _require_device_domain(dom, grid):
    # dom None (the production field) or a prime-field domain of modulus p; anything else
    # (e.g. the reference's FloatDomain, which has no .p) is rejected, never truncated
    if dom is not None and getattr(dom, "p", None) != P:
        raise ValueError("device polynomial engine supports only the production scalar field")
    if grid is not None:
        for d, nodes in zip(grid.shape, grid.axes):
            if tuple(int(z) % P for z in nodes) != tuple(range(1, d + 1)):
                raise ValueError("device polynomial engine supports only the default grid (nodes 1..d)")


def _shape_arr(shape):
    return (C.c_uint32 * len(shape))(*shape)


def interpolate_lagrange(dom, values, grid: Grid) -> MultiPoly:
    """Unique interpolant with per-axis degree < d_j matching `values` on `grid`."""
    _require_device_domain(dom, grid)
    shape = tuple(grid.shape)
    n = check_shape(shape)
    ctx = _lib.Context.get()
    ptr, dt, keep = _conv.device_input(values, n, f"cuda:{ctx.device}")
    if dt != _lib.DTYPE_FP_LIMBS:
        raise ValueError("interpolate_lagrange takes field elements (quantize floats first)")
    limbs = keep.clone()
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_interpolate(ctx.handle, limbs.data_ptr(), _shape_arr(shape), len(shape)),
                  "interpolate_lagrange")
        ctx.check(_lib.lib().tc_ctx_synchronize(ctx.handle))
    return MultiPoly(shape, tuple(_conv.limbs_to_ints(limbs)))


def evaluate(dom, f: MultiPoly, point) -> int:
    _require_device_domain(dom, None)
    if len(point) != len(f.shape):
        raise ValueError("evaluation point arity does not match polynomial")
    ctx = _lib.Context.get()
    ptr, dt, keep = _conv.device_input(f.coeffs, len(f.coeffs), f"cuda:{ctx.device}")
    y = C.create_string_buffer(21)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_evaluate(ctx.handle, ptr, _shape_arr(f.shape), len(f.shape),
                                         b"".join(encode_scalar(int(w)) for w in point), y), "evaluate")
    return int.from_bytes(y.raw, "little")


def open_quotients(dom, f: MultiPoly, point):
    """f - f(w) = sum_i q_i (X_i - w_i): returns ([q_1..q_m], y), each q_i in f's shape."""
    _require_device_domain(dom, None)
    if len(point) != len(f.shape):
        raise ValueError("point arity does not match polynomial")
    m = len(f.shape)
    n = len(f.coeffs)
    ctx = _lib.Context.get()
    ptr, dt, keep = _conv.device_input(f.coeffs, n, f"cuda:{ctx.device}")
    q = _conv.empty_limbs(m * n, f"cuda:{ctx.device}")
    y = C.create_string_buffer(21)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_open_quotients(ctx.handle, ptr, _shape_arr(f.shape), m,
                                               b"".join(encode_scalar(int(w)) for w in point), q.data_ptr(), y),
                  "open_quotients")
    flat = _conv.limbs_to_ints(q)
    qs = [MultiPoly(tuple(f.shape), tuple(flat[a * n:(a + 1) * n])) for a in range(m)]
    return qs, int.from_bytes(y.raw, "little")


# ---------------------------------------------------------------- wire format (mvpoly.py:567-631)
WIRE_VERSION = 1


def _header(magic: bytes, shape) -> bytes:
    import struct
    return magic + struct.pack("<HH", WIRE_VERSION, len(shape)) + b"".join(struct.pack("<I", d) for d in shape)


def _read_header(raw: bytes, magic: bytes):
    import struct
    if raw[:4] != magic:
        raise ValueError(f"bad magic, expected {magic!r}")
    version, m = struct.unpack_from("<HH", raw, 4)
    if version != WIRE_VERSION:
        raise ValueError(f"unsupported version {version}")
    shape = struct.unpack_from("<" + "I" * m, raw, 8)
    return tuple(shape), 8 + 4 * m


def poly_to_bytes(backend, f: MultiPoly) -> bytes:
    """TCPL: header then 21-byte canonical coefficients (backend accepted for drop-in use)."""
    return _header(b"TCPL", f.shape) + b"".join(encode_scalar(int(c)) for c in f.coeffs)


def poly_from_bytes(backend, raw: bytes) -> MultiPoly:
    from .curve import decode_scalar
    raw = bytes(raw)
    shape, off = _read_header(raw, b"TCPL")
    n = check_shape(shape)
    if len(raw) != off + 21 * n:
        raise ValueError("polynomial payload length mismatch")
    return MultiPoly(shape, tuple(decode_scalar(raw[off + 21 * k: off + 21 * (k + 1)]) for k in range(n)))


def tensor_to_bytes(backend, shape, values) -> bytes:
    """TCTN: header then 21-byte canonical field elements."""
    n = check_shape(shape)
    values = list(values)
    if len(values) != n:
        raise ValueError("tensor size does not match shape")
    return _header(b"TCTN", shape) + b"".join(encode_scalar(int(v)) for v in values)


def tensor_from_bytes(backend, raw: bytes):
    from .curve import decode_scalar
    raw = bytes(raw)
    shape, off = _read_header(raw, b"TCTN")
    n = check_shape(shape)
    if len(raw) != off + 21 * n:
        raise ValueError("tensor payload length mismatch")
    return shape, [decode_scalar(raw[off + 21 * k: off + 21 * (k + 1)]) for k in range(n)]
