"""TensorCommitments: setup / commit / open / verify on the B200.

Drop-in for the spec-only `commit` module of the reference and
`setup_srs` of `algebra`, with the reference's types: points are affine
(x, y) int tuples or None (backend.py:15-17), scalars are ints in [0, p).

Every compute step (SRS generation, quantisation, interpolation, MSM, quotients) runs in
libtcb200.so on the GPU; `tc_verify` is the CPU verifier (product of
pairings SPEC.md:313) implemented natively in the same library.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

from . import _conv, _lib
from .curve import (ELEM_BYTES, P, decode_elem, decode_elems, decode_scalar, encode_elem, encode_scalar,
                    hash_to_scalar)
from .mvpoly import Grid, check_shape, default_grid

SCALE_BITS = 16   # protocol.quantize fixed-point scale

_ROUTES = {"auto": _lib.ROUTE_AUTO, "monomial": _lib.ROUTE_MONOMIAL, "lagrange": _lib.ROUTE_LAGRANGE}


def shape_header(magic: bytes, shape) -> bytes:
    """magic ‖ <HH version=1, m> ‖ <I d_j>×m — the wire header of mvpoly.py:567-572."""
    return magic + struct.pack("<HH", 1, len(shape)) + b"".join(struct.pack("<I", d) for d in shape)


def derive_taus(shape, entropy: bytes):
    """Frozen trapdoor PRF (SPEC.md:81 leaves it open):
    tau_j = hash_to_scalar(entropy ‖ u32le(j) ‖ TCSR header(shape), tag=b"srs/tau")."""
    hdr = shape_header(b"TCSR", shape)
    return tuple(hash_to_scalar(bytes(entropy) + struct.pack("<I", j) + hdr, b"srs/tau") for j in range(len(shape)))


@dataclass(frozen=True)
class Trapdoors:
    """only the trusted setup and tests may hold these."""
    taus: tuple


@dataclass(frozen=True)
class Commitment:
    """a single group element."""
    elem: object

    def to_bytes(self) -> bytes:
        return encode_elem(self.elem)


@dataclass(frozen=True)
class TensorOpening:
    """claimed value y and m quotient commitments."""
    y: int
    proofs: tuple

    def to_bytes(self, point) -> bytes:
        """TCOP wire format: magic, m (u16), omega, y, m proof elements."""
        out = [b"TCOP", struct.pack("<H", len(self.proofs))]
        out += [encode_scalar(w) for w in point]
        out.append(encode_scalar(self.y))
        out += [encode_elem(e) for e in self.proofs]
        return b"".join(out)

    @staticmethod
    def from_bytes(raw: bytes):
        """Inverse of to_bytes: returns (point, TensorOpening); ValueError on malformed input."""
        raw = bytes(raw)
        if raw[:4] != b"TCOP":
            raise ValueError("bad magic, expected b'TCOP'")
        (m,) = struct.unpack_from("<H", raw, 4)
        need = 6 + 21 * (m + 1) + ELEM_BYTES * m
        if len(raw) != need:
            raise ValueError("opening payload length mismatch")
        off = 6
        point = tuple(decode_scalar(raw[off + 21 * i: off + 21 * (i + 1)]) for i in range(m))
        off += 21 * m
        y = decode_scalar(raw[off: off + 21])
        off += 21
        proofs = tuple(decode_elem(raw[off + ELEM_BYTES * i: off + ELEM_BYTES * (i + 1)]) for i in range(m))
        return point, TensorOpening(y, proofs)


class Srs:
    """Structured reference string resident in device memory.

    monomial_elems / lagrange_elems are materialised on the host lazily (they are
    large); the kernels use the device copy directly.
    """

    def __init__(self, shape, handle, device, axis_elems, grid=None):
        self.shape = tuple(int(d) for d in shape)
        self._h = handle
        self.device = device
        self.axis_elems = tuple(axis_elems)
        self.grid = grid if grid is not None else default_grid(None, self.shape)
        self._cache = {}

    @property
    def size(self) -> int:
        return int(_lib.lib().tc_srs_size(self._h))

    @property
    def handle(self):
        return self._h

    def has(self, which: int) -> bool:
        return bool(_lib.lib().tc_srs_has(self._h, which))

    def export_range(self, which: int, start: int, count: int):
        """Elements [start, start+count) of the monomial / Lagrange SRS as points."""
        ctx = _lib.Context.get(self.device)
        buf = C.create_string_buffer(max(1, count) * ELEM_BYTES)
        with ctx.lock:
            ctx.bind_stream()
            ctx.check(_lib.lib().tc_srs_export(ctx.handle, self._h, which, start, count, buf), "tc_srs_export")
        return decode_elems(buf.raw, count)

    def _export(self, which):
        if which not in self._cache:
            self._cache[which] = self.export_range(which, 0, self.size)
        return self._cache[which]

    @property
    def monomial_elems(self):
        return self._export(_lib.SRS_MONOMIAL)

    @property
    def lagrange_elems(self):
        return self._export(_lib.SRS_LAGRANGE)

    def prepare(self, dtype="float16", scale_bits: int = SCALE_BITS) -> "Srs":
        """Build the tables commits of `dtype` inputs read (fp16: the exponent table of the
        Lagrange basis) now instead of on the first commit.  Returns self."""
        code = {"float16": _lib.DTYPE_F16, "bfloat16": _lib.DTYPE_BF16, "float32": _lib.DTYPE_F32}.get(str(dtype).replace("torch.", ""), 0)
        ctx = _lib.Context.get(self.device)
        with ctx.lock:
            ctx.bind_stream()
            ctx.check(_lib.lib().tc_srs_prepare(ctx.handle, self._h, code, scale_bits), "prepare")
        return self

    def table_bytes(self) -> dict:
        """Device bytes held by this SRS: exponent table, window tables, bases."""
        e, w, b = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _lib.check(_lib.lib().tc_srs_table_bytes(self._h, C.byref(e), C.byref(w), C.byref(b)), None, "table_bytes")
        return {"exptab_bytes": e.value, "window_table_bytes": w.value, "basis_bytes": b.value}

    def derive_lagrange(self) -> "Srs":
        """Derive the Lagrange elements (and sub-grid sets) from the monomial elements on the
        device, without the trapdoors (a no-op when present).  Returns self."""
        ctx = _lib.Context.get(self.device)
        with ctx.lock:
            ctx.bind_stream()
            ctx.check(_lib.lib().tc_srs_derive_lagrange(ctx.handle, self._h), "derive_lagrange")
        self._cache.pop(_lib.SRS_LAGRANGE, None)
        return self

    def to_bytes(self) -> bytes:
        """TCSR file: header, monomial elements, axis elements, grid."""
        out = [shape_header(b"TCSR", self.shape)]
        out += [encode_elem(e) for e in self.monomial_elems]
        out += [encode_elem(e) for e in self.axis_elems]
        for nodes in self.grid.axes:
            out += [encode_scalar(z) for z in nodes]
        return b"".join(out)

    @classmethod
    def from_bytes(cls, raw: bytes, device=None) -> "Srs":
        if raw[:4] != b"TCSR":
            raise ValueError("bad magic, expected b'TCSR'")
        version, m = struct.unpack_from("<HH", raw, 4)
        if version != 1:
            raise ValueError(f"unsupported version {version}")
        shape = struct.unpack_from("<" + "I" * m, raw, 8)
        n = check_shape(shape)
        off = 8 + 4 * m
        mono = raw[off:off + n * ELEM_BYTES]
        off += n * ELEM_BYTES
        axis = raw[off:off + m * ELEM_BYTES]
        if len(mono) != n * ELEM_BYTES or len(axis) != m * ELEM_BYTES:
            raise ValueError("srs payload length mismatch")
        return load_srs(shape, mono, axis, device=device)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None and _lib._lib is not None:
            try:
                _lib.lib().tc_srs_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass

    def __repr__(self):
        return f"Srs(shape={self.shape})"


def _shape_arr(shape):
    return (C.c_uint32 * len(shape))(*shape)


def setup_srs(shape, entropy: bytes, *, lagrange: bool = True, monomial: bool = True, device=None):
    """setup_srs(shape, entropy) -> (Srs, Trapdoors).

    Monomial elements g^{prod tau_j^{i_j}} (lex order) and — used by the fast commit
    route — the grid-Lagrange elements g^{prod L_{j,i_j}(tau_j)}, both generated on the
    GPU by fixed-base scalar multiplication."""
    shape = tuple(int(d) for d in shape)
    check_shape(shape)
    taus = derive_taus(shape, entropy)
    ctx = _lib.Context.get(device)
    flags = (_lib.SRS_MONOMIAL if monomial else 0) | (_lib.SRS_LAGRANGE if lagrange else 0)
    h = C.c_void_p()
    taus_b = b"".join(encode_scalar(t) for t in taus)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_srs_generate(ctx.handle, _shape_arr(shape), len(shape), taus_b, flags, C.byref(h)),
                  "setup_srs")
    axis_buf = C.create_string_buffer(len(shape) * ELEM_BYTES)
    _lib.lib().tc_srs_export_axis(h, axis_buf)
    srs = Srs(shape, h, ctx.device, decode_elems(axis_buf.raw, len(shape)))
    return srs, Trapdoors(taus)


def load_srs(shape, monomial43: bytes, axis43: bytes, device=None) -> Srs:
    """Srs from public points only (e.g. a TCSR file).  The Lagrange elements
    and sub-grid sets the fast commit / open routes use are derived on the device from the
    monomial elements alone (tc_srs_derive_lagrange): no trapdoor is needed."""
    shape = tuple(int(d) for d in shape)
    check_shape(shape)
    ctx = _lib.Context.get(device)
    h = C.c_void_p()
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_srs_load(ctx.handle, _shape_arr(shape), len(shape), bytes(monomial43), bytes(axis43),
                                         C.byref(h)), "load_srs")
    return Srs(shape, h, ctx.device, decode_elems(axis43, len(shape), validate=True))


def _route(route) -> int:
    try:
        return _ROUTES[route]
    except KeyError:
        raise ValueError(f"unknown route {route!r}") from None


def tc_commit(srs: Srs, T, *, scale_bits: int = SCALE_BITS, route: str = "auto") -> Commitment:
    """C_T = g^{f_T(tau)}.

    T: field tensor (sequence of ints / integer array) or a float tensor (torch / numpy),
    which is quantised on the device at 2^scale_bits first."""
    ctx = _lib.Context.get(srs.device)
    ptr, dt, keep = _conv.device_input(T, srs.size, f"cuda:{ctx.device}")
    out = C.create_string_buffer(ELEM_BYTES)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_commit(ctx.handle, srs.handle, ptr, dt, scale_bits, _route(route), out), "tc_commit")
    del keep
    return Commitment(decode_elem(out.raw, validate=False))


def _host_floats(tensors):
    """CPU float tensors / arrays of one dtype -> (contiguous torch tensors, dtype code), else None."""
    import numpy as np
    import torch

    out = []
    for T in tensors:
        if isinstance(T, np.ndarray) and T.dtype.kind == "f":
            T = torch.from_numpy(np.ascontiguousarray(T))
        if not (isinstance(T, torch.Tensor) and T.device.type == "cpu" and T.dtype in _conv._float_codes()):
            return None
        out.append(T.detach().contiguous())
    if not out or len({t.dtype for t in out}) != 1:
        return None
    return out, _conv._float_codes()[out[0].dtype]


def tc_commit_many(srs: Srs, tensors, *, scale_bits: int = SCALE_BITS, route: str = "auto", group: int = 0):
    """Commit several tensors of the SRS's shape (one C call).  Host (CPU) float tensors go
    through tc_commit_batch_host: uploaded in groups on a copy stream, overlapped with the
    commitments of the groups already on the device (pin them for full overlap)."""
    ctx = _lib.Context.get(srs.device)
    tensors = list(tensors)
    host = _host_floats(tensors)
    if host is not None:
        ts, code = host
        for t in ts:
            if t.numel() != srs.size:
                raise ValueError("tensor size does not match grid shape")
        arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
        out = C.create_string_buffer(ELEM_BYTES * len(ts))
        with ctx.lock:
            ctx.bind_stream()
            ctx.check(_lib.lib().tc_commit_batch_host(ctx.handle, srs.handle, arr, len(ts), code, scale_bits,
                                                      _route(route), int(group), out), "tc_commit_many")
        return [Commitment(decode_elem(out.raw[i * ELEM_BYTES:(i + 1) * ELEM_BYTES], validate=False))
                for i in range(len(ts))]
    keeps, ptrs, dts = [], [], set()
    for T in tensors:
        ptr, dt, keep = _conv.device_input(T, srs.size, f"cuda:{ctx.device}")
        ptrs.append(ptr)
        dts.add(dt)
        keeps.append(keep)
    if len(dts) > 1:
        raise ValueError("tc_commit_many: all tensors must share one dtype")
    if not ptrs:
        return []
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    out = C.create_string_buffer(ELEM_BYTES * len(ptrs))
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_commit_batch(ctx.handle, srs.handle, arr, len(ptrs), dts.pop(), scale_bits,
                                             _route(route), out), "tc_commit_many")
    del keeps
    return [Commitment(decode_elem(out.raw[i * ELEM_BYTES:(i + 1) * ELEM_BYTES], validate=False))
            for i in range(len(ptrs))]


def _tree_buffers(count: int, B: int):
    """Output buffers of the device tree calls for `count` leaves over arity B."""
    L, cap = 1, B
    while cap < count:
        cap *= B
        L += 1
    n_nodes = sum(B ** (L - 1 - l) for l in range(L))
    n_vals = sum(B ** (L - l) for l in range(L))
    return (L, C.create_string_buffer(ELEM_BYTES * count), C.create_string_buffer(ELEM_BYTES * n_nodes),
            C.create_string_buffer(24 * n_vals), C.c_uint64(n_nodes), C.c_uint64(n_vals))


def _tree_result(count, L, comms, nodes, vals):
    raw = comms.raw
    commitments = [Commitment(decode_elem(raw[i * ELEM_BYTES:(i + 1) * ELEM_BYTES], validate=False))
                   for i in range(count)]
    return commitments, nodes.raw, vals.raw, L


def tc_commit_tree(srs: Srs, tensors, node_srs: Srs, *, scale_bits: int = SCALE_BITS, route: str = "auto"):
    """Commit device tensors of the SRS's shape AND build their Terkle tree over `node_srs`
    in one C call (tc_commit_tree: leaf hashing and every tree level on the device, one
    readback).  Returns (commitments, node encodings, level values, depth): node encodings
    are 43-byte commitments level by level (bottom first), level values the canonical
    24-byte child values of every level (leaves zero-padded to B^L first)."""
    ctx = _lib.Context.get(srs.device)
    keeps, ptrs, dts = [], [], set()
    for T in tensors:
        ptr, dt, keep = _conv.device_input(T, srs.size, f"cuda:{ctx.device}")
        ptrs.append(ptr)
        dts.add(dt)
        keeps.append(keep)
    if len(dts) != 1:
        raise ValueError("tc_commit_tree: all tensors must share one dtype")
    L, comms, nodes, vals, cn, cv = _tree_buffers(len(ptrs), node_srs.size)
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_commit_tree(ctx.handle, srs.handle, arr, len(ptrs), dts.pop(), scale_bits,
                                            _route(route), node_srs.handle, comms, nodes, C.byref(cn), vals,
                                            C.byref(cv)), "tc_commit_tree")
    del keeps
    return _tree_result(len(ptrs), L, comms, nodes, vals)


def tc_commit_tree_launch(ctx, srs: Srs, tensors, node_srs: Srs, *, scale_bits: int = SCALE_BITS,
                          route: str = "auto"):
    """First half of tc_commit_tree on pipeline context `ctx` (_lib.Context.pipeline): enqueue
    the commitments, leaf hashing, tree and readback, return without waiting for them.  CUDA
    tensors are ordered after torch's current stream; CPU float tensors are uploaded on the
    context's copy stream.  Returns the state tc_commit_tree_finish takes (it keeps the
    inputs alive until then)."""
    import torch

    tensors = list(tensors)
    host = _host_floats(tensors)
    conv = None
    if host is None:
        # conversions (contiguous copies, H2D limbs, cross-device moves) are enqueued on
        # torch's current stream: do them BEFORE the pipeline stream is ordered after it
        conv = [_conv.device_input(T, srs.size, f"cuda:{ctx.device}") for T in tensors]
    with ctx.lock:
        # the context's stream runs after everything already queued on torch's stream (the
        # inputs' producers and conversions, SRS setup)
        ctx.fixed_stream.wait_stream(torch.cuda.current_stream(ctx.device))
        if host is not None:
            ts, code = host
            for t in ts:
                if t.numel() != srs.size:
                    raise ValueError("tensor size does not match grid shape")
            arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
            keep = ts
            ctx.check(_lib.lib().tc_commit_stream_tree_launch(ctx.handle, srs.handle, arr, len(ts), code, scale_bits,
                                                              _route(route), node_srs.handle),
                      "tc_commit_tree_launch")
        else:
            ptrs = [c[0] for c in conv]
            dts = {c[1] for c in conv}
            keeps = [c[2] for c in conv]
            if len(dts) != 1:
                raise ValueError("tc_commit_tree: all tensors must share one dtype")
            arr = (C.c_void_p * len(ptrs))(*ptrs)
            keep = keeps
            ctx.check(_lib.lib().tc_commit_tree_launch(ctx.handle, srs.handle, arr, len(ptrs), dts.pop(), scale_bits,
                                                       _route(route), node_srs.handle), "tc_commit_tree_launch")
    return ctx, len(tensors), node_srs.size, keep


def tc_commit_tree_finish(state):
    """Second half: wait for the launched work, return what tc_commit_tree returns."""
    ctx, count, B, _keep = state
    L, comms, nodes, vals, cn, cv = _tree_buffers(count, B)
    with ctx.lock:
        ctx.check(_lib.lib().tc_commit_tree_finish(ctx.handle, comms, nodes, C.byref(cn), vals, C.byref(cv)),
                  "tc_commit_tree_finish")
    return _tree_result(count, L, comms, nodes, vals)


def _stream_args(srs: Srs, cur, nxt):
    hc = _host_floats(list(cur))
    if hc is None:
        raise ValueError("tc_commit_stream: cur must be CPU float tensors of one dtype")
    ts, code = hc
    for t in ts:
        if t.numel() != srs.size:
            raise ValueError("tensor size does not match grid shape")
    arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    narr = None
    if nxt is not None:
        hn = _host_floats(list(nxt))
        if hn is None or hn[1] != code or len(hn[0]) != len(ts):
            raise ValueError("tc_commit_stream: nxt must match cur (count, dtype, CPU)")
        if any(t.numel() != srs.size for t in hn[0]):
            raise ValueError("tensor size does not match grid shape")
        narr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in hn[0]])
    return ts, code, arr, narr


def tc_commit_stream_tree(srs: Srs, cur, nxt, node_srs: Srs, *, scale_bits: int = SCALE_BITS,
                          route: str = "auto"):
    """tc_commit_stream and the Terkle tree of its commitments on the device in one call
    (tc_commit_stream_tree); returns what tc_commit_tree returns."""
    ctx = _lib.Context.get(srs.device)
    ts, code, arr, narr = _stream_args(srs, cur, nxt)
    L, comms, nodes, vals, cn, cv = _tree_buffers(len(ts), node_srs.size)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_commit_stream_tree(ctx.handle, srs.handle, arr, narr, len(ts), code, scale_bits,
                                                   _route(route), node_srs.handle, comms, nodes, C.byref(cn),
                                                   vals, C.byref(cv)), "tc_commit_stream_tree")
    return _tree_result(len(ts), L, comms, nodes, vals)


def tc_commit_stream(srs: Srs, cur, nxt=None, *, scale_bits: int = SCALE_BITS, route: str = "auto"):
    """Streaming commits of host (CPU) float tensors, one call per forward: commits `cur`
    while the upload of `nxt` (the next forward's tensors, or None) runs on the copy stream.
    `cur` is consumed from the prefetched device slot when it is the previous call's `nxt`.
    Tensors passed as `nxt` must not change until the call that commits them returns."""
    ctx = _lib.Context.get(srs.device)
    ts, code, arr, narr = _stream_args(srs, cur, nxt)
    out = C.create_string_buffer(ELEM_BYTES * len(ts))
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_commit_stream(ctx.handle, srs.handle, arr, narr, len(ts), code, scale_bits,
                                              _route(route), out), "tc_commit_stream")
    return [Commitment(decode_elem(out.raw[i * ELEM_BYTES:(i + 1) * ELEM_BYTES], validate=False))
            for i in range(len(ts))]


def tc_open(srs: Srs, T, point, *, scale_bits: int = SCALE_BITS, route: str = "auto") -> TensorOpening:
    """y = f_T(omega), pi_i = g^{q_i(tau)} from open_quotients."""
    if len(point) != len(srs.shape):
        raise ValueError("point arity does not match polynomial")
    ctx = _lib.Context.get(srs.device)
    ptr, dt, keep = _conv.device_input(T, srs.size, f"cuda:{ctx.device}")
    m = len(srs.shape)
    om = b"".join(encode_scalar(int(w)) for w in point)
    y = C.create_string_buffer(21)
    pis = C.create_string_buffer(ELEM_BYTES * m)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_open(ctx.handle, srs.handle, ptr, dt, scale_bits, om, _route(route), y, pis), "tc_open")
    del keep
    return TensorOpening(int.from_bytes(y.raw, "little"), decode_elems(pis.raw, m))


_OPEN_POOL = None


def _open_pool():
    global _OPEN_POOL
    if _OPEN_POOL is None:
        import concurrent.futures as cf

        _OPEN_POOL = cf.ThreadPoolExecutor(max_workers=max(8, _OPEN_PARALLEL), thread_name_prefix="tc-open")
    return _OPEN_POOL


def _open_bins(tensors, nbins: int):
    """Split opening indices into nbins sets, all openings of one tensor in one set (its
    slice commitments are built once), balancing a rough cost: a tensor opened k >= 6 times
    costs its slice commitments plus a little per opening, otherwise k full quotient MSMs."""
    groups = {}
    for i, T in enumerate(tensors):
        groups.setdefault(id(T), []).append(i)
    cost = lambda ids: 3.0 + 0.05 * len(ids) if len(ids) >= 6 else 1.4 * len(ids)
    bins = [[] for _ in range(nbins)]
    load = [0.0] * nbins
    for ids in sorted(groups.values(), key=cost, reverse=True):
        j = min(range(nbins), key=lambda b: load[b])
        bins[j] += ids
        load[j] += cost(ids)
    return [sorted(b) for b in bins if b]


_OPEN_PARALLEL = int(__import__("os").environ.get("TC_OPEN_PARALLEL", "4"))   # contexts (A/B: 1 146 ms, 2 122, 4 111, 6 111, 8 124)


def tc_open_many(srs: Srs, tensors, points, *, scale_bits: int = SCALE_BITS, route: str = "auto",
                 parallel: int = None):
    """tc_open for many (tensor, point) pairs (tc_open_batch): the quotient MSMs of a group
    of openings run as one batched pipeline per axis.  With `parallel` > 1 and enough
    openings, the pairs are split by tensor over that many device contexts driven from
    worker threads, so one set's latency-bound MSM tails overlap the other's compute.  Same
    bytes as calling tc_open on each pair."""
    tensors, points = list(tensors), list(points)
    if parallel is None:
        parallel = _OPEN_PARALLEL
    if len(tensors) != len(points):
        raise ValueError("tensors and points differ in length")
    if not tensors:
        return []
    m = len(srs.shape)
    for pt in points:
        if len(pt) != m:
            raise ValueError("point arity does not match polynomial")
    # device inputs on the calling thread's stream (the same layer opened many times is
    # converted once)
    cache, conv = {}, []
    for T in tensors:
        if id(T) not in cache:
            cache[id(T)] = _conv.device_input(T, srs.size, f"cuda:{srs.device}")
        conv.append(cache[id(T)])
    if len({c[1] for c in conv}) > 1:
        raise ValueError("tc_open_many: all tensors must share one dtype")
    if parallel > 1 and len(tensors) >= 32:
        import torch

        bins = _open_bins(tensors, parallel)
        if len(bins) > 1:
            cur = torch.cuda.current_stream(srs.device)

            def work(ids):
                ctx = _lib.Context.pipeline(srs.device, 0)   # one per worker thread
                ctx.fixed_stream.wait_stream(cur)
                return ids, _open_batch(ctx, srs, [conv[i] for i in ids], [points[i] for i in ids], scale_bits,
                                        route)

            out = [None] * len(tensors)
            for ids, ops in _open_pool().map(work, bins):
                for i, op in zip(ids, ops):
                    out[i] = op
            return out
    return _open_batch(_lib.Context.get(srs.device), srs, conv, points, scale_bits, route, bind=True)


def _open_batch(ctx, srs: Srs, conv, points, scale_bits, route, bind=False):
    """One tc_open_batch call on `ctx` over device inputs (ptr, dtype, keep-alive)."""
    m = len(srs.shape)
    ptrs = [c[0] for c in conv]
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    om = b"".join(encode_scalar(int(w)) for pt in points for w in pt)
    ys = C.create_string_buffer(21 * len(ptrs))
    pis = C.create_string_buffer(ELEM_BYTES * m * len(ptrs))
    with ctx.lock:
        if bind:
            ctx.bind_stream()
        ctx.check(_lib.lib().tc_open_batch(ctx.handle, srs.handle, arr, len(ptrs), conv[0][1], scale_bits, om,
                                           _route(route), ys, pis), "tc_open_many")
    raw_y, raw_p = ys.raw, pis.raw
    return [TensorOpening(int.from_bytes(raw_y[21 * i:21 * (i + 1)], "little"),
                          decode_elems(raw_p[ELEM_BYTES * m * i:ELEM_BYTES * m * (i + 1)], m))
            for i in range(len(ptrs))]


def tc_verify(srs: Srs, C_T, point, opening: TensorOpening) -> bool:
    """e(C g^-y, g) == prod_i e(pi_i, axis_i g^-omega_i). CPU."""
    m = len(srs.shape)
    if len(opening.proofs) != m:
        raise ValueError("proof count does not match tensor order")
    if len(point) != m:
        raise ValueError("point arity does not match polynomial")
    elem = C_T.elem if isinstance(C_T, Commitment) else C_T
    ok = C.c_int(0)
    st = _lib.lib().tc_verify_host(
        m,
        b"".join(encode_elem(a) for a in srs.axis_elems),
        encode_elem(elem),
        b"".join(encode_scalar(int(w)) for w in point),
        encode_scalar(int(opening.y)),
        b"".join(encode_elem(e) for e in opening.proofs),
        C.byref(ok),
    )
    _lib.check(st, None, "tc_verify")
    return bool(ok.value)


def pair(a, b):
    """The reference's modified Tate pairing e(a, b) (backend.py:219-291), on the CPU."""
    out = C.create_string_buffer(42)
    _lib.check(_lib.lib().tc_pairing(encode_elem(a), encode_elem(b), out), None, "pair")
    return (int.from_bytes(out.raw[:21], "little"), int.from_bytes(out.raw[21:], "little"))


def g_mul(k: int):
    """k * g on the host (test helper)."""
    out = C.create_string_buffer(ELEM_BYTES)
    _lib.lib().tc_host_g_mul(encode_scalar(int(k) % P), out)
    return decode_elem(out.raw, validate=False)


__all__ = ["Commitment", "Grid", "Srs", "TensorOpening", "Trapdoors", "derive_taus", "g_mul", "load_srs", "pair",
           "setup_srs", "tc_commit", "tc_commit_many", "tc_open", "tc_verify"]
