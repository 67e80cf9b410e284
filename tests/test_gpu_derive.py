"""Trapdoor-free Lagrange SRS.

A published SRS carries only monomial elements (TCSR).  tc_srs_derive_lagrange (run by
tc_srs_load) derives the grid-Lagrange elements and the sub-grid sets from them on the
device; they must equal, byte for byte, the elements the trusted setup computes from the
trapdoors, and commits / openings on a loaded SRS must take the Lagrange route with the
same bytes."""
import ctypes as C
import random
import time

import numpy as np
import pytest

from oracle import tc_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _raw_generate(shape, taus, flags):
    from paper_2602_12630_b200 import _lib
    ctx = _lib.Context.get(0)
    h = C.c_void_p()
    tb = b"".join(int(t).to_bytes(21, "little") for t in taus)
    arr = (C.c_uint32 * len(shape))(*shape)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_srs_generate(ctx.handle, arr, len(shape), tb, flags, C.byref(h)), "generate")
    return ctx, h


def _raw_export(ctx, h, which, count):
    from paper_2602_12630_b200 import _lib
    buf = C.create_string_buffer(max(1, count) * 43)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_srs_export(ctx.handle, h, which, 0, count, buf), "export")
    return buf.raw[:count * 43]


def _sub_total(shape):
    return sum(int(np.prod(shape[i:])) for i in range(1, len(shape)))


@pytest.mark.parametrize("shape,taus", [
    ((5,), None),
    ((3, 4, 5), None),
    ((2, 2, 2), None),
    ((4, 8, 16), None),
    ((1, 7, 1, 3), None),
    ((4, 8), (2, 5)),            # trapdoors ON grid nodes: Lagrange elements hit the identity
    ((6, 3), (7, 3)),            # one axis on a node, one beside it
])
def test_derived_lagrange_equals_trapdoor_setup(shape, taus):
    from paper_2602_12630_b200 import _lib
    rng = random.Random(hash(shape) & 0xffff)
    taus = taus or [rng.randrange(1, O.P) for _ in shape]
    n = int(np.prod(shape))
    ctx, h_full = _raw_generate(shape, taus, _lib.SRS_MONOMIAL | _lib.SRS_LAGRANGE)
    _, h_mono = _raw_generate(shape, taus, _lib.SRS_MONOMIAL)
    try:
        assert not _lib.lib().tc_srs_has(h_mono, _lib.SRS_LAGRANGE)
        ctx.check(_lib.lib().tc_srs_derive_lagrange(ctx.handle, h_mono), "derive")
        assert _raw_export(ctx, h_mono, _lib.SRS_LAGRANGE, n) == _raw_export(ctx, h_full, _lib.SRS_LAGRANGE, n)
        if len(shape) > 1:
            tot = _sub_total(shape)
            assert _raw_export(ctx, h_mono, _lib.SRS_SUBGRID, tot) == _raw_export(ctx, h_full, _lib.SRS_SUBGRID, tot)
        # spot-check against the oracle's exponents (backend.py exp of g)
        exps = O.lagrange_exponents(shape, list(taus))
        got = _raw_export(ctx, h_mono, _lib.SRS_LAGRANGE, n)
        for i in sorted({0, n // 2, n - 1}):
            assert got[43 * i:43 * (i + 1)] == O.encode_elem(O.ec_mul(O.G, exps[i]))
    finally:
        _lib.lib().tc_srs_destroy(h_full)
        _lib.lib().tc_srs_destroy(h_mono)


def test_tcsr_round_trip_takes_lagrange_route():
    """setup_srs -> Srs.to_bytes (TCSR) -> Srs.from_bytes: the bytes round-trip,
    the loaded SRS has the trapdoor-identical Lagrange elements, and commits / openings on it
    (Lagrange route) equal those on the generated SRS."""
    import paper_2602_12630_b200 as tcb
    shape = (4, 8, 16)
    srs, td = tcb.setup_srs(shape, b"tcsr-round-trip")
    raw = srs.to_bytes()
    loaded = tcb.Srs.from_bytes(raw)
    assert loaded.to_bytes() == raw
    assert loaded.has(4) and loaded.lagrange_elems == srs.lagrange_elems
    x = torch.from_numpy((np.random.default_rng(3).standard_t(3, 512) * 2).astype(np.float16)).cuda()
    want = O.commit_trapdoor(O.quantize(x.cpu().numpy().astype(np.float64), 16), shape, list(td.taus))
    for route in ("lagrange", "monomial", "auto"):
        assert tcb.tc_commit(loaded, x, route=route).elem == want
    pt = [random.Random(9).randrange(O.P) for _ in shape]
    op_l, op_g = tcb.tc_open(loaded, x, pt, route="lagrange"), tcb.tc_open(srs, x, pt)
    assert op_l == op_g
    assert tcb.tc_verify(loaded, tcb.Commitment(want), pt, op_l)
    grid_pt = [2, 5, 16]
    assert tcb.tc_open(loaded, x, grid_pt, route="lagrange") == tcb.tc_open(srs, x, grid_pt, route="monomial")


def test_tcsr_malformed_rejected():
    import paper_2602_12630_b200 as tcb
    srs, _ = tcb.setup_srs((2, 3), b"bad")
    raw = srs.to_bytes()
    with pytest.raises(ValueError):
        tcb.Srs.from_bytes(b"TCSX" + raw[4:])
    with pytest.raises(ValueError):
        tcb.Srs.from_bytes(raw[:40])
    bad = bytearray(raw)
    bad[8 + 4 * 2 + 5] ^= 1      # corrupt the first point's x: no longer on the curve
    with pytest.raises(ValueError):
        tcb.Srs.from_bytes(bytes(bad))


@pytest.mark.parametrize("shape", [(32, 32, 32, 64)])
def test_derived_lagrange_full_size(shape):
    """Config-3 SRS (2^21 points): the monomial elements exported and re-loaded through
    tc_srs_load (which derives the Lagrange set) give the trapdoor setup's Lagrange and
    sub-grid elements byte for byte; the derivation time is printed."""
    from paper_2602_12630_b200 import _lib
    taus = [int(t) for t in __import__("paper_2602_12630_b200").derive_taus(shape, b"tc-b200/config3")]
    n = int(np.prod(shape))
    ctx, h_full = _raw_generate(shape, taus, _lib.SRS_MONOMIAL | _lib.SRS_LAGRANGE)
    mono = _raw_export(ctx, h_full, _lib.SRS_MONOMIAL, n)
    axis = C.create_string_buffer(43 * len(shape))
    _lib.lib().tc_srs_export_axis(h_full, axis)
    h = C.c_void_p()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_srs_load(ctx.handle, (C.c_uint32 * 4)(*shape), 4, mono, axis.raw, C.byref(h)), "load")
    torch.cuda.synchronize()
    print(f"tc_srs_load incl. Lagrange derivation of {shape}: {time.perf_counter() - t0:.3f} s")
    try:
        assert _raw_export(ctx, h, _lib.SRS_LAGRANGE, n) == _raw_export(ctx, h_full, _lib.SRS_LAGRANGE, n)
        tot = _sub_total(shape)
        assert _raw_export(ctx, h, _lib.SRS_SUBGRID, tot) == _raw_export(ctx, h_full, _lib.SRS_SUBGRID, tot)
    finally:
        _lib.lib().tc_srs_destroy(h_full)
        _lib.lib().tc_srs_destroy(h)
