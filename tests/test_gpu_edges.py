"""SPEC examples and edge cases through the public API: zero and
constant tensors, degenerate shapes (single element, unit axes), the coefficient-count
limit, arity / size / dtype errors, non-finite and overflowing inputs, empty batches,
completeness over many small random instances and rejection of perturbed openings."""
import random

import numpy as np
import pytest

from oracle import tc_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


SHAPES = [(1,), (7,), (3, 1, 2), (1, 1), (2, 2), (4, 4, 4, 4)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_zero_and_constant_tensors(shape):
    """T all-zeros -> identity; T constant c -> g^c; opening a
    constant tensor at any point gives y = c and identity proofs."""
    import paper_2602_12630_b200 as tcb
    n = int(np.prod(shape))
    srs, _ = tcb.setup_srs(shape, b"edges-%d" % n)
    zero = torch.zeros(n, dtype=torch.float16, device="cuda")
    for route in ("lagrange", "monomial"):
        assert tcb.tc_commit(srs, zero, route=route).elem is None
    c = 12345
    const = [c] * n
    for route in ("lagrange", "monomial"):
        assert tcb.tc_commit(srs, const, route=route).elem == O.ec_mul(O.G, c)
    pt = [random.Random(n).randrange(O.P) for _ in shape]
    op = tcb.tc_open(srs, const, pt)
    assert op.y == c and all(e is None for e in op.proofs)
    assert tcb.tc_verify(srs, tcb.Commitment(O.ec_mul(O.G, c)), pt, op)


def test_errors_match_reference_exception_types():
    import paper_2602_12630_b200 as tcb
    with pytest.raises(ValueError):
        tcb.setup_srs((8192, 8193), b"too-big")            # > 2^26 coefficients (mvpoly.py:24)
    with pytest.raises(ValueError):
        tcb.setup_srs((4, 0), b"zero-axis")
    srs, _ = tcb.setup_srs((4, 8), b"errors")
    with pytest.raises(ValueError):
        tcb.tc_commit(srs, torch.zeros(31, dtype=torch.float16, device="cuda"))   # size mismatch
    with pytest.raises(ValueError):
        tcb.tc_open(srs, [1] * 32, [1, 2, 3])                # point arity
    op = tcb.tc_open(srs, [1] * 32, [5, 6])
    with pytest.raises(ValueError):
        tcb.tc_verify(srs, tcb.Commitment(O.G), [5, 6], tcb.TensorOpening(op.y, op.proofs[:1]))
    with pytest.raises(ValueError):
        tcb.tc_commit(srs, torch.full((32,), float("nan"), device="cuda"))
    with pytest.raises(ValueError):   # |v| 2^scale_bits >= p / 2
        tcb.tc_commit(srs, torch.full((32,), 2.0 ** 30, dtype=torch.float64, device="cuda"), scale_bits=140)
    with pytest.raises(ValueError):
        tcb.prover_commit([], srs)
    assert tcb.tc_open_many(srs, [], []) == []
    assert tcb.tc_commit_many(srs, []) == []
    # the context recovers after every error
    x = torch.from_numpy(np.arange(32, dtype=np.float32) / 7).cuda()
    want = O.commit_trapdoor(O.quantize(x.cpu().numpy().astype(np.float64), 16), (4, 8),
                             list(tcb.derive_taus((4, 8), b"errors")))
    assert tcb.tc_commit(srs, x).elem == want


def test_completeness_and_binding_small_random():
    """honest openings of random small instances (shapes <= 4^4, random
    points, grid points) verify; y + 1, swapped proofs, a proof replaced by g, and a proof
    reused from another instance are rejected."""
    import paper_2602_12630_b200 as tcb
    rng = random.Random(2026)
    shapes = [(2, 2), (4, 4, 4, 4), (3, 4), (4, 1, 3), (2, 2, 2, 2)]
    for si, shape in enumerate(shapes):
        srs, _ = tcb.setup_srs(shape, b"complete-%d" % si)
        n = int(np.prod(shape))
        tensors = [[rng.randrange(O.P) for _ in range(n)] for _ in range(4)]
        pts = [[rng.randrange(O.P) for _ in shape] for _ in range(3)] + [[rng.randrange(1, d + 1) for d in shape]]
        comms = tcb.tc_commit_many(srs, tensors)
        ops = tcb.tc_open_many(srs, tensors, pts, parallel=1)
        for k, (C, pt, op) in enumerate(zip(comms, pts, ops)):
            assert tcb.tc_verify(srs, C, pt, op)
            assert not tcb.tc_verify(srs, C, pt, tcb.TensorOpening((op.y + 1) % O.P, op.proofs))
            if len(shape) > 1 and op.proofs[0] != op.proofs[1]:
                sw = (op.proofs[1], op.proofs[0]) + tuple(op.proofs[2:])
                assert not tcb.tc_verify(srs, C, pt, tcb.TensorOpening(op.y, sw))
            assert not tcb.tc_verify(srs, C, pt, tcb.TensorOpening(op.y, (O.G,) + tuple(op.proofs[1:])))
            other = ops[(k + 1) % len(ops)]
            if other.proofs != op.proofs:
                assert not tcb.tc_verify(srs, C, pt, tcb.TensorOpening(op.y, other.proofs))


def test_split_slice_commitments_open_like_tc_open():
    """The multi-GPU opening route on one GPU: slice commitments computed in three row
    chunks (tc_open_slices, as three ranks would), concatenated, and openings from them
    (tc_open_batch_sliced) equal tc_open byte for byte, grid-node challenges included."""
    import paper_2602_12630_b200 as tcb
    from paper_2602_12630_b200.dist import _open_sliced
    from paper_2602_12630_b200 import _conv, _lib
    shape = (8, 8, 16)
    srs, _ = tcb.setup_srs(shape, b"split-slices")
    x = torch.from_numpy((np.random.default_rng(8).standard_t(3, 1024) * 3).astype(np.float16)).cuda()
    ctx = _lib.Context.get(0)
    chunks = []
    for lo, hi in ((0, 2), (2, 5), (5, 8)):
        buf = torch.zeros(((hi - lo) * 8, 43), dtype=torch.uint8, device="cuda")
        ptr, dt, keep = _conv.device_input(x, srs.size, "cuda:0")
        with ctx.lock:
            ctx.bind_stream()
            ctx.check(_lib.lib().tc_open_slices(ctx.handle, srs.handle, ptr, dt, 16, lo, hi, buf.data_ptr()), "slices")
        chunks.append(buf)
    H = torch.cat(chunks).contiguous()
    rng = random.Random(12)
    pts = [[rng.randrange(O.P) for _ in shape] for _ in range(5)] + [[3, 8, 1], [rng.randrange(O.P), 2, 16]]
    got = _open_sliced(srs, x, H, pts)
    for pt, op in zip(pts, got):
        assert op == tcb.tc_open(srs, x, pt)
