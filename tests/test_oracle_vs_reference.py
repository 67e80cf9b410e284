"""Property tests: the oracle restatement equals the reference imported live from
/root/reference (build container only; skipped on the GPU box)."""
import random

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import tc_oracle as O

shapes = st.lists(st.integers(1, 5), min_size=1, max_size=3).filter(lambda s: 1 <= __import__("math").prod(s) <= 125)


@settings(max_examples=60, deadline=None)
@given(shape=shapes, seed=st.integers(0, 2 ** 32))
def test_interpolation_division_match_reference(reference, shape, seed):
    backend, field, mvpoly = reference
    dom = field.PrimeField(O.P)
    rng = random.Random(seed)
    n = 1
    for d in shape:
        n *= d
    vals = [dom.rand(rng) if rng.random() < 0.7 else rng.randrange(-3, 4) % O.P for _ in range(n)]
    grid = mvpoly.default_grid(dom, tuple(shape))
    f = mvpoly.interpolate_lagrange(dom, vals, grid)
    mine = O.interpolate_lagrange(vals, tuple(shape))
    assert mine == list(f.coeffs)
    pt = [dom.rand(rng) if rng.random() < 0.7 else rng.randrange(1, 6) for _ in shape]
    qs, y = mvpoly.open_quotients(dom, f, pt)
    mqs, my = O.open_quotients(mine, tuple(shape), pt)
    assert my == y and mqs == [list(q.coeffs) for q in qs]
    assert O.evaluate(mine, tuple(shape), pt) == mvpoly.evaluate(dom, f, pt)
    assert O.barycentric_eval(vals, tuple(shape), pt) == mvpoly.barycentric_eval(dom, vals, grid, pt)
    # SPEC.md:689 opening identity, coefficient-exact
    acc = [0] * n
    for i, q in enumerate(mqs):
        prod = O.multiply_by_linear(q, tuple(shape), i, pt[i] % O.P)
        acc = [(a + b) % O.P for a, b in zip(acc, prod)]
    acc[0] = (acc[0] + my) % O.P
    assert acc == mine


@settings(max_examples=40, deadline=None)
@given(a=st.integers(0, 2 ** 170), b=st.integers(0, 2 ** 170))
def test_group_ops_match_reference(reference, a, b):
    backend, _, _ = reference
    be = backend.make_backend("production")
    pa, pb = be.exp(be.g, a), be.exp(be.g, b)
    assert O.ec_mul(O.G, a) == pa
    assert O.ec_add(pa, pb) == be.mul(pa, pb)
    assert O.ec_add(pa, O.ec_neg(pa)) is None
    assert O.encode_elem(pa) == be.encode_elem(pa)
    assert O.decode_elem(be.encode_elem(pb)) == be.decode_elem(be.encode_elem(pb))


def test_pairing_matches_reference(reference):
    backend, _, _ = reference
    be = backend.make_backend("production")
    rng = random.Random(2)
    for _ in range(3):
        a, b = rng.randrange(O.P), rng.randrange(O.P)
        P1, P2 = be.exp(be.g, a), be.exp(be.g, b)
        assert O.pairing(P1, P2) == be.pair(P1, P2)


@settings(max_examples=200, deadline=None)
@given(data=st.binary(max_size=80), tag=st.binary(max_size=16))
def test_hash_to_scalar_matches_reference(reference, data, tag):
    backend, _, _ = reference
    be = backend.make_backend("production")
    assert O.hash_to_scalar(data, tag) == be.hash_to_scalar(data, tag)
