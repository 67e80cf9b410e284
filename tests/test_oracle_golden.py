"""Pin the CPU oracle against golden vectors generated from the reference
(tests/golden/make_golden.py).  Runs everywhere, no GPU, no reference tree."""
import random

import numpy as np
import pytest

from oracle import tc_oracle as O
from tests.golden_io import elem, ints, load


def test_constants():
    assert O.P == 2 ** 161 + 2 ** 24 + 1
    assert O.Q == 120 * O.P - 1
    assert O.on_curve(O.G)
    assert O.ec_mul(O.G, O.P) is None            # g has order p


def test_field_golden():
    for c in load("primitives.json")["field"]:
        a, b = int(c["a"], 16), int(c["b"], 16)
        assert (a + b) % O.P == int(c["add"], 16)
        assert (a - b) % O.P == int(c["sub"], 16)
        assert a * b % O.P == int(c["mul"], 16)
        assert O.fp_inv(a) == int(c["inv"], 16)
    with pytest.raises(ZeroDivisionError):
        O.fp_inv(O.P)


def test_exp_and_mul_golden():
    g = load("primitives.json")
    for c in g["exp"]:
        assert O.encode_elem(O.ec_mul(O.G, int(c["k"], 16))).hex() == c["elem"]
    for c in g["mul"]:
        assert O.encode_elem(O.ec_add(elem(c["a"]), elem(c["b"]))).hex() == c["sum"]


def test_pairing_golden():
    for c in load("primitives.json")["pair"]:
        a, b = int(c["a"], 16), int(c["b"], 16)
        t = O.pairing(O.ec_mul(O.G, a), O.ec_mul(O.G, b))
        assert [hex(t[0]), hex(t[1])] == c["t"]


def test_hash_and_encoding_golden():
    g = load("primitives.json")
    for c in g["h2s"]:
        assert O.hash_to_scalar(bytes.fromhex(c["data"]), bytes.fromhex(c["tag"])) == int(c["v"], 16)
    for c in g["enc"]:
        assert O.encode_scalar(int(c["s"], 16)).hex() == c["bytes"]


@pytest.mark.parametrize("case", load("mvpoly.json"), ids=lambda c: "x".join(map(str, c["shape"])))
def test_mvpoly_golden(case):
    shape = tuple(case["shape"])
    vals = ints(case["values"])
    coeffs = O.interpolate_lagrange(vals, shape)
    assert coeffs == ints(case["coeffs"])
    pt = ints(case["point"])
    assert O.evaluate(coeffs, shape, pt) == int(case["eval"], 16)
    qs, y = O.open_quotients(coeffs, shape, pt)
    assert y == int(case["y"], 16)
    assert qs == [ints(q) for q in case["quotients"]]
    assert O.barycentric_eval(vals, shape, pt) == int(case["bary"], 16)
    qg, yg = O.open_quotients(coeffs, shape, case["grid_point"])
    assert yg == int(case["grid_y"], 16)
    assert qg == [ints(q) for q in case["grid_quotients"]]


@pytest.mark.parametrize("case", load("commit_small.json"), ids=lambda c: "x".join(map(str, c["shape"])) + "-" + c["kind"])
def test_commit_small_golden(case):
    shape = tuple(case["shape"])
    entropy = bytes.fromhex(case["entropy"])
    taus = O.derive_taus(shape, entropy)
    assert taus == ints(case["taus"])
    srs = [O.ec_mul(O.G, e) for e in O.monomial_exponents(shape, taus)]
    assert [O.encode_elem(e).hex() for e in srs] == case["srs"]
    axis = [elem(a) for a in case["axis"]]
    vals = ints(case["values"])
    C = O.tc_commit(srs, vals, shape)
    assert O.encode_elem(C).hex() == case["commitment"]
    pt = ints(case["point"])
    y, proofs = O.tc_open(srs, vals, shape, pt)
    assert y == int(case["y"], 16)
    assert [O.encode_elem(e).hex() for e in proofs] == case["proofs"]
    # trapdoor oracle agrees with the MSM route
    assert O.commit_trapdoor(vals, shape, taus) == C
    yt, pt_proofs = O.open_trapdoor(vals, shape, taus, pt)
    assert yt == y and pt_proofs == proofs
    assert O.tc_verify(axis, C, pt, y, proofs) is True
    assert O.tc_verify(axis, C, pt, (y + 1) % O.P, proofs) is False


def test_quantize_spec_examples():
    # SPEC.md:542-544
    assert O.quantize(np.array([0.0, 1.5, -1.0]), 16) == [0, 98304, O.P - 65536]
    # round half to even at the 2^-16 grid
    half = 2.0 ** -17
    assert O.quantize(np.array([half, 3 * half, -half, -3 * half]), 16) == [0, 2, 0, O.P - 2]
    with pytest.raises(ValueError):
        O.quantize(np.array([np.inf]))
    with pytest.raises(ValueError):
        O.quantize(np.array([np.nan]))
    with pytest.raises(ValueError):
        O.quantize(np.array([2.0 ** 150]), 16)


def test_spec_kats():
    # SPEC.md:125-127 lex_index
    assert O.lex_index((0, 0), (3, 3)) == 0
    assert O.lex_index((1, 2), (3, 3)) == 5
    assert O.lex_index((1, 2, 3), (2, 3, 4)) == 23
    # T[i,j] = z_i z_j on {1,2}^2 -> X1*X2
    assert O.interpolate_lagrange([1, 2, 2, 4], (2, 2)) == [0, 0, 0, 1]
    # X^2 / (X - 3) -> q = X + 3, r = 9
    q, r = O.divide_by_linear([0, 0, 1], (3,), 0, 3)
    assert q == [3, 1, 0] and r == [9, 0, 0]
    # X1*X2 at (2,3) -> q1 = X2, q2 = 2, y = 6
    qs, y = O.open_quotients([0, 0, 0, 1], (2, 2), (2, 3))
    assert qs[0] == [0, 1, 0, 0] and qs[1] == [2, 0, 0, 0] and y == 6


def test_terkle_oracle_structure():
    leaves = list(range(1, 33))
    levels, values = O.terkle_build(leaves, (2, 2, 2), lambda z: O.ec_mul(O.G, sum(z) % O.P))
    assert [len(lv) for lv in levels] == [8, 1]
    assert O.terkle_depth(1, 8) == 1 and O.terkle_depth(8, 8) == 1 and O.terkle_depth(9, 8) == 2
    assert O.terkle_child_point(5, (2, 2, 2)) == [2, 1, 2]


@pytest.mark.parametrize("shape", [(4,), (3, 5), (8, 4, 2), (2, 3, 4, 5)])
def test_barycentric_eval_small_matches(shape):
    """The numpy limb contraction used for full-size configs equals barycentric_eval."""
    import numpy as np
    g = np.random.default_rng(len(shape))
    n = int(np.prod(shape))
    q = g.integers(-(1 << 29), 1 << 29, n)
    pt = [int(g.integers(0, 1 << 62)) * (1 << 99) % O.P for _ in shape]
    pt[0] = 2 if shape[0] >= 2 else pt[0]          # a grid node on the leading axis
    assert O.barycentric_eval_small(q, shape, pt) == O.barycentric_eval([int(v) % O.P for v in q], shape, pt)
    pt[0] = 123456789
    assert O.barycentric_eval_small(q, shape, pt) == O.barycentric_eval([int(v) % O.P for v in q], shape, pt)


def test_quantize_signed_matches():
    import numpy as np
    x = np.random.default_rng(0).standard_t(3, 4096).astype(np.float16)
    assert [int(v) % O.P for v in O.quantize_signed(x, 16)] == O.quantize(x, 16)
