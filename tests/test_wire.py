"""Wire formats: TCPL / TCTN byte-identical with the reference (mvpoly.py:567-631), TCOP and
TCTP round trips."""
import random

import pytest

from oracle import tc_oracle as O


def test_tcpl_tctn_match_reference(reference):
    backend, field, mvpoly = reference
    from paper_2602_12630_b200 import mvpoly as M
    be = backend.make_backend("production")
    rng = random.Random(1)
    shape = (3, 4)
    vals = [rng.randrange(O.P) for _ in range(12)]
    f = M.MultiPoly(shape, tuple(vals))
    ref_f = mvpoly.MultiPoly(shape, tuple(vals))
    assert M.poly_to_bytes(None, f) == mvpoly.poly_to_bytes(be, ref_f)
    assert M.tensor_to_bytes(None, shape, vals) == mvpoly.tensor_to_bytes(be, shape, vals)
    assert M.poly_from_bytes(None, mvpoly.poly_to_bytes(be, ref_f)) == f
    assert M.tensor_from_bytes(None, mvpoly.tensor_to_bytes(be, shape, vals)) == (shape, vals)


def test_wire_errors():
    from paper_2602_12630_b200 import mvpoly as M
    raw = M.tensor_to_bytes(None, (2,), [1, 2])
    with pytest.raises(ValueError):
        M.tensor_from_bytes(None, raw[:-1])
    with pytest.raises(ValueError):
        M.poly_from_bytes(None, raw)
    with pytest.raises(ValueError):
        M.tensor_from_bytes(None, raw[:-21] + (O.P).to_bytes(21, "little"))


def test_tcop_tctp_roundtrip():
    from paper_2602_12630_b200.authtree import MembershipProof, TreeConfig
    from paper_2602_12630_b200.commit import TensorOpening
    g2 = O.ec_mul(O.G, 2)
    op = TensorOpening(12345, (O.G, None, g2))
    pt = (1, 2, O.P - 1)
    assert TensorOpening.from_bytes(op.to_bytes(pt)) == (pt, op)
    pf = MembershipProof(13, (O.G, g2), (op, TensorOpening(7, (g2, g2, None))))
    raw = pf.to_bytes(TreeConfig())
    assert raw[:4] == b"TCTP"
    assert MembershipProof.from_bytes(raw) == pf
    with pytest.raises(ValueError):
        MembershipProof.from_bytes(raw[:-1])
