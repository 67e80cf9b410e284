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


def test_tcop_tctp_cross_checked_with_oracle_verifier():
    """Openings and membership proofs produced by the ORACLE (the reference's arithmetic),
    serialised through the package's TCOP / TCTP encoders, decode to
    objects the oracle verifiers accept; the TCOP byte layout is checked field by field."""
    import struct

    from paper_2602_12630_b200.authtree import MembershipProof, TreeConfig
    from paper_2602_12630_b200.commit import TensorOpening
    rng = random.Random(4)
    shape = (2, 3)
    srs_elems, axis, taus = O.setup_srs(shape, b"wire")
    vals = [rng.randrange(O.P) for _ in range(6)]
    C = O.tc_commit(srs_elems, vals, shape)
    pt = [rng.randrange(O.P) for _ in shape]
    y, proofs = O.tc_open(srs_elems, vals, shape, pt)
    raw = TensorOpening(y, tuple(proofs)).to_bytes(pt)
    assert raw[:4] == b"TCOP" and struct.unpack_from("<H", raw, 4)[0] == 2
    assert raw[6:6 + 42] == b"".join(O.encode_scalar(w) for w in pt)
    assert raw[48:69] == O.encode_scalar(y)
    assert raw[69:] == b"".join(O.encode_elem(e) for e in proofs)
    pt2, op2 = TensorOpening.from_bytes(raw)
    assert O.tc_verify(axis, C, list(pt2), op2.y, list(op2.proofs))
    assert not O.tc_verify(axis, C, list(pt2), (op2.y + 1) % O.P, list(op2.proofs))
    # a two-level Terkle membership proof (node shape (2,2), 5 leaves -> 16 slots)
    node_shape = (2, 2)
    n_srs, n_axis, _ = O.setup_srs(node_shape, b"wire-node")
    leaves = [rng.randrange(O.P) for _ in range(5)]
    levels, values = O.terkle_build(leaves, node_shape, lambda z: O.tc_commit(n_srs, z, node_shape))
    i = 4
    nodes, ops = [], []
    pos = i
    for lv in range(len(levels)):
        u, slot = divmod(pos, 4)
        z = values[lv][4 * u:4 * u + 4]
        yy, pp = O.tc_open(n_srs, z, node_shape, O.terkle_child_point(slot, node_shape))
        nodes.append(levels[lv][u])
        ops.append(TensorOpening(yy, tuple(pp)))
        pos = u
    raw = MembershipProof(i, tuple(nodes), tuple(ops)).to_bytes(TreeConfig(shape=node_shape))
    pf = MembershipProof.from_bytes(raw)
    assert O.terkle_verify(levels[-1][0], i, leaves[i], list(pf.nodes), [(o.y, o.proofs) for o in pf.openings],
                           node_shape, n_axis)
