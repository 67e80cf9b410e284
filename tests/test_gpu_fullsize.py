"""Full-size parity against the reference-pinned oracle (BASELINE configs 3, 4 and 5).

* config 3: all 32 layers' commitments equal the trapdoor oracle g^{f_T(tau)} and the
  32-leaf Terkle root equals the oracle tree (oracle node commitments: interpolation +
  naive MSM over the node SRS);
* config 4: on that tree, 256 seeded challenges (the bench's) plus grid-node challenges:
  every tc_open_many opening verifies under the oracle's product-of-pairings verifier
  (O.tc_verify, pinned to the reference by tests/test_oracle_vs_reference.py), a spread of
  openings covering every production route equals the trapdoor opening
  (y, pi_i = g^{q_i(tau)}), tampered openings are rejected, and every membership proof
  verifies under the oracle's Terkle check;
* config 5: all 40 layers of [4,2048,5120] (41,943,040 elements each) commit to the oracle
  values and the 40-leaf root equals the oracle tree.

The oracle work runs in a process pool on the host cores (barycentric_eval_small: exact
numpy limb contraction of the leading axis, pinned by tests/test_oracle_golden.py)."""
import multiprocessing as mp
import os
import random
import sys

import numpy as np
import pytest

from oracle import tc_oracle as O

pytestmark = [pytest.mark.gpu,
              # the oracle pool forks a process whose CUDA / torch threads the children never use
              pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")]

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


_HOST = {}   # layer arrays shared with forked oracle workers


def _commit_one(args):
    key, l, shape, taus = args
    q = O.quantize_signed(_HOST[key][l].reshape(-1).astype(np.float64), 16)
    return O.ec_mul(O.G, O.barycentric_eval_small(q, shape, taus))


def _open_one(args):
    key, l, shape, taus, pt = args
    q = O.quantize_signed(_HOST[key][l].reshape(-1).astype(np.float64), 16)
    m = len(shape)
    ev = [O.barycentric_eval_small(q, shape, [pt[j] if j < i else taus[j] for j in range(m)]) for i in range(m + 1)]
    proofs = [O.ec_mul(O.G, (ev[i] - ev[i + 1]) * O.fp_inv(taus[i] - pt[i]) % O.P) for i in range(m)]
    return ev[m], proofs


def _verify_one(args):
    axis, c, pt, y, proofs = args
    return O.tc_verify(axis, c, pt, y, proofs)


def _pool():
    return mp.get_context("fork").Pool(max(1, min(16, os.cpu_count() or 1)))


def _oracle_root(comms, node_srs_elems, node_shape=(2, 2, 2)):
    levels, _ = O.terkle_build([O.leaf_of_commitment(c) for c in comms], node_shape,
                               lambda z: O.tc_commit(node_srs_elems, z, node_shape))
    return levels[-1][0]


@pytest.fixture(scope="module")
def config3():
    import bench
    import paper_2602_12630_b200 as tcb
    cfg = bench.CONFIGS[3]
    host = bench.make_layers_host(cfg, range(cfg["layers"]))
    _HOST["c3"] = host
    srs, td = tcb.setup_srs(cfg["shape"], b"tc-b200/config3")
    layers = [torch.from_numpy(h).cuda() for h in host]
    comms, root, tree = tcb.prover_commit(layers, srs, return_tree=True)
    with _pool() as pool:
        want = pool.map(_commit_one, [("c3", l, cfg["shape"], list(td.taus)) for l in range(cfg["layers"])])
    return dict(cfg=cfg, srs=srs, td=td, layers=layers, comms=comms, root=root, tree=tree, want=want)


def test_config3_all_layers_and_root(config3):
    import paper_2602_12630_b200 as tcb
    assert [c.elem for c in config3["comms"]] == config3["want"]
    node = tcb.authtree.node_srs(tcb.TreeConfig())
    assert config3["root"].elem == _oracle_root(config3["want"], list(node.monomial_elems))
    # the bench's forward pipeline gives the same root
    (_, root_p, _), = list(tcb.prover_commit_pipeline([config3["layers"]], config3["srs"], depth=3))
    assert root_p == config3["root"]


def _config4_challenges(n_layers, shape):
    """The bench's 256 challenges (bench.run_openings) + 8 grid-node challenges."""
    score = np.random.default_rng(4).pareto(1.5, n_layers) + 1e-3
    picks = np.random.default_rng(5).choice(n_layers, size=256, p=score / score.sum())
    rng = random.Random(6)
    chals = [(int(l), [rng.randrange(O.P) for _ in shape]) for l in picks]
    g = random.Random(7)
    for k in range(8):
        l = int(picks[k % 3])      # heavily challenged layers (slice route) and others
        l = l if k < 4 else (int(picks[-1]) + k) % n_layers
        pt = [g.randrange(O.P) for _ in shape]
        for a in range(len(shape)):
            if (k >> a) & 1 or k == 0:
                pt[a] = g.randrange(1, shape[a] + 1)   # grid node on this axis
        chals.append((l, pt))
    return chals


def test_config4_full_openings_and_membership(config3):
    import paper_2602_12630_b200 as tcb
    srs, td, layers, comms, tree = (config3[k] for k in ("srs", "td", "layers", "comms", "tree"))
    shape = config3["cfg"]["shape"]
    chals = _config4_challenges(len(layers), shape)
    ops = tcb.tc_open_many(srs, [layers[l] for l, _ in chals], [pt for _, pt in chals])
    axis = list(srs.axis_elems)
    with _pool() as pool:
        ok = pool.map(_verify_one, [(axis, comms[l].elem, pt, op.y, list(op.proofs)) for (l, pt), op in zip(chals, ops)])
        assert all(ok), [i for i, v in enumerate(ok) if not v][:10]
        # trapdoor equality on openings covering every route: layers opened >= 6 times (slice
        # commitments, exponent-table multi-base MSMs), rarely opened layers (grouped quotient
        # MSMs), grid-node challenges (derivative weights)
        counts = {}
        for l, _ in chals:
            counts[l] = counts.get(l, 0) + 1
        hot = [i for i, (l, _) in enumerate(chals[:256]) if counts[l] >= 6][:6]
        cold = [i for i, (l, _) in enumerate(chals[:256]) if counts[l] < 6][:6]
        grid = list(range(256, len(chals)))
        assert len(hot) >= 4 and len(cold) >= 4
        pick = hot + cold + grid
        want = pool.map(_open_one, [("c3", chals[i][0], shape, list(td.taus), chals[i][1]) for i in pick])
    for i, (y, proofs) in zip(pick, want):
        assert ops[i].y == y and list(ops[i].proofs) == proofs, i
    # tampering is rejected by the oracle verifier
    l, pt = chals[0]
    op = ops[0]
    assert not O.tc_verify(axis, comms[l].elem, pt, (op.y + 1) % O.P, list(op.proofs))
    assert not O.tc_verify(axis, comms[l].elem, pt, op.y, [op.proofs[1], op.proofs[0]] + list(op.proofs[2:]))
    assert not O.tc_verify(axis, comms[(l + 1) % 32].elem, pt, op.y, list(op.proofs))
    # membership proofs for every challenged layer, checked by the oracle's Terkle verifier
    node = tree.srs
    proofs = tcb.prove_many(tree, [l for l, _ in chals])
    root = config3["root"].elem
    for (l, _), pf in zip(chals, proofs):
        leaf = O.leaf_of_commitment(comms[l].elem)
        assert O.terkle_verify(root, l, leaf, list(pf.nodes), [(o.y, o.proofs) for o in pf.openings], (2, 2, 2),
                               list(node.axis_elems))
    pf = proofs[0]
    l0 = chals[0][0]
    assert not O.terkle_verify(root, (l0 + 1) % 32, O.leaf_of_commitment(comms[l0].elem), list(pf.nodes),
                               [(o.y, o.proofs) for o in pf.openings], (2, 2, 2), list(node.axis_elems))


def test_config5_all_layers_and_root():
    """Config 5 on one GPU: 40 layers x 41,943,040 elements, grid (64,128,64,80)."""
    import bench
    import paper_2602_12630_b200 as tcb
    cfg = bench.CONFIGS[5]
    dev = torch.device("cuda", 0)
    layers = bench.make_layers_device(cfg, range(cfg["layers"]), dev)
    _HOST["c5"] = [t.cpu().numpy() for t in layers]
    srs, td = tcb.setup_srs(cfg["shape"], b"tc-b200/config5")
    comms, root = tcb.prover_commit(layers, srs)
    with _pool() as pool:
        want = pool.map(_commit_one, [("c5", l, cfg["shape"], list(td.taus)) for l in range(cfg["layers"])])
    assert [c.elem for c in comms] == want
    node = tcb.authtree.node_srs(tcb.TreeConfig())
    assert root.elem == _oracle_root(want, list(node.monomial_elems))
    del _HOST["c5"]
