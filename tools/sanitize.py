"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every production
kernel family on a small (16,16,16,16) batch — fp16 commits on both routes (exponent-table
plan with the block-private counting sort and sorted scatter), the device Terkle tree,
openings (grouped quotient MSMs, slice-commitment route, grid nodes), the Lagrange
derivation from a monomial-only SRS, and the distributed points/tree launch."""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_12630_b200 as tcb  # noqa: E402
from paper_2602_12630_b200.dist import prover_commit_dist  # noqa: E402

shape = (16, 16, 16, 16)
srs, td = tcb.setup_srs(shape, b"sanitize")
g = np.random.default_rng(0)
xs = [torch.from_numpy((g.standard_t(3, 65536) * 2).astype(np.float16)).cuda() for _ in range(4)]
comms, root, tree = tcb.prover_commit(xs, srs, return_tree=True)
mono = tcb.tc_commit_many(srs, xs[:2], route="monomial")
assert [c.elem for c in mono] == [c.elem for c in comms[:2]]
rng = random.Random(1)
pts = [[rng.randrange(tcb.P) for _ in shape] for _ in range(8)] + [[3, 5, 16, 1]]
ops = tcb.tc_open_many(srs, [xs[0]] * 7 + [xs[1], xs[2]], pts, parallel=1)
assert all(tcb.tc_verify(srs, comms[i], pt, op) for i, pt, op in zip([0] * 7 + [1, 2], pts, ops))
pf = tcb.prove_many(tree, [0, 3])
m_srs, _ = tcb.setup_srs((4, 8, 16), b"sanitize-derive", lagrange=False)
m_srs.derive_lagrange()
c2, r2, _ = prover_commit_dist(dict(enumerate(xs)), srs, 4, 0, 1)
assert r2 == root
torch.cuda.synchronize()
print("sanitize workload ok")
