"""Determinism / correctness probe: config-3 commitments computed repeatedly (device path
and host-streaming path) must be identical; mismatching layers are checked against the
trapdoor oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
host = [torch.from_numpy(h) for h in bench.make_layers_host(cfg, range(32))]
dev = [h.cuda() for h in host]
srs, td = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=0)
runs = [[c.elem for c in tcb.tc_commit_many(srs, dev)] for _ in range(4)]
runs.append([c.elem for c in tcb.tc_commit_many(srs, [h.pin_memory() for h in host])])
bad = sorted({l for r in runs[1:] for l in range(32) if r[l] != runs[0][l]})
print("layers differing between runs:", bad)
if bad and "--oracle" in sys.argv:
    from oracle import tc_oracle as O
    for l in bad[:2]:
        want = O.commit_trapdoor(O.quantize(host[l].numpy().reshape(-1).astype(np.float64), 16), cfg["shape"],
                                 list(td.taus))
        print("layer", l, "runs equal to oracle:", [r[l] == want for r in runs])
