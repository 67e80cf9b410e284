"""Config-4 openings for profiling: the bench workload (256 challenges, Pareto layer
scores) through tc_open_many inside the NVTX range "open"; prints the wall time."""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
layers = [torch.from_numpy(h).cuda() for h in bench.make_layers_host(cfg, range(32))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=0)
if os.environ.get("TC_C4_COMMIT"):
    comms, root, tree = tcb.prover_commit(layers, srs, return_tree=True)
score = np.random.default_rng(4).pareto(1.5, 32) + 1e-3
picks = np.random.default_rng(5).choice(32, size=256, p=score / score.sum())
rng = random.Random(6)
chals = [(int(l), [rng.randrange(tcb.P) for _ in cfg["shape"]]) for l in picks]
ts, pts = [layers[l] for l, _ in chals], [pt for _, pt in chals]
tcb.tc_open_many(srs, ts[:16], pts[:16])
torch.cuda.synchronize()
for rep in range(int(os.environ.get("TC_C4_REPS", "1"))):
    torch.cuda.nvtx.range_push("open")
    t0 = time.perf_counter()
    tcb.tc_open_many(srs, ts, pts, **({"parallel": 1} if os.environ.get("TC_C4_SERIAL") else {}))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    torch.cuda.nvtx.range_pop()
    print(f"256 openings: {wall * 1e3:.1f} ms ({256 / wall:.0f} /s)")
if os.environ.get("TC_C4_COMMIT"):
    t0 = time.perf_counter()
    proofs = [tcb.prove(tree, l) for l, _ in chals]
    print(f"membership proofs: {(time.perf_counter() - t0) * 1e3:.1f} ms")
