"""Where the host time of ONE lone prover_commit goes (cProfile, config 3)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
layers = [torch.from_numpy(h).cuda() for h in bench.make_layers_host(cfg, range(32))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=0)
srs.prepare("float16")
for _ in range(3):
    tcb.prover_commit(layers, srs)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    tcb.prover_commit(layers, srs)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
