"""Monomial-route config-3 step (interpolate -> 162-bit MSM) for profiling."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
layers = [torch.from_numpy(h).cuda() for h in bench.make_layers_host(cfg, range(32))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/profile", device=0)
tcb.tc_commit_many(srs, layers, route="monomial")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("mono")
t0 = time.perf_counter()
tcb.tc_commit_many(srs, layers, route="monomial")
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(f"monomial route: {1e3 * (time.perf_counter() - t0):.1f} ms")
