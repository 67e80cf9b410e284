"""Config-4 style openings for profiling: 16 openings of config-3 layers inside NVTX "open"."""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
K = int(os.environ.get("TC_PROFILE_OPENINGS", "16"))
layers = [torch.from_numpy(h).cuda() for h in bench.make_layers_host(cfg, range(4))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/profile", device=0)
rng = random.Random(1)
pts = [[rng.randrange(tcb.P) for _ in cfg["shape"]] for _ in range(K)]
ts = [layers[k % 4] for k in range(K)]
tcb.tc_open_many(srs, ts, pts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.nvtx.range_push("open")
e0.record()
tcb.tc_open_many(srs, ts, pts)
e1.record()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ms per opening", e0.elapsed_time(e1) / K)
