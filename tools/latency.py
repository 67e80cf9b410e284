"""Lone-forward latency of prover_commit on config 3 (CUDA events around one forward with
nothing else in flight), min / median of 15, plus the root for cross-checking builds."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
dev = torch.device("cuda", 0)
layers = [torch.from_numpy(h).to(dev) for h in bench.make_layers_host(cfg, range(cfg["layers"]))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=0)
srs.prepare("float16")
ts = []
for i in range(18):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    comms, root = tcb.prover_commit(layers, srs)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
print(os.environ.get("TC_LIB", "default"), "latency ms min %.3f med %.3f" % (min(ts), statistics.median(ts)),
      root.to_bytes().hex()[:16])
