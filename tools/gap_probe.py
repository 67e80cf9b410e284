"""Idle gaps on the GPU timeline of the config-3 prover step (torch.profiler / CUPTI kernel
and memcpy records): the largest gaps between consecutive device activities and their
neighbours, to attribute the difference between the step's event time and its kernel sum."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
dev = torch.device("cuda", 0)
layers = [torch.from_numpy(h).to(dev) for h in bench.make_layers_host(cfg, range(32))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/profile", device=0)
tcfg = tcb.TreeConfig(shape=bench.NODE_SHAPE)
node = tcb.authtree.node_srs(tcfg, device=0)


def step():
    return tcb.prover_commit(layers, srs, tree_config=tcfg, node_srs=node)[1]


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in evs)
span = evs[-1].time_range.end - evs[0].time_range.start
print(f"3 steps: span {span / 1e3:.3f} ms, device busy {busy / 1e3:.3f} ms, idle {(span - busy) / 1e3:.3f} ms")
gaps = []
for a, b in zip(evs, evs[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 0:
        gaps.append((g, a.name[:50], b.name[:50]))
gaps.sort(reverse=True)
for g, a, b in gaps[:25]:
    print(f"{g:8.1f} us  after {a:50s} before {b}")
