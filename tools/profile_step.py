"""One config-3 prover step for profiling: setup + 1 warm step, then ONE step inside the
NVTX range "step" (ncu --nvtx --nvtx-include "step/" selects exactly its launches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[int(os.environ.get("TC_PROFILE_CONFIG", "3"))]
n_layers = int(os.environ.get("TC_PROFILE_LAYERS", cfg["layers"]))
dev = torch.device("cuda", 0)
if cfg is bench.CONFIGS[5]:
    layers = bench.make_layers_device(cfg, range(n_layers), dev)
else:
    layers = [torch.from_numpy(h).to(dev) for h in bench.make_layers_host(cfg, range(n_layers))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/profile", device=0)
tcfg = tcb.TreeConfig(shape=bench.NODE_SHAPE)
node = tcb.authtree.node_srs(tcfg, device=0)


def step():
    # the bench's step: protocol.prover_commit (tc_commit_tree: commitments, device leaf
    # hashing and the tree in one call)
    return tcb.prover_commit(layers, srs, tree_config=tcfg, node_srs=node)[1]


step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
root = step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("root", root.to_bytes().hex()[:32])

if os.environ.get("TC_PROFILE_TIME"):
    import time
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    print("step ms", e0.elapsed_time(e1) / 10, "layers", n_layers)
