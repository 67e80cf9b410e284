"""Config-3 forwards through prover_commit (one at a time) vs prover_commit_pipeline (two
contexts): ms per forward by CUDA-synchronised wall time over K forwards."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

cfg = bench.CONFIGS[3]
dev = torch.device("cuda", 0)
layers = [torch.from_numpy(h).to(dev) for h in bench.make_layers_host(cfg, range(32))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/profile", device=0)
tcfg = tcb.TreeConfig(shape=bench.NODE_SHAPE)
node = tcb.authtree.node_srs(tcfg, device=0)
K = int(os.environ.get("K", "20"))
for depth in (0, 2, 3, 0, 2):
    for _ in range(2):
        if depth:
            roots = [r for _, r, _ in tcb.prover_commit_pipeline([layers] * K, srs, tree_config=tcfg,
                                                                  node_srs=node, depth=depth)]
        else:
            roots = [tcb.prover_commit(layers, srs, tree_config=tcfg, node_srs=node)[1] for _ in range(K)]
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    if depth:
        roots = [r for _, r, _ in tcb.prover_commit_pipeline([layers] * K, srs, tree_config=tcfg, node_srs=node,
                                                              depth=depth)]
    else:
        roots = [tcb.prover_commit(layers, srs, tree_config=tcfg, node_srs=node)[1] for _ in range(K)]
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / K
    print(f"depth {depth}: {ms:.3f} ms per forward, roots equal {len(set(r.to_bytes() for r in roots)) == 1}")
