"""torchrun worker for tests/test_gpu_multirank.py: the multi-GPU prover paths (dist.py) on
`WORLD_SIZE` ranks; rank 0 prints one JSON line with the roots, commitments and proof bytes."""
import hashlib
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2602_12630_b200 as tcb
    from paper_2602_12630_b200.dist import open_many_dist, prover_commit_dist, prover_commit_pipeline_dist

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    n_layers, shape = int(os.environ.get("TC_T_LAYERS", "7")), (8, 8, 16)
    torch.cuda.set_device(0)
    dist.init_process_group(os.environ.get("TC_DIST_BACKEND", "gloo"))
    g = np.random.default_rng(3)
    host = [(g.standard_t(3, 1024) * (1 + l)).astype(np.float16) for l in range(n_layers)]
    layers = {l: torch.from_numpy(h).cuda() for l, h in enumerate(host)}
    srs, _ = tcb.setup_srs(shape, b"dist-test")
    comms, root, tree = prover_commit_dist(layers, srs, n_layers, rank, world)
    roots = [r.to_bytes().hex() for _, r, _ in prover_commit_pipeline_dist(
        [layers, {l: t.cpu() for l, t in layers.items()}, layers], srs, n_layers, rank, world, depth=2)]
    rng = random.Random(5)
    chals = [(l, [rng.randrange(tcb.P) for _ in shape]) for l in [0, 0, 0, 0, 0, 0, 0, 1, 2, 3] + list(range(n_layers))]
    ops, pfs = open_many_dist(srs, layers, chals, rank, world, tree=tree)
    blob = b"".join(op.to_bytes(pt) for op, (_, pt) in zip(ops, chals))
    blob += b"".join(p.to_bytes(tree.config) for p in pfs)
    if rank == 0:
        print(json.dumps({"root": root.to_bytes().hex(), "pipeline_roots": roots,
                          "comms": [c.to_bytes().hex() for c in comms],
                          "proofs_sha": hashlib.sha256(blob).hexdigest()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
