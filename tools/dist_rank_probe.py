"""Per-rank cost of the multi-GPU path on one GPU: the dist pipeline (device part encodings,
device tree) at world size 1 over all 32 config-3 layers vs the single-GPU forward pipeline,
and over the 4 layers one of 8 ranks owns (the per-rank work at N = 8, without the
all-gather).  Prints ms per forward (CUDA events, K forwards)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402
from paper_2602_12630_b200.dist import prover_commit_pipeline_dist  # noqa: E402

cfg = bench.CONFIGS[3]
dev = torch.device("cuda", 0)
layers = [torch.from_numpy(h).to(dev) for h in bench.make_layers_host(cfg, range(cfg["layers"]))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=0)
srs.prepare("float16")
K = 20
DEPTH = int(os.environ.get("TC_PROBE_DEPTH", "3"))


def timed(fn):
    fn(max(3, DEPTH + 2))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    root = fn(K)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, root


def pipe(n):
    def f(k):
        r = None
        for _, r, _ in tcb.prover_commit_pipeline([layers[:n]] * k, srs, depth=DEPTH):
            pass
        return r
    return f


def dpipe(n):
    d = dict(enumerate(layers[:n]))

    def f(k):
        r = None
        for _, r, _ in prover_commit_pipeline_dist([d] * k, srs, n, 0, 1, depth=DEPTH):
            pass
        return r
    return f


for n in [int(x) for x in os.environ.get("TC_PROBE_LAYERS", "32,4").split(",")]:
    a, ra = timed(pipe(n))
    b, rb = timed(dpipe(n))
    print(f"{n} layers: forward pipeline {a:.3f} ms, dist pipeline (world 1) {b:.3f} ms, roots equal {ra == rb}")
