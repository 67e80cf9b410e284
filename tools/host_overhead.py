"""Host-side cost per forward of the forward pipeline (cProfile over K forwards of n layers):
where the Python / ctypes time goes when the GPU work per forward is short."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_12630_b200 as tcb  # noqa: E402

n = int(os.environ.get("TC_HO_LAYERS", "4"))
cfg = bench.CONFIGS[3]
layers = [torch.from_numpy(h).cuda() for h in bench.make_layers_host(cfg, range(n))]
srs, _ = tcb.setup_srs(cfg["shape"], b"tc-b200/config3", device=0)
srs.prepare("float16")
K = 40


def run(k):
    for _ in tcb.prover_commit_pipeline([layers] * k, srs, depth=3):
        pass


run(5)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
run(K)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(14)
