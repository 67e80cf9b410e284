"""Probe: kernels of ONE single-layer config-3 commit (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_12630_b200 as tcb

n = 512 * 4096
x = torch.from_numpy((np.random.default_rng(3).standard_t(3, n) * 2).astype(np.float16)).cuda()
srs, _ = tcb.setup_srs((32, 32, 32, 64), b"probe", device=0)
tcb.tc_commit_many(srs, [x])
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("one")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tcb.tc_commit_many(srs, [x])
e1.record()
torch.cuda.synchronize()
print("one-layer commit ms", e0.elapsed_time(e1))
