"""Probe: H2D copy cost of the e2e path (torch copy_ vs tc_commit_batch_host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_12630_b200 as tcb

dev = torch.device("cuda", 0)
n = 512 * 4096
L = 32
host = [torch.from_numpy((np.random.default_rng(l).standard_t(3, n) * 2).astype(np.float16)).pin_memory() for l in range(L)]
print("pinned:", all(h.is_pinned() for h in host))
devs = [torch.empty(n, dtype=torch.float16, device=dev) for _ in range(L)]
srs, _ = tcb.setup_srs((32, 32, 32, 64), b"probe", device=0)

def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

def torch_copy():
    for d, h in zip(devs, host):
        d.copy_(h, non_blocking=True)

print("torch copy ms", ev_time(torch_copy))
print("device commit ms", ev_time(lambda: tcb.tc_commit_many(srs, devs)))
for g in (32, 8):
    print("host commit g=%d ms" % g, ev_time(lambda: tcb.tc_commit_many(srs, host, group=g)))
s = torch.cuda.Stream()
def side_copy():
    with torch.cuda.stream(s):
        for d, h in zip(devs, host):
            d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s)
print("side-stream torch copy ms", ev_time(side_copy))
for g in (1, 4, 8, 16, 32):
    def grouped():
        for i in range(0, L, g):
            tcb.tc_commit_many(srs, devs[i:i + g])
    print("device commit in groups of %d: ms" % g, ev_time(grouped))
