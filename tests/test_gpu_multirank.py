"""Multi-rank prover paths on ONE GPU: torchrun ranks share the device (gloo moves the one
gather through host memory; the ranks' kernels never wait on one another).  Roots,
commitments and every proof byte must be identical for world sizes 1, 2, 3 and 4 — 3 and 4
do not divide the 7 layers, so layers are split into chunks whose partial MSM sums are
combined after the gather — and the bench's multi-rank path must reproduce the one-rank
config-3 root."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(world, script_args, extra_env, port):
    env = dict(os.environ, TC_DIST_BACKEND="gloo", **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}"] + script_args
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_dist_prover_identical_across_world_sizes():
    res = {w: _torchrun(w, [os.path.join(ROOT, "tests", "_dist_worker.py")], {}, 29540 + w) for w in (1, 2, 3, 4)}
    for w in (2, 3, 4):
        assert res[w]["root"] == res[1]["root"], w
        assert res[w]["comms"] == res[1]["comms"], w
        assert res[w]["pipeline_roots"] == [res[1]["root"]] * 3, w
        assert res[w]["proofs_sha"] == res[1]["proofs_sha"], w
    # and equal to the single-process prover_commit
    import numpy as np
    import paper_2602_12630_b200 as tcb
    g = np.random.default_rng(3)
    host = [(g.standard_t(3, 1024) * (1 + l)).astype(np.float16) for l in range(7)]
    srs, _ = tcb.setup_srs((8, 8, 16), b"dist-test")
    comms, root = tcb.prover_commit([torch.from_numpy(h).cuda() for h in host], srs)
    assert root.to_bytes().hex() == res[1]["root"]
    assert [c.to_bytes().hex() for c in comms] == res[1]["comms"]


def _bench(prefix, extra):
    env = dict(os.environ, **extra)
    out = subprocess.run(prefix + [os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1", "--no-cpu",
                                   "--no-forward", "--no-monomial"] + (["--gpus", "2"] if len(prefix) > 1 else []),
                         capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def test_bench_two_ranks_same_root_as_one():
    one = _bench([sys.executable], {})
    two = _bench([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                  "--master-addr=127.0.0.1", "--master-port=29533"], {"TC_DIST_BACKEND": "gloo"})
    assert two["n_gpus"] == 2 and two["config"]["parallelism"] == "layers/2"
    assert two["root"] == one["root"]


def test_bench_config4_two_ranks():
    """bench.py --config 4 under torchrun with 2 ranks: openings split by cost over the
    ranks, every proof gathered to every rank; the bench verifies a sample of openings and
    membership proofs on each rank before reporting."""
    env = dict(os.environ, TC_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--config", "4", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0


_NCCL1 = r'''
import os, sys, json
sys.path.insert(0, os.environ["TC_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2602_12630_b200 as tcb
from paper_2602_12630_b200.dist import prover_commit_pipeline_dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
g = np.random.default_rng(3)
host = [(g.standard_t(3, 1024) * (1 + l)).astype(np.float16) for l in range(7)]
layers = {l: torch.from_numpy(h).cuda() for l, h in enumerate(host)}
srs, _ = tcb.setup_srs((8, 8, 16), b"dist-test")
roots = [r.to_bytes().hex() for _, r, _ in prover_commit_pipeline_dist([layers] * 4, srs, 7, 0, 1, depth=3)]
print(json.dumps({"roots": roots}))
dist.destroy_process_group()
'''


def test_nccl_device_gather_one_rank():
    """The NCCL all-gather of the part encodings (device buffers, issued on the pipeline
    context's stream) on a one-rank NCCL group, forced on: four pipelined forwards give the
    single-process root."""
    env = dict(os.environ, TC_DIST_FORCE_GATHER="1", TC_ROOT=ROOT)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                          "--master-addr=127.0.0.1", "--master-port=29539", "--no-python",
                          sys.executable, "-c", _NCCL1], capture_output=True, text=True, env=env, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    roots = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])["roots"]
    import numpy as np
    import paper_2602_12630_b200 as tcb
    g = np.random.default_rng(3)
    host = [(g.standard_t(3, 1024) * (1 + l)).astype(np.float16) for l in range(7)]
    srs, _ = tcb.setup_srs((8, 8, 16), b"dist-test")
    _, root = tcb.prover_commit([torch.from_numpy(h).cuda() for h in host], srs)
    assert roots == [root.to_bytes().hex()] * 4
