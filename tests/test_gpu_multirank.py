"""Multi-rank bench path on ONE GPU: two torchrun ranks share the device (gloo for the
single gather collective; the kernels of the two ranks never wait on each other).  The
Terkle root must equal the single-rank root: every commitment is computed whole on one
rank, and EC addition is exact."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(cmd_prefix, extra_env):
    env = dict(os.environ, **extra_env)
    out = subprocess.run(cmd_prefix + [os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1", "--no-cpu",
                                       "--no-forward", "--no-monomial"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def test_two_ranks_same_root_as_one():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    one = _bench([sys.executable], {})
    two = _bench([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                  "--master-addr=127.0.0.1", "--master-port=29533"], {"TC_DIST_BACKEND": "gloo"})
    assert two["n_gpus"] == 2 and two["config"]["parallelism"] == "layers/2"
    assert two["root"] == one["root"]
