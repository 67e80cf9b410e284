"""Host check of the twisted Edwards MSM arithmetic (csrc/ec.cuh: extended-coordinate adds on
the a = -1 model of the 2-isogenous curve E': Y^2 = X^3 - 4X, bases phi([1/2] P), results
psi(.)) against the XYZZ / Montgomery affine arithmetic the reference's curve y^2 = x^3 + x
(backend.py:102-146) is written in: round trips, sums, doublings, P + P and P - P through
the mixed add, the neutral element, small multiples.  The same __host__ __device__ code runs
in the kernels; compiled here with nvcc (host only)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not os.path.exists(NVCC) and not shutil.which("nvcc"), reason="nvcc not available")
def test_edwards_vs_montgomery_host(tmp_path):
    exe = tmp_path / "ed_check"
    subprocess.run([NVCC, "-std=c++17", "--expt-relaxed-constexpr", "-o", str(exe),
                    os.path.join(ROOT, "tools", "ed_check.cu")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert '"bad": 0' in out.stdout
