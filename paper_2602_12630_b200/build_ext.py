"""Build libtcb200.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtcb200.so")
SOURCES = ["capi.cu", "msm.cu", "small_msm.cu", "srs.cu", "derive.cu", "quantize.cu", "interp.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-I" + os.path.join(os.path.dirname(HERE), "include")]


def _compile(src, build_dir, extra):
    obj = os.path.join(build_dir, src.replace(".cu", ".o"))
    cmd = [NVCC] + FLAGS + list(extra) + ["-c", os.path.join(CSRC, src), "-o", obj]
    subprocess.run(cmd, check=True)
    return obj


def _stale(out):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    for root in (CSRC, os.path.join(os.path.dirname(HERE), "include")):
        for f in os.listdir(root):
            if os.path.getmtime(os.path.join(root, f)) > t:
                return True
    return os.path.getmtime(__file__) > t


def build(force=False, verbose=True, out=OUT, extra=()):
    """Compile every CUDA source for sm_100a and link the shared library `out`.
    `extra`: additional nvcc flags (e.g. -DTC_MULV=0 for A/B variants)."""
    if not force and not _stale(out):
        return out
    build_dir = os.path.join(HERE, "_build", os.path.basename(out).replace(".so", ""))
    os.makedirs(build_dir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, build_dir, extra), SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp"] + objs
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    if verbose:
        print("built", out, file=sys.stderr)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--force"]
    out = OUT
    extra = []
    for a in args:
        if a.startswith("--out="):
            out = os.path.abspath(a[6:])
        else:
            extra.append(a)
    build(force="--force" in sys.argv or bool(extra), out=out, extra=extra)
