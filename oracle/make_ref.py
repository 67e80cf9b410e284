"""Recipe for oracle/_ref: the UNMODIFIED reference implementation of the path, for the
bench's reference arm (`bench.py --impl reference`, cpu_baseline kind "reference").

The reference (/root/reference/pkg/src/tensorcommit) is pure CPython with stdlib imports
only, so "building" it is copying its three shipped modules, byte for byte, into
oracle/_ref/tensorcommit/ (a namespace package, as in the reference: no __init__.py) and
recording their SHA-256.  oracle/_ref is git-ignored (reference sources never enter the
repository history) but travels to the GPU box with the working tree.  Only bench.py's
reference / cpu_baseline legs import it — never the product path.
"""
import hashlib
import json
import os
import shutil
import sys

SRC = "/root/reference/pkg/src/tensorcommit"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_ref", "tensorcommit")
MODULES = ("field.py", "backend.py", "mvpoly.py")


def build(src=SRC, dst=DST) -> bool:
    """Copy the reference modules; False when the reference tree is absent (GPU box)."""
    if not all(os.path.isfile(os.path.join(src, m)) for m in MODULES):
        return False
    os.makedirs(dst, exist_ok=True)
    manifest = {}
    for m in MODULES:
        shutil.copyfile(os.path.join(src, m), os.path.join(dst, m))
        with open(os.path.join(dst, m), "rb") as fh:
            manifest[m] = hashlib.sha256(fh.read()).hexdigest()
    with open(os.path.join(os.path.dirname(dst), "MANIFEST.json"), "w") as fh:
        json.dump({"source": src, "sha256": manifest}, fh, indent=1)
    return True


def load():
    """(backend, field, mvpoly) modules of the copied reference, or None."""
    root = os.path.dirname(DST)
    if not os.path.isdir(DST):
        return None
    if root not in sys.path:
        sys.path.insert(0, root)
    from tensorcommit import backend, field, mvpoly   # noqa: E402
    return backend, field, mvpoly


if __name__ == "__main__":
    print("copied" if build() else "reference tree absent")
