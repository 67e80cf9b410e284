"""INTEGRATION.md's reference-side ctypes binding, executed verbatim: loading a published SRS
(reference-generated points from tests/golden/commit_small.json) through tc_srs_load and
committing field elements through tc_commit must give the reference's commitment."""
import os
import re
import types

import pytest

from oracle import tc_oracle as O
from tests.golden_io import ints, load

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def stub():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        code = re.search(r"```python\n(# tensorcommit/b200.py.*?)```", fh.read(), re.S).group(1)
    os.environ["TC_B200_LIB"] = os.path.join(ROOT, "paper_2602_12630_b200", "libtcb200.so")
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


@pytest.mark.parametrize("case", load("commit_small.json"), ids=lambda c: "x".join(map(str, c["shape"])) + "-" + c["kind"])
def test_integration_stub_matches_reference(stub, case):
    backend = types.SimpleNamespace(encode_elem=O.encode_elem, decode_elem=O.decode_elem)
    srs = types.SimpleNamespace(shape=tuple(case["shape"]),
                                monomial_elems=[O.decode_elem(bytes.fromhex(e)) for e in case["srs"]],
                                axis_elems=[O.decode_elem(bytes.fromhex(e)) for e in case["axis"]])
    h = stub["load_srs"](backend, srs)
    got = stub["tc_commit"](backend, h, ints(case["values"]))
    assert O.encode_elem(got).hex() == case["commitment"]
