"""Regression tests for defects found by review."""
import random

import numpy as np
import pytest

from oracle import tc_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("scale_bits", [16, 24, 25, 28, 33, 40])
def test_fp16_zeros_subnormals_large_scale(scale_bits):
    """msm.cu key3: the speculative exponent-table path (fp16, n >= 2^16, Lagrange basis)
    must not treat zeros / subnormals (exponent field 0) as normal values when
    scale_bits >= 25; commitment and opening (quantize_device) must agree with the oracle."""
    import paper_2602_12630_b200 as tcb
    shape = (16, 16, 16, 16)
    n = 65536
    srs, td = tcb.setup_srs(shape, b"adv-scale-bits")
    g = np.random.default_rng(scale_bits)
    x = (g.standard_t(3, n) * 2).astype(np.float16)
    x[g.choice(n, 4096, replace=False)] = 0
    sub = g.choice(n, 4096, replace=False)
    x[sub] = (g.integers(1, 1024, 4096) * np.float16(2.0 ** -24)).astype(np.float16)   # subnormals
    x[:8] = np.array([0, -0.0, 2 ** -24, -(2 ** -24), 6.1e-5, -6.1e-5, 1023 * 2 ** -24, 65504], np.float16)
    xd = torch.from_numpy(x).cuda()
    vals = O.quantize(x.astype(np.float64), scale_bits)
    want = O.commit_trapdoor(vals, shape, list(td.taus))
    for route in ("lagrange", "monomial"):
        assert tcb.tc_commit(srs, xd, scale_bits=scale_bits, route=route).elem == want, route
    pt = [random.Random(scale_bits).randrange(O.P) for _ in shape]
    op = tcb.tc_open(srs, xd, pt, scale_bits=scale_bits)
    assert tcb.tc_verify(srs, tcb.Commitment(want), pt, op)


def test_stream_prefetch_dropped_when_consumer_stops():
    """A prover_commit_stream consumer that stops early leaves the next forward prefetched;
    a later stream whose host buffers reuse those addresses with new contents must commit
    the new contents (the generator's cleanup drops the prefetch)."""
    import paper_2602_12630_b200 as tcb
    shape = (4, 8, 16)
    srs, td = tcb.setup_srs(shape, b"adv-stream")
    g = np.random.default_rng(1)
    a = [torch.from_numpy(g.standard_normal(512).astype(np.float16)).pin_memory() for _ in range(3)]
    b = [torch.from_numpy(g.standard_normal(512).astype(np.float16)).pin_memory() for _ in range(3)]
    gen = tcb.prover_commit_stream([a, b], srs)
    next(gen)            # commits a, prefetches b
    gen.close()          # consumer stops
    for t in b:
        t.mul_(3.0)      # same host buffers, new contents
    (comms, root, _), = list(tcb.prover_commit_stream([b], srs))
    for t, c in zip(b, comms):
        assert c.elem == O.commit_trapdoor(O.quantize(t.numpy().astype(np.float64), 16), shape, list(td.taus))


def test_pipeline_orders_after_input_conversions():
    """tc_commit_tree_launch converts inputs (here: non-contiguous CUDA views that need a
    .contiguous() copy on torch's stream) BEFORE ordering the pipeline stream after torch's
    stream; the pipelined commitments equal the one-shot ones."""
    import paper_2602_12630_b200 as tcb
    shape = (8, 8, 8)
    srs, td = tcb.setup_srs(shape, b"adv-order")
    g = np.random.default_rng(2)
    base = torch.from_numpy(g.standard_normal((4, 2 * 512)).astype(np.float32)).cuda()
    fwds = []
    for k in range(4):
        big = base * (k + 1)
        fwds.append([big[i, ::2] for i in range(4)])   # strided views
    got = [r[0] for r in tcb.prover_commit_pipeline(fwds, srs, depth=3)]
    for fwd, comms in zip(fwds, got):
        for t, c in zip(fwd, comms):
            assert c.elem == O.commit_trapdoor(O.quantize(t.cpu().numpy().astype(np.float64), 16), shape,
                                               list(td.taus))
