"""Activation capture (SPEC.md:526-534 infer_and_capture) and the captured tensors feeding
prover_commit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _toy(seed=42):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.ReLU(), torch.nn.Linear(32, 16), torch.nn.ReLU())


def test_capture_cpu_deterministic():
    from paper_2602_12630_b200.capture import infer_and_capture
    m = _toy()
    x = torch.ones(2, 16)
    out1, t1 = infer_and_capture(m, x)
    out2, t2 = infer_and_capture(m, x)
    assert len(t1) == 4 and [tuple(t.shape) for t in t1] == [(2, 32), (2, 32), (2, 16), (2, 16)]
    assert all(torch.equal(a, b) for a, b in zip(t1, t2))          # SPEC.md:533 determinism
    z_out, z = infer_and_capture(torch.nn.Sequential(torch.nn.Linear(16, 8, bias=False)), torch.zeros(1, 16))
    assert torch.count_nonzero(z[0]) == 0


@pytest.mark.gpu
def test_capture_then_prover_commit():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_12630_b200 as tcb
    from oracle import tc_oracle as O
    m = torch.nn.Sequential(torch.nn.Linear(64, 64), torch.nn.GELU(), torch.nn.Linear(64, 64)).cuda().half()
    x = torch.randn(8, 64, device="cuda", dtype=torch.float16)
    _, acts = tcb.infer_and_capture(m, x)
    srs, td = tcb.setup_srs((8, 8, 8), b"capture")
    comms, root, tree = tcb.prover_commit(acts, srs, return_tree=True)
    for a, c in zip(acts, comms):
        vals = O.quantize(a.float().cpu().numpy().astype(np.float64), 16)
        assert c.elem == O.commit_trapdoor(vals, (8, 8, 8), list(td.taus))
