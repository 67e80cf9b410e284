"""Multi-rank host logic of the prover (layer partition + one all-gather of commitments +
identical Terkle leaves on every rank), world_size 2 over gloo on CPU."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2602_12630_b200.dist import allgather_commitments, layer_partition


def test_layer_partition_covers_all():
    for n in (1, 5, 32, 40):
        for world in (1, 2, 3, 4, 8):
            parts = [layer_partition(n, r, world) for r in range(world)]
            flat = [l for p in parts for l in p]
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        layer_partition(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_layers, q):
    import torch.distributed as dist

    from oracle import tc_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = layer_partition(n_layers, rank, world)
    # stand-in commitments: g^(layer+1), encoded exactly like the real ones
    local = [O.encode_elem(O.ec_mul(O.G, l + 1)) for l in mine]
    encs = allgather_commitments(local, n_layers, rank, world)
    leaves = [O.hash_to_scalar(e, O.LEAF_TAG) for e in encs]
    q.put((rank, encs, leaves))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_layers", [5, 8])
def test_allgather_commitments_gloo(n_layers):
    from oracle import tc_oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_layers, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [O.encode_elem(O.ec_mul(O.G, l + 1)) for l in range(n_layers)]
    for rank, encs, leaves in res:
        assert encs == want
        assert leaves == [O.hash_to_scalar(e, O.LEAF_TAG) for e in want]
