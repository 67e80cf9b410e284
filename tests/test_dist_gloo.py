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


# ---------------------------------------------------------------- layer-chunk partition (dist.py)
def test_work_partition_covers_everything_once():
    from paper_2602_12630_b200.dist import gather_layout, work_partition
    for n_layers, n in ((7, 1024), (32, 2 ** 21), (40, 41943040), (1, 5), (3, 7)):
        for world in (1, 2, 3, 4, 5, 8):
            allp = work_partition(n_layers, n, world)
            seen = {}
            for parts in allp:
                for l, s, c in parts:
                    assert 0 <= s and c > 0 and s + c <= n
                    seen.setdefault(l, []).append((s, c))
            for l in range(n_layers):
                segs = sorted(seen[l])
                assert segs[0][0] == 0 and sum(c for _, c in segs) == n
                assert all(a[0] + a[1] == b[0] for a, b in zip(segs, segs[1:]))
            sizes = [sum(c for _, _, c in p) for p in allp]
            assert max(sizes) - min(sizes) <= 1
            if n_layers % world == 0:
                assert all(c == n for p in allp for _, _, c in p)     # whole layers only
            per, rows, layer_of = gather_layout(allp)
            assert layer_of == sorted(layer_of) and len(rows) == len(layer_of)


def _chunk_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import tc_oracle as O
    from paper_2602_12630_b200.dist import _gather_rows, gather_layout, part_inputs, work_partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape, taus, n_layers = (2, 4), [12345, 678], 5
    layers = {l: torch.arange(8, dtype=torch.int64) * (l + 1) - 3 for l in range(n_layers)}
    allp = work_partition(n_layers, 8, world)
    ins = part_inputs(layers, allp[rank], 8)
    per, rows, layer_of = gather_layout(allp)
    buf = torch.zeros((per, 43), dtype=torch.uint8)
    for i, t in enumerate(ins):   # stand-in for tc_commit_points_launch: the chunk's exact commitment
        pt = O.commit_trapdoor([int(v) % O.P for v in t.tolist()], shape, taus)
        buf[i] = torch.frombuffer(bytearray(O.encode_elem(pt)), dtype=torch.uint8)
    got = _gather_rows(buf, world, None, False)[torch.tensor(rows)]
    comms = [None] * n_layers      # stand-in for tc_tree_from_points_launch's per-layer sum
    for row, l in zip(got, layer_of):
        comms[l] = O.ec_add(comms[l], O.decode_elem(bytes(row.tolist())))
    q.put((rank, [O.encode_elem(c) for c in comms]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_layer_chunks_partial_sums_gloo(world):
    """Ranks commit zero-masked chunks of layers; summing the gathered partial commitments
    per layer gives every layer's whole commitment on every rank (linearity of the
    Lagrange-route commitment), for world sizes that do not divide the layer count."""
    from oracle import tc_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [O.encode_elem(O.commit_trapdoor([(v * (l + 1) - 3) % O.P for v in range(8)], (2, 4), [12345, 678]))
            for l in range(5)]
    for _, encs in res:
        assert encs == want


def test_hot_layer_plan_balances_and_covers():
    """Multi-GPU openings: every challenge assigned exactly once, hot layers' openings dealt
    out to every rank, slice-commitment rows cover the first axis once."""
    from paper_2602_12630_b200.dist import hot_layer_plan
    import numpy as np
    score = np.random.default_rng(4).pareto(1.5, 32) + 1e-3
    picks = [int(l) for l in np.random.default_rng(5).choice(32, size=256, p=score / score.sum())]
    for world in (1, 2, 3, 4, 8):
        hot, rows, parts = hot_layer_plan(picks, world, 32, 4)
        assert sorted(i for p in parts for i in p) == list(range(256))
        assert all(p == sorted(p) for p in parts)
        assert rows[0][0] == 0 and rows[-1][1] == 32 and all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert hot == sorted(l for l in set(picks) if picks.count(l) >= 6)
        for l in hot:
            owners = [r for r, p in enumerate(parts) if any(picks[i] == l for i in p)]
            assert len(owners) == min(world, picks.count(l))
