"""Multi-GPU partitioning of the prover.

Per-layer commitments are independent, so ranks split the layers with no data-path
collective; the only exchange is ONE all-gather of the 43-byte commitments (NCCL over
NVLink on GPUs, gloo in the CPU tests), after which every rank builds the (tiny) Terkle
tree and holds the same root.  EC points cannot be summed by NCCL reductions, so a
gather (not a reduce) is the right primitive; the root is identical for any world size
because each commitment is computed whole on one rank.
"""
from __future__ import annotations

ELEM_BYTES = 43


def layer_partition(n_layers: int, rank: int, world: int):
    """Contiguous balanced blocks: rank r owns layers [lo, hi)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_layers, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def allgather_commitments(local: list, n_layers: int, rank: int, world: int, device=None, group=None):
    """local: encoded commitments (43 B each) of this rank's layers (layer_partition order).
    Returns the n_layers encodings in layer order, on every rank."""
    import torch
    import torch.distributed as dist

    per = max(len(layer_partition(n_layers, r, world)) for r in range(world))
    buf = torch.zeros((per, ELEM_BYTES), dtype=torch.uint8)
    for i, enc in enumerate(local):
        buf[i] = torch.frombuffer(bytearray(enc), dtype=torch.uint8)
    if device is not None:
        buf = buf.to(device)
    out = torch.empty((world * per, ELEM_BYTES), dtype=torch.uint8, device=buf.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    out = out.cpu()
    result = []
    for r in range(world):
        ids = layer_partition(n_layers, r, world)
        for i in range(len(ids)):
            result.append(bytes(out[r * per + i].tolist()))
    return result
