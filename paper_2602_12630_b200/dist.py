"""Multi-GPU prover (north star: "partitioned across the GPUs by layer and by
MSM point-chunk, with a single tiny NCCL gather to combine partial group sums and roots").

Commitments.  The (layer, element) space of a forward — n_layers x N samples — is cut into
`world` contiguous ranges, one per rank (one process per GPU).  A range covers whole layers
and at most one chunk at each end: a chunk's commitment is a PARTIAL SUM of its layer's
commitment, because the Lagrange-route commitment C_T = sum_w T[w] g^{L_w(tau)} is linear
in the samples, so a chunk is committed as a zero-masked copy of the layer.  When world
divides n_layers (configs 3 and 5 on 1/2/4/8 GPUs) every range is whole layers and no
chunk exists.  Each rank writes its parts' 43-byte encodings into a device buffer
(tc_commit_points_launch), ONE all-gather (NCCL over NVLink; gloo in the CPU tests)
exchanges them, and every rank sums the parts per layer, hashes the leaves and builds the
Terkle tree on the device (tc_tree_from_points_launch) — the same commitments and root on
every rank and for every world size (EC addition is associative; affine output is
canonical).  Everything is stream-ordered on the context's stream: forward k+1's MSMs run
while forward k's gather and tree complete (prover_commit_pipeline_dist).

Openings (config 4).  A layer opened many times ("hot") opens from its slice commitments
H[c', c] (d0 x d0 MSMs over the tensor's slices c' and the SRS slices c): those MSMs are
split by rows c' over the ranks (point-chunks of the layer), ONE all-gather assembles every
hot layer's H on every rank, and the hot openings are dealt out evenly; the other openings
go to ranks by a cost model; the results are all-gathered so every rank holds every proof
(open_many_dist).
"""
from __future__ import annotations

import ctypes as C
import os

ELEM_BYTES = 43


# --------------------------------------------------------------------------- partitioning
def layer_partition(n_layers: int, rank: int, world: int):
    """Contiguous balanced blocks of whole layers: rank r owns layers [lo, hi)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_layers, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def work_partition(n_layers: int, n_elems: int, world: int):
    """Every rank's share of the flattened (layer, element) space: rank r gets elements
    [r T / W, (r + 1) T / W) of T = n_layers n_elems, as a list of parts
    (layer, start, count) in ascending order.  Whole layers when world divides n_layers."""
    if world < 1 or n_layers < 1 or n_elems < 1:
        raise ValueError("bad partition arguments")
    T = n_layers * n_elems
    out = []
    for r in range(world):
        a, b = r * T // world, (r + 1) * T // world
        parts = []
        while a < b:
            l, s = divmod(a, n_elems)
            c = min(b - a, n_elems - s)
            parts.append((l, s, c))
            a += c
        out.append(parts)
    return out


def gather_layout(parts_all):
    """Rows of the padded all-gather buffer (world x per rows) that hold real parts, in
    global order, and the layer of each part."""
    per = max(1, max(len(p) for p in parts_all))
    rows = [r * per + i for r, p in enumerate(parts_all) for i in range(len(p))]
    layer_of = [l for p in parts_all for (l, _, _) in p]
    return per, rows, layer_of


def part_inputs(layers, parts, n_elems):
    """Device inputs of this rank's parts: whole layers as given, a chunk as a zero-masked
    copy of its layer (same grid positions, zeros elsewhere).  layers: layer -> tensor."""
    import torch

    out = []
    for l, s, c in parts:
        t = layers[l]
        if c == n_elems:
            out.append(t)
        else:
            flat = t.reshape(-1)
            m = torch.zeros_like(flat)
            m[s:s + c] = flat[s:s + c]
            out.append(m)
    return out


def _gather_rows(buf, world, group, device_ok: bool):
    """All-gather a (per, 43) uint8 tensor from every rank -> (world * per, 43) on buf's
    device.  NCCL gathers device buffers in place on the current stream; gloo (CPU tests,
    several ranks sharing one GPU) goes through host memory."""
    import torch
    import torch.distributed as dist

    if device_ok or buf.device.type == "cpu":
        out = torch.empty((world * buf.shape[0], buf.shape[1]), dtype=buf.dtype, device=buf.device)
        dist.all_gather_into_tensor(out, buf, group=group)
        return out
    host = buf.cpu()
    out = torch.empty((world * host.shape[0], host.shape[1]), dtype=host.dtype)
    dist.all_gather_into_tensor(out, host, group=group)
    return out.to(buf.device, non_blocking=False)


# --------------------------------------------------------------------------- commitments
class DistProver:
    """prover_commit over `world` ranks (one process per GPU): launch(layers) commits this
    rank's parts, all-gathers every rank's part encodings and launches the device tree on a
    pipeline context; finish(state) returns (commitments, root, tree) for ALL layers."""

    def __init__(self, srs, n_layers: int, rank: int, world: int, *, group=None, tree_config=None, node_srs=None,
                 scale_bits: int = 16, route: str = "auto", depth: int = 4):
        import torch
        import torch.distributed as dist

        from . import authtree
        from ._lib import Context

        self.srs, self.n_layers, self.rank, self.world, self.group = srs, n_layers, rank, world, group
        self.cfg = tree_config or authtree.TreeConfig()
        self.node = node_srs or authtree.node_srs(self.cfg, device=srs.device)
        self.scale_bits, self.route = scale_bits, route
        self.parts_all = work_partition(n_layers, srs.size, world)
        self.parts = self.parts_all[rank]
        self.per, rows, layer_of = gather_layout(self.parts_all)
        self.layer_of = (C.c_uint32 * len(layer_of))(*layer_of)
        self.nparts = len(layer_of)
        self.ctxs = [Context.pipeline(srs.device, k) for k in range(max(1, depth))]
        self.dev = torch.device("cuda", srs.device)
        self.rows = torch.tensor(rows, dtype=torch.long, device=self.dev)
        # TC_DIST_FORCE_GATHER=1: run the all-gather even for one rank (tests the NCCL call
        # and its stream ordering on a single GPU)
        self.force_gather = os.environ.get("TC_DIST_FORCE_GATHER", "0") not in ("", "0") and dist.is_initialized()
        backend = dist.get_backend(group) if (world > 1 or self.force_gather) else "nccl"
        self.device_gather = backend == "nccl"
        self._k = 0

    def layers_needed(self):
        """The layers this rank's parts read."""
        return sorted({l for l, _, _ in self.parts})

    def launch(self, layers: dict):
        """layers: layer index -> tensor (CUDA, or CPU float: copied on the context's stream)
        for at least layers_needed().  Returns the state finish() takes."""
        import torch

        from . import _conv, _lib
        from .commit import _route

        ctx = self.ctxs[self._k % len(self.ctxs)]
        self._k += 1
        with ctx.lock:
            ctx.fixed_stream.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(ctx.fixed_stream):
                dev_layers = {l: (t if t.is_cuda else t.to(self.dev, non_blocking=True)) for l, t in layers.items()
                              if l in set(self.layers_needed())}
                ins = part_inputs(dev_layers, self.parts, self.srs.size)
                conv = [_conv.device_input(t, self.srs.size, f"cuda:{self.srs.device}") for t in ins]
                if len({c[1] for c in conv}) > 1:
                    raise ValueError("all layers must share one dtype")
                buf = torch.zeros((self.per, ELEM_BYTES), dtype=torch.uint8, device=self.dev)
                if conv:
                    arr = (C.c_void_p * len(conv))(*[c[0] for c in conv])
                    ctx.check(_lib.lib().tc_commit_points_launch(ctx.handle, self.srs.handle, arr, len(conv),
                                                                 conv[0][1], self.scale_bits, _route(self.route),
                                                                 buf.data_ptr()), "tc_commit_points_launch")
                if self.world > 1 or self.force_gather:
                    gathered = _gather_rows(buf, self.world, self.group, self.device_gather)
                    allp = gathered.index_select(0, self.rows)
                else:
                    allp = buf[:self.nparts]
                allp = allp.contiguous()
                ctx.check(_lib.lib().tc_tree_from_points_launch(ctx.handle, self.node.handle, allp.data_ptr(),
                                                                self.layer_of, self.nparts, self.n_layers),
                          "tc_tree_from_points_launch")
        return ctx, (dev_layers, ins, conv, buf, allp)

    def finish(self, state):
        from . import authtree
        from .commit import tc_commit_tree_finish

        ctx, _keep = state
        commitments, nodes, vals, depth = tc_commit_tree_finish((ctx, self.n_layers, self.node.size, _keep))
        tree = authtree.tree_from_device(self.cfg, self.n_layers, depth, nodes, vals, self.node)
        return commitments, tree.root, tree


def prover_commit_dist(layers: dict, srs, n_layers: int, rank: int, world: int, **kw):
    """One forward: (commitments of all n_layers, root, tree), identical on every rank."""
    p = DistProver(srs, n_layers, rank, world, depth=1, **kw)
    return p.finish(p.launch(layers))


def prover_commit_pipeline_dist(forwards, srs, n_layers: int, rank: int, world: int, *, depth: int = 4, **kw):
    """prover_commit_dist over a stream of forwards (each a dict layer -> tensor holding at
    least this rank's layers), yielding (commitments, root, tree) per forward in order;
    `depth` contexts keep forwards in flight so one forward's gather and tree overlap the
    next forward's MSMs."""
    p = DistProver(srs, n_layers, rank, world, depth=depth, **kw)
    pending = []
    try:
        for fwd in forwards:
            pending.append(p.launch(fwd))
            if len(pending) == len(p.ctxs):
                yield p.finish(pending.pop(0))
        while pending:
            yield p.finish(pending.pop(0))
    finally:
        for st in pending:
            try:
                p.finish(st)
            except Exception:
                pass


def allgather_commitments(local: list, n_layers: int, rank: int, world: int, device=None, group=None):
    """local: encoded commitments (43 B each) of this rank's whole layers (layer_partition
    order).  Returns the n_layers encodings in layer order, on every rank (host path)."""
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


# --------------------------------------------------------------------------- openings
def _open_sliced(srs, T, d_h43, points, scale_bits=16):
    """Openings of ONE tensor from its assembled slice commitments (tc_open_batch_sliced)."""
    from . import _conv, _lib
    from .commit import TensorOpening
    from .curve import ELEM_BYTES, decode_elems, encode_scalar

    ctx = _lib.Context.get(srs.device)
    ptr, dt, keep = _conv.device_input(T, srs.size, f"cuda:{srs.device}")
    m = len(srs.shape)
    om = b"".join(encode_scalar(int(w)) for pt in points for w in pt)
    ys = C.create_string_buffer(21 * max(1, len(points)))
    pis = C.create_string_buffer(ELEM_BYTES * m * max(1, len(points)))
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_open_batch_sliced(ctx.handle, srs.handle, ptr, d_h43.data_ptr(), len(points), dt,
                                                  scale_bits, om, ys, pis), "tc_open_batch_sliced")
    del keep
    return [TensorOpening(int.from_bytes(ys.raw[21 * i:21 * (i + 1)], "little"),
                          decode_elems(pis.raw[ELEM_BYTES * m * i:ELEM_BYTES * m * (i + 1)], m))
            for i in range(len(points))]


def hot_layer_plan(layer_of_chal, world: int, d0: int, m: int, precomp_min: int = 6):
    """Multi-GPU openings: the layers opened >= precomp_min times ("hot") share their slice
    commitments H (d0 x d0 MSMs) by ROWS — rank r computes rows [r d0 / W, (r+1) d0 / W), one
    all-gather assembles every H on every rank — and their openings are dealt out evenly
    (contiguous chunks per rank); the other ("cold") challenges go to ranks longest-first by
    tc_open_many's cost model on top of that load.  Returns (hot layers, per-rank row ranges,
    per-rank challenge indices)."""
    groups = {}
    for i, l in enumerate(layer_of_chal):
        groups.setdefault(l, []).append(i)
    hot = sorted(l for l, ids in groups.items() if len(ids) >= precomp_min and m >= 2 and d0 * d0 <= 4096)
    rows = [(r * d0 // world, (r + 1) * d0 // world) for r in range(world)]
    out = [[] for _ in range(world)]
    load = [0.0] * world
    for l in hot:
        ids = groups[l]
        for r in range(world):
            part = ids[r * len(ids) // world:(r + 1) * len(ids) // world]
            out[r] += part
            load[r] += 3.0 / world + 0.05 * len(part)
    cold = sorted((ids for l, ids in groups.items() if l not in hot), key=lambda ids: (-len(ids), ids[0]))
    for ids in cold:
        r = min(range(world), key=lambda j: (load[j], j))
        out[r] += ids
        load[r] += 1.4 * len(ids)
    return hot, rows, [sorted(o) for o in out]


def open_many_dist(srs, layers: dict, chals, rank: int, world: int, *, group=None, tree=None, scale_bits: int = 16,
                   **kw):
    """Config-4 openings over `world` ranks.  chals: list of (layer, point); layers: layer ->
    tensor for the hot layers and this rank's challenges (hot_layer_plan).  Hot layers' slice
    commitments are split by rows over the ranks (MSM point-chunks: each row is a set of
    d0 MSMs over one tensor slice) and all-gathered; every rank then opens its share.
    Returns (openings, proofs): every challenge's TensorOpening and — with `tree` — its
    Terkle membership proof, on every rank, in challenge order (same bytes as tc_open_many /
    prove_many on one GPU)."""
    import torch
    import torch.distributed as dist

    from . import _conv, _lib
    from .authtree import MembershipProof, prove_many
    from .commit import TensorOpening, tc_open_many

    m, d0 = len(srs.shape), srs.shape[0]
    if world == 1:
        ops = tc_open_many(srs, [layers[l] for l, _ in chals], [pt for _, pt in chals], scale_bits=scale_bits, **kw)
        pfs = prove_many(tree, [l for l, _ in chals]) if tree is not None else None
        return ops, pfs
    hot, rows, assign = hot_layer_plan([l for l, _ in chals], world, d0, m)
    mine = assign[rank]
    dev = torch.device("cuda", srs.device)
    H = {}
    if hot:
        per = max(hi - lo for lo, hi in rows) * d0
        buf = torch.zeros((len(hot), per, ELEM_BYTES), dtype=torch.uint8, device=dev)
        ctx = _lib.Context.get(srs.device)
        lo, hi = rows[rank]
        for h, l in enumerate(hot):
            ptr, dt, keep = _conv.device_input(layers[l], srs.size, f"cuda:{srs.device}")
            with ctx.lock:
                ctx.bind_stream()
                ctx.check(_lib.lib().tc_open_slices(ctx.handle, srs.handle, ptr, dt, scale_bits, lo, hi,
                                                    buf[h].data_ptr()), "tc_open_slices")
            del keep
        backend = dist.get_backend(group)
        gathered = _gather_rows(buf.reshape(-1, ELEM_BYTES), world, group, backend == "nccl")
        gathered = gathered.reshape(world, len(hot), per, ELEM_BYTES)
        for h, l in enumerate(hot):
            H[l] = torch.cat([gathered[r, h, :(rows[r][1] - rows[r][0]) * d0] for r in range(world)]).contiguous()
    ops = {}
    hot_mine = {}
    cold_mine = []
    for i in mine:
        l = chals[i][0]
        if l in H:
            hot_mine.setdefault(l, []).append(i)
        else:
            cold_mine.append(i)
    for l, ids in hot_mine.items():
        for i, op in zip(ids, _open_sliced(srs, layers[l], H[l], [chals[i][1] for i in ids], scale_bits)):
            ops[i] = op
    if cold_mine:
        got = tc_open_many(srs, [layers[chals[i][0]] for i in cold_mine], [chals[i][1] for i in cold_mine],
                           scale_bits=scale_bits, **kw)
        for i, op in zip(cold_mine, got):
            ops[i] = op
    pfs = prove_many(tree, [chals[i][0] for i in mine]) if (tree is not None and mine) else []
    local = [(i, ops[i].to_bytes(chals[i][1]), pfs[k].to_bytes(tree.config) if pfs else None)
             for k, i in enumerate(mine)]
    allr = [None] * world
    dist.all_gather_object(allr, local, group=group)
    openings, proofs = [None] * len(chals), [None] * len(chals)
    for part in allr:
        for i, ob, pb in part:
            openings[i] = TensorOpening.from_bytes(ob)[1]
            if pb is not None:
                proofs[i] = MembershipProof.from_bytes(pb)
    return openings, (proofs if tree is not None else None)
