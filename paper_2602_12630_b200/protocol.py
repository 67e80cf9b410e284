"""Prover side of the protocol harness, hot-path subset:

quantize       SPEC.md:536-544 — RNE(v * 2^16) into F_p on the device (K1)
prover_commit  SPEC.md:546-554 — per-layer commitments + Terkle root over their leaves
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _conv, _lib
from . import authtree
from .authtree import TreeConfig, build, leaf_of
from .commit import (SCALE_BITS, tc_commit_many, tc_commit_stream, tc_commit_stream_tree, tc_commit_tree,
                     tc_commit_tree_finish, tc_commit_tree_launch)


@dataclass
class FieldTensor:
    """Quantised tensor resident on the device: canonical limbs, shape (n, 6) int32."""
    limbs: object
    shape: tuple

    def tolist(self):
        return _conv.limbs_to_ints(self.limbs)

    def __len__(self):
        return int(self.limbs.shape[0])


def quantize(tensor, scale_bits: int = SCALE_BITS) -> FieldTensor:
    """Round-to-nearest-even fixed point: q = RNE(v * 2^scale_bits), negatives -> p - |q|.
    ValueError on non-finite values or |v| * 2^scale_bits >= p/2."""
    import numpy as np
    import torch

    if isinstance(tensor, np.ndarray):
        tensor = torch.from_numpy(np.ascontiguousarray(tensor))
    if not isinstance(tensor, torch.Tensor) or not tensor.is_floating_point():
        tensor = torch.as_tensor(tensor, dtype=torch.float64)
    ctx = _lib.Context.get(tensor.device if tensor.is_cuda else None)
    dev = f"cuda:{ctx.device}"
    t = tensor.detach().to(dev).contiguous()
    n = t.numel()
    out = _conv.empty_limbs(n, dev)
    code = _conv._float_codes()[t.dtype]
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_quantize(ctx.handle, t.data_ptr(), code, n, scale_bits, out.data_ptr()), "quantize")
    return FieldTensor(out, tuple(tensor.shape))


def _device_tree_ok(tensors, srs, node) -> bool:
    """tc_commit_tree applies: CUDA tensors on the SRS's device, a Lagrange node SRS of <= 64
    points (the device tree path of tc_terkle_build)."""
    try:
        import torch
    except ImportError:
        return False
    if node is None or node.size > 64 or not node.has(_lib.SRS_LAGRANGE):
        return False
    return all(isinstance(T, torch.Tensor) and T.is_cuda and T.device.index == srs.device for T in tensors)


def prover_commit(tensors, srs_pool, *, tree_config: TreeConfig = None, scale_bits: int = SCALE_BITS,
                  route: str = "auto", node_srs=None, return_tree: bool = False):
    """prover_commit(tensors, srs) -> (per-layer commitments, Terkle root).

    Per-layer commitments C_l = tc_commit(srs[shape_l], quantize(T_l)) and a Terkle tree
    over leaves hash_to_scalar(encode_elem(C_l), b"terkle/leaf").
    srs_pool: an Srs (all layers share it) or a mapping shape -> Srs.
    return_tree=True also returns the tree (for membership proofs): (commitments, root, tree)."""
    out = _prover_commit(tensors, srs_pool, tree_config, scale_bits, route, node_srs)
    return out if return_tree else out[:2]


def _prover_commit(tensors, srs_pool, tree_config, scale_bits, route, node_srs):
    tensors = list(tensors)
    if not tensors:
        raise ValueError("no tensors to commit")
    groups = {}
    for idx, T in enumerate(tensors):
        srs = srs_pool if not isinstance(srs_pool, dict) else None
        if srs is None:
            key = tuple(T.shape) if hasattr(T, "shape") else None
            srs = srs_pool.get(key)
            if srs is None:
                raise ValueError(f"no srs for tensor shape {key}")
        groups.setdefault(id(srs), (srs, []))[1].append(idx)
    cfg = tree_config or TreeConfig()
    if len(groups) == 1:
        srs = next(iter(groups.values()))[0]
        node = node_srs or authtree.node_srs(cfg, device=srs.device)
        if _device_tree_ok(tensors, srs, node):
            # commitments, leaf hashes and the whole tree on the device, one readback
            commitments, nodes, vals, depth = tc_commit_tree(srs, tensors, node, scale_bits=scale_bits, route=route)
            tree = authtree.tree_from_device(cfg, len(tensors), depth, nodes, vals, node)
            return commitments, tree.root, tree
    commitments = [None] * len(tensors)
    for srs, idxs in groups.values():
        cs = tc_commit_many(srs, [tensors[i] for i in idxs], scale_bits=scale_bits, route=route)
        for i, c in zip(idxs, cs):
            commitments[i] = c
    tree, root = build(cfg, [leaf_of(c) for c in commitments], srs=node_srs)
    return commitments, root, tree


def prover_commit_pipeline(forwards, srs, *, tree_config: TreeConfig = None, node_srs=None,
                           scale_bits: int = SCALE_BITS, route: str = "auto", depth: int = 2):
    """prover_commit over a stream of forwards (each a list of same-shape tensors: CUDA, or
    CPU floats uploaded on the fly), yielding (commitments, root, tree) per forward in order.
    `depth` device contexts (own streams and scratch, shared SRS) take the forwards in turn,
    so forward k+1's sort and accumulation overlap forward k's latency-bound tail (bucket
    weighting, affine conversion, tree) and its host-side decoding."""
    cfg = tree_config or TreeConfig()
    node = node_srs or authtree.node_srs(cfg, device=srs.device)
    if node.size > 64 or not node.has(_lib.SRS_LAGRANGE):
        for fwd in forwards:   # no device tree: the plain per-forward path
            yield prover_commit(list(fwd), srs, tree_config=cfg, scale_bits=scale_bits, route=route,
                                node_srs=node_srs, return_tree=True)
        return
    ctxs = [_lib.Context.pipeline(srs.device, k) for k in range(max(1, depth))]
    pending = []
    try:
        for k, fwd in enumerate(forwards):
            state = tc_commit_tree_launch(ctxs[k % len(ctxs)], srs, list(fwd), node, scale_bits=scale_bits,
                                          route=route)
            pending.append(state)
            if len(pending) == len(ctxs):
                yield _finish_tree(pending.pop(0), cfg, node)
        while pending:
            yield _finish_tree(pending.pop(0), cfg, node)
    finally:
        # an error or an early exit leaves launches in flight: collect them so their
        # contexts can be launched on again
        for state in pending:
            try:
                tc_commit_tree_finish(state)
            except Exception:
                pass


def _finish_tree(state, cfg, node):
    commitments, nodes, vals, depth = tc_commit_tree_finish(state)
    tree = authtree.tree_from_device(cfg, len(commitments), depth, nodes, vals, node)
    return commitments, tree.root, tree


def prover_commit_stream(batches, srs, *, tree_config: TreeConfig = None, node_srs=None,
                         scale_bits: int = SCALE_BITS, route: str = "auto"):
    """prover_commit over a stream of forwards (an iterable of per-forward lists of HOST
    tensors sharing one SRS): yields (commitments, root, tree) per forward.  The upload of
    forward k+1's activations overlaps the commitments of forward k (tc_commit_stream)."""
    cfg = tree_config or TreeConfig()
    it = iter(batches)
    try:
        cur = list(next(it))
    except StopIteration:
        return
    try:
        yield from _stream_forwards(it, cur, srs, cfg, node_srs, scale_bits, route)
    finally:
        # a consumer that stops early (or an error) leaves the last prefetch pending: drop
        # it, so a later stream whose buffers reuse these host addresses uploads afresh
        ctx = _lib.Context.get(srs.device)
        with ctx.lock:
            _lib.lib().tc_commit_stream_reset(ctx.handle)


def _stream_forwards(it, cur, srs, cfg, node_srs, scale_bits, route):
    while cur is not None:
        try:
            nxt = list(next(it))
        except StopIteration:
            nxt = None
        node = node_srs or authtree.node_srs(cfg, device=srs.device)
        if node.size <= 64 and node.has(_lib.SRS_LAGRANGE):
            # commitments, leaf hashes and the tree on the device, one readback per forward
            commitments, nodes, vals, depth = tc_commit_stream_tree(srs, cur, nxt, node, scale_bits=scale_bits,
                                                                    route=route)
            tree = authtree.tree_from_device(cfg, len(commitments), depth, nodes, vals, node)
            yield commitments, tree.root, tree
        else:
            commitments = tc_commit_stream(srs, cur, nxt, scale_bits=scale_bits, route=route)
            tree, root = build(cfg, [leaf_of(c) for c in commitments], srs=node)
            yield commitments, root, tree
        cur = nxt
