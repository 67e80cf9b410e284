"""Terkle trees with node commitments on the GPU.

A node gathers its B = prod(d) children as a tensor Z_u of shape d and stores
C_u = tc_commit(Z_u); a child node enters its parent as
hash_to_scalar(encode_elem(C_child), b"terkle/node").  Leaves are padded
with field zero to B^L, L = max(1, ceil(log_B n)).
Membership proofs open each node on the path at its child's grid point kappa + 1
(default grid, nodes 1..d) and carry the node commitments below the root.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

from . import _lib
from .commit import Commitment, Srs, TensorOpening, setup_srs, tc_open, tc_verify
from .curve import ELEM_BYTES, P, decode_elem, encode_elem, encode_scalar, hash_to_scalar
from .mvpoly import check_shape

NODE_TAG = b"terkle/node"
LEAF_TAG = b"terkle/leaf"
DEFAULT_NODE_SHAPE = (2, 2, 2)


@dataclass(frozen=True)
class TreeConfig:
    """SPEC.md:335-338 (terkle kind only: Merkle / Verkle are out of scope)."""
    kind: str = "terkle"
    shape: tuple = DEFAULT_NODE_SHAPE

    def __post_init__(self):
        if self.kind != "terkle":
            raise ValueError("only kind='terkle' is provided by the B200 prover")
        if check_shape(self.shape) < 2:
            raise ValueError("tree arity must be >= 2")

    @property
    def arity(self) -> int:
        return check_shape(self.shape)


class TerkleTree:
    """A built tree: levels[l][u] = node commitment point (bottom level first), values[l] =
    the child values of level l (flat, lex per node); n = true leaf count (root metadata,
    SPEC.md:395).  A tree read back from the device keeps the raw encodings and decodes
    levels / values on first use (prove); the root alone is decoded eagerly-cheaply."""

    def __init__(self, config: TreeConfig, n: int, depth: int, levels=None, values=None, srs: Srs = None,
                 raw=None):
        self.config, self.n, self.depth, self.srs = config, n, depth, srs
        self._levels, self._values, self._raw = levels, values, raw
        # node openings already computed: (level, node, slot) -> TensorOpening.  prove() is a
        # pure function of the (immutable) tree, so repeated challenges reuse them
        self._openings = {}

    def _decode(self):
        nodes_raw, values_raw = self._raw
        B = self.config.arity
        levels, values, pos, vpos = [], [], 0, 0
        for l in range(self.depth):
            k = B ** (self.depth - 1 - l)
            levels.append([decode_elem(nodes_raw[(pos + u) * ELEM_BYTES:(pos + u + 1) * ELEM_BYTES], validate=False)
                           for u in range(k)])
            pos += k
            w = B ** (self.depth - l)
            values.append([int.from_bytes(values_raw[24 * (vpos + j):24 * (vpos + j + 1)], "little")
                           for j in range(w)])
            vpos += w
        self._levels, self._values = levels, values

    @property
    def levels(self):
        if self._levels is None:
            self._decode()
        return self._levels

    @property
    def values(self):
        if self._values is None:
            self._decode()
        return self._values

    @property
    def root(self) -> Commitment:
        if self._levels is None:   # the top node is the last encoding of the bottom-first list
            nodes_raw = self._raw[0]
            B = self.config.arity
            total = sum(B ** (self.depth - 1 - l) for l in range(self.depth))
            return Commitment(decode_elem(nodes_raw[(total - 1) * ELEM_BYTES:total * ELEM_BYTES], validate=False))
        return Commitment(self.levels[-1][0])

    def __repr__(self):
        return f"TerkleTree(config={self.config}, n={self.n}, depth={self.depth})"


@dataclass(frozen=True)
class MembershipProof:
    """Per level (bottom first): the node commitment and its opening at the child's point."""
    index: int
    nodes: tuple
    openings: tuple

    def to_bytes(self, config: "TreeConfig") -> bytes:
        """TCTP wire format: magic, kind byte (2 = terkle), depth u16, leaf
        index u64, then per level a length-prefixed payload: node point ‖ TCOP opening."""
        out = [b"TCTP", bytes([2]), struct.pack("<HQ", len(self.nodes), self.index)]
        for lvl, (node, op) in enumerate(zip(self.nodes, self.openings)):
            slot = (self.index // config.arity ** lvl) % config.arity
            payload = encode_elem(node) + op.to_bytes(child_point(slot, config.shape))
            out.append(struct.pack("<I", len(payload)) + payload)
        return b"".join(out)

    @staticmethod
    def from_bytes(raw: bytes) -> "MembershipProof":
        raw = bytes(raw)
        if raw[:4] != b"TCTP" or len(raw) < 15 or raw[4] != 2:
            raise ValueError("bad terkle proof header")
        depth, index = struct.unpack_from("<HQ", raw, 5)
        off, nodes, ops = 15, [], []
        for _ in range(depth):
            if off + 4 > len(raw):
                raise ValueError("truncated terkle proof")
            (ln,) = struct.unpack_from("<I", raw, off)
            off += 4
            payload = raw[off: off + ln]
            if len(payload) != ln or ln < ELEM_BYTES:
                raise ValueError("truncated terkle proof")
            nodes.append(decode_elem(payload[:ELEM_BYTES]))
            ops.append(TensorOpening.from_bytes(payload[ELEM_BYTES:])[1])
            off += ln
        if off != len(raw):
            raise ValueError("trailing bytes in terkle proof")
        return MembershipProof(index, tuple(nodes), tuple(ops))


_NODE_SRS = {}


def node_srs(config: TreeConfig, entropy: bytes = b"tc-b200/terkle", device=None) -> Srs:
    key = (config.shape, entropy, device)
    if key not in _NODE_SRS:
        _NODE_SRS[key] = setup_srs(config.shape, entropy, device=device)[0]
    return _NODE_SRS[key]


def tree_depth(n: int, arity: int) -> int:
    if n < 1:
        raise ValueError("empty leaf list")
    L, cap = 1, arity
    while cap < n:
        cap *= arity
        L += 1
    return L


def child_point(slot: int, shape):
    """Flat child slot -> grid point kappa + 1 (lex, last axis fastest)."""
    pt = []
    for d in reversed(shape):
        pt.append(slot % d + 1)
        slot //= d
    return tuple(reversed(pt))


def build(config: TreeConfig, leaves, *, srs: Srs = None):
    """(tree, root commitment) for field-element leaves."""
    leaves = [int(v) % P for v in leaves]
    if not leaves:
        raise ValueError("empty leaf list")
    srs = srs or node_srs(config)
    B = config.arity
    L = tree_depth(len(leaves), B)
    total_nodes = sum(B ** (L - 1 - l) for l in range(L))
    ctx = _lib.Context.get(srs.device)
    out = C.create_string_buffer(total_nodes * ELEM_BYTES)
    cnt = C.c_uint64(total_nodes)
    with ctx.lock:
        ctx.bind_stream()
        ctx.check(_lib.lib().tc_terkle_build(ctx.handle, srs.handle, b"".join(encode_scalar(v) for v in leaves),
                                             len(leaves), out, C.byref(cnt)), "terkle build")
    raw = out.raw
    levels, values, pos = [], [], 0
    vals = leaves + [0] * (B ** L - len(leaves))
    for l in range(L):
        k = B ** (L - 1 - l)
        nodes = [decode_elem(raw[(pos + u) * ELEM_BYTES:(pos + u + 1) * ELEM_BYTES], validate=False) for u in range(k)]
        pos += k
        levels.append(nodes)
        values.append(vals)
        vals = [hash_to_scalar(encode_elem(c), NODE_TAG) for c in nodes]
    tree = TerkleTree(config, len(leaves), L, levels, values, srs)
    return tree, tree.root


def tree_from_device(config: TreeConfig, n: int, depth: int, nodes_raw: bytes, values_raw: bytes,
                     srs: Srs) -> TerkleTree:
    """The TerkleTree of tc_commit_tree's outputs (node encodings level by level, every
    level's child values as 24-byte LE limbs) — the same object `build` returns, decoded
    lazily (a forward's readback costs the host ~100 us of Python decoding otherwise)."""
    return TerkleTree(config, n, depth, srs=srs, raw=(bytes(nodes_raw), bytes(values_raw)))


def prove(tree: TerkleTree, i: int) -> MembershipProof:
    """L openings, one per level."""
    if not 0 <= i < tree.n:
        raise IndexError(f"leaf index {i} out of range")
    B = tree.config.arity
    nodes, openings = [], []
    pos = i
    for l in range(tree.depth):
        u, slot = divmod(pos, B)
        op = tree._openings.get((l, u, slot))
        if op is None:
            Z = tree.values[l][u * B:(u + 1) * B]
            op = tree._openings[(l, u, slot)] = tc_open(tree.srs, Z, child_point(slot, tree.config.shape))
        nodes.append(tree.levels[l][u])
        openings.append(op)
        pos = u
    return MembershipProof(i, tuple(nodes), tuple(openings))


def prove_many(tree: TerkleTree, indices) -> list:
    """prove() for many leaves: the node openings none of them has memoised yet are computed
    together (one tc_open_many call: for the tiny node SRS, every quotient MSM in one
    table-kernel launch), then each proof is assembled as prove() does."""
    from .commit import tc_open_many

    B = tree.config.arity
    need = {}
    for i in indices:
        if not 0 <= i < tree.n:
            raise IndexError(f"leaf index {i} out of range")
        pos = i
        for l in range(tree.depth):
            u, slot = divmod(pos, B)
            if (l, u, slot) not in tree._openings:
                need[(l, u, slot)] = None
            pos = u
    if need:
        keys = list(need)
        zs = [tree.values[l][u * B:(u + 1) * B] for l, u, _ in keys]
        pts = [child_point(slot, tree.config.shape) for _, _, slot in keys]
        for key, op in zip(keys, tc_open_many(tree.srs, zs, pts)):
            tree._openings[key] = op
    return [prove(tree, i) for i in indices]


def verify(root, i: int, leaf: int, proof: MembershipProof, config: TreeConfig, *, srs: Srs = None) -> bool:
    """Every level's opening verifies, opens the expected child value, and the top node
    is the root."""
    srs = srs or node_srs(config)
    root_elem = root.elem if isinstance(root, Commitment) else root
    B = config.arity
    if len(proof.nodes) != len(proof.openings) or not proof.nodes:
        raise ValueError("malformed proof")
    if proof.index != i:
        return False
    expected = int(leaf) % P
    pos = i
    for node, op in zip(proof.nodes, proof.openings):
        u, slot = divmod(pos, B)
        if not isinstance(op, TensorOpening) or len(op.proofs) != len(config.shape):
            raise ValueError("malformed proof")
        if op.y != expected:
            return False
        if not tc_verify(srs, Commitment(node), child_point(slot, config.shape), op):
            return False
        expected = hash_to_scalar(encode_elem(node), NODE_TAG)
        pos = u
    return pos == 0 and proof.nodes[-1] == root_elem


def leaf_of(c) -> int:
    """Per-layer commitment -> Terkle leaf."""
    elem = c.elem if isinstance(c, Commitment) else c
    return hash_to_scalar(encode_elem(elem), LEAF_TAG)
