"""Host-side constants and canonical encodings of the production curve.

Everything here is O(1)-per-element byte plumbing around the C ABI; the group and
field arithmetic itself runs in libtcb200.so.  Layouts follow the reference exactly:
encode_elem / decode_elem (backend.py:309-333), encode_scalar / decode_scalar
(backend.py:335-344), hash_to_scalar (backend.py:346-348), constants
(backend.py:102-108).
"""
from __future__ import annotations

import hashlib

P = (1 << 161) + (1 << 24) + 1      # scalar field / subgroup order
Q = 120 * P - 1                     # base field of E: y^2 = x^3 + x
G = (251143519239308603259454152668007805633320126757058,
     36213243983195114554803697526372907779067409015054)
SCALAR_BYTES = 21
COORD_BYTES = 21
ELEM_BYTES = 43
IDENTITY = None


def on_curve(e) -> bool:
    if e is None:
        return True
    x, y = e
    return 0 <= x < Q and 0 <= y < Q and (y * y - x * x * x - x) % Q == 0


def encode_elem(e) -> bytes:
    if e is None:
        return bytes(ELEM_BYTES)
    x, y = e
    return b"\x04" + x.to_bytes(COORD_BYTES, "little") + y.to_bytes(COORD_BYTES, "little")


def decode_elem(raw: bytes, validate: bool = True):
    raw = bytes(raw)
    if len(raw) != ELEM_BYTES:
        raise ValueError("bad element length")
    if raw[0] == 0:
        if any(raw[1:]):
            raise ValueError("bad infinity encoding")
        return None
    if raw[0] != 4:
        raise ValueError("bad point flag")
    pt = (int.from_bytes(raw[1:1 + COORD_BYTES], "little"), int.from_bytes(raw[1 + COORD_BYTES:], "little"))
    if validate and not on_curve(pt):
        raise ValueError("point not on curve")
    return pt


def decode_elems(raw: bytes, count: int, validate: bool = False):
    return tuple(decode_elem(raw[i * ELEM_BYTES:(i + 1) * ELEM_BYTES], validate) for i in range(count))


def encode_scalar(s: int) -> bytes:
    return (s % P).to_bytes(SCALAR_BYTES, "little")


def decode_scalar(raw: bytes) -> int:
    if len(raw) != SCALAR_BYTES:
        raise ValueError("bad scalar length")
    v = int.from_bytes(raw, "little")
    if v >= P:
        raise ValueError("scalar out of range")
    return v


def hash_to_scalar(data: bytes, tag: bytes = b"") -> int:
    return int.from_bytes(hashlib.sha256(b"tc/h2f/" + tag + b"/" + data).digest(), "little") % P


def scalars_le21(values) -> bytes:
    return b"".join(encode_scalar(int(v)) for v in values)
