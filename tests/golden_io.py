"""Loaders for the committed golden vectors (tests/golden/*.json)."""
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def ints(xs):
    return [int(x, 16) for x in xs]


def elem(hexstr):
    from oracle import tc_oracle as O
    return O.decode_elem(bytes.fromhex(hexstr))
