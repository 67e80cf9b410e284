"""Scalar domain object with the reference's duck-typed `dom` protocol (field.py:1-8).

Host-side only (Python ints): the device engine works on limbs; this class exists so
callers can keep passing a `dom` exactly as they do with tensorcommit.field.PrimeField.
"""
from __future__ import annotations

from .curve import P


class PrimeField:
    __slots__ = ("p", "zero", "one")

    def __init__(self, p: int = P):
        if p < 2:
            raise ValueError("field order must be at least 2")
        self.p = p
        self.zero = 0
        self.one = 1 % p

    def from_int(self, n) -> int:
        return int(n) % self.p

    def add(self, a, b):
        return (a + b) % self.p

    def sub(self, a, b):
        return (a - b) % self.p

    def mul(self, a, b):
        return a * b % self.p

    def neg(self, a):
        return -a % self.p

    def inv(self, a):
        if a % self.p == 0:
            raise ZeroDivisionError("inverse of zero in prime field")
        return pow(a, self.p - 2, self.p)

    def div(self, a, b):
        return a * self.inv(b) % self.p

    def is_zero(self, a) -> bool:
        return a % self.p == 0

    def rand(self, rng) -> int:
        return rng.randrange(self.p)

    def __eq__(self, other):
        return isinstance(other, PrimeField) and other.p == self.p

    def __hash__(self):
        return hash(("PrimeField", self.p))

    def __repr__(self):
        return f"PrimeField(0x{self.p:x})"
