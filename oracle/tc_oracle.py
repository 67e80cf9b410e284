"""CPU ORACLE for the TensorCommitments prover path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The shipped package
(``paper_2602_12630_b200``) must never call into it.

It restates, in plain CPython big-int arithmetic, the reference algorithm of
the prover hot path (``/root/reference/pkg/src/tensorcommit``):

* scalar field F_p                      — field.py:13-61 (PrimeField)
* curve group over F_q                  — backend.py:102-348 (PairingBackend)
* lexicographic layout / interpolation  — mvpoly.py:27-247
* evaluation, division, open_quotients  — mvpoly.py:140-161, 452-534
* barycentric evaluation                — mvpoly.py:313-371
* the spec-only entry points            — SPEC.md:53-61 (setup_srs),
  276-304 (tc_commit/tc_open/tc_verify), 348-376 (Terkle build/prove/verify),
  536-554 (quantize, prover_commit)

Parity pinning: every primitive here is checked against the reference
imported from ``/root/reference/pkg/src`` (tests/test_oracle_vs_reference.py,
only when that tree exists) and against golden vectors generated from the
reference by ``tests/golden/make_golden.py`` (tests/test_oracle_golden.py,
runs everywhere).  The spec-only entry points are compositions of those
pinned primitives plus the conventions frozen in DESIGN.md ("Conventions"),
which the reference leaves open.
"""

from __future__ import annotations

import hashlib
import math
import struct

# ---------------------------------------------------------------------------
# constants — backend.py:102-108
# ---------------------------------------------------------------------------
P = (1 << 161) + (1 << 24) + 1          # subgroup order / scalar field (backend.py:103)
COFACTOR = 120                           # backend.py:104
Q = COFACTOR * P - 1                     # curve base field (backend.py:105)
GX = 251143519239308603259454152668007805633320126757058   # backend.py:106
GY = 36213243983195114554803697526372907779067409015054    # backend.py:107
G = (GX, GY)
SCALAR_BYTES = 21                        # backend.py:180
COORD_BYTES = 21                         # backend.py:181
ELEM_BYTES = 43                          # backend.py:182
MAX_COEFFS = 1 << 26                     # mvpoly.py:24
SCALE_BITS = 16


class BackendError(RuntimeError):
    """Mirror of backend.py:26-27."""


# ---------------------------------------------------------------------------
# F_p helpers — field.py:28-52
# ---------------------------------------------------------------------------
def fp_inv(a: int) -> int:
    """field.py:40-43: ZeroDivisionError on 0, else a^-1 mod p."""
    a %= P
    if a == 0:
        raise ZeroDivisionError("inverse of zero in prime field")
    return pow(a, P - 2, P)


def fp_rand(rng) -> int:
    """field.py:51-52 — PrimeField.rand(rng) = rng.randrange(p)."""
    return rng.randrange(P)


# ---------------------------------------------------------------------------
# curve arithmetic — backend.py:111-217
# Points are affine (x, y) int tuples, None = point at infinity.
# ---------------------------------------------------------------------------
def _dbl_jac(pt):
    """Jacobian doubling on y^2 = x^3 + x (a = 1); backend.py:111-123."""
    X, Y, Z = pt
    xx = X * X % Q
    yy = Y * Y % Q
    y4 = yy * yy % Q
    zz = Z * Z % Q
    s = 2 * ((X + yy) ** 2 - xx - y4) % Q
    mm = (3 * xx + zz * zz) % Q
    x3 = (mm * mm - 2 * s) % Q
    y3 = (mm * (s - x3) - 8 * y4) % Q
    z3 = ((Y + Z) ** 2 - yy - zz) % Q
    return (x3, y3, z3)


def _madd_jac(pt, xa, ya):
    """Jacobian + affine; None when the sum is infinity (backend.py:126-146)."""
    X, Y, Z = pt
    zz = Z * Z % Q
    u2 = xa * zz % Q
    s2 = ya * Z % Q * zz % Q
    h = (u2 - X) % Q
    r = 2 * (s2 - Y) % Q
    if h == 0:
        return _dbl_jac(pt) if r == 0 else None
    hh = h * h % Q
    i4 = 4 * hh % Q
    j = h * i4 % Q
    v = X * i4 % Q
    x3 = (r * r - j - 2 * v) % Q
    y3 = (r * (v - x3) - 2 * Y * j) % Q
    z3 = ((Z + h) ** 2 - zz - hh) % Q
    return (x3, y3, z3)


def _jac_affine(pt):
    """backend.py:149-155."""
    if pt is None:
        return None
    X, Y, Z = pt
    zi = pow(Z, Q - 2, Q)
    zi2 = zi * zi % Q
    return (X * zi2 % Q, Y * zi2 % Q * zi % Q)


def ec_add(a, b):
    """Affine group operation, PairingBackend.mul (backend.py:185-200)."""
    if a is None:
        return b
    if b is None:
        return a
    x1, y1 = a
    x2, y2 = b
    if x1 == x2:
        if (y1 + y2) % Q == 0:
            return None
        lam = (3 * x1 * x1 + 1) * pow(2 * y1, Q - 2, Q) % Q
    else:
        lam = (y2 - y1) * pow((x2 - x1) % Q, Q - 2, Q) % Q
    x3 = (lam * lam - x1 - x2) % Q
    return (x3, (lam * (x1 - x3) - y1) % Q)


def ec_neg(a):
    return None if a is None else (a[0], (-a[1]) % Q)


def ec_mul(base, k: int):
    """Scalar multiplication, PairingBackend.exp (backend.py:202-217):
    k reduced mod p, MSB-first double-and-add in Jacobian coordinates."""
    k %= P
    if base is None or k == 0:
        return None
    xa, ya = base
    acc = None
    for bit in bin(k)[2:]:
        if acc is not None:
            acc = _dbl_jac(acc)
        if bit == "1":
            acc = (xa, ya, 1) if acc is None else _madd_jac(acc, xa, ya)
    return _jac_affine(acc)


def on_curve(e) -> bool:
    """PairingBackend.validate_elem (backend.py:299-306)."""
    if e is None:
        return True
    x, y = e
    return 0 <= x < Q and 0 <= y < Q and (y * y - x * x * x - x) % Q == 0


# --- F_q2 = F_q[i]/(i^2+1) and the modified Tate pairing (backend.py:158-291)
def _f2mul(u, v):
    return ((u[0] * v[0] - u[1] * v[1]) % Q, (u[0] * v[1] + u[1] * v[0]) % Q)


def _f2sqr(u):
    return ((u[0] - u[1]) * (u[0] + u[1]) % Q, 2 * u[0] * u[1] % Q)


_LOOP_BITS = bin(P)[3:]  # backend.py:108


def pairing(S, T):
    """e(S, T) = t_p(S, phi(T)), phi(x, y) = (-x, i*y); backend.py:219-291.

    Miller loop over the bits of p below the MSB with the doubling and
    chord lines evaluated at phi(T), then the final exponentiation
    f -> (conj(f)/f)^120."""
    if S is None or T is None:
        return (1, 0)
    xq = (-T[0]) % Q
    yq = T[1]
    xp, yp = S
    f = (1, 0)
    X, Y, Z = xp, yp, 1
    for bit in _LOOP_BITS:
        xx = X * X % Q
        yy = Y * Y % Q
        y4 = yy * yy % Q
        zz = Z * Z % Q
        s = 2 * ((X + yy) ** 2 - xx - y4) % Q
        mm = (3 * xx + zz * zz) % Q
        line = ((-2 * yy - mm * (xq * zz - X)) % Q, 2 * Y * Z % Q * zz % Q * yq % Q)
        f = _f2mul(_f2sqr(f), line)
        x3 = (mm * mm - 2 * s) % Q
        y3 = (mm * (s - x3) - 8 * y4) % Q
        Z = ((Y + Z) ** 2 - yy - zz) % Q
        X, Y = x3, y3
        if bit == "1":
            zz = Z * Z % Q
            u2 = xp * zz % Q
            s2 = yp * Z % Q * zz % Q
            h = (u2 - X) % Q
            num = (s2 - Y) % Q
            if h == 0 and num == 0:
                raise BackendError("pairing argument of unexpected order")
            if h != 0:
                den = h * Z % Q
                line = ((-den * yp - num * (xq - xp)) % Q, den * yq % Q)
                f = _f2mul(f, line)
                hh = h * h % Q
                i4 = 4 * hh % Q
                j = h * i4 % Q
                v = X * i4 % Q
                r = 2 * num % Q
                x3 = (r * r - j - 2 * v) % Q
                y3 = (r * (v - x3) - 2 * Y * j) % Q
                Z = ((Z + h) ** 2 - zz - hh) % Q
                X, Y = x3, y3
            else:
                X, Y, Z = 0, 1, 0
    norm = (f[0] * f[0] + f[1] * f[1]) % Q
    ni = pow(norm, Q - 2, Q)
    finv = (f[0] * ni % Q, (-f[1]) * ni % Q)
    base = _f2mul((f[0], (-f[1]) % Q), finv)  # conj(f) / f
    out = (1, 0)
    e = COFACTOR
    while e:
        if e & 1:
            out = _f2mul(out, base)
        base = _f2sqr(base)
        e >>= 1
    return out


def target_mul(x, y):
    """backend.py:293-294."""
    return _f2mul(x, y)


# ---------------------------------------------------------------------------
# encodings and hash-to-field — backend.py:309-348
# ---------------------------------------------------------------------------
def encode_elem(e) -> bytes:
    if e is None:
        return bytes(ELEM_BYTES)
    return b"\x04" + e[0].to_bytes(COORD_BYTES, "little") + e[1].to_bytes(COORD_BYTES, "little")


def decode_elem(raw: bytes):
    if len(raw) != ELEM_BYTES:
        raise ValueError("bad element length")
    if raw[0] == 0:
        if any(raw[1:]):
            raise ValueError("bad infinity encoding")
        return None
    if raw[0] != 4:
        raise ValueError("bad point flag")
    pt = (int.from_bytes(raw[1:22], "little"), int.from_bytes(raw[22:], "little"))
    if not on_curve(pt):
        raise ValueError("point not on curve")
    return pt


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
    """backend.py:346-348."""
    d = hashlib.sha256(b"tc/h2f/" + tag + b"/" + data).digest()
    return int.from_bytes(d, "little") % P


# ---------------------------------------------------------------------------
# layout — mvpoly.py:27-133
# ---------------------------------------------------------------------------
def check_shape(shape) -> int:
    """mvpoly.py:27-38."""
    if len(shape) == 0:
        raise ValueError("shape needs at least one axis")
    n = 1
    for d in shape:
        if d < 1:
            raise ValueError(f"axis degree bound must be >= 1, got {d}")
        n *= d
    if n > MAX_COEFFS:
        raise ValueError(f"coefficient array of {n} entries exceeds limit")
    return n


def lex_strides(shape):
    """mvpoly.py:41-47 — last axis fastest."""
    out = []
    acc = 1
    for d in reversed(shape):
        out.append(acc)
        acc *= d
    return tuple(reversed(out))


def lex_index(idx, shape) -> int:
    """mvpoly.py:50-59."""
    if len(idx) != len(shape):
        raise ValueError("index arity does not match shape")
    off = 0
    for i, d in zip(idx, shape):
        if not 0 <= i < d:
            raise IndexError(f"index {idx} out of bounds for shape {shape}")
        off = off * d + i
    return off


def default_nodes(d: int):
    """default_grid axis nodes 1..d (mvpoly.py:130-133)."""
    return [r + 1 for r in range(d)]


def _fibers(shape, axis):
    """Yield (base, step) for every 1-D fiber along `axis` (mvpoly.py:168-186)."""
    strides = lex_strides(shape)
    step = strides[axis]
    d = shape[axis]
    outer = 1
    for j in range(axis):
        outer *= shape[j]
    for o in range(outer):
        for i in range(step):
            yield o * d * step + i, step


# ---------------------------------------------------------------------------
# interpolation — mvpoly.py:193-247
# ---------------------------------------------------------------------------
def lagrange_matrix(nodes):
    """Column l = monomial coefficients of the l-th Lagrange basis polynomial
    (master polynomial / (X - z_l) scaled by 1/prod_{r!=l}(z_l - z_r));
    mvpoly.py:193-218.  Returned as rows[l][k]."""
    d = len(nodes)
    master = [1]
    for z in nodes:
        nxt = [0] * (len(master) + 1)
        for k, c in enumerate(master):
            nxt[k + 1] = (nxt[k + 1] + c) % P
            nxt[k] = (nxt[k] - c * z) % P
        master = nxt
    rows = []
    for l, z in enumerate(nodes):
        quo = [0] * d
        carry = master[d]
        for k in range(d - 1, -1, -1):
            quo[k] = carry
            carry = (master[k] + carry * z) % P
        w = 1
        for r, zr in enumerate(nodes):
            if r != l:
                w = w * (z - zr) % P
        wi = fp_inv(w)
        rows.append([c * wi % P for c in quo])
    return rows


def interpolate_lagrange(values, shape, axes_nodes=None):
    """mvpoly.py:233-247: per-axis sample->coefficient transform, axis 0 first.
    Returns the flat lex coefficient list."""
    n = check_shape(shape)
    flat = [v % P for v in values]
    if len(flat) != n:
        raise ValueError("tensor size does not match grid shape")
    for axis, d in enumerate(shape):
        nodes = axes_nodes[axis] if axes_nodes else default_nodes(d)
        rows = lagrange_matrix(nodes)
        for base, step in _fibers(shape, axis):
            fib = flat[base: base + d * step: step]
            out = [0] * d
            for l, v in enumerate(fib):
                if v:
                    row = rows[l]
                    for k in range(d):
                        out[k] += v * row[k]
            flat[base: base + d * step: step] = [c % P for c in out]
    return flat


def evaluate(coeffs, shape, point) -> int:
    """Nested Horner of the monomial form, mvpoly.py:140-161."""
    if len(point) != len(shape):
        raise ValueError("evaluation point arity does not match polynomial")
    cur = list(coeffs)
    # contract the last axis first (same value as the reference's recursion)
    for axis in range(len(shape) - 1, -1, -1):
        d = shape[axis]
        x = point[axis] % P
        nxt = []
        for b in range(len(cur) // d):
            acc = 0
            for k in range(d - 1, -1, -1):
                acc = (acc * x + cur[b * d + k]) % P
            nxt.append(acc)
        cur = nxt
    return cur[0]


def divide_by_linear(coeffs, shape, axis, v):
    """f = q*(X_axis - v) + r, q and r keep f's shape; mvpoly.py:452-484."""
    n = len(coeffs)
    qc = [0] * n
    rc = list(coeffs)
    d = shape[axis]
    if d > 1:
        for base, step in _fibers(shape, axis):
            carry = rc[base + (d - 1) * step]
            rc[base + (d - 1) * step] = 0
            for c in range(d - 2, -1, -1):
                pos = base + c * step
                qc[pos] = carry
                carry = (rc[pos] + v * carry) % P
                rc[pos] = 0
            rc[base] = carry
    return qc, rc


def open_quotients(coeffs, shape, point):
    """mvpoly.py:521-534: peel one variable at a time; returns (q_list, y)."""
    if len(point) != len(shape):
        raise ValueError("point arity does not match polynomial")
    qs = []
    rem = list(coeffs)
    for axis, w in enumerate(point):
        q, rem = divide_by_linear(rem, shape, axis, w % P)
        qs.append(q)
    return qs, rem[0]


def multiply_by_linear(coeffs, shape, axis, v):
    """q * (X_axis - v) (mvpoly.py:487-518), for the division identity."""
    out = [0] * len(coeffs)
    d = shape[axis]
    for base, step in _fibers(shape, axis):
        if coeffs[base + (d - 1) * step] % P:
            raise ValueError("product would overflow the degree bound")
        for c in range(d - 1):
            pos = base + c * step
            fc = coeffs[pos]
            out[pos + step] = (out[pos + step] + fc) % P
            out[pos] = (out[pos] - fc * v) % P
    return out


def barycentric_weights(nodes):
    """mvpoly.py:313-323."""
    ws = []
    for l, z in enumerate(nodes):
        w = 1
        for r, zr in enumerate(nodes):
            if r != l:
                w = w * (z - zr) % P
        ws.append(fp_inv(w))
    return ws


def lagrange_at(nodes, x):
    """Normalised barycentric factors L_l(x) for one axis (mvpoly.py:326-337)."""
    x %= P
    for l, z in enumerate(nodes):
        if x == z % P:
            return [1 if r == l else 0 for r in range(len(nodes))]
    ws = barycentric_weights(nodes)
    terms = [ws[l] * fp_inv(x - z) % P for l, z in enumerate(nodes)]
    tinv = fp_inv(sum(terms) % P)
    return [t * tinv % P for t in terms]


def contract_leading(values, shape, factors):
    """Contract the leading axis of a lex tensor against per-node factors."""
    d = shape[0]
    block = len(values) // d
    out = [0] * block
    for l in range(d):
        f = factors[l]
        if f:
            seg = values[l * block:(l + 1) * block]
            for b in range(block):
                out[b] += f * seg[b]
    return [v % P for v in out]


def barycentric_eval(values, shape, point, axes_nodes=None):
    """mvpoly.py:340-371: evaluate the interpolant at `point` by contracting
    the leading axis repeatedly, without forming coefficients."""
    if len(point) != len(shape):
        raise ValueError("evaluation point arity does not match grid")
    flat = [v % P for v in values]
    if len(flat) != check_shape(shape):
        raise ValueError("tensor size does not match grid shape")
    for j in range(len(shape)):
        nodes = axes_nodes[j] if axes_nodes else default_nodes(shape[j])
        flat = contract_leading(flat, shape[j:], lagrange_at(nodes, point[j]))
    return flat[0]


def barycentric_eval_small(q, shape, point, axes_nodes=None):
    """barycentric_eval for a tensor of SMALL signed integers (numpy int64, |q| < 2^30, e.g.
    quantised fp16 activations): the first contraction (the leading axis, all but N/d_0 of
    the work) runs exactly in numpy over 24-bit limbs of the Lagrange factors — each limb
    sum stays below 2^63 — and the remaining axes as in barycentric_eval.  Same value as
    barycentric_eval(q mod p, ...); test-only speed-up for full-size configs."""
    import numpy as np

    q = np.asarray(q, dtype=np.int64).reshape(-1)
    n = check_shape(shape)
    if q.size != n:
        raise ValueError("tensor size does not match grid shape")
    if len(point) != len(shape):
        raise ValueError("evaluation point arity does not match grid")
    if q.size and int(np.abs(q).max()) >= 1 << 30:
        raise ValueError("barycentric_eval_small needs |q| < 2^30")
    d0 = shape[0]
    nodes = axes_nodes[0] if axes_nodes else default_nodes(d0)
    fac = lagrange_at(nodes, point[0])
    LB, NL = 24, 7                                        # 7 x 24 bits >= 162
    limbs = np.array([[(f >> (LB * k)) & ((1 << LB) - 1) for f in fac] for k in range(NL)], dtype=np.int64)
    acc = limbs @ q.reshape(d0, n // d0)                  # (NL, N/d0), |entries| < 2^24 2^30 2^7
    rows = [r.tolist() for r in acc]
    flat = [sum(rows[k][b] << (LB * k) for k in range(NL)) % P for b in range(n // d0)]
    for j in range(1, len(shape)):
        nj = axes_nodes[j] if axes_nodes else default_nodes(shape[j])
        flat = contract_leading(flat, shape[j:], lagrange_at(nj, point[j]))
    return flat[0]


def quantize_signed(values, scale_bits: int = SCALE_BITS):
    """quantize() as signed int64 (numpy) for inputs whose |v| 2^scale_bits < 2^62."""
    import numpy as np

    flat = np.asarray(values).reshape(-1).astype(np.float64)
    if not np.all(np.isfinite(flat)):
        raise ValueError("quantize: non-finite value")
    scaled = np.ldexp(flat, scale_bits)
    if not np.all(np.abs(scaled) < 2.0 ** 62):
        raise ValueError("quantize_signed: magnitude too large for int64")
    return np.rint(scaled).astype(np.int64)


# ---------------------------------------------------------------------------
# quantize — SPEC.md:536-544, 605
# ---------------------------------------------------------------------------
def quantize(values, scale_bits: int = SCALE_BITS):
    """q = round-half-even(v * 2^scale_bits); negatives map to p - |q|;
    ValueError when |v| * 2^scale_bits >= p/2 or v is not finite
    (SPEC.md:536-544).  Works on the exact binary value of each input:
    fp16/fp32 inputs widen to float64 exactly and v * 2^k stays exact."""
    import numpy as np
    from fractions import Fraction

    arr = np.asarray(values)
    if arr.dtype.kind != "f":
        arr = arr.astype(np.float64)
    flat = arr.reshape(-1).astype(np.float64)
    if not np.all(np.isfinite(flat)):
        raise ValueError("quantize: non-finite value")
    scaled = np.ldexp(flat, scale_bits)
    if np.all(np.abs(scaled) < 2.0 ** 62):
        q = np.rint(scaled).astype(np.int64)          # rint = round half to even
        return [int(v) % P for v in q.tolist()]
    out = []
    for v in flat.tolist():
        x = Fraction(v) * (1 << scale_bits)
        if 2 * abs(x) >= P:
            raise ValueError("quantize: value overflows the field half-range")
        out.append(round(x) % P)                      # Fraction.__round__ is half-even
    return out


def signed_of(v: int) -> int:
    """Field element -> centred signed integer in (-p/2, p/2]."""
    v %= P
    return v - P if v > P // 2 else v


# ---------------------------------------------------------------------------
# SRS — SPEC.md:44-61, 81, 87 (conventions frozen in DESIGN.md)
# ---------------------------------------------------------------------------
def shape_header(magic: bytes, shape) -> bytes:
    """Wire header magic ‖ <HH version=1, m> ‖ <I d_j>×m (mvpoly.py:567-572)."""
    return magic + struct.pack("<HH", 1, len(shape)) + b"".join(struct.pack("<I", d) for d in shape)


def derive_taus(shape, entropy: bytes):
    """Frozen convention (SPEC.md:81 asks only for a PRF on the entropy):
    tau_j = hash_to_scalar(entropy ‖ u32le(j) ‖ TCSR shape header, b"srs/tau")."""
    hdr = shape_header(b"TCSR", shape)
    return [hash_to_scalar(entropy + struct.pack("<I", j) + hdr, b"srs/tau") for j in range(len(shape))]


def monomial_exponents(shape, taus):
    """prod_j tau_j^{i_j} for every multi-index in lex order."""
    flat = [1]
    for d, t in zip(shape, taus):
        pw = [pow(t, e, P) for e in range(d)]
        flat = [a * b % P for a in flat for b in pw]
    return flat


def lagrange_exponents(shape, taus, axes_nodes=None):
    """prod_j L_{j,i_j}(tau_j) for every grid index in lex order."""
    flat = [1]
    for j, (d, t) in enumerate(zip(shape, taus)):
        nodes = axes_nodes[j] if axes_nodes else default_nodes(d)
        lj = lagrange_at(nodes, t)
        flat = [a * b % P for a in flat for b in lj]
    return flat


def setup_srs(shape, entropy: bytes):
    """Returns (monomial_elems, axis_elems, taus): G_i = g^{prod tau_j^{i_j}}
    (SPEC.md:44-50); axis_elems[j] = g^{tau_j}."""
    check_shape(shape)
    taus = derive_taus(shape, entropy)
    elems = [ec_mul(G, e) for e in monomial_exponents(shape, taus)]
    axis = [ec_mul(G, t) for t in taus]
    return elems, axis, taus


# ---------------------------------------------------------------------------
# commitment scheme — SPEC.md:276-304
# ---------------------------------------------------------------------------
def msm_naive(scalars, bases):
    """prod_k bases_k^{a_k} as the reference composes it: fold `mul` over
    `exp` terms (backend.py:185-217; SPEC.md:279, 315 'naive' strategy)."""
    acc = None
    for a, b in zip(scalars, bases):
        if a % P:
            acc = ec_add(acc, ec_mul(b, a))
    return acc


def tc_commit(srs_elems, values, shape):
    """C_T = MSM(srs, interpolate_lagrange(T))."""
    coeffs = interpolate_lagrange(values, shape)
    return msm_naive(coeffs, srs_elems)


def tc_open(srs_elems, values, shape, point):
    """(y, [pi_1..pi_m]) with pi_i = MSM(srs, q_i)."""
    coeffs = interpolate_lagrange(values, shape)
    qs, y = open_quotients(coeffs, shape, point)
    return y, [msm_naive(q, srs_elems) for q in qs]


def tc_verify(axis_elems, commitment, point, y, proofs) -> bool:
    """Product-of-pairings check:
    e(C * g^-y, g) == prod_i e(pi_i, axis_i * g^-w_i)."""
    if len(proofs) != len(axis_elems) or len(point) != len(axis_elems):
        raise ValueError("proof count does not match tensor order")
    lhs = pairing(ec_add(commitment, ec_mul(G, (-y) % P)), G)
    rhs = (1, 0)
    for pi, ax, w in zip(proofs, axis_elems, point):
        rhs = target_mul(rhs, pairing(pi, ec_add(ax, ec_mul(G, (-w) % P))))
    return lhs == rhs


# --- trapdoor oracles: O(N) field work instead of an MSM
def commit_trapdoor(values, shape, taus):
    """g^{f_T(tau)} via barycentric evaluation (mvpoly.py:340-371)."""
    return ec_mul(G, barycentric_eval(values, shape, taus))


def open_trapdoor(values, shape, taus, point):
    """pi_i = g^{q_i(tau)}: r_{i-1}(X) = f(w_<i, X_>=i), so
    q_i(tau) = (f(w_<i, tau_>=i) - f(w_<=i, tau_>i)) / (tau_i - w_i)."""
    m = len(shape)
    ev = []
    for i in range(m + 1):
        pt = [point[j] if j < i else taus[j] for j in range(m)]
        ev.append(barycentric_eval(values, shape, pt))
    y = ev[m]
    proofs = []
    for i in range(m):
        num = (ev[i] - ev[i + 1]) % P
        proofs.append(ec_mul(G, num * fp_inv(taus[i] - point[i]) % P))
    return y, proofs


# ---------------------------------------------------------------------------
# Terkle trees — SPEC.md:335-376, 394-397
# ---------------------------------------------------------------------------
LEAF_TAG = b"terkle/leaf"
NODE_TAG = b"terkle/node"


def terkle_depth(n: int, arity: int) -> int:
    """L = max(1, ceil(log_B n)) node levels."""
    if n < 1:
        raise ValueError("empty leaf list")
    L, cap = 1, arity
    while cap < n:
        cap *= arity
        L += 1
    return L


def terkle_build(leaves, node_shape, commit_fn):
    """Bottom-up: pad leaves with 0 to B^L; every node commits to its B
    children as a node_shape tensor; a node's parent entry is
    hash_to_scalar(encode_elem(C_u), b"terkle/node").

    commit_fn(values) -> point.  Returns levels: list (bottom first) of
    lists of node commitments, and the per-level child-value lists."""
    B = check_shape(node_shape)
    L = terkle_depth(len(leaves), B)
    vals = [v % P for v in leaves] + [0] * (B ** L - len(leaves))
    levels, values = [], []
    for _ in range(L):
        values.append(vals)
        nodes = [commit_fn(vals[k * B:(k + 1) * B]) for k in range(len(vals) // B)]
        levels.append(nodes)
        vals = [hash_to_scalar(encode_elem(c), NODE_TAG) for c in nodes]
    return levels, values


def terkle_child_point(pos: int, node_shape):
    """Child slot -> grid point (kappa + 1 on the default grid)."""
    idx = []
    for d in reversed(node_shape):
        idx.append(pos % d + 1)
        pos //= d
    return list(reversed(idx))


def terkle_verify(root, i: int, leaf: int, nodes, openings, node_shape, axis_elems) -> bool:
    """Membership check: for every level (bottom first) the opening
    (y, proofs) of the node at its child's grid point verifies (tc_verify, product of
    pairings) and opens the expected child value; the next expected value is the node's
    hash; the top node is the root."""
    B = check_shape(node_shape)
    expected = leaf % P
    pos = i
    for node, (y, proofs) in zip(nodes, openings):
        u, slot = divmod(pos, B)
        if y != expected:
            return False
        if not tc_verify(axis_elems, node, terkle_child_point(slot, node_shape), y, list(proofs)):
            return False
        expected = hash_to_scalar(encode_elem(node), NODE_TAG)
        pos = u
    return pos == 0 and len(nodes) > 0 and nodes[-1] == root


def leaf_of_commitment(c) -> int:
    """Per-layer commitment -> tree leaf."""
    return hash_to_scalar(encode_elem(c), LEAF_TAG)
