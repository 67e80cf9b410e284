"""Generate golden vectors for the prover path FROM THE REFERENCE ITSELF.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
Writes tests/golden/*.json.  Everything here calls the reference's own
primitives (tensorcommit.field / backend / mvpoly); the spec-only entry
points (setup_srs, tc_commit, tc_open, tc_verify, Terkle) are composed from
those primitives exactly as SPEC.md describes them, with the conventions
frozen in DESIGN.md.  Nothing in this file is imported at test time.
"""
import json
import os
import random
import struct
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from tensorcommit import backend as B   # noqa: E402
from tensorcommit import field as F     # noqa: E402
from tensorcommit import mvpoly as M    # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
be = B.make_backend("production")
dom = F.PrimeField(be.order)
p = be.order


def hx(v):
    return hex(v)


def enc(e):
    return be.encode_elem(e).hex()


def shape_header(magic, shape):
    return magic + struct.pack("<HH", 1, len(shape)) + b"".join(struct.pack("<I", d) for d in shape)


def taus_for(shape, entropy):
    hdr = shape_header(b"TCSR", shape)
    return [be.hash_to_scalar(entropy + struct.pack("<I", j) + hdr, b"srs/tau") for j in range(len(shape))]


def monomial_srs(shape, taus):
    exps = [1]
    for d, t in zip(shape, taus):
        pw = [pow(t, e, p) for e in range(d)]
        exps = [a * b % p for a in exps for b in pw]
    return [be.exp(be.g, e) for e in exps]


def msm(scalars, bases):
    acc = be.identity
    for a, b in zip(scalars, bases):
        if a % p:
            acc = be.mul(acc, be.exp(b, a))
    return acc


def verify(axis_elems, C, point, y, proofs):
    g = be.g
    lhs = be.pair(be.mul(C, be.exp(g, (-y) % p)), g)
    rhs = be.target_identity
    for pi, ax, w in zip(proofs, axis_elems, point):
        rhs = be.target_mul(rhs, be.pair(pi, be.mul(ax, be.exp(g, (-w) % p))))
    return lhs == rhs


def quantize_np(x):
    # RNE(v * 2^16), negatives -> p - |q|
    q = np.rint(np.ldexp(np.asarray(x, dtype=np.float64), 16)).astype(np.int64)
    return [int(v) % p for v in q.tolist()]


def primitives():
    rng = random.Random(1234)
    out = {"field": [], "exp": [], "mul": [], "pair": [], "h2s": [], "enc": []}
    for _ in range(16):
        a, b = dom.rand(rng), dom.rand(rng)
        out["field"].append({"a": hx(a), "b": hx(b), "add": hx(dom.add(a, b)), "sub": hx(dom.sub(a, b)),
                             "mul": hx(dom.mul(a, b)), "inv": hx(dom.inv(a))})
    ks = [0, 1, 2, 3, p - 1, p, p + 5, 2 ** 161, 2 ** 162 + 7] + [dom.rand(rng) for _ in range(12)] + [rng.randrange(1 << 32) for _ in range(4)]
    pts = {}
    for k in ks:
        e = be.exp(be.g, k)
        pts[k] = e
        out["exp"].append({"k": hx(k), "elem": enc(e)})
    g2 = be.exp(be.g, 2)
    cases = [(be.g, be.g), (be.g, g2), (be.g, be.exp(be.g, p - 1)), (None, be.g), (be.g, None), (None, None)]
    for _ in range(8):
        cases.append((be.exp(be.g, dom.rand(rng)), be.exp(be.g, dom.rand(rng))))
    for a, b in cases:
        out["mul"].append({"a": enc(a), "b": enc(b), "sum": enc(be.mul(a, b))})
    for a, b in [(1, 1), (2, 3), (3, 2), (dom.rand(rng), dom.rand(rng)), (0, 5)]:
        ea, eb = be.exp(be.g, a), be.exp(be.g, b)
        t = be.pair(ea, eb)
        out["pair"].append({"a": hx(a), "b": hx(b), "t": [hx(t[0]), hx(t[1])]})
    for data, tag in [(b"", b""), (b"abc", b"terkle/leaf"), (bytes(43), b"terkle/node"), (bytes(range(43)), b"srs/tau")]:
        out["h2s"].append({"data": data.hex(), "tag": tag.hex(), "v": hx(be.hash_to_scalar(data, tag))})
    for s in [0, 1, p - 1, dom.rand(rng)]:
        out["enc"].append({"s": hx(s), "bytes": be.encode_scalar(s).hex()})
    return out


def mvpoly_cases():
    rng = random.Random(99)
    out = []
    for shape in [(1,), (4,), (7,), (3, 3), (2, 3, 4), (4, 4, 4), (5, 5, 5), (2, 2, 2, 2), (3, 1, 4), (16,), (4, 4, 4, 4)]:
        n = 1
        for d in shape:
            n *= d
        vals = [dom.rand(rng) if rng.random() < 0.8 else rng.randrange(100) for _ in range(n)]
        grid = M.default_grid(dom, shape)
        f = M.interpolate_lagrange(dom, vals, grid)
        pt = [dom.rand(rng) for _ in shape]
        qs, y = M.open_quotients(dom, f, pt)
        gp = [rng.randrange(1, d + 1) for d in shape]          # a grid-node challenge
        qg, yg = M.open_quotients(dom, f, gp)
        out.append({"shape": list(shape), "values": [hx(v) for v in vals], "coeffs": [hx(c) for c in f.coeffs],
                    "point": [hx(v) for v in pt], "eval": hx(M.evaluate(dom, f, pt)), "y": hx(y),
                    "quotients": [[hx(c) for c in q.coeffs] for q in qs],
                    "bary": hx(M.barycentric_eval(dom, vals, grid, pt)),
                    "grid_point": gp, "grid_y": hx(yg), "grid_quotients": [[hx(c) for c in q.coeffs] for q in qg]})
    return out


def commit_cases():
    """Small spec-composed commit/open/verify instances."""
    rng = random.Random(7)
    out = []
    for shape, entropy in [((1,), b"seed-a"), ((2, 2), b"seed-b"), ((3,), b"seed-c"), ((2, 3), b"seed-d"), ((2, 2, 2), b"seed-e"), ((4, 4), b"seed-f")]:
        n = 1
        for d in shape:
            n *= d
        taus = taus_for(shape, entropy)
        srs = monomial_srs(shape, taus)
        axis = [be.exp(be.g, t) for t in taus]
        grid = M.default_grid(dom, shape)
        for kind in ["random", "zeros", "const"]:
            if kind == "random":
                vals = [dom.rand(rng) for _ in range(n)]
            elif kind == "zeros":
                vals = [0] * n
            else:
                vals = [12345] * n
            f = M.interpolate_lagrange(dom, vals, grid)
            C = msm(f.coeffs, srs)
            pt = [dom.rand(rng) for _ in shape]
            qs, y = M.open_quotients(dom, f, pt)
            proofs = [msm(q.coeffs, srs) for q in qs]
            ok = verify(axis, C, pt, y, proofs)
            bad = verify(axis, C, pt, (y + 1) % p, proofs)
            assert ok and not bad
            out.append({"shape": list(shape), "entropy": entropy.hex(), "taus": [hx(t) for t in taus],
                        "srs": [enc(e) for e in srs], "axis": [enc(e) for e in axis], "kind": kind,
                        "values": [hx(v) for v in vals], "commitment": enc(C), "point": [hx(v) for v in pt],
                        "y": hx(y), "proofs": [enc(e) for e in proofs], "verify": ok, "verify_y_plus_1": bad})
    return out


def config1():
    """BASELINE config 1: 4096 N(0,1) fp32 from seed 0 -> (64,64); commit;
    open + verify at 4 challenge points from PrimeField.rand(Random(s))."""
    t0 = time.time()
    x = np.random.default_rng(0).standard_normal(4096, dtype=np.float32)
    vals = quantize_np(x)
    shape = (64, 64)
    entropy = b"tc-b200/config1"
    taus = taus_for(shape, entropy)
    srs = monomial_srs(shape, taus)
    axis = [be.exp(be.g, t) for t in taus]
    grid = M.default_grid(dom, shape)
    f = M.interpolate_lagrange(dom, vals, grid)
    C = msm(f.coeffs, srs)
    import hashlib
    opens = []
    for s in range(4):
        r = random.Random(s)
        pt = [dom.rand(r) for _ in shape]
        qs, y = M.open_quotients(dom, f, pt)
        proofs = [msm(q.coeffs, srs) for q in qs]
        ok = verify(axis, C, pt, y, proofs)
        assert ok
        opens.append({"seed": s, "point": [hx(v) for v in pt], "y": hx(y), "proofs": [enc(e) for e in proofs], "verify": ok})
    srs_digest = hashlib.sha256(b"".join(be.encode_elem(e) for e in srs)).hexdigest()
    coeff_digest = hashlib.sha256(b"".join(be.encode_scalar(c) for c in f.coeffs)).hexdigest()
    print("config1 done in %.1fs" % (time.time() - t0))
    return {"shape": list(shape), "entropy": entropy.hex(), "taus": [hx(t) for t in taus],
            "values_digest": hashlib.sha256(b"".join(be.encode_scalar(v) for v in vals)).hexdigest(),
            "srs_digest": srs_digest, "srs_head": [enc(e) for e in srs[:8]], "axis": [enc(e) for e in axis],
            "coeff_digest": coeff_digest, "coeff_head": [hx(c) for c in f.coeffs[:8]],
            "commitment": enc(C), "openings": opens}


def config2():
    """BASELINE config 2: same 4096 values at m = 1, 2, 3, 4, 6."""
    import hashlib
    x = np.random.default_rng(0).standard_normal(4096, dtype=np.float32)
    vals = quantize_np(x)
    out = []
    for shape in [(4096,), (64, 64), (16, 16, 16), (8, 8, 8, 8), (4, 4, 4, 4, 4, 4)]:
        t0 = time.time()
        entropy = b"tc-b200/config2"
        taus = taus_for(shape, entropy)
        srs = monomial_srs(shape, taus)
        f = M.interpolate_lagrange(dom, vals, M.default_grid(dom, shape))
        C = msm(f.coeffs, srs)
        out.append({"shape": list(shape), "entropy": entropy.hex(), "taus": [hx(t) for t in taus],
                    "srs_digest": hashlib.sha256(b"".join(be.encode_elem(e) for e in srs)).hexdigest(),
                    "coeff_digest": hashlib.sha256(b"".join(be.encode_scalar(c) for c in f.coeffs)).hexdigest(),
                    "coeff_head": [hx(c) for c in f.coeffs[:8]], "commitment": enc(C)})
        print("config2", shape, "%.1fs" % (time.time() - t0))
    return out


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as fh:
        json.dump(obj, fh, indent=0)


if __name__ == "__main__":
    which = sys.argv[1:] or ["primitives", "mvpoly", "commit", "config1", "config2"]
    if "primitives" in which:
        dump("primitives.json", primitives())
    if "mvpoly" in which:
        dump("mvpoly.json", mvpoly_cases())
    if "commit" in which:
        dump("commit_small.json", commit_cases())
    if "config1" in which:
        dump("config1.json", config1())
    if "config2" in which:
        dump("config2.json", config2())
