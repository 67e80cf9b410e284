// Group arithmetic on E: y^2 = x^3 + x over F_q (a = 1, b = 0), the reference's
// production curve (backend.py:9-13, 102-108).
//
// The reference works in Jacobian coordinates (backend.py:111-146) and converts every
// result to affine with one inversion (backend.py:149-155).  Here accumulators live in
// XYZZ coordinates (x = X/ZZ, y = Y/ZZZ): a mixed affine add is 8M+2S and needs no
// doubling-specific branches in the common case, which is what Pippenger bucket
// accumulation spends nearly all its time in.  Affine outputs are canonical, so any
// coordinate system yields the reference's bytes exactly.
//
// Affine points are stored in Montgomery form; the point at infinity is flagged with
// x.v[5] = 0xFFFFFFFF (never a valid lazy field element, whose top limb is < 2*0xF0).
#pragma once
#include "field.cuh"

namespace tc {

struct Aff {
  Fe x, y;
};
struct Xyzz {
  Fe X, Y, ZZ, ZZZ;
};

static constexpr uint32_t AFF_INF_TAG = 0xFFFFFFFFu;

TC_HD bool aff_is_inf(const Aff& p) { return p.x.v[5] == AFF_INF_TAG; }
TC_HD Aff aff_inf() {
  Aff p;
  for (int i = 0; i < 6; i++) p.x.v[i] = AFF_INF_TAG, p.y.v[i] = 0;
  return p;
}
TC_HD Aff aff_neg(const Aff& p) {
  if (aff_is_inf(p)) return p;
  return Aff{p.x, Fq::neg(p.y)};
}

TC_HD Xyzz xyzz_inf() {
  Xyzz r;
  r.X = Fq::one();
  r.Y = Fq::one();
  r.ZZ = Fq::zero();
  r.ZZZ = Fq::zero();
  return r;
}
TC_HD bool xyzz_is_inf(const Xyzz& p) { return Fq::is_zero(p.ZZ); }
TC_HD Xyzz xyzz_from_aff(const Aff& p) {
  if (aff_is_inf(p)) return xyzz_inf();
  return Xyzz{p.x, p.y, Fq::one(), Fq::one()};
}
TC_HD Xyzz xyzz_neg(const Xyzz& p) { return Xyzz{p.X, Fq::neg(p.Y), p.ZZ, p.ZZZ}; }

// 2 * (x, y) for an affine point, result in XYZZ (mdbl-2008-s-1, a = 1)
TC_HD Xyzz xyzz_dbl_aff(const Aff& p) {
  Fe U = Fq::dbl(p.y);
  Fe V = Fq::sqr(U);
  Fe W = Fq::mul(U, V);
  Fe S = Fq::mul(p.x, V);
  Fe xx = Fq::sqr(p.x);
  Fe M = Fq::add(Fq::add(Fq::dbl(xx), xx), Fq::one());
  Xyzz r;
  r.X = Fq::sub(Fq::sqr(M), Fq::dbl(S));
  r.Y = Fq::sub(Fq::mul(M, Fq::sub(S, r.X)), Fq::mul(W, p.y));
  r.ZZ = V;
  r.ZZZ = W;
  return r;
}

// 2P in XYZZ (dbl-2008-s-1 with a = 1: M = 3X^2 + ZZ^2).  Y = 0 gives ZZ3 = 0 = infinity.
TC_HD Xyzz xyzz_dbl(const Xyzz& p) {
  Fe U = Fq::dbl(p.Y);
  Fe V = Fq::sqr(U);
  Fe W = Fq::mul(U, V);
  Fe S = Fq::mul(p.X, V);
  Fe xx = Fq::sqr(p.X);
  Fe M = Fq::add(Fq::add(Fq::dbl(xx), xx), Fq::sqr(p.ZZ));
  Xyzz r;
  r.X = Fq::sub(Fq::sqr(M), Fq::dbl(S));
  r.Y = Fq::sub(Fq::mul(M, Fq::sub(S, r.X)), Fq::mul(W, p.Y));
  r.ZZ = Fq::mul(V, p.ZZ);
  r.ZZZ = Fq::mul(W, p.ZZZ);
  return r;
}

// acc += q (q affine, madd-2008-s) with every exceptional case handled.
TC_HD void xyzz_add_aff(Xyzz& acc, const Aff& q) {
  if (aff_is_inf(q)) return;
  if (xyzz_is_inf(acc)) {
    acc = xyzz_from_aff(q);
    return;
  }
  Fe U2 = Fq::mul(q.x, acc.ZZ);
  Fe S2 = Fq::mul(q.y, acc.ZZZ);
  Fe P = Fq::sub(U2, acc.X);
  Fe R = Fq::sub(S2, acc.Y);
  if (Fq::is_zero(P)) {
    if (Fq::is_zero(R)) {
      acc = xyzz_dbl_aff(q);
    } else {
      acc = xyzz_inf();
    }
    return;
  }
  Fe PP = Fq::sqr(P);
  Fe PPP = Fq::mul(P, PP);
  Fe Qv = Fq::mul(acc.X, PP);
  Fe X3 = Fq::sub(Fq::sub(Fq::sqr(R), PPP), Fq::dbl(Qv));
  Fe Y3 = Fq::sub(Fq::mul(R, Fq::sub(Qv, X3)), Fq::mul(acc.Y, PPP));
  acc.ZZ = Fq::mul(acc.ZZ, PP);
  acc.ZZZ = Fq::mul(acc.ZZZ, PPP);
  acc.X = X3;
  acc.Y = Y3;
}

// acc += q, both XYZZ (add-2008-s)
TC_HD void xyzz_add(Xyzz& acc, const Xyzz& q) {
  if (xyzz_is_inf(q)) return;
  if (xyzz_is_inf(acc)) {
    acc = q;
    return;
  }
  Fe U1 = Fq::mul(acc.X, q.ZZ);
  Fe U2 = Fq::mul(q.X, acc.ZZ);
  Fe S1 = Fq::mul(acc.Y, q.ZZZ);
  Fe S2 = Fq::mul(q.Y, acc.ZZZ);
  Fe P = Fq::sub(U2, U1);
  Fe R = Fq::sub(S2, S1);
  if (Fq::is_zero(P)) {
    if (Fq::is_zero(R)) {
      acc = xyzz_dbl(acc);
    } else {
      acc = xyzz_inf();
    }
    return;
  }
  Fe PP = Fq::sqr(P);
  Fe PPP = Fq::mul(P, PP);
  Fe Qv = Fq::mul(U1, PP);
  Fe X3 = Fq::sub(Fq::sub(Fq::sqr(R), PPP), Fq::dbl(Qv));
  Fe Y3 = Fq::sub(Fq::mul(R, Fq::sub(Qv, X3)), Fq::mul(S1, PPP));
  acc.ZZ = Fq::mul(Fq::mul(acc.ZZ, q.ZZ), PP);
  acc.ZZZ = Fq::mul(Fq::mul(acc.ZZZ, q.ZZZ), PPP);
  acc.X = X3;
  acc.Y = Y3;
}

// k * P for a small non-negative k (bucket-segment offsets), double-and-add MSB first
TC_HD Xyzz xyzz_mul_small(const Xyzz& p, uint32_t k) {
  Xyzz r = xyzz_inf();
  bool started = false;
  for (int b = 31; b >= 0; b--) {
    if (started) r = xyzz_dbl(r);
    if ((k >> b) & 1u) {
      if (started) {
        xyzz_add(r, p);
      } else {
        r = p;
        started = true;
      }
    }
  }
  return r;
}

// XYZZ -> affine (Montgomery form).  One field inversion of ZZ*ZZZ.
TC_HD Aff xyzz_to_aff(const Xyzz& p) {
  if (xyzz_is_inf(p)) return aff_inf();
  Fe t = Fq::inv(Fq::mul(p.ZZ, p.ZZZ));
  Fe izz = Fq::mul(t, p.ZZZ);   // 1/ZZ
  Fe izzz = Fq::mul(t, p.ZZ);   // 1/ZZZ
  return Aff{Fq::mul(p.X, izz), Fq::mul(p.Y, izzz)};
}

// Same, given a precomputed inverse of ZZ*ZZZ (batch inversion).
TC_HD Aff xyzz_to_aff_with_inv(const Xyzz& p, const Fe& inv_zz_zzz) {
  Fe izz = Fq::mul(inv_zz_zzz, p.ZZZ);
  Fe izzz = Fq::mul(inv_zz_zzz, p.ZZ);
  return Aff{Fq::mul(p.X, izz), Fq::mul(p.Y, izzz)};
}

// canonical little-endian affine coordinates (what encode_elem serialises)
TC_HD void aff_to_canonical(const Aff& p, uint32_t out_x[6], uint32_t out_y[6], bool* inf) {
  if (aff_is_inf(p)) {
    *inf = true;
    for (int i = 0; i < 6; i++) out_x[i] = out_y[i] = 0;
    return;
  }
  *inf = false;
  Fe x = Fq::from_mont(p.x), y = Fq::from_mont(p.y);
  for (int i = 0; i < 6; i++) out_x[i] = x.v[i], out_y[i] = y.v[i];
}

// 43-byte encoding (backend.py:309-317): 0x04 || x LE21 || y LE21, infinity = 43 zero bytes
TC_HD void aff_encode43(const Aff& p, uint8_t out[43]) {
  uint32_t x[6], y[6];
  bool inf;
  aff_to_canonical(p, x, y, &inf);
  if (inf) {
    for (int i = 0; i < 43; i++) out[i] = 0;
    return;
  }
  out[0] = 4;
  for (int i = 0; i < 21; i++) {
    out[1 + i] = (uint8_t)(x[i / 4] >> (8 * (i % 4)));
    out[22 + i] = (uint8_t)(y[i / 4] >> (8 * (i % 4)));
  }
}

}  // namespace tc
