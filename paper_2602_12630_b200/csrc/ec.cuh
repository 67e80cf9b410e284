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
  Fe t = Fq::inv_pref(Fq::mul(p.ZZ, p.ZZZ));
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

// ---- twisted Edwards model for the MSM: the 2-isogenous curve, a = -1 ------------------
// E: y^2 = x^3 + x has the rational 2-torsion point (0, 0); the 2-isogeny with that kernel,
//   phi(x, y) = ((x^2 + 1) / x, y (1 - x^2) / x^2),
// maps E onto E': Y^2 = X^3 - 4X, and its dual psi(X, Y) = (Y^2 / (4 X^2), Y (-4 - X^2) / (8 X^2))
// maps back with psi(phi(P)) = 2P.  E' has all three 2-torsion points; through X = u - 2,
// u = sqrt(8) w it is the Montgomery curve B v^2 = w^3 + A w^2 + w (A = -6 / sqrt 8) whose
// twisted Edwards model, after scaling, has a = -1 and a non-square d' — the model of the
// fastest mixed addition (Hisil-Wong-Carter-Dawson madd-2008-hwcd-3: 7M with the table
// storing 2d' x y, against 8M for E's own a = 2 model).  a = -1 is not a square mod q, so the
// unified formulas have exceptional inputs, but only of order 2 or 4: every point here lies
// in the order-p subgroup (p odd), where they never occur.
//
// Convention: an Edwards point stands for an E point P as phi([h] P), h = 2^-1 mod p
// (= 2^160 + 2^23 + 1: 160 doublings and 2 additions).  Every MSM base is converted that way
// (aff_to_ed), group operations commute with phi o [h], and ext_to_aff returns
// psi(phi([h] S)) = 2 h S = S — the reference's point, canonical affine, bytes unchanged.
// Both maps are closed rational functions of one inversion each (derivation and check in
// DESIGN.md "Edwards model"; tests/test_edwards_host.py runs them on the host).
// 16-byte aligned so every load / store is LDG.128 / STG.128 (EdAff padded 72 -> 80 B)
struct alignas(16) EdAff {
  Fe x, y, t;
};
struct alignas(16) Ext {
  Fe X, Y, Z, T;
};

#if defined(__CUDACC__)
// explicit 128-bit loads (the struct copy alone leaves ptxas with 24 scalar loads)
TC_D void unpack4(const uint4* q, uint32_t* w, int n4) {
#pragma unroll
  for (int i = 0; i < n4; i++) {
    const uint4 a = q[i];
    w[4 * i] = a.x, w[4 * i + 1] = a.y, w[4 * i + 2] = a.z, w[4 * i + 3] = a.w;
  }
}
TC_D Ext ld_ext(const Ext* p) {
  uint32_t w[24];
  unpack4((const uint4*)p, w, 6);
  Ext r;
#pragma unroll
  for (int i = 0; i < 6; i++) r.X.v[i] = w[i], r.Y.v[i] = w[6 + i], r.Z.v[i] = w[12 + i], r.T.v[i] = w[18 + i];
  return r;
}
TC_D EdAff ld_edaff(const EdAff* p) {
  uint32_t w[20];
  unpack4((const uint4*)p, w, 5);
  EdAff r;
#pragma unroll
  for (int i = 0; i < 6; i++) r.x.v[i] = w[i], r.y.v[i] = w[6 + i], r.t.v[i] = w[12 + i];
  return r;
}
#endif

// Packed storage of an Edwards affine point for the MSM bases: canonical x, y, t (168 bits
// each, q < 2^168) in 504 bits = ONE 64-byte line (two DRAM sectors instead of the three an
// 80-byte EdAff straddles; the config-3 table shrinks 168 -> 134 MB, closer to L2)
struct alignas(64) EdPk {
  uint32_t w[16];
};
TC_HD void pk_put(uint32_t w[16], const Fe& a, int word, int sh) {
  const Fe c = Fq::canon(a);
  for (int i = 0; i < 6; i++) {
    const uint64_t v = (uint64_t)c.v[i] << sh;
    w[word + i] |= (uint32_t)v;
    if (word + i + 1 < 16) w[word + i + 1] |= (uint32_t)(v >> 32);
  }
}
TC_HD EdPk pack_ed(const EdAff& p) {
  EdPk r;
  for (int i = 0; i < 16; i++) r.w[i] = 0;
  pk_put(r.w, p.x, 0, 0);
  pk_put(r.w, p.y, 5, 8);
  pk_put(r.w, p.t, 10, 16);
  return r;
}
#if defined(__CUDACC__)
TC_D EdAff ld_edpk(const EdPk* p) {
  uint32_t w[16];
  unpack4((const uint4*)p, w, 4);
  EdAff r;
#pragma unroll
  for (int i = 0; i < 5; i++) {
    r.x.v[i] = w[i];
    r.y.v[i] = __funnelshift_r(w[5 + i], w[6 + i], 8);
    r.t.v[i] = __funnelshift_r(w[10 + i], w[11 + i], 16);
  }
  r.x.v[5] = w[5] & 0xFFu;
  r.y.v[5] = __funnelshift_r(w[10], w[11], 8) & 0xFFu;
  r.t.v[5] = (w[15] >> 16) & 0xFFu;
  return r;
}
#endif

// constants of the a = -1 model in Montgomery form (tools: DESIGN.md "Edwards model")
TC_HD Fe ed1_s8() { return Fe{{0xf0e3fc7fu, 0x7af10ac5u, 0xd178846bu, 0xb9b458afu, 0x365aaf7eu, 0x0000007bu}}; }   // sqrt(8)
TC_HD Fe ed1_c1() { return Fe{{0x224fdc49u, 0xbe788564u, 0xe8bc4235u, 0x5cda2c57u, 0x9b2d57bfu, 0x00000095u}}; }   // 1 / (sqrt(8) s)
TC_HD Fe ed1_k() { return Fe{{0xb90be8e9u, 0x4db37eccu, 0x2e59caf6u, 0x4b8bd7c2u, 0x73bfc60fu, 0x00000089u}}; }    // 2 d'
TC_HD Fe ed1_kinv() { return Fe{{0x899ae3edu, 0x75132055u, 0x74698d42u, 0x2d1d0a0fu, 0xa3100e7cu, 0x00000071u}}; } // 1 / (2 d')
TC_HD Fe ed1_cx() { return Fe{{0x993cdc1eu, 0x0e3bd4e3u, 0xba1dee52u, 0x192e9d40u, 0x26954205u, 0x000000b3u}}; }   // 1 / (4 s^2)
TC_HD Fe ed1_cy() { return Fe{{0xd5b076b1u, 0xdefc42b1u, 0xf45e211au, 0xae6d162bu, 0xcd96abdfu, 0x00000052u}}; }   // -1 / (8 s)

TC_HD Ext ext_zero() { return Ext{Fq::zero(), Fq::one(), Fq::one(), Fq::zero()}; }
// table points carry t = 2 d' x y; the accumulator's T = X Y / Z
TC_HD Ext ext_from_aff(const EdAff& p) { return Ext{p.x, p.y, Fq::one(), Fq::mul(p.t, ed1_kinv())}; }
TC_HD EdAff edaff_from_xy(const Fe& x, const Fe& y) { return EdAff{x, y, Fq::mul(Fq::mul(x, y), ed1_k())}; }
TC_HD EdAff edaff_neg(const EdAff& p) { return EdAff{Fq::neg(p.x), p.y, Fq::neg(p.t)}; }
TC_HD Ext ext_neg(const Ext& p) { return Ext{Fq::neg(p.X), p.Y, p.Z, Fq::neg(p.T)}; }

// acc += q (q affine with t = 2 d' x y): madd-2008-hwcd-3, a = -1 — 7 products, 7 reductions
// (E and H from unreduced products, Fq::lazy_e_h1)
TC_HD void ext_madd(Ext& acc, const EdAff& q) {
  // Statement order matters to ptxas's register allocation in k_accum_aff (80 registers at
  // 6 blocks per SM): C, F and G first, so T1, Z1 and t2 are dead before the two wide
  // products of E / H, then the outputs in the order T, Z, Y, X.  Swept over both halves'
  // orders and all 24 output orders (tools/ab_libs40.sh): 4.276 -> 4.182 ms per forward,
  // accumulation 0.857 -> 0.882 of the IMAD peak; the previous order spilled 28 bytes per
  // thread, this one none.
  const Fe C = Fq::mul(acc.T, q.t);               // 2 d' T1 T2
  const Fe D = Fq::dbl(acc.Z);                    // 2 Z1
  const Fe F = Fq::sub(D, C);
  const Fe G = Fq::add(D, C);
  Fe E, H;
  Fq::lazy_e_h1(acc.X, acc.Y, q.x, q.y, E, H);   // E = 2(X1 y2 + Y1 x2), H = 2(Y1 y2 + X1 x2)
  acc.T = Fq::mul(E, H);
  acc.Z = Fq::mul(F, G);
  acc.Y = Fq::mul(G, H);
  acc.X = Fq::mul(E, F);
}

// acc += q, both extended: add-2008-hwcd-3, a = -1 (9M)
TC_HD void ext_add(Ext& acc, const Ext& q) {
  Fe E, H;
  Fq::lazy_e_h1(acc.X, acc.Y, q.X, q.Y, E, H);
  const Fe C = Fq::mul(Fq::mul(acc.T, q.T), ed1_k());
  const Fe D = Fq::dbl(Fq::mul(acc.Z, q.Z));
  const Fe F = Fq::sub(D, C);
  const Fe G = Fq::add(D, C);
  acc.X = Fq::mul(E, F);
  acc.Y = Fq::mul(G, H);
  acc.T = Fq::mul(E, H);
  acc.Z = Fq::mul(F, G);
}

// 2P: dbl-2008-hwcd, a = -1 (4M + 4S)
TC_HD Ext ext_dbl(const Ext& p) {
  const Fe A = Fq::sqr(p.X);
  const Fe B = Fq::sqr(p.Y);
  const Fe C = Fq::dbl(Fq::sqr(p.Z));
  const Fe E = Fq::sub(Fq::sub(Fq::sqr(Fq::add(p.X, p.Y)), A), B);
  const Fe G = Fq::sub(B, A);         // a A + B
  const Fe F = Fq::sub(G, C);
  const Fe H = Fq::neg(Fq::add(A, B));   // a A - B
  return Ext{Fq::mul(E, F), Fq::mul(G, H), Fq::mul(F, G), Fq::mul(E, H)};
}

// k * P for a small non-negative k, double-and-add from the MSB
TC_HD Ext ext_mul_small(const Ext& p, uint32_t k) {
  Ext r = ext_zero();
  bool started = false;
  for (int b = 31; b >= 0; b--) {
    if (started) r = ext_dbl(r);
    if ((k >> b) & 1u) {
      if (started) {
        ext_add(r, p);
      } else {
        r = p;
        started = true;
      }
    }
  }
  return r;
}

// k * P through the non-adjacent form (k = 2^10 - 1 costs 10 doublings + 1 add, not
// 10 + 9): the latency-bound window re-basing multiplies by mlo - 1 = 1023
TC_HD Ext ext_mul_small_naf(const Ext& p, uint32_t k) {
  if (k == 0) return ext_zero();
  int8_t naf[34];
  int len = 0;
  uint64_t v = k;
  while (v) {
    int d = 0;
    if (v & 1u) {
      d = 2 - (int)(v & 3u);   // +1 or -1
      v -= (uint64_t)(int64_t)d;
    }
    naf[len++] = (int8_t)d;
    v >>= 1;
  }
  const Ext np = ext_neg(p);
  Ext r = naf[len - 1] > 0 ? p : np;
  for (int i = len - 2; i >= 0; i--) {
    r = ext_dbl(r);
    if (naf[i] > 0) ext_add(r, p);
    if (naf[i] < 0) ext_add(r, np);
  }
  return r;
}

// Edwards (X:Y:Z:T) on E' -> psi -> canonical-ready Montgomery-form affine point of E:
// with N = sqrt8 (Z + Y) - 2 (Z - Y) and one inversion of D = X^2 N^2 (Z - Y),
//   x = ((Z + Y) Z)^2 (Z - Y) / (4 s^2 D),  y = -(Z + Y) Z (4 (Z - Y)^2 + N^2) X / (8 s D).
// The neutral element (X = 0) -> infinity.  ext_to_aff_den / _with_inv: batch-inversion form.
TC_HD Fe ext_to_aff_den(const Ext& p) {
  if (Fq::is_zero(p.X)) return Fq::one();
  const Fe zm = Fq::sub(p.Z, p.Y);
  const Fe N = Fq::sub(Fq::mul(ed1_s8(), Fq::add(p.Z, p.Y)), Fq::dbl(zm));
  return Fq::mul(Fq::mul(Fq::sqr(p.X), Fq::sqr(N)), zm);
}
TC_HD Aff ext_to_aff_with_inv(const Ext& p, const Fe& inv) {
  if (Fq::is_zero(p.X)) return aff_inf();
  const Fe zp = Fq::add(p.Z, p.Y), zm = Fq::sub(p.Z, p.Y);
  const Fe N = Fq::sub(Fq::mul(ed1_s8(), zp), Fq::dbl(zm));
  const Fe zpz = Fq::mul(zp, p.Z);
  const Fe x = Fq::mul(Fq::mul(Fq::mul(Fq::sqr(zpz), zm), inv), ed1_cx());
  const Fe w = Fq::add(Fq::dbl(Fq::dbl(Fq::sqr(zm))), Fq::sqr(N));   // 4 (Z - Y)^2 + N^2
  const Fe y = Fq::mul(Fq::mul(Fq::mul(Fq::mul(zpz, w), p.X), inv), ed1_cy());
  return Aff{x, y};
}
TC_HD Aff ext_to_aff(const Ext& p) {
  if (Fq::is_zero(p.X)) return aff_inf();
  return ext_to_aff_with_inv(p, Fq::inv_pref(ext_to_aff_den(p)));
}

// [h] P on E, h = 2^-1 mod p = 2^160 + 2^23 + 1 (XYZZ: 160 doublings, 2 mixed adds)
TC_HD Xyzz xyzz_mul_half(const Aff& p) {
  if (aff_is_inf(p)) return xyzz_inf();
  Xyzz acc = xyzz_from_aff(p);
  for (int b = 159; b >= 0; b--) {
    acc = xyzz_dbl(acc);
    if (b == 23 || b == 0) xyzz_add_aff(acc, p);
  }
  return acc;
}

// E affine point Q (already [h]-scaled) -> E' Edwards (x_e, y_e, 2 d' x_e y_e):
//   x_e = c1 x (x + 1) / (y (1 - x)),  y_e = ((x + 1)^2 - sqrt8 x) / ((x + 1)^2 + sqrt8 x),
// one inversion of den = y (1 - x) ((x + 1)^2 + sqrt8 x) (never 0 in the odd-order subgroup:
// its zeros are points of order 2 or 4).  Infinity -> the neutral (0, 1).
TC_HD Fe aff_ed_den(const Aff& q) {
  if (aff_is_inf(q)) return Fq::one();
  const Fe x1 = Fq::add(q.x, Fq::one());
  const Fe sq = Fq::add(Fq::sqr(x1), Fq::mul(ed1_s8(), q.x));
  return Fq::mul(Fq::mul(q.y, Fq::sub(Fq::one(), q.x)), sq);
}
TC_HD EdAff aff_to_ed_with_inv(const Aff& q, const Fe& inv) {
  if (aff_is_inf(q)) return EdAff{Fq::zero(), Fq::one(), Fq::zero()};
  const Fe x1 = Fq::add(q.x, Fq::one());
  const Fe a = Fq::sqr(x1), sx = Fq::mul(ed1_s8(), q.x);
  const Fe xe = Fq::mul(Fq::mul(Fq::mul(Fq::mul(ed1_c1(), q.x), x1), Fq::add(a, sx)), inv);
  const Fe ye = Fq::mul(Fq::mul(Fq::sub(a, sx), Fq::mul(q.y, Fq::sub(Fq::one(), q.x))), inv);
  return edaff_from_xy(xe, ye);
}
// the model's image of an E point that is ALREADY [h]-scaled
TC_HD EdAff aff_to_ed_noh(const Aff& q) { return aff_to_ed_with_inv(q, Fq::inv_pref(aff_ed_den(q))); }
// the model's image of an E point P: phi([h] P)
TC_HD EdAff aff_to_ed(const Aff& p) {
  const Aff q = xyzz_to_aff(xyzz_mul_half(p));
  return aff_to_ed_noh(q);
}

}  // namespace tc
