// Host check of the twisted Edwards MSM arithmetic (ec.cuh: a = -1 model of the 2-isogenous
// curve, bases phi([1/2] P), results psi(.)) against the XYZZ/affine
// Montgomery arithmetic: random multiples of g, sums, doublings, P - P, neutral.
// nvcc -std=c++17 --expt-relaxed-constexpr -o /tmp/ed_check tools/ed_check.cu && /tmp/ed_check
#include <cstdio>
#include <random>
#include "../paper_2602_12630_b200/csrc/ec.cuh"
using namespace tc;

static Aff g_aff() {
  Fe x{{0xbe9bb8c2u, 0x9f4698deu, 0x2e04a40bu, 0x96df9421u, 0xd6e0e406u, 0x000000abu}};
  Fe y{{0xca83210eu, 0x0d3911f8u, 0x28e6ecd6u, 0xfcd508bdu, 0xc7320595u, 0x00000018u}};
  return Aff{Fq::to_mont(x), Fq::to_mont(y)};
}
static bool aff_eq(const Aff& a, const Aff& b) {
  if (aff_is_inf(a) || aff_is_inf(b)) return aff_is_inf(a) == aff_is_inf(b);
  return Fq::eq(a.x, b.x) && Fq::eq(a.y, b.y);
}
static Aff mul_small(const Aff& g, uint32_t k) {
  Xyzz acc = xyzz_inf();
  for (uint32_t i = 0; i < k; i++) xyzz_add_aff(acc, g);
  return xyzz_to_aff(acc);
}
int main() {
  std::mt19937 rng(5);
  Aff g = g_aff();
  int bad = 0, n = 0;
  for (int it = 0; it < 40; it++) {
    uint32_t a = rng() % 50 + 1, b = rng() % 50 + 1;
    Aff P = mul_small(g, a), Q = mul_small(g, b);
    EdAff Pe = aff_to_ed(P), Qe = aff_to_ed(Q);
    // round trip
    bad += !aff_eq(ext_to_aff(ext_from_aff(Pe)), P); n++;
    // mixed add vs Montgomery sum
    Aff R = mul_small(g, a + b);
    Ext acc = ext_from_aff(Pe);
    ext_madd(acc, Qe);
    bad += !aff_eq(ext_to_aff(acc), R); n++;
    // full add, from the neutral element
    Ext z = ext_zero();
    ext_add(z, ext_from_aff(Pe));
    ext_add(z, acc);   // P + (P + Q)
    bad += !aff_eq(ext_to_aff(z), mul_small(g, 2 * a + b)); n++;
    // doubling, and P + P through madd (complete: no special case)
    bad += !aff_eq(ext_to_aff(ext_dbl(ext_from_aff(Pe))), mul_small(g, 2 * a)); n++;
    Ext pp = ext_from_aff(Pe);
    ext_madd(pp, Pe);
    bad += !aff_eq(ext_to_aff(pp), mul_small(g, 2 * a)); n++;
    // P + (-P) = neutral -> infinity
    Ext pm = ext_from_aff(Pe);
    ext_madd(pm, edaff_neg(Pe));
    bad += !aff_is_inf(ext_to_aff(pm)); n++;
    // neutral + P via madd
    Ext zz = ext_zero();
    ext_madd(zz, Qe);
    bad += !aff_eq(ext_to_aff(zz), Q); n++;
    // small scalar multiple (binary and NAF)
    bad += !aff_eq(ext_to_aff(ext_mul_small(ext_from_aff(Pe), 7)), mul_small(g, 7 * a)); n++;
    for (uint32_t k : {1u, 2u, 3u, 7u, 11u, 1023u, 1024u, 4095u})
      bad += !aff_eq(ext_to_aff(ext_mul_small_naf(ext_from_aff(Pe), k)), ext_to_aff(ext_mul_small(ext_from_aff(Pe), k))), n++;
    // infinity in -> neutral
    bad += !aff_is_inf(ext_to_aff(ext_from_aff(aff_to_ed(aff_inf())))); n++;
  }
  // binary-Euclid inversion == Fermat inversion (F_q and F_p, random + edge values)
  std::mt19937_64 r64(9);
  for (int it = 0; it < 300; it++) {
    Fe a;
    for (int i = 0; i < 5; i++) a.v[i] = (uint32_t)r64();
    a.v[5] = (uint32_t)(r64() % 0x1E0);
    if (it == 0) a = Fq::one();
    if (it == 1) a = Fq::zero();
    if (it == 2) a = Fe{{0x78000076u, 0, 0, 0, 0, 0xF0u}};   // q - 1 (canonical, as Montgomery value)
    bad += !Fq::eq(Fq::inv_fast(a), Fq::inv(a)); n++;
    Fe b = a;
    b.v[5] &= 0x3u;
    bad += !Fp::eq(Fp::inv_fast(b), Fp::inv(b)); n++;
  }
  // lazy E / H against the reduced formulas on lazy operands close to 2m (the sums exceed 2m)
  for (int it = 0; it < 2000; it++) {
    Fe a[4];
    for (int j = 0; j < 4; j++) {
      for (int i = 0; i < 5; i++) a[j].v[i] = (uint32_t)r64();
      a[j].v[5] = (uint32_t)(0x1D0 + r64() % 0x10);   // in [2m - 2^164, 2m): lazy, near the top
      if (it & 1) a[j].v[5] = (uint32_t)(r64() % 0x1E0);
      a[j] = Fq::red2(a[j]);
    }
    Fe E, H;
    Fq::lazy_e_h(a[0], a[1], a[2], a[3], E, H);
    const Fe A = Fq::mul(a[0], a[2]), B = Fq::mul(a[1], a[3]);
    const Fe E2 = Fq::add(Fq::mul(a[0], a[3]), Fq::mul(a[1], a[2]));
    const Fe H2 = Fq::sub(B, Fq::dbl(A));
    bad += !Fq::eq(E, E2) || !Fq::eq(H, H2); n++;
    // outputs stay lazy (< 2m)
    bad += (E.v[5] >= 0x1E0u) || (H.v[5] >= 0x1E0u); n++;
  }
  printf("{\"edwards_checks\": %d, \"bad\": %d}\n", n, bad);
  return bad != 0;
}
