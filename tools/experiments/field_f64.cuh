// F_q arithmetic on the FP64 pipe.
//
// B200 (sm_100a) keeps full-rate FP64: DFMA issues at 64 lanes/clk/SM, the same rate as
// IMAD, on a SEPARATE pipe (measured: 8 DFMA + 8 IMAD chains per thread run in 0.57x the
// time of 16 of either; tools/imad_peak.cu, profiles/r01_imad_peak.json).  The integer
// Montgomery product (field.cuh) saturates the fma-heavy pipe while the FP64 pipe idles,
// so warps that do their F_q products in doubles run alongside warps that use IMAD.
//
// Representation ("FeD"): value = sum_k v[k] * 2^(24 k), k = 0..6, every v[k] an integer
// held exactly in a double; limbs are SIGNED and only loosely normalised.  Montgomery form
// with R' = 2^168 (7 x 24 bits; q = 120 p - 1 < 2^168, backend.py:104-105).  In 24-bit
// limbs q = [119, 120, 0, 0, 0, 0, 120 * 2^17]: three small non-zero limbs, so each of the
// 7 reduction steps costs 4 DFMA instead of 7.
//
// Exactness: every intermediate is an integer below 2^53 in magnitude.
//   * product inputs: limbs |v| <= 2^24 + 2^10 ("N1": a normalised element, or the sum /
//     difference of two).  Column sums: <= 7 * 2^48.01 < 2^50.9; reduction adds at most
//     u * Q6 < 2^47.9 and small carries, so every column stays < 2^51 — the bound the
//     1.5 * 2^52 "magic" extraction of the low word needs.
//   * mul/sqr outputs are normalised: limbs 0..5 in [-2^23, 2^23], limb 6 the rest, and
//     a top-limb range fix keeps |value| < 1.1 q.
//   * add/sub/dbl are limb-wise; callers normalise (norm()) before a product when an
//     operand is the sum of more than two normalised values.
#pragma once
#include "../../paper_2602_12630_b200/csrc/field.cuh"

namespace tc {

struct FeD {
  double v[7];
};

struct FqD {
  static constexpr double MAG = 6755399441055744.0;      // 1.5 * 2^52
  static constexpr double T24 = 16777216.0;              // 2^24
  static constexpr double I24 = 1.0 / 16777216.0;        // 2^-24
  static constexpr double Q0 = 119.0, Q1 = 120.0, Q6 = 15728640.0;   // q limbs 0, 1, 6
  static constexpr double IQ6 = 1.0 / 15728640.0;
  static constexpr uint32_t NP24 = 0x0226b9u;            // -q^-1 mod 2^24
  static constexpr uint32_t MAGHI = 0x43380000u;         // high word of MAG

  TC_HD static FeD zero() {
    FeD r;
#pragma unroll
    for (int k = 0; k < 7; k++) r.v[k] = 0.0;
    return r;
  }

#if defined(__CUDA_ARCH__)
  TC_D static double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
  // low 32 bits of an integer-valued double c, |c| < 2^51 (two's complement)
  TC_D static uint32_t lo32(double c) { return (uint32_t)__double2loint(c + MAG); }
  // u in [0, 2^32) -> double, exact
  TC_D static double from_u32(uint32_t u) { return __hiloint2double((int)MAGHI, (int)u) - MAG; }
  // round-to-nearest integer of x, |x| < 2^51
  TC_D static double rint_(double x) { return (x + MAG) - MAG; }
#else
  static double fma_(double a, double b, double c) { return __builtin_fma(a, b, c); }
  static uint32_t lo32(double c) {
    volatile double t = c + MAG;
    uint64_t bits;
    __builtin_memcpy(&bits, (const void*)&t, 8);
    return (uint32_t)bits;
  }
  static double from_u32(uint32_t u) { return (double)u; }
  static double rint_(double x) {
    volatile double t = x + MAG;
    return t - MAG;
  }
#endif

  TC_HD static FeD add(const FeD& a, const FeD& b) {
    FeD r;
#pragma unroll
    for (int k = 0; k < 7; k++) r.v[k] = a.v[k] + b.v[k];
    return r;
  }
  TC_HD static FeD sub(const FeD& a, const FeD& b) {
    FeD r;
#pragma unroll
    for (int k = 0; k < 7; k++) r.v[k] = a.v[k] - b.v[k];
    return r;
  }
  TC_HD static FeD neg(const FeD& a) {
    FeD r;
#pragma unroll
    for (int k = 0; k < 7; k++) r.v[k] = -a.v[k];
    return r;
  }
  TC_HD static FeD dbl(const FeD& a) { return add(a, a); }

  // carry-normalise limbs 0..5 into [-2^23, 2^23]; limb 6 takes the rest
  TC_HD static void norm_in(double r[7]) {
#pragma unroll
    for (int k = 0; k < 6; k++) {
      const double c = rint_(r[k] * I24);
      r[k] = fma_(c, -T24, r[k]);
      r[k + 1] += c;
    }
  }
  // |value| -> below ~1.1 q: subtract round(value / q) * q estimated from the top limb
  TC_HD static void range_fix(double r[7]) {
    const double k = rint_(r[6] * IQ6);
    r[0] = fma_(k, -Q0, r[0]);
    r[1] = fma_(k, -Q1, r[1]);
    r[6] = fma_(k, -Q6, r[6]);
  }
  TC_HD static FeD norm(const FeD& a) {
    FeD r = a;
    norm_in(r.v);
    range_fix(r.v);
    return r;
  }

  // Montgomery reduction of the 13 product columns c[0..12] -> c * 2^-168 mod q
  TC_HD static FeD redc(double c[13]) {
#pragma unroll
    for (int i = 0; i < 7; i++) {
      const uint32_t u = (lo32(c[i]) * NP24) & 0xFFFFFFu;
      const double ud = from_u32(u);
      const double ci = fma_(ud, Q0, c[i]);   // = 0 mod 2^24
      c[i + 1] = fma_(ud, Q1, c[i + 1]);
      c[i + 1] = fma_(ci, I24, c[i + 1]);
      c[i + 6] = fma_(ud, Q6, c[i + 6]);
    }
    FeD r;
#pragma unroll
    for (int k = 0; k < 6; k++) r.v[k] = c[7 + k];
    r.v[6] = 0.0;
    norm_in(r.v);
    range_fix(r.v);
    return r;
  }

  TC_HD static FeD mul(const FeD& a, const FeD& b) {
    double c[13];
#pragma unroll
    for (int k = 0; k < 13; k++) c[k] = 0.0;
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = 0; j < 7; j++) c[i + j] = fma_(a.v[i], b.v[j], c[i + j]);
    return redc(c);
  }

  TC_HD static FeD sqr(const FeD& a) {
    double c[13], d[7];
#pragma unroll
    for (int k = 0; k < 7; k++) d[k] = a.v[k] + a.v[k];
#pragma unroll
    for (int k = 0; k < 13; k++) c[k] = 0.0;
#pragma unroll
    for (int i = 0; i < 7; i++) {
      c[2 * i] = fma_(a.v[i], a.v[i], c[2 * i]);
#pragma unroll
      for (int j = i + 1; j < 7; j++) c[i + j] = fma_(d[i], a.v[j], c[i + j]);
    }
    return redc(c);
  }

  // ---- conversions ------------------------------------------------------------------
  // A 6 x u32 integer (< 2^192, e.g. a lazy [0, 2q) value) -> 7 limbs of 24 bits
  // (limb 6 takes bits 144..191).  Exact; no modular change.
  TC_HD static FeD from_words(const Fe& x) {
    FeD r;
    const uint32_t* w = x.v;
    r.v[0] = from_u32(w[0] & 0xFFFFFFu);
    r.v[1] = from_u32(((w[0] >> 24) | (w[1] << 8)) & 0xFFFFFFu);
    r.v[2] = from_u32(((w[1] >> 16) | (w[2] << 16)) & 0xFFFFFFu);
    r.v[3] = from_u32(w[2] >> 8);
    r.v[4] = from_u32(w[3] & 0xFFFFFFu);
    r.v[5] = from_u32(((w[3] >> 24) | (w[4] << 8)) & 0xFFFFFFu);
    r.v[6] = from_u32(((w[4] >> 16) | (w[5] << 16)));   // < 2^32 for values < 2^176
    return r;
  }

  // exact integer value of a (any limbs within the invariants) reduced into [0, 2q):
  // two's-complement 224-bit accumulation, then a multiple of q added/subtracted.
  TC_HD static Fe to_words_lazy(const FeD& a) {
    FeD t = norm(a);   // limbs 0..5 in [-2^23, 2^23], |value| < 1.1 q
    // signed limbs -> 7 x 32-bit two's complement words of the value + 2q (positive)
    int64_t acc = 0;
    uint32_t w[7];
    // value = sum t_k 2^(24k); emit 32-bit words
    // build as 64-bit chunks: bit offset 24k
    int64_t limb[7];
#pragma unroll
    for (int k = 0; k < 7; k++) limb[k] = (int64_t)t.v[k];
    // add 2q to make it positive: 2q limbs (24-bit) = [238, 240, 0, 0, 0, 0, 2 * Q6]
    limb[0] += 238;
    limb[1] += 240;
    limb[6] += 31457280;
    // carry-propagate into non-negative 24-bit digits
#pragma unroll
    for (int k = 0; k < 6; k++) {
      int64_t c = limb[k] >> 24;   // arithmetic shift = floor division
      limb[k] -= c << 24;
      limb[k + 1] += c;
    }
    // pack 7 digits (top one up to ~26 bits) into words
    uint64_t d[7];
#pragma unroll
    for (int k = 0; k < 7; k++) d[k] = (uint64_t)limb[k];
    w[0] = (uint32_t)(d[0] | (d[1] << 24));
    w[1] = (uint32_t)((d[1] >> 8) | (d[2] << 16));
    w[2] = (uint32_t)((d[2] >> 16) | (d[3] << 8));
    w[3] = (uint32_t)(d[4] | (d[5] << 24));
    w[4] = (uint32_t)((d[5] >> 8) | (d[6] << 16));
    w[5] = (uint32_t)(d[6] >> 16);
    (void)acc;
    (void)w[6];
    Fe r{{w[0], w[1], w[2], w[3], w[4], w[5]}};
    // value + 2q in [0.9q, 3.1q) -> [0, 2q)
    r = Fq::red2(r);
    r = Fq::red2(r);
    return r;
  }
};

}  // namespace tc
