// Exact fixed-point quantisation of one float (protocol.quantize):
// |q| = round-half-even(|v| * 2^k) computed from the binary representation (sign, integer
// mantissa, exponent), never through a float multiply.  Shared by the standalone quantise
// kernel (K1) and the MSM digit kernel, which fuses quantisation into its scalar load.
#pragma once
#include "field.cuh"

namespace tc {

constexpr uint32_t QF_NONFINITE = 1u, QF_OVERFLOW = 2u;

struct Decoded {
  bool neg;
  bool nonfinite;
  uint64_t mant;   // integer mantissa (implicit bit included)
  int exp2;        // value = mant * 2^exp2
};

// dtype codes as in include/tc_b200.h: 1 f16, 2 bf16, 3 f32, 4 f64
template <int DT>
TC_D Decoded decode_float(const void* in, uint64_t i) {
  Decoded d;
  if (DT == 1) {
    uint32_t b = ((const uint16_t*)in)[i];
    uint32_t e = (b >> 10) & 0x1f, m = b & 0x3ff;
    d.neg = b >> 15;
    d.nonfinite = (e == 0x1f);
    d.mant = e ? (m | 0x400u) : m;
    d.exp2 = (e ? (int)e : 1) - 25;
  } else if (DT == 2) {
    uint32_t b = ((const uint16_t*)in)[i];
    uint32_t e = (b >> 7) & 0xff, m = b & 0x7f;
    d.neg = b >> 15;
    d.nonfinite = (e == 0xff);
    d.mant = e ? (m | 0x80u) : m;
    d.exp2 = (e ? (int)e : 1) - 134;
  } else if (DT == 3) {
    uint32_t b = ((const uint32_t*)in)[i];
    uint32_t e = (b >> 23) & 0xff, m = b & 0x7fffffu;
    d.neg = b >> 31;
    d.nonfinite = (e == 0xff);
    d.mant = e ? (m | 0x800000u) : m;
    d.exp2 = (e ? (int)e : 1) - 150;
  } else {
    uint64_t b = ((const uint64_t*)in)[i];
    uint32_t e = (uint32_t)(b >> 52) & 0x7ff;
    uint64_t m = b & 0xfffffffffffffull;
    d.neg = b >> 63;
    d.nonfinite = (e == 0x7ff);
    d.mant = e ? (m | (1ull << 52)) : m;
    d.exp2 = (e ? (int)e : 1) - 1075;
  }
  return d;
}

// |q| = RNE(mant * 2^sh) as 6 limbs; false when |q| >= (p+1)/2 (i.e. |v| 2^k >= p/2)
TC_D bool rne_magnitude(uint64_t mant, int sh, Fe& q) {
  for (int i = 0; i < 6; i++) q.v[i] = 0;
  if (mant == 0) return true;
  if (sh < 0) {
    int s = -sh;
    if (s > 63) return true;   // mant < 2^53 -> value < 1/2 -> 0
    uint64_t iq = mant >> s;
    uint64_t rem = mant & ((1ull << s) - 1ull);
    uint64_t half = 1ull << (s - 1);
    if (rem > half || (rem == half && (iq & 1ull))) iq++;
    q.v[0] = (uint32_t)iq;
    q.v[1] = (uint32_t)(iq >> 32);
    return true;
  }
  int top = 64 - __clzll((long long)mant) + sh;   // bit length of |q|
  if (top > 162) return false;
  int limb = sh >> 5, bit = sh & 31;
  uint64_t lo = mant << bit;
  uint32_t hi = bit ? (uint32_t)(mant >> (64 - bit)) : 0u;
  if (limb < 6) q.v[limb] = (uint32_t)lo;
  if (limb + 1 < 6) q.v[limb + 1] = (uint32_t)(lo >> 32);
  if (limb + 2 < 6) q.v[limb + 2] = hi;
  // (p+1)/2 = 2^160 + 2^23 + 1
  bool over = (q.v[5] > 1u) ||
              (q.v[5] == 1u && ((q.v[4] | q.v[3] | q.v[2] | q.v[1]) != 0u || q.v[0] >= 0x00800001u));
  return !over;
}

// magnitude + sign of the quantised value; flags |= QF_* on error (value then 0)
template <int DT>
TC_D void quantize_signed(const void* in, uint64_t i, int scale_bits, Fe& mag, bool& neg, uint32_t& flags) {
  Decoded d = decode_float<DT>(in, i);
  neg = d.neg;
  if (d.nonfinite) {
    flags |= QF_NONFINITE;
    for (int k = 0; k < 6; k++) mag.v[k] = 0;
  } else if (!rne_magnitude(d.mant, d.exp2 + scale_bits, mag)) {
    flags |= QF_OVERFLOW;
    for (int k = 0; k < 6; k++) mag.v[k] = 0;
  }
}

// canonical F_p element of a signed magnitude: p - |q| for negatives (q != 0)
TC_D Fe signed_to_fp(const Fe& q, bool neg) {
  if (!neg || (q.v[0] | q.v[1] | q.v[2] | q.v[3] | q.v[4] | q.v[5]) == 0) return q;
  Fe r;
  uint64_t t = (uint64_t)FpParams::M0 - q.v[0];
  r.v[0] = (uint32_t)t;
  uint32_t br = (uint32_t)(t >> 63);
  for (int k = 1; k < 5; k++) {
    t = 0ull - q.v[k] - br;
    r.v[k] = (uint32_t)t;
    br = (uint32_t)(t >> 63);
  }
  r.v[5] = FpParams::M5 - q.v[5] - br;
  return r;
}

// centred magnitude of a canonical F_p element: a <= (p-1)/2 -> (a, +), else (p - a, -)
TC_D void centre_fp(const Fe& a, Fe& mag, bool& neg) {
  bool big = (a.v[5] > 1u) ||
             (a.v[5] == 1u && ((a.v[4] | a.v[3] | a.v[2] | a.v[1]) != 0u || a.v[0] > 0x00800000u));
  if (big) {
    uint64_t t = (uint64_t)FpParams::M0 - a.v[0];
    mag.v[0] = (uint32_t)t;
    uint32_t br = (uint32_t)(t >> 63);
    for (int i = 1; i < 5; i++) {
      t = 0ull - a.v[i] - br;
      mag.v[i] = (uint32_t)t;
      br = (uint32_t)(t >> 63);
    }
    mag.v[5] = FpParams::M5 - a.v[5] - br;
    neg = true;
  } else {
    mag = a;
    neg = false;
  }
}

}  // namespace tc
