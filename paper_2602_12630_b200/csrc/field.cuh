// 6 x u32 Montgomery arithmetic for the two prime fields of the TensorCommitments
// curve (reference: /root/reference/pkg/src/tensorcommit/backend.py:102-108):
//
//   p = 2^161 + 2^24 + 1         scalar field / subgroup order   limbs [0x01000001,0,0,0,0,0x2]
//   q = 120 p - 1                curve base field                limbs [0x78000077,0,0,0,0,0xF0]
//
// Both moduli have only limbs 0 and 5 non-zero, so Montgomery reduction (R = 2^192)
// costs 6 word products against limb 0 plus one 6-limb multiply by the small top limb,
// instead of the 36 products of a dense modulus.  The 6x6 schoolbook product is written as
// even/odd mad.lo.cc / madc.hi.cc chains, which ptxas fuses into IMAD.WIDE.U32(.X) with
// carry in/out (one instruction per 32x32->64 partial product).
//
// Representation invariant ("lazy"): every element is kept in [0, 2m).  Because
// 4m < 2^192 = R, a Montgomery product of two such elements is again < 2m, so no final
// conditional subtraction is needed inside mul; add/sub re-normalise into [0, 2m) with
// one trial subtraction of 2m.  canon() maps [0, 2m) -> [0, m) for output and equality.
//
// Everything is __host__ __device__: the host path (plain C, 64-bit words) is what the
// CPU self-tests and the host-side pairing verifier use; the device path uses PTX.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define TC_HD __host__ __device__ __forceinline__
#define TC_D __device__ __forceinline__
#else
#define TC_HD inline
#define TC_D inline
#endif

namespace tc {

struct Fe {
  uint32_t v[6];
};

// --- field parameter packs -------------------------------------------------------------
struct FpParams {   // scalar field F_p (field.py PrimeField(backend.order))
  static constexpr uint32_t M0 = 0x01000001u, M5 = 0x2u;
  static constexpr uint32_t NP = 0x00ffffffu;         // -p^{-1} mod 2^32
  // R mod p and R^2 mod p (R = 2^192)
  static constexpr uint32_t ONE0 = 0x81000001u, ONE1 = 0xff7fffffu, ONE2 = 0xffffffffu,
                            ONE3 = 0xffffffffu, ONE4 = 0xffffffffu, ONE5 = 0x1u;
  static constexpr uint32_t R20 = 0x0u, R21 = 0x40000000u, R22 = 0x800000u, R23 = 0x4000u,
                            R24 = 0x0u, R25 = 0x0u;
};
struct FqParams {   // curve base field F_q
  static constexpr uint32_t M0 = 0x78000077u, M5 = 0xF0u;
  static constexpr uint32_t NP = 0xb10226b9u;         // -q^{-1} mod 2^32
  static constexpr uint32_t ONE0 = 0x89111119u, ONE1 = 0xff7fffffu, ONE2 = 0xffffffffu,
                            ONE3 = 0xffffffffu, ONE4 = 0xffffffffu, ONE5 = 0xfu;
  static constexpr uint32_t R20 = 0xc70123b5u, R21 = 0x3ef01234u, R22 = 0x11900000u,
                            R23 = 0x11115111u, R24 = 0x11111111u, R25 = 0xe1u;
};

template <class PM>
struct Field {
  // ---- constants ----
  TC_HD static Fe zero() { return Fe{{0, 0, 0, 0, 0, 0}}; }
  TC_HD static Fe one() { return Fe{{PM::ONE0, PM::ONE1, PM::ONE2, PM::ONE3, PM::ONE4, PM::ONE5}}; }
  TC_HD static Fe r2() { return Fe{{PM::R20, PM::R21, PM::R22, PM::R23, PM::R24, PM::R25}}; }
  TC_HD static Fe modulus() { return Fe{{PM::M0, 0, 0, 0, 0, PM::M5}}; }

  // ---- 6-limb helpers (portable) ----
  // r = a - (k*m) where k*m has limbs [k*M0 lo.., 0,0,0, k*M5]; returns borrow
  TC_HD static uint32_t sub_km(Fe& r, const Fe& a, uint32_t km0, uint32_t km5) {
#if defined(__CUDA_ARCH__)
    uint32_t b;
    asm("sub.cc.u32  %0, %7, %13;\n\t"
        "subc.cc.u32 %1, %8, 0;\n\t"
        "subc.cc.u32 %2, %9, 0;\n\t"
        "subc.cc.u32 %3, %10, 0;\n\t"
        "subc.cc.u32 %4, %11, 0;\n\t"
        "subc.cc.u32 %5, %12, %14;\n\t"
        "subc.u32    %6, 0, 0;\n\t"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(b)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(km0), "r"(km5));
    return b & 1u;
#else
    uint64_t t = (uint64_t)a.v[0] - km0;
    r.v[0] = (uint32_t)t;
    uint32_t br = (uint32_t)(t >> 63);
    for (int i = 1; i < 5; i++) {
      t = (uint64_t)a.v[i] - br;
      r.v[i] = (uint32_t)t;
      br = (uint32_t)(t >> 63);
    }
    t = (uint64_t)a.v[5] - km5 - br;
    r.v[5] = (uint32_t)t;
    return (uint32_t)(t >> 63);
#endif
  }

  TC_HD static Fe select(bool c, const Fe& a, const Fe& b) {
    Fe r;
#pragma unroll
    for (int i = 0; i < 6; i++) r.v[i] = c ? a.v[i] : b.v[i];
    return r;
  }

  // [0, 4m) -> [0, 2m)
  TC_HD static Fe red2(const Fe& a) {
    Fe t;
    uint32_t br = sub_km(t, a, 2u * PM::M0, 2u * PM::M5);
    return select(br != 0, a, t);
  }
  // [0, 2m) -> [0, m)
  TC_HD static Fe canon(const Fe& a) {
    Fe t;
    uint32_t br = sub_km(t, a, PM::M0, PM::M5);
    return select(br != 0, a, t);
  }

  TC_HD static Fe add(const Fe& a, const Fe& b) {
    Fe r;
#if defined(__CUDA_ARCH__)
    asm("add.cc.u32  %0, %6, %12;\n\t"
        "addc.cc.u32 %1, %7, %13;\n\t"
        "addc.cc.u32 %2, %8, %14;\n\t"
        "addc.cc.u32 %3, %9, %15;\n\t"
        "addc.cc.u32 %4, %10, %16;\n\t"
        "addc.u32    %5, %11, %17;\n\t"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]));
#else
    uint64_t c = 0;
    for (int i = 0; i < 6; i++) {
      c += (uint64_t)a.v[i] + b.v[i];
      r.v[i] = (uint32_t)c;
      c >>= 32;
    }
#endif
    return red2(r);
  }

  TC_HD static Fe sub(const Fe& a, const Fe& b) {
    Fe r;
    uint32_t br;
#if defined(__CUDA_ARCH__)
    asm("sub.cc.u32  %0, %7, %13;\n\t"
        "subc.cc.u32 %1, %8, %14;\n\t"
        "subc.cc.u32 %2, %9, %15;\n\t"
        "subc.cc.u32 %3, %10, %16;\n\t"
        "subc.cc.u32 %4, %11, %17;\n\t"
        "subc.cc.u32 %5, %12, %18;\n\t"
        "subc.u32    %6, 0, 0;\n\t"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(br)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]));
    // if negative add 2m
    uint32_t k0 = br ? 2u * PM::M0 : 0u, k5 = br ? 2u * PM::M5 : 0u;
    asm("add.cc.u32  %0, %0, %6;\n\t"
        "addc.cc.u32 %1, %1, 0;\n\t"
        "addc.cc.u32 %2, %2, 0;\n\t"
        "addc.cc.u32 %3, %3, 0;\n\t"
        "addc.cc.u32 %4, %4, 0;\n\t"
        "addc.u32    %5, %5, %7;\n\t"
        : "+r"(r.v[0]), "+r"(r.v[1]), "+r"(r.v[2]), "+r"(r.v[3]), "+r"(r.v[4]), "+r"(r.v[5])
        : "r"(k0), "r"(k5));
#else
    uint64_t t = 0;
    br = 0;
    for (int i = 0; i < 6; i++) {
      t = (uint64_t)a.v[i] - b.v[i] - br;
      r.v[i] = (uint32_t)t;
      br = (uint32_t)(t >> 63);
    }
    if (br) {
      uint64_t c = (uint64_t)r.v[0] + 2u * PM::M0;
      r.v[0] = (uint32_t)c;
      c >>= 32;
      for (int i = 1; i < 5; i++) {
        c += r.v[i];
        r.v[i] = (uint32_t)c;
        c >>= 32;
      }
      r.v[5] = (uint32_t)(c + r.v[5] + 2u * PM::M5);
    }
#endif
    return r;
  }

  TC_HD static Fe neg(const Fe& a) { return sub(zero(), a); }
  TC_HD static Fe dbl(const Fe& a) { return add(a, a); }

  // ---- Montgomery product ----
  // T[0..11] = a * b
  TC_HD static void mul_wide(uint32_t T[12], const Fe& a, const Fe& b) {
#if defined(__CUDA_ARCH__)
#pragma unroll
    for (int i = 0; i < 12; i++) T[i] = 0;
#pragma unroll
    for (int i = 0; i < 6; i++) {
      const uint32_t bi = b.v[i];
      asm("mad.lo.cc.u32  %0, %7, %10, %0;\n\t"
          "madc.hi.cc.u32 %1, %7, %10, %1;\n\t"
          "madc.lo.cc.u32 %2, %8, %10, %2;\n\t"
          "madc.hi.cc.u32 %3, %8, %10, %3;\n\t"
          "madc.lo.cc.u32 %4, %9, %10, %4;\n\t"
          "madc.hi.cc.u32 %5, %9, %10, %5;\n\t"
          "addc.u32       %6, %6, 0;\n\t"
          : "+r"(T[i + 0]), "+r"(T[i + 1]), "+r"(T[i + 2]), "+r"(T[i + 3]), "+r"(T[i + 4]),
            "+r"(T[i + 5]), "+r"(T[i + 6])
          : "r"(a.v[0]), "r"(a.v[2]), "r"(a.v[4]), "r"(bi));
      if (i < 5) {
        asm("mad.lo.cc.u32  %0, %7, %10, %0;\n\t"
            "madc.hi.cc.u32 %1, %7, %10, %1;\n\t"
            "madc.lo.cc.u32 %2, %8, %10, %2;\n\t"
            "madc.hi.cc.u32 %3, %8, %10, %3;\n\t"
            "madc.lo.cc.u32 %4, %9, %10, %4;\n\t"
            "madc.hi.cc.u32 %5, %9, %10, %5;\n\t"
            "addc.u32       %6, %6, 0;\n\t"
            : "+r"(T[i + 1]), "+r"(T[i + 2]), "+r"(T[i + 3]), "+r"(T[i + 4]), "+r"(T[i + 5]),
              "+r"(T[i + 6]), "+r"(T[(i + 7) < 12 ? (i + 7) : 11])
            : "r"(a.v[1]), "r"(a.v[3]), "r"(a.v[5]), "r"(bi));
      } else {
        asm("mad.lo.cc.u32  %0, %6, %9, %0;\n\t"
            "madc.hi.cc.u32 %1, %6, %9, %1;\n\t"
            "madc.lo.cc.u32 %2, %7, %9, %2;\n\t"
            "madc.hi.cc.u32 %3, %7, %9, %3;\n\t"
            "madc.lo.cc.u32 %4, %8, %9, %4;\n\t"
            "madc.hi.u32    %5, %8, %9, %5;\n\t"
            : "+r"(T[i + 1]), "+r"(T[i + 2]), "+r"(T[i + 3]), "+r"(T[i + 4]), "+r"(T[i + 5]),
              "+r"(T[i + 6])
            : "r"(a.v[1]), "r"(a.v[3]), "r"(a.v[5]), "r"(bi));
      }
    }
#else
    for (int i = 0; i < 12; i++) T[i] = 0;
    for (int i = 0; i < 6; i++) {
      uint64_t c = 0;
      for (int j = 0; j < 6; j++) {
        c += (uint64_t)a.v[j] * b.v[i] + T[i + j];
        T[i + j] = (uint32_t)c;
        c >>= 32;
      }
      T[i + 6] = (uint32_t)c;
    }
#endif
  }

  // Montgomery reduction of T (< m * R) exploiting limbs 1..4 of m being zero.
  TC_HD static Fe redc(const uint32_t T[12]) {
    uint32_t u[6];
    uint64_t s, carry = 0;
#pragma unroll
    for (int i = 0; i < 6; i++) {
      s = (uint64_t)T[i] + carry;
      if (i == 5) s += (uint64_t)u[0] * PM::M5;
      u[i] = (uint32_t)s * PM::NP;
      s += (uint64_t)u[i] * PM::M0;
      carry = s >> 32;
    }
    Fe r;
    s = (uint64_t)T[6] + carry + (uint64_t)u[1] * PM::M5;
    r.v[0] = (uint32_t)s;
    s = (s >> 32) + T[7] + (uint64_t)u[2] * PM::M5;
    r.v[1] = (uint32_t)s;
    s = (s >> 32) + T[8] + (uint64_t)u[3] * PM::M5;
    r.v[2] = (uint32_t)s;
    s = (s >> 32) + T[9] + (uint64_t)u[4] * PM::M5;
    r.v[3] = (uint32_t)s;
    s = (s >> 32) + T[10] + (uint64_t)u[5] * PM::M5;
    r.v[4] = (uint32_t)s;
    s = (s >> 32) + T[11];
    r.v[5] = (uint32_t)s;
    return r;
  }

  TC_HD static Fe mul(const Fe& a, const Fe& b) {
    uint32_t T[12];
    mul_wide(T, a, b);
    return redc(T);
  }
  TC_HD static Fe sqr(const Fe& a) { return mul(a, a); }

  // multiply by a small integer k < 2^20 (result < 2m): k*a < 2^20 * 2m, then reduce by
  // folding the top limb with one Montgomery-free trial loop.  Used for small node
  // constants (grid nodes 1..d) in interpolation / division.
  TC_HD static Fe mul_small(const Fe& a, uint32_t k) { return mul(a, to_mont_small(k)); }

  TC_HD static Fe to_mont_small(uint32_t k) {
    Fe t = zero();
    t.v[0] = k;
    return mul(t, r2());
  }

  TC_HD static bool is_zero(const Fe& a) {
    Fe c = canon(a);
    return (c.v[0] | c.v[1] | c.v[2] | c.v[3] | c.v[4] | c.v[5]) == 0;
  }
  TC_HD static bool eq(const Fe& a, const Fe& b) { return is_zero(sub(a, b)); }

  // canonical little-endian integer  <->  Montgomery form
  TC_HD static Fe to_mont(const Fe& x) { return mul(x, r2()); }
  TC_HD static Fe from_mont(const Fe& a) {
    uint32_t T[12] = {a.v[0], a.v[1], a.v[2], a.v[3], a.v[4], a.v[5], 0, 0, 0, 0, 0, 0};
    return canon(redc(T));
  }

  // a^(m-2) by left-to-right square and multiply over the fixed exponent
  TC_HD static Fe inv(const Fe& a) {
    // m - 2: limbs [M0 - 2, 0, 0, 0, 0, M5]
    Fe r = one();
    const uint32_t e[6] = {PM::M0 - 2u, 0, 0, 0, 0, PM::M5};
    bool started = false;
    for (int limb = 5; limb >= 0; limb--) {
      for (int bit = 31; bit >= 0; bit--) {
        if (started) r = sqr(r);
        if ((e[limb] >> bit) & 1u) {
          r = started ? mul(r, a) : a;
          started = true;
        }
      }
    }
    return r;
  }
};

using Fp = Field<FpParams>;
using Fq = Field<FqParams>;

}  // namespace tc
