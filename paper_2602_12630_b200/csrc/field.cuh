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

#if defined(__CUDACC__)
// Modulus constants for the device reduction, read from the constant bank.  Kept out of
// immediates on purpose: with visible constants ptxas proves lo(u*M0 + s) = 0 and rewrites
// the full-rate IMAD.WIDE into half-rate IMAD.HI + carry fix-ups.
// [field][M0, M5, NP, pad]; field 0 = F_p, 1 = F_q
static __constant__ uint32_t tc_cmod[2][4] = {{0x01000001u, 0x2u, 0x00ffffffu, 0u},
                                              {0x78000077u, 0xF0u, 0xb10226b9u, 0u}};
#endif

// --- field parameter packs -------------------------------------------------------------
struct FpParams {   // scalar field F_p (field.py PrimeField(backend.order))
  static constexpr int IDX = 0;
  static constexpr uint32_t M0 = 0x01000001u, M5 = 0x2u;
  static constexpr uint32_t NP = 0x00ffffffu;         // -p^{-1} mod 2^32
  static constexpr uint64_t NP64 = 0xffff000000ffffffull;   // -p^{-1} mod 2^64 (host 64-bit path)
  // R mod p and R^2 mod p (R = 2^192)
  static constexpr uint32_t ONE0 = 0x81000001u, ONE1 = 0xff7fffffu, ONE2 = 0xffffffffu,
                            ONE3 = 0xffffffffu, ONE4 = 0xffffffffu, ONE5 = 0x1u;
  static constexpr uint32_t R20 = 0x0u, R21 = 0x40000000u, R22 = 0x800000u, R23 = 0x4000u,
                            R24 = 0x0u, R25 = 0x0u;
  // 8 p^2 limbs 0..11 (the non-zero ones) for lazy reduction
  static constexpr uint32_t K0 = 0x10000008u, K1 = 0x80000u, K2 = 0x0u, K5 = 0x20000020u, K6 = 0x0u, K10 = 0x20u;
  // R^3 mod p (binary-inversion result -> Montgomery form)
  static constexpr uint32_t R30 = 0x11000011u, R31 = 0x0u, R32 = 0xe0000000u, R33 = 0xff9fffffu,
                            R34 = 0xffff9fffu, R35 = 0x1u;
};
struct FqParams {   // curve base field F_q
  static constexpr int IDX = 1;
  static constexpr uint32_t M0 = 0x78000077u, M5 = 0xF0u;
  static constexpr uint32_t NP = 0xb10226b9u;         // -q^{-1} mod 2^32
  static constexpr uint64_t NP64 = 0x9a42bf71b10226b9ull;   // -q^{-1} mod 2^64 (host 64-bit path)
  static constexpr uint32_t ONE0 = 0x89111119u, ONE1 = 0xff7fffffu, ONE2 = 0xffffffffu,
                            ONE3 = 0xffffffffu, ONE4 = 0xffffffffu, ONE5 = 0xfu;
  static constexpr uint32_t R20 = 0xc70123b5u, R21 = 0x3ef01234u, R22 = 0x11900000u,
                            R23 = 0x11115111u, R24 = 0x11111111u, R25 = 0xe1u;
  // 8 q^2 limbs 0..11 (the non-zero ones) for lazy reduction
  static constexpr uint32_t K0 = 0x8001ba88u, K1 = 0xc200037cu, K2 = 0x1u, K5 = 0x6f900u, K6 = 0x708u, K10 = 0x70800u;
  static constexpr uint32_t R30 = 0x07d3b44au, R31 = 0x148e4c4fu, R32 = 0xd7b0eddfu, R33 = 0xbc809907u,
                            R34 = 0x67894c9au, R35 = 0xc5u;
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
#if defined(__CUDA_ARCH__)
  // (r0..r5) += x0*b, x1*b, x2*b as three 64-bit register pairs in one carry chain, carry
  // out added into c.  ptxas fuses each mad.lo.cc/madc.hi.cc pair into one
  // IMAD.WIDE.U32(.X) on an aligned register pair.
  TC_D static void chain3(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t& r4, uint32_t& r5,
                          uint32_t& c, uint32_t x0, uint32_t x1, uint32_t x2, uint32_t b) {
    asm("mad.lo.cc.u32  %0, %7, %10, %0;\n\t"
        "madc.hi.cc.u32 %1, %7, %10, %1;\n\t"
        "madc.lo.cc.u32 %2, %8, %10, %2;\n\t"
        "madc.hi.cc.u32 %3, %8, %10, %3;\n\t"
        "madc.lo.cc.u32 %4, %9, %10, %4;\n\t"
        "madc.hi.cc.u32 %5, %9, %10, %5;\n\t"
        "addc.u32       %6, %6, 0;\n\t"
        : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3), "+r"(r4), "+r"(r5), "+r"(c)
        : "r"(x0), "r"(x1), "r"(x2), "r"(b));
  }
  TC_D static void chain3_last(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t& r4, uint32_t& r5,
                               uint32_t x0, uint32_t x1, uint32_t x2, uint32_t b) {
    asm("mad.lo.cc.u32  %0, %6, %9, %0;\n\t"
        "madc.hi.cc.u32 %1, %6, %9, %1;\n\t"
        "madc.lo.cc.u32 %2, %7, %9, %2;\n\t"
        "madc.hi.cc.u32 %3, %7, %9, %3;\n\t"
        "madc.lo.cc.u32 %4, %8, %9, %4;\n\t"
        "madc.hi.u32    %5, %8, %9, %5;\n\t"
        : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3), "+r"(r4), "+r"(r5)
        : "r"(x0), "r"(x1), "r"(x2), "r"(b));
  }
  TC_D static void chain2(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t& c, uint32_t x0,
                          uint32_t x1, uint32_t b) {
    asm("mad.lo.cc.u32  %0, %5, %7, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %7, %1;\n\t"
        "madc.lo.cc.u32 %2, %6, %7, %2;\n\t"
        "madc.hi.cc.u32 %3, %6, %7, %3;\n\t"
        "addc.u32       %4, %4, 0;\n\t"
        : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3), "+r"(c)
        : "r"(x0), "r"(x1), "r"(b));
  }
  TC_D static void chain1(uint32_t& r0, uint32_t& r1, uint32_t& c, uint32_t x0, uint32_t b) {
    asm("mad.lo.cc.u32  %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32       %2, %2, 0;\n\t"
        : "+r"(r0), "+r"(r1), "+r"(c)
        : "r"(x0), "r"(b));
  }
  TC_D static uint64_t madwide(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
    return r;
  }
#endif

#if defined(__CUDA_ARCH__)
  // T = ev + od * 2^32 (the even / odd partial-product accumulators of mul_wide)
  TC_D static void merge_eo(uint32_t T[12], const uint32_t ev[12], const uint32_t od[12]) {
    T[0] = ev[0];
    asm("add.cc.u32  %0, %11, %22;\n\t"
        "addc.cc.u32 %1, %12, %23;\n\t"
        "addc.cc.u32 %2, %13, %24;\n\t"
        "addc.cc.u32 %3, %14, %25;\n\t"
        "addc.cc.u32 %4, %15, %26;\n\t"
        "addc.cc.u32 %5, %16, %27;\n\t"
        "addc.cc.u32 %6, %17, %28;\n\t"
        "addc.cc.u32 %7, %18, %29;\n\t"
        "addc.cc.u32 %8, %19, %30;\n\t"
        "addc.cc.u32 %9, %20, %31;\n\t"
        "addc.u32    %10, %21, %32;\n\t"
        : "=r"(T[1]), "=r"(T[2]), "=r"(T[3]), "=r"(T[4]), "=r"(T[5]), "=r"(T[6]), "=r"(T[7]), "=r"(T[8]),
          "=r"(T[9]), "=r"(T[10]), "=r"(T[11])
        : "r"(ev[1]), "r"(ev[2]), "r"(ev[3]), "r"(ev[4]), "r"(ev[5]), "r"(ev[6]), "r"(ev[7]), "r"(ev[8]),
          "r"(ev[9]), "r"(ev[10]), "r"(ev[11]), "r"(od[0]), "r"(od[1]), "r"(od[2]), "r"(od[3]), "r"(od[4]),
          "r"(od[5]), "r"(od[6]), "r"(od[7]), "r"(od[8]), "r"(od[9]), "r"(od[10]));
  }
#endif

  // T[0..11] = a * b
#if defined(__CUDA_ARCH__)
  // operand scanning, one row per limb of b: two 7-limb carry chains per row
  TC_D static void mul_wide_rows(uint32_t T[12], const Fe& a, const Fe& b) {
#pragma unroll
    for (int i = 0; i < 12; i++) T[i] = 0;
#pragma unroll
    for (int i = 0; i < 6; i++) {
      const uint32_t bi = b.v[i];
      chain3(T[i + 0], T[i + 1], T[i + 2], T[i + 3], T[i + 4], T[i + 5], T[i + 6], a.v[0], a.v[2], a.v[4], bi);
      if (i < 5)
        chain3(T[i + 1], T[i + 2], T[i + 3], T[i + 4], T[i + 5], T[i + 6], T[i + 7], a.v[1], a.v[3], a.v[5], bi);
      else
        chain3_last(T[i + 1], T[i + 2], T[i + 3], T[i + 4], T[i + 5], T[i + 6], a.v[1], a.v[3], a.v[5], bi);
    }
  }
#endif

#ifndef TC_MULV
// 0: even/odd pair accumulators (every IMAD.WIDE on an aligned pair, no realigning moves),
// 1: operand-scanning rows.  Row form was faster with XYZZ; with the Edwards adds the
// even/odd form wins (k_accum_aff 5.98 -> 5.83 ms, config-3 step 10.14 -> 9.89 ms)
#define TC_MULV 0
#endif
#ifndef TC_E_H1_2ARR
#define TC_E_H1_2ARR 0
#endif
#ifndef TC_SQRV
#define TC_SQRV 1   // 0: square through the generic product, 1: dedicated 21-product square (3% faster accumulation)
#endif

  TC_HD static void mul_wide(uint32_t T[12], const Fe& a, const Fe& b) {
#if defined(__CUDA_ARCH__) && TC_MULV == 1
    mul_wide_rows(T, a, b);
#elif defined(__CUDA_ARCH__)
    // Even/odd split: ev[t] collects products whose 64-bit pair starts at even position t,
    // od[t] those starting at odd position t+1 (od is shifted by one limb), so every
    // partial product is one IMAD.WIDE into an aligned register pair with no MOVs.
    uint32_t ev[12], od[12];
#pragma unroll
    for (int i = 0; i < 12; i++) ev[i] = od[i] = 0;
    const uint32_t a0 = a.v[0], a1 = a.v[1], a2 = a.v[2], a3 = a.v[3], a4 = a.v[4], a5 = a.v[5];
    // row 0
    chain3(ev[0], ev[1], ev[2], ev[3], ev[4], ev[5], ev[6], a0, a2, a4, b.v[0]);
    chain3(od[0], od[1], od[2], od[3], od[4], od[5], od[6], a1, a3, a5, b.v[0]);
    // row 1
    chain3(ev[2], ev[3], ev[4], ev[5], ev[6], ev[7], ev[8], a1, a3, a5, b.v[1]);
    chain3(od[0], od[1], od[2], od[3], od[4], od[5], od[6], a0, a2, a4, b.v[1]);
    // row 2
    chain3(ev[2], ev[3], ev[4], ev[5], ev[6], ev[7], ev[8], a0, a2, a4, b.v[2]);
    chain3(od[2], od[3], od[4], od[5], od[6], od[7], od[8], a1, a3, a5, b.v[2]);
    // row 3
    chain3(ev[4], ev[5], ev[6], ev[7], ev[8], ev[9], ev[10], a1, a3, a5, b.v[3]);
    chain3(od[2], od[3], od[4], od[5], od[6], od[7], od[8], a0, a2, a4, b.v[3]);
    // row 4
    chain3(ev[4], ev[5], ev[6], ev[7], ev[8], ev[9], ev[10], a0, a2, a4, b.v[4]);
    chain3(od[4], od[5], od[6], od[7], od[8], od[9], od[10], a1, a3, a5, b.v[4]);
    // row 5
    chain3_last(ev[6], ev[7], ev[8], ev[9], ev[10], ev[11], a1, a3, a5, b.v[5]);
    chain3(od[4], od[5], od[6], od[7], od[8], od[9], od[10], a0, a2, a4, b.v[5]);
    merge_eo(T, ev, od);
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
#ifndef TC_REDCV
#define TC_REDCV 0   // 0: plain C (ptxas picks IMAD.HI for the known-zero low halves), 1: explicit IMAD.WIDE
#endif
#if defined(__CUDA_ARCH__) && TC_REDCV == 1
    // word-serial: u_i = s_i * n' makes position i vanish; s carries into position i+1.
    // Every 32x32 product is one full-rate IMAD.WIDE (never the half-rate IMAD.HI).
    const uint32_t M0 = tc_cmod[PM::IDX][0], M5 = tc_cmod[PM::IDX][1], NP = tc_cmod[PM::IDX][2];
    uint32_t u[6];
    uint64_t s = T[0];
#pragma unroll
    for (int i = 0; i < 6; i++) {
      u[i] = (uint32_t)s * NP;
      s = madwide(u[i], M0, s) >> 32;
      if (i < 5) s += T[i + 1];
      if (i == 4) s = madwide(u[0], M5, s);   // u_0 * M5 lands on position 5
    }
    Fe r;
    s = madwide(u[1], M5, s + T[6]);
    r.v[0] = (uint32_t)s;
    s = madwide(u[2], M5, (s >> 32) + T[7]);
    r.v[1] = (uint32_t)s;
    s = madwide(u[3], M5, (s >> 32) + T[8]);
    r.v[2] = (uint32_t)s;
    s = madwide(u[4], M5, (s >> 32) + T[9]);
    r.v[3] = (uint32_t)s;
    s = madwide(u[5], M5, (s >> 32) + T[10]);
    r.v[4] = (uint32_t)s;
    r.v[5] = (uint32_t)(s >> 32) + T[11];
    return r;
#else
    uint32_t u[6];
    uint64_t s, carry = 0;
#pragma unroll
    for (int i = 0; i < 6; i++) {
      s = (uint64_t)T[i] + carry;
      if (i == 5) s += mul_m5(u[0]);
      u[i] = (uint32_t)s * PM::NP;
      s += (uint64_t)u[i] * PM::M0;
      carry = s >> 32;
    }
    Fe r;
    s = (uint64_t)T[6] + carry + mul_m5(u[1]);
    r.v[0] = (uint32_t)s;
    s = (s >> 32) + T[7] + mul_m5(u[2]);
    r.v[1] = (uint32_t)s;
    s = (s >> 32) + T[8] + mul_m5(u[3]);
    r.v[2] = (uint32_t)s;
    s = (s >> 32) + T[9] + mul_m5(u[4]);
    r.v[3] = (uint32_t)s;
    s = (s >> 32) + T[10] + mul_m5(u[5]);
    r.v[4] = (uint32_t)s;
    s = (s >> 32) + T[11];
    r.v[5] = (uint32_t)s;
    return r;
#endif
  }

  // u * M5 for the small top limb of the modulus (q: 0xF0 = 2^8 - 2^4, p: 2).  p's is a
  // shift.  q's: TC_REDC_SHIFT=1 forms 2^8 u - 2^4 u with 64-bit shifts (LEA + IMAD.SHL +
  // SHF), 0 (default) one IMAD.WIDE — which one schedules better depends on the rest of the
  // accumulation loop: shifts won with the earlier add orderings (k_accum_aff 4.03 -> 3.97 ms),
  // the product wins with the tuned mixed-add order (4.182 -> 4.164 ms per forward)
#ifndef TC_REDC_SHIFT
#define TC_REDC_SHIFT 0
#endif
  TC_HD static uint64_t mul_m5(uint32_t u) {
#if defined(__CUDA_ARCH__)
    if (PM::M5 == 2u) return (uint64_t)u << 1;
#if TC_REDC_SHIFT
    if (PM::M5 == 0xF0u) {
      uint64_t r;
      asm("{.reg .u64 a, b;\n\t"
          "cvt.u64.u32 a, %1;\n\t"
          "shl.b64 b, a, 8;\n\t"
          "shl.b64 a, a, 4;\n\t"
          "sub.u64 %0, b, a;}"
          : "=l"(r) : "r"(u));
      return r;
    }
#endif
#endif
    return (uint64_t)u * PM::M5;
  }

#if !defined(__CUDA_ARCH__) && defined(__SIZEOF_INT128__)
  // Host: the same Montgomery product (R = 2^192, lazy [0, 2m)) on 3 x 64-bit limbs with
  // 128-bit products — ~5x fewer multiplies than the 32-bit limb loops, for the CPU
  // verifier (pairings), opening weights and setup tables.
  static Fe mul_host64(const Fe& a, const Fe& b) {
    typedef unsigned __int128 u128;
    const uint64_t A[3] = {a.v[0] | (uint64_t)a.v[1] << 32, a.v[2] | (uint64_t)a.v[3] << 32,
                           a.v[4] | (uint64_t)a.v[5] << 32};
    const uint64_t B[3] = {b.v[0] | (uint64_t)b.v[1] << 32, b.v[2] | (uint64_t)b.v[3] << 32,
                           b.v[4] | (uint64_t)b.v[5] << 32};
    uint64_t t[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 3; i++) {
      uint64_t c = 0;
      for (int j = 0; j < 3; j++) {
        const u128 x = (u128)A[j] * B[i] + t[i + j] + c;
        t[i + j] = (uint64_t)x;
        c = (uint64_t)(x >> 64);
      }
      t[i + 3] = c;
    }
    // modulus in 64-bit limbs: m0 = M0, m1 = 0, m2 = M5 << 32
    const uint64_t m0 = PM::M0, m2 = (uint64_t)PM::M5 << 32;
    for (int i = 0; i < 3; i++) {
      const uint64_t u = t[i] * PM::NP64;
      u128 x = (u128)u * m0 + t[i];
      uint64_t c = (uint64_t)(x >> 64);
      x = (u128)t[i + 1] + c;
      t[i + 1] = (uint64_t)x;
      c = (uint64_t)(x >> 64);
      x = (u128)u * m2 + t[i + 2] + c;
      t[i + 2] = (uint64_t)x;
      c = (uint64_t)(x >> 64);
      for (int k = i + 3; k < 7 && c; k++) {
        x = (u128)t[k] + c;
        t[k] = (uint64_t)x;
        c = (uint64_t)(x >> 64);
      }
    }
    Fe r;
    for (int k = 0; k < 3; k++) r.v[2 * k] = (uint32_t)t[3 + k], r.v[2 * k + 1] = (uint32_t)(t[3 + k] >> 32);
    return r;
  }
#endif

  TC_HD static Fe mul(const Fe& a, const Fe& b) {
#if !defined(__CUDA_ARCH__) && defined(__SIZEOF_INT128__)
    return mul_host64(a, b);
#else
    uint32_t T[12];
    mul_wide(T, a, b);
    return redc(T);
#endif
  }

  // ---- 12-limb (unreduced product) arithmetic for lazy reduction --------------------------
  // r = a - b (a >= b as integers)
  TC_HD static void w12_sub(uint32_t r[12], const uint32_t a[12], const uint32_t b[12]) {
#if defined(__CUDA_ARCH__)
    asm("sub.cc.u32  %0, %12, %24;\n\t"
        "subc.cc.u32 %1, %13, %25;\n\t"
        "subc.cc.u32 %2, %14, %26;\n\t"
        "subc.cc.u32 %3, %15, %27;\n\t"
        "subc.cc.u32 %4, %16, %28;\n\t"
        "subc.cc.u32 %5, %17, %29;\n\t"
        "subc.cc.u32 %6, %18, %30;\n\t"
        "subc.cc.u32 %7, %19, %31;\n\t"
        "subc.cc.u32 %8, %20, %32;\n\t"
        "subc.cc.u32 %9, %21, %33;\n\t"
        "subc.cc.u32 %10, %22, %34;\n\t"
        "subc.u32    %11, %23, %35;\n\t"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(a[8]),
          "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]),
          "r"(b[6]), "r"(b[7]), "r"(b[8]), "r"(b[9]), "r"(b[10]), "r"(b[11]));
#else
    uint64_t br = 0;
    for (int i = 0; i < 12; i++) {
      const uint64_t t = (uint64_t)a[i] - b[i] - br;
      r[i] = (uint32_t)t;
      br = (t >> 63) & 1u;
    }
#endif
  }
  // r = a + K where K = 8 m^2 (a multiple of m: adding it leaves redc's result unchanged mod m)
  TC_HD static void w12_add_8mm(uint32_t r[12], const uint32_t a[12]) {
    const uint32_t K[12] = {PM::K0, PM::K1, PM::K2, 0, 0, PM::K5, PM::K6, 0, 0, 0, PM::K10, 0};
#if defined(__CUDA_ARCH__)
    asm("add.cc.u32  %0, %12, %24;\n\t"
        "addc.cc.u32 %1, %13, %25;\n\t"
        "addc.cc.u32 %2, %14, %26;\n\t"
        "addc.cc.u32 %3, %15, %27;\n\t"
        "addc.cc.u32 %4, %16, %28;\n\t"
        "addc.cc.u32 %5, %17, %29;\n\t"
        "addc.cc.u32 %6, %18, %30;\n\t"
        "addc.cc.u32 %7, %19, %31;\n\t"
        "addc.cc.u32 %8, %20, %32;\n\t"
        "addc.cc.u32 %9, %21, %33;\n\t"
        "addc.cc.u32 %10, %22, %34;\n\t"
        "addc.u32    %11, %23, %35;\n\t"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(a[8]),
          "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(K[0]), "r"(K[1]), "r"(K[2]), "r"(K[3]), "r"(K[4]), "r"(K[5]),
          "r"(K[6]), "r"(K[7]), "r"(K[8]), "r"(K[9]), "r"(K[10]), "r"(K[11]));
#else
    uint64_t c = 0;
    for (int i = 0; i < 12; i++) {
      c += (uint64_t)a[i] + K[i];
      r[i] = (uint32_t)c;
      c >>= 32;
    }
#endif
  }
  // Lazy pair for Edwards adds: with A = a1 b1, B = a2 b2 (unreduced) and P = (a1+a2)(b1+b2),
  //   E = P - A - B = a1 b2 + a2 b1 >= 0 (exact)  and  H = B - 2A + 8m^2 > 0,
  // both < 12 m^2 < m R, reduced ONCE each: 3 products, 2 reductions (instead of 3 + 3).
  // The sums must NOT be reduced: (a1 + a2 - 2m)(...) would make P - A - B negative.
  // a1 + a2 < 4m < 2^170 fits the 6 limbs; P < 16 m^2, P - A - B < 8 m^2.
  TC_HD static Fe add_raw(const Fe& a, const Fe& b) {
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
    return r;
  }
  // r = a + b (12 limbs, no overflow for the bounded products here)
  TC_HD static void w12_add(uint32_t r[12], const uint32_t a[12], const uint32_t b[12]) {
#if defined(__CUDA_ARCH__)
    asm("add.cc.u32  %0, %12, %24;\n\t"
        "addc.cc.u32 %1, %13, %25;\n\t"
        "addc.cc.u32 %2, %14, %26;\n\t"
        "addc.cc.u32 %3, %15, %27;\n\t"
        "addc.cc.u32 %4, %16, %28;\n\t"
        "addc.cc.u32 %5, %17, %29;\n\t"
        "addc.cc.u32 %6, %18, %30;\n\t"
        "addc.cc.u32 %7, %19, %31;\n\t"
        "addc.cc.u32 %8, %20, %32;\n\t"
        "addc.cc.u32 %9, %21, %33;\n\t"
        "addc.cc.u32 %10, %22, %34;\n\t"
        "addc.u32    %11, %23, %35;\n\t"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(a[8]),
          "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]),
          "r"(b[6]), "r"(b[7]), "r"(b[8]), "r"(b[9]), "r"(b[10]), "r"(b[11]));
#else
    uint64_t c = 0;
    for (int i = 0; i < 12; i++) {
      c += (uint64_t)a[i] + b[i];
      r[i] = (uint32_t)c;
      c >>= 32;
    }
#endif
  }
  // Lazy pair for the a = -1 Edwards adds (ec.cuh): A = (Y1 - X1)(y2 - x2) with the lazy
  // [0, 2m) differences, B = (Y1 + X1)(y2 + x2) with unreduced sums, then
  //   E = B - A + 8m^2 = 2 (X1 y2 + Y1 x2)  and  H = B + A = 2 (X1 x2 + Y1 y2)   (mod m),
  // 2 products and 2 reductions.  A < 4m^2, B < 16m^2 (sums < 4m): E < 24m^2, H < 20m^2 < m R.
  TC_HD static void lazy_e_h1(const Fe& X1, const Fe& Y1, const Fe& x2, const Fe& y2, Fe& E, Fe& H) {
#if TC_E_H1_2ARR
    // two 12-limb arrays: E_raw = B + 8m^2 - A in place, then H_raw = E_raw + 2A
    // (= B + A + 8m^2 < 28 m^2)
    uint32_t A[12], B[12];
    mul_wide(A, sub(Y1, X1), sub(y2, x2));
    mul_wide(B, add_raw(Y1, X1), add_raw(y2, x2));
    w12_add_8mm(B, B);
    w12_sub(B, B, A);
    E = redc(B);
    w12_add(A, A, A);
    w12_add(A, A, B);
    H = redc(A);
#else
    uint32_t A[12], B[12], T[12];
    mul_wide(A, sub(Y1, X1), sub(y2, x2));
    mul_wide(B, add_raw(Y1, X1), add_raw(y2, x2));
    w12_add(T, B, A);
    H = redc(T);
    w12_add_8mm(B, B);
    w12_sub(B, B, A);
    E = redc(B);
#endif
  }
  TC_HD static void lazy_e_h(const Fe& a1, const Fe& a2, const Fe& b1, const Fe& b2, Fe& E, Fe& H) {
    uint32_t A[12], B[12], P[12];
    mul_wide(A, a1, b1);
    mul_wide(B, a2, b2);
    mul_wide(P, add_raw(a1, a2), add_raw(b1, b2));
    w12_sub(P, P, A);
    w12_sub(P, P, B);
    E = redc(P);
    w12_add_8mm(B, B);
    w12_sub(B, B, A);
    w12_sub(B, B, A);
    H = redc(B);
  }

#if defined(__CUDA_ARCH__)
  // T = a^2: the 15 cross products once (even/odd pair chains), doubled, plus the 6
  // squares on the diagonal — 21 IMAD.WIDE instead of 36.
  TC_D static void sqr_wide(uint32_t T[12], const Fe& a) {
    uint32_t ev[12], od[12];
#pragma unroll
    for (int i = 0; i < 12; i++) ev[i] = od[i] = 0;
    const uint32_t a0 = a.v[0], a1 = a.v[1], a2 = a.v[2], a3 = a.v[3], a4 = a.v[4], a5 = a.v[5];
    chain3(od[0], od[1], od[2], od[3], od[4], od[5], od[6], a1, a3, a5, a0);   // pos 1,3,5
    chain2(ev[2], ev[3], ev[4], ev[5], ev[6], a2, a4, a0);                     // pos 2,4
    chain2(od[2], od[3], od[4], od[5], od[6], a2, a4, a1);                     // pos 3,5
    chain2(ev[4], ev[5], ev[6], ev[7], ev[8], a3, a5, a1);                     // pos 4,6
    chain2(od[4], od[5], od[6], od[7], od[8], a3, a5, a2);                     // pos 5,7
    chain1(ev[6], ev[7], ev[8], a4, a2);                                       // pos 6
    chain1(od[6], od[7], od[8], a4, a3);                                       // pos 7
    chain1(ev[8], ev[9], ev[10], a5, a3);                                      // pos 8
    chain1(od[8], od[9], od[10], a5, a4);                                      // pos 9
    // C = ev + od * 2^32 (positions 1..11), then 2C + diagonal
    uint32_t C[12];
    C[0] = 0;
    asm("add.cc.u32  %0, %11, %21;\n\t"
        "addc.cc.u32 %1, %12, %22;\n\t"
        "addc.cc.u32 %2, %13, %23;\n\t"
        "addc.cc.u32 %3, %14, %24;\n\t"
        "addc.cc.u32 %4, %15, %25;\n\t"
        "addc.cc.u32 %5, %16, %26;\n\t"
        "addc.cc.u32 %6, %17, %27;\n\t"
        "addc.cc.u32 %7, %18, %28;\n\t"
        "addc.cc.u32 %8, %19, %29;\n\t"
        "addc.cc.u32 %9, %20, %30;\n\t"
        "addc.u32    %10, 0, %31;\n\t"
        : "=r"(C[1]), "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]), "=r"(C[8]),
          "=r"(C[9]), "=r"(C[10]), "=r"(C[11])
        : "r"(ev[1]), "r"(ev[2]), "r"(ev[3]), "r"(ev[4]), "r"(ev[5]), "r"(ev[6]), "r"(ev[7]), "r"(ev[8]),
          "r"(ev[9]), "r"(ev[10]), "r"(od[0]), "r"(od[1]), "r"(od[2]), "r"(od[3]), "r"(od[4]), "r"(od[5]),
          "r"(od[6]), "r"(od[7]), "r"(od[8]), "r"(od[9]), "r"(od[10]));
#pragma unroll
    for (int i = 11; i > 0; i--) T[i] = __funnelshift_l(C[i - 1], C[i], 1);
    T[0] = 0;
    asm("mad.lo.cc.u32  %0, %12, %12, %0;\n\t"
        "madc.hi.cc.u32 %1, %12, %12, %1;\n\t"
        "madc.lo.cc.u32 %2, %13, %13, %2;\n\t"
        "madc.hi.cc.u32 %3, %13, %13, %3;\n\t"
        "madc.lo.cc.u32 %4, %14, %14, %4;\n\t"
        "madc.hi.cc.u32 %5, %14, %14, %5;\n\t"
        "madc.lo.cc.u32 %6, %15, %15, %6;\n\t"
        "madc.hi.cc.u32 %7, %15, %15, %7;\n\t"
        "madc.lo.cc.u32 %8, %16, %16, %8;\n\t"
        "madc.hi.cc.u32 %9, %16, %16, %9;\n\t"
        "madc.lo.cc.u32 %10, %17, %17, %10;\n\t"
        "madc.hi.u32    %11, %17, %17, %11;\n\t"
        : "+r"(T[0]), "+r"(T[1]), "+r"(T[2]), "+r"(T[3]), "+r"(T[4]), "+r"(T[5]), "+r"(T[6]), "+r"(T[7]),
          "+r"(T[8]), "+r"(T[9]), "+r"(T[10]), "+r"(T[11])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5));
  }
#endif

  TC_HD static Fe sqr(const Fe& a) {
#if defined(__CUDA_ARCH__) && TC_SQRV == 1
    uint32_t T[12];
    sqr_wide(T, a);
    return redc(T);
#else
    return mul(a, a);
#endif
  }

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

  // ---- binary extended Euclid ----------------------------------------------------------
  // ~2 x 168 iterations of 6-limb shifts / subtractions instead of the ~180 Montgomery
  // products of Fermat's a^(m-2).  Faster on the host (the CPU verifier, setup); on the
  // device it measured SLOWER than Fermat (k_final 95 -> 150 us: divergent data-dependent
  // loops), so device code keeps inv().  Variable time (public data only).
  // a (Montgomery, lazy) -> a^-1 (Montgomery).
  TC_HD static bool w_even(const Fe& a) { return (a.v[0] & 1u) == 0; }
  TC_HD static bool w_is_one(const Fe& a) { return a.v[0] == 1u && (a.v[1] | a.v[2] | a.v[3] | a.v[4] | a.v[5]) == 0; }
  TC_HD static void w_shr1(Fe& a) {
    for (int i = 0; i < 5; i++) a.v[i] = (a.v[i] >> 1) | (a.v[i + 1] << 31);
    a.v[5] >>= 1;
  }
  TC_HD static bool w_ge(const Fe& a, const Fe& b) {
    for (int i = 5; i >= 0; i--)
      if (a.v[i] != b.v[i]) return a.v[i] > b.v[i];
    return true;
  }
  TC_HD static void w_sub(Fe& a, const Fe& b) {   // a -= b, a >= b
    uint64_t br = 0;
    for (int i = 0; i < 6; i++) {
      const uint64_t t = (uint64_t)a.v[i] - b.v[i] - br;
      a.v[i] = (uint32_t)t;
      br = (t >> 63) & 1u;
    }
  }
  TC_HD static void w_add(Fe& a, const Fe& b) {   // a += b, no overflow of 192 bits
    uint64_t c = 0;
    for (int i = 0; i < 6; i++) {
      c += (uint64_t)a.v[i] + b.v[i];
      a.v[i] = (uint32_t)c;
      c >>= 32;
    }
  }
  // x / 2 mod m for x in [0, m)
  TC_HD static void w_half(Fe& x) {
    if (!w_even(x)) w_add(x, modulus());   // x + m < 2m < 2^192
    w_shr1(x);
  }
  // x - y mod m for x, y in [0, m)
  TC_HD static void w_subm(Fe& x, const Fe& y) {
    if (w_ge(x, y)) {
      w_sub(x, y);
    } else {
      w_add(x, modulus());
      w_sub(x, y);
    }
  }
  TC_HD static Fe inv_fast(const Fe& a_mont) {
    Fe u = canon(a_mont);
    if ((u.v[0] | u.v[1] | u.v[2] | u.v[3] | u.v[4] | u.v[5]) == 0) return zero();
    Fe v = modulus(), x1 = Fe{{1u, 0, 0, 0, 0, 0}}, x2 = zero();
    // invariants: x1 a = u, x2 a = v (mod m), u, v odd-reduced; gcd(u, v) = 1
    while (!w_is_one(u) && !w_is_one(v)) {
      while (w_even(u)) w_shr1(u), w_half(x1);
      while (w_even(v)) w_shr1(v), w_half(x2);
      if (w_ge(u, v)) {
        w_sub(u, v);
        w_subm(x1, x2);
      } else {
        w_sub(v, u);
        w_subm(x2, x1);
      }
    }
    // (aR)^-1 = a^-1 R^-1; times R^3 through one Montgomery product -> a^-1 R
    const Fe r3{{PM::R30, PM::R31, PM::R32, PM::R33, PM::R34, PM::R35}};
    return mul(w_is_one(u) ? x1 : x2, r3);
  }


  // ---- Bernstein-Yang "safegcd" inversion (variable-time divsteps, batches of 30 on
  // signed 30-bit limbs, after libsecp256k1's modinv32_var): ~13 batches of cheap 32-bit
  // steps + 6-limb matrix updates instead of Fermat's 167 dependent squarings — the
  // single-thread latency that sits on the commit / tree tail (ext_to_aff per MSM, per
  // Terkle node).  tools/tail_latency.cu measures both.
  TC_HD static void to30(const Fe& a, int32_t r[6]) {
    const uint32_t M = 0x3FFFFFFFu;
    r[0] = (int32_t)(a.v[0] & M);
    r[1] = (int32_t)(((a.v[0] >> 30) | (a.v[1] << 2)) & M);
    r[2] = (int32_t)(((a.v[1] >> 28) | (a.v[2] << 4)) & M);
    r[3] = (int32_t)(((a.v[2] >> 26) | (a.v[3] << 6)) & M);
    r[4] = (int32_t)(((a.v[3] >> 24) | (a.v[4] << 8)) & M);
    r[5] = (int32_t)((a.v[4] >> 22) | (a.v[5] << 10));   // < 2^28 for the moduli here
  }
  TC_HD static Fe from30(const int32_t r[6]) {   // limbs in [0, 2^30), value < 2^192
    const uint32_t a0 = (uint32_t)r[0], a1 = (uint32_t)r[1], a2 = (uint32_t)r[2], a3 = (uint32_t)r[3],
                   a4 = (uint32_t)r[4], a5 = (uint32_t)r[5];
    return Fe{{a0 | (a1 << 30), (a1 >> 2) | (a2 << 28), (a2 >> 4) | (a3 << 26), (a3 >> 6) | (a4 << 24),
               (a4 >> 8) | (a5 << 22), a5 >> 10}};
  }
  TC_HD static int ctz32(uint32_t x) {
#if defined(__CUDA_ARCH__)
    return __ffs((int)x) - 1;
#else
    return __builtin_ctz(x);
#endif
  }
  // 30 divsteps on the low words: transition matrix [u v; q r] (scaled by 2^30), new eta
  TC_HD static int32_t divsteps30(int32_t eta, uint32_t f0, uint32_t g0, int32_t& tu, int32_t& tv, int32_t& tq,
                                  int32_t& tr) {
    uint32_t u = 1, v = 0, q = 0, r = 1;
    uint32_t f = f0, g = g0;
    int i = 30;
    for (;;) {
      const int zeros = ctz32(g | (0xFFFFFFFFu << i));   // sentinel: count only up to i
      g >>= zeros;
      u <<= zeros;
      v <<= zeros;
      eta -= zeros;
      i -= zeros;
      if (i == 0) break;
      if (eta < 0) {   // swap (f, g), (u, q), (v, r); negate the old f, u, v
        uint32_t t;
        eta = -eta;
        t = f, f = g, g = 0u - t;
        t = u, u = q, q = 0u - t;
        t = v, v = r, r = 0u - t;
      }
      const int limit = (eta + 1) > i ? i : (eta + 1);
      const uint32_t m = (0xFFFFFFFFu >> (32 - limit)) & 255u;
      // -(f^-1) mod 256 by Newton's iteration (f odd: f * f = 1 mod 8)
      uint32_t y = f;
      y *= 2u - f * y;
      y *= 2u - f * y;
      const uint32_t w = (g * (0u - y)) & m;
      g += f * w;
      q += u * w;
      r += v * w;
    }
    tu = (int32_t)u, tv = (int32_t)v, tq = (int32_t)q, tr = (int32_t)r;
    return eta;
  }
  TC_HD static Fe inv_bygcd(const Fe& a_mont) {
    const Fe x = canon(a_mont);
    if ((x.v[0] | x.v[1] | x.v[2] | x.v[3] | x.v[4] | x.v[5]) == 0) return zero();
    const int32_t M30 = 0x3FFFFFFF;
    int32_t md[6], f[6], g[6], d[6] = {0, 0, 0, 0, 0, 0}, e[6] = {1, 0, 0, 0, 0, 0};
    to30(modulus(), md);
    to30(x, g);
    for (int i = 0; i < 6; i++) f[i] = md[i];
    const uint32_t minv30 = (0u - PM::NP) & 0x3FFFFFFFu;   // modulus^-1 mod 2^30
    int len = 6;
    int32_t eta = -1;
    for (;;) {
      int32_t u, v, q, r;
      eta = divsteps30(eta, (uint32_t)f[0], (uint32_t)g[0], u, v, q, r);
      {   // [d, e] <- t [d, e] / 2^30 mod m (d, e stay in (-2m, m))
        const int32_t sd = d[5] >> 31, se = e[5] >> 31;
        int32_t mdd = (u & sd) + (v & se), mee = (q & sd) + (r & se);
        int64_t cd = (int64_t)u * d[0] + (int64_t)v * e[0];
        int64_t ce = (int64_t)q * d[0] + (int64_t)r * e[0];
        mdd -= (int32_t)((minv30 * (uint32_t)cd + (uint32_t)mdd) & (uint32_t)M30);
        mee -= (int32_t)((minv30 * (uint32_t)ce + (uint32_t)mee) & (uint32_t)M30);
        cd += (int64_t)md[0] * mdd;
        ce += (int64_t)md[0] * mee;
        cd >>= 30;
        ce >>= 30;
        for (int i = 1; i < 6; i++) {
          cd += (int64_t)u * d[i] + (int64_t)v * e[i] + (int64_t)md[i] * mdd;
          ce += (int64_t)q * d[i] + (int64_t)r * e[i] + (int64_t)md[i] * mee;
          d[i - 1] = (int32_t)cd & M30;
          cd >>= 30;
          e[i - 1] = (int32_t)ce & M30;
          ce >>= 30;
        }
        d[5] = (int32_t)cd;
        e[5] = (int32_t)ce;
      }
      {   // [f, g] <- t [f, g] / 2^30 (exact)
        int64_t cf = (int64_t)u * f[0] + (int64_t)v * g[0];
        int64_t cg = (int64_t)q * f[0] + (int64_t)r * g[0];
        cf >>= 30;
        cg >>= 30;
        for (int i = 1; i < len; i++) {
          cf += (int64_t)u * f[i] + (int64_t)v * g[i];
          cg += (int64_t)q * f[i] + (int64_t)r * g[i];
          f[i - 1] = (int32_t)cf & M30;
          cf >>= 30;
          g[i - 1] = (int32_t)cg & M30;
          cg >>= 30;
        }
        f[len - 1] = (int32_t)cf;
        g[len - 1] = (int32_t)cg;
      }
      if (g[0] == 0) {
        int32_t c = 0;
        for (int j = 1; j < len; j++) c |= g[j];
        if (c == 0) break;
      }
      const int32_t fn = f[len - 1], gn = g[len - 1];
      int32_t c = (len - 2) >> 31;
      c |= fn ^ (fn >> 31);
      c |= gn ^ (gn >> 31);
      if (c == 0) {   // both top limbs 0 / -1: fold them into the limb below
        f[len - 2] = (int32_t)((uint32_t)f[len - 2] | ((uint32_t)fn << 30));
        g[len - 2] = (int32_t)((uint32_t)g[len - 2] | ((uint32_t)gn << 30));
        --len;
      }
    }
    // d = +-x^-1 in (-2m, m): fold in the sign of f (= +-1), bring to [0, m)
    {
      const int32_t add1 = d[5] >> 31, neg = f[len - 1] >> 31;
      for (int i = 0; i < 6; i++) d[i] += md[i] & add1;
      for (int i = 0; i < 6; i++) d[i] = (d[i] ^ neg) - neg;
      for (int i = 0; i < 5; i++) d[i + 1] += d[i] >> 30, d[i] &= M30;
      const int32_t add2 = d[5] >> 31;
      for (int i = 0; i < 6; i++) d[i] += md[i] & add2;
      for (int i = 0; i < 5; i++) d[i + 1] += d[i] >> 30, d[i] &= M30;
    }
    // (aR)^-1 = a^-1 R^-1; times R^3 through one Montgomery product -> a^-1 R
    const Fe r3{{PM::R30, PM::R31, PM::R32, PM::R33, PM::R34, PM::R35}};
    return mul(from30(d), r3);
  }

  // single-thread (latency-bound) inversions: safegcd on host and device (Fermat `inv`
  // stays for the batch kernels, where its branch-free schedule keeps warps converged)
  TC_HD static Fe inv_pref(const Fe& a) {
#if defined(__CUDA_ARCH__)
#ifndef TC_INV_FERMAT
    return inv_bygcd(a);
#else
    return inv(a);
#endif
#else
    return inv_bygcd(a);
#endif
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
