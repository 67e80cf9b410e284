// SHA-256 (FIPS 180-4) for hash_to_scalar (backend.py:346-348):
//   int.from_bytes(sha256(b"tc/h2f/" + tag + b"/" + data), "little") mod p
// Used for Terkle child values.  __host__ __device__, short messages only.
#pragma once
#include <cstdint>
#include <cstring>

#include "field.cuh"

namespace tc {

struct Sha256 {
  uint32_t h[8];
  uint8_t buf[64];
  uint32_t blen;
  uint64_t total;

  TC_HD static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

  TC_HD void init() {
    const uint32_t iv[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                            0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    for (int i = 0; i < 8; i++) h[i] = iv[i];
    blen = 0;
    total = 0;
  }

  TC_HD void block(const uint8_t* p) {
    const uint32_t K[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; i++)
      w[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) | ((uint32_t)p[4 * i + 2] << 8) | p[4 * i + 3];
    for (int i = 16; i < 64; i++) {
      uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; i++) {
      uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
      uint32_t ch = (e & f) ^ (~e & g);
      uint32_t t1 = hh + S1 + ch + K[i] + w[i];
      uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
      uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
      uint32_t t2 = S0 + mj;
      hh = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += hh;
  }

  TC_HD void update(const uint8_t* p, uint32_t n) {
    total += n;
    while (n) {
      uint32_t take = 64 - blen < n ? 64 - blen : n;
      for (uint32_t i = 0; i < take; i++) buf[blen + i] = p[i];
      blen += take;
      p += take;
      n -= take;
      if (blen == 64) {
        block(buf);
        blen = 0;
      }
    }
  }

  TC_HD void final(uint8_t out[32]) {
    uint64_t bits = total * 8;
    uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (blen != 56) update(&zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; i++) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    update(len, 8);
    for (int i = 0; i < 8; i++) {
      out[4 * i] = (uint8_t)(h[i] >> 24);
      out[4 * i + 1] = (uint8_t)(h[i] >> 16);
      out[4 * i + 2] = (uint8_t)(h[i] >> 8);
      out[4 * i + 3] = (uint8_t)h[i];
    }
  }
};

// hash_to_scalar(data, tag) -> canonical F_p (backend.py:346-348)
TC_HD Fe hash_to_scalar(const uint8_t* data, uint32_t n, const uint8_t* tag, uint32_t tn) {
  Sha256 s;
  s.init();
  const uint8_t pre[7] = {'t', 'c', '/', 'h', '2', 'f', '/'};
  const uint8_t slash = '/';
  s.update(pre, 7);
  s.update(tag, tn);
  s.update(&slash, 1);
  s.update(data, n);
  uint8_t dg[32];
  s.final(dg);
  // 256-bit little-endian integer mod p: x = lo + hi * 2^192 with hi < 2^64;
  // reduce via Montgomery: (x mod p) = redc(lo_part * R2) + redc(hi * 2^192 * R2) ...
  // simpler: x mod p = from_mont( to_mont(lo) + to_mont(hi) * (2^192 mod p in Montgomery) )
  Fe lo, hi;
  for (int i = 0; i < 6; i++)
    lo.v[i] = (uint32_t)dg[4 * i] | ((uint32_t)dg[4 * i + 1] << 8) | ((uint32_t)dg[4 * i + 2] << 16) |
              ((uint32_t)dg[4 * i + 3] << 24);
  hi.v[0] = (uint32_t)dg[24] | ((uint32_t)dg[25] << 8) | ((uint32_t)dg[26] << 16) | ((uint32_t)dg[27] << 24);
  hi.v[1] = (uint32_t)dg[28] | ((uint32_t)dg[29] << 8) | ((uint32_t)dg[30] << 16) | ((uint32_t)dg[31] << 24);
  for (int i = 2; i < 6; i++) hi.v[i] = 0;
  // lo may exceed 2p (it is < 2^192): to_mont handles any input < 2^192 since
  // lo * R2 < 2^192 * p < p * R.  2^192 mod p in Montgomery form is R2 (= R * R mod p).
  Fe a = Fp::to_mont(lo);
  Fe b = Fp::mul(Fp::to_mont(hi), Fp::r2());
  return Fp::from_mont(Fp::add(Fp::red2(a), Fp::red2(b)));
}

}  // namespace tc
