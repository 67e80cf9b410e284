// SHA-256 (FIPS 180-4) for hash_to_scalar (backend.py:346-348):
//   int.from_bytes(sha256(b"tc/h2f/" + tag + b"/" + data), "little") mod p
// Used for Terkle child values.  __host__ __device__, short messages only.
#pragma once
#include <cstdint>
#include <cstring>

#include "ec.cuh"

namespace tc {

#define TC_SHA256_K                                                                                           \
  {0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,     \
   0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,     \
   0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,     \
   0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,     \
   0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,     \
   0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,     \
   0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,     \
   0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u}
#if defined(__CUDACC__)
static __constant__ uint32_t sha256_k[64] = TC_SHA256_K;
#endif
inline const uint32_t* sha256_k_host() {
  static const uint32_t k[64] = TC_SHA256_K;
  return k;
}

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

  // round constants: __constant__ on the device (uniform loads), a static table on the host
  TC_HD static uint32_t K(int i) {
#if defined(__CUDA_ARCH__)
    return sha256_k[i];
#else
    return sha256_k_host()[i];
#endif
  }

  // one compression; fully unrolled so the 16-word message window stays in registers
  TC_HD void block(const uint8_t* p) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; i++)
      w[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) | ((uint32_t)p[4 * i + 2] << 8) | p[4 * i + 3];
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    // 4 passes of 16 unrolled rounds: message-window indices stay compile-time (registers)
    // while the code is reused (the latency-bound tail kernels run it once per launch,
    // straight-line code would miss the instruction cache on every line)
#pragma unroll 1
    for (int r = 0; r < 64; r += 16) {
#pragma unroll
      for (int j = 0; j < 16; j++) {
        if (r) {
          const uint32_t x15 = w[(j + 1) & 15], x2 = w[(j + 14) & 15];
          const uint32_t s0 = rotr(x15, 7) ^ rotr(x15, 18) ^ (x15 >> 3);
          const uint32_t s1 = rotr(x2, 17) ^ rotr(x2, 19) ^ (x2 >> 10);
          w[j] += s0 + w[(j + 9) & 15] + s1;
        }
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + S1 + ch + K(r + j) + w[j];
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = S0 + mj;
        hh = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + t2;
      }
    }
    h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += hh;
  }

  // one compression over 16 big-endian message words already in registers
  TC_HD void block_words(const uint32_t* m) {
    uint8_t p[64];
#pragma unroll
    for (int i = 0; i < 16; i++)
      p[4 * i] = (uint8_t)(m[i] >> 24), p[4 * i + 1] = (uint8_t)(m[i] >> 16), p[4 * i + 2] = (uint8_t)(m[i] >> 8),
      p[4 * i + 3] = (uint8_t)m[i];
    block(p);
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

// hash_to_scalar(encode_elem(P), tag) for the Terkle tags b"terkle/leaf" / b"terkle/node"
// (backend.py:309-317, 346-348) with the 62-byte message
// "tc/h2f/" || tag || "/" || (0x04 || x LE21 || y LE21) and its SHA-256 padding assembled
// as 32 words at compile-time byte positions (registers, no byte buffer), two compressions.
TC_HD Fe hash_point_to_scalar(const Aff& P, bool node) {
  uint32_t xc[6], yc[6];
  bool inf;
  aff_to_canonical(P, xc, yc, &inf);
  const char* pre = "tc/h2f/terkle/";
  uint32_t m[32];
#pragma unroll
  for (int wd = 0; wd < 32; wd++) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int i = 4 * wd + b;
      uint32_t byte;
      if (i < 14) {
        byte = (uint8_t)pre[i];
      } else if (i < 18) {
        byte = (uint8_t)(node ? "node"[i - 14] : "leaf"[i - 14]);
      } else if (i == 18) {
        byte = '/';
      } else if (i == 19) {
        byte = inf ? 0u : 4u;
      } else if (i < 41) {
        const int k = i - 20;
        byte = inf ? 0u : (xc[k >> 2] >> (8 * (k & 3))) & 0xffu;
      } else if (i < 62) {
        const int k = i - 41;
        byte = inf ? 0u : (yc[k >> 2] >> (8 * (k & 3))) & 0xffu;
      } else if (i == 62) {
        byte = 0x80u;
      } else if (i < 120) {
        byte = 0u;
      } else {
        byte = (uint32_t)((62ull * 8ull >> (8 * (127 - i))) & 0xffu);   // message length in bits, big-endian
      }
      v = (v << 8) | byte;
    }
    m[wd] = v;
  }
  Sha256 s;
  s.init();
  s.block_words(m);
  s.block_words(m + 16);
  // the digest as a little-endian 256-bit integer: byte-swap the big-endian state words
  Fe lo, hi;
  auto bswap = [](uint32_t x) { return (x >> 24) | ((x >> 8) & 0xff00u) | ((x << 8) & 0xff0000u) | (x << 24); };
#pragma unroll
  for (int i = 0; i < 6; i++) lo.v[i] = bswap(s.h[i]);
  hi.v[0] = bswap(s.h[6]);
  hi.v[1] = bswap(s.h[7]);
#pragma unroll
  for (int i = 2; i < 6; i++) hi.v[i] = 0;
  const Fe a = Fp::to_mont(lo);
  const Fe b = Fp::mul(Fp::to_mont(hi), Fp::r2());
  return Fp::from_mont(Fp::add(Fp::red2(a), Fp::red2(b)));
}

}  // namespace tc
