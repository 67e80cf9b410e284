// K1: quantise real activations into F_p (protocol.quantize, scale 2^16
// SPEC.md:605):  q = round-half-even(v * 2^k); q < 0 -> p - |q|; error when v is not
// finite or |v| * 2^k >= p/2.
//
// The rounding is done on the exact binary value (sign, exponent, integer mantissa), never
// through a float multiply, so fp32 inputs up to 2^128 and fp64 inputs of any magnitude
// quantise exactly like the oracle's arbitrary-precision restatement.  HBM-bound:
// 2-8 B read + 24 B written per element, grid-stride with vectorised 16 B stores.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr uint32_t QF_NONFINITE = 1u, QF_OVERFLOW = 2u;

struct Decoded {
  bool neg;
  bool nonfinite;
  uint64_t mant;   // integer mantissa (implicit bit included)
  int exp2;        // value = mant * 2^exp2
};

template <int DT>
__device__ __forceinline__ Decoded decode(const void* in, uint64_t i) {
  Decoded d;
  if (DT == TC_DTYPE_F16) {
    uint32_t b = ((const uint16_t*)in)[i];
    uint32_t e = (b >> 10) & 0x1f, m = b & 0x3ff;
    d.neg = b >> 15;
    d.nonfinite = (e == 0x1f);
    d.mant = e ? (m | 0x400u) : m;
    d.exp2 = (e ? (int)e : 1) - 25;
  } else if (DT == TC_DTYPE_BF16) {
    uint32_t b = ((const uint16_t*)in)[i];
    uint32_t e = (b >> 7) & 0xff, m = b & 0x7f;
    d.neg = b >> 15;
    d.nonfinite = (e == 0xff);
    d.mant = e ? (m | 0x80u) : m;
    d.exp2 = (e ? (int)e : 1) - 134;
  } else if (DT == TC_DTYPE_F32) {
    uint32_t b = ((const uint32_t*)in)[i];
    uint32_t e = (b >> 23) & 0xff, m = b & 0x7fffffu;
    d.neg = b >> 31;
    d.nonfinite = (e == 0xff);
    d.mant = e ? (m | 0x800000u) : m;
    d.exp2 = (e ? (int)e : 1) - 150;
  } else {   // F64
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

// |q| = RNE(mant * 2^sh) as 6 limbs; returns false when |q| >= (p+1)/2 (overflow)
__device__ __forceinline__ bool magnitude(uint64_t mant, int sh, Fe& q) {
  for (int i = 0; i < 6; i++) q.v[i] = 0;
  if (mant == 0) return true;
  if (sh < 0) {
    int s = -sh;
    if (s > 63) return true;   // < 2^53 / 2^64 < 1/2 -> 0
    uint64_t iq = mant >> s;
    uint64_t rem = mant & ((1ull << s) - 1ull);
    uint64_t half = 1ull << (s - 1);
    if (rem > half || (rem == half && (iq & 1ull))) iq++;
    q.v[0] = (uint32_t)iq;
    q.v[1] = (uint32_t)(iq >> 32);
    return true;
  }
  // mant < 2^53, |q| = mant << sh; overflow test against (p+1)/2 = 2^160 + 2^23 + 1
  int top = 64 - __clzll(mant) + sh;   // bit length of |q|
  if (top > 162) return false;
  int limb = sh >> 5, bit = sh & 31;
  // spread mant << bit across limbs [limb, limb+2]
  uint64_t lo = mant << bit;
  uint32_t hi = bit ? (uint32_t)(mant >> (64 - bit)) : 0u;
  if (limb < 6) q.v[limb] = (uint32_t)lo;
  if (limb + 1 < 6) q.v[limb + 1] = (uint32_t)(lo >> 32);
  if (limb + 2 < 6) q.v[limb + 2] = hi;
  // q >= 2^160 + 2^23 + 1 ?
  bool over = (q.v[5] > 1u) ||
              (q.v[5] == 1u && ((q.v[4] | q.v[3] | q.v[2] | q.v[1]) != 0u || q.v[0] >= 0x00800001u));
  return !over;
}

template <int DT>
__global__ void k_quantize(const void* in, uint64_t n, int scale_bits, Fe* out, uint32_t* flags) {
  uint32_t f = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Decoded d = decode<DT>(in, i);
    Fe q;
    if (d.nonfinite) {
      f |= QF_NONFINITE;
      q = Fe{{0, 0, 0, 0, 0, 0}};
    } else if (!magnitude(d.mant, d.exp2 + scale_bits, q)) {
      f |= QF_OVERFLOW;
      q = Fe{{0, 0, 0, 0, 0, 0}};
    } else if (d.neg && (q.v[0] | q.v[1] | q.v[2] | q.v[3] | q.v[4] | q.v[5])) {
      // p - |q|
      uint64_t t = (uint64_t)FpParams::M0 - q.v[0];
      uint32_t r0 = (uint32_t)t, br = (uint32_t)(t >> 63);
      Fe r;
      r.v[0] = r0;
#pragma unroll
      for (int k = 1; k < 5; k++) {
        t = 0ull - q.v[k] - br;
        r.v[k] = (uint32_t)t;
        br = (uint32_t)(t >> 63);
      }
      r.v[5] = FpParams::M5 - q.v[5] - br;
      q = r;
    }
    uint4* o = (uint4*)(out + i);   // 24 B element = 1.5 x uint4; write as 3 x uint2
    (void)o;
    uint2* o2 = (uint2*)(out + i);
    o2[0] = make_uint2(q.v[0], q.v[1]);
    o2[1] = make_uint2(q.v[2], q.v[3]);
    o2[2] = make_uint2(q.v[4], q.v[5]);
  }
  if (f) atomicOr(flags, f);
}

template <int DT>
__global__ void k_quantize_i64(const void* in, uint64_t n, int scale_bits, int64_t* out,
                               uint32_t* flags) {
  uint32_t f = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Decoded d = decode<DT>(in, i);
    Fe q;
    int64_t v = 0;
    if (d.nonfinite) {
      f |= QF_NONFINITE;
    } else if (!magnitude(d.mant, d.exp2 + scale_bits, q)) {
      f |= QF_OVERFLOW;
    } else if (q.v[2] | q.v[3] | q.v[4] | q.v[5] | (q.v[1] & 0x80000000u)) {
      f |= 4u;   // does not fit int64: caller must use the limb path
    } else {
      uint64_t u = ((uint64_t)q.v[1] << 32) | q.v[0];
      v = d.neg ? -(int64_t)u : (int64_t)u;
    }
    out[i] = v;
  }
  if (f) atomicOr(flags, f);
}

template <class K>
int launch_dtype(tc_ctx* ctx, int dtype, K&& k) {
  switch (dtype) {
    case TC_DTYPE_F16: return k(std::integral_constant<int, TC_DTYPE_F16>());
    case TC_DTYPE_BF16: return k(std::integral_constant<int, TC_DTYPE_BF16>());
    case TC_DTYPE_F32: return k(std::integral_constant<int, TC_DTYPE_F32>());
    case TC_DTYPE_F64: return k(std::integral_constant<int, TC_DTYPE_F64>());
    default: return tcrt::fail(ctx, TC_ERR_ARGUMENT, "quantize: unsupported dtype %d", dtype);
  }
}

int check_flags(tc_ctx* ctx) {
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  uint32_t f = ctx->h_flags[0];
  if (f & QF_NONFINITE) return tcrt::fail(ctx, TC_ERR_VALUE, "quantize: non-finite value");
  if (f & QF_OVERFLOW) return tcrt::fail(ctx, TC_ERR_VALUE, "quantize: value overflows the field half-range");
  if (f & 4u) return tcrt::fail(ctx, TC_ERR_OVERFLOW, "quantize: value does not fit int64");
  return TC_OK;
}

}  // namespace

namespace tcrt {

int quantize_device(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits, Fe* d_out) {
  if (scale_bits < 0 || scale_bits > 160) return fail(ctx, TC_ERR_VALUE, "quantize: scale_bits out of range");
  TC_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, sizeof(uint32_t), ctx->stream));
  if (n) {
    unsigned grid = std::min<unsigned>(blocks_for(n, 256), (unsigned)ctx->num_sms * 16);
    int s = launch_dtype(ctx, dtype, [&](auto dt) -> int {
      k_quantize<decltype(dt)::value><<<grid, 256, 0, ctx->stream>>>(d_in, n, scale_bits, d_out, ctx->d_flags);
      TC_LAUNCHED(ctx);
      return TC_OK;
    });
    if (s) return s;
  }
  return check_flags(ctx);
}

int quantize_i64_device(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits, int64_t* d_out) {
  if (scale_bits < 0 || scale_bits > 160) return fail(ctx, TC_ERR_VALUE, "quantize: scale_bits out of range");
  TC_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, sizeof(uint32_t), ctx->stream));
  if (n) {
    unsigned grid = std::min<unsigned>(blocks_for(n, 256), (unsigned)ctx->num_sms * 16);
    int s = launch_dtype(ctx, dtype, [&](auto dt) -> int {
      k_quantize_i64<decltype(dt)::value><<<grid, 256, 0, ctx->stream>>>(d_in, n, scale_bits, d_out, ctx->d_flags);
      TC_LAUNCHED(ctx);
      return TC_OK;
    });
    if (s) return s;
  }
  return check_flags(ctx);
}

}  // namespace tcrt
