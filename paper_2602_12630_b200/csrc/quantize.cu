// K1: quantise real activations into F_p (protocol.quantize, scale 2^16
// SPEC.md:605):  q = round-half-even(v * 2^k); q < 0 -> p - |q|; error when v is not
// finite or |v| * 2^k >= p/2.
//
// The rounding works on the exact binary value (quant.cuh), so fp32 inputs up to 2^128 and
// fp64 inputs of any magnitude quantise exactly like the oracle's arbitrary-precision
// restatement.  HBM-bound: 2-8 B read + 24 B written per element.  (The commit path does
// not call this kernel: the MSM digit kernel fuses the same quantisation into its load.)
#include "quant.cuh"
#include "tc_internal.cuh"

using namespace tc;

namespace {

template <int DT>
__global__ void k_quantize(const void* in, uint64_t n, int scale_bits, Fe* out, uint32_t* flags) {
  uint32_t f = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Fe mag;
    bool neg;
    quantize_signed<DT>(in, i, scale_bits, mag, neg, f);
    Fe q = signed_to_fp(mag, neg);
    uint2* o2 = (uint2*)(out + i);
    o2[0] = make_uint2(q.v[0], q.v[1]);
    o2[1] = make_uint2(q.v[2], q.v[3]);
    o2[2] = make_uint2(q.v[4], q.v[5]);
  }
  if (f) atomicOr(flags, f);
}

}  // namespace

namespace tcrt {

int quantize_flags_to_status(tc_ctx* ctx, uint32_t f) {
  if (f & QF_NONFINITE) return fail(ctx, TC_ERR_VALUE, "quantize: non-finite value");
  if (f & QF_OVERFLOW) return fail(ctx, TC_ERR_VALUE, "quantize: value overflows the field half-range");
  return TC_OK;
}

int quantize_device(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits, Fe* d_out) {
  if (scale_bits < 0 || scale_bits > 160) return fail(ctx, TC_ERR_VALUE, "quantize: scale_bits out of range");
  cudaStream_t st = ctx->stream;
  TC_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, sizeof(uint32_t), st));
  if (n) {
    unsigned grid = std::min<unsigned>(blocks_for(n, 256), (unsigned)ctx->num_sms * 16);
    switch (dtype) {
      case TC_DTYPE_F16: k_quantize<1><<<grid, 256, 0, st>>>(d_in, n, scale_bits, d_out, ctx->d_flags); break;
      case TC_DTYPE_BF16: k_quantize<2><<<grid, 256, 0, st>>>(d_in, n, scale_bits, d_out, ctx->d_flags); break;
      case TC_DTYPE_F32: k_quantize<3><<<grid, 256, 0, st>>>(d_in, n, scale_bits, d_out, ctx->d_flags); break;
      case TC_DTYPE_F64: k_quantize<4><<<grid, 256, 0, st>>>(d_in, n, scale_bits, d_out, ctx->d_flags); break;
      default: return fail(ctx, TC_ERR_ARGUMENT, "quantize: unsupported dtype %d", dtype);
    }
    TC_LAUNCHED(ctx);
  }
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return quantize_flags_to_status(ctx, ctx->h_flags[0]);
}

}  // namespace tcrt
