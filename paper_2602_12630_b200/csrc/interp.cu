// K2 / K4: the polynomial side of the prover on the device.
//
// interpolate_device  — mvpoly.interpolate_lagrange (mvpoly.py:233-247): for each axis j the
//   d_j x d_j matrix B_j (column l = monomial coefficients of the l-th Lagrange basis
//   polynomial on nodes 1..d_j, mvpoly.py:193-218) is applied to every fibre along axis j
//   (mvpoly.py:168-186).  A block stages FB whole fibres in shared memory; each output
//   coefficient is a length-d_j dot product accumulated as full 384-bit products and
//   Montgomery-reduced ONCE (sum < 4 d p^2 < p R for d < 2^28), so a MAC costs the 6x6
//   product only.  B_j is kept in Montgomery form and the samples canonical, so the
//   reduction lands directly on canonical coefficients.
// open_quotients_device — mvpoly.open_quotients (mvpoly.py:521-534) built from
//   divide_by_linear (mvpoly.py:452-484): after dividing along axis a the remainder is
//   independent of X_0..X_a, i.e. supported on the lex prefix of length prod_{t>a} d_t, so
//   axis a only touches fibres of that prefix (one thread per fibre, synthetic division).
// evaluate_device — mvpoly.evaluate (mvpoly.py:140-161): per-axis Horner contraction.
#include "tc_internal.cuh"

using namespace tc;

namespace {

// acc[0..11] += a * b  (12-limb accumulator; callers keep the sum below 2^384)
__device__ __forceinline__ void mac_wide(uint32_t acc[12], const Fe& a, const Fe& b) {
  uint32_t T[12];
  Fp::mul_wide(T, a, b);
  asm("add.cc.u32  %0, %0, %12;\n\t"
      "addc.cc.u32 %1, %1, %13;\n\t"
      "addc.cc.u32 %2, %2, %14;\n\t"
      "addc.cc.u32 %3, %3, %15;\n\t"
      "addc.cc.u32 %4, %4, %16;\n\t"
      "addc.cc.u32 %5, %5, %17;\n\t"
      "addc.cc.u32 %6, %6, %18;\n\t"
      "addc.cc.u32 %7, %7, %19;\n\t"
      "addc.cc.u32 %8, %8, %20;\n\t"
      "addc.cc.u32 %9, %9, %21;\n\t"
      "addc.cc.u32 %10, %10, %22;\n\t"
      "addc.u32    %11, %11, %23;\n\t"
      : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),
        "+r"(acc[6]), "+r"(acc[7]), "+r"(acc[8]), "+r"(acc[9]), "+r"(acc[10]), "+r"(acc[11])
      : "r"(T[0]), "r"(T[1]), "r"(T[2]), "r"(T[3]), "r"(T[4]), "r"(T[5]), "r"(T[6]), "r"(T[7]),
        "r"(T[8]), "r"(T[9]), "r"(T[10]), "r"(T[11]));
}

__device__ __forceinline__ uint64_t fibre_addr(uint64_t f, uint32_t l, uint32_t d, uint64_t stride) {
  uint64_t o = f / stride, i = f - o * stride;
  return o * d * stride + (uint64_t)l * stride + i;
}

// one block = FB fibres along an axis with extent d and stride `stride`
__global__ void __launch_bounds__(256) k_interp_axis(Fe* data, const Fe* Bm, uint32_t d, uint64_t stride,
                                                     uint64_t nfib, uint32_t FB) {
  extern __shared__ Fe sh[];   // FB * d samples, fibre-major
  uint64_t f0 = (uint64_t)blockIdx.x * FB;
  uint32_t nloc = (nfib - f0 < FB) ? (uint32_t)(nfib - f0) : FB;
  uint32_t tot = nloc * d;
  const bool contiguous = (stride == 1);
  for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    uint32_t fl, l;
    if (contiguous) {
      fl = idx / d;
      l = idx - fl * d;
    } else {
      l = idx / nloc;
      fl = idx - l * nloc;
    }
    sh[fl * d + l] = data[fibre_addr(f0 + fl, l, d, stride)];
  }
  __syncthreads();
  for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    uint32_t fl, k;
    if (contiguous) {
      fl = idx / d;
      k = idx - fl * d;
    } else {
      k = idx / nloc;
      fl = idx - k * nloc;
    }
    uint32_t acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const Fe* v = sh + fl * d;
    for (uint32_t l = 0; l < d; l++) mac_wide(acc, v[l], Bm[(uint64_t)l * d + k]);
    Fe r = Fp::canon(Fp::redc(acc));
    // every sample of this block was staged before any write, fibres are disjoint
    data[fibre_addr(f0 + fl, k, d, stride)] = r;
  }
}

// divide the prefix-supported remainder r by (X_a - v) along axis a (extent d, stride s):
// fibres i in [0, s); q written at the same offsets; r keeps only its X_a^0 slice
__global__ void k_divide_axis(Fe* r, Fe* q, uint32_t d, uint64_t s, Fe v_mont) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= s) return;
  Fe carry = r[(uint64_t)(d - 1) * s + i];
  if (d > 1) r[(uint64_t)(d - 1) * s + i] = Fp::zero();
  for (int c = (int)d - 2; c >= 0; c--) {
    uint64_t pos = (uint64_t)c * s + i;
    q[pos] = Fp::canon(carry);
    carry = Fp::add(r[pos], Fp::mul(v_mont, carry));
    r[pos] = Fp::zero();
  }
  r[i] = Fp::canon(carry);
}

// Lagrange-route opening along the leading axis (extent d, `rest` trailing elements):
// rn[r] = sum_k r[k, r] lam[k];  q[k, r] = (r[k, r] - rn[r]) * inv[k]
__global__ void k_open_axis_lag(const Fe* r, uint32_t d, uint64_t rest, const Fe* lam, const Fe* inv, const Fe* der,
                                int sj, Fe* rn, Fe* q) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rest) return;
  uint32_t acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (uint32_t k = 0; k < d; k++) mac_wide(acc, r[(uint64_t)k * rest + i], lam[k]);
  const Fe next = Fp::canon(Fp::redc(acc));
  rn[i] = next;
  if (!q) return;   // caller commits this axis another way (slice-commitment openings)
  for (uint32_t k = 0; k < d; k++) {
    const uint64_t pos = (uint64_t)k * rest + i;
    if ((int)k == sj) {   // omega on the node x_k: derivative of the fibre interpolant
      uint32_t dacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (uint32_t t = 0; t < d; t++) mac_wide(dacc, r[(uint64_t)t * rest + i], der[t]);
      q[pos] = Fp::canon(Fp::redc(dacc));
    } else {
      q[pos] = Fp::canon(Fp::mul(Fp::sub(r[pos], next), inv[k]));
    }
  }
}

// Slice-commitment opening scalars (tc_open_batch): for opening o with axis-0 weights
// lam = L_c'(omega_0) and inv = 1/(c + 1 - omega_0) (Montgomery form, as k_open_axis_lag
// takes them; tabs[o] = lam[d] ++ inv[d]), s[o][c' d + c] = (delta_{c c'} - lam[c']) inv[c]
// (canonical out), so pi_0 = sum s * H[c', c].
__global__ void k_slice_scalars(const Fe* tabs, const int* sj, uint32_t d, uint32_t count, Fe* out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t dd = (uint64_t)d * d;
  if (t >= dd * count) return;
  const uint64_t o = t / dd;
  const uint32_t cp = (uint32_t)((t % dd) / d), c = (uint32_t)(t % d);
  const Fe* lam = tabs + o * 3 * d;
  const Fe* inv = lam + d;
  if ((int)c == sj[o]) {   // omega_0 on the node x_c: q_0 there is sum_c' der[c'] T[c', .]
    out[t] = Fp::from_mont(lam[2 * d + cp]);
    return;
  }
  const Fe x = Fp::sub(c == cp ? Fp::one() : Fp::zero(), lam[cp]);   // Montgomery
  out[t] = Fp::from_mont(Fp::mul(x, inv[c]));                        // canonical
}

// k_open_axis_lag for `cnt` openings in one launch: thread (o, i); opening o reads r_in[o]
// (device pointer table), its weights at tabs + o * tstride + {0, dsum, 2 dsum}, writes
// rn + o * rest and (unless q is null) q + o * qstride.  The per-opening kernels are
// latency-bound (d sequential MACs per thread); a group's openings now share the launch.
__global__ void k_open_axis_lag_b(const Fe* const* r_in, uint32_t d, uint64_t rest, const Fe* tabs, uint64_t tstride,
                                  uint32_t dsum, const int* sj, Fe* rn, Fe* q, uint64_t qstride, uint32_t cnt) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= rest * cnt) return;
  const uint32_t o = (uint32_t)(t / rest);
  const uint64_t i = t % rest;
  const Fe* r = r_in[o];
  const Fe* lam = tabs + o * tstride;
  const Fe* inv = lam + dsum;
  const Fe* der = lam + 2 * dsum;
  uint32_t acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (uint32_t k = 0; k < d; k++) mac_wide(acc, r[(uint64_t)k * rest + i], lam[k]);
  const Fe next = Fp::canon(Fp::redc(acc));
  rn[(uint64_t)o * rest + i] = next;
  if (!q) return;
  Fe* qo = q + o * qstride;
  const int s = sj[o];
  for (uint32_t k = 0; k < d; k++) {
    const uint64_t pos = (uint64_t)k * rest + i;
    if ((int)k == s) {
      uint32_t dacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (uint32_t u = 0; u < d; u++) mac_wide(dacc, r[(uint64_t)u * rest + i], der[u]);
      qo[pos] = Fp::canon(Fp::redc(dacc));
    } else {
      qo[pos] = Fp::canon(Fp::mul(Fp::sub(r[pos], next), inv[k]));
    }
  }
}

// out[rest] = sum_k c[k, rest] x^k  (Horner along the leading axis of extent d)
__global__ void k_horner_lead(const Fe* c, Fe* out, uint32_t d, uint64_t rest, Fe x_mont) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rest) return;
  Fe acc = c[(uint64_t)(d - 1) * rest + i];
  for (int k = (int)d - 2; k >= 0; k--) acc = Fp::add(Fp::mul(acc, x_mont), c[(uint64_t)k * rest + i]);
  out[i] = Fp::canon(acc);
}

// ---- host-side B_j (Montgomery form), cached per extent d ----
std::vector<Fe> lagrange_matrix_host(uint32_t d) {
  using F = Fp;
  std::vector<Fe> master(d + 1, F::zero());
  master[0] = F::one();
  uint32_t deg = 0;
  for (uint32_t z = 1; z <= d; z++) {   // multiply by (X - z)
    Fe zm = F::to_mont_small(z);
    for (int k = (int)deg + 1; k >= 0; k--) {
      Fe lower = (k > 0) ? master[k - 1] : F::zero();
      master[k] = F::sub(lower, F::mul(master[k], zm));
    }
    deg++;
  }
  // w_l = prod_{r != l} (l - r) over nodes 1..d: l! * (d-1-l)! * (-1)^(d-1-l)
  std::vector<Fe> fact(d + 1);
  fact[0] = F::one();
  for (uint32_t i = 1; i <= d; i++) fact[i] = F::mul(fact[i - 1], F::to_mont_small(i));
  std::vector<Fe> B((size_t)d * d);
  std::vector<Fe> q(d);
  for (uint32_t l = 0; l < d; l++) {
    Fe zm = F::to_mont_small(l + 1);
    Fe carry = master[d];
    for (int k = (int)d - 1; k >= 0; k--) {
      q[k] = carry;
      carry = F::add(master[k], F::mul(carry, zm));
    }
    Fe w = F::mul(fact[l], fact[d - 1 - l]);
    if ((d - 1 - l) & 1u) w = F::neg(w);
    Fe wi = F::inv(w);
    for (uint32_t k = 0; k < d; k++) B[(size_t)l * d + k] = F::canon(F::mul(q[k], wi));
  }
  return B;
}

}  // namespace

namespace tcrt {

int interpolate_device(tc_ctx* ctx, Fe* d_vals, const uint32_t* shape, int m) {
  cudaStream_t st = ctx->stream;
  uint64_t n = 1;
  for (int j = 0; j < m; j++) n *= shape[j];
  uint64_t stride = n;
  for (int j = 0; j < m; j++) {
    uint32_t d = shape[j];
    stride /= d;
    if (d == 1) continue;   // degree-0 axis: identity transform
    std::string key = "interp.B." + std::to_string(d);
    Fe* dB;
    bool have = ctx->scratch.count(key + ".ready") != 0;
    TC_TRY(scratch_t(ctx, key.c_str(), (uint64_t)d * d, &dB));
    if (!have) {
      std::vector<Fe> B = lagrange_matrix_host(d);
      TC_CUDA(ctx, cudaMemcpyAsync(dB, B.data(), B.size() * sizeof(Fe), cudaMemcpyHostToDevice, st));
      TC_CUDA(ctx, cudaStreamSynchronize(st));
      ctx->scratch[key + ".ready"] = tc_ctx::Buf{};
    }
    uint32_t FB = std::max<uint32_t>(1u, 2048u / d);
    uint64_t nfib = n / d;
    size_t smem = (size_t)FB * d * sizeof(Fe);
    if (smem > 48 * 1024)
      TC_CUDA(ctx, cudaFuncSetAttribute(k_interp_axis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    unsigned grid = (unsigned)((nfib + FB - 1) / FB);
    k_interp_axis<<<grid, 256, smem, st>>>(d_vals, dB, d, stride, nfib, FB);
    TC_LAUNCHED(ctx);
  }
  return TC_OK;
}

// r (scratch copy of the coefficients) is consumed; quotients are m x n, zero outside
// their support.  omega canonical; returns y canonical on the host.
int open_quotients_device(tc_ctx* ctx, const Fe* d_coeffs, const uint32_t* shape, int m,
                          const Fe* omega_canon, Fe* d_quotients, Fe* h_y) {
  cudaStream_t st = ctx->stream;
  uint64_t n = 1;
  for (int j = 0; j < m; j++) n *= shape[j];
  Fe* r;
  TC_TRY(scratch_t(ctx, "open.rem", n, &r));
  TC_CUDA(ctx, cudaMemcpyAsync(r, d_coeffs, n * sizeof(Fe), cudaMemcpyDeviceToDevice, st));
  TC_CUDA(ctx, cudaMemsetAsync(d_quotients, 0, (uint64_t)m * n * sizeof(Fe), st));
  uint64_t span = n;   // remainder support: lex prefix of length span
  for (int a = 0; a < m; a++) {
    uint32_t d = shape[a];
    uint64_t s = span / d;
    Fe vm = Fp::to_mont(omega_canon[a]);
    k_divide_axis<<<blocks_for(s, 128), 128, 0, st>>>(r, d_quotients + (uint64_t)a * n, d, s, vm);
    TC_LAUNCHED(ctx);
    span = s;
  }
  TC_CUDA(ctx, cudaMemcpyAsync(h_y, r, sizeof(Fe), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return TC_OK;
}

int open_quotients_lagrange_device(tc_ctx* ctx, Fe* d_vals, const uint32_t* shape, int m, const LagW& W,
                                   Fe* d_quotients, Fe* h_y, bool skip_q0) {
  cudaStream_t st = ctx->stream;
  uint64_t n = 1;
  uint32_t dsum = 0;
  for (int j = 0; j < m; j++) n *= shape[j], dsum += shape[j];
  Fe *tabs, *bufA, *bufB;
  TC_TRY(scratch_t(ctx, "openlag.tabs", 3 * (uint64_t)dsum, &tabs));
  TC_TRY(scratch_t(ctx, "openlag.rA", n / shape[0] + 1, &bufA));
  TC_TRY(scratch_t(ctx, "openlag.rB", (m > 1 ? n / shape[0] / shape[1] : 1) + 1, &bufB));
  // weights + inverses -> device through the pinned staging area, one copy
  Fe* stage = (Fe*)((char*)ctx->h_stage + 512 * 1024);
  if ((size_t)3 * dsum * sizeof(Fe) > 256 * 1024) return fail(ctx, TC_ERR_VALUE, "open: axes too long");
  memcpy(stage, W.lam.data(), dsum * sizeof(Fe));
  memcpy(stage + dsum, W.inv.data(), dsum * sizeof(Fe));
  memcpy(stage + 2 * dsum, W.der.data(), dsum * sizeof(Fe));
  TC_CUDA(ctx, cudaMemcpyAsync(tabs, stage, 3 * dsum * sizeof(Fe), cudaMemcpyHostToDevice, st));
  Fe* r = d_vals;
  uint64_t span = n;
  uint32_t off = 0;
  for (int a = 0; a < m; a++) {
    const uint32_t d = shape[a];
    const uint64_t rest = span / d;
    // r_{a+1} alternates between two buffers (A holds r_1, B is large enough for r_2..);
    // kernels are stream-ordered, so r_a is never overwritten while it is read
    Fe* rn = (a & 1) ? bufB : bufA;
    k_open_axis_lag<<<blocks_for(rest, 128), 128, 0, st>>>(r, d, rest, tabs + off, tabs + dsum + off,
                                                           tabs + 2 * dsum + off, W.sj[a], rn,
                                                           (a == 0 && skip_q0) ? nullptr : d_quotients + (uint64_t)a * n);
    TC_LAUNCHED(ctx);
    r = rn;
    span = rest;
    off += d;
  }
  TC_CUDA(ctx, cudaMemcpyAsync(h_y, r, sizeof(Fe), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return TC_OK;
}

// open_quotients_lagrange_device for `cnt` openings at once: vals[o] (device), weights Ws[o];
// opening o's quotient a goes to qouts + (o m + a) n; y[o] returned on the host
int open_quotients_lagrange_batch(tc_ctx* ctx, const Fe* const* vals, int cnt, const uint32_t* shape, int m,
                                  const std::vector<LagW>& Ws, Fe* qouts, Fe* h_y, bool skip_q0,
                                  const uint64_t* qoff, const uint64_t* qstride) {
  cudaStream_t st = ctx->stream;
  uint64_t n = 1;
  uint32_t dsum = 0;
  for (int j = 0; j < m; j++) n *= shape[j], dsum += shape[j];
  const uint64_t tstride = 3 * (uint64_t)dsum;
  Fe *tabs, *bufA, *bufB;
  int* d_sj;
  const Fe** d_rin;
  TC_TRY(scratch_t(ctx, "openb.tabs", tstride * cnt, &tabs));
  TC_TRY(scratch_t(ctx, "openb.sj", (uint64_t)m * cnt, &d_sj));
  TC_TRY(scratch_t(ctx, "openb.rin", (uint64_t)m * cnt, (Fe***)&d_rin));
  TC_TRY(scratch_t(ctx, "openb.rA", (n / shape[0]) * cnt + 1, &bufA));
  TC_TRY(scratch_t(ctx, "openb.rB", (m > 1 ? n / shape[0] / shape[1] : 1) * cnt + 1, &bufB));
  // host tables: weights per opening, the sj of every (axis, opening), input pointers per axis
  std::vector<Fe> th(tstride * cnt);
  std::vector<int> sh((size_t)m * cnt);
  std::vector<const Fe*> rin((size_t)m * cnt);
  for (int o = 0; o < cnt; o++) {
    memcpy(&th[o * tstride], Ws[o].lam.data(), dsum * sizeof(Fe));
    memcpy(&th[o * tstride + dsum], Ws[o].inv.data(), dsum * sizeof(Fe));
    memcpy(&th[o * tstride + 2 * dsum], Ws[o].der.data(), dsum * sizeof(Fe));
    for (int a = 0; a < m; a++) sh[(size_t)a * cnt + o] = Ws[o].sj[a];
  }
  uint64_t span = n;
  for (int a = 0; a < m; a++) {
    const uint64_t rest_in = span;
    for (int o = 0; o < cnt; o++)
      rin[(size_t)a * cnt + o] = a == 0 ? vals[o] : ((a & 1) ? bufA : bufB) + (uint64_t)o * rest_in;
    span /= shape[a];
  }
  // pageable sources: synchronous copies complete before the host vectors go away
  TC_CUDA(ctx, cudaMemcpyAsync(tabs, th.data(), th.size() * sizeof(Fe), cudaMemcpyHostToDevice, st));
  TC_CUDA(ctx, cudaMemcpyAsync(d_sj, sh.data(), sh.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  TC_CUDA(ctx, cudaMemcpyAsync(d_rin, rin.data(), rin.size() * sizeof(Fe*), cudaMemcpyHostToDevice, st));
  span = n;
  uint32_t off = 0;
  for (int a = 0; a < m; a++) {
    const uint32_t d = shape[a];
    const uint64_t rest = span / d;
    Fe* rn = (a & 1) ? bufB : bufA;   // r_{a+1}: A for odd a+1 ... (stream order keeps r_a intact)
    // quotient a of opening o at qouts + qoff[a] + o qstride[a] (default: (o m + a) n)
    Fe* q = (a == 0 && skip_q0) ? nullptr : qouts + (qoff ? qoff[a] : (uint64_t)a * n);
    k_open_axis_lag_b<<<blocks_for(rest * cnt, 128), 128, 0, st>>>(d_rin + (size_t)a * cnt, d, rest, tabs + off,
                                                                   tstride, dsum, d_sj + (size_t)a * cnt, rn, q,
                                                                   qstride ? qstride[a] : (uint64_t)m * n,
                                                                   (uint32_t)cnt);
    TC_LAUNCHED(ctx);
    span = rest;
    off += d;
  }
  // y_o = r_m of opening o (one element each)
  Fe* last = (m & 1) ? bufA : bufB;
  TC_CUDA(ctx, cudaMemcpyAsync(h_y, last, cnt * sizeof(Fe), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return TC_OK;
}

int slice_scalars_device(tc_ctx* ctx, const std::vector<Fe>& tabs_host, const std::vector<int>& sj, uint32_t d,
                         uint32_t count, Fe* d_out) {
  cudaStream_t st = ctx->stream;
  Fe* tabs;
  int* d_sj;
  TC_TRY(scratch_t(ctx, "openh.tabs", tabs_host.size(), &tabs));
  TC_TRY(scratch_t(ctx, "openh.sj", sj.size(), &d_sj));
  // pageable sources: synchronise before the host vectors can change
  TC_CUDA(ctx, cudaMemcpyAsync(tabs, tabs_host.data(), tabs_host.size() * sizeof(Fe), cudaMemcpyHostToDevice, st));
  TC_CUDA(ctx, cudaMemcpyAsync(d_sj, sj.data(), sj.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  const uint64_t tot = (uint64_t)d * d * count;
  k_slice_scalars<<<blocks_for(tot, 128), 128, 0, st>>>(tabs, d_sj, d, count, d_out);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

int evaluate_device(tc_ctx* ctx, const Fe* d_coeffs, const uint32_t* shape, int m,
                    const Fe* point_canon, Fe* h_y) {
  cudaStream_t st = ctx->stream;
  uint64_t n = 1;
  for (int j = 0; j < m; j++) n *= shape[j];
  Fe *bufA, *bufB;
  TC_TRY(scratch_t(ctx, "eval.a", n, &bufA));
  TC_TRY(scratch_t(ctx, "eval.b", n, &bufB));
  const Fe* src = d_coeffs;
  uint64_t rest = n;
  for (int a = 0; a < m; a++) {
    uint32_t d = shape[a];
    rest /= d;
    Fe* dst = (a & 1) ? bufB : bufA;
    k_horner_lead<<<blocks_for(rest, 128), 128, 0, st>>>(src, dst, d, rest, Fp::to_mont(point_canon[a]));
    TC_LAUNCHED(ctx);
    src = dst;
  }
  TC_CUDA(ctx, cudaMemcpyAsync(h_y, src, sizeof(Fe), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return TC_OK;
}

}  // namespace tcrt
