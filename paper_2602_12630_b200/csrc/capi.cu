// C ABI of libtcb200.so (include/tc_b200.h): context / SRS management and the prover entry
// points (quantize, interpolate, evaluate, open_quotients, msm, commit, open, Terkle build),
// plus the CPU-side verifier primitive (pairing) that the reference keeps on the host.
#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>

#include "sha256.cuh"
#include "tc_internal.cuh"

using namespace tc;

// ======================================================================================
// runtime helpers
// ======================================================================================
namespace tcrt {

int fail(tc_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

int func_smem(tc_ctx* ctx, const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  TC_CUDA(ctx, cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, func, bytes})) return TC_OK;
  TC_CUDA(ctx, cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({dev, func, bytes});
  return TC_OK;
}

int scratch(tc_ctx* ctx, const char* name, size_t bytes, void** out) {
  auto& b = ctx->scratch[name];
  if (b.n < bytes + (ctx->guard ? GUARD_BYTES : 0)) {
    if (b.p) {
      cudaError_t e = cudaFreeAsync(b.p, ctx->stream);
      if (e != cudaSuccess) return fail(ctx, TC_ERR_CUDA, "cudaFreeAsync(%s): %s", name, cudaGetErrorString(e));
      b.p = nullptr;
      b.n = 0;
    }
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMallocAsync(&b.p, want, ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, TC_ERR_MEMORY, "scratch %s: cannot allocate %zu bytes: %s", name, want, cudaGetErrorString(e));
    }
    b.n = want;
  }
  *out = b.p;
  if (ctx->guard) {
    // out-of-bounds-write canary right after the requested size (want >= bytes + 256)
    TC_CUDA(ctx, cudaMemsetAsync((char*)b.p + bytes, 0xA5, GUARD_BYTES, ctx->stream));
    ctx->guards[name] = std::make_pair((char*)b.p + bytes, bytes);
  }
  return TC_OK;
}

}  // namespace tcrt

namespace {
__global__ void k_check_guard(const uint8_t* g, uint32_t n, uint32_t* bad) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
    if (g[i] != 0xA5) {
      atomicAdd(bad, 1u);
      return;
    }
}
}  // namespace

int tc_ctx_check_guards(tc_ctx* ctx, uint64_t* bad_buffers) {
  if (!ctx || !bad_buffers) return TC_ERR_ARGUMENT;
  *bad_buffers = 0;
  if (!ctx->guard) return tcrt::fail(ctx, TC_ERR_VALUE, "scratch guards are off (set TC_SCRATCH_GUARD=1 before creating the context)");
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::string bad;
  for (auto& kv : ctx->guards) {
    TC_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream));
    k_check_guard<<<1, 256, 0, ctx->stream>>>((const uint8_t*)kv.second.first, tcrt::GUARD_BYTES, ctx->d_flags);
    TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
    TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->h_flags[0]) {
      ++*bad_buffers;
      bad += kv.first + "(" + std::to_string(kv.second.second) + " B) ";
    }
  }
  if (*bad_buffers) tcrt::fail(ctx, TC_ERR_VALUE, "write past the end of scratch: %s", bad.c_str());
  return TC_OK;
}

using tcrt::fail;

namespace {

// ---- host encodings (backend.py:309-348) ----
bool le21_to_fe(const uint8_t* b, Fe& out) {
  for (int i = 0; i < 6; i++) out.v[i] = 0;
  for (int i = 0; i < 21; i++) out.v[i / 4] |= (uint32_t)b[i] << (8 * (i % 4));
  // < p ?
  Fe t;
  return Fp::sub_km(t, out, FpParams::M0, FpParams::M5) != 0;
}
void fe_to_le21(const Fe& a, uint8_t* b) {
  for (int i = 0; i < 21; i++) b[i] = (uint8_t)(a.v[i / 4] >> (8 * (i % 4)));
}
// decode_elem (backend.py:319-333); false on malformed / off-curve
bool decode43(const uint8_t* raw, Aff& out) {
  if (raw[0] == 0) {
    for (int i = 1; i < 43; i++)
      if (raw[i]) return false;
    out = aff_inf();
    return true;
  }
  if (raw[0] != 4) return false;
  Fe x, y;
  for (int i = 0; i < 6; i++) x.v[i] = y.v[i] = 0;
  for (int i = 0; i < 21; i++) {
    x.v[i / 4] |= (uint32_t)raw[1 + i] << (8 * (i % 4));
    y.v[i / 4] |= (uint32_t)raw[22 + i] << (8 * (i % 4));
  }
  Fe t;
  if (!Fq::sub_km(t, x, FqParams::M0, FqParams::M5) || !Fq::sub_km(t, y, FqParams::M0, FqParams::M5)) return false;
  Fe xm = Fq::to_mont(x), ym = Fq::to_mont(y);
  Fe lhs = Fq::sqr(ym);
  Fe rhs = Fq::add(Fq::mul(Fq::sqr(xm), xm), xm);
  if (!Fq::eq(lhs, rhs)) return false;
  out = Aff{Fq::canon(xm), Fq::canon(ym)};
  return true;
}

Aff g_host() {
  Fe x{{0xbe9bb8c2u, 0x9f4698deu, 0x2e04a40bu, 0x96df9421u, 0xd6e0e406u, 0x000000abu}};
  Fe y{{0xca83210eu, 0x0d3911f8u, 0x28e6ecd6u, 0xfcd508bdu, 0xc7320595u, 0x00000018u}};
  return Aff{Fq::to_mont(x), Fq::to_mont(y)};
}

// k * P on the host (canonical scalar k < 2^192), MSB-first double-and-add
Xyzz host_mul(const Aff& P, const Fe& k) {
  Xyzz acc = xyzz_inf();
  bool started = false;
  for (int b = 191; b >= 0; b--) {
    if (started) acc = xyzz_dbl(acc);
    if ((k.v[b >> 5] >> (b & 31)) & 1u) {
      xyzz_add_aff(acc, P);
      started = true;
    }
  }
  return acc;
}
Aff host_aff(const Xyzz& p) {
  Aff r = xyzz_to_aff(p);
  if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
  return r;
}
Fe fp_neg_canon(const Fe& a) {   // (-a) mod p, canonical input
  Fe z{{0, 0, 0, 0, 0, 0}};
  return Fp::canon(Fp::sub(z, a));
}

// ---- device encode/decode of SRS point arrays ----
__global__ void k_encode43(const Aff* pts, uint64_t n, uint8_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  aff_encode43(pts[i], out + i * 43);
}
__global__ void k_decode43(const uint8_t* raw, uint64_t n, Aff* out, uint32_t* bad) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* r = raw + i * 43;
  if (r[0] == 0) {
    bool ok = true;
    for (int k = 1; k < 43; k++) ok &= (r[k] == 0);
    if (!ok) atomicOr(bad, 1u);
    out[i] = aff_inf();
    return;
  }
  Fe x, y;
  for (int k = 0; k < 6; k++) x.v[k] = y.v[k] = 0;
  for (int k = 0; k < 21; k++) {
    x.v[k / 4] |= (uint32_t)r[1 + k] << (8 * (k % 4));
    y.v[k / 4] |= (uint32_t)r[22 + k] << (8 * (k % 4));
  }
  Fe t;
  bool inrange = Fq::sub_km(t, x, FqParams::M0, FqParams::M5) && Fq::sub_km(t, y, FqParams::M0, FqParams::M5);
  Fe xm = Fq::to_mont(x), ym = Fq::to_mont(y);
  bool on = Fq::eq(Fq::sqr(ym), Fq::add(Fq::mul(Fq::sqr(xm), xm), xm));
  if (r[0] != 4 || !inrange || !on) atomicOr(bad, 1u);
  out[i] = Aff{Fq::canon(xm), Fq::canon(ym)};
}

__global__ void k_field_op(int op, const Fe* a, const Fe* b, Fe* out, uint64_t n) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  Fe r;
  switch (op) {
    case 0: r = Fq::from_mont(Fq::mul(Fq::to_mont(a[i]), Fq::to_mont(b[i]))); break;
    case 1: r = Fp::from_mont(Fp::mul(Fp::to_mont(a[i]), Fp::to_mont(b[i]))); break;
    case 2: r = Fq::canon(Fq::add(a[i], b[i])); break;
    case 3: r = Fq::canon(Fq::sub(a[i], b[i])); break;
    case 5: r = Fq::from_mont(Fq::sqr(Fq::to_mont(a[i]))); break;
    case 6: r = Fp::from_mont(Fp::sqr(Fp::to_mont(a[i]))); break;
    default: r = Fq::from_mont(Fq::inv(Fq::to_mont(a[i]))); break;
  }
  out[i] = r;
}

// 16 independent dependent-chains of mad.lo.u32 per thread: saturates the IMAD pipe
__global__ void k_imad_peak(uint32_t* sink, uint32_t seed, int iters) {
  uint32_t a[16];
  const uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = seed * (i + 3) + threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s ^= a[i];
  if (s == 0x7f4a7c15u) sink[0] = s;
}

// read one device Aff result and encode it on the host
int fetch_encode(tc_ctx* ctx, const Aff* d_pt, uint8_t* out43) {
  Aff h;
  TC_CUDA(ctx, cudaMemcpyAsync(&h, d_pt, sizeof(Aff), cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  aff_encode43(h, out43);
  return TC_OK;
}

uint64_t shape_size(const uint32_t* shape, int m) {
  uint64_t n = 1;
  for (int j = 0; j < m; j++) n *= shape[j];
  return n;
}

int check_shape(tc_ctx* ctx, const uint32_t* shape, int m) {
  if (m < 1 || m > TC_MAX_AXES) return fail(ctx, TC_ERR_VALUE, "shape needs 1..%d axes, got %d", TC_MAX_AXES, m);
  uint64_t n = 1;
  for (int j = 0; j < m; j++) {
    if (shape[j] < 1) return fail(ctx, TC_ERR_VALUE, "axis degree bound must be >= 1, got %u", shape[j]);
    n *= shape[j];
    if (n > (1ull << 26)) return fail(ctx, TC_ERR_VALUE, "coefficient array exceeds limit 2^26");
  }
  return TC_OK;
}

// canonical F_p tensor of the SRS shape from a device input of any dtype
int load_field_tensor(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits, Fe** out,
                      const char* name) {
  Fe* buf;
  TC_TRY(tcrt::scratch_t(ctx, name, n, &buf));
  if (dtype == TC_DTYPE_FP_LIMBS) {
    TC_CUDA(ctx, cudaMemcpyAsync(buf, d_in, n * sizeof(Fe), cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    TC_TRY(tcrt::quantize_device(ctx, d_in, dtype, n, scale_bits, buf));
  }
  *out = buf;
  return TC_OK;
}

// ---- per-axis SRS exponent tables (host, F_p Montgomery arithmetic) ----
// monomial: tau^e, e < d ; Lagrange on nodes 1..d: L_a(tau) = prod_{b != a} (tau - b)/(a - b)
void axis_tables(const Fe& tau_c, uint32_t d, bool lagrange, std::vector<Fe>& out) {
  Fe tau = Fp::to_mont(tau_c);
  if (!lagrange) {
    Fe acc = Fp::one();
    for (uint32_t e = 0; e < d; e++) {
      out.push_back(Fp::from_mont(acc));
      acc = Fp::mul(acc, tau);
    }
    return;
  }
  // exact node?
  for (uint32_t a = 0; a < d; a++) {
    if (Fp::eq(tau, Fp::to_mont_small(a + 1))) {
      for (uint32_t b = 0; b < d; b++) out.push_back(b == a ? Fp::from_mont(Fp::one()) : Fp::zero());
      return;
    }
  }
  // master = prod (tau - b); L_a = master / (tau - a) / w_a,  w_a = a! (d-1-a)! (-1)^(d-1-a)
  std::vector<Fe> diff(d), fact(d + 1);
  Fe master = Fp::one();
  for (uint32_t b = 0; b < d; b++) {
    diff[b] = Fp::sub(tau, Fp::to_mont_small(b + 1));
    master = Fp::mul(master, diff[b]);
  }
  fact[0] = Fp::one();
  for (uint32_t i = 1; i <= d; i++) fact[i] = Fp::mul(fact[i - 1], Fp::to_mont_small(i));
  // batch-invert diff[a] * w_a
  std::vector<Fe> den(d), pref(d);
  Fe run = Fp::one();
  for (uint32_t a = 0; a < d; a++) {
    Fe w = Fp::mul(fact[a], fact[d - 1 - a]);
    if ((d - 1 - a) & 1u) w = Fp::neg(w);
    den[a] = Fp::mul(diff[a], w);
    pref[a] = run;
    run = Fp::mul(run, den[a]);
  }
  Fe inv = Fp::inv_fast(run);
  std::vector<Fe> res(d);
  for (int a = (int)d - 1; a >= 0; a--) {
    Fe ia = Fp::mul(inv, pref[a]);
    inv = Fp::mul(inv, den[a]);
    res[a] = Fp::from_mont(Fp::mul(master, ia));
  }
  out.insert(out.end(), res.begin(), res.end());
}

// g^{prod_j tab_j[i_j]} for every lex index of `shape` into the preallocated dst
int srs_fill_points(tc_ctx* ctx, const uint32_t* shape, int m, const Fe* taus, bool lagrange, Aff* dst) {
  std::vector<Fe> tabs;
  uint64_t n = 1;
  for (int j = 0; j < m; j++) axis_tables(taus[j], shape[j], lagrange, tabs), n *= shape[j];
  Fe* d_exps;
  TC_TRY(tcrt::scratch_t(ctx, "srs.exps", n, &d_exps));
  TC_TRY(tcrt::srs_exponents(ctx, tabs, shape, m, n, d_exps));
  TC_TRY(tcrt::fixed_base_g(ctx, d_exps, n, dst));
  return TC_OK;
}

int srs_build_points(tc_ctx* ctx, tc_srs* srs, const std::vector<Fe>& taus, bool lagrange, Aff** dst) {
  TC_CUDA(ctx, cudaMalloc(dst, srs->n * sizeof(Aff)));
  return srs_fill_points(ctx, srs->shape, srs->m, taus.data(), lagrange, *dst);
}

// Edwards copies of every basis the Pippenger pipeline may read (built at setup, so the
// shared read-only SRS is never mutated by a commit)
int srs_build_edwards(tc_ctx* ctx, tc_srs* srs) {
  const EdPk* e;
  if (srs->n <= SMALL_MSM_MAX && !srs->sublag) return TC_OK;   // node SRSs use the table kernel
  if (srs->monomial) TC_TRY(tcrt::srs_edwards(ctx, srs, TC_SRS_MONOMIAL, &e));
  if (srs->lagrange) TC_TRY(tcrt::srs_edwards(ctx, srs, TC_SRS_LAGRANGE, &e));
  if (srs->sublag) TC_TRY(tcrt::srs_edwards(ctx, srs, 0, &e));
  return TC_OK;
}

// sub-grid Lagrange sets for the suffixes i = 1..m-1 (Lagrange-route opening quotients):
// offsets and allocation
int srs_alloc_sublag(tc_ctx* ctx, tc_srs* srs) {
  uint64_t total = 0;
  for (int i = 1; i < srs->m; i++) {
    uint64_t ni = 1;
    for (int j = i; j < srs->m; j++) ni *= srs->shape[j];
    srs->sublag_off[i] = total;
    total += ni;
  }
  TC_CUDA(ctx, cudaMalloc(&srs->sublag, total * sizeof(Aff)));
  return TC_OK;
}

int srs_build_sublag(tc_ctx* ctx, tc_srs* srs, const std::vector<Fe>& taus) {
  if (srs->m < 2) return TC_OK;
  TC_TRY(srs_alloc_sublag(ctx, srs));
  for (int i = 1; i < srs->m; i++)
    TC_TRY(srs_fill_points(ctx, srs->shape + i, srs->m - i, taus.data() + i, true, srs->sublag + srs->sublag_off[i]));
  return TC_OK;
}

// Lagrange elements and sub-grid sets from the monomial elements alone (no trapdoor): the
// suffix set i is the Lagrange transform of the first prod_{j>=i} d_j monomial elements
// (lex indices with zero leading coordinates = g^{prod_{j>=i} tau_j^{i_j}}) over axes i..m-1
int srs_derive_lagrange(tc_ctx* ctx, tc_srs* srs) {
  if (!srs->monomial) return fail(ctx, TC_ERR_VALUE, "srs has no monomial elements to derive from");
  if (srs->lagrange) return TC_OK;
  const EdPk* mono;
  TC_TRY(tcrt::srs_edwards(ctx, srs, TC_SRS_MONOMIAL, &mono));
  // derive into buffers the SRS does not own yet: a failure leaves it monomial-only, never
  // with a half-computed Lagrange set the routes would trust
  Aff *lag = nullptr, *sub = nullptr;
  auto cleanup = [&](int s) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(lag);
    cudaFree(sub);
    return s;
  };
  if (cudaMalloc(&lag, srs->n * sizeof(Aff)) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, TC_ERR_MEMORY, "derive: Lagrange set of %llu points", (unsigned long long)srs->n);
  }
  int s = tcrt::derive_lagrange_device(ctx, mono, srs->shape, srs->m, lag);
  if (s) return cleanup(s);
  uint64_t off[TC_MAX_AXES] = {0}, total = 0;
  for (int i = 1; i < srs->m; i++) {
    uint64_t ni = 1;
    for (int j = i; j < srs->m; j++) ni *= srs->shape[j];
    off[i] = total;
    total += ni;
  }
  if (srs->m > 1) {
    if (cudaMalloc(&sub, total * sizeof(Aff)) != cudaSuccess) {
      cudaGetLastError();
      return cleanup(fail(ctx, TC_ERR_MEMORY, "derive: sub-grid sets of %llu points", (unsigned long long)total));
    }
    for (int i = 1; i < srs->m && !s; i++)
      s = tcrt::derive_lagrange_device(ctx, mono, srs->shape + i, srs->m - i, sub + off[i]);
    if (s) return cleanup(s);
  }
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return cleanup(fail(ctx, TC_ERR_CUDA, "derive: %s", cudaGetErrorString(cudaGetLastError())));
  srs->lagrange = lag;
  srs->sublag = sub;
  for (int i = 0; i < TC_MAX_AXES; i++) srs->sublag_off[i] = off[i];
  TC_TRY(srs_build_edwards(ctx, srs));
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return TC_OK;
}

// ---- host pairing (backend.py:219-291), restated over the shared F_q core ----
struct F2 {
  Fe a, b;
};
F2 f2mul(const F2& u, const F2& v) {
  return F2{Fq::sub(Fq::mul(u.a, v.a), Fq::mul(u.b, v.b)), Fq::add(Fq::mul(u.a, v.b), Fq::mul(u.b, v.a))};
}
F2 f2sqr(const F2& u) {
  return F2{Fq::mul(Fq::sub(u.a, u.b), Fq::add(u.a, u.b)), Fq::dbl(Fq::mul(u.a, u.b))};
}

// returns false on "pairing argument of unexpected order" (BackendError)
bool host_pairing(const Aff& S, const Aff& T, F2& out) {
  if (aff_is_inf(S) || aff_is_inf(T)) {
    out = F2{Fq::one(), Fq::zero()};
    return true;
  }
  Fe xq = Fq::neg(T.x), yq = T.y, xp = S.x, yp = S.y;
  F2 f{Fq::one(), Fq::zero()};
  Fe X = xp, Y = yp, Z = Fq::one();
  // bits of p below the MSB: p = 2^161 + 2^24 + 1 -> bits 160..0
  for (int bit = 160; bit >= 0; bit--) {
    Fe XX = Fq::sqr(X), YY = Fq::sqr(Y), YYYY = Fq::sqr(YY), ZZ = Fq::sqr(Z);
    Fe t = Fq::add(X, YY);
    Fe Sd = Fq::dbl(Fq::sub(Fq::sub(Fq::sqr(t), XX), YYYY));
    Fe M = Fq::add(Fq::add(Fq::dbl(XX), XX), Fq::sqr(ZZ));
    // tangent line at R evaluated at (xq, i*yq)
    Fe lr = Fq::sub(Fq::neg(Fq::dbl(YY)), Fq::mul(M, Fq::sub(Fq::mul(xq, ZZ), X)));
    Fe li = Fq::mul(Fq::mul(Fq::mul(Fq::dbl(Y), Z), ZZ), yq);
    f = f2mul(f2sqr(f), F2{lr, li});
    Fe X3 = Fq::sub(Fq::sqr(M), Fq::dbl(Sd));
    Fe Y3 = Fq::sub(Fq::mul(M, Fq::sub(Sd, X3)), Fq::dbl(Fq::dbl(Fq::dbl(YYYY))));
    Fe Z3 = Fq::sub(Fq::sub(Fq::sqr(Fq::add(Y, Z)), YY), ZZ);
    X = X3, Y = Y3, Z = Z3;
    bool set = (bit == 0) || (bit == 24);
    if (set) {
      ZZ = Fq::sqr(Z);
      Fe U2 = Fq::mul(xp, ZZ);
      Fe S2 = Fq::mul(Fq::mul(yp, Z), ZZ);
      Fe H = Fq::sub(U2, X);
      Fe num = Fq::sub(S2, Y);
      bool hz = Fq::is_zero(H), nz = Fq::is_zero(num);
      if (hz && nz) return false;
      if (!hz) {
        Fe den = Fq::mul(H, Z);
        Fe lr2 = Fq::sub(Fq::neg(Fq::mul(den, yp)), Fq::mul(num, Fq::sub(xq, xp)));
        Fe li2 = Fq::mul(den, yq);
        f = f2mul(f, F2{lr2, li2});
        Fe HH = Fq::sqr(H);
        Fe I = Fq::dbl(Fq::dbl(HH));
        Fe J = Fq::mul(H, I);
        Fe V = Fq::mul(X, I);
        Fe r2 = Fq::dbl(num);
        Fe X4 = Fq::sub(Fq::sub(Fq::sqr(r2), J), Fq::dbl(V));
        Fe Y4 = Fq::sub(Fq::mul(r2, Fq::sub(V, X4)), Fq::dbl(Fq::mul(Y, J)));
        Fe Z4 = Fq::sub(Fq::sub(Fq::sqr(Fq::add(Z, H)), ZZ), HH);
        X = X4, Y = Y4, Z = Z4;
      } else {
        X = Fq::zero(), Y = Fq::one(), Z = Fq::zero();
      }
    }
  }
  // final exponentiation: (conj(f) / f)^120
  Fe norm = Fq::add(Fq::sqr(f.a), Fq::sqr(f.b));
  Fe ni = Fq::inv_fast(norm);
  Fe inva = Fq::mul(f.a, ni), invb = Fq::neg(Fq::mul(f.b, ni));
  F2 g{Fq::add(Fq::mul(f.a, inva), Fq::mul(f.b, invb)), Fq::sub(Fq::mul(f.a, invb), Fq::mul(f.b, inva))};
  F2 o{Fq::one(), Fq::zero()};
  for (uint32_t e = 120; e; e >>= 1) {
    if (e & 1u) o = f2mul(o, g);
    g = f2sqr(g);
  }
  out = F2{Fq::canon(o.a), Fq::canon(o.b)};
  return true;
}

bool f2_eq(const F2& u, const F2& v) { return Fq::eq(u.a, v.a) && Fq::eq(u.b, v.b); }

}  // namespace

// ======================================================================================
// exported ABI
// ======================================================================================
extern "C" {

int tc_abi_version(void) { return TC_ABI_VERSION; }

int tc_ctx_create(int device, void* cuda_stream, tc_ctx** out) {
  if (!out) return TC_ERR_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return TC_ERR_CUDA;
  }
  if (device < 0 || device >= count) return TC_ERR_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return TC_ERR_CUDA;
  tc_ctx* ctx = new tc_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)cuda_stream;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) ctx->num_sms = prop.multiProcessorCount;
  ctx->h_stage_bytes = 1 << 20;
  ctx->guard = getenv("TC_SCRATCH_GUARD") && atoi(getenv("TC_SCRATCH_GUARD")) != 0;
  if (getenv("TC_L2_FETCH")) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(getenv("TC_L2_FETCH")));
  if (cudaMalloc(&ctx->d_flags, 64) != cudaSuccess || cudaMallocHost(&ctx->h_flags, 64) != cudaSuccess ||
      cudaMallocHost(&ctx->h_stage, ctx->h_stage_bytes) != cudaSuccess) {
    delete ctx;
    return TC_ERR_CUDA;
  }
  *out = ctx;
  return TC_OK;
}

int tc_ctx_destroy(tc_ctx* ctx) {
  if (!ctx) return TC_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->scratch)
    if (kv.second.p) cudaFreeAsync(kv.second.p, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->d_flags);
  cudaFreeHost(ctx->h_flags);
  cudaFreeHost(ctx->h_stage);
  if (ctx->ev[0]) cudaEventDestroy(ctx->ev[0]), cudaEventDestroy(ctx->ev[1]);
  for (cudaEvent_t e : ctx->copy_ev) cudaEventDestroy(e);
  for (auto& sl : ctx->slot)
    if (sl.ready) cudaEventDestroy(sl.ready);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->h_res) cudaFreeHost(ctx->h_res);
  if (ctx->h_off) cudaFreeHost(ctx->h_off);
  if (ctx->res_ev) cudaEventDestroy(ctx->res_ev);
  if (ctx->ev_mid) cudaEventDestroy(ctx->ev_mid);
  if (ctx->ev_tail) cudaEventDestroy(ctx->ev_tail);
  if (ctx->tail_stream) cudaStreamDestroy(ctx->tail_stream);
  delete ctx;
  return TC_OK;
}

int tc_ctx_set_pipelined(tc_ctx* ctx, int on) {
  if (!ctx) return TC_ERR_ARGUMENT;
  ctx->pipelined = on != 0;
  return TC_OK;
}

int tc_ctx_set_stream(tc_ctx* ctx, void* s) {
  if (!ctx) return TC_ERR_ARGUMENT;
  ctx->stream = (cudaStream_t)s;
  return TC_OK;
}

int tc_ctx_synchronize(tc_ctx* ctx) {
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return TC_OK;
}

const char* tc_ctx_last_error(const tc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
uint64_t tc_ctx_launch_count(const tc_ctx* ctx) { return ctx ? ctx->launches : 0; }

int tc_ctx_set_profiling(tc_ctx* ctx, int on) {
  if (!ctx) return TC_ERR_ARGUMENT;
  if (on && !ctx->ev[0]) {
    TC_CUDA(ctx, cudaEventCreate(&ctx->ev[0]));
    TC_CUDA(ctx, cudaEventCreate(&ctx->ev[1]));
  }
  ctx->prof = on != 0;
  ctx->stats.clear();
  return TC_OK;
}

int tc_ctx_kernel_stats(const tc_ctx* ctx, const char* name, double* ms, uint64_t* launches, double* units) {
  if (!ctx || !name || !ms || !launches || !units) return TC_ERR_ARGUMENT;
  auto it = ctx->stats.find(name);
  if (it == ctx->stats.end()) {
    *ms = 0, *launches = 0, *units = 0;
    return TC_OK;
  }
  *ms = it->second.ms;
  *launches = it->second.launches;
  *units = it->second.units;
  return TC_OK;
}

// ---- SRS ----
int tc_srs_generate(tc_ctx* ctx, const uint32_t* shape, int m, const uint8_t* taus_le21, int flags, tc_srs** out) {
  if (!ctx || !shape || !taus_le21 || !out) return TC_ERR_ARGUMENT;
  TC_TRY(check_shape(ctx, shape, m));
  if (!(flags & (TC_SRS_MONOMIAL | TC_SRS_LAGRANGE))) return fail(ctx, TC_ERR_ARGUMENT, "srs flags");
  std::vector<Fe> taus(m);
  for (int j = 0; j < m; j++)
    if (!le21_to_fe(taus_le21 + 21 * j, taus[j])) return fail(ctx, TC_ERR_VALUE, "trapdoor %d out of range", j);
  tc_srs* srs = new tc_srs();
  srs->device = ctx->device;
  srs->m = m;
  for (int j = 0; j < m; j++) srs->shape[j] = shape[j];
  srs->n = shape_size(shape, m);
  int s = TC_OK;
  if (flags & TC_SRS_MONOMIAL) s = srs_build_points(ctx, srs, taus, false, &srs->monomial);
  if (!s && (flags & TC_SRS_LAGRANGE)) s = srs_build_points(ctx, srs, taus, true, &srs->lagrange);
  if (!s && (flags & TC_SRS_LAGRANGE)) s = srs_build_sublag(ctx, srs, taus);
  s = s ? s : srs_build_edwards(ctx, srs);
  if (!s) {   // axis elements g^{tau_j}
    Fe* d_t;
    Aff* d_a;
    s = tcrt::scratch_t(ctx, "srs.axis_t", m, &d_t);
    if (!s) s = tcrt::scratch_t(ctx, "srs.axis_a", m, &d_a);
    if (!s && cudaMemcpyAsync(d_t, taus.data(), m * sizeof(Fe), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
      s = fail(ctx, TC_ERR_CUDA, "copy taus");
    if (!s) s = tcrt::fixed_base_g(ctx, d_t, m, d_a);
    if (!s && cudaMemcpyAsync(srs->axis, d_a, m * sizeof(Aff), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
      s = fail(ctx, TC_ERR_CUDA, "copy axis");
    if (!s && cudaStreamSynchronize(ctx->stream) != cudaSuccess) s = fail(ctx, TC_ERR_CUDA, "sync");
  }
  if (s) {
    tc_srs_destroy(srs);
    return s;
  }
  *out = srs;
  return TC_OK;
}

int tc_srs_load(tc_ctx* ctx, const uint32_t* shape, int m, const uint8_t* monomial43, const uint8_t* axis43, tc_srs** out) {
  if (!ctx || !shape || !monomial43 || !axis43 || !out) return TC_ERR_ARGUMENT;
  TC_TRY(check_shape(ctx, shape, m));
  tc_srs* srs = new tc_srs();
  srs->device = ctx->device;
  srs->m = m;
  for (int j = 0; j < m; j++) srs->shape[j] = shape[j];
  srs->n = shape_size(shape, m);
  for (int j = 0; j < m; j++) {
    if (!decode43(axis43 + 43 * j, srs->axis[j])) {
      delete srs;
      return fail(ctx, TC_ERR_VALUE, "axis element %d: bad encoding or point not on curve", j);
    }
  }
  uint8_t* d_raw;
  int s = tcrt::scratch_t(ctx, "srs.raw", srs->n * 43, &d_raw);
  if (!s && cudaMalloc(&srs->monomial, srs->n * sizeof(Aff)) != cudaSuccess) s = fail(ctx, TC_ERR_MEMORY, "srs alloc");
  if (!s && cudaMemcpyAsync(d_raw, monomial43, srs->n * 43, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
    s = fail(ctx, TC_ERR_CUDA, "copy srs");
  if (!s && cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream) != cudaSuccess) s = fail(ctx, TC_ERR_CUDA, "memset");
  if (!s) {
    k_decode43<<<tcrt::blocks_for(srs->n, 128), 128, 0, ctx->stream>>>(d_raw, srs->n, srs->monomial, ctx->d_flags);
    ctx->launches++;
    if (cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      s = fail(ctx, TC_ERR_CUDA, "decode srs: %s", cudaGetErrorString(cudaGetLastError()));
    else if (ctx->h_flags[0])
      s = fail(ctx, TC_ERR_VALUE, "srs element: bad encoding or point not on curve");
  }
  if (!s) s = srs_build_edwards(ctx, srs);
  // a published SRS has no Lagrange elements: derive them (and the sub-grid sets) from the
  // monomial ones, so commits and openings on it take the Lagrange route
  if (!s) s = srs_derive_lagrange(ctx, srs);
  if (s) {
    tc_srs_destroy(srs);
    return s;
  }
  *out = srs;
  return TC_OK;
}

int tc_srs_derive_lagrange(tc_ctx* ctx, tc_srs* srs) {
  if (!ctx || !srs) return TC_ERR_ARGUMENT;
  TC_CUDA(ctx, cudaSetDevice(srs->device));
  return srs_derive_lagrange(ctx, srs);
}

int tc_srs_export(tc_ctx* ctx, const tc_srs* srs, int which, uint64_t offset, uint64_t count, uint8_t* out43) {
  if (!ctx || !srs || !out43) return TC_ERR_ARGUMENT;
  const Aff* pts = (which == TC_SRS_LAGRANGE) ? srs->lagrange : (which == TC_SRS_SUBGRID) ? srs->sublag : srs->monomial;
  if (!pts) return fail(ctx, TC_ERR_VALUE, "srs has no elements of kind %d", which);
  const uint64_t total = which == TC_SRS_SUBGRID ? srs->sublag_off[srs->m - 1] + srs->shape[srs->m - 1] : srs->n;
  if (offset > total || count > total - offset)
    return fail(ctx, TC_ERR_INDEX, "srs export range [%llu, +%llu) out of bounds (%llu elements of kind %d)",
                (unsigned long long)offset, (unsigned long long)count, (unsigned long long)total, which);
  if (count == 0) return TC_OK;
  uint8_t* d_raw;
  TC_TRY(tcrt::scratch_t(ctx, "srs.raw", count * 43, &d_raw));
  k_encode43<<<tcrt::blocks_for(count, 128), 128, 0, ctx->stream>>>(pts + offset, count, d_raw);
  TC_LAUNCHED(ctx);
  TC_CUDA(ctx, cudaMemcpyAsync(out43, d_raw, count * 43, cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return TC_OK;
}

int tc_srs_table_bytes(const tc_srs* srs, uint64_t* exptab_bytes, uint64_t* wintab_bytes, uint64_t* basis_bytes) {
  if (!srs || !exptab_bytes || !wintab_bytes || !basis_bytes) return TC_ERR_ARGUMENT;
  *exptab_bytes = (uint64_t)srs->exptab_depth * srs->n * sizeof(EdPk);
  *wintab_bytes = srs->wintab_bytes;
  const uint64_t nsub = srs->sublag && srs->m > 1 ? srs->sublag_off[srs->m - 1] + srs->shape[srs->m - 1] : 0;
  uint64_t b = 0;
  if (srs->monomial) b += srs->n * sizeof(Aff);
  if (srs->lagrange) b += srs->n * sizeof(Aff);
  if (srs->sublag) b += nsub * sizeof(Aff);
  if (srs->ed_monomial) b += srs->n * sizeof(EdPk);
  if (srs->ed_lagrange) b += srs->n * sizeof(EdPk);
  if (srs->ed_sublag) b += nsub * sizeof(EdPk);
  *basis_bytes = b;
  return TC_OK;
}

int tc_srs_prepare(tc_ctx* ctx, tc_srs* srs, int dtype, int scale_bits) {
  if (!ctx || !srs) return TC_ERR_ARGUMENT;
  TC_CUDA(ctx, cudaSetDevice(srs->device));
  if (dtype != TC_DTYPE_F16 || !srs->lagrange || srs->n <= SMALL_MSM_MAX) return TC_OK;
  const EdPk* lag;
  TC_TRY(tcrt::srs_edwards(ctx, srs, TC_SRS_LAGRANGE, &lag));
  const EdPk* tab;
  const int depth = scale_bits + 6;   // any finite fp16 input (the speculative plan's depth)
  if ((uint64_t)depth * srs->n >= (1ull << 31)) return TC_OK;
  const int s = tcrt::srs_exp_table(ctx, srs, lag, srs->n, depth, &tab);
  if (s == TC_ERR_MEMORY) return TC_OK;   // commits fall back to the float-exponent groups
  return s;
}

int tc_srs_export_axis(const tc_srs* srs, uint8_t* out43) {
  if (!srs || !out43) return TC_ERR_ARGUMENT;
  for (int j = 0; j < srs->m; j++) aff_encode43(srs->axis[j], out43 + 43 * j);
  return TC_OK;
}

int tc_srs_has(const tc_srs* srs, int which) {
  if (!srs) return 0;
  return which == TC_SRS_LAGRANGE ? srs->lagrange != nullptr
         : which == TC_SRS_SUBGRID ? srs->sublag != nullptr : srs->monomial != nullptr;
}

uint64_t tc_srs_size(const tc_srs* srs) { return srs ? srs->n : 0; }

int tc_srs_destroy(tc_srs* srs) {
  if (!srs) return TC_OK;
  cudaSetDevice(srs->device);
  if (srs->monomial) cudaFree(srs->monomial);
  if (srs->lagrange) cudaFree(srs->lagrange);
  for (auto* t : srs->small_tab)
    if (t) cudaFree(t);
  if (srs->sublag) cudaFree(srs->sublag);
  for (auto* e : {srs->ed_monomial, srs->ed_lagrange, srs->ed_sublag})
    if (e) cudaFree(e);
  for (auto& kv : srs->wintab) cudaFree(kv.second);
  if (srs->exptab) cudaFree(srs->exptab);
  for (auto* t : srs->retired) cudaFree(t);
  delete srs;
  return TC_OK;
}

// ---- polynomial entry points ----
int tc_quantize(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits, uint32_t* d_out) {
  if (!ctx || (n && (!d_in || !d_out))) return TC_ERR_ARGUMENT;
  if (dtype == TC_DTYPE_FP_LIMBS) return fail(ctx, TC_ERR_ARGUMENT, "quantize: input already field elements");
  return tcrt::quantize_device(ctx, d_in, dtype, n, scale_bits, (Fe*)d_out);
}

int tc_interpolate(tc_ctx* ctx, uint32_t* d_limbs, const uint32_t* shape, int m) {
  if (!ctx || !d_limbs || !shape) return TC_ERR_ARGUMENT;
  TC_TRY(check_shape(ctx, shape, m));
  return tcrt::interpolate_device(ctx, (Fe*)d_limbs, shape, m);
}

int tc_evaluate(tc_ctx* ctx, const uint32_t* d_coeffs, const uint32_t* shape, int m, const uint8_t* point_le21,
                uint8_t* out_y21) {
  if (!ctx || !d_coeffs || !shape || !point_le21 || !out_y21) return TC_ERR_ARGUMENT;
  TC_TRY(check_shape(ctx, shape, m));
  std::vector<Fe> pt(m);
  for (int j = 0; j < m; j++)
    if (!le21_to_fe(point_le21 + 21 * j, pt[j])) return fail(ctx, TC_ERR_VALUE, "point coordinate %d out of range", j);
  Fe y;
  TC_TRY(tcrt::evaluate_device(ctx, (const Fe*)d_coeffs, shape, m, pt.data(), &y));
  fe_to_le21(y, out_y21);
  return TC_OK;
}

int tc_open_quotients(tc_ctx* ctx, const uint32_t* d_coeffs, const uint32_t* shape, int m, const uint8_t* omega_le21,
                      uint32_t* d_quotients, uint8_t* out_y21) {
  if (!ctx || !d_coeffs || !shape || !omega_le21 || !d_quotients || !out_y21) return TC_ERR_ARGUMENT;
  TC_TRY(check_shape(ctx, shape, m));
  std::vector<Fe> om(m);
  for (int j = 0; j < m; j++)
    if (!le21_to_fe(omega_le21 + 21 * j, om[j])) return fail(ctx, TC_ERR_VALUE, "point coordinate %d out of range", j);
  Fe y;
  TC_TRY(tcrt::open_quotients_device(ctx, (const Fe*)d_coeffs, shape, m, om.data(), (Fe*)d_quotients, &y));
  fe_to_le21(y, out_y21);
  return TC_OK;
}

int tc_msm(tc_ctx* ctx, const tc_srs* srs, int which, const uint32_t* d_scalars, uint64_t n, uint8_t* out43) {
  if (!ctx || !srs || !out43 || (n && !d_scalars)) return TC_ERR_ARGUMENT;
  const EdPk* bases;
  TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), which, &bases));
  if (n > srs->n) return fail(ctx, TC_ERR_VALUE, "msm: %llu scalars for an srs of %llu elements",
                              (unsigned long long)n, (unsigned long long)srs->n);
  Aff* d_out;
  TC_TRY(tcrt::scratch_t(ctx, "msm.out", 1, &d_out));
  TC_TRY(tcrt::msm_device(ctx, tcrt::SCALAR_FP_CANON, d_scalars, bases, n, d_out));
  return fetch_encode(ctx, d_out, out43);
}

// copy L device results to the host (pinned staging) and encode them
static int fetch_encode_many(tc_ctx* ctx, const Aff* d_pts, int L, uint8_t* out43) {
  for (int base = 0; base < L;) {
    int k = std::min<int>(L - base, (int)(ctx->h_stage_bytes / sizeof(Aff)));
    TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_stage, d_pts + base, k * sizeof(Aff), cudaMemcpyDeviceToHost, ctx->stream));
    TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const Aff* h = (const Aff*)ctx->h_stage;
    for (int i = 0; i < k; i++) aff_encode43(h[i], out43 + 43 * (base + i));
    base += k;
  }
  return TC_OK;
}

// L MSMs over the SRS's `which` elements: the fixed-base table kernel for small SRSs
// (Terkle nodes), the batched Pippenger pipeline otherwise
static int msm_quotients(tc_ctx* ctx, const tc_srs* srs, const void* const* ptrs, int L, const EdPk* bases,
                         uint64_t n, Aff* d_out);

static int msm_srs(tc_ctx* ctx, const tc_srs* srs, int which, int dtype, int scale_bits, const void* const* ptrs,
                   int L, Aff* d_out) {
  if (!((which == TC_SRS_LAGRANGE) ? srs->lagrange : srs->monomial))
    return fail(ctx, TC_ERR_VALUE, "srs has no elements of kind %d", which);
  if (srs->n > SMALL_MSM_MAX) {
    const EdPk* bases;
    TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), which, &bases));
    // full-width field-element scalars (the monomial route's coefficients) over a large
    // basis: the fixed-base window table, as for the opening quotients (one shared window
    // of buckets, no Horner chain)
    static const bool no_fb = getenv("TC_COMMIT_NO_WINTAB") != nullptr;
    if (dtype == TC_DTYPE_FP_LIMBS && srs->n >= tcrt::FB_SMALL_N && !no_fb)
      return msm_quotients(ctx, srs, ptrs, L, bases, srs->n, d_out);
    return tcrt::msm_batch_device(ctx, dtype, scale_bits, ptrs, L, bases, srs->n, d_out, nullptr, 0,
                                  which == TC_SRS_LAGRANGE ? const_cast<tc_srs*>(srs) : nullptr);
  }
  std::vector<const void*> fp(ptrs, ptrs + L);
  if (dtype != TC_DTYPE_FP_LIMBS) {   // quantise first: the table kernel takes field elements
    Fe* q;
    TC_TRY(tcrt::scratch_t(ctx, "small.q_in", (uint64_t)L * srs->n, &q));
    for (int i = 0; i < L; i++) {
      TC_TRY(tcrt::quantize_device(ctx, ptrs[i], dtype, srs->n, scale_bits, q + (uint64_t)i * srs->n));
      fp[i] = q + (uint64_t)i * srs->n;
    }
  }
  return tcrt::small_msm_device(ctx, const_cast<tc_srs*>(srs), which, fp.data(), L, d_out);
}

// count tensors of the SRS shape in one batched MSM pipeline; points stay on the device
static int commit_many_dev(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                           int scale_bits, int route, Aff* d_out) {
  const uint64_t n = srs->n;
  bool lag = (route == TC_ROUTE_LAGRANGE) || (route == TC_ROUTE_AUTO && srs->lagrange);
  if (lag && !srs->lagrange) return fail(ctx, TC_ERR_VALUE, "srs has no Lagrange elements");
  if (!lag && !srs->monomial) return fail(ctx, TC_ERR_VALUE, "srs has no monomial elements");
  if (count == 0) return TC_OK;
  if (lag) {
    // C_T = sum_grid T[w] * g^{L_w(tau)}: no interpolation; the raw grid values (quantised
    // inside the digit kernel for float inputs) are the scalars
    TC_TRY(msm_srs(ctx, srs, TC_SRS_LAGRANGE, dtype, scale_bits, d_ins, count, d_out));
  } else {
    // SPEC.md:279 verbatim: interpolate every tensor, then MSM over the monomial SRS
    // groups of layers bound the coefficient scratch (config 5: 1 layer = 41.9M elements)
    const int G = (int)std::max<uint64_t>(1, (1ull << 24) / n);
    Fe* coeffs;
    TC_TRY(tcrt::scratch_t(ctx, "commit.coeffs", (uint64_t)std::min(G, count) * n, &coeffs));
    for (int g0 = 0; g0 < count; g0 += G) {
      const int gc = std::min(G, count - g0);
      std::vector<const void*> ptrs(gc);
      for (int i = 0; i < gc; i++) {
        Fe* dst = coeffs + (uint64_t)i * n;
        if (dtype == TC_DTYPE_FP_LIMBS) {
          TC_CUDA(ctx, cudaMemcpyAsync(dst, d_ins[g0 + i], n * sizeof(Fe), cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
          TC_TRY(tcrt::quantize_device(ctx, d_ins[g0 + i], dtype, n, scale_bits, dst));
        }
        TC_TRY(tcrt::interpolate_device(ctx, dst, srs->shape, srs->m));
        ptrs[i] = dst;
      }
      TC_TRY(msm_srs(ctx, srs, TC_SRS_MONOMIAL, TC_DTYPE_FP_LIMBS, 0, ptrs.data(), gc, d_out + g0));
    }
  }
  return TC_OK;
}

static int commit_many(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype, int scale_bits,
                       int route, uint8_t* out43) {
  if (count == 0) return commit_many_dev(ctx, srs, d_ins, 0, dtype, scale_bits, route, nullptr);
  Aff* d_out;
  TC_TRY(tcrt::scratch_t(ctx, "commit.out", (uint64_t)count, &d_out));
  TC_TRY(commit_many_dev(ctx, srs, d_ins, count, dtype, scale_bits, route, d_out));
  return fetch_encode_many(ctx, d_out, count, out43);
}

// Terkle geometry for n leaves over a node SRS of B points: L levels, cap = B^L slots,
// node count and child-value count over all levels
static void terkle_geometry(uint64_t n, uint64_t B, uint64_t& L, uint64_t& cap, uint64_t& nodes, uint64_t& values) {
  L = 1, cap = B;
  while (cap < n) cap *= B, L++;
  nodes = 0, values = 0;
  uint64_t w = cap;
  for (uint64_t l = 0; l < L; l++) values += w, w /= B, nodes += w;
}

// Pipeline contexts (tc_ctx_set_pipelined): the forward's post-accumulation tail runs on a
// low-priority stream of the context (msm_batch_device switches to it after the level-0
// accumulation when tail_split is set), so other forwards' sort and accumulation blocks are
// dispatched first.  tail_end orders the context's own stream after the tail.
static int tail_begin(tc_ctx* ctx) {
  static const bool split = getenv("TC_TAIL_SPLIT") ? atoi(getenv("TC_TAIL_SPLIT")) != 0 : true;
  if (!split || !ctx->pipelined) return TC_OK;
  if (!ctx->tail_stream) {
    int lo = 0, hi = 0;
    TC_CUDA(ctx, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TC_CUDA(ctx, cudaStreamCreateWithPriority(&ctx->tail_stream, cudaStreamNonBlocking, lo));
  }
  ctx->tail_split = true;
  return TC_OK;
}

static int tail_end(tc_ctx* ctx, cudaStream_t home) {
  ctx->tail_split = false;
  if (ctx->stream == home) return TC_OK;
  const cudaStream_t tail = ctx->stream;
  ctx->stream = home;
  if (!ctx->ev_tail) TC_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_tail, cudaEventDisableTiming));
  TC_CUDA(ctx, cudaEventRecord(ctx->ev_tail, tail));
  TC_CUDA(ctx, cudaStreamWaitEvent(home, ctx->ev_tail, 0));
  return TC_OK;
}

// commit + leaves + tree on the ctx stream; the results are copied (asynchronously) into the
// ctx's pinned result buffer and `res_ev` recorded — tc_commit_tree_finish collects them
static int commit_tree_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                              int scale_bits, int route, const tc_srs* node_srs) {
  if (!ctx || !srs || !d_ins || !node_srs) return TC_ERR_ARGUMENT;
  if (count <= 0) return fail(ctx, TC_ERR_VALUE, "empty leaf list");
  if (ctx->res_pending) return fail(ctx, TC_ERR_VALUE, "commit_tree: previous launch not finished on this context");
  const uint64_t B = node_srs->n;
  if (B < 2) return fail(ctx, TC_ERR_VALUE, "tree arity must be >= 2");
  if (!node_srs->lagrange || B > SMALL_MSM_MAX)
    return fail(ctx, TC_ERR_VALUE, "device tree needs a Lagrange node SRS of <= %llu points",
                (unsigned long long)SMALL_MSM_MAX);
  uint64_t L, cap, total_nodes, total_values;
  terkle_geometry((uint64_t)count, B, L, cap, total_nodes, total_values);
  // commitments and node points in one buffer (one readback), leaves and level values
  Aff* d_all;
  Fe *d_vals, *d_levels;
  TC_TRY(tcrt::scratch_t(ctx, "tree.pts", (uint64_t)count + total_nodes, &d_all));
  TC_TRY(tcrt::scratch_t(ctx, "tree.vals", cap, &d_vals));
  TC_TRY(tcrt::scratch_t(ctx, "tree.levels", total_values, &d_levels));
  // the MSM batch hands over its window sums (deferred finish) so the commitments, leaves
  // and every tree level run as ONE single-block tail kernel; any other MSM plan writes the
  // points and the tree runs level by level
  static const bool no_tail = getenv("TC_NO_TREE_TAIL") != nullptr;
  ctx->defer_req = !no_tail && cap <= 1024;
  ctx->defer_wsum = nullptr;
  // pipeline contexts: the post-accumulation tail on the low-priority stream (tail_begin);
  // the context's stream is restored below, ordered after it
  cudaStream_t home = ctx->stream;
  TC_TRY(tail_begin(ctx));
  const int cs = commit_many_dev(ctx, srs, d_ins, count, dtype, scale_bits, route, d_all);
  ctx->defer_req = false;
  ctx->tail_split = false;
  if (cs) {
    ctx->stream = home;
    return cs;
  }
  if (ctx->defer_wsum) {
    if (ctx->defer_L != count) return fail(ctx, TC_ERR_VALUE, "deferred finish: %d of %d MSMs", ctx->defer_L, count);
    TC_TRY(tcrt::tree_tail_device(ctx, const_cast<tc_srs*>(node_srs), ctx->defer_wsum, count, ctx->defer_nwin, cap,
                                  (int)L, d_all, d_levels));
    ctx->defer_wsum = nullptr;
  } else {
    TC_TRY(tcrt::leaf_hash_device(ctx, d_all, count, cap, d_vals));
    TC_TRY(tcrt::terkle_device(ctx, const_cast<tc_srs*>(node_srs), d_vals, cap, (int)L, d_all + count, d_levels));
  }
  const size_t pts_b = (size_t)(count + total_nodes) * sizeof(Aff), vals_b = (size_t)total_values * sizeof(Fe);
  if (ctx->h_res_bytes < pts_b + vals_b) {
    if (ctx->h_res) cudaFreeHost(ctx->h_res);
    ctx->h_res = nullptr;
    ctx->h_res_bytes = 0;
    TC_CUDA(ctx, cudaHostAlloc(&ctx->h_res, pts_b + vals_b, cudaHostAllocDefault));
    ctx->h_res_bytes = pts_b + vals_b;
  }
  if (!ctx->res_ev) TC_CUDA(ctx, cudaEventCreateWithFlags(&ctx->res_ev, cudaEventDisableTiming));
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_res, d_all, pts_b, cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaMemcpyAsync((char*)ctx->h_res + pts_b, d_levels, vals_b, cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaEventRecord(ctx->res_ev, ctx->stream));
  if (ctx->stream != home) {   // back on the context's own stream, ordered after the tail
    TC_CUDA(ctx, cudaStreamWaitEvent(home, ctx->res_ev, 0));
    ctx->stream = home;
  }
  ctx->res_pending = true;
  ctx->res_count = (uint64_t)count, ctx->res_nodes = total_nodes, ctx->res_values = total_values;
  return TC_OK;
}

int tc_commit_tree_finish(tc_ctx* ctx, uint8_t* out_comms43, uint8_t* out_nodes43, uint64_t* inout_node_count,
                          uint8_t* out_values24, uint64_t* inout_value_count) {
  if (!ctx || !out_comms43 || !out_nodes43 || !inout_node_count || !out_values24 || !inout_value_count)
    return TC_ERR_ARGUMENT;
  if (!ctx->res_pending) return fail(ctx, TC_ERR_VALUE, "commit_tree: nothing launched on this context");
  if (*inout_node_count < ctx->res_nodes || *inout_value_count < ctx->res_values)
    return fail(ctx, TC_ERR_VALUE, "need room for %llu nodes and %llu values", (unsigned long long)ctx->res_nodes,
                (unsigned long long)ctx->res_values);
  TC_CUDA(ctx, cudaEventSynchronize(ctx->res_ev));
  ctx->res_pending = false;
  const Aff* pts = (const Aff*)ctx->h_res;
  for (uint64_t i = 0; i < ctx->res_count; i++) aff_encode43(pts[i], out_comms43 + 43 * i);
  for (uint64_t i = 0; i < ctx->res_nodes; i++) aff_encode43(pts[ctx->res_count + i], out_nodes43 + 43 * i);
  memcpy(out_values24, (const char*)ctx->h_res + (ctx->res_count + ctx->res_nodes) * sizeof(Aff),
         ctx->res_values * sizeof(Fe));
  *inout_node_count = ctx->res_nodes;
  *inout_value_count = ctx->res_values;
  return TC_OK;
}

int tc_commit_tree_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                          int scale_bits, int route, const tc_srs* node_srs) {
  return commit_tree_launch(ctx, srs, d_ins, count, dtype, scale_bits, route, node_srs);
}

// ---- multi-GPU building blocks (dist.py) ----------------------------------------------
// Each rank commits its share of the (layer, element) space — whole layers, or a layer's
// contiguous chunk given as a zero-masked copy (a Lagrange-route commitment is linear in
// the samples, so a chunk's MSM is a partial sum of the layer's commitment) — into device
// encodings; ONE all-gather exchanges them; every rank then sums the partials per layer
// and hashes the tree on the device.
int tc_commit_points_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                            int scale_bits, int route, uint8_t* d_out43) {
  if (!ctx || !srs || (count > 0 && (!d_ins || !d_out43)) || count < 0) return TC_ERR_ARGUMENT;
  if (count == 0) return TC_OK;
  Aff* d_pts;
  TC_TRY(tcrt::scratch_t(ctx, "dist.pts", (uint64_t)count, &d_pts));
  cudaStream_t home = ctx->stream;
  TC_TRY(tail_begin(ctx));
  const int cs = commit_many_dev(ctx, srs, d_ins, count, dtype, scale_bits, route, d_pts);
  ctx->tail_split = false;
  if (!cs) {
    k_encode43<<<tcrt::blocks_for(count, 64), 64, 0, ctx->stream>>>(d_pts, count, d_out43);
    TC_LAUNCHED(ctx);
  }
  const int te = tail_end(ctx, home);
  return cs ? cs : te;
}

// sum the partial points of each layer (CSR offsets `off`, n_layers + 1 entries)
__global__ void k_combine_parts(const Aff* parts, const uint32_t* off, int n_layers, Aff* out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n_layers) return;
  const uint32_t a = off[l], b = off[l + 1];
  if (b - a == 1) {
    out[l] = parts[a];
    return;
  }
  Xyzz acc = xyzz_inf();
  for (uint32_t k = a; k < b; k++) xyzz_add_aff(acc, parts[k]);
  Aff r = xyzz_to_aff(acc);
  if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
  out[l] = r;
}

int tc_tree_from_points_launch(tc_ctx* ctx, const tc_srs* node_srs, const uint8_t* d_parts43,
                               const uint32_t* layer_of, uint64_t nparts, int n_layers) {
  if (!ctx || !node_srs || !d_parts43 || nparts == 0 || n_layers <= 0) return TC_ERR_ARGUMENT;
  if (ctx->res_pending) return fail(ctx, TC_ERR_VALUE, "commit_tree: previous launch not finished on this context");
  const uint64_t B = node_srs->n;
  if (B < 2 || !node_srs->lagrange || B > SMALL_MSM_MAX)
    return fail(ctx, TC_ERR_VALUE, "device tree needs a Lagrange node SRS of 2..%llu points",
                (unsigned long long)SMALL_MSM_MAX);
  // CSR offsets of the parts per layer (parts of one layer must be adjacent, layers ascending)
  std::vector<uint32_t> off(n_layers + 1, 0);
  if (layer_of) {
    if (nparts > (1ull << 20)) return fail(ctx, TC_ERR_VALUE, "too many parts");
    for (uint64_t k = 0; k < nparts; k++) {
      const uint32_t l = layer_of[k];
      if (l >= (uint32_t)n_layers || (k && l < layer_of[k - 1]))
        return fail(ctx, TC_ERR_VALUE, "parts must be grouped by ascending layer (< %d)", n_layers);
      off[l + 1]++;
    }
    for (int l = 0; l < n_layers; l++) {
      if (!off[l + 1]) return fail(ctx, TC_ERR_VALUE, "layer %d has no part", l);
      off[l + 1] += off[l];
    }
  } else {
    if (nparts != (uint64_t)n_layers) return fail(ctx, TC_ERR_VALUE, "one part per layer expected");
    for (int l = 0; l <= n_layers; l++) off[l] = (uint32_t)l;
  }
  uint64_t L, cap, total_nodes, total_values;
  terkle_geometry((uint64_t)n_layers, B, L, cap, total_nodes, total_values);
  Aff *d_parts, *d_all;
  Fe *d_vals, *d_levels;
  uint32_t* d_off;
  TC_TRY(tcrt::scratch_t(ctx, "dist.parts", nparts, &d_parts));
  TC_TRY(tcrt::scratch_t(ctx, "dist.off", (uint64_t)n_layers + 1, &d_off));
  TC_TRY(tcrt::scratch_t(ctx, "tree.pts", (uint64_t)n_layers + total_nodes, &d_all));
  TC_TRY(tcrt::scratch_t(ctx, "tree.vals", cap, &d_vals));
  TC_TRY(tcrt::scratch_t(ctx, "tree.levels", total_values, &d_levels));
  // the offsets go up through a pinned buffer of this ctx used by nothing else: its previous
  // upload belonged to the previous launch on this ctx, which tc_commit_tree_finish waited
  // for — no stream synchronisation here, so the launch stays asynchronous
  const size_t off_b = sizeof(uint32_t) * off.size();
  if (ctx->h_off_bytes < off_b) {
    if (ctx->h_off) cudaFreeHost(ctx->h_off);
    ctx->h_off = nullptr;
    ctx->h_off_bytes = 0;
    TC_CUDA(ctx, cudaHostAlloc(&ctx->h_off, off_b, cudaHostAllocDefault));
    ctx->h_off_bytes = off_b;
  }
  memcpy(ctx->h_off, off.data(), off_b);
  TC_CUDA(ctx, cudaMemcpyAsync(d_off, ctx->h_off, off_b, cudaMemcpyHostToDevice, ctx->stream));
  TC_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream));
  k_decode43<<<tcrt::blocks_for(nparts, 64), 64, 0, ctx->stream>>>(d_parts43, nparts, d_parts, ctx->d_flags);
  TC_LAUNCHED(ctx);
  k_combine_parts<<<tcrt::blocks_for(n_layers, 32), 32, 0, ctx->stream>>>(d_parts, d_off, n_layers, d_all);
  TC_LAUNCHED(ctx);
  TC_TRY(tcrt::leaf_hash_device(ctx, d_all, n_layers, cap, d_vals));
  TC_TRY(tcrt::terkle_device(ctx, const_cast<tc_srs*>(node_srs), d_vals, cap, (int)L, d_all + n_layers, d_levels));
  const size_t pts_b = (size_t)(n_layers + total_nodes) * sizeof(Aff), vals_b = (size_t)total_values * sizeof(Fe);
  if (ctx->h_res_bytes < pts_b + vals_b) {
    if (ctx->h_res) cudaFreeHost(ctx->h_res);
    ctx->h_res = nullptr;
    ctx->h_res_bytes = 0;
    TC_CUDA(ctx, cudaHostAlloc(&ctx->h_res, pts_b + vals_b, cudaHostAllocDefault));
    ctx->h_res_bytes = pts_b + vals_b;
  }
  if (!ctx->res_ev) TC_CUDA(ctx, cudaEventCreateWithFlags(&ctx->res_ev, cudaEventDisableTiming));
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_res, d_all, pts_b, cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaMemcpyAsync((char*)ctx->h_res + pts_b, d_levels, vals_b, cudaMemcpyDeviceToHost, ctx->stream));
  TC_CUDA(ctx, cudaEventRecord(ctx->res_ev, ctx->stream));
  ctx->res_pending = true;
  ctx->res_count = (uint64_t)n_layers, ctx->res_nodes = total_nodes, ctx->res_values = total_values;
  return TC_OK;
}

static int commit_tree_impl(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                            int scale_bits, int route, const tc_srs* node_srs, uint8_t* out_comms43,
                            uint8_t* out_nodes43, uint64_t* inout_node_count, uint8_t* out_values24,
                            uint64_t* inout_value_count) {
  if (!out_comms43 || !out_nodes43 || !inout_node_count || !out_values24 || !inout_value_count)
    return TC_ERR_ARGUMENT;
  TC_TRY(commit_tree_launch(ctx, srs, d_ins, count, dtype, scale_bits, route, node_srs));
  return tc_commit_tree_finish(ctx, out_comms43, out_nodes43, inout_node_count, out_values24, inout_value_count);
}

int tc_commit_tree(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype, int scale_bits,
                   int route, const tc_srs* node_srs, uint8_t* out_comms43, uint8_t* out_nodes43,
                   uint64_t* inout_node_count, uint8_t* out_values24, uint64_t* inout_value_count) {
  return commit_tree_impl(ctx, srs, d_ins, count, dtype, scale_bits, route, node_srs, out_comms43, out_nodes43,
                          inout_node_count, out_values24, inout_value_count);
}

int tc_commit(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits, int route, uint8_t* out43) {
  if (!ctx || !srs || !d_in || !out43) return TC_ERR_ARGUMENT;
  const void* ptrs[1] = {d_in};
  return commit_many(ctx, srs, ptrs, 1, dtype, scale_bits, route, out43);
}

int tc_commit_batch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype, int scale_bits,
                    int route, uint8_t* out43) {
  if (!ctx || !srs || !d_ins || !out43 || count < 0) return TC_ERR_ARGUMENT;
  return commit_many(ctx, srs, d_ins, count, dtype, scale_bits, route, out43);
}

static int dtype_size(int dtype, size_t* esz) {
  switch (dtype) {
    case TC_DTYPE_F16: case TC_DTYPE_BF16: *esz = 2; return TC_OK;
    case TC_DTYPE_F32: *esz = 4; return TC_OK;
    case TC_DTYPE_F64: *esz = 8; return TC_OK;
    case TC_DTYPE_FP_LIMBS: *esz = sizeof(Fe); return TC_OK;
    default: return TC_ERR_ARGUMENT;
  }
}

static int ensure_copy_stream(tc_ctx* ctx) {
  if (!ctx->copy_stream) TC_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  return TC_OK;
}

// Host-resident inputs: the layers are uploaded on a copy stream in groups of `group`
// (0 = one group) and the ctx stream commits each group once it is resident.  Splitting a
// forward into several MSM batches was measured SLOWER on config 3 (groups of 8: +3.4 ms of
// per-batch reduction tails for 1.9 ms of hidden upload), so the default is one group; the
// overlap that pays is across forwards (tc_commit_stream).
int tc_commit_batch_host(tc_ctx* ctx, const tc_srs* srs, const void* const* h_ins, int count, int dtype,
                         int scale_bits, int route, int group, uint8_t* out43) {
  if (!ctx || !srs || !h_ins || !out43 || count < 0 || group < 0) return TC_ERR_ARGUMENT;
  if (count == 0) return TC_OK;
  size_t esz;
  if (dtype_size(dtype, &esz)) return fail(ctx, TC_ERR_ARGUMENT, "commit_batch_host: unsupported dtype %d", dtype);
  for (int i = 0; i < count; i++)
    if (!h_ins[i]) return TC_ERR_ARGUMENT;
  static const int G_ENV = getenv("TC_PIPE_GROUP") ? atoi(getenv("TC_PIPE_GROUP")) : 0;
  int G = group ? group : (G_ENV > 0 ? G_ENV : count);
  G = std::min(G, count);
  const int ngroups = (count + G - 1) / G;
  const size_t bytes = (size_t)srs->n * esz;
  uint8_t* stage;
  TC_TRY(tcrt::scratch(ctx, "host.stage", bytes * count, (void**)&stage));
  TC_TRY(ensure_copy_stream(ctx));
  while ((int)ctx->copy_ev.size() < ngroups) {
    cudaEvent_t e;
    TC_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->copy_ev.push_back(e);
  }
  // the staging buffer may still be read by earlier work on the ctx stream
  TC_CUDA(ctx, cudaEventRecord(ctx->copy_ev[0], ctx->stream));
  TC_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[0], 0));
  for (int g = 0; g < ngroups; g++) {
    for (int i = g * G; i < std::min(count, (g + 1) * G); i++)
      TC_CUDA(ctx, cudaMemcpyAsync(stage + bytes * i, h_ins[i], bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
    TC_CUDA(ctx, cudaEventRecord(ctx->copy_ev[g], ctx->copy_stream));
  }
  std::vector<const void*> ptrs(count);
  for (int i = 0; i < count; i++) ptrs[i] = stage + bytes * i;
  for (int g = 0; g < ngroups; g++) {
    const int g0 = g * G, gc = std::min(G, count - g0);
    TC_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->copy_ev[g], 0));
    TC_TRY(commit_many(ctx, srs, ptrs.data() + g0, gc, dtype, scale_bits, route, out43 + 43 * (size_t)g0));
  }
  return TC_OK;
}

// upload `count` host tensors into stream slot s (copy stream), record its ready event
static int slot_upload(tc_ctx* ctx, int s, const void* const* h, int count, int dtype, uint64_t n, size_t esz) {
  auto& sl = ctx->slot[s];
  uint8_t* dst;
  TC_TRY(tcrt::scratch(ctx, s ? "stream.slot1" : "stream.slot0", (size_t)n * esz * count, (void**)&dst));
  if (!sl.ready) TC_CUDA(ctx, cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
  for (int i = 0; i < count; i++)
    TC_CUDA(ctx, cudaMemcpyAsync(dst + (size_t)n * esz * i, h[i], (size_t)n * esz, cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
  TC_CUDA(ctx, cudaEventRecord(sl.ready, ctx->copy_stream));
  sl.host.assign(h, h + count);
  sl.dtype = dtype;
  sl.n = n;
  sl.valid = true;
  return TC_OK;
}

// Streaming commits, one call per forward: commits h_cur and, before the commit starts,
// enqueues the upload of h_next (the next forward's activations; may be NULL) on the copy
// stream, so the PCIe transfer of forward k+1 runs under the MSMs of forward k.  h_cur is
// consumed from the slot a previous call prefetched it into (same pointers, count, dtype),
// else uploaded now.  Host buffers passed as h_next must not change until the call that
// commits them returns.
// device pointers of this forward's tensors (from the prefetched slot, or uploaded now) and
// the next forward's upload started on the copy stream
static int stream_prepare(tc_ctx* ctx, const tc_srs* srs, const void* const* h_cur, const void* const* h_next,
                          int count, int dtype, std::vector<const void*>& ptrs) {
  size_t esz;
  if (dtype_size(dtype, &esz)) return fail(ctx, TC_ERR_ARGUMENT, "commit_stream: unsupported dtype %d", dtype);
  for (int i = 0; i < count; i++)
    if (!h_cur[i] || (h_next && !h_next[i])) return TC_ERR_ARGUMENT;
  TC_TRY(ensure_copy_stream(ctx));
  const uint64_t n = srs->n;
  int s = -1;
  for (int k = 0; k < 2 && s < 0; k++) {
    const auto& sl = ctx->slot[k];
    if (sl.valid && sl.dtype == dtype && sl.n == n && (int)sl.host.size() == count &&
        std::equal(sl.host.begin(), sl.host.end(), h_cur))
      s = k;
  }
  if (s < 0) {
    // h_cur is not a pending prefetch: any prefetched slot belongs to a stream of forwards
    // that was abandoned (its buffers may be reused with other contents), drop both
    ctx->slot[0].valid = ctx->slot[1].valid = false;
    s = 0;
    // slot 0 may still be read by earlier work on the ctx stream
    if (!ctx->slot[0].ready) TC_CUDA(ctx, cudaEventCreateWithFlags(&ctx->slot[0].ready, cudaEventDisableTiming));
    TC_CUDA(ctx, cudaEventRecord(ctx->slot[0].ready, ctx->stream));
    TC_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->slot[0].ready, 0));
    TC_TRY(slot_upload(ctx, 0, h_cur, count, dtype, n, esz));
  }
  uint8_t* cur;
  TC_TRY(tcrt::scratch(ctx, s ? "stream.slot1" : "stream.slot0", (size_t)n * esz * count, (void**)&cur));
  TC_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->slot[s].ready, 0));
  ctx->slot[s].valid = false;   // consumed by this call
  if (h_next) {
    // the other slot was last read by a previous call, which finished (commits end with a
    // host synchronisation); order the copy after everything on the ctx stream anyway
    auto& o = ctx->slot[1 - s];
    if (!o.ready) TC_CUDA(ctx, cudaEventCreateWithFlags(&o.ready, cudaEventDisableTiming));
    TC_CUDA(ctx, cudaEventRecord(o.ready, ctx->stream));
    TC_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, o.ready, 0));
    TC_TRY(slot_upload(ctx, 1 - s, h_next, count, dtype, n, esz));
  }
  ptrs.resize(count);
  for (int i = 0; i < count; i++) ptrs[i] = cur + (size_t)n * esz * i;
  return TC_OK;
}

int tc_commit_stream_reset(tc_ctx* ctx) {
  if (!ctx) return TC_ERR_ARGUMENT;
  ctx->slot[0].valid = ctx->slot[1].valid = false;
  return TC_OK;
}

int tc_commit_stream(tc_ctx* ctx, const tc_srs* srs, const void* const* h_cur, const void* const* h_next, int count,
                     int dtype, int scale_bits, int route, uint8_t* out43) {
  if (!ctx || !srs || !h_cur || !out43 || count < 0) return TC_ERR_ARGUMENT;
  if (count == 0) return TC_OK;
  std::vector<const void*> ptrs;
  TC_TRY(stream_prepare(ctx, srs, h_cur, h_next, count, dtype, ptrs));
  return commit_many(ctx, srs, ptrs.data(), count, dtype, scale_bits, route, out43);
}

int tc_commit_stream_tree_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* h_cur, int count, int dtype,
                                 int scale_bits, int route, const tc_srs* node_srs) {
  if (!ctx || !srs || !h_cur || count <= 0) return TC_ERR_ARGUMENT;
  if (ctx->res_pending) return fail(ctx, TC_ERR_VALUE, "commit_tree: previous launch not finished on this context");
  std::vector<const void*> ptrs;
  TC_TRY(stream_prepare(ctx, srs, h_cur, nullptr, count, dtype, ptrs));
  return commit_tree_launch(ctx, srs, ptrs.data(), count, dtype, scale_bits, route, node_srs);
}

int tc_commit_stream_tree(tc_ctx* ctx, const tc_srs* srs, const void* const* h_cur, const void* const* h_next,
                          int count, int dtype, int scale_bits, int route, const tc_srs* node_srs,
                          uint8_t* out_comms43, uint8_t* out_nodes43, uint64_t* inout_node_count,
                          uint8_t* out_values24, uint64_t* inout_value_count) {
  if (!ctx || !srs || !h_cur || count <= 0) return TC_ERR_ARGUMENT;
  std::vector<const void*> ptrs;
  TC_TRY(stream_prepare(ctx, srs, h_cur, h_next, count, dtype, ptrs));
  return commit_tree_impl(ctx, srs, ptrs.data(), count, dtype, scale_bits, route, node_srs, out_comms43,
                          out_nodes43, inout_node_count, out_values24, inout_value_count);
}

// L_k(omega_a) (canonical) and 1 / (k + 1 - omega_a) for every axis, concatenated
// barycentric weights w_i = 1 / prod_{t != i} (x_i - x_t) of the default grid x = 1..d and
// their inverses, both in Montgomery form, cached per extent
static const std::pair<std::vector<Fe>, std::vector<Fe>>& bary_weights(uint32_t d) {
  static std::mutex mu;
  static std::map<uint32_t, std::pair<std::vector<Fe>, std::vector<Fe>>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(d);
  if (it != cache.end()) return it->second;
  std::vector<Fe> w(d), winv(d);
  for (uint32_t i = 0; i < d; i++) {
    Fe prod = Fp::one();
    for (uint32_t t = 0; t < d; t++) {
      if (t == i) continue;
      const Fe diff = Fp::sub(Fp::to_mont_small(i + 1), Fp::to_mont_small(t + 1));
      prod = Fp::mul(prod, diff);
    }
    winv[i] = Fp::canon(prod);
    w[i] = Fp::canon(Fp::inv_fast(prod));
  }
  return cache.emplace(d, std::make_pair(w, winv)).first->second;
}

// MSM of canonical F_p scalars (opening quotients) over an SRS base range: through the
// range's fixed-base window table (one shared bucket window, no Horner chain; built on first
// use) when the table fits the budget, else the windowed Pippenger pipeline.
static int msm_quotients(tc_ctx* ctx, const tc_srs* srs, const void* const* ptrs, int L, const EdPk* bases,
                         uint64_t n, Aff* d_out) {
  static const uint64_t BUDGET = getenv("TC_WINTAB_MB") ? strtoull(getenv("TC_WINTAB_MB"), nullptr, 10) << 20
                                                        : (4096ull << 20);
  const int c = tcrt::fb_width(n);
  if (n * tcrt::fb_ndig(c) * sizeof(EdPk) <= BUDGET) {
    const EdPk* tab;
    TC_TRY(tcrt::srs_window_table(ctx, const_cast<tc_srs*>(srs), bases, n, &tab));
    return tcrt::msm_batch_device(ctx, TC_DTYPE_FP_LIMBS, 0, ptrs, L, tab, n, d_out, nullptr, c);
  }
  return tcrt::msm_batch_device(ctx, TC_DTYPE_FP_LIMBS, 0, ptrs, L, bases, n, d_out);
}

// Lagrange-route opening weights for every axis (see tcrt::LagW)
static void lag_weights(const tc_srs* srs, const std::vector<Fe>& om, tcrt::LagW& W) {
  W.lam.clear();
  W.inv.clear();
  W.der.clear();
  W.sj.assign(srs->m, -1);
  for (int a = 0; a < srs->m; a++) {
    const uint32_t d = srs->shape[a];
    int j = -1;   // omega_a = x_j ?
    for (uint32_t k = 0; k < d && j < 0; k++) {
      Fe z{{k + 1, 0, 0, 0, 0, 0}};
      if (memcmp(z.v, om[a].v, sizeof z.v) == 0) j = (int)k;
    }
    W.sj[a] = j;
    std::vector<Fe> la;
    axis_tables(om[a], d, true, la);   // L_k(omega_a), canonical (one-hot on a node)
    const Fe w = Fp::to_mont(om[a]);
    std::vector<Fe> diff(d), pref(d);
    Fe run = Fp::one();
    for (uint32_t k = 0; k < d; k++) {
      diff[k] = (int)k == j ? Fp::one() : Fp::sub(Fp::to_mont_small(k + 1), w);   // x_k - omega
      pref[k] = run;
      run = Fp::mul(run, diff[k]);
    }
    Fe iv = Fp::inv_fast(run);
    std::vector<Fe> ik(d);
    for (int k = (int)d - 1; k >= 0; k--) {
      ik[k] = Fp::canon(Fp::mul(iv, pref[k]));
      iv = Fp::mul(iv, diff[k]);
    }
    std::vector<Fe> dk(d, Fp::zero());
    if (j >= 0) {
      // L_i'(x_j) = (w_i / w_j) / (x_j - x_i) = -(w_i / w_j) inv[i]  (i != j),
      // L_j'(x_j) = sum_{i != j} 1 / (x_j - x_i) = -sum_{i != j} inv[i]
      ik[j] = Fp::zero();
      const auto& bw = bary_weights(d);
      const Fe wj_inv = bw.second[j];
      Fe sum = Fp::zero();
      for (uint32_t i = 0; i < d; i++) {
        if ((int)i == j) continue;
        dk[i] = Fp::canon(Fp::neg(Fp::mul(Fp::mul(bw.first[i], wj_inv), ik[i])));   // all Montgomery
        sum = Fp::add(sum, ik[i]);
      }
      dk[j] = Fp::canon(Fp::neg(sum));
    }
    for (uint32_t k = 0; k < d; k++) W.lam.push_back(Fp::canon(Fp::to_mont(la[k])));
    W.inv.insert(W.inv.end(), ik.begin(), ik.end());
    W.der.insert(W.der.end(), dk.begin(), dk.end());
  }
}

int tc_open(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits, const uint8_t* omega_le21,
            int route, uint8_t* out_y21, uint8_t* out_pi43) {
  if (!ctx || !srs || !d_in || !omega_le21 || !out_y21 || !out_pi43) return TC_ERR_ARGUMENT;
  const uint64_t n = srs->n;
  const int m = srs->m;
  std::vector<Fe> om(m);
  for (int j = 0; j < m; j++)
    if (!le21_to_fe(omega_le21 + 21 * j, om[j])) return fail(ctx, TC_ERR_VALUE, "point coordinate %d out of range", j);
  Fe* vals;
  TC_TRY(load_field_tensor(ctx, d_in, dtype, n, scale_bits, &vals, "open.vals"));
  // Lagrange route: quotients evaluated on the grid straight from the samples (no
  // interpolation), committed over the (sub-grid) Lagrange elements.  On an axis where
  // omega is a grid node x_j (verifier challenges are grid points) the
  // quotient's value at x_j is the derivative of the fibre interpolant, a contraction with
  // the weights L_i'(x_j) (lag_weights).
  const bool lag_ok = srs->lagrange && (m == 1 || srs->sublag);
  // tiny SRSs (Terkle nodes): the monomial route's quotients go to the fixed-base table
  // kernel in one call; the Lagrange route would run m Pippenger pipelines
  if (route == TC_ROUTE_AUTO && n <= SMALL_MSM_MAX && srs->monomial) route = TC_ROUTE_MONOMIAL;
  if (route == TC_ROUTE_LAGRANGE && !lag_ok)
    return fail(ctx, TC_ERR_VALUE, "srs has no Lagrange elements");
  if (lag_ok && route != TC_ROUTE_MONOMIAL) {
    tcrt::LagW W;
    lag_weights(srs, om, W);
    Fe* qs;
    TC_TRY(tcrt::scratch_t(ctx, "open.q", (uint64_t)m * n, &qs));
    Fe y;
    TC_TRY(tcrt::open_quotients_lagrange_device(ctx, vals, srs->shape, m, W, qs, &y));
    fe_to_le21(y, out_y21);
    Aff* d_out;
    TC_TRY(tcrt::scratch_t(ctx, "open.out", (uint64_t)m, &d_out));
    uint64_t span = n;
    const EdPk *ed_lag, *ed_sub = nullptr;
    TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), TC_SRS_LAGRANGE, &ed_lag));
    if (m > 1) TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), 0, &ed_sub));
    for (int a = 0; a < m; a++) {
      const EdPk* bases = a == 0 ? ed_lag : ed_sub + srs->sublag_off[a];
      const void* ptr = qs + (uint64_t)a * n;
      TC_TRY(msm_quotients(ctx, srs, &ptr, 1, bases, span, d_out + a));
      span /= srs->shape[a];
    }
    return fetch_encode_many(ctx, d_out, m, out_pi43);
  }
  if (!srs->monomial) return fail(ctx, TC_ERR_VALUE, "tc_open needs the monomial srs");
  TC_TRY(tcrt::interpolate_device(ctx, vals, srs->shape, m));
  Fe* qs;
  TC_TRY(tcrt::scratch_t(ctx, "open.q", (uint64_t)m * n, &qs));
  Fe y;
  TC_TRY(tcrt::open_quotients_device(ctx, vals, srs->shape, m, om.data(), qs, &y));
  fe_to_le21(y, out_y21);
  // the m quotient MSMs in one batch (quotient a is zero outside its lex-prefix support,
  // and zero scalars emit no bucket entries)
  Aff* d_out;
  TC_TRY(tcrt::scratch_t(ctx, "open.out", (uint64_t)m, &d_out));
  std::vector<const void*> ptrs(m);
  for (int a = 0; a < m; a++) ptrs[a] = qs + (uint64_t)a * n;
  TC_TRY(msm_srs(ctx, srs, TC_SRS_MONOMIAL, TC_DTYPE_FP_LIMBS, 0, ptrs.data(), m, d_out));
  return fetch_encode_many(ctx, d_out, m, out_pi43);
}

// Many openings against one SRS (config 4).  Two batched strategies, both exact:
//  * grouped: the Lagrange-route quotients of up to G openings are evaluated, then every
//    axis a runs ONE batched MSM over the (sub-grid) Lagrange bases shared by all of them,
//    so the per-MSM fixed costs are paid once per group;
//  * slice commitments (a tensor opened >= TC_OPEN_PRECOMP_MIN times, m >= 2): with
//    R = N / d_0, H[c', c] = sum_rest T[c', rest] G[c, rest] (d_0^2 small-scalar MSMs over
//    the slices of the Lagrange SRS, computed once per tensor as one multi-base batch), and
//    pi_0 = sum_{c, c'} (delta_{c c'} - L_c'(omega_0)) / (c + 1 - omega_0) * H[c', c]
//    (the axis-0 quotient q_0(a) = (T[a] - sum_c' L_c'(omega_0) T[c', a_rest]) / (a_0 + 1
//    - omega_0), regrouped) — a d_0^2-point MSM per opening instead of an N-point one.
// route = monomial goes through tc_open (interpolation + monomial SRS) per opening.
// H[c', c] for the tensor slices c' in [row_lo, row_hi) over every SRS slice c (the
// slice-commitment route's d0 x d0 MSMs of n / d0 points, multi-base batch) into out
static int slice_commitments(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits,
                             uint32_t row_lo, uint32_t row_hi, Aff* out) {
  const EdPk* ed_lag;
  TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), TC_SRS_LAGRANGE, &ed_lag));
  size_t esz = 0;
  if (dtype_size(dtype, &esz)) return fail(ctx, TC_ERR_ARGUMENT, "open: unsupported dtype %d", dtype);
  const uint32_t d0 = srs->shape[0];
  const uint64_t R = srs->n / d0;
  const uint32_t nh = (row_hi - row_lo) * d0;
  if (nh == 0) return TC_OK;
  std::vector<const void*> hp(nh);
  std::vector<uint32_t> boff(nh);
  for (uint32_t cp = row_lo; cp < row_hi; cp++)
    for (uint32_t c = 0; c < d0; c++) {
      hp[(cp - row_lo) * d0 + c] = (const uint8_t*)d_in + esz * R * cp;
      boff[(cp - row_lo) * d0 + c] = (uint32_t)(R * c);
    }
  return tcrt::msm_batch_device(ctx, dtype, scale_bits, hp.data(), (int)nh, ed_lag, R, out, boff.data(), 0,
                                const_cast<tc_srs*>(srs));
}

static int open_batch_impl(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                           int scale_bits, const uint8_t* omegas_le21, int route, uint8_t* out_y21,
                           uint8_t* out_pi43, const uint8_t* d_h43);

int tc_open_batch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype, int scale_bits,
                  const uint8_t* omegas_le21, int route, uint8_t* out_y21, uint8_t* out_pi43) {
  return open_batch_impl(ctx, srs, d_ins, count, dtype, scale_bits, omegas_le21, route, out_y21, out_pi43, nullptr);
}

int tc_open_slices(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits, uint32_t row_lo,
                   uint32_t row_hi, uint8_t* d_out43) {
  if (!ctx || !srs || !d_in || row_lo > row_hi || (row_hi > row_lo && !d_out43)) return TC_ERR_ARGUMENT;
  if (srs->m < 2 || !srs->lagrange) return fail(ctx, TC_ERR_VALUE, "slice commitments need m >= 2 and a Lagrange SRS");
  if (row_hi > srs->shape[0]) return fail(ctx, TC_ERR_INDEX, "slice rows beyond the first axis");
  const uint32_t nh = (row_hi - row_lo) * srs->shape[0];
  if (nh == 0) return TC_OK;
  Aff* pts;
  TC_TRY(tcrt::scratch_t(ctx, "opens.pts", (uint64_t)nh, &pts));
  TC_TRY(slice_commitments(ctx, srs, d_in, dtype, scale_bits, row_lo, row_hi, pts));
  k_encode43<<<tcrt::blocks_for(nh, 64), 64, 0, ctx->stream>>>(pts, nh, d_out43);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

int tc_open_batch_sliced(tc_ctx* ctx, const tc_srs* srs, const void* d_in, const uint8_t* d_h43, int count,
                         int dtype, int scale_bits, const uint8_t* omegas_le21, uint8_t* out_y21, uint8_t* out_pi43) {
  if (!ctx || !srs || !d_in || !d_h43 || count < 0) return TC_ERR_ARGUMENT;
  if (srs->m < 2 || !srs->lagrange || !srs->sublag)
    return fail(ctx, TC_ERR_VALUE, "sliced openings need m >= 2 and the Lagrange / sub-grid sets");
  std::vector<const void*> ins((size_t)count, d_in);
  return open_batch_impl(ctx, srs, ins.data(), count, dtype, scale_bits, omegas_le21, TC_ROUTE_LAGRANGE, out_y21,
                         out_pi43, d_h43);
}

static int open_batch_impl(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                           int scale_bits, const uint8_t* omegas_le21, int route, uint8_t* out_y21,
                           uint8_t* out_pi43, const uint8_t* d_h43) {
  if (!ctx || !srs || (count && (!d_ins || !omegas_le21 || !out_y21 || !out_pi43)) || count < 0)
    return TC_ERR_ARGUMENT;
  const uint64_t n = srs->n;
  const int m = srs->m;
  std::vector<int> lag, tiny_ops;
  for (int i = 0; i < count; i++) {
    if (!d_ins[i]) return TC_ERR_ARGUMENT;
    std::vector<Fe> om(m);
    for (int j = 0; j < m; j++)
      if (!le21_to_fe(omegas_le21 + 21 * ((size_t)i * m + j), om[j]))
        return fail(ctx, TC_ERR_VALUE, "opening %d: point coordinate %d out of range", i, j);
    const bool lag_ok = srs->lagrange && (m == 1 || srs->sublag);
    // tiny SRSs (Terkle nodes) open fastest one by one on tc_open's table-kernel route
    // (measured: 0.17 ms per node opening vs ~4 ms through batched pipelines)
    const bool tiny = n <= SMALL_MSM_MAX && srs->monomial && route == TC_ROUTE_AUTO;
    if (lag_ok && route != TC_ROUTE_MONOMIAL && !tiny)
      lag.push_back(i);
    else if (tiny)
      tiny_ops.push_back(i);
    else
      TC_TRY(tc_open(ctx, srs, d_ins[i], dtype, scale_bits, omegas_le21 + 21 * (size_t)i * m, route,
                     out_y21 + 21 * (size_t)i, out_pi43 + 43 * (size_t)i * m));
  }
  if (!tiny_ops.empty()) {
    // tiny SRSs (Terkle node openings): tc_open's monomial route for all of them with no
    // host round trip per opening — interpolation and synthetic division per tensor, every
    // quotient MSM in ONE table-kernel launch, one readback of the points and the values
    const uint64_t K = tiny_ops.size();
    Fe *tv, *tq, *ty;
    Aff* tout;
    TC_TRY(tcrt::scratch_t(ctx, "opent.vals", K * n, &tv));
    TC_TRY(tcrt::scratch_t(ctx, "opent.q", K * m * n, &tq));
    TC_TRY(tcrt::scratch_t(ctx, "opent.y", K, &ty));
    TC_TRY(tcrt::scratch_t(ctx, "opent.out", K * m, &tout));
    std::vector<const void*> ptrs(K * m);
    std::vector<Fe> om(m);
    for (uint64_t k = 0; k < K; k++) {
      const int i = tiny_ops[k];
      Fe* v = tv + k * n;
      if (dtype == TC_DTYPE_FP_LIMBS)
        TC_CUDA(ctx, cudaMemcpyAsync(v, d_ins[i], n * sizeof(Fe), cudaMemcpyDeviceToDevice, ctx->stream));
      else
        TC_TRY(tcrt::quantize_device(ctx, d_ins[i], dtype, n, scale_bits, v));
      TC_TRY(tcrt::interpolate_device(ctx, v, srs->shape, m));
      for (int j = 0; j < m; j++) le21_to_fe(omegas_le21 + 21 * ((size_t)i * m + j), om[j]);
      TC_TRY(tcrt::open_quotients_device(ctx, v, srs->shape, m, om.data(), tq + k * m * n, nullptr, ty + k));
      for (int a = 0; a < m; a++) ptrs[k * m + a] = tq + (k * m + a) * n;
    }
    TC_TRY(msm_srs(ctx, srs, TC_SRS_MONOMIAL, TC_DTYPE_FP_LIMBS, 0, ptrs.data(), (int)(K * m), tout));
    std::vector<uint8_t> enc(K * m * 43);
    TC_TRY(fetch_encode_many(ctx, tout, (int)(K * m), enc.data()));
    std::vector<Fe> ys(K);
    TC_CUDA(ctx, cudaMemcpy(ys.data(), ty, K * sizeof(Fe), cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < K; k++) {
      const int i = tiny_ops[k];
      fe_to_le21(Fp::canon(ys[k]), out_y21 + 21 * (size_t)i);
      memcpy(out_pi43 + 43 * (size_t)i * m, enc.data() + 43 * k * m, 43 * (size_t)m);
    }
  }
  if (lag.empty()) return TC_OK;
  const EdPk *ed_lag, *ed_sub = nullptr;
  TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), TC_SRS_LAGRANGE, &ed_lag));
  if (m > 1) TC_TRY(tcrt::srs_edwards(ctx, const_cast<tc_srs*>(srs), 0, &ed_sub));
  size_t esz = 0;
  if (dtype_size(dtype, &esz)) return fail(ctx, TC_ERR_ARGUMENT, "open: unsupported dtype %d", dtype);

  // split: tensors opened often enough take the slice-commitment route
  static const int PMIN = getenv("TC_OPEN_PRECOMP_MIN") ? atoi(getenv("TC_OPEN_PRECOMP_MIN")) : 6;
  const uint32_t d0 = srs->shape[0];
  std::map<const void*, std::vector<int>> by_tensor;
  for (int i : lag) by_tensor[d_ins[i]].push_back(i);
  std::vector<std::vector<int>> jobs;   // each job: openings sharing one strategy (+ tensor)
  std::vector<const void*> job_h;       // tensor whose slice commitments the job uses, or null
  std::vector<int> rest;
  for (int i : lag) {
    auto& v = by_tensor[d_ins[i]];
    if (m >= 2 && ((PMIN > 0 && (int)v.size() >= PMIN) || d_h43) && d0 * d0 <= 4096) {
      if (v.front() == i) jobs.push_back(v), job_h.push_back(d_ins[i]);
    } else {
      rest.push_back(i);
    }
  }
  static const uint64_t G_ENV = getenv("TC_OPEN_GROUP") ? (uint64_t)atoi(getenv("TC_OPEN_GROUP")) : 0;
  const int G = (int)std::max<uint64_t>(1, G_ENV ? G_ENV : (1ull << 24) / n);
  for (size_t g0 = 0; g0 < rest.size(); g0 += G) {
    jobs.push_back(std::vector<int>(rest.begin() + g0, rest.begin() + std::min(rest.size(), g0 + G)));
    job_h.push_back(nullptr);
  }

  constexpr uint64_t GS_MAX = 256;   // openings per sliced group
  Fe *qall, *sc = nullptr;
  Aff *d_out, *hpts = nullptr;
  EdPk* hed = nullptr;
  uint64_t compact = 0;   // per-opening quotient values of axes >= 1 (sliced layout)
  {
    uint64_t sp = n;
    for (int a = 1; a < m; a++) sp /= srs->shape[a - 1], compact += sp;
  }
  const uint64_t GO = std::max<uint64_t>(G, GS_MAX);   // openings per group, either layout
  TC_TRY(tcrt::scratch_t(ctx, "openb.q", std::max<uint64_t>((uint64_t)G * m * n, GS_MAX * compact), &qall));
  TC_TRY(tcrt::scratch_t(ctx, "openb.out", GO * m, &d_out));
  std::vector<uint8_t> enc((size_t)GO * m * 43);
  std::vector<Fe> om(m), stabs;
  std::vector<int> ssj;
  for (size_t jb = 0; jb < jobs.size(); jb++) {
    const std::vector<int>& ops = jobs[jb];
    const bool sliced = job_h[jb] != nullptr;
    if (sliced) {
      // H[c', c]: d0^2 MSMs of R points, MSM (c', c) = tensor slice c' over SRS slice c
      const uint32_t nh = d0 * d0;
      TC_TRY(tcrt::scratch_t(ctx, "openh.pts", (uint64_t)nh, &hpts));
      TC_TRY(tcrt::scratch_t(ctx, "openh.ed", (uint64_t)nh, &hed));
      TC_TRY(tcrt::scratch_t(ctx, "openh.s", GO * nh, &sc));
      if (d_h43) {
        // slice commitments computed elsewhere (each rank a share of the rows, all-gathered:
        // dist.open_many_dist) — only decode them
        TC_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream));
        k_decode43<<<tcrt::blocks_for(nh, 64), 64, 0, ctx->stream>>>(d_h43, nh, hpts, ctx->d_flags);
        TC_LAUNCHED(ctx);
      } else {
        TC_TRY(slice_commitments(ctx, srs, job_h[jb], dtype, scale_bits, 0, d0, hpts));
      }
      TC_TRY(tcrt::to_edwards_device(ctx, hpts, nh, hed));
    }
    // sliced jobs keep only the quotients of axes >= 1 (n / d0 + ... per opening), packed
    // per axis, so a whole tensor's openings form ONE group: one quotient launch per axis
    // and one MSM pipeline per axis instead of one per 8 openings
    const int GJ = sliced ? (int)std::min<uint64_t>(GS_MAX, ops.size()) : G;
    std::vector<uint64_t> qoff(m, 0), qstr(m, 0);
    for (size_t g0 = 0; g0 < ops.size(); g0 += GJ) {
      const int gc = (int)std::min<size_t>(GJ, ops.size() - g0);
      if (sliced) {
        uint64_t acc = 0, sp = n;
        for (int a = 0; a < m; a++) {
          sp /= srs->shape[a];   // axis a's quotient lives on axes >= a: n / (d0 .. d_(a-1)) values
          const uint64_t span_a = sp * srs->shape[a];
          qoff[a] = a == 0 ? 0 : acc;
          qstr[a] = a == 0 ? 0 : span_a;
          if (a) acc += span_a * gc;
        }
      }
      stabs.clear();
      ssj.clear();
      // field values of the group's tensors (one copy per distinct tensor), then the
      // quotients of all gc openings with one launch per axis
      std::vector<tcrt::LagW> Ws(gc);
      std::vector<const Fe*> vptr(gc);
      std::map<const void*, const Fe*> loaded;
      Fe* vbuf;
      TC_TRY(tcrt::scratch_t(ctx, "openb.vals", (uint64_t)(sliced ? 1 : gc) * n, &vbuf));
      for (int k = 0; k < gc; k++) {
        const int i = ops[g0 + k];
        for (int j = 0; j < m; j++) le21_to_fe(omegas_le21 + 21 * ((size_t)i * m + j), om[j]);
        lag_weights(srs, om, Ws[k]);
        if (sliced) {
          stabs.insert(stabs.end(), Ws[k].lam.begin(), Ws[k].lam.begin() + d0);
          stabs.insert(stabs.end(), Ws[k].inv.begin(), Ws[k].inv.begin() + d0);
          stabs.insert(stabs.end(), Ws[k].der.begin(), Ws[k].der.begin() + d0);
          ssj.push_back(Ws[k].sj[0]);
        }
        auto it = loaded.find(d_ins[i]);
        if (it == loaded.end()) {
          Fe* dst = vbuf + (uint64_t)loaded.size() * n;
          if (dtype == TC_DTYPE_FP_LIMBS)
            TC_CUDA(ctx, cudaMemcpyAsync(dst, d_ins[i], n * sizeof(Fe), cudaMemcpyDeviceToDevice, ctx->stream));
          else
            TC_TRY(tcrt::quantize_device(ctx, d_ins[i], dtype, n, scale_bits, dst));
          it = loaded.emplace(d_ins[i], dst).first;
        }
        vptr[k] = it->second;
      }
      std::vector<Fe> ys(gc);
      TC_TRY(tcrt::open_quotients_lagrange_batch(ctx, vptr.data(), gc, srs->shape, m, Ws, qall, ys.data(), sliced,
                                                 sliced ? qoff.data() : nullptr, sliced ? qstr.data() : nullptr));
      for (int k = 0; k < gc; k++) fe_to_le21(Fp::canon(ys[k]), out_y21 + 21 * (size_t)ops[g0 + k]);
      uint64_t span = n;
      std::vector<const void*> ptrs(gc);
      for (int a = 0; a < m; a++) {
        if (a == 0 && sliced) {
          const uint32_t nh = d0 * d0;
          TC_TRY(tcrt::slice_scalars_device(ctx, stabs, ssj, d0, (uint32_t)gc, sc));
          for (int k = 0; k < gc; k++) ptrs[k] = sc + (uint64_t)k * nh;
          TC_TRY(tcrt::msm_batch_device(ctx, TC_DTYPE_FP_LIMBS, 0, ptrs.data(), gc, hed, nh, d_out));
        } else {
          const EdPk* bases = a == 0 ? ed_lag : ed_sub + srs->sublag_off[a];
          for (int k = 0; k < gc; k++)
            ptrs[k] = sliced ? qall + qoff[a] + (uint64_t)k * qstr[a] : qall + ((uint64_t)k * m + a) * n;
          TC_TRY(msm_quotients(ctx, srs, ptrs.data(), gc, bases, span,
                                        d_out + (uint64_t)a * gc));
        }
        span /= srs->shape[a];
      }
      TC_TRY(fetch_encode_many(ctx, d_out, m * gc, enc.data()));
      for (int a = 0; a < m; a++)
        for (int k = 0; k < gc; k++)
          memcpy(out_pi43 + 43 * ((size_t)ops[g0 + k] * m + a), enc.data() + 43 * ((size_t)a * gc + k), 43);
    }
  }
  return TC_OK;
}

// ---- Terkle ----
int tc_terkle_build(tc_ctx* ctx, const tc_srs* node_srs, const uint8_t* leaves_le21, uint64_t n, uint8_t* out_nodes43,
                    uint64_t* inout_count) {
  if (!ctx || !node_srs || !leaves_le21 || !out_nodes43 || !inout_count) return TC_ERR_ARGUMENT;
  if (n == 0) return fail(ctx, TC_ERR_VALUE, "empty leaf list");
  const uint64_t B = node_srs->n;
  if (B < 2) return fail(ctx, TC_ERR_VALUE, "tree arity must be >= 2");
  uint64_t L = 1, cap = B;
  while (cap < n) cap *= B, L++;
  uint64_t total_nodes = 0, w = cap;
  for (uint64_t l = 0; l < L; l++) w /= B, total_nodes += w;
  if (*inout_count < total_nodes) return fail(ctx, TC_ERR_VALUE, "need room for %llu nodes", (unsigned long long)total_nodes);
  std::vector<Fe> vals(cap);
  for (uint64_t i = 0; i < cap; i++) {
    if (i < n) {
      if (!le21_to_fe(leaves_le21 + 21 * i, vals[i])) return fail(ctx, TC_ERR_VALUE, "leaf %llu out of range", (unsigned long long)i);
    } else {
      vals[i] = Fe{{0, 0, 0, 0, 0, 0}};
    }
  }
  Fe* d_vals;
  Aff* d_out;
  TC_TRY(tcrt::scratch_t(ctx, "terkle.vals", cap, &d_vals));
  TC_TRY(tcrt::scratch_t(ctx, "terkle.out", cap / B, &d_out));
  bool lag = node_srs->lagrange != nullptr;
  if (lag && B <= SMALL_MSM_MAX) {
    // device-resident tree: one upload, L launches (hashing on the device), one readback
    Aff* d_pts;
    TC_TRY(tcrt::scratch_t(ctx, "terkle.pts", total_nodes, &d_pts));
    // pageable source: the synchronous copy completes before `vals` goes away
    TC_CUDA(ctx, cudaMemcpy(d_vals, vals.data(), cap * sizeof(Fe), cudaMemcpyHostToDevice));
    TC_TRY(tcrt::terkle_device(ctx, const_cast<tc_srs*>(node_srs), d_vals, cap, (int)L, d_pts));
    TC_TRY(fetch_encode_many(ctx, d_pts, (int)total_nodes, out_nodes43));
    *inout_count = total_nodes;
    return TC_OK;
  }
  uint64_t written = 0;
  const uint8_t tag[] = {'t', 'e', 'r', 'k', 'l', 'e', '/', 'n', 'o', 'd', 'e'};
  for (uint64_t l = 0; l < L; l++) {
    const uint64_t nodes = vals.size() / B;
    // pageable source: the synchronous copy completes before `vals` is reused
    TC_CUDA(ctx, cudaMemcpy(d_vals, vals.data(), vals.size() * sizeof(Fe), cudaMemcpyHostToDevice));
    std::vector<const void*> ptrs(nodes);
    for (uint64_t u = 0; u < nodes; u++) {
      Fe* z = d_vals + u * B;
      if (!lag) TC_TRY(tcrt::interpolate_device(ctx, z, node_srs->shape, node_srs->m));
      ptrs[u] = z;
    }
    // every node of the level in one batched MSM
    TC_TRY(msm_srs(ctx, node_srs, lag ? TC_SRS_LAGRANGE : TC_SRS_MONOMIAL, TC_DTYPE_FP_LIMBS, 0, ptrs.data(),
                   (int)nodes, d_out));
    uint8_t* enc = out_nodes43 + 43 * written;
    TC_TRY(fetch_encode_many(ctx, d_out, (int)nodes, enc));
    std::vector<Fe> next(nodes);
    for (uint64_t u = 0; u < nodes; u++) next[u] = hash_to_scalar(enc + 43 * u, 43, tag, sizeof tag);
    written += nodes;
    vals.swap(next);
  }
  *inout_count = written;
  return TC_OK;
}

// ---- host verifier primitive ----
int tc_pairing(const uint8_t* a43, const uint8_t* b43, uint8_t* out42) {
  if (!a43 || !b43 || !out42) return TC_ERR_ARGUMENT;
  Aff a, b;
  if (!decode43(a43, a) || !decode43(b43, b)) return TC_ERR_VALUE;
  F2 r;
  if (!host_pairing(a, b, r)) return TC_ERR_BACKEND;
  Fe ra = Fq::from_mont(r.a), rb = Fq::from_mont(r.b);
  fe_to_le21(ra, out42);
  fe_to_le21(rb, out42 + 21);
  return TC_OK;
}

// tc_verify (product-of-pairings form SPEC.md:313), CPU only
int tc_verify_host(int m, const uint8_t* axis43, const uint8_t* c43, const uint8_t* omega_le21, const uint8_t* y21,
                   const uint8_t* proofs43, int* ok) {
  if (!axis43 || !c43 || !omega_le21 || !y21 || !proofs43 || !ok || m < 1) return TC_ERR_ARGUMENT;
  Aff C, g = g_host();
  if (!decode43(c43, C)) return TC_ERR_VALUE;
  Fe y;
  if (!le21_to_fe(y21, y)) return TC_ERR_VALUE;
  Xyzz lhs_pt = host_mul(g, fp_neg_canon(y));
  if (!aff_is_inf(C)) xyzz_add_aff(lhs_pt, C);
  F2 lhs, rhs{Fq::one(), Fq::zero()};
  if (!host_pairing(host_aff(lhs_pt), g, lhs)) return TC_ERR_BACKEND;
  for (int i = 0; i < m; i++) {
    Aff pi, ax;
    Fe w;
    if (!decode43(proofs43 + 43 * i, pi) || !decode43(axis43 + 43 * i, ax) || !le21_to_fe(omega_le21 + 21 * i, w))
      return TC_ERR_VALUE;
    Xyzz t = host_mul(g, fp_neg_canon(w));
    if (!aff_is_inf(ax)) xyzz_add_aff(t, ax);
    F2 e;
    if (!host_pairing(pi, host_aff(t), e)) return TC_ERR_BACKEND;
    rhs = f2mul(rhs, e);
  }
  *ok = f2_eq(lhs, rhs) ? 1 : 0;
  return TC_OK;
}

// ---- self-test hooks ----
int tc_host_fq_mul(const uint32_t* a, const uint32_t* b, uint32_t* out) {
  Fe x, y;
  memcpy(x.v, a, 24);
  memcpy(y.v, b, 24);
  Fe r = Fq::from_mont(Fq::mul(Fq::to_mont(x), Fq::to_mont(y)));
  memcpy(out, r.v, 24);
  return TC_OK;
}
int tc_host_fp_mul(const uint32_t* a, const uint32_t* b, uint32_t* out) {
  Fe x, y;
  memcpy(x.v, a, 24);
  memcpy(y.v, b, 24);
  Fe r = Fp::from_mont(Fp::mul(Fp::to_mont(x), Fp::to_mont(y)));
  memcpy(out, r.v, 24);
  return TC_OK;
}
int tc_host_g_mul(const uint8_t* k_le21, uint8_t* out43) {
  Fe k;
  for (int i = 0; i < 6; i++) k.v[i] = 0;
  for (int i = 0; i < 21; i++) k.v[i / 4] |= (uint32_t)k_le21[i] << (8 * (i % 4));
  aff_encode43(host_aff(host_mul(g_host(), k)), out43);
  return TC_OK;
}
int tc_host_field_inv(int field, int method, const uint32_t* a, uint32_t* out) {
  if (!a || !out || field < 0 || field > 1 || method < 0 || method > 2) return TC_ERR_ARGUMENT;
  Fe x, r;
  for (int i = 0; i < 6; i++) x.v[i] = a[i];
  if (field == 0) {
    const Fe m = Fq::to_mont(x);
    r = Fq::from_mont(method == 0 ? Fq::inv_bygcd(m) : method == 1 ? Fq::inv(m) : Fq::inv_fast(m));
  } else {
    const Fe m = Fp::to_mont(x);
    r = Fp::from_mont(method == 0 ? Fp::inv_bygcd(m) : method == 1 ? Fp::inv(m) : Fp::inv_fast(m));
  }
  for (int i = 0; i < 6; i++) out[i] = r.v[i];
  return TC_OK;
}

int tc_host_hash_point(const uint8_t* p43, int node, uint8_t* out21) {
  if (!p43 || !out21) return TC_ERR_ARGUMENT;
  Aff a;
  if (!decode43(p43, a)) return TC_ERR_VALUE;
  fe_to_le21(hash_point_to_scalar(a, node != 0), out21);
  return TC_OK;
}

int tc_host_hash_to_scalar(const uint8_t* data, uint32_t n, const uint8_t* tag, uint32_t tn, uint8_t* out21) {
  fe_to_le21(hash_to_scalar(data, n, tag, tn), out21);
  return TC_OK;
}

// integer-multiply pipe peak (IMAD, mad.lo.u32) at the current clocks: the roofline
// denominator for the integer-bound kernels (MEASURED_PEAKS.json carries none)
int tc_measure_imad_peak(tc_ctx* ctx, double* tops) {
  if (!ctx || !tops) return TC_ERR_ARGUMENT;
  uint32_t* d_sink;
  TC_TRY(tcrt::scratch_t(ctx, "imad.sink", 4, &d_sink));
  cudaEvent_t e0, e1;
  TC_CUDA(ctx, cudaEventCreate(&e0));
  TC_CUDA(ctx, cudaEventCreate(&e1));
  const int iters = 8192, threads = 512, blocks = ctx->num_sms * 4;
  double best = 0;
  for (int rep = 0; rep < 4; rep++) {
    TC_CUDA(ctx, cudaEventRecord(e0, ctx->stream));
    k_imad_peak<<<blocks, threads, 0, ctx->stream>>>(d_sink, 0x9e3779b9u + rep, iters);
    TC_CUDA(ctx, cudaEventRecord(e1, ctx->stream));
    TC_CUDA(ctx, cudaEventSynchronize(e1));
    float ms = 0;
    TC_CUDA(ctx, cudaEventElapsedTime(&ms, e0, e1));
    double ops = (double)blocks * threads * iters * 16;
    best = std::max(best, ops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *tops = best;
  return TC_OK;
}

int tc_debug_field(tc_ctx* ctx, int op, const uint32_t* d_a, const uint32_t* d_b, uint32_t* d_out, uint64_t n) {
  if (!ctx) return TC_ERR_ARGUMENT;
  k_field_op<<<tcrt::blocks_for(n, 128), 128, 0, ctx->stream>>>(op, (const Fe*)d_a, (const Fe*)d_b, (Fe*)d_out, n);
  TC_LAUNCHED(ctx);
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return TC_OK;
}

}  // extern "C"
