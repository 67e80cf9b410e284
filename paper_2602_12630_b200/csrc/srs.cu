// K5: structured reference string generation (setup_srs; Srs SPEC.md:44-50).
//
// Every SRS element is g^{e_i} for a known exponent e_i (monomial: prod_j tau_j^{i_j};
// Lagrange: prod_j L_{j,i_j}(tau_j)).  The reference would run `exp` (double-and-add,
// backend.py:202-217, ~1.9 ms each) per element.  Here the base g is fixed, so:
//   k_gtable   — table G[w][j] = (j+1) * 2^{8w} * g, 21 windows x 255 entries (affine)
//   k_exps     — e_i from per-axis tables (lex index decomposition, m-1 F_p products)
//   k_fixed    — e_i * g = sum over the 21 bytes of e_i of one table entry (21 mixed adds),
//                K points per thread converted to affine with ONE shared inversion
//                (Montgomery batch trick)
#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr int GT_WIN = 21;     // 21 x 8 bits = 168 >= 162
constexpr int GT_ENT = 255;
constexpr int FB_K = 8;        // points per thread sharing one inversion

__device__ __forceinline__ Aff g_aff() {
  // generator (backend.py:106-107), canonical -> Montgomery
  Fe x{{0xbe9bb8c2u, 0x9f4698deu, 0x2e04a40bu, 0x96df9421u, 0xd6e0e406u, 0x000000abu}};
  Fe y{{0xca83210eu, 0x0d3911f8u, 0x28e6ecd6u, 0xfcd508bdu, 0xc7320595u, 0x00000018u}};
  return Aff{Fq::to_mont(x), Fq::to_mont(y)};
}

__global__ void k_gtable(Aff* table) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= GT_WIN * GT_ENT) return;
  uint32_t w = t / GT_ENT, j = t % GT_ENT + 1;
  // k = j << 8w, double-and-add from the MSB
  Aff g = g_aff();
  Xyzz acc = xyzz_inf();
  int top = 8 * w + 7;
  bool started = false;
  for (int b = top; b >= 0; b--) {
    if (started) acc = xyzz_dbl(acc);
    int bit = (b >= (int)(8 * w)) ? (int)((j >> (b - 8 * w)) & 1u) : 0;
    if (bit) {
      xyzz_add_aff(acc, g);
      started = true;
    }
  }
  Aff r = xyzz_to_aff(acc);
  r.x = Fq::canon(r.x);
  r.y = Fq::canon(r.y);
  table[t] = r;
}

// e_i = prod_j tab_j[i_j] (canonical F_p); tabs are concatenated per-axis tables
__global__ void k_exps(const Fe* tabs, const uint32_t* tab_off, const uint32_t* shape, int m,
                       uint64_t n, Fe* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t rem = i;
  Fe acc = Fp::one();   // Montgomery 1
  for (int j = m - 1; j >= 0; j--) {
    uint32_t d = shape[j];
    uint32_t ij = (uint32_t)(rem % d);
    rem /= d;
    // mul by canonical value: mont(acc) * canon(x) -> mont(acc * x / R) ... keep acc in
    // Montgomery form by multiplying with Montgomery(x) = x*R.
    acc = Fp::mul(acc, Fp::to_mont(tabs[tab_off[j] + ij]));
  }
  out[i] = Fp::from_mont(acc);
}

__global__ void __launch_bounds__(128) k_fixed(const Aff* table, const Fe* exps, uint64_t n, Aff* out) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t i0 = t * FB_K;
  if (i0 >= n) return;
  Xyzz pts[FB_K];
  Fe pref[FB_K];
  Fe run = Fq::one();
  int cnt = (n - i0 < (uint64_t)FB_K) ? (int)(n - i0) : FB_K;
  for (int k = 0; k < cnt; k++) {
    Fe e = exps[i0 + k];
    Xyzz acc = xyzz_inf();
#pragma unroll 1
    for (int w = 0; w < GT_WIN; w++) {
      uint32_t byte = (e.v[w >> 2] >> (8 * (w & 3))) & 0xffu;
      if (byte) xyzz_add_aff(acc, table[w * GT_ENT + byte - 1]);
    }
    pts[k] = acc;
    // Montgomery batch inversion: pref[k] = product of ZZ*ZZZ of finite points before k
    pref[k] = run;
    if (!xyzz_is_inf(acc)) run = Fq::mul(run, Fq::mul(acc.ZZ, acc.ZZZ));
  }
  Fe inv = Fq::inv(run);
  for (int k = cnt - 1; k >= 0; k--) {
    Aff r;
    if (xyzz_is_inf(pts[k])) {
      r = aff_inf();
    } else {
      Fe iz = Fq::mul(inv, pref[k]);                    // 1 / (ZZ*ZZZ)_k
      inv = Fq::mul(inv, Fq::mul(pts[k].ZZ, pts[k].ZZZ));
      r = xyzz_to_aff_with_inv(pts[k], iz);
      r.x = Fq::canon(r.x);
      r.y = Fq::canon(r.y);
    }
    out[i0 + k] = r;
  }
}

// E affine points -> the MSM's Edwards model phi([h] P) (ec.cuh): [h] P in XYZZ, then two
// Montgomery batch inversions over K points per thread (XYZZ -> affine, affine -> Edwards).
// K = FB_K for SRS-sized inputs; K = 1 for small ones (an opening's d0^2 slice commitments),
// whose conversion is latency-bound: 1024 points at 8 per thread ran on 128 threads of one SM
// (3.2 ms of serial doublings), one per thread spreads them over the GPU
template <int K>
__global__ void __launch_bounds__(128) k_to_edwards(const Aff* in, uint64_t n, EdPk* out) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t i0 = t * K;
  if (i0 >= n) return;
  const int cnt = (n - i0 < (uint64_t)K) ? (int)(n - i0) : K;
  Xyzz h[K];
  Fe pref[K];
  Fe run = Fq::one();
  for (int k = 0; k < cnt; k++) {
    h[k] = xyzz_mul_half(in[i0 + k]);
    pref[k] = run;
    if (!xyzz_is_inf(h[k])) run = Fq::mul(run, Fq::mul(h[k].ZZ, h[k].ZZZ));
  }
  Fe inv = Fq::inv_pref(run);
  Aff q[K];
  for (int k = cnt - 1; k >= 0; k--) {
    if (xyzz_is_inf(h[k])) {
      q[k] = aff_inf();
    } else {
      const Fe iz = Fq::mul(inv, pref[k]);
      inv = Fq::mul(inv, Fq::mul(h[k].ZZ, h[k].ZZZ));
      q[k] = xyzz_to_aff_with_inv(h[k], iz);
    }
  }
  run = Fq::one();
  for (int k = 0; k < cnt; k++) {
    pref[k] = run;
    run = Fq::mul(run, aff_ed_den(q[k]));
  }
  inv = Fq::inv_pref(run);
  for (int k = cnt - 1; k >= 0; k--) {
    const Fe den = aff_ed_den(q[k]);
    const Fe ik = Fq::mul(inv, pref[k]);
    inv = Fq::mul(inv, den);
    out[i0 + k] = pack_ed(aff_to_ed_with_inv(q[k], ik));
  }
}

// out[i] = 2^c in[i] (Edwards affine with t = 2 d' x y): c doublings in extended coordinates, the
// Z of FB_K points per thread inverted with one shared inversion
__global__ void __launch_bounds__(128) k_win_step(const EdPk* in, uint64_t n, int c, EdPk* out) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t i0 = t * FB_K;
  if (i0 >= n) return;
  const int cnt = (n - i0 < (uint64_t)FB_K) ? (int)(n - i0) : FB_K;
  Ext pts[FB_K];
  Fe pref[FB_K];
  Fe run = Fq::one();
  for (int k = 0; k < cnt; k++) {
    Ext e = ext_from_aff(ld_edpk(in + i0 + k));
    for (int j = 0; j < c; j++) e = ext_dbl(e);
    pts[k] = e;
    pref[k] = run;
    run = Fq::mul(run, e.Z);   // Z != 0 on the (complete) Edwards curve
  }
  Fe inv = Fq::inv(run);
  for (int k = cnt - 1; k >= 0; k--) {
    const Fe iz = Fq::mul(inv, pref[k]);
    inv = Fq::mul(inv, pts[k].Z);
    const Fe x = Fq::mul(pts[k].X, iz), y = Fq::mul(pts[k].Y, iz);
    out[i0 + k] = pack_ed(edaff_from_xy(x, y));
  }
}

}  // namespace

namespace tcrt {

int srs_window_table(tc_ctx* ctx, tc_srs* srs, const EdPk* bases, uint64_t n, const EdPk** out) {
  std::lock_guard<std::mutex> guard(srs->mu);
  auto it = srs->wintab.find(bases);
  if (it != srs->wintab.end()) {
    *out = it->second;
    return TC_OK;
  }
  const int c = fb_width(n), nd = fb_ndig(c);
  EdPk* tab = nullptr;
  if (cudaMalloc(&tab, std::max<uint64_t>(n, 1) * nd * sizeof(EdPk)) != cudaSuccess)
    return fail(ctx, TC_ERR_MEMORY, "window table alloc (%llu points)", (unsigned long long)(n * nd));
  TC_CUDA(ctx, cudaMemcpyAsync(tab, bases, n * sizeof(EdPk), cudaMemcpyDeviceToDevice, ctx->stream));
  for (int w = 1; w < nd; w++) {
    k_win_step<<<blocks_for((n + FB_K - 1) / FB_K, 128), 128, 0, ctx->stream>>>(tab + (w - 1) * n, n, c,
                                                                                tab + w * n);
    TC_LAUNCHED(ctx);
  }
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));   // shared with other contexts' streams
  srs->wintab[bases] = tab;
  srs->wintab_bytes += std::max<uint64_t>(n, 1) * nd * sizeof(EdPk);
  *out = tab;
  return TC_OK;
}

int srs_exp_table(tc_ctx* ctx, tc_srs* srs, const EdPk* bases, uint64_t n, int depth, const EdPk** out) {
  std::lock_guard<std::mutex> guard(srs->mu);
  if (srs->exptab && srs->exptab_depth >= depth) {
    *out = srs->exptab;
    return TC_OK;
  }
  // budget: TC_EXPTAB_GB (default 96) and 8 GB of device memory left free
  static const uint64_t cap = (getenv("TC_EXPTAB_GB") ? strtoull(getenv("TC_EXPTAB_GB"), nullptr, 10) : 96ull) << 30;
  const uint64_t bytes = (uint64_t)depth * n * sizeof(EdPk);
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  if (bytes > cap || bytes > fr || fr - bytes < (8ull << 30)) return TC_ERR_MEMORY;
  EdPk* tab = nullptr;
  if (cudaMalloc(&tab, bytes) != cudaSuccess) {
    cudaGetLastError();
    return TC_ERR_MEMORY;
  }
  // a shallower table may still be read by kernels other contexts (threads) launched with
  // the pointer they got earlier: retire it, freed with the SRS (tc_srs_destroy)
  if (srs->exptab) srs->retired.push_back(srs->exptab);
  TC_CUDA(ctx, cudaMemcpyAsync(tab, bases, n * sizeof(EdPk), cudaMemcpyDeviceToDevice, ctx->stream));
  for (int k = 1; k < depth; k++) {
    k_win_step<<<blocks_for((n + FB_K - 1) / FB_K, 128), 128, 0, ctx->stream>>>(tab + (uint64_t)(k - 1) * n, n, 1,
                                                                                tab + (uint64_t)k * n);
    TC_LAUNCHED(ctx);
  }
  // other contexts (other streams) read the table from now on: finish building it first
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  srs->exptab = tab;
  srs->exptab_depth = depth;
  *out = tab;
  return TC_OK;
}

int to_edwards_device(tc_ctx* ctx, const Aff* d_in, uint64_t n, EdPk* d_out) {
  if (n == 0) return TC_OK;
  if (n <= (uint64_t)ctx->num_sms * 128 * 4)
    k_to_edwards<1><<<blocks_for(n, 64), 64, 0, ctx->stream>>>(d_in, n, d_out);
  else
    k_to_edwards<FB_K><<<blocks_for((n + FB_K - 1) / FB_K, 128), 128, 0, ctx->stream>>>(d_in, n, d_out);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

int srs_edwards(tc_ctx* ctx, tc_srs* srs, int which, const EdPk** out) {
  const Aff* src;
  EdPk** dst;
  uint64_t n = srs->n;
  if (which == TC_SRS_LAGRANGE) {
    src = srs->lagrange, dst = &srs->ed_lagrange;
  } else if (which == TC_SRS_MONOMIAL) {
    src = srs->monomial, dst = &srs->ed_monomial;
  } else {
    src = srs->sublag, dst = &srs->ed_sublag;
    n = srs->m > 1 ? srs->sublag_off[srs->m - 1] + srs->shape[srs->m - 1] : 0;
  }
  if (!src) return fail(ctx, TC_ERR_VALUE, "srs has no elements of kind %d", which);
  std::lock_guard<std::mutex> guard(srs->mu);
  if (!*dst) {
    EdPk* p = nullptr;
    if (cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(EdPk)) != cudaSuccess)
      return fail(ctx, TC_ERR_MEMORY, "srs edwards alloc");
    TC_TRY(to_edwards_device(ctx, src, n, p));
    TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));   // shared with other contexts' streams
    *dst = p;
  }
  *out = *dst;
  return TC_OK;
}

int fixed_base_g(tc_ctx* ctx, const Fe* d_exps, uint64_t n, Aff* d_out) {
  cudaStream_t st = ctx->stream;
  Aff* table;
  TC_TRY(scratch_t(ctx, "srs.gtable", GT_WIN * GT_ENT, &table));
  // the table depends only on g: build it once per context
  static_assert(GT_WIN * GT_ENT < 8192, "table size");
  if (!ctx->scratch.count("srs.gtable.ready")) {
    k_gtable<<<blocks_for(GT_WIN * GT_ENT, 64), 64, 0, st>>>(table);
    TC_LAUNCHED(ctx);
    ctx->scratch["srs.gtable.ready"] = tc_ctx::Buf{};
  }
  if (n == 0) return TC_OK;
  uint64_t threads = (n + FB_K - 1) / FB_K;
  k_fixed<<<blocks_for(threads, 128), 128, 0, st>>>(table, d_exps, n, d_out);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

int srs_exponents(tc_ctx* ctx, const std::vector<Fe>& tabs_host, const uint32_t* shape, int m,
                  uint64_t n, Fe* d_exps) {
  cudaStream_t st = ctx->stream;
  std::vector<uint32_t> off(m), shp(shape, shape + m);
  uint32_t acc = 0;
  for (int j = 0; j < m; j++) {
    off[j] = acc;
    acc += shape[j];
  }
  Fe* d_tabs;
  uint32_t *d_off, *d_shape;
  TC_TRY(scratch_t(ctx, "srs.tabs", tabs_host.size(), &d_tabs));
  TC_TRY(scratch_t(ctx, "srs.off", m, &d_off));
  TC_TRY(scratch_t(ctx, "srs.shape", m, &d_shape));
  TC_CUDA(ctx, cudaMemcpyAsync(d_tabs, tabs_host.data(), tabs_host.size() * sizeof(Fe), cudaMemcpyHostToDevice, st));
  TC_CUDA(ctx, cudaMemcpyAsync(d_off, off.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  TC_CUDA(ctx, cudaMemcpyAsync(d_shape, shp.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  k_exps<<<blocks_for(n, 256), 256, 0, st>>>(d_tabs, d_off, d_shape, m, n, d_exps);
  TC_LAUNCHED(ctx);
  // the host vectors above are pageable: make the copies complete before they go away
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return TC_OK;
}

}  // namespace tcrt
