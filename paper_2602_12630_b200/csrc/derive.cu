// Trapdoor-free Lagrange SRS.
//
// A published SRS (TCSR) carries only the monomial elements
// G_i = g^{prod_j tau_j^{i_j}}.  The fast commit route needs the grid-Lagrange elements
// L_w = g^{prod_j L_{j,w_j}(tau_j)} (nodes 1..d_j, mvpoly.py:130-133) and, for the
// Lagrange-route openings, the same for every axis suffix.  L_w = sum_i C[w, i] G_i with
// C = (x)_j C_j, C_j[k, l] = coefficient of X^l in L_{j,k}(X) — the TRANSPOSE of the
// Lagrange->monomial interpolation matrix of mvpoly.py:193-230.  Applying it "in the
// exponent" with full scalars would cost d_j scalar multiplications per element and axis;
// instead the transpose of the Newton-form interpolation is applied, axis by axis:
//
//   1. monomial -> Newton basis N_l(X) = prod_{t=1..l} (X - t): in place on each fibre,
//        for l = 1..d-1, s = d-1 down to l:  B[s] -= l * B[s-1]
//      (R_{l,t} = tau^t N_l(tau) g satisfies R_{l,t} = R_{l-1,t+1} - l R_{l-1,t}; afterwards
//      B[l] = N_l(tau) g) — small-integer multiply-subtracts only;
//   2. one scalar per element: B[i] *= prod_j 1 / (i_j)!   (all axes at once);
//   3. Newton -> Lagrange: L_{k+1} = sum_{l>=k} (-1)^{l-k} C(l, k) N_l / l!, i.e. the Taylor
//      shift sum_l U_l (y - 1)^l:  for i = 0..d-2, k = d-2 down to i:  B[k] -= B[k+1]
//      — subtractions only.
//
// The three stages are separable linear maps, so they commute across axes.  Points live
// in the extended twisted Edwards coordinates of the MSM model (ec.cuh: the neutral element,
// which appears when a trapdoor hits a grid node, needs no special case); the result is
// mapped back to canonical affine points of the reference curve, so the bytes equal the
// trapdoor-generated elements (g^{L_w(tau)} is unique).  Cost per element: sum_j (d_j - 1)/2 small
// multiplications + one 162-bit multiplication + sum_j (d_j - 1)/2 additions.
#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr int DV_K = 8;   // points per thread sharing one inversion (final affine map)

TC_D Ext ld_ext_g(const Ext* p) { return ld_ext(p); }
TC_D void st_ext(Ext* p, const Ext& e) {
  uint4* q = (uint4*)p;
  const uint32_t* w[4] = {e.X.v, e.Y.v, e.Z.v, e.T.v};
  uint32_t a[24];
#pragma unroll
  for (int c = 0; c < 4; c++)
#pragma unroll
    for (int i = 0; i < 6; i++) a[6 * c + i] = w[c][i];
#pragma unroll
  for (int i = 0; i < 6; i++) q[i] = make_uint4(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]);
}

TC_D void ext_sub(Ext& acc, const Ext& q) { ext_add(acc, ext_neg(q)); }

// packed Edwards affine basis -> extended working points
__global__ void k_dv_load(const EdPk* __restrict__ in, uint64_t n, Ext* __restrict__ out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  st_ext(out + i, ext_from_aff(ld_edpk(in + i)));
}

// fibre f of an axis with d nodes and stride s (product of the later axes): elements
// base + k s, base = (f / s) d s + f % s; consecutive threads take consecutive f, so their
// accesses are adjacent whenever s > 1
__device__ __forceinline__ uint64_t fibre_base(uint64_t f, uint32_t d, uint64_t s) {
  return (f / s) * d * s + f % s;
}

// stage 1: monomial -> Newton basis along one axis
__global__ void __launch_bounds__(128) k_dv_newton(Ext* __restrict__ w, uint64_t nfib, uint32_t d, uint64_t s) {
  const uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (f >= nfib) return;
  Ext* b = w + fibre_base(f, d, s);
#pragma unroll 1
  for (uint32_t l = 1; l < d; l++) {
    Ext cur = ld_ext_g(b + (uint64_t)(d - 1) * s);   // old B[s]
#pragma unroll 1
    for (uint32_t k = d - 1; k >= l; k--) {
      const Ext prev = ld_ext_g(b + (uint64_t)(k - 1) * s);   // old B[k-1]
      ext_sub(cur, ext_mul_small_naf(prev, l));
      st_ext(b + (uint64_t)k * s, cur);
      cur = prev;
    }
  }
}

// stage 2: B[i] *= e_i (canonical F_p scalar), double-and-add from the top bit
__global__ void __launch_bounds__(128) k_dv_scale(Ext* __restrict__ w, const Fe* __restrict__ e, uint64_t n) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Fe k = e[i];
  const Ext p = ld_ext_g(w + i);
  Ext r = ext_zero();
  bool started = false;
#pragma unroll 1
  for (int b = 191; b >= 0; b--) {
    if (started) r = ext_dbl(r);
    if ((k.v[b >> 5] >> (b & 31)) & 1u) {
      if (started) {
        ext_add(r, p);
      } else {
        r = p;
        started = true;
      }
    }
  }
  st_ext(w + i, r);
}

// stage 3: Newton -> Lagrange (Taylor shift by -1) along one axis
__global__ void __launch_bounds__(128) k_dv_taylor(Ext* __restrict__ w, uint64_t nfib, uint32_t d, uint64_t s) {
  const uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (f >= nfib || d < 2) return;
  Ext* b = w + fibre_base(f, d, s);
#pragma unroll 1
  for (uint32_t i = 0; i + 1 < d; i++) {
    Ext nxt = ld_ext_g(b + (uint64_t)(d - 1) * s);   // B[k+1], already updated in this pass
#pragma unroll 1
    for (int k = (int)d - 2; k >= (int)i; k--) {
      Ext v = ld_ext_g(b + (uint64_t)k * s);
      ext_sub(v, nxt);
      st_ext(b + (uint64_t)k * s, v);
      nxt = v;
    }
  }
}

// Edwards points of the MSM model -> canonical E affine (ec.cuh ext_to_aff: psi, one
// inversion), DV_K points per thread sharing one inversion; the neutral element -> infinity
__global__ void __launch_bounds__(128) k_dv_store(const Ext* __restrict__ w, uint64_t n, Aff* __restrict__ out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t i0 = t * DV_K;
  if (i0 >= n) return;
  const int cnt = (n - i0 < (uint64_t)DV_K) ? (int)(n - i0) : DV_K;
  Fe pref[DV_K];
  Fe run = Fq::one();
  for (int k = 0; k < cnt; k++) {
    const Ext p = ld_ext_g(w + i0 + k);
    pref[k] = run;
    run = Fq::mul(run, ext_to_aff_den(p));
  }
  Fe inv = Fq::inv(run);
  for (int k = cnt - 1; k >= 0; k--) {
    const Ext p = ld_ext_g(w + i0 + k);
    const Fe den = ext_to_aff_den(p);
    const Fe ik = Fq::mul(inv, pref[k]);
    inv = Fq::mul(inv, den);
    Aff r = ext_to_aff_with_inv(p, ik);
    if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
    out[i0 + k] = r;
  }
}

// 1 / l! mod p for l < d (canonical), per axis, concatenated
void inv_fact_tables(const uint32_t* shape, int m, std::vector<Fe>& out) {
  for (int j = 0; j < m; j++) {
    Fe f = Fp::one();   // Montgomery
    std::vector<Fe> fact(shape[j]);
    for (uint32_t l = 0; l < shape[j]; l++) {
      if (l) f = Fp::mul(f, Fp::to_mont_small(l));
      fact[l] = f;
    }
    for (uint32_t l = 0; l < shape[j]; l++) out.push_back(Fp::from_mont(Fp::inv_fast(fact[l])));
  }
}

}  // namespace

namespace tcrt {

static int derive_run(tc_ctx* ctx, const EdPk* d_mono, const uint32_t* shape, int m, uint64_t n, Ext* w, Fe* e,
                      Aff* d_out);

// Lagrange elements of `shape` (n points, lex order) from the Edwards monomial elements of
// the same shape; `out` receives canonical Montgomery-curve affine points.
int derive_lagrange_device(tc_ctx* ctx, const EdPk* d_mono, const uint32_t* shape, int m, Aff* d_out) {
  cudaStream_t st = ctx->stream;
  uint64_t n = 1;
  for (int j = 0; j < m; j++) n *= shape[j];
  if (n == 0) return TC_OK;
  // setup-only working memory (96 + 24 B per point: 4.8 GB for config 5), released on return
  Ext* w = nullptr;
  Fe* e = nullptr;
  if (cudaMalloc(&w, n * sizeof(Ext)) != cudaSuccess || cudaMalloc(&e, n * sizeof(Fe)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(w);
    return fail(ctx, TC_ERR_MEMORY, "derive: working memory for %llu points", (unsigned long long)n);
  }
  const int s = derive_run(ctx, d_mono, shape, m, n, w, e, d_out);
  cudaStreamSynchronize(st);
  cudaFree(w);
  cudaFree(e);
  return s;
}

static int derive_run(tc_ctx* ctx, const EdPk* d_mono, const uint32_t* shape, int m, uint64_t n, Ext* w, Fe* e,
                      Aff* d_out) {
  cudaStream_t st = ctx->stream;
  k_dv_load<<<blocks_for(n, 256), 256, 0, st>>>(d_mono, n, w);
  TC_LAUNCHED(ctx);
  for (int j = 0; j < m; j++) {
    if (shape[j] < 2) continue;
    uint64_t s = 1;
    for (int k = j + 1; k < m; k++) s *= shape[k];
    const uint64_t nfib = n / shape[j];
    k_dv_newton<<<blocks_for(nfib, 128), 128, 0, st>>>(w, nfib, shape[j], s);
    TC_LAUNCHED(ctx);
  }
  std::vector<Fe> tabs;
  inv_fact_tables(shape, m, tabs);
  TC_TRY(srs_exponents(ctx, tabs, shape, m, n, e));
  k_dv_scale<<<blocks_for(n, 128), 128, 0, st>>>(w, e, n);
  TC_LAUNCHED(ctx);
  for (int j = 0; j < m; j++) {
    if (shape[j] < 2) continue;
    uint64_t s = 1;
    for (int k = j + 1; k < m; k++) s *= shape[k];
    const uint64_t nfib = n / shape[j];
    k_dv_taylor<<<blocks_for(nfib, 128), 128, 0, st>>>(w, nfib, shape[j], s);
    TC_LAUNCHED(ctx);
  }
  k_dv_store<<<blocks_for((n + DV_K - 1) / DV_K, 128), 128, 0, st>>>(w, n, d_out);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

}  // namespace tcrt
