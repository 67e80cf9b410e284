// Small fixed-base MSMs (Terkle node commitments, and the quotient MSMs of
// node openings): L independent MSMs over an SRS of only B <= 64 points with full 162-bit
// scalars.  Pippenger is the wrong tool here (its window-combination Horner is ~160
// sequential doublings); instead every SRS point gets a byte-window table
//     tab[k][w][j] = (j+1) * 2^{8w} * G_k   (21 windows x 255 entries, twisted Edwards affine)
// built once per SRS, and one warp per MSM sums the <= 21*B table entries selected by the
// scalar bytes (complete 8M mixed adds), reduces across lanes with shuffles and converts
// to canonical Montgomery affine.
#include "sha256.cuh"
#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr int SW = 21;    // byte windows (168 >= 162 bits)
constexpr int SE = 255;   // non-zero byte values

// Q[k][w] = 2^{8w} G_k  (one thread per point, sequential doublings)
__global__ void k_tab_bases(const Aff* pts, uint32_t B, Xyzz* q) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= B) return;
  Xyzz acc = xyzz_mul_half(pts[k]);   // the MSM model's bases are phi([h] G_k) (ec.cuh)
  for (int w = 0; w < SW; w++) {
    q[k * SW + w] = acc;
    for (int i = 0; i < 8; i++) acc = xyzz_dbl(acc);
  }
}

// tab[k][w][j] = (j+1) Q[k][w], twisted Edwards affine (x, y, xy): the MSM kernel then
// runs complete, branch-free 8M mixed adds
__global__ void k_tab_fill(const Xyzz* q, uint32_t B, EdAff* tab) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * SW * SE) return;
  uint32_t j = t % SE + 1, kw = t / SE;
  const Xyzz base = q[kw];
  Xyzz acc = xyzz_inf();
  for (int b = 7; b >= 0; b--) {
    acc = xyzz_dbl(acc);
    if ((j >> b) & 1u) xyzz_add(acc, base);
  }
  Aff r = xyzz_to_aff(acc);
  if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
  const EdAff e = aff_to_ed_noh(r);   // r = (j+1) 2^{8w} [h] G_k
  tab[t] = EdAff{Fq::red2(e.x), Fq::red2(e.y), Fq::red2(e.t)};
}

__device__ __forceinline__ Ext shfl_ext(const Ext& p, int src) {
  Ext r;
#pragma unroll
  for (int i = 0; i < 6; i++) {
    r.X.v[i] = __shfl_down_sync(0xffffffffu, p.X.v[i], src);
    r.Y.v[i] = __shfl_down_sync(0xffffffffu, p.Y.v[i], src);
    r.Z.v[i] = __shfl_down_sync(0xffffffffu, p.Z.v[i], src);
    r.T.v[i] = __shfl_down_sync(0xffffffffu, p.T.v[i], src);
  }
  return r;
}

// one warp per MSM; scalars are canonical F_p limbs: ptrs[l][k], k < B
__global__ void __launch_bounds__(128) k_small_msm(const Fe* const* ptrs, uint32_t L, uint32_t B, const EdAff* tab,
                                                   Aff* out) {
  const uint32_t l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (l >= L) return;   // whole warps exit together
  const Fe* s = ptrs[l];
  Ext acc = ext_zero();
  for (uint32_t kw = lane; kw < B * SW; kw += 32) {
    const uint32_t k = kw / SW, w = kw % SW;
    const uint32_t byte = (s[k].v[w >> 2] >> (8 * (w & 3))) & 0xffu;
    if (byte) ext_madd(acc, ld_edaff(tab + (uint64_t)kw * SE + byte - 1));
  }
#pragma unroll 1   // one copy of the add: these latency-bound kernels would miss the icache
  for (int o = 16; o; o >>= 1) {
    Ext other = shfl_ext(acc, o);
    if (lane < (uint32_t)o) ext_add(acc, other);
  }
  if (lane == 0) {
    Aff r = ext_to_aff(acc);
    if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
    out[l] = r;
  }
}

// Terkle leaves on the device: vals[i] = hash_to_scalar(encode_elem(C_i), "terkle/leaf")
// (backend.py:309-317, 346-348) for i < count, zero padding up to cap
__global__ void k_leaf_hash(const Aff* comms, uint32_t count, uint64_t cap, Fe* vals) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= cap) return;
  if (i >= count) {
    vals[i] = Fe{{0, 0, 0, 0, 0, 0}};
    return;
  }
  vals[i] = hash_point_to_scalar(comms[i], false);
}

// The tail of a forward's commit + tree (the deferred MSM finish): warp l sums MSM l's
// prescaled window sums, converts the commitment to canonical affine and hashes its leaf
// (the inversions of all MSMs run in parallel, 4 warps per SM); warps >= count write the
// zero padding up to cap.  One launch instead of k_final_sum + k_leaf_hash.
__global__ void __launch_bounds__(128) k_final_leaf(const Ext* wsum, uint32_t count, int nwin, uint32_t cap, Aff* pts,
                                                    Fe* vals) {
  const uint32_t l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (l >= cap) return;   // whole warps
  if (l >= count) {
    if (lane == 0) vals[l] = Fe{{0, 0, 0, 0, 0, 0}};
    return;
  }
  Ext acc = ext_zero();
  for (int k = (int)lane; k < nwin; k += 32) ext_add(acc, ld_ext(wsum + (uint64_t)l * nwin + k));
  if (nwin > 1) {
#pragma unroll 1
    for (int o = 16; o; o >>= 1) {
      Ext other = shfl_ext(acc, o);
      if (lane < (uint32_t)o) ext_add(acc, other);
    }
  }
  if (lane == 0) {
    Aff r = ext_to_aff(acc);
    if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
    pts[l] = r;
    vals[l] = hash_point_to_scalar(r, false);
  }
}

// One Terkle level with one BLOCK per node: the node's B x 21 byte-window entries spread
// over TL_THREADS lanes (one mixed add each for B = 8), warp shuffles, then the warps'
// partial sums through shared memory; thread 0 converts, stores and hashes for the parent.
constexpr int TL_THREADS = 256;
__global__ void __launch_bounds__(TL_THREADS) k_terkle_level_b(const Fe* vals, uint32_t B, const EdAff* tab, Aff* pts,
                                                               Fe* next) {
  __shared__ Ext part[TL_THREADS / 32];
  const uint32_t u = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const Fe* sv = vals + (uint64_t)u * B;
  Ext acc = ext_zero();
  for (uint32_t kw = t; kw < B * SW; kw += TL_THREADS) {
    const uint32_t k = kw / SW, wi = kw % SW;
    const uint32_t byte = (sv[k].v[wi >> 2] >> (8 * (wi & 3))) & 0xffu;
    if (byte) ext_madd(acc, ld_edaff(tab + (uint64_t)kw * SE + byte - 1));
  }
#pragma unroll 1   // one copy of the add: these latency-bound kernels would miss the icache
  for (int o = 16; o; o >>= 1) {
    Ext other = shfl_ext(acc, o);
    if (lane < (uint32_t)o) ext_add(acc, other);
  }
  if (lane == 0) part[w] = acc;
  __syncthreads();
  if (t >= 32) return;
  acc = t < TL_THREADS / 32 ? part[t] : ext_zero();
#pragma unroll 1
  for (int o = TL_THREADS / 64; o; o >>= 1) {
    Ext other = shfl_ext(acc, o);
    if (lane < (uint32_t)o) ext_add(acc, other);
  }
  if (t == 0) {
    Aff r = ext_to_aff(acc);
    if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
    pts[u] = r;
    if (next) next[u] = hash_point_to_scalar(r, true);
  }
}

}  // namespace

namespace tcrt {

int leaf_hash_device(tc_ctx* ctx, const Aff* d_comms, int count, uint64_t cap, Fe* d_vals) {
  k_leaf_hash<<<blocks_for(cap, 64), 64, 0, ctx->stream>>>(d_comms, (uint32_t)count, cap, d_vals);
  TC_LAUNCHED(ctx);
  return TC_OK;
}


// build (once) the byte-window tables of the SRS's `which` elements
static int small_tables(tc_ctx* ctx, tc_srs* srs, int which, const EdAff** out) {
  std::lock_guard<std::mutex> guard(srs->mu);
  const int idx = (which == TC_SRS_LAGRANGE) ? 1 : 0;
  if (!srs->small_tab[idx]) {
    const Aff* pts = idx ? srs->lagrange : srs->monomial;
    if (!pts) return fail(ctx, TC_ERR_VALUE, "srs has no elements of kind %d", which);
    const uint32_t B = (uint32_t)srs->n;
    Xyzz* q;
    TC_TRY(scratch_t(ctx, "small.q", (uint64_t)B * SW, &q));
    EdAff* tab = nullptr;
    TC_CUDA(ctx, cudaMalloc(&tab, (size_t)B * SW * SE * sizeof(EdAff)));
    k_tab_bases<<<blocks_for(B, 32), 32, 0, ctx->stream>>>(pts, B, q);
    TC_LAUNCHED(ctx);
    k_tab_fill<<<blocks_for((uint64_t)B * SW * SE, 128), 128, 0, ctx->stream>>>(q, B, tab);
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    srs->small_tab[idx] = tab;
  }
  *out = srs->small_tab[idx];
  return TC_OK;
}

int small_msm_device(tc_ctx* ctx, tc_srs* srs, int which, const void* const* h_ptrs, int L, Aff* d_out) {
  if (L <= 0) return TC_OK;
  if (srs->n > ::SMALL_MSM_MAX) return fail(ctx, TC_ERR_VALUE, "small msm: srs too large");
  const EdAff* tab;
  TC_TRY(small_tables(ctx, srs, which, &tab));
  const Fe** d_ptrs;
  TC_TRY(scratch_t(ctx, "small.ptrs", (uint64_t)L, (Fe***)&d_ptrs));
  memcpy(ctx->h_stage, h_ptrs, sizeof(void*) * L);
  TC_CUDA(ctx, cudaMemcpyAsync(d_ptrs, ctx->h_stage, sizeof(void*) * L, cudaMemcpyHostToDevice, ctx->stream));
  k_small_msm<<<blocks_for((uint64_t)L * 32, 128), 128, 0, ctx->stream>>>(d_ptrs, (uint32_t)L, (uint32_t)srs->n, tab,
                                                                          d_out);
  TC_LAUNCHED(ctx);
  // the pointer upload reads h_stage asynchronously: finish before h_stage is reused
  TC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return TC_OK;
}

int tree_tail_device(tc_ctx* ctx, tc_srs* node_srs, const Ext* wsum, int count, int nwin, uint64_t cap, int L,
                     Aff* d_pts, Fe* d_levels) {
  const EdAff* tab;
  TC_TRY(small_tables(ctx, node_srs, TC_SRS_LAGRANGE, &tab));
  const uint32_t B = (uint32_t)node_srs->n;
  // level 0's child values (the leaves) go straight into d_levels
  k_final_leaf<<<blocks_for(cap * 32, 128), 128, 0, ctx->stream>>>(wsum, (uint32_t)count, nwin, (uint32_t)cap, d_pts,
                                                                  d_levels);
  TC_LAUNCHED(ctx);
  uint64_t width = cap, in_off = 0, pts_off = count;
  for (int l = 0; l < L; l++) {
    const uint32_t nodes = (uint32_t)(width / B);
    Fe* out = l + 1 < L ? d_levels + in_off + width : nullptr;
    k_terkle_level_b<<<nodes, TL_THREADS, 0, ctx->stream>>>(d_levels + in_off, B, tab, d_pts + pts_off, out);
    TC_LAUNCHED(ctx);
    in_off += width;
    pts_off += nodes;
    width = nodes;
  }
  return TC_OK;
}

// The whole Terkle tree over `cap` (= B^L, zero-padded) canonical leaf values already on
// the device: L launches, no host synchronisation between levels; node points (level by
// level, bottom first) in d_pts.  Lagrange node SRS (grid values are the node tensor).
int terkle_device(tc_ctx* ctx, tc_srs* srs, Fe* d_vals, uint64_t cap, int L, Aff* d_pts, Fe* d_levels) {
  const EdAff* tab;
  TC_TRY(small_tables(ctx, srs, TC_SRS_LAGRANGE, &tab));
  const uint32_t B = (uint32_t)srs->n;
  Fe* cur = d_vals;
  Fe* nxt;
  TC_TRY(scratch_t(ctx, "terkle.next", cap / B + 1, &nxt));
  uint64_t written = 0, width = cap;
  if (d_levels) {   // keep every level's child values: level l's inputs at d_levels + sum of wider levels
    TC_CUDA(ctx, cudaMemcpyAsync(d_levels, d_vals, cap * sizeof(Fe), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  uint64_t lvl_off = cap;
  for (int l = 0; l < L; l++) {
    const uint32_t nodes = (uint32_t)(width / B);
    Fe* out_vals = (l + 1 < L) ? (d_levels ? d_levels + lvl_off : (cur == d_vals ? nxt : d_vals)) : nullptr;
    if (l + 1 < L) lvl_off += nodes;
    k_terkle_level_b<<<nodes, TL_THREADS, 0, ctx->stream>>>(cur, B, tab, d_pts + written, out_vals);
    TC_LAUNCHED(ctx);
    written += nodes;
    width = nodes;
    if (out_vals) cur = out_vals;
  }
  return TC_OK;
}

}  // namespace tcrt
