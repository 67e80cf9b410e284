// K3: batched Pippenger multi-scalar multiplication
//     out[l] = sum_k a_{l,k} * G_k      l = 0..L-1, all L MSMs over the SAME bases G.
//
// The reference composes one MSM as a fold of `exp` (double-and-add, backend.py:202-217)
// and `mul` (affine add, backend.py:185-200) — 1.5 ms per term on a CPU core
// designates it the single performance hot-spot.  The prover runs many MSMs against one
// SRS (32 layers per forward, m quotients per opening, 8 nodes per Terkle level), so the
// whole batch goes through ONE pipeline:
//   1. k_scan_bits    — max bit length of the centred scalar magnitudes + quantisation
//                       errors (scalars are either canonical F_p limbs or raw floats that
//                       are quantised on the fly, fusing K1 into the MSM)
//   2. k_digits       — signed c-bit window digits; only NON-ZERO digits are emitted,
//                       compacted per block: key = (l*nwin + w)*B + |d|-1, value =
//                       point index | sign<<31
//   3. radix sort     — (key, value) by bucket, CUB onesweep over the used key bits
//   4. k_bounds       — [start, end) of every bucket
//   5. levels         — load-balanced segmented reduction: each bucket is cut into pieces
//                       of <= T entries, one thread per piece (XYZZ accumulator, mixed
//                       affine adds at level 0); piece sums feed the next level until every
//                       bucket is one point (heavy-tailed activations make a few buckets
//                       huge — they get split, not serialised)
//   6. k_bucket_reduce— per (msm, window, segment of buckets): sum_b b * B_b by running sums
//   7. k_window_sum, k_final — segments -> window sums -> Horner over windows -> affine
// Affine outputs are canonical and the group is abelian, so any window size, bucket order
// or coordinate system reproduces the reference's bytes exactly.
#include <cub/cub.cuh>

#include "quant.cuh"
#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr uint32_t SIGN_BIT = 0x80000000u;
constexpr int DT_LIMBS = 0;   // template code for canonical F_p scalars

__device__ __forceinline__ uint32_t bitlen6(const Fe& a) {
#pragma unroll
  for (int i = 5; i >= 0; i--)
    if (a.v[i]) return 32u * i + 32u - __clz(a.v[i]);
  return 0u;
}

template <int DT>
__device__ __forceinline__ void load_scalar(const void* p, uint64_t i, int scale_bits, Fe& mag, bool& neg,
                                            uint32_t& flags) {
  if (DT == DT_LIMBS) {
    const uint2* q = (const uint2*)((const Fe*)p + i);
    uint2 a = q[0], b = q[1], c = q[2];
    Fe v{{a.x, a.y, b.x, b.y, c.x, c.y}};
    centre_fp(v, mag, neg);
  } else {
    quantize_signed<DT>(p, i, scale_bits, mag, neg, flags);
  }
}

__device__ __forceinline__ uint32_t window_bits(const Fe& m, int lo, int c) {
  int limb = lo >> 5, sh = lo & 31;
  if (limb >= 6) return 0;
  uint64_t w = m.v[limb];
  if (limb + 1 < 6) w |= (uint64_t)m.v[limb + 1] << 32;
  return (uint32_t)(w >> sh) & ((1u << c) - 1u);
}

template <int DT>
__global__ void k_scan_bits(const void* const* ptrs, uint64_t n, int scale_bits, uint32_t* out) {
  const void* p = ptrs[blockIdx.y];
  uint32_t mx = 0, f = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Fe mag;
    bool neg;
    load_scalar<DT>(p, i, scale_bits, mag, neg, f);
    mx = max(mx, bitlen6(mag));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    f |= __shfl_xor_sync(0xffffffffu, f, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx) atomicMax(out, mx);
    if (f) atomicOr(out + 1, f);
  }
}

// signed digits of `mag`: calls emit(w, |d|, digit_negative) for every non-zero digit
template <class F>
__device__ __forceinline__ void for_digits(const Fe& mag, int c, int nwin, F&& emit) {
  const uint32_t half = 1u << (c - 1), full = 1u << c;
  uint32_t carry = 0;
  for (int w = 0; w < nwin; w++) {
    uint32_t d = window_bits(mag, w * c, c) + carry;
    bool dn = false;
    if (d > half) {   // d - 2^c, carry into the next window
      d = full - d;
      dn = true;
      carry = 1;
    } else {
      carry = 0;
    }
    if (d) emit(w, d, dn);
  }
}

template <int DT>
__global__ void __launch_bounds__(256) k_digits(const void* const* ptrs, uint64_t n, int scale_bits, int c, int nwin,
                                                uint32_t* keys, uint32_t* vals, uint32_t* count) {
  __shared__ uint32_t warp_tot[8];
  __shared__ uint32_t base;
  const uint32_t l = blockIdx.y;
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t B = 1u << (c - 1);
  Fe mag;
  bool neg = false;
  uint32_t f = 0, cnt = 0;
  if (i < n) {
    load_scalar<DT>(ptrs[l], i, scale_bits, mag, neg, f);
    for_digits(mag, c, nwin, [&](int, uint32_t, bool) { cnt++; });
  }
  // block-wide exclusive scan of cnt
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      uint32_t t = warp_tot[w];
      warp_tot[w] = s;
      s += t;
    }
    base = s ? atomicAdd(count, s) : 0u;
  }
  __syncthreads();
  uint32_t pos = base + warp_tot[wid] + incl - cnt;
  if (cnt) {
    const uint32_t key0 = l * (uint32_t)nwin * B;
    for_digits(mag, c, nwin, [&](int w, uint32_t d, bool dn) {
      keys[pos] = key0 + (uint32_t)w * B + d - 1u;
      vals[pos] = (uint32_t)i | ((neg != dn) ? SIGN_BIT : 0u);
      pos++;
    });
  }
}

__global__ void k_bounds(const uint32_t* keys, const uint32_t* count, uint32_t* bstart, uint32_t* bend) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t E = *count;
  if (j >= E) return;
  uint32_t k = keys[j];
  if (j == 0 || keys[j - 1] != k) bstart[k] = (uint32_t)j;
  if (j + 1 == E || keys[j + 1] != k) bend[k] = (uint32_t)j + 1u;
}

// pieces per bucket; np has nb+1 entries (last = 0).  Sizes from [bstart, bend) or from
// the previous level's offsets (prev_off != nullptr).
__global__ void k_piece_count(const uint32_t* bstart, const uint32_t* bend, const uint32_t* prev_off, uint32_t nb,
                              uint32_t T, uint32_t* np) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nb) return;
  if (k == nb) {
    np[k] = 0;
    return;
  }
  uint32_t sz = prev_off ? prev_off[k + 1] - prev_off[k] : bend[k] - bstart[k];
  np[k] = (sz + T - 1) / T;
}

__device__ __forceinline__ uint32_t find_bucket(const uint32_t* off, uint32_t nb, uint32_t p) {
  uint32_t lo = 0, hi = nb;   // off[lo] <= p < off[hi]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= p)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// level 0: entries are (sign | point index) into the shared affine bases
__global__ void __launch_bounds__(128) k_accum_aff(const uint32_t* vals, const Aff* bases, const uint32_t* bstart,
                                                   const uint32_t* bend, const uint32_t* off, uint32_t nb, uint32_t T,
                                                   Xyzz* out) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t total = off[nb];
  if (p >= total) return;
  uint32_t k = find_bucket(off, nb, p);
  uint32_t a = bstart[k] + (p - off[k]) * T;
  uint32_t b = min(a + T, bend[k]);
  Xyzz acc = xyzz_inf();
  for (uint32_t j = a; j < b; j++) {
    uint32_t v = vals[j];
    Aff q = bases[v & ~SIGN_BIT];
    if (v & SIGN_BIT) q.y = Fq::neg(q.y);
    xyzz_add_aff(acc, q);
  }
  out[p] = acc;
}

// level >= 1: bucket k's entries are in[prev_off[k] .. prev_off[k+1])
__global__ void __launch_bounds__(128) k_accum_xyzz(const Xyzz* in, const uint32_t* prev_off, const uint32_t* off,
                                                    uint32_t nb, uint32_t T, Xyzz* out) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t total = off[nb];
  if (p >= total) return;
  uint32_t k = find_bucket(off, nb, p);
  uint32_t a = prev_off[k] + (p - off[k]) * T;
  uint32_t b = min(a + T, prev_off[k + 1]);
  Xyzz acc = in[a];
  for (uint32_t j = a + 1; j < b; j++) xyzz_add(acc, in[j]);
  out[p] = acc;
}

__global__ void k_gather_buckets(const Xyzz* in, const uint32_t* off, uint32_t nb, Xyzz* buckets) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  buckets[k] = (off[k + 1] > off[k]) ? in[off[k]] : xyzz_inf();
}

// per (window, segment): sum_{b in seg} (b+1) * B_b via running sums from the top
__global__ void __launch_bounds__(128) k_bucket_reduce(const Xyzz* buckets, uint32_t B, uint32_t nwin_total,
                                                       uint32_t LS, Xyzz* segs) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t nseg = B / LS;
  if (t >= nwin_total * nseg) return;
  uint32_t w = t / nseg, s = t % nseg;
  uint32_t lo = s * LS;
  const Xyzz* bw = buckets + (uint64_t)w * B;
  Xyzz run = xyzz_inf(), sum = xyzz_inf();
  for (int b = (int)(lo + LS) - 1; b >= (int)lo; b--) {
    xyzz_add(run, bw[b]);
    xyzz_add(sum, run);
  }
  if (lo) {   // sum_b (b - lo + 1) B_b + lo * sum_b B_b
    Xyzz extra = xyzz_mul_small(run, lo);
    xyzz_add(sum, extra);
  }
  segs[t] = sum;
}

__global__ void __launch_bounds__(128) k_window_sum(const Xyzz* segs, uint32_t nseg, Xyzz* wsum) {
  __shared__ Xyzz sh[128];
  uint32_t w = blockIdx.x;
  Xyzz acc = xyzz_inf();
  for (uint32_t s = threadIdx.x; s < nseg; s += blockDim.x) xyzz_add(acc, segs[(uint64_t)w * nseg + s]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (uint32_t st = blockDim.x / 2; st; st >>= 1) {
    if (threadIdx.x < st) {
      Xyzz a = sh[threadIdx.x];
      xyzz_add(a, sh[threadIdx.x + st]);
      sh[threadIdx.x] = a;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) wsum[w] = sh[0];
}

// Horner over the windows of MSM l: sum_w 2^{c w} S_{l,w}, then canonical affine
__global__ void k_final(const Xyzz* wsum, uint32_t L, uint32_t nwin, uint32_t c, Aff* out) {
  uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const Xyzz* ws = wsum + (uint64_t)l * nwin;
  Xyzz acc = ws[nwin - 1];
  for (int w = (int)nwin - 2; w >= 0; w--) {
    for (uint32_t i = 0; i < c; i++) acc = xyzz_dbl(acc);
    xyzz_add(acc, ws[w]);
  }
  Aff r = xyzz_to_aff(acc);
  if (!aff_is_inf(r)) {
    r.x = Fq::canon(r.x);
    r.y = Fq::canon(r.y);
  }
  out[l] = r;
}

__global__ void k_fill_inf(Aff* out, uint32_t L) {
  uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < L) out[l] = aff_inf();
}

uint32_t bitlen_u32(uint32_t v) { return v ? 32u - __builtin_clz(v) : 0u; }

// window size minimising ~ nwin * (entries + 2.5 * buckets) per MSM
int choose_c(uint64_t n, uint32_t nbits) {
  int best_c = 4;
  double best = 1e300;
  for (int c = 4; c <= 20; c++) {
    uint32_t nwin = (nbits + 1 + c - 1) / c;
    double cost = (double)nwin * ((double)n + 2.5 * (double)(1u << (c - 1)));
    if (cost < best) {
      best = cost;
      best_c = c;
    }
  }
  return best_c;
}

template <class F>
int dispatch_dt(tc_ctx* ctx, int dtype, F&& f) {
  switch (dtype) {
    case TC_DTYPE_FP_LIMBS: f(std::integral_constant<int, DT_LIMBS>()); return TC_OK;
    case TC_DTYPE_F16: f(std::integral_constant<int, 1>()); return TC_OK;
    case TC_DTYPE_BF16: f(std::integral_constant<int, 2>()); return TC_OK;
    case TC_DTYPE_F32: f(std::integral_constant<int, 3>()); return TC_OK;
    case TC_DTYPE_F64: f(std::integral_constant<int, 4>()); return TC_OK;
    default: return tcrt::fail(ctx, TC_ERR_ARGUMENT, "msm: unsupported scalar dtype %d", dtype);
  }
}

}  // namespace

namespace tcrt {

int quantize_flags_to_status(tc_ctx* ctx, uint32_t f);

int msm_batch_device(tc_ctx* ctx, int dtype, int scale_bits, const void* const* h_ptrs, int L, const Aff* d_bases,
                     uint64_t n, Aff* d_out) {
  cudaStream_t st = ctx->stream;
  if (L <= 0) return TC_OK;
  if (n >= (1ull << 31)) return fail(ctx, TC_ERR_VALUE, "msm: too many points (%llu)", (unsigned long long)n);
  if (dtype != TC_DTYPE_FP_LIMBS && (scale_bits < 0 || scale_bits > 160))
    return fail(ctx, TC_ERR_VALUE, "quantize: scale_bits out of range");
  if (n == 0) {
    k_fill_inf<<<blocks_for(L, 64), 64, 0, st>>>(d_out, (uint32_t)L);
    TC_LAUNCHED(ctx);
    return TC_OK;
  }
  // scalar pointers -> device (pinned staging; the syncs below keep it alive)
  const void** d_ptrs;
  TC_TRY(scratch_t(ctx, "msm.ptrs", (uint64_t)L, (void***)&d_ptrs));
  memcpy(ctx->h_stage, h_ptrs, sizeof(void*) * L);
  TC_CUDA(ctx, cudaMemcpyAsync(d_ptrs, ctx->h_stage, sizeof(void*) * L, cudaMemcpyHostToDevice, st));

  // 1. magnitude bits + quantisation status
  uint32_t* d_small;
  TC_TRY(scratch_t(ctx, "msm.small", 8, &d_small));
  TC_CUDA(ctx, cudaMemsetAsync(d_small, 0, 8 * sizeof(uint32_t), st));
  {
    unsigned gx = std::min<unsigned>(blocks_for(n, 256), std::max(1u, (unsigned)ctx->num_sms * 8 / (unsigned)L + 1));
    int s = dispatch_dt(ctx, dtype, [&](auto dt) {
      k_scan_bits<decltype(dt)::value><<<dim3(gx, L), 256, 0, st>>>(d_ptrs, n, scale_bits, d_small);
    });
    if (s) return s;
    TC_LAUNCHED(ctx);
  }
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags, d_small, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  const uint32_t nbits = ctx->h_flags[0];
  TC_TRY(quantize_flags_to_status(ctx, ctx->h_flags[1]));
  if (nbits == 0) {
    k_fill_inf<<<blocks_for(L, 64), 64, 0, st>>>(d_out, (uint32_t)L);
    TC_LAUNCHED(ctx);
    return TC_OK;
  }

  const int c = choose_c(n, nbits);
  const uint32_t nwin = (nbits + 1 + c - 1) / c;
  const uint32_t B = 1u << (c - 1);
  const uint64_t nb64 = (uint64_t)L * nwin * B;
  if (nb64 >= (1ull << 31)) return fail(ctx, TC_ERR_VALUE, "msm batch too large (%llu buckets)", (unsigned long long)nb64);
  const uint32_t nb = (uint32_t)nb64;
  const uint64_t cap = (uint64_t)L * n * nwin;
  const int end_bit = (int)bitlen_u32(nb - 1);

  // 2. non-zero digits, compacted
  uint32_t *keys, *vals, *keys2, *vals2;
  TC_TRY(scratch_t(ctx, "msm.keys", cap, &keys));
  TC_TRY(scratch_t(ctx, "msm.vals", cap, &vals));
  TC_TRY(scratch_t(ctx, "msm.keys2", cap, &keys2));
  TC_TRY(scratch_t(ctx, "msm.vals2", cap, &vals2));
  uint32_t* d_count = d_small + 2;
  {
    int s = dispatch_dt(ctx, dtype, [&](auto dt) {
      k_digits<decltype(dt)::value><<<dim3(blocks_for(n, 256), L), 256, 0, st>>>(d_ptrs, n, scale_bits, c, (int)nwin,
                                                                                  keys, vals, d_count);
    });
    if (s) return s;
    TC_LAUNCHED(ctx);
  }
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags + 2, d_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  const uint64_t E = ctx->h_flags[2];
  if (E == 0) {
    k_fill_inf<<<blocks_for(L, 64), 64, 0, st>>>(d_out, (uint32_t)L);
    TC_LAUNCHED(ctx);
    return TC_OK;
  }

  // 3. sort by bucket
  size_t tmp_bytes = 0;
  cub::DoubleBuffer<uint32_t> dk(keys, keys2), dv(vals, vals2);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int)E, 0, end_bit, st);
  void* d_tmp;
  TC_TRY(scratch(ctx, "msm.cubtmp", tmp_bytes, &d_tmp));
  TC_CUDA(ctx, cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, dk, dv, (int)E, 0, end_bit, st));
  ctx->launches += 1 + (end_bit + 7) / 8;
  const uint32_t* skeys = dk.Current();
  const uint32_t* svals = dv.Current();

  // 4. bucket bounds
  uint32_t *bstart, *bend;
  TC_TRY(scratch_t(ctx, "msm.bstart", (uint64_t)nb + 1, &bstart));
  TC_TRY(scratch_t(ctx, "msm.bend", (uint64_t)nb + 1, &bend));
  TC_CUDA(ctx, cudaMemsetAsync(bstart, 0, ((uint64_t)nb + 1) * sizeof(uint32_t), st));
  TC_CUDA(ctx, cudaMemsetAsync(bend, 0, ((uint64_t)nb + 1) * sizeof(uint32_t), st));
  k_bounds<<<blocks_for(E, 256), 256, 0, st>>>(skeys, d_count, bstart, bend);
  TC_LAUNCHED(ctx);

  // 5. levels of load-balanced segmented reduction (a bucket holds <= n entries)
  // level 0 sums runs of T affine entries; later levels sum T1 partial points per thread
  // (short sequential chains keep the latency of the few huge buckets low)
  const uint32_t T = (E >= (1u << 20)) ? 32u : (E >= (1u << 14) ? 16u : 8u);
  const uint32_t T1 = 8u;
  int levels = 1;
  for (uint64_t capT = T; capT < n; capT *= T1) levels++;
  const uint64_t max_items = (E + T - 1) / T + nb;
  uint32_t *offA, *offB, *np;
  Xyzz *itemsA, *itemsB, *buckets;
  TC_TRY(scratch_t(ctx, "msm.offA", (uint64_t)nb + 1, &offA));
  TC_TRY(scratch_t(ctx, "msm.offB", (uint64_t)nb + 1, &offB));
  TC_TRY(scratch_t(ctx, "msm.np", (uint64_t)nb + 1, &np));
  TC_TRY(scratch_t(ctx, "msm.itemsA", max_items, &itemsA));
  TC_TRY(scratch_t(ctx, "msm.itemsB", max_items, &itemsB));
  TC_TRY(scratch_t(ctx, "msm.buckets", nb, &buckets));
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, np, offA, (int)(nb + 1), st);
  void* d_scan;
  TC_TRY(scratch(ctx, "msm.scantmp", scan_bytes, &d_scan));

  k_piece_count<<<blocks_for((uint64_t)nb + 1, 256), 256, 0, st>>>(bstart, bend, nullptr, nb, T, np);
  TC_LAUNCHED(ctx);
  TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, np, offA, (int)(nb + 1), st));
  ctx->launches += 2;
  if (ctx->prof) TC_CUDA(ctx, cudaEventRecord(ctx->ev[0], st));
  k_accum_aff<<<blocks_for(max_items, 128), 128, 0, st>>>(svals, d_bases, bstart, bend, offA, nb, T, itemsA);
  TC_LAUNCHED(ctx);
  if (ctx->prof) {
    TC_CUDA(ctx, cudaEventRecord(ctx->ev[1], st));
    TC_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    TC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
    auto& s = ctx->stats["msm.accumulate"];
    s.ms += ms;
    s.launches += 1;
    s.units += (double)E;
  }
  uint64_t items_bound = max_items;
  for (int lv = 1; lv < levels; lv++) {
    k_piece_count<<<blocks_for((uint64_t)nb + 1, 256), 256, 0, st>>>(nullptr, nullptr, offA, nb, T1, np);
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, np, offB, (int)(nb + 1), st));
    ctx->launches += 2;
    uint64_t bound = (items_bound + T1 - 1) / T1 + nb;
    k_accum_xyzz<<<blocks_for(bound, 128), 128, 0, st>>>(itemsA, offA, offB, nb, T1, itemsB);
    TC_LAUNCHED(ctx);
    items_bound = bound;
    std::swap(offA, offB);
    std::swap(itemsA, itemsB);
  }
  k_gather_buckets<<<blocks_for(nb, 256), 256, 0, st>>>(itemsA, offA, nb, buckets);
  TC_LAUNCHED(ctx);

  // 6-7. bucket reduction, window sums, Horner, affine
  const uint32_t nw_total = (uint32_t)L * nwin;
  // segment length: enough threads to cover the GPU, short running-sum chains
  uint32_t LS = 32u;
  while (LS > 2u && (uint64_t)nw_total * B / LS < (uint64_t)ctx->num_sms * 256u) LS >>= 1;
  LS = std::min<uint32_t>(B, LS);
  const uint32_t nseg = B / LS;
  Xyzz *segs, *wsum;
  TC_TRY(scratch_t(ctx, "msm.segs", (uint64_t)nw_total * nseg, &segs));
  TC_TRY(scratch_t(ctx, "msm.wsum", nw_total, &wsum));
  k_bucket_reduce<<<blocks_for((uint64_t)nw_total * nseg, 128), 128, 0, st>>>(buckets, B, nw_total, LS, segs);
  TC_LAUNCHED(ctx);
  k_window_sum<<<nw_total, 128, 0, st>>>(segs, nseg, wsum);
  TC_LAUNCHED(ctx);
  k_final<<<blocks_for(L, 32), 32, 0, st>>>(wsum, (uint32_t)L, nwin, (uint32_t)c, d_out);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

int msm_device(tc_ctx* ctx, ScalarKind kind, const void* d_scalars, const Aff* d_bases, uint64_t n, Aff* d_out) {
  if (kind != SCALAR_FP_CANON) return fail(ctx, TC_ERR_ARGUMENT, "msm: scalar kind");
  const void* ptrs[1] = {d_scalars};
  return msm_batch_device(ctx, TC_DTYPE_FP_LIMBS, 0, ptrs, 1, d_bases, n, d_out);
}

}  // namespace tcrt
