// K3: Pippenger multi-scalar multiplication  C = sum_k a_k * G_k  over the curve of
// backend.py:102-108.  The reference composes this as a fold of `exp` (double-and-add,
// backend.py:202-217) and `mul` (affine add, backend.py:185-200) — 1.5 ms per term on a
// CPU core; SPEC.md:315 designates it the single performance hot-spot.
//
// Pipeline (all on the context stream, no host synchronisation):
//   1. k_maxbits      — bit length of the largest centred scalar magnitude (|a| or p-a)
//   2. k_digits       — signed c-bit window digits; key = window*B + |digit|-1, value =
//                       point index | sign<<31; zero digits get a sentinel key
//   3. radix sort     — (key, value) pairs by bucket (CUB onesweep over the used key bits)
//   4. k_bounds       — [start, end) of every bucket in the sorted order
//   5. levels         — load-balanced segmented reduction: every bucket is cut into pieces
//                       of <= T entries, one thread per piece sums its entries (XYZZ
//                       accumulator, mixed affine adds at level 0), piece sums become the
//                       entries of the next level until each bucket is a single point
//   6. k_bucket_reduce— per (window, segment of buckets) running sums: sum_b b * B_b
//   7. k_window_sum / k_final — add segments per window, Horner over windows with c
//                       doublings, one inversion to canonical affine
// Because affine points are canonical and the group is abelian, any window size,
// bucket order or coordinate system reproduces the reference's bytes exactly.
#include <cub/cub.cuh>

#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr uint32_t SIGN_BIT = 0x80000000u;

// centred magnitude of a canonical F_p element: a <= (p-1)/2 -> a, else p - a (negated)
__device__ __forceinline__ void centre_fp(const Fe& a, Fe& mag, bool& neg) {
  // (p-1)/2 = 2^160 + 2^23 -> limbs [0x00800000, 0, 0, 0, 0, 1]
  bool big = (a.v[5] > 1u) ||
             (a.v[5] == 1u && ((a.v[4] | a.v[3] | a.v[2] | a.v[1]) != 0u || a.v[0] > 0x00800000u));
  if (big) {
    Fe pm{{FpParams::M0, 0, 0, 0, 0, FpParams::M5}};
    uint64_t t = (uint64_t)pm.v[0] - a.v[0];
    mag.v[0] = (uint32_t)t;
    uint32_t br = (uint32_t)(t >> 63);
#pragma unroll
    for (int i = 1; i < 6; i++) {
      t = (uint64_t)pm.v[i] - a.v[i] - br;
      mag.v[i] = (uint32_t)t;
      br = (uint32_t)(t >> 63);
    }
    neg = true;
  } else {
    mag = a;
    neg = false;
  }
}

__device__ __forceinline__ uint32_t bitlen6(const Fe& a) {
#pragma unroll
  for (int i = 5; i >= 0; i--)
    if (a.v[i]) return 32u * i + 32u - __clz(a.v[i]);
  return 0u;
}

template <int KIND>
__device__ __forceinline__ void load_scalar(const void* s, uint64_t i, Fe& mag, bool& neg) {
  if (KIND == tcrt::SCALAR_FP_CANON) {
    const Fe a = ((const Fe*)s)[i];
    centre_fp(a, mag, neg);
  } else {
    int64_t v = ((const int64_t*)s)[i];
    neg = v < 0;
    uint64_t u = neg ? (uint64_t)(-(v + 1)) + 1u : (uint64_t)v;
    mag = Fe{{(uint32_t)u, (uint32_t)(u >> 32), 0, 0, 0, 0}};
  }
}

template <int KIND>
__global__ void k_maxbits(const void* s, uint64_t n, uint32_t* out) {
  uint32_t mx = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Fe mag;
    bool neg;
    load_scalar<KIND>(s, i, mag, neg);
    mx = max(mx, bitlen6(mag));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// window w of the magnitude: bits [c*w, c*w + c)
__device__ __forceinline__ uint32_t window_bits(const Fe& m, int lo, int c) {
  int limb = lo >> 5, sh = lo & 31;
  uint64_t w = m.v[limb];
  if (limb + 1 < 6) w |= (uint64_t)m.v[limb + 1] << 32;
  return (uint32_t)(w >> sh) & ((1u << c) - 1u);
}

template <int KIND>
__global__ void k_digits(const void* s, uint64_t n, int c, int nwin, uint32_t* keys,
                         uint32_t* vals, uint32_t* nnz) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t cnt = 0;
  if (i < n) {
    Fe mag;
    bool neg;
    load_scalar<KIND>(s, i, mag, neg);
    const uint32_t half = 1u << (c - 1), full = 1u << c, B = half;
    const uint32_t sentinel = (uint32_t)nwin * B;
    uint32_t carry = 0;
    for (int w = 0; w < nwin; w++) {
      uint32_t d = window_bits(mag, w * c, c) + carry;
      bool dneg = false;
      if (d > half) {   // d - 2^c, carry into the next window
        d = full - d;
        dneg = true;
        carry = 1;
      } else {
        carry = 0;
      }
      uint64_t o = (uint64_t)w * n + i;
      if (d == 0) {
        keys[o] = sentinel;
        vals[o] = 0;
      } else {
        keys[o] = (uint32_t)w * B + d - 1u;
        vals[o] = (uint32_t)i | ((neg != dneg) ? SIGN_BIT : 0u);
        cnt++;
      }
    }
  }
  // warp-aggregated count of non-zero digits
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nnz, cnt);
}

__global__ void k_bounds(const uint32_t* keys, const uint32_t* nnz, uint32_t* bstart,
                         uint32_t* bend) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t E = *nnz;
  if (j >= E) return;
  uint32_t k = keys[j];
  if (j == 0 || keys[j - 1] != k) bstart[k] = (uint32_t)j;
  if (j + 1 == E || keys[j + 1] != k) bend[k] = (uint32_t)j + 1u;
}

// pieces per bucket for this level; np has nb+1 entries (last = 0)
__global__ void k_piece_count(const uint32_t* bstart, const uint32_t* bend, uint32_t nb,
                              uint32_t T, uint32_t* np) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nb) return;
  if (k == nb) {
    np[k] = 0;
    return;
  }
  uint32_t sz = bend[k] - bstart[k];
  np[k] = (sz + T - 1) / T;
}

__device__ __forceinline__ uint32_t find_bucket(const uint32_t* off, uint32_t nb, uint32_t p) {
  // largest k with off[k] <= p  (off is non-decreasing, off[nb] = total)
  uint32_t lo = 0, hi = nb;   // invariant: off[lo] <= p < off[hi]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= p)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// level 0: entries are (sign | point index) into the affine bases
__global__ void __launch_bounds__(128) k_accum_aff(const uint32_t* vals, const Aff* bases,
                                                   const uint32_t* bstart, const uint32_t* bend,
                                                   const uint32_t* off, uint32_t nb, uint32_t T,
                                                   Xyzz* out) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t total = off[nb];
  if (p >= total) return;
  uint32_t k = find_bucket(off, nb, p);
  uint32_t piece = p - off[k];
  uint32_t a = bstart[k] + piece * T;
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

// level >= 1: entries are XYZZ partial sums; bucket k's entries are [off_prev[k], off_prev[k+1])
__global__ void __launch_bounds__(128) k_accum_xyzz(const Xyzz* in, const uint32_t* prev_off,
                                                    const uint32_t* off, uint32_t nb, uint32_t T,
                                                    Xyzz* out) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t total = off[nb];
  if (p >= total) return;
  uint32_t k = find_bucket(off, nb, p);
  uint32_t piece = p - off[k];
  uint32_t a = prev_off[k] + piece * T;
  uint32_t b = min(a + T, prev_off[k + 1]);
  Xyzz acc = in[a];
  for (uint32_t j = a + 1; j < b; j++) xyzz_add(acc, in[j]);
  out[p] = acc;
}

__global__ void k_piece_count_off(const uint32_t* prev_off, uint32_t nb, uint32_t T,
                                  uint32_t* np) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nb) return;
  if (k == nb) {
    np[k] = 0;
    return;
  }
  uint32_t sz = prev_off[k + 1] - prev_off[k];
  np[k] = (sz + T - 1) / T;
}

// buckets[k] = the single remaining piece (or infinity)
__global__ void k_gather_buckets(const Xyzz* in, const uint32_t* off, uint32_t nb, Xyzz* buckets) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  buckets[k] = (off[k + 1] > off[k]) ? in[off[k]] : xyzz_inf();
}

// per (window, segment): sum_{b in seg} (b+1) * B_b  via running sums from the top
__global__ void __launch_bounds__(128) k_bucket_reduce(const Xyzz* buckets, uint32_t B,
                                                       uint32_t nwin, uint32_t LS, Xyzz* segs) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t nseg = B / LS;
  if (t >= nwin * nseg) return;
  uint32_t w = t / nseg, s = t % nseg;
  uint32_t lo = s * LS;
  const Xyzz* bw = buckets + (uint64_t)w * B;
  Xyzz run = xyzz_inf(), sum = xyzz_inf();
  for (int b = (int)(lo + LS) - 1; b >= (int)lo; b--) {
    xyzz_add(run, bw[b]);
    xyzz_add(sum, run);
  }
  // sum = sum_b (b - lo + 1) B_b ; add lo * run to get sum_b (b + 1) B_b
  if (lo) {
    Xyzz extra = xyzz_mul_small(run, lo);
    xyzz_add(sum, extra);
  }
  segs[t] = sum;
}

// tree-sum nseg segments of every window (one block per window)
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

// Horner over windows: sum_w 2^{c w} S_w, then canonical affine
__global__ void k_final(const Xyzz* wsum, uint32_t nwin, uint32_t c, Aff* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Xyzz acc = wsum[nwin - 1];
  for (int w = (int)nwin - 2; w >= 0; w--) {
    for (uint32_t i = 0; i < c; i++) acc = xyzz_dbl(acc);
    xyzz_add(acc, wsum[w]);
  }
  Aff r = xyzz_to_aff(acc);
  if (!aff_is_inf(r)) {
    r.x = Fq::canon(r.x);
    r.y = Fq::canon(r.y);
  }
  *out = r;
}

uint32_t bitlen_u32(uint32_t v) { return v ? 32u - __builtin_clz(v) : 0u; }

// cost model: mixed adds for digits + ~2.5 equivalent adds per bucket in the reduction
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

}  // namespace

namespace tcrt {

int msm_device(tc_ctx* ctx, ScalarKind kind, const void* d_scalars, const Aff* d_bases,
               uint64_t n, Aff* d_out) {
  cudaStream_t st = ctx->stream;
  if (n == 0) {
    Aff inf = aff_inf();
    TC_CUDA(ctx, cudaMemcpyAsync(d_out, &inf, sizeof(Aff), cudaMemcpyHostToDevice, st));
    TC_CUDA(ctx, cudaStreamSynchronize(st));
    return TC_OK;
  }
  if (n >= (1ull << 31)) return fail(ctx, TC_ERR_VALUE, "msm: too many points (%llu)", (unsigned long long)n);

  // 1. scalar magnitude bits (one small readback chooses the window layout)
  uint32_t* d_small;
  TC_TRY(scratch_t(ctx, "msm.small", 8, &d_small));
  TC_CUDA(ctx, cudaMemsetAsync(d_small, 0, 8 * sizeof(uint32_t), st));
  unsigned gb = std::min<unsigned>(blocks_for(n, 256), (unsigned)ctx->num_sms * 8);
  if (kind == SCALAR_FP_CANON)
    k_maxbits<SCALAR_FP_CANON><<<gb, 256, 0, st>>>(d_scalars, n, d_small);
  else
    k_maxbits<SCALAR_I64><<<gb, 256, 0, st>>>(d_scalars, n, d_small);
  TC_LAUNCHED(ctx);
  uint32_t nbits = 0;
  TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags, d_small, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  nbits = ctx->h_flags[0];
  if (nbits == 0) {   // every scalar is zero: identity
    Aff inf = aff_inf();
    TC_CUDA(ctx, cudaMemcpyAsync(d_out, &inf, sizeof(Aff), cudaMemcpyHostToDevice, st));
    TC_CUDA(ctx, cudaStreamSynchronize(st));
    return TC_OK;
  }

  const int c = choose_c(n, nbits);
  const uint32_t nwin = (nbits + 1 + c - 1) / c;
  const uint32_t B = 1u << (c - 1);
  const uint32_t nb = nwin * B;
  const uint64_t E = n * nwin;
  const int end_bit = (int)bitlen_u32(nb);   // sentinel nb fits

  uint32_t *keys, *vals, *keys2, *vals2, *bstart, *bend;
  TC_TRY(scratch_t(ctx, "msm.keys", E, &keys));
  TC_TRY(scratch_t(ctx, "msm.vals", E, &vals));
  TC_TRY(scratch_t(ctx, "msm.keys2", E, &keys2));
  TC_TRY(scratch_t(ctx, "msm.vals2", E, &vals2));
  TC_TRY(scratch_t(ctx, "msm.bstart", nb + 1, &bstart));
  TC_TRY(scratch_t(ctx, "msm.bend", nb + 1, &bend));

  // 2. digits
  uint32_t* d_nnz = d_small + 1;
  if (kind == SCALAR_FP_CANON)
    k_digits<SCALAR_FP_CANON><<<blocks_for(n, 256), 256, 0, st>>>(d_scalars, n, c, nwin, keys, vals, d_nnz);
  else
    k_digits<SCALAR_I64><<<blocks_for(n, 256), 256, 0, st>>>(d_scalars, n, c, nwin, keys, vals, d_nnz);
  TC_LAUNCHED(ctx);

  // 3. sort by bucket
  size_t tmp_bytes = 0;
  cub::DoubleBuffer<uint32_t> dk(keys, keys2), dv(vals, vals2);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int)E, 0, end_bit, st);
  void* d_tmp;
  TC_TRY(scratch(ctx, "msm.cubtmp", tmp_bytes, &d_tmp));
  TC_CUDA(ctx, cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, dk, dv, (int)E, 0, end_bit, st));
  ctx->launches += 4;
  const uint32_t* skeys = dk.Current();
  const uint32_t* svals = dv.Current();

  // 4. bucket bounds
  TC_CUDA(ctx, cudaMemsetAsync(bstart, 0, (nb + 1) * sizeof(uint32_t), st));
  TC_CUDA(ctx, cudaMemsetAsync(bend, 0, (nb + 1) * sizeof(uint32_t), st));
  k_bounds<<<blocks_for(E, 256), 256, 0, st>>>(skeys, d_nnz, bstart, bend);
  TC_LAUNCHED(ctx);

  // 5. levels of load-balanced segmented reduction
  const uint32_t T = (E >= (1u << 20)) ? 32u : (E >= (1u << 14) ? 16u : 8u);
  int levels = 1;
  for (uint64_t cap = T; cap < n; cap *= T) levels++;   // a bucket holds <= n entries
  uint64_t max_items = (E + T - 1) / T + nb;
  uint32_t *offA, *offB;
  Xyzz *itemsA, *itemsB, *buckets;
  TC_TRY(scratch_t(ctx, "msm.offA", nb + 1, &offA));
  TC_TRY(scratch_t(ctx, "msm.offB", nb + 1, &offB));
  TC_TRY(scratch_t(ctx, "msm.itemsA", max_items, &itemsA));
  TC_TRY(scratch_t(ctx, "msm.itemsB", max_items, &itemsB));
  TC_TRY(scratch_t(ctx, "msm.buckets", nb, &buckets));
  uint32_t* np;
  TC_TRY(scratch_t(ctx, "msm.np", nb + 1, &np));
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, np, offA, (int)(nb + 1), st);
  void* d_scan;
  TC_TRY(scratch(ctx, "msm.scantmp", scan_bytes, &d_scan));

  k_piece_count<<<blocks_for(nb + 1, 256), 256, 0, st>>>(bstart, bend, nb, T, np);
  TC_LAUNCHED(ctx);
  TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, np, offA, (int)(nb + 1), st));
  ctx->launches += 2;
  if (ctx->prof) TC_CUDA(ctx, cudaEventRecord(ctx->ev[0], st));
  k_accum_aff<<<blocks_for(max_items, 128), 128, 0, st>>>(svals, d_bases, bstart, bend, offA, nb, T, itemsA);
  TC_LAUNCHED(ctx);
  if (ctx->prof) {
    // one extra sync per MSM while profiling: read the kernel time and its entry count
    TC_CUDA(ctx, cudaEventRecord(ctx->ev[1], st));
    TC_CUDA(ctx, cudaMemcpyAsync(ctx->h_flags + 4, d_nnz, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    TC_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    TC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
    auto& s = ctx->stats["msm.accumulate"];
    s.ms += ms;
    s.launches += 1;
    s.units += (double)ctx->h_flags[4];
  }
  uint64_t items_bound = max_items;
  for (int l = 1; l < levels; l++) {
    k_piece_count_off<<<blocks_for(nb + 1, 256), 256, 0, st>>>(offA, nb, T, np);
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, np, offB, (int)(nb + 1), st));
    ctx->launches += 2;
    uint64_t bound = (items_bound + T - 1) / T + nb;
    k_accum_xyzz<<<blocks_for(bound, 128), 128, 0, st>>>(itemsA, offA, offB, nb, T, itemsB);
    TC_LAUNCHED(ctx);
    items_bound = bound;
    std::swap(offA, offB);
    std::swap(itemsA, itemsB);
  }
  k_gather_buckets<<<blocks_for(nb, 256), 256, 0, st>>>(itemsA, offA, nb, buckets);
  TC_LAUNCHED(ctx);

  // 6. bucket reduction
  uint32_t LS = std::min<uint32_t>(B, 32u);
  uint32_t nseg = B / LS;
  Xyzz *segs, *wsum;
  TC_TRY(scratch_t(ctx, "msm.segs", (uint64_t)nwin * nseg, &segs));
  TC_TRY(scratch_t(ctx, "msm.wsum", nwin, &wsum));
  k_bucket_reduce<<<blocks_for((uint64_t)nwin * nseg, 128), 128, 0, st>>>(buckets, B, nwin, LS, segs);
  TC_LAUNCHED(ctx);
  k_window_sum<<<nwin, 128, 0, st>>>(segs, nseg, wsum);
  TC_LAUNCHED(ctx);
  k_final<<<1, 32, 0, st>>>(wsum, nwin, (uint32_t)c, d_out);
  TC_LAUNCHED(ctx);
  return TC_OK;
}

}  // namespace tcrt
