// K3: batched Pippenger multi-scalar multiplication
//     out[l] = sum_k a_{l,k} * G_k      l = 0..L-1, all L MSMs over the SAME bases G.
//
// The reference composes one MSM as a fold of `exp` (double-and-add, backend.py:202-217)
// and `mul` (affine add, backend.py:185-200) — 1.5 ms per term on a CPU core
// designates it the single performance hot-spot.  The prover runs many MSMs against one
// SRS (32 layers per forward, m quotients per opening, 8 nodes per Terkle level), so the
// whole batch goes through ONE pipeline:
//   1. k_scan_bits(_v) — exact maximum bit length + quantisation errors of the scalars
//                       (canonical F_p limbs, or raw floats quantised on the fly: K1 is
//                       fused into the MSM), bit-length histogram on a sample
//   2. window plan    — (host) mode 3: fp16 / bf16 over the SRS's exponent table (one
//                       entry per element, one window of 2^MB - 1 buckets), mode 1
//                       float-exponent groups when the table does not fit, mode 2 fixed-base
//                       digit windows over a window table (opening quotients), else signed
//                       windows from a DP over the histogram (#digits + kappa * #buckets)
//   3. counting sort  — count entries per bucket, exclusive scan, scatter (table index |
//                       sign << 31) into bucket slices: block-private shared-memory counters
//                       (k_fpb_pass, k_fpb_scatter_sorted) for modes 3 / 1, RED atomics
//                       into counter copies otherwise (k_digits_fp / k_digits_v /
//                       k_count_digits)
//   4. levels         — load-balanced segmented reduction: buckets are cut into pieces of
//                       <= T entries (one thread per piece, extended twisted Edwards
//                       accumulator, complete 8M mixed adds with lazy reduction, ec.cuh);
//                       single-piece buckets are final at once, multi-piece buckets (the
//                       heavy tail) feed further levels of T1-way reduction
//   5. weighting      — sum_j (mlo + j) B_j per window: recursive segmentation
//                       (k_wsum_level / k_wsum_final), or one block per window for small
//                       batches (k_wsum_block); k_final / k_final_sum combine the windows
//                       and convert to canonical Montgomery affine
// Affine outputs are canonical and the group is abelian, so any window layout, bucket
// order or coordinate system reproduces the reference's bytes exactly.  The bases are the
// SRS points mapped to the twisted Edwards model of the curve (tc_srs::ed_*, built once per
// SRS); results are mapped back to Montgomery affine by k_final.
#include <cub/cub.cuh>

#include "quant.cuh"
#include "tc_internal.cuh"

using namespace tc;

namespace {

constexpr uint32_t SIGN_BIT = 0x80000000u;
constexpr int DT_LIMBS = 0;   // template code for canonical F_p scalars
constexpr int MAXW = 48;      // windows per scalar (>= ceil(163 / 4))
constexpr int NHIST = 168;    // bit-length histogram bins
constexpr uint32_t HIST_SAMPLE = 8;   // histogram taken on every 8th element (k_scan_bits)

// mode 0: signed-digit windows (bits [off, off + width) of the magnitude; bucket j of
//         window w holds digit j + 1).
// mode 1: float-exponent groups for fp16 / bf16 inputs.  A quantised fp value is
//         |q| = m 2^k with at most MB = 11 (fp16) / 8 (bf16) significant bits, so group k
//         holds m = |q| >> k: k = 0 takes |q| < 2^MB (m in [1, 2^MB)), k >= 1 takes
//         bitlen(|q|) = MB + k (m in [2^(MB-1), 2^MB)).  ONE bucket entry per element (no
//         carry window) and K * 2^(MB-1) buckets per MSM, none of them empty by construction
//         of fp16 (a signed-window plan of the same data leaves ~85% of its 2^17 low-window
//         buckets empty: fp16 has 1024 mantissas per octave).  Bucket j of group w holds
//         weight mlo[w] + j; the groups are combined with weight 2^off[w] (off[w] = w).
// mode 3: mode 1 with the exponent in the base: entry (i, g) reads 2^g G_i from the SRS's
//         exponent table (srs_exp_table, level pitch tpitch), so every group shares ONE
//         window of 2^MB - 1 buckets of weight m.
// mode 2: fixed-base windows (openings: canonical F_p scalars against an SRS range with a
//         window table, srs_window_table).  The scalar's ndig signed digits of cdig bits
//         index the table copies 2^(cdig w) B, so all digits share ONE window of buckets:
//         nwin = 1, no Horner doublings, and the bucket reduction is ndig x smaller.
struct WinPlan {
  int nwin;
  int mode;                  // 0 signed windows, 1 float-exponent groups, 2 fixed-base windows
  int mbits;                 // mode 1: significant bits of the input format
  int ndig, cdig;            // mode 2: digit windows and their width
  uint32_t nbm;              // buckets per MSM
  uint8_t off[MAXW];         // window w: first bit (mode 0) / exponent k (mode 1)
  uint8_t width[MAXW];       // mode 0: c_w
  uint32_t mlo[MAXW];        // weight of the window's first bucket (mode 0: 1)
  uint32_t base[MAXW + 1];   // first bucket of window w inside one MSM
  uint32_t tpitch;           // mode 3: points per exponent-table level (entry = g tpitch + i)
  const uint32_t* ktab = nullptr;   // mode 3, fp16: per |bit pattern| key | g << 16 (0xFFFFFFFF: no entry)
};

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

// out[0] = quantisation flags, out[1..NHIST] = bit-length histogram
template <int DT>
__global__ void k_scan_bits(const void* const* ptrs, uint64_t n, int scale_bits, uint32_t* out) {
  __shared__ uint32_t hist[NHIST];
  for (int i = threadIdx.x; i < NHIST; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const void* p = ptrs[blockIdx.y];
  uint32_t f = 0, bmax = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t bl;
    if (DT >= 1 && DT <= 3) {
      // fp16 / bf16 / fp32: |q| < 2^145 never overflows the field half-range, so only the
      // bit length is needed: from the exponent, an upper bound that is exact except that
      // rounding up may add one bit (the window plan only needs an upper bound)
      Decoded d = decode_float<DT>(p, i);
      if (d.nonfinite) f |= QF_NONFINITE;
      const int sh = d.exp2 + scale_bits;
      const int mb = d.mant ? 64 - __clzll((long long)d.mant) : 0;
      const int b = d.nonfinite ? 0 : (sh >= 0 ? mb + sh : mb + sh + 1);
      bl = (uint32_t)(b > 0 ? (b < NHIST - 1 ? b : NHIST - 1) : 0);
    } else {
      Fe mag;
      bool neg;
      load_scalar<DT>(p, i, scale_bits, mag, neg, f);
      bl = bitlen6(mag);
    }
    // the histogram only steers the window plan (any plan is exact), so it is taken on
    // 1/HIST_SAMPLE of the elements: contended shared atomics were the kernel's cost.  The
    // maximum bit length (which the plan must cover) and the error flags see every element.
    if ((i & (HIST_SAMPLE - 1)) == 0) atomicAdd(&hist[bl], 1u);
    bmax = max(bmax, bl);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    f |= __shfl_xor_sync(0xffffffffu, f, o);
    bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  }
  if ((threadIdx.x & 31) == 0 && f) atomicOr(out, f);
  if ((threadIdx.x & 31) == 0 && bmax) atomicMax(out + NHIST + 1, bmax);
  __syncthreads();
  for (int i = threadIdx.x; i < NHIST; i += blockDim.x)
    if (hist[i]) atomicAdd(out + 1 + i, hist[i]);
}

// ---- counting-sort layout (default): digits -> bucket counts -> scan -> scatter -------
// The radix sort of (key, value) pairs costs 3 onesweep passes over all entries plus a
// bounds pass.  Instead, the digits are produced twice from the (2 B/elem) inputs:
//   k_count_digits   — per-bucket entry counts (global RED atomics; windows with few
//                      buckets, where one bucket takes thousands of hits, are aggregated
//                      per warp first with __match_any_sync)
//   exclusive scan   — bucket starts (bucket k = [bstart[k], bstart[k+1]))
//   k_scatter_digits — each entry claims a slot with an atomic on its bucket cursor and
//                      writes its value (point index | sign); the order inside a bucket is
//                      arbitrary, which EC addition does not see
constexpr uint32_t HOT_BUCKETS = 1024;   // windows with <= this many buckets are warp-aggregated

template <bool SCATTER>
__device__ __forceinline__ void bucket_hit(uint32_t key, bool hot, bool active, uint32_t val, uint32_t* cnt,
                                           uint32_t* vals) {
  // hot is warp-uniform (same window for every lane)
  if (hot) {
    const uint32_t act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const uint32_t peers = __match_any_sync(act, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) {
      if (SCATTER)
        base = atomicAdd(cnt + key, (uint32_t)__popc(peers));
      else
        atomicAdd(cnt + key, (uint32_t)__popc(peers));
    }
    if (SCATTER) {
      base = __shfl_sync(peers, base, leader);
      vals[base + __popc(peers & ((1u << lane) - 1u))] = val;
    }
  } else if (active) {
    if (SCATTER)
      vals[atomicAdd(cnt + key, 1u)] = val;
    else
      atomicAdd(cnt + key, 1u);
  }
}

template <int DT, bool SCATTER>
__global__ void __launch_bounds__(256) k_count_digits(const void* const* ptrs, uint64_t n, int scale_bits, WinPlan P,
                                                      uint32_t* cnt, uint32_t* vals) {
  const uint32_t l = blockIdx.y;
  const void* p = ptrs[l];
  const uint32_t key0 = l * P.nbm;
  uint32_t f = 0;
  // whole warps iterate together (the hot-window aggregation needs converged lanes)
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nr = (n + 31) & ~31ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nr; i += stride) {
    const bool in = i < n;
    Fe mag;
    bool neg = false;
    if (in) load_scalar<DT>(p, i, scale_bits, mag, neg, f);
    else mag = Fe{{0, 0, 0, 0, 0, 0}};
    uint32_t carry = 0;
    if (P.mode == 2) {   // fixed-base digit windows, one shared set of buckets
      const int c = P.cdig;
      const uint32_t half = 1u << (c - 1), full = 1u << c;
      for (int w = 0; w < P.ndig; w++) {
        uint32_t d = window_bits(mag, w * c, c) + carry;
        bool dn = false;
        if (d > half) {
          d = full - d, dn = true, carry = 1;
        } else {
          carry = 0;
        }
        bucket_hit<SCATTER>(key0 + d - 1u, false, d != 0,
                            (uint32_t)((uint64_t)w * n + i) | ((neg != dn) ? SIGN_BIT : 0u), cnt, vals);
      }
      continue;
    }
    for (int w = 0; w < P.nwin; w++) {
      const int c = P.width[w];
      const uint32_t half = 1u << (c - 1), full = 1u << c;
      uint32_t d = window_bits(mag, P.off[w], c) + carry;
      bool dn = false;
      if (d > half) {
        d = full - d;
        dn = true;
        carry = 1;
      } else {
        carry = 0;
      }
      const uint32_t key = key0 + P.base[w] + d - 1u;
      bucket_hit<SCATTER>(key, half <= HOT_BUCKETS, d != 0, (uint32_t)i | ((neg != dn) ? SIGN_BIT : 0u), cnt, vals);
    }
  }
}

// ---- fast path: float inputs whose quantised magnitudes fit 63 bits (fp16 at the
// reference's scale 2^16 always does).  One block = 2048 consecutive elements of one MSM,
// 8 per thread from one 16-byte load (two for fp32); magnitudes and digits in uint64.
// Few-bucket ("hot") windows are counted in shared memory and claimed from the global
// cursors with ONE atomic per (block, bucket); the blocks are scheduled MSM after MSM,
// so the scattered 4-byte writes of the MSMs in flight stay in L2 until their sectors
// are complete.
constexpr int V_EPT = 8;
constexpr int HOT_MAXW = 4;        // hot windows per plan handled by the fast path
constexpr uint32_t HOT_MAXB = 2048;

struct HotPlan {
  int nhot;
  uint8_t win[HOT_MAXW];       // hot window ids
  uint16_t hbase[HOT_MAXW];    // first shared counter of each hot window
  uint32_t nhotb;              // shared counters in use
  int8_t slot[MAXW];           // window -> hot slot or -1
};

template <int DT>
__device__ __forceinline__ void load_raw8(const void* p, uint64_t i0, uint64_t n, uint32_t raw[V_EPT]) {
  if (i0 + V_EPT <= n) {
    if (DT == 1 || DT == 2) {
      const uint4 a = *(const uint4*)((const uint16_t*)p + i0);
      const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int k = 0; k < 4; k++) raw[2 * k] = w[k] & 0xffffu, raw[2 * k + 1] = w[k] >> 16;
    } else {
      const uint4 a = *(const uint4*)((const uint32_t*)p + i0), b = *((const uint4*)((const uint32_t*)p + i0) + 1);
      raw[0] = a.x, raw[1] = a.y, raw[2] = a.z, raw[3] = a.w, raw[4] = b.x, raw[5] = b.y, raw[6] = b.z, raw[7] = b.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < V_EPT; k++) {
      const uint64_t i = i0 + k;
      raw[k] = i < n ? ((DT == 1 || DT == 2) ? (uint32_t)((const uint16_t*)p)[i] : ((const uint32_t*)p)[i]) : 0u;
    }
  }
}

// |RNE(v * 2^scale_bits)| < 2^63 and its sign from raw fp16 / bf16 / fp32 bits (non-finite
// values were rejected by k_scan_bits before this runs; they map to 0 here)
template <int DT>
__device__ __forceinline__ uint64_t quant64(uint32_t b, int scale_bits, bool& neg) {
  uint32_t e, m;
  int ex;
  if (DT == 1) {
    e = (b >> 10) & 0x1f, m = b & 0x3ff, neg = b >> 15;
    if (e == 0x1f) return 0;
    m = e ? (m | 0x400u) : m, ex = (e ? (int)e : 1) - 25;
  } else if (DT == 2) {
    e = (b >> 7) & 0xff, m = b & 0x7f, neg = b >> 15;
    if (e == 0xff) return 0;
    m = e ? (m | 0x80u) : m, ex = (e ? (int)e : 1) - 134;
  } else {
    e = (b >> 23) & 0xff, m = b & 0x7fffffu, neg = b >> 31;
    if (e == 0xff) return 0;
    m = e ? (m | 0x800000u) : m, ex = (e ? (int)e : 1) - 150;
  }
  const int sh = ex + scale_bits;
  if (sh >= 0) return (uint64_t)m << sh;
  const int s = -sh;
  if (s > 31) return 0;   // m < 2^24 -> value < 1/2
  const uint32_t iq = m >> s, rem = m & ((1u << s) - 1u), half = 1u << (s - 1);
  return (uint64_t)(iq + ((rem > half || (rem == half && (iq & 1u))) ? 1u : 0u));
}

// nc: counter copies per bucket (mode 1): block b counts into copy b % nc, so the ~100-300
// hits a popular fp16 bucket takes per MSM are spread over nc addresses (same-address L2
// atomics serialise); bucket k's copies are adjacent, so one scan gives every copy its
// own slice of the bucket and the bucket stays contiguous
template <int DT, bool SCATTER>
__global__ void __launch_bounds__(256) k_digits_v(const void* const* ptrs, uint64_t n, int scale_bits, WinPlan P,
                                                  HotPlan H, uint32_t* cnt, uint32_t* vals, uint32_t nc) {
  __shared__ uint32_t hcnt[HOT_MAXB];
  const uint32_t l = blockIdx.y;
  const void* p = ptrs[l];
  const uint32_t key0 = l * P.nbm;
  for (uint32_t h = threadIdx.x; h < H.nhotb; h += blockDim.x) hcnt[h] = 0;
  __syncthreads();
  const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * V_EPT;
  uint32_t raw[V_EPT];
  load_raw8<DT>(p, i0, n, raw);
  uint32_t hd[V_EPT][HOT_MAXW];   // hot digits: counter index | local rank << 12 | sign << 31
#pragma unroll
  for (int k = 0; k < V_EPT; k++) {
#pragma unroll
    for (int j = 0; j < HOT_MAXW; j++) hd[k][j] = 0xffffffffu;
    bool neg;
    const uint64_t mag = (i0 + k < n) ? quant64<DT>(raw[k], scale_bits, neg) : 0ull;
    if (P.mode == 1) {   // float-exponent group: one entry per non-zero element
      if (!mag) continue;
      const int bl = 64 - __clzll((long long)mag);
      const int g = bl > P.mbits ? bl - P.mbits : 0;
      const uint32_t key = key0 + P.base[g] + (uint32_t)(mag >> g) - P.mlo[g];
      const uint32_t val = (uint32_t)(i0 + k) | (neg ? SIGN_BIT : 0u);
      uint32_t* c = cnt + (uint64_t)key * nc + blockIdx.x % nc;
      if (SCATTER)
        vals[atomicAdd(c, 1u)] = val;
      else
        atomicAdd(c, 1u);
      continue;
    }
    uint32_t carry = 0;
    for (int w = 0; w < P.nwin; w++) {
      const int c = P.width[w];
      const uint32_t half = 1u << (c - 1), full = 1u << c;
      uint32_t d = (uint32_t)((mag >> P.off[w]) & (full - 1u)) + carry;
      bool dn = false;
      if (d > half) {
        d = full - d, dn = true, carry = 1;
      } else {
        carry = 0;
      }
      if (!d) continue;
      const int hs = H.slot[w];
      if (hs >= 0) {
        const uint32_t h = H.hbase[hs] + d - 1u;
        const uint32_t r = atomicAdd(&hcnt[h], 1u);
        hd[k][hs] = h | (r << 12) | ((neg != dn) ? SIGN_BIT : 0u);
      } else if (SCATTER) {
        vals[atomicAdd(cnt + key0 + P.base[w] + d - 1u, 1u)] = (uint32_t)(i0 + k) | ((neg != dn) ? SIGN_BIT : 0u);
      } else {
        atomicAdd(cnt + key0 + P.base[w] + d - 1u, 1u);
      }
    }
  }
  if (H.nhot == 0) return;
  __syncthreads();
  // one global atomic per used hot bucket of this block; hcnt becomes the claimed base
  for (int hs = 0; hs < H.nhot; hs++) {
    const int w = H.win[hs];
    const uint32_t nbw = 1u << (P.width[w] - 1);
    for (uint32_t j = threadIdx.x; j < nbw; j += blockDim.x) {
      const uint32_t h = H.hbase[hs] + j, c = hcnt[h];
      if (!c) continue;
      const uint32_t b = atomicAdd(cnt + key0 + P.base[w] + j, c);
      if (SCATTER) hcnt[h] = b;
    }
  }
  if (!SCATTER) return;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < V_EPT; k++)
#pragma unroll
    for (int j = 0; j < HOT_MAXW; j++) {
      const uint32_t v = hd[k][j];
      if (v != 0xffffffffu)
        vals[hcnt[v & 0xfffu] + ((v >> 12) & 0x7ffffu)] = (uint32_t)(i0 + k) | (v & SIGN_BIT);
    }
}

// k_scan_bits for fp16 / bf16 / fp32: 8 elements per thread from 16-byte loads
template <int DT>
__global__ void __launch_bounds__(256) k_scan_bits_v(const void* const* ptrs, uint64_t n, int scale_bits, uint32_t* out) {
  __shared__ uint32_t hist[NHIST];
  for (int i = threadIdx.x; i < NHIST; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const void* p = ptrs[blockIdx.y];
  uint32_t f = 0, bmax = 0;
  for (uint64_t i0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * V_EPT; i0 < n;
       i0 += (uint64_t)gridDim.x * blockDim.x * V_EPT) {
    uint32_t raw[V_EPT];
    load_raw8<DT>(p, i0, n, raw);
#pragma unroll
    for (int k = 0; k < V_EPT; k++) {
      if (i0 + k >= n) break;
      uint32_t e, m;
      int ex;
      bool nf;
      const uint32_t b = raw[k];
      if (DT == 1) {
        e = (b >> 10) & 0x1f, m = b & 0x3ff, nf = e == 0x1f;
        m = e ? (m | 0x400u) : m, ex = (e ? (int)e : 1) - 25;
      } else if (DT == 2) {
        e = (b >> 7) & 0xff, m = b & 0x7f, nf = e == 0xff;
        m = e ? (m | 0x80u) : m, ex = (e ? (int)e : 1) - 134;
      } else {
        e = (b >> 23) & 0xff, m = b & 0x7fffffu, nf = e == 0xff;
        m = e ? (m | 0x800000u) : m, ex = (e ? (int)e : 1) - 150;
      }
      if (nf) f |= QF_NONFINITE;
      const int sh = ex + scale_bits;
      const int mb = m ? 32 - __clz(m) : 0;
      const int bl0 = nf ? 0 : (sh >= 0 ? mb + sh : mb + sh + 1);
      const uint32_t bl = (uint32_t)(bl0 > 0 ? (bl0 < NHIST - 1 ? bl0 : NHIST - 1) : 0);
      if (k == 0 && ((i0 / V_EPT) & (HIST_SAMPLE / V_EPT > 1 ? HIST_SAMPLE / V_EPT - 1 : 0)) == 0) atomicAdd(&hist[bl], 1u);
      bmax = max(bmax, bl);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    f |= __shfl_xor_sync(0xffffffffu, f, o);
    bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  }
  if ((threadIdx.x & 31) == 0 && f) atomicOr(out, f);
  if ((threadIdx.x & 31) == 0 && bmax) atomicMax(out + NHIST + 1, bmax);
  __syncthreads();
  for (int i = threadIdx.x; i < NHIST; i += blockDim.x)
    if (hist[i]) atomicAdd(out + 1 + i, hist[i]);
}

// largest bucket (sets the number of reduction levels)
__global__ void k_max_bucket(const uint32_t* bstart, uint32_t nb, uint32_t* out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = k < nb ? bstart[k + 1] - bstart[k] : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// bucket starts from the per-copy exclusive scan: bstart[k] = S[k * nc], k = 0..nb
__global__ void k_copy_starts(const uint32_t* S, uint32_t nb, uint32_t nc, uint32_t* bstart) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k <= nb) bstart[k] = S[(uint64_t)k * nc];
}

// mode-1 (float-exponent) digit pass: one entry per element; the 8 slot claims of a
// thread are issued back to back before any of its stores (the atomics' latency overlaps)
template <int DT, bool SCATTER>
__global__ void __launch_bounds__(256) k_digits_fp(const void* const* ptrs, uint64_t n, int scale_bits, WinPlan P,
                                                   uint32_t* __restrict__ cnt, uint32_t* __restrict__ vals,
                                                   uint32_t nc) {
  const uint32_t l = blockIdx.y;
  const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * V_EPT;
  const uint32_t key0 = l * P.nbm, copy = blockIdx.x % nc;
  uint32_t raw[V_EPT], ctr[V_EPT], val[V_EPT];
  load_raw8<DT>(ptrs[l], i0, n, raw);
  uint32_t live = 0;
#pragma unroll
  for (int k = 0; k < V_EPT; k++) {
    bool neg;
    const uint64_t mag = (i0 + k < n) ? quant64<DT>(raw[k], scale_bits, neg) : 0ull;
    const int bl = mag ? 64 - __clzll((long long)mag) : 0;
    const int g = bl > P.mbits ? bl - P.mbits : 0;
    ctr[k] = (key0 + P.base[g] + (uint32_t)(mag >> g) - P.mlo[g]) * nc + copy;
    val[k] = (uint32_t)(i0 + k) | (neg ? SIGN_BIT : 0u);
    live |= (mag ? 1u : 0u) << k;
  }
  if (SCATTER) {
    uint32_t slot[V_EPT];
#pragma unroll
    for (int k = 0; k < V_EPT; k++)
      if (live >> k & 1u) slot[k] = atomicAdd(cnt + ctr[k], 1u);
    // (measured: the scattered stores of the MSMs in flight combine in L2 — DRAM writes
    // = the 268 MB of entries; the pass is bound by the 67 M returning atomics)
#pragma unroll
    for (int k = 0; k < V_EPT; k++)
      if (live >> k & 1u) vals[slot[k]] = val[k];
  } else {
#pragma unroll
    for (int k = 0; k < V_EPT; k++)
      if (live >> k & 1u) atomicAdd(cnt + ctr[k], 1u);
  }
}

// Counting sort with block-private bucket counters (modes 1 and 3, no global atomics).
// Block (x, l) owns chunk x of MSM l and keeps that MSM's nbm bucket counters in shared
// memory.  k_fpb_pass<.., false>: shared-memory atomics, then the block's counts stored
// chunk-major (cnt[(l S + x) nbm + b], coalesced).  k_fpb_totals / cub scan / k_fpb_starts
// turn them into bucket starts and, in place, the start of every (chunk, bucket) run.
// Scatter: mode 3 k_fpb_scatter_sorted (slice-local counting sort, below); mode 1
// k_fpb_pass<.., true>: the block loads its run starts into shared memory and hands out
// slots with shared-memory atomics, launched a few MSMs at a time so the vals region being
// written stays resident in L2 while the runs' partial sectors fill (one launch over all
// MSMs let them leave L2 half-written: 1.30 ms vs 0.81 ms for the global-atomic scatter).
__device__ __forceinline__ uint32_t fp_key(const WinPlan& P, uint64_t mag, uint32_t& g) {
  const int bl = 64 - __clzll((long long)mag);
  g = bl > P.mbits ? (uint32_t)(bl - P.mbits) : 0u;
  // mode 3: one window of m = |q| >> g in [1, 2^mbits), the exponent goes to the base
  return P.mode == 3 ? (uint32_t)(mag >> g) - 1u : P.base[g] + (uint32_t)(mag >> g) - P.mlo[g];
}

// mode-3 bucket key straight from the fp16 bits: a normal value with exponent field e >=
// 25 - scale_bits quantises exactly to (1024 + mantissa) 2^(e - 25 + scale_bits), so its key
// is 1023 + mantissa and its table level e - 25 + scale_bits (the general path — RNE
// rounding of small values, zeros, subnormals, non-finite — through quant64 / fp_key
// otherwise).
// Returns false for a zero (no entry).
template <int DT>
__device__ __forceinline__ bool key3(uint32_t raw, bool in, int scale_bits, const WinPlan& P, uint32_t& key,
                                     uint32_t& g, bool& neg) {
  if (DT == 1 && P.ktab) {
    // branch-free: one cached table load per element (built by k_build_ktab from the same
    // quant64 / fp_key as below, so every bit pattern maps exactly as the general path)
    if (!in) return false;
    const uint32_t e = __ldg(P.ktab + (raw & 0x7fffu));
    key = e & 0xffffu;
    g = e >> 16;
    neg = (raw >> 15) != 0;
    return e != 0xffffffffu;
  }
  if (DT == 1 && in) {
    const int e = (int)((raw >> 10) & 0x1fu);
    // e == 0 (zero / subnormal) never takes this path, whatever scale_bits admits
    if (e != 0 && e >= 25 - scale_bits && e != 0x1f) {
      key = 1023u + (raw & 0x3ffu);
      g = (uint32_t)(e - 25 + scale_bits);
      neg = (raw >> 15) != 0;
      return true;
    }
  }
  const uint64_t mag = in ? quant64<DT>(raw, scale_bits, neg) : 0ull;
  if (!mag) return false;
  key = fp_key(P, mag, g);
  return true;
}

// the fp16 key table of the exponent-table plan: entry r (r = |bit pattern|) = the bucket key
// | table level g << 16 of the quantised magnitude, 0xFFFFFFFF when it quantises to zero (or
// is not finite: the count pass flags those from the raw bits)
__global__ void k_build_ktab(uint32_t* tab, int scale_bits, WinPlan P) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 32768u) return;
  bool neg;
  const uint64_t mag = ((r & 0x7c00u) == 0x7c00u) ? 0ull : quant64<1>(r, scale_bits, neg);
  uint32_t g = 0, key = 0;
  if (mag) key = fp_key(P, mag, g);
  tab[r] = mag ? (key | (g << 16)) : 0xffffffffu;
}

template <int DT, bool SCATTER>
__global__ void __launch_bounds__(1024) k_fpb_pass(const void* const* ptrs, uint64_t n, int scale_bits, WinPlan P,
                                                   uint32_t* __restrict__ cnt, uint32_t* __restrict__ vals,
                                                   uint64_t chunk, uint32_t l0, uint32_t* flags) {
  extern __shared__ uint32_t h[];
  const uint32_t l = l0 + blockIdx.y, S = gridDim.x;
  const uint64_t c0 = (uint64_t)blockIdx.x * chunk;
  const uint64_t c1 = min(n, c0 + chunk);
  const void* p = ptrs[l];
  uint32_t* row = cnt + ((uint64_t)l * S + blockIdx.x) * P.nbm;
  for (uint32_t b = threadIdx.x; b < P.nbm; b += blockDim.x) h[b] = SCATTER ? row[b] : 0u;
  __syncthreads();
  uint32_t nf = 0;   // fused scan (speculative fp16 plan): non-finite inputs
  for (uint64_t i0 = c0 + (uint64_t)threadIdx.x * V_EPT; i0 < c1; i0 += (uint64_t)blockDim.x * V_EPT) {
    uint32_t raw[V_EPT];
    load_raw8<DT>(p, i0, c1, raw);
#pragma unroll
    for (int k = 0; k < V_EPT; k++) {
      if (!SCATTER && DT == 1 && (raw[k] & 0x7c00u) == 0x7c00u) nf = 1u;
      bool neg;
      uint32_t g, key;
      bool hit;
      if (P.mode == 3) {
        hit = key3<DT>(raw[k], i0 + k < c1, scale_bits, P, key, g, neg);
      } else {
        const uint64_t mag = (i0 + k < c1) ? quant64<DT>(raw[k], scale_bits, neg) : 0ull;
        hit = mag != 0;
        if (hit) key = fp_key(P, mag, g);
      }
      if (hit) {
        const uint32_t slot = atomicAdd(h + key, 1u);
        // mode 3 entries index the exponent table: 2^g G_i at g n + i
        if (SCATTER) vals[slot] = ((P.mode == 3 ? g * P.tpitch : 0u) + (uint32_t)(i0 + k)) | (neg ? SIGN_BIT : 0u);
      }
    }
  }
  if (SCATTER) return;
  if (flags && __any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) atomicOr(flags, QF_NONFINITE);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < P.nbm; b += blockDim.x) row[b] = h[b];
}

// mode-3 scatter with a block-local counting sort of every 8192-element slice: the slice's
// entries are ranked per bucket in shared memory, staged in bucket order together with their
// global slot, and written out by consecutive threads — entries of one bucket (about 4 per
// slice over 2^11 - 1 buckets) land in consecutive addresses from consecutive lanes, so
// they share store transactions instead of costing one scattered 4-byte store each.
#ifndef TC_FPB_THREADS
#define TC_FPB_THREADS 1024   // block size of the block-private count / scatter passes
#endif
#ifndef TC_FPS_THREADS
#define TC_FPS_THREADS 1024   // 16384-element slices: ~8 entries per bucket per slice (A/B: 512 -> 4.75 ms step, 1024 -> 4.70)
#endif
constexpr int FPS_THREADS = TC_FPS_THREADS, FPS_EPT = 16, FPS_SLICE = FPS_THREADS * FPS_EPT;   // 8192
constexpr int FPS_CPT = 2048 / FPS_THREADS;   // bucket counters per thread in the slice scan
template <int DT>
__global__ void __launch_bounds__(FPS_THREADS, 1024 / FPS_THREADS) k_fpb_scatter_sorted(const void* const* ptrs, uint64_t n,
                                                                        int scale_bits, WinPlan P,
                                                                        const uint32_t* __restrict__ cnt,
                                                                        uint32_t* __restrict__ vals, uint64_t chunk,
                                                                        uint32_t l0) {
  extern __shared__ uint32_t sm[];
  const uint32_t NB = P.nbm;                  // <= 2047 (mode 3)
  uint32_t* h = sm;                           // run cursors (global slots)
  uint32_t* lo = sm + 2048;                   // per-slice counts -> exclusive offsets, lo[2048] = total
  uint2* stg = (uint2*)(sm + 2 * 2048 + 32);  // staged (slot, entry), bucket order
  __shared__ uint32_t wsum[FPS_THREADS / 32];
  const uint32_t t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t l = l0 + blockIdx.y, S = gridDim.x;
  const uint32_t* row = cnt + ((uint64_t)l * S + blockIdx.x) * NB;
  for (uint32_t b = t; b < NB; b += FPS_THREADS) h[b] = row[b];
  const uint64_t c0 = (uint64_t)blockIdx.x * chunk;
  const uint64_t c1 = min(n, c0 + chunk);
  const void* p = ptrs[l];
  // the next slice's fp16 / bf16 words are loaded (packed, 2 x 16 B per thread) while the
  // current slice is ranked, scanned, staged and written (the pass was load-latency bound)
  auto ld16 = [&](uint64_t i0, uint4& w) {
    if (i0 + V_EPT <= c1) {
      w = *(const uint4*)((const uint16_t*)p + i0);
    } else {
      uint32_t r[V_EPT];
      load_raw8<DT>(p, i0, c1, r);
      w = make_uint4(r[0] | r[1] << 16, r[2] | r[3] << 16, r[4] | r[5] << 16, r[6] | r[7] << 16);
    }
  };
  uint4 cur[2];
  if (c0 < c1) {
    ld16(c0 + (uint64_t)t * V_EPT, cur[0]);
    ld16(c0 + FPS_SLICE / 2 + (uint64_t)t * V_EPT, cur[1]);
  }
  for (uint64_t base = c0; base < c1; base += FPS_SLICE) {
    for (uint32_t b = t; b < 2048; b += FPS_THREADS) lo[b] = 0u;
    __syncthreads();
    uint32_t key[FPS_EPT], rk[FPS_EPT], val[FPS_EPT];
#pragma unroll
    for (int half = 0; half < 2; half++) {
      const uint64_t i0 = base + (uint64_t)half * (FPS_SLICE / 2) + (uint64_t)t * V_EPT;
      const uint32_t wv[4] = {cur[half].x, cur[half].y, cur[half].z, cur[half].w};
#pragma unroll
      for (int k = 0; k < V_EPT; k++) {
        const int e = half * V_EPT + k;
        const uint32_t rawk = (wv[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        bool neg;
        uint32_t g, kk;
        key[e] = 0xffffffffu;
        if (key3<DT>(rawk, i0 + k < c1, scale_bits, P, kk, g, neg)) {
          key[e] = kk;
          val[e] = (g * P.tpitch + (uint32_t)(i0 + k)) | (neg ? SIGN_BIT : 0u);
          rk[e] = atomicAdd(lo + key[e], 1u);
        }
      }
    }
    if (base + FPS_SLICE < c1) {
      ld16(base + FPS_SLICE + (uint64_t)t * V_EPT, cur[0]);
      ld16(base + FPS_SLICE + FPS_SLICE / 2 + (uint64_t)t * V_EPT, cur[1]);
    }
    __syncthreads();
    // exclusive scan of lo[0..2048): FPS_CPT counters per thread, warp shuffles, warp totals
    uint32_t c[FPS_CPT], sum = 0;
#pragma unroll
    for (int j = 0; j < FPS_CPT; j++) c[j] = lo[FPS_CPT * t + j], sum += c[j];
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      uint32_t w = lane < FPS_THREADS / 32 ? wsum[lane] : 0u, wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= (uint32_t)o) wi += y;
      }
      if (lane < FPS_THREADS / 32) wsum[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = wsum[wid] + inc - sum;
#pragma unroll
    for (int j = 0; j < FPS_CPT; j++) lo[FPS_CPT * t + j] = run, run += c[j];
    if (t == FPS_THREADS - 1) lo[2048] = run;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < FPS_EPT; e++)
      if (key[e] != 0xffffffffu) stg[lo[key[e]] + rk[e]] = make_uint2(h[key[e]] + rk[e], val[e]);
    __syncthreads();
    for (uint32_t b = t; b < NB; b += FPS_THREADS) h[b] += lo[b + 1] - lo[b];
    const uint32_t tot = lo[2048];
    for (uint32_t s2 = t; s2 < tot; s2 += FPS_THREADS) {
      const uint2 q = stg[s2];
      vals[q.x] = q.y;
    }
    __syncthreads();
  }
}

// mode-2 (fixed-base window) count with block-private counters: block (x, l) counts the
// signed digits of chunk x of MSM l in shared memory (2^(c-1) counters) and flushes each
// non-zero counter with one RED — the scatter (k_count_digits) keeps its global cursors
// ROWS: the block's counts are stored chunk-major (cnt[(l S + x) nbm + b], as k_fpb_pass) for
// the block-private scatter k_scatter_fb instead of being added into global counters
template <bool ROWS>
__global__ void __launch_bounds__(1024) k_count_fb(const void* const* ptrs, uint64_t n, WinPlan P,
                                                   uint32_t* __restrict__ cnt, uint64_t chunk) {
  extern __shared__ uint32_t h[];
  const uint32_t l = blockIdx.y;
  const uint64_t c0 = (uint64_t)blockIdx.x * chunk;
  const uint64_t c1 = min(n, c0 + chunk);
  const void* p = ptrs[l];
  for (uint32_t b = threadIdx.x; b < P.nbm; b += blockDim.x) h[b] = 0u;
  __syncthreads();
  const int c = P.cdig;
  const uint32_t half = 1u << (c - 1), full = 1u << c;
  for (uint64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    Fe mag;
    bool neg;
    uint32_t f = 0;
    load_scalar<DT_LIMBS>(p, i, 0, mag, neg, f);
    uint32_t carry = 0;
    for (int w = 0; w < P.ndig; w++) {
      uint32_t d = window_bits(mag, w * c, c) + carry;
      if (d > half) {
        d = full - d, carry = 1;
      } else {
        carry = 0;
      }
      if (d) atomicAdd(h + d - 1u, 1u);
    }
  }
  __syncthreads();
  if (ROWS) {
    uint32_t* row = cnt + ((uint64_t)l * gridDim.x + blockIdx.x) * P.nbm;
    for (uint32_t b = threadIdx.x; b < P.nbm; b += blockDim.x) row[b] = h[b];
    return;
  }
  uint32_t* out = cnt + (uint64_t)l * P.nbm;
  for (uint32_t b = threadIdx.x; b < P.nbm; b += blockDim.x)
    if (h[b]) atomicAdd(out + b, h[b]);
}

// mode-2 scatter with block-private cursors: block (x, l) loads the run starts of chunk x of
// MSM l (k_fpb_starts over k_count_fb<true>'s rows) into shared memory and hands out slots
// with shared-memory atomics — no global atomics (the global-cursor scatter is bound by
// L2 atomic throughput: 738 M digits of a config-3 monomial step in 10.7 ms).  A chunk's
// run per bucket holds ~n ndig / (S nbm) entries, so its sectors fill within the block.
__global__ void __launch_bounds__(1024) k_scatter_fb(const void* const* ptrs, uint64_t n, WinPlan P,
                                                     const uint32_t* __restrict__ runs, uint32_t* __restrict__ vals,
                                                     uint64_t chunk, uint32_t l0) {
  extern __shared__ uint32_t h[];
  const uint32_t l = l0 + blockIdx.y;
  const uint64_t c0 = (uint64_t)blockIdx.x * chunk;
  const uint64_t c1 = min(n, c0 + chunk);
  const void* p = ptrs[l];
  const uint32_t* row = runs + ((uint64_t)l * gridDim.x + blockIdx.x) * P.nbm;
  for (uint32_t b = threadIdx.x; b < P.nbm; b += blockDim.x) h[b] = row[b];
  __syncthreads();
  const int c = P.cdig;
  const uint32_t half = 1u << (c - 1), full = 1u << c;
  for (uint64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    Fe mag;
    bool neg;
    uint32_t f = 0;
    load_scalar<DT_LIMBS>(p, i, 0, mag, neg, f);
    uint32_t carry = 0;
    for (int w = 0; w < P.ndig; w++) {
      uint32_t d = window_bits(mag, w * c, c) + carry;
      bool dn = false;
      if (d > half) {
        d = full - d, dn = true, carry = 1;
      } else {
        carry = 0;
      }
      if (d) vals[atomicAdd(h + d - 1u, 1u)] = (uint32_t)((uint64_t)w * n + i) | ((neg != dn) ? SIGN_BIT : 0u);
    }
  }
}

// tot[l nbm + b] = sum over chunks of cnt[(l S + x) nbm + b]  (loads batched 8 deep: the
// chunk rows are independent, a one-at-a-time loop is latency bound)
__global__ void k_fpb_totals(const uint32_t* cnt, uint32_t nbm, uint32_t L, uint32_t S, uint32_t* tot) {
  const uint64_t key = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= (uint64_t)L * nbm) return;
  const uint64_t l = key / nbm, b = key - l * nbm;
  const uint32_t* c = cnt + l * S * nbm + b;
  uint32_t t = 0;
  for (uint32_t x0 = 0; x0 < S; x0 += 8) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = (x0 + k < S) ? __ldg(c + (uint64_t)(x0 + k) * nbm) : 0u;
#pragma unroll
    for (int k = 0; k < 8; k++) t += v[k];
  }
  tot[key] = t;
}

// counts -> run starts, in place: run (x, b) of MSM l starts at bstart[l nbm + b] plus the
// counts of the earlier chunks
__global__ void k_fpb_starts(uint32_t* __restrict__ cnt, uint32_t nbm, uint32_t L, uint32_t S,
                             const uint32_t* __restrict__ bstart) {
  const uint64_t key = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= (uint64_t)L * nbm) return;
  const uint64_t l = key / nbm, b = key - l * nbm;
  uint32_t* c = cnt + l * S * nbm + b;
  uint32_t run = bstart[key];
  for (uint32_t x0 = 0; x0 < S; x0 += 8) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = (x0 + k < S) ? c[(uint64_t)(x0 + k) * nbm] : 0u;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (x0 + k < S) c[(uint64_t)(x0 + k) * nbm] = run;
      run += v[k];
    }
  }
}

// level 0 piece counts: np[k] = ceil(size/T) (threads), npm[k] = np[k] if > 1 (items);
// an empty bucket is set to the neutral element here (every other bucket is written by
// the accumulation levels), so the bucket array needs no separate fill pass
// buckets from `tail` on take pieces of Ts entries (the accumulation dispatches them last:
// short pieces there shorten its final wave)
__device__ __forceinline__ uint32_t piece_len(uint32_t k, uint32_t T, uint32_t tail, uint32_t Ts) {
  return k >= tail ? Ts : T;
}

__global__ void k_count0(const uint32_t* bstart, const uint32_t* bend, uint32_t nb, uint32_t T, uint32_t tail,
                         uint32_t Ts, uint32_t* np, uint32_t* npm, Ext* buckets) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nb) return;
  const uint32_t Tk = piece_len(k, T, tail, Ts);
  uint32_t c = (k == nb) ? 0u : (bend[k] - bstart[k] + Tk - 1) / Tk;
  np[k] = c;
  npm[k] = c > 1 ? c : 0u;
  if (k < nb && c == 0) buckets[k] = ext_zero();
}

// level >= 1: items of bucket k are [off_in[k], off_in[k+1]) (0 or >= 2 of them)
__global__ void k_count(const uint32_t* off_in, uint32_t nb, uint32_t T, uint32_t* np, uint32_t* npm) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nb) return;
  uint32_t c = (k == nb) ? 0u : (off_in[k + 1] - off_in[k] + T - 1) / T;
  np[k] = c;
  npm[k] = c > 1 ? c : 0u;
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

// level 0: entries are (sign | point index) into the shared Edwards affine bases.  A bucket
// that fits in one piece is final (written to buckets[k]); otherwise its piece sums go to
// items.  The accumulator starts as the piece's first point, then one complete 8M mixed
// add per entry (no exceptional cases, ec.cuh).
#ifndef TC_M3_SMALL_E
#define TC_M3_SMALL_E (1ull << 24)   // exponent-table batches below this many entries take 16-entry pieces
#endif
#ifndef TC_ACCUM_PF
#define TC_ACCUM_PF 1   // A/B (config 3): 0 -> 3.982 ms, 1 -> 3.909 (MINB 4), 2 (+L2 prefetch) -> 4.15, 3 (point in registers) -> 4.14
#endif
#ifndef TC_ACCUM_MINB
#define TC_ACCUM_MINB 6   // min resident blocks per SM for k_accum_aff (a = -1 model, PF 1): 4 -> 112 registers, 3.768 ms; 5 -> 95, 3.641; 6 -> 80 + 24 B stack, 3.629; 7 -> 72 + 68 B spills, 0.844 vs 0.857 of the peak (the a = 2 model ran best at 4 / 96)
#endif
__global__ void __launch_bounds__(128, TC_ACCUM_MINB) k_accum_aff(const uint32_t* vals, const EdPk* bases, const uint32_t* bstart,
                                                   const uint32_t* bend, const uint32_t* toff, const uint32_t* ooff,
                                                   uint32_t nb, uint32_t T, uint32_t tail, uint32_t Ts,
                                                   Ext* items, Ext* buckets, const uint32_t* boff, uint32_t nbm) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t total = toff[nb];
  if (p >= total) return;
  uint32_t k = find_bucket(toff, nb, p);
  if (boff) bases += boff[k / nbm];   // multi-base batch: MSM l reads bases + boff[l]
  uint32_t piece = p - toff[k];
  const uint32_t Tk = piece_len(k, T, tail, Ts);
  uint32_t a = bstart[k] + piece * Tk;
  uint32_t b = min(a + Tk, bend[k]);
  uint32_t v = vals[a];
  EdAff q = ld_edpk(bases + (v & ~SIGN_BIT));
  if (v & SIGN_BIT) q = edaff_neg(q);
  Ext acc = ext_from_aff(q);
#if TC_ACCUM_PF == 3
  // the next point in registers (gathered during the current add), its index two ahead
  uint32_t vn = a + 1 < b ? vals[a + 1] : 0u;
  uint32_t vnn = a + 2 < b ? vals[a + 2] : 0u;
  EdAff qn = ld_edpk(bases + (vn & ~SIGN_BIT));
  for (uint32_t j = a + 1; j < b; j++) {
    q = qn;
    v = vn;
    vn = vnn;
    if (j + 1 < b) qn = ld_edpk(bases + (vn & ~SIGN_BIT));
    vnn = j + 2 < b ? vals[j + 2] : 0u;
    if (v & SIGN_BIT) q = edaff_neg(q);
    ext_madd(acc, q);
  }
#elif TC_ACCUM_PF
  // software-pipelined entry index: the next point's address is known one add ahead, so
  // its gather (and, PF 2, an L2 prefetch of its line) overlaps the current add
  uint32_t vn = a + 1 < b ? vals[a + 1] : 0u;
  for (uint32_t j = a + 1; j < b; j++) {
    v = vn;
#if TC_ACCUM_PF >= 2
    if (j + 1 < b) {
      vn = vals[j + 1];
      asm volatile("prefetch.global.L2 [%0];" ::"l"(bases + (vn & ~SIGN_BIT)));
    }
#else
    vn = j + 1 < b ? vals[j + 1] : 0u;
#endif
    q = ld_edpk(bases + (v & ~SIGN_BIT));
    if (v & SIGN_BIT) q = edaff_neg(q);
    ext_madd(acc, q);
  }
#else
  for (uint32_t j = a + 1; j < b; j++) {
    v = vals[j];
    q = ld_edpk(bases + (v & ~SIGN_BIT));
    if (v & SIGN_BIT) q = edaff_neg(q);
    ext_madd(acc, q);
  }
#endif
  if (toff[k + 1] - toff[k] == 1)
    buckets[k] = acc;
  else
    items[ooff[k] + piece] = acc;
}

// level >= 1: bucket k's items are in[iofs[k] .. iofs[k+1])
__global__ void __launch_bounds__(128) k_accum_ext(const Ext* in, const uint32_t* iofs, const uint32_t* toff,
                                                    const uint32_t* ooff, uint32_t nb, uint32_t T, Ext* out,
                                                    Ext* buckets) {
  // grid-stride: the launch is sized from a host-side bound (no read-back of the level's
  // piece count), so a bounded grid avoids launching mostly-empty blocks on deep levels
  const uint32_t total = toff[nb];
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < total; p += gridDim.x * blockDim.x) {
    const uint32_t k = find_bucket(toff, nb, p);
    const uint32_t piece = p - toff[k];
    const uint32_t a = iofs[k] + piece * T;
    const uint32_t b = min(a + T, iofs[k + 1]);
    Ext acc = ld_ext(in + a);
    for (uint32_t j = a + 1; j < b; j++) ext_add(acc, ld_ext(in + j));
    if (toff[k + 1] - toff[k] == 1)
      buckets[k] = acc;
    else
      out[ooff[k] + piece] = acc;
  }
}

// ---- weighted bucket sums A_g = sum_j (j+1) x_j by recursive segmentation ----------------
// Split each group into segments of SEG items: per segment k, T_k = sum x_j and
// U_k = sum (j - SEG k + 1) x_j (running sums).  Then
//     A(x) = sum_k U_k + SEG * sum_k k T_k = sum_k U_k + SEG * A(T) - SEG * S,
// S = sum x.  Recursing on T (SEG x fewer items per level) and carrying
//     D = sum_{levels r} SEG^{r-1} sum_k U_{r,k}
// in a second stream gives, after R levels (every group reduced to one item, T = S),
//     A(x) = D - S * (SEG^R - SEG) / (SEG - 1).
// No per-segment scalar multiplications and SEG x more parallelism than one thread per
// window; every level is one launch over all groups of the batch.
// segment length SEG = 2^lg (runtime: TC_MSM_SEG_LG, default 3)

struct GroupTab {   // per group: input offset, input count, output offset (device)
  const uint32_t* in_off;
  const uint32_t* in_cnt;
  const uint32_t* out_off;
  uint32_t ngroups;
};

__global__ void __launch_bounds__(128) k_wsum_level(const Ext* Tin, const Ext* Din, GroupTab G, uint32_t total_out,
                                                    uint32_t dbl_shift, uint32_t SEG, Ext* Tout, Ext* Dout) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= total_out) return;
  uint32_t lo = 0, hi = G.ngroups;   // group g with out_off[g] <= o < out_off[g+1]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (G.out_off[mid] <= o)
      lo = mid;
    else
      hi = mid;
  }
  const uint32_t g = lo, k = o - G.out_off[g];
  const uint32_t a = G.in_off[g] + k * SEG;
  const uint32_t len = min(SEG, G.in_cnt[g] - k * SEG);
  Ext run = ext_zero(), u = ext_zero();
  for (int j = (int)len - 1; j >= 0; j--) {
    ext_add(run, ld_ext(Tin + a + j));
    ext_add(u, run);
  }
  Tout[o] = run;
  // D_out = sum of D_in over the segment + SEG^{r-1} * U
  for (uint32_t i = 0; i < dbl_shift; i++) u = ext_dbl(u);
  if (Din)
    for (uint32_t j = 0; j < len; j++) ext_add(u, ld_ext(Din + a + j));
  Dout[o] = u;
}

// One block per (MSM, window) for windows of <= WB_THREADS * WB_CHUNK buckets (the
// float-exponent groups): W = sum_j (mlo + j) B_j in ONE launch instead of recursive
// levels.  Thread t takes the chunk [t C, t C + C) (C = WB_CHUNK, a power of two) and forms
// T_t = sum of the chunk and U_t = sum (j - tC + 1) B_j by running sums; then
//     A = sum_j (j+1) B_j = sum_t U_t + C * sum_t t T_t,   sum_t t T_t = sum_{t>=1} R_t,
// R_t = sum_{s>=t} T_s (a shared-memory suffix scan), S = R_0, and W = A + (mlo - 1) S.
// Serial depth ~ 2C + 2 log2(threads) + log2(C) + log2(mlo) adds instead of ~27 per level.
#ifndef TC_WB_THREADS
#define TC_WB_THREADS 256   // A/B: 512 -> lone forward 5.02 ms, pipelined 4.471; 256 -> 4.99, 4.457; 128 -> 5.00, 4.458
#endif
constexpr int WB_THREADS = TC_WB_THREADS;
constexpr int WB_CHUNK_LG = TC_WB_THREADS == 512 ? 2 : (TC_WB_THREADS == 256 ? 3 : 4);   // 2048 buckets

// prescale: also multiply the window sum by 2^off[w] (its weight in the scalar), so the
// windows of an MSM only need to be ADDED (k_final_sum): the doublings of all windows run
// in parallel blocks instead of one Horner chain
__global__ void __launch_bounds__(WB_THREADS, 1) k_wsum_block(const Ext* buckets, WinPlan P, Ext* W, int prescale) {
  extern __shared__ Ext wb_smem[];
  Ext* sh = wb_smem;
  Ext* su = wb_smem + WB_THREADS;
  const uint32_t g = blockIdx.x, l = g / P.nwin, w = g % P.nwin, t = threadIdx.x;
  const uint32_t nbw = P.base[w + 1] - P.base[w];
  const Ext* b = buckets + (uint64_t)l * P.nbm + P.base[w];
  const uint32_t C = 1u << WB_CHUNK_LG, a = t * C, e = min(a + C, nbw);
  Ext run = ext_zero(), u = ext_zero();
  for (int j = (int)e - 1; j >= (int)a; j--) {
    ext_add(run, ld_ext(b + j));
    ext_add(u, run);
  }
  sh[t] = run;
  su[t] = u;
  __syncthreads();
  // inclusive suffix scan R_t = sum_{s >= t} T_s (Hillis-Steele).  The scan and reduction
  // loops stay rolled: one copy of the Edwards add instead of nine straight-line ones keeps
  // this latency-bound kernel in the instruction cache
#pragma unroll 1
  for (uint32_t o = 1; o < WB_THREADS; o <<= 1) {
    Ext v = sh[t];
    if (t + o < WB_THREADS) ext_add(v, sh[t + o]);
    __syncthreads();
    sh[t] = v;
    __syncthreads();
  }
  const Ext S = sh[0];
  // reduce sum_{t>=1} R_t (into sh) and sum_t U_t (into su)
  if (t == 0) sh[0] = ext_zero();
  __syncthreads();
#pragma unroll 1
  for (uint32_t o = WB_THREADS / 2; o; o >>= 1) {
    if (t < o) {
      Ext x = sh[t], y = su[t];
      ext_add(x, sh[t + o]);
      ext_add(y, su[t + o]);
      sh[t] = x;
      su[t] = y;
    }
    __syncthreads();
  }
  if (t != 0) return;
  Ext A = sh[0];
  for (int i = 0; i < WB_CHUNK_LG; i++) A = ext_dbl(A);
  ext_add(A, su[0]);
  const uint32_t c = P.mlo[w] - 1u;
  if (c) ext_add(A, ext_mul_small_naf(S, c));
  if (prescale)
    for (int i = 0; i < P.off[w]; i++) A = ext_dbl(A);
  W[g] = A;
}

// W_g = D_g - c * S_g + (mlo_w - 1) * S_g: sum_j (j+1) x_j re-based to the window's weights
__global__ void k_wsum_final(const Ext* T, const Ext* D, uint32_t ngroups, uint32_t c, WinPlan P, Ext* W) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  Ext w = D[g];
  const int64_t coef = (int64_t)P.mlo[g % P.nwin] - 1 - (int64_t)c;
  if (coef) {
    Ext s = ext_mul_small_naf(T[g], (uint32_t)(coef < 0 ? -coef : coef));
    ext_add(w, coef < 0 ? ext_neg(s) : s);
  }
  W[g] = w;
}

// Horner over the windows of MSM l: acc = 2^{c_w} acc + S_w from the top, then affine
__global__ void k_final(const Ext* wsum, uint32_t L, WinPlan P, Aff* out) {
  uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const Ext* ws = wsum + (uint64_t)l * P.nwin;
  Ext acc = ws[P.nwin - 1];
  for (int w = P.nwin - 2; w >= 0; w--) {
    for (int i = 0; i < P.off[w + 1] - P.off[w]; i++) acc = ext_dbl(acc);
    ext_add(acc, ws[w]);
  }
  Aff r = ext_to_aff(acc);
  if (!aff_is_inf(r)) {
    r.x = Fq::canon(r.x);
    r.y = Fq::canon(r.y);
  }
  out[l] = r;
}

// one warp per MSM: sum of its (prescaled) window sums by a shuffle tree, then affine
__global__ void k_final_sum(const Ext* wsum, uint32_t L, int nwin, Aff* out) {
  const uint32_t l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (l >= L) return;   // whole warps
  Ext acc = ext_zero();
  for (int w = (int)lane; w < nwin; w += 32) ext_add(acc, ld_ext(wsum + (uint64_t)l * nwin + w));
#pragma unroll 1
  for (int o = 16; o; o >>= 1) {
    Ext other;
#pragma unroll
    for (int i = 0; i < 6; i++) {
      other.X.v[i] = __shfl_down_sync(0xffffffffu, acc.X.v[i], o);
      other.Y.v[i] = __shfl_down_sync(0xffffffffu, acc.Y.v[i], o);
      other.Z.v[i] = __shfl_down_sync(0xffffffffu, acc.Z.v[i], o);
      other.T.v[i] = __shfl_down_sync(0xffffffffu, acc.T.v[i], o);
    }
    if (lane < (uint32_t)o) ext_add(acc, other);
  }
  if (lane == 0) {
    Aff r = ext_to_aff(acc);
    if (!aff_is_inf(r)) r = Aff{Fq::canon(r.x), Fq::canon(r.y)};
    out[l] = r;
  }
}

__global__ void k_fill_inf(Aff* out, uint32_t L) {
  uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < L) out[l] = aff_inf();
}

// Window plan from the bit-length histogram.  Window w (bits [o, o+c)) holds a non-zero
// digit roughly iff the magnitude has bit length > o (carries included), so it costs
// E_w = #{elements with bitlen > o} bucket entries plus L * 2^(c-1) buckets, each costing
// ~KAPPA entries in the running-sum reduction.  DP over window boundaries.
WinPlan plan_windows(const uint32_t* hist, uint32_t nbits, uint64_t L) {
  // KAPPA: cost of one bucket in bucket-entry units (~2.4 full XYZZ adds in the recursive
  // bucket weighting + sort-key width).  tools/ab_kappa.sh on config 3: KAPPA 2..6 picks
  // an 18-bit low window, 13.95 ms/step (vs 15.4 ms at KAPPA 64 / 10-bit windows and
  // 17.7 ms for uniform 16-bit windows).
  static const double KAPPA = getenv("TC_MSM_KAPPA") ? atof(getenv("TC_MSM_KAPPA")) : 4.0;
  const int top = (int)nbits + 1;   // bits to cover incl. the final carry
  double above[NHIST + 2];          // above[o] = #elements with bitlen > o
  double acc = 0;
  for (int b = NHIST; b >= 0; b--) {
    above[b] = acc;
    if (b < NHIST) acc += hist[b];
  }
  above[NHIST + 1] = 0;
  static const int CMAX = getenv("TC_MSM_CMAX") ? atoi(getenv("TC_MSM_CMAX")) : 20;
  static const int CMIN_ENV = getenv("TC_MSM_CMIN") ? atoi(getenv("TC_MSM_CMIN")) : 4;
  const int CMIN = std::max(CMIN_ENV, (top + MAXW - 1) / MAXW);   // at most MAXW windows
  std::vector<double> best(top + CMAX + 1, 1e300);
  std::vector<int> from(top + CMAX + 1, -1);
  best[0] = 0;
  for (int o = 0; o < top; o++) {
    if (best[o] >= 1e299) continue;
    for (int c = CMIN; c <= CMAX; c++) {
      // a window may overshoot the top: the bits above nbits are zero
      const int dst = std::min(o + c, top);
      const double cost = best[o] + (o <= NHIST ? above[o] : 0) + KAPPA * (double)L * (double)(1u << (c - 1));
      if (cost < best[dst]) {
        best[dst] = cost;
        from[dst] = o * 64 + c;   // window start and width
      }
    }
  }
  // backtrack
  int pos = top;
  std::vector<std::pair<int, int>> wins;
  while (pos > 0) {
    int f = from[pos];
    int o = f / 64, c = f % 64;
    wins.push_back({o, c});
    pos = o;
  }
  WinPlan P;
  P.mode = 0;
  P.mbits = 0;
  P.ndig = P.cdig = 0;
  P.nwin = (int)wins.size();
  uint32_t b = 0;
  for (int w = 0; w < P.nwin; w++) {
    auto oc = wins[P.nwin - 1 - w];
    P.off[w] = (uint8_t)oc.first;
    P.width[w] = (uint8_t)oc.second;
    P.mlo[w] = 1;
    P.base[w] = b;
    b += 1u << (oc.second - 1);
  }
  P.base[P.nwin] = b;
  P.nbm = b;
  if (getenv("TC_MSM_DEBUG")) {
    fprintf(stderr, "[tc msm] L=%llu nbits=%u windows:", (unsigned long long)L, nbits);
    for (int w = 0; w < P.nwin; w++) fprintf(stderr, " [%d,+%d)", P.off[w], P.width[w]);
    fprintf(stderr, " buckets/msm=%u\n", P.nbm);
  }
  return P;
}

// mode-2 plan: one window of 2^(c-1) buckets shared by all digit windows
WinPlan plan_fb(int c) {
  WinPlan P;
  P.mode = 2;
  P.mbits = 0;
  P.ndig = tcrt::fb_ndig(c);
  P.cdig = c;
  P.nwin = 1;
  P.off[0] = 0;
  P.width[0] = (uint8_t)c;
  P.mlo[0] = 1;
  P.base[0] = 0;
  P.base[1] = P.nbm = 1u << (c - 1);
  return P;
}

// mode-1 plan: groups k = 0 .. nbits - MB (see WinPlan)
WinPlan plan_fp(uint32_t nbits, int mb) {
  WinPlan P;
  P.mode = 1;
  P.ndig = P.cdig = 0;
  P.mbits = mb;
  P.nwin = nbits > (uint32_t)mb ? (int)nbits - mb + 1 : 1;
  uint32_t b = 0;
  for (int w = 0; w < P.nwin; w++) {
    P.off[w] = (uint8_t)w;
    P.width[w] = 0;
    P.mlo[w] = w ? 1u << (mb - 1) : 1u;
    P.base[w] = b;
    b += w ? 1u << (mb - 1) : (1u << mb) - 1u;
  }
  P.base[P.nwin] = b;
  P.nbm = b;
  return P;
}

// mode 3: the float-exponent plan over an exponent table (srs_exp_table): entry (i, g)
// reads the base 2^g G_i, so all groups share ONE window of 2^mb - 1 buckets of weight m
WinPlan plan_fpx(int mb, uint32_t pitch) {
  WinPlan P;
  P.tpitch = pitch;
  P.mode = 3;
  P.ndig = P.cdig = 0;
  P.mbits = mb;
  P.nwin = 1;
  P.off[0] = 0;
  P.width[0] = 0;
  P.mlo[0] = 1;
  P.base[0] = 0;
  P.base[1] = (1u << mb) - 1u;
  P.nbm = P.base[1];
  return P;
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

// fp16 inputs on the exponent-table plan classify every element with one table load
// (k_build_ktab, per context and scale_bits) instead of the per-element branches of key3
static int attach_ktab(tc_ctx* ctx, int dtype, int scale_bits, WinPlan& P) {
  P.ktab = nullptr;
  static const bool off = getenv("TC_NO_KTAB") != nullptr;
  if (off || dtype != TC_DTYPE_F16) return TC_OK;
  const std::string key = "msm.ktab." + std::to_string(scale_bits);
  uint32_t* tab;
  const bool have = ctx->scratch.count(key + ".ready") != 0;
  TC_TRY(scratch_t(ctx, key.c_str(), 32768, &tab));
  if (!have) {
    k_build_ktab<<<128, 256, 0, ctx->stream>>>(tab, scale_bits, P);
    TC_LAUNCHED(ctx);
    ctx->scratch[key + ".ready"] = tc_ctx::Buf{};
  }
  P.ktab = tab;
  return TC_OK;
}

int msm_batch_device(tc_ctx* ctx, int dtype, int scale_bits, const void* const* h_ptrs, int L, const EdPk* d_bases,
                     uint64_t n, Aff* d_out, const uint32_t* h_boff, int fbw, tc_srs* exp_srs) {
  if (fbw && (dtype != TC_DTYPE_FP_LIMBS || n * fb_ndig(fbw) >= (1ull << 31)))
    return fail(ctx, TC_ERR_VALUE, "msm: window-table MSMs take field-element scalars, < 2^31 table points");
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
  // bound the scratch of one pipeline: at most 2^28 fp16 / bf16 values (one bucket entry
  // each under the float-exponent plan: 1 GiB of entries), 2^26 other floats (<= 3-4
  // windows) or 2^24 full field elements (~14 windows) per batch; larger batches run in
  // groups (config 5: 6 layers of 41.9 M per pipeline instead of 1, so the reduction tails
  // are paid 7 times per step instead of 40)
  {
    static const uint64_t PER16 = getenv("TC_MSM_PER16") ? strtoull(getenv("TC_MSM_PER16"), nullptr, 10) : (1ull << 28);
    const uint64_t per = (dtype == TC_DTYPE_FP_LIMBS) ? (1ull << 24)
                         : (dtype == TC_DTYPE_F16 || dtype == TC_DTYPE_BF16) ? PER16 : (1ull << 26);
    const uint64_t G = std::max<uint64_t>(1, per / n);
    if ((uint64_t)L > G) {
      const bool defer = ctx->defer_req;   // several pipelines: each finishes its own points
      ctx->defer_req = false;
      for (int l0 = 0; l0 < L; l0 += (int)G) {
        const int cnt = (int)std::min<uint64_t>(G, (uint64_t)(L - l0));
        const int st2 = msm_batch_device(ctx, dtype, scale_bits, h_ptrs + l0, cnt, d_bases, n, d_out + l0,
                                         h_boff ? h_boff + l0 : nullptr, fbw, exp_srs);
        if (st2) {
          ctx->defer_req = defer;
          return st2;
        }
      }
      ctx->defer_req = defer;
      return TC_OK;
    }
  }
  // scalar pointers -> device (pinned staging; the syncs below keep it alive)
  const void** d_ptrs;
  TC_TRY(scratch_t(ctx, "msm.ptrs", (uint64_t)L, (void***)&d_ptrs));
  memcpy(ctx->h_stage, h_ptrs, sizeof(void*) * L);
  TC_CUDA(ctx, cudaMemcpyAsync(d_ptrs, ctx->h_stage, sizeof(void*) * L, cudaMemcpyHostToDevice, st));
  uint32_t* d_boff = nullptr;
  if (h_boff) {   // per-MSM base offsets (staged behind the pointers)
    if (sizeof(void*) * L + sizeof(uint32_t) * L > 65536) return fail(ctx, TC_ERR_VALUE, "msm: batch too large");
    TC_TRY(scratch_t(ctx, "msm.boff", (uint64_t)L, &d_boff));
    memcpy((char*)ctx->h_stage + sizeof(void*) * L, h_boff, sizeof(uint32_t) * L);
    TC_CUDA(ctx, cudaMemcpyAsync(d_boff, (char*)ctx->h_stage + sizeof(void*) * L, sizeof(uint32_t) * L,
                                 cudaMemcpyHostToDevice, st));
  }

  // 1. bit-length histogram + quantisation status
  uint32_t* d_small;
  const int NSMALL = NHIST + 8;
  TC_TRY(scratch_t(ctx, "msm.small", NSMALL, &d_small));
  TC_CUDA(ctx, cudaMemsetAsync(d_small, 0, NSMALL * sizeof(uint32_t), st));
  // fp16 over an exponent table deep enough for ANY finite input (|q| < 2^(16 + scale_bits):
  // scale_bits + 6 groups) needs nothing from the scan: the plan is fixed, so the scan is
  // fused into the count pass (its non-finite flag read back with the entry count) and the
  // pipeline has no host round trip before the sort (speculative mode 3)
  static const bool no_spec = getenv("TC_MSM_NO_SPEC") != nullptr;
  static const uint64_t EXP_MIN_N0 =
      getenv("TC_MSM_EXP_MIN_N") ? strtoull(getenv("TC_MSM_EXP_MIN_N"), nullptr, 10) : (1ull << 14);
  const EdPk* spec_tab = nullptr;
  if (!no_spec && !fbw && dtype == TC_DTYPE_F16 && scale_bits + 16 <= 61 && exp_srs &&
      d_bases == exp_srs->ed_lagrange && n >= EXP_MIN_N0 && n >= (1u << 16) && !getenv("TC_MSM_NO_EXPTAB") &&
      !getenv("TC_MSM_NO_BLKCNT") && !getenv("TC_MSM_GENERIC_DIGITS") &&
      (uint64_t)(scale_bits + 6) * exp_srs->n < (1ull << 31)) {
    bool al = true;
    for (int l = 0; l < L && al; l++) al = ((uintptr_t)h_ptrs[l] & 15u) == 0;
    if (!al || srs_exp_table(ctx, exp_srs, d_bases, exp_srs->n, scale_bits + 6, &spec_tab) != TC_OK)
      spec_tab = nullptr;
  }
  if (!spec_tab) {
    unsigned gx = std::min<unsigned>(blocks_for(n, 256), std::max(1u, (unsigned)ctx->num_sms * 8 / (unsigned)L + 1));
    bool vec = true;   // 16-byte loads need aligned inputs
    for (int l = 0; l < L; l++) vec = vec && ((uintptr_t)h_ptrs[l] & 15u) == 0;
    int s = dispatch_dt(ctx, dtype, [&](auto dt) {
      constexpr int D = decltype(dt)::value;
      if constexpr (D >= 1 && D <= 3) {
        if (vec) {
          k_scan_bits_v<D><<<dim3(gx, L), 256, 0, st>>>(d_ptrs, n, scale_bits, d_small);
          return;
        }
      }
      k_scan_bits<D><<<dim3(gx, L), 256, 0, st>>>(d_ptrs, n, scale_bits, d_small);
    });
    if (s) return s;
    TC_LAUNCHED(ctx);
  }
  uint32_t* h_small = (uint32_t*)((char*)ctx->h_stage + 65536);
  uint32_t hist[NHIST];   // sampled counts scaled back to the population
  uint32_t nbits;
  if (spec_tab) {
    nbits = (uint32_t)(16 + scale_bits);   // upper bound: the plan does not need the maximum
    for (int b = 0; b < NHIST; b++) hist[b] = 0;
  } else {
    TC_CUDA(ctx, cudaMemcpyAsync(h_small, d_small, (NHIST + 2) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    TC_CUDA(ctx, cudaStreamSynchronize(st));
    TC_TRY(quantize_flags_to_status(ctx, h_small[0]));
    for (int b = 0; b < NHIST; b++) hist[b] = h_small[1 + b] * HIST_SAMPLE;
    nbits = std::min<uint32_t>(h_small[NHIST + 1], NHIST - 1);   // exact maximum
    if (nbits) hist[nbits] = std::max<uint32_t>(hist[nbits], 1u);
  }
  if (nbits == 0) {
    k_fill_inf<<<blocks_for(L, 64), 64, 0, st>>>(d_out, (uint32_t)L);
    TC_LAUNCHED(ctx);
    return TC_OK;
  }

  // 2. window plan: float-exponent groups for large fp16 / bf16 batches on the vectorised
  //    digit path, signed windows from the histogram DP otherwise
  static const bool generic_digits = getenv("TC_MSM_GENERIC_DIGITS") != nullptr;
  static const uint64_t FP_MIN_N = getenv("TC_MSM_FP_MIN_N") ? strtoull(getenv("TC_MSM_FP_MIN_N"), nullptr, 10)
                                                            : (1ull << 18);
  bool vec_ok = (dtype == TC_DTYPE_F16 || dtype == TC_DTYPE_BF16 || dtype == TC_DTYPE_F32) && nbits <= 61 &&
                !generic_digits;
  for (int l = 0; l < L && vec_ok; l++) vec_ok = ((uintptr_t)h_ptrs[l] & 15u) == 0;   // 16-byte vector loads
  const int fp_mb = dtype == TC_DTYPE_F16 ? 11 : (dtype == TC_DTYPE_BF16 ? 8 : 0);
  const bool fpmode = vec_ok && fp_mb && n >= FP_MIN_N && (int)nbits - fp_mb + 1 <= MAXW;
  WinPlan P = fbw ? plan_fb(fbw) : fpmode ? plan_fp(nbits, fp_mb) : plan_windows(hist, nbits, (uint64_t)L);
  P.tpitch = 0;
  // exponent-table plan (mode 3) when the caller's bases lie in a Lagrange basis whose table
  // (depth = the batch's exponent groups) fits in memory; its 2^mb - 1 buckets per MSM pay
  // off from a few times that many points (slice commitments: 1024 MSMs of 65536)
  static const bool no_exp = getenv("TC_MSM_NO_EXPTAB") != nullptr;
  static const uint64_t EXP_MIN_N =
      getenv("TC_MSM_EXP_MIN_N") ? strtoull(getenv("TC_MSM_EXP_MIN_N"), nullptr, 10) : (1ull << 14);
  const EdPk* bases = d_bases;
  const int groups = fp_mb ? std::max(1, (int)nbits - fp_mb + 1) : 0;
  if (spec_tab) {
    P = plan_fpx(fp_mb, (uint32_t)exp_srs->n);
    TC_TRY(attach_ktab(ctx, dtype, scale_bits, P));
    bases = spec_tab;
  } else if (!fbw && exp_srs && d_bases == exp_srs->ed_lagrange && !no_exp && !getenv("TC_MSM_NO_BLKCNT") && vec_ok &&
      fp_mb && n >= EXP_MIN_N &&
      groups <= MAXW && (uint64_t)groups * exp_srs->n < (1ull << 31)) {
    const EdPk* tab = nullptr;
    // fp16: ask for the depth ANY finite input needs (scale_bits + 6) so the table is built
    // once instead of regrown batch by batch; the batch's own depth when that does not fit
    const int full = dtype == TC_DTYPE_F16 ? scale_bits + 6 : 0;
    const bool full_ok = full > groups && (uint64_t)full * exp_srs->n < (1ull << 31);
    if ((full_ok && srs_exp_table(ctx, exp_srs, d_bases, exp_srs->n, full, &tab) == TC_OK) ||
        srs_exp_table(ctx, exp_srs, d_bases, exp_srs->n, groups, &tab) == TC_OK) {
      P = plan_fpx(fp_mb, (uint32_t)exp_srs->n);
      TC_TRY(attach_ktab(ctx, dtype, scale_bits, P));
      bases = tab;   // multi-base batches (h_boff) index inside the table's level 0 as before
    }
  }
  if (P.nwin > MAXW) return fail(ctx, TC_ERR_VALUE, "msm: window plan too long");
  const uint64_t nb64 = (uint64_t)L * P.nbm;
  if (nb64 >= (1ull << 31)) return fail(ctx, TC_ERR_VALUE, "msm batch too large (%llu buckets)", (unsigned long long)nb64);
  const uint32_t nb = (uint32_t)nb64;
  const uint64_t cap = (uint64_t)L * n * ((P.mode == 1 || P.mode == 3) ? 1 : P.mode == 2 ? P.ndig : P.nwin);

  // 3. non-zero digits, compacted
  uint32_t* vals;
  TC_TRY(scratch_t(ctx, "msm.vals", cap, &vals));
  const uint32_t* svals;
  uint32_t *bstart, *bend;
  uint64_t E;
  bool have_maxb = false;   // exact largest bucket known (counting layout)
  uint32_t maxb = 0;
  // level 0 of the bucket accumulation: piece tables (k_count0 + scans) and k_accum_aff.
  // E_plan sizes pieces and scratch (an upper bound is fine: surplus threads exit on the
  // device-side piece count); the block-counter path queues it BEFORE the host waits for
  // the entry count, so the GPU goes from the scatter straight into the accumulation
  struct Level0 {
    uint32_t T = 0, T1 = 0, tail = 0, Ts = 0, Tmin = 0;
    uint64_t max_items = 0;
    uint32_t *np, *npm, *toff, *offA, *offB;
    Ext *itemsA, *itemsB, *buckets;
    void* d_scan;
    size_t scan_bytes = 0;
  } L0;
  bool early0 = false;
  auto level0 = [&](uint64_t E_plan) -> int {
    static const uint32_t T_ENV = getenv("TC_MSM_T") ? (uint32_t)atoi(getenv("TC_MSM_T")) : 16u;   // sweep (config 3): 8 6.75, 12 6.66, 16 6.54, 24 6.60, 32 6.64 ms
    static const uint32_t T1_ENV = getenv("TC_MSM_T1") ? (uint32_t)atoi(getenv("TC_MSM_T1")) : 8u;
    // piece length: 16 entries balances config 3 (~114 entries per bucket); dense buckets
    // (config 5: ~2300 per bucket) take longer pieces (fewer items for the tail levels:
    // 6-layer batch 22.0 -> 21.5 ms at 64)
    uint32_t T = (E_plan >= (1u << 20)) ? T_ENV : (E_plan >= (1u << 14) ? 16u : 8u);
    // exponent-table plan (mode 3, ~1000 entries per bucket): pieces of 32 with 16 items per
    // reduction thread (A/B over 40 forwards: T 64 / T1 8 -> 4.479 ms per step, 32 / 16 ->
    // 4.463, 24 / 8 -> 4.480; shorter pieces shorten the accumulation's last wave, the
    // wider reduction keeps the item levels at two)
    const bool m3 = P.mode == 3 && !getenv("TC_MSM_T") && !getenv("TC_MSM_T1");
    if (!getenv("TC_MSM_T") && E_plan >= (1u << 20)) {
      const uint64_t per_bucket = E_plan / std::max<uint64_t>(1, nb);
      // smaller batches (a multi-GPU rank's few layers) have fewer waves: shorter pieces still
      // (4 layers: 0.706 -> 0.686 ms per pipelined forward at 16; 32 layers: 16 is slower)
      const uint32_t tmax = m3 ? (E_plan < TC_M3_SMALL_E ? 16u : 32u) : 64u;
      while (T < tmax && (uint64_t)T * 16 <= per_bucket) T *= 2;
    }
    L0.T = T;
    L0.T1 = (m3 && T >= 16) ? 16u : T1_ENV;
    // items = pieces of multi-piece buckets: ceil(sz/T) <= 2 sz / T for sz > T
    L0.max_items = 2 * ((E_plan + std::max<uint32_t>(4u, T / 4) - 1) / std::max<uint32_t>(4u, T / 4)) + 2;
    TC_TRY(scratch_t(ctx, "msm.np", (uint64_t)nb + 1, &L0.np));
    TC_TRY(scratch_t(ctx, "msm.npm", (uint64_t)nb + 1, &L0.npm));
    TC_TRY(scratch_t(ctx, "msm.toff", (uint64_t)nb + 1, &L0.toff));
    TC_TRY(scratch_t(ctx, "msm.offA", (uint64_t)nb + 1, &L0.offA));
    TC_TRY(scratch_t(ctx, "msm.offB", (uint64_t)nb + 1, &L0.offB));
    TC_TRY(scratch_t(ctx, "msm.itemsA", L0.max_items, &L0.itemsA));
    TC_TRY(scratch_t(ctx, "msm.itemsB", L0.max_items, &L0.itemsB));
    TC_TRY(scratch_t(ctx, "msm.buckets", nb, &L0.buckets));
    L0.scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, L0.scan_bytes, L0.np, L0.toff, (int)(nb + 1), st);
    TC_TRY(scratch(ctx, "msm.scantmp", L0.scan_bytes, &L0.d_scan));
    // the last TC_MSM_TAIL_PCT % of the buckets take quarter-length pieces (off by default:
    // config 3, 3 % -> 4.496 ms per step vs 4.457 — the accumulation's last wave shrinks by
    // 25 us but the short pieces need one more reduction level)
    static const uint32_t TAIL_PCT = getenv("TC_MSM_TAIL_PCT") ? (uint32_t)atoi(getenv("TC_MSM_TAIL_PCT")) : 0u;
    const uint32_t tail = TAIL_PCT ? (uint32_t)((uint64_t)nb * (100 - std::min(TAIL_PCT, 100u)) / 100) : nb;
    const uint32_t Ts = std::max<uint32_t>(4u, T / 4);
    L0.tail = tail;
    L0.Ts = Ts;
    k_count0<<<blocks_for((uint64_t)nb + 1, 256), 256, 0, st>>>(bstart, bend, nb, T, tail, Ts, L0.np, L0.npm,
                                                                L0.buckets);
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(L0.d_scan, L0.scan_bytes, L0.np, L0.toff, (int)(nb + 1), st));
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(L0.d_scan, L0.scan_bytes, L0.npm, L0.offA, (int)(nb + 1), st));
    ctx->launches += 4;
    if (ctx->prof) TC_CUDA(ctx, cudaEventRecord(ctx->ev[0], st));
    // pieces <= sum_k ceil(size_k / T_k) <= E / min(T_k) + nb; surplus threads exit
    const uint32_t Tmin = tail < nb ? Ts : T;
    L0.Tmin = Tmin;
    k_accum_aff<<<blocks_for((E_plan + Tmin - 1) / Tmin + nb, 128), 128, 0, st>>>(svals, bases, bstart, bend, L0.toff,
                                                                              L0.offA, nb, T, tail, Ts, L0.itemsA,
                                                                              L0.buckets, d_boff, P.nbm);
    TC_LAUNCHED(ctx);
    if (ctx->prof) TC_CUDA(ctx, cudaEventRecord(ctx->ev[1], st));
    return TC_OK;
  };
  // counting-sort layout: count, scan, scatter (no keys stored, no radix passes)
  uint32_t *cnt, *cursor;
  static const uint32_t NC_ENV = getenv("TC_MSM_NC") ? (uint32_t)atoi(getenv("TC_MSM_NC")) : 16u;   // sweep: 1 9.04, 4 7.79, 8 7.53, 16 7.40, 32 7.37 ms
  // mode 1 with block-private counters (k_fpb_pass) when one MSM's counters fit twice per
  // SM in shared memory; otherwise NC interleaved counter copies spread the global atomics
  static const bool no_blk = getenv("TC_MSM_NO_BLKCNT") != nullptr;
  static const uint32_t FPB_LG_ENV = getenv("TC_MSM_FPB_LG") ? (uint32_t)atoi(getenv("TC_MSM_FPB_LG")) : 8u;
  const size_t blk_smem = (size_t)P.nbm * sizeof(uint32_t);
  // ... and when one MSM's entries (4 B each) fit in L2 with room to spare: the scatter's
  // short per-(chunk, bucket) runs must stay in L2 until their sectors fill (config 5,
  // 168 MB of entries per MSM: 157.7 ms with block counters vs 138.4 ms without)
  // (mode 3: 2^mb - 1 buckets per MSM, so every (chunk, bucket) run is long and fills its
  // sectors quickly whatever the MSM size)
  // mode 2 (fixed-base digit windows of canonical scalars): block-private counters and
  // cursors over 2^(c-1) buckets (TC_MSM_NO_FB_SCATTER: the global-cursor scatter)
  static const bool no_fbs = getenv("TC_MSM_NO_FB_SCATTER") != nullptr;
  const bool fbs = P.mode == 2 && dtype == TC_DTYPE_FP_LIMBS && !no_fbs && blk_smem <= 64 * 1024 &&
                   n >= (1u << 14) && (uint64_t)n * P.ndig < (1ull << 31);
  const bool blkcnt = P.mode == 3 || fbs ||
                      (P.mode == 1 && vec_ok && !no_blk && blk_smem <= 100 * 1024 && n >= (1u << 16) &&
                       n * sizeof(uint32_t) <= (16ull << 20) && dtype != TC_DTYPE_F32);
  if (blkcnt) {
    // S chunks per MSM so that one scatter launch (LG MSMs) is about one wave of 2 blocks/SM
    // LG MSMs per scatter launch: their entries (LG n 4 B) stay within 64 MB of L2
    const uint64_t ent_per_msm = n * (P.mode == 2 ? (uint64_t)P.ndig : 1ull);
    const uint32_t LG = P.mode == 3 ? std::max(1u, std::min(getenv("TC_MSM_FPB_LG") ? FPB_LG_ENV : (uint32_t)L,
                                                            (uint32_t)L))
                                    : std::max<uint32_t>(1u, std::min(std::min(FPB_LG_ENV, (uint32_t)L),
                                                                      (uint32_t)((64ull << 20) / (ent_per_msm * sizeof(uint32_t)))));
    const uint64_t conc = (uint64_t)ctx->num_sms * 2;
    const uint64_t step = std::max<uint64_t>(1024ull * V_EPT, (uint64_t)FPS_SLICE);   // chunks hold whole slices
    const uint64_t S0 = std::max<uint64_t>(1, std::min<uint64_t>(conc / LG, n / step));
    const uint64_t chunk = ((n + S0 - 1) / S0 + step - 1) / step * step;
    const uint32_t Sx = (uint32_t)((n + chunk - 1) / chunk);
    if (fbs) {
      TC_TRY(func_smem(ctx, (const void*)k_count_fb<true>, 64 * 1024));
      TC_TRY(func_smem(ctx, (const void*)k_scatter_fb, 64 * 1024));
    }
    TC_TRY(func_smem(ctx, (const void*)k_fpb_pass<1, false>, 100 * 1024));
    TC_TRY(func_smem(ctx, (const void*)k_fpb_pass<1, true>, 100 * 1024));
    TC_TRY(func_smem(ctx, (const void*)k_fpb_pass<2, false>, 100 * 1024));
    TC_TRY(func_smem(ctx, (const void*)k_fpb_pass<2, true>, 100 * 1024));
    uint32_t *runs, *tot;
    TC_TRY(scratch_t(ctx, "msm.fpbruns", (uint64_t)nb * Sx, &runs));
    TC_TRY(scratch_t(ctx, "msm.bcount", (uint64_t)nb + 1, &tot));
    TC_TRY(scratch_t(ctx, "msm.bstart", (uint64_t)nb + 1, &bstart));
    TC_CUDA(ctx, cudaMemsetAsync(tot + nb, 0, sizeof(uint32_t), st));
    if (getenv("TC_MSM_DEBUG"))
      fprintf(stderr, "[tc msm] L=%d n=%llu mode=%d (block counters: %u chunks x %llu) groups=%d buckets/msm=%u\n", L,
              (unsigned long long)n, P.mode, Sx, (unsigned long long)chunk, P.nwin, P.nbm);
    static const bool no_sorted = getenv("TC_MSM_NO_SORTED_SCATTER") != nullptr;
    const bool sorted = P.mode == 3 && !no_sorted;
    const size_t fps_smem = (2 * 2048 + 32) * sizeof(uint32_t) + FPS_SLICE * sizeof(uint2);
    if (sorted) {
      TC_TRY(func_smem(ctx, (const void*)k_fpb_scatter_sorted<1>, (int)fps_smem));
      TC_TRY(func_smem(ctx, (const void*)k_fpb_scatter_sorted<2>, (int)fps_smem));
    }
    // the fp16 key table pays in the ALU-bound count pass (131 -> 100 us on config 3) but not
    // in the barrier-bound slice-sorted scatter (366 -> 458 us: its key phase is latency
    // bound and the table load adds to it), which keeps the branchy key3 path
    WinPlan Pns = P;
    Pns.ktab = nullptr;
    auto pass = [&](bool scatter, uint32_t l0, uint32_t nl) {
      if (fbs) {
        if (scatter)
          k_scatter_fb<<<dim3(Sx, nl), 1024, blk_smem, st>>>(d_ptrs, n, P, runs, vals, chunk, l0);
        else
          k_count_fb<true><<<dim3(Sx, nl), 1024, blk_smem, st>>>(d_ptrs, n, P, runs, chunk);
        return;
      }
      if (scatter && sorted) {
        if (dtype == TC_DTYPE_F16)
          k_fpb_scatter_sorted<1><<<dim3(Sx, nl), FPS_THREADS, fps_smem, st>>>(d_ptrs, n, scale_bits, Pns, runs, vals,
                                                                               chunk, l0);
        else
          k_fpb_scatter_sorted<2><<<dim3(Sx, nl), FPS_THREADS, fps_smem, st>>>(d_ptrs, n, scale_bits, Pns, runs, vals,
                                                                               chunk, l0);
        return;
      }
      if (dtype == TC_DTYPE_F16) {
        if (scatter)
          k_fpb_pass<1, true><<<dim3(Sx, nl), TC_FPB_THREADS, blk_smem, st>>>(d_ptrs, n, scale_bits, P, runs, vals, chunk, l0,
                                                                     nullptr);
        else
          k_fpb_pass<1, false><<<dim3(Sx, nl), TC_FPB_THREADS, blk_smem, st>>>(d_ptrs, n, scale_bits, P, runs, vals, chunk, l0,
                                                                      spec_tab ? d_small : nullptr);
      } else {
        if (scatter)
          k_fpb_pass<2, true><<<dim3(Sx, nl), TC_FPB_THREADS, blk_smem, st>>>(d_ptrs, n, scale_bits, P, runs, vals, chunk, l0,
                                                                     nullptr);
        else
          k_fpb_pass<2, false><<<dim3(Sx, nl), TC_FPB_THREADS, blk_smem, st>>>(d_ptrs, n, scale_bits, P, runs, vals, chunk, l0,
                                                                      nullptr);
      }
    };
    pass(false, 0, (uint32_t)L);
    TC_LAUNCHED(ctx);
    k_fpb_totals<<<blocks_for(nb, 256), 256, 0, st>>>(runs, P.nbm, (uint32_t)L, Sx, tot);
    TC_LAUNCHED(ctx);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, tot, bstart, (int)(nb + 1), st);
    void* d_sb;
    TC_TRY(scratch(ctx, "msm.scantmp0", sb, &d_sb));
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_sb, sb, tot, bstart, (int)(nb + 1), st));
    ctx->launches += 2;
    k_fpb_starts<<<blocks_for(nb, 256), 256, 0, st>>>(runs, P.nbm, (uint32_t)L, Sx, bstart);
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cudaMemcpyAsync(h_small, bstart + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    k_max_bucket<<<blocks_for(nb, 256), 256, 0, st>>>(bstart, nb, d_small + NHIST + 3);   // zeroed with d_small
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cudaMemcpyAsync(h_small + 1, d_small + NHIST + 3, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    if (spec_tab)   // the fused scan's flags, checked after the synchronisation below
      TC_CUDA(ctx, cudaMemcpyAsync(h_small + 2, d_small, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    have_maxb = true;
    for (uint32_t l0 = 0; l0 < (uint32_t)L; l0 += LG) {
      pass(true, l0, std::min<uint32_t>(LG, (uint32_t)L - l0));
      TC_LAUNCHED(ctx);
    }
    svals = vals;
    bend = bstart + 1;
    static const bool no_early = getenv("TC_MSM_NO_EARLY0") != nullptr;
    if (!no_early && P.mode != 2 && n * (uint64_t)L < (1ull << 31)) {   // every element at most one entry (modes 1 / 3)
      // the host waits for the entry count / largest bucket (an event after the scatter),
      // NOT for the accumulation queued behind it
      if (!ctx->ev_mid) TC_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_mid, cudaEventDisableTiming));
      TC_CUDA(ctx, cudaEventRecord(ctx->ev_mid, st));
      TC_TRY(level0((uint64_t)L * n));
      early0 = true;
      TC_CUDA(ctx, cudaEventSynchronize(ctx->ev_mid));
    } else {
      TC_CUDA(ctx, cudaStreamSynchronize(st));
    }
    E = h_small[0];
    maxb = h_small[1];
    if (spec_tab) TC_TRY(quantize_flags_to_status(ctx, h_small[2]));
  } else {
  const uint32_t NC = P.mode == 1 ? std::max(1u, NC_ENV) : 1u;
  const uint64_t ncnt = (uint64_t)nb * NC + 1;
  if (ncnt >= (1ull << 31)) return fail(ctx, TC_ERR_VALUE, "msm: too many bucket counters");
  uint32_t* S;
  TC_TRY(scratch_t(ctx, "msm.bcount", ncnt, &cnt));
  TC_TRY(scratch_t(ctx, "msm.bstart", (uint64_t)nb + 1, &bstart));
  TC_TRY(scratch_t(ctx, "msm.cursor", ncnt, &cursor));
  if (NC > 1) {
    TC_TRY(scratch_t(ctx, "msm.bscan", ncnt, &S));
  } else {
    S = bstart;
  }
  TC_CUDA(ctx, cudaMemsetAsync(cnt, 0, ncnt * sizeof(uint32_t), st));
  // fast path (k_digits_v) for fp16 / bf16 / fp32 with magnitudes below 2^62 and at most
  // HOT_MAXW few-bucket windows; the generic kernel otherwise
  HotPlan H{};
  H.nhot = 0;
  H.nhotb = 0;
  bool fast = vec_ok;
  for (int w = 0; w < MAXW; w++) H.slot[w] = -1;
  for (int w = 0; w < P.nwin && P.mode == 0; w++) {
    H.slot[w] = -1;
    const uint32_t nbw = 1u << (P.width[w] - 1);
    if (nbw <= HOT_BUCKETS) {
      if (H.nhot == HOT_MAXW || H.nhotb + nbw > HOT_MAXB) {
        fast = false;
        continue;
      }
      H.slot[w] = (int8_t)H.nhot;
      H.win[H.nhot] = (uint8_t)w;
      H.hbase[H.nhot] = (uint16_t)H.nhotb;
      H.nhotb += nbw;
      H.nhot++;
    }
  }
  if (P.mode == 1 && !fast) return fail(ctx, TC_ERR_VALUE, "msm: float-exponent plan needs the vector path");
  if (getenv("TC_MSM_DEBUG"))
    fprintf(stderr, "[tc msm] L=%d n=%llu mode=%d groups=%d buckets/msm=%u\n", L, (unsigned long long)n, P.mode,
            P.nwin, P.nbm);
  const unsigned gxv = blocks_for(n, 256 * V_EPT);
  const unsigned gx = std::min<unsigned>(blocks_for(n, 256), std::max(1u, (unsigned)ctx->num_sms * 16 / (unsigned)L + 1));
  TC_TRY(func_smem(ctx, (const void*)k_count_fb<false>, 64 * 1024));
  int s = dispatch_dt(ctx, dtype, [&](auto dt) {
    constexpr int D = decltype(dt)::value;
    if constexpr (D >= 1 && D <= 3) {
      if (fast) {
        if (P.mode == 1) {
          k_digits_fp<D, false><<<dim3(gxv, L), 256, 0, st>>>(d_ptrs, n, scale_bits, P, cnt, nullptr, NC);
        } else {
          k_digits_v<D, false><<<dim3(gxv, L), 256, 0, st>>>(d_ptrs, n, scale_bits, P, H, cnt, nullptr, NC);
        }
        return;
      }
    }
    static const bool no_fbc = getenv("TC_MSM_NO_FB_BLKCNT") != nullptr;
    if (D == DT_LIMBS && P.mode == 2 && NC == 1 && !no_fbc && P.nbm * sizeof(uint32_t) <= 64 * 1024) {
      // block-private counters: chunks of >= 16 K scalars, about two waves of 1024 threads
      const uint64_t conc = (uint64_t)ctx->num_sms * 3;
      const uint64_t S = std::max<uint64_t>(1, std::min<uint64_t>((conc + L - 1) / (uint64_t)L, n >> 14));
      const uint64_t chunk = (n + S - 1) / S;
      k_count_fb<false><<<dim3((unsigned)((n + chunk - 1) / chunk), L), 1024, P.nbm * sizeof(uint32_t), st>>>(
          d_ptrs, n, P, cnt, chunk);
      return;
    }
    k_count_digits<D, false><<<dim3(gx, L), 256, 0, st>>>(d_ptrs, n, scale_bits, P, cnt, nullptr);
  });
  if (s) return s;
  TC_LAUNCHED(ctx);
  size_t sb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sb, cnt, S, (int)ncnt, st);
  void* d_sb;
  TC_TRY(scratch(ctx, "msm.scantmp0", sb, &d_sb));
  TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_sb, sb, cnt, S, (int)ncnt, st));
  ctx->launches += 2;
  if (NC > 1) {
    k_copy_starts<<<blocks_for((uint64_t)nb + 1, 256), 256, 0, st>>>(S, nb, NC, bstart);
    TC_LAUNCHED(ctx);
  }
  TC_CUDA(ctx, cudaMemcpyAsync(cursor, S, ncnt * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  TC_CUDA(ctx, cudaMemcpyAsync(h_small, S + (ncnt - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  k_max_bucket<<<blocks_for(nb, 256), 256, 0, st>>>(bstart, nb, d_small + NHIST + 3);   // zeroed with d_small
  TC_LAUNCHED(ctx);
  TC_CUDA(ctx, cudaMemcpyAsync(h_small + 1, d_small + NHIST + 3, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  have_maxb = true;
  s = dispatch_dt(ctx, dtype, [&](auto dt) {
    constexpr int D = decltype(dt)::value;
    if constexpr (D >= 1 && D <= 3) {
      if (fast) {
        if (P.mode == 1)
          k_digits_fp<D, true><<<dim3(gxv, L), 256, 0, st>>>(d_ptrs, n, scale_bits, P, cursor, vals, NC);
        else
          k_digits_v<D, true><<<dim3(gxv, L), 256, 0, st>>>(d_ptrs, n, scale_bits, P, H, cursor, vals, NC);
        return;
      }
    }
    k_count_digits<D, true><<<dim3(gx, L), 256, 0, st>>>(d_ptrs, n, scale_bits, P, cursor, vals);
  });
  if (s) return s;
  TC_LAUNCHED(ctx);
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  E = h_small[0];
  maxb = h_small[1];
  }   // counting layout with global counters
  if (E == 0) {
    k_fill_inf<<<blocks_for(L, 64), 64, 0, st>>>(d_out, (uint32_t)L);
    TC_LAUNCHED(ctx);
    return TC_OK;
  }
  svals = vals;
  bend = bstart + 1;

  // 6. levels (a bucket holds <= n entries); level 0 may already be queued (early0)
  if (!early0) TC_TRY(level0(E));
  if (ctx->tail_split && ctx->tail_stream && ctx->stream != ctx->tail_stream) {
    // the rest of this forward on the context's low-priority tail stream (tc_ctx::tail_split)
    if (!ctx->ev_tail) TC_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_tail, cudaEventDisableTiming));
    TC_CUDA(ctx, cudaEventRecord(ctx->ev_tail, st));
    TC_CUDA(ctx, cudaStreamWaitEvent(ctx->tail_stream, ctx->ev_tail, 0));
    ctx->main_stream = ctx->stream;
    ctx->stream = ctx->tail_stream;
    st = ctx->tail_stream;
  }
  if (ctx->prof) {
    TC_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    TC_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
    auto& st_ = ctx->stats["msm.accumulate"];
    st_.ms += ms;
    st_.launches += 1;
    st_.units += (double)E;   // bucket entries accumulated
  }
  int levels = 1;   // enough for the largest bucket (<= n entries when its size is unknown)
  // the shortest pieces (tail buckets) leave the most items per bucket
  for (uint64_t capT = L0.Tmin; capT < (have_maxb ? (uint64_t)maxb : n); capT *= L0.T1) levels++;
  const uint32_t T1 = L0.T1;
  const uint64_t max_items = L0.max_items;
  uint32_t *np = L0.np, *npm = L0.npm, *toff = L0.toff, *offA = L0.offA, *offB = L0.offB;
  Ext *itemsA = L0.itemsA, *itemsB = L0.itemsB, *buckets = L0.buckets;
  void* d_scan = L0.d_scan;
  size_t scan_bytes = L0.scan_bytes;
  uint64_t items_bound = max_items;
  for (int lv = 1; lv < levels; lv++) {
    k_count<<<blocks_for((uint64_t)nb + 1, 256), 256, 0, st>>>(offA, nb, T1, np, npm);
    TC_LAUNCHED(ctx);
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, np, toff, (int)(nb + 1), st));
    TC_CUDA(ctx, cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, npm, offB, (int)(nb + 1), st));
    ctx->launches += 4;
    // every piece holds >= 1 item, and a multi-piece bucket of c >= 2 items yields
    // ceil(c/T1) <= c items: both threads and the next level's items are <= items_bound
    const unsigned gext = (unsigned)std::min<uint64_t>(blocks_for(items_bound, 128), (uint64_t)ctx->num_sms * 16);
    k_accum_ext<<<gext, 128, 0, st>>>(itemsA, offA, toff, offB, nb, T1, itemsB, buckets);
    TC_LAUNCHED(ctx);
    std::swap(offA, offB);
    std::swap(itemsA, itemsB);
  }

  // 7-8. bucket reduction, window sums, Horner, affine
  const uint32_t nw_total = (uint32_t)L * P.nwin;
  static const uint32_t SEG_LG = getenv("TC_MSM_SEG_LG") ? (uint32_t)atoi(getenv("TC_MSM_SEG_LG")) : 3u;
  const uint32_t SEG = 1u << SEG_LG;
  uint32_t maxw = 0;
  for (int w = 0; w < P.nwin; w++) maxw = std::max(maxw, P.base[w + 1] - P.base[w]);
  static const bool no_block = getenv("TC_MSM_NO_WSUM_BLOCK") != nullptr;
  // latency-bound small batches (multi-GPU ranks, openings): one block per window; large
  // batches keep the level recursion, which has more parallelism (measured: 4 layers
  // 1.58 -> 1.51 ms per step, 32 layers 7.01 -> 7.11 ms with the block kernel)
  static const uint32_t WB_MAXG = getenv("TC_WB_MAXG") ? (uint32_t)atoi(getenv("TC_WB_MAXG")) : 256u;
  if (!no_block && maxw <= (uint32_t)WB_THREADS << WB_CHUNK_LG && nw_total <= WB_MAXG) {
    Ext* wsum;
    TC_TRY(scratch_t(ctx, "msm.wsum", nw_total, &wsum));
    const size_t smem = 2 * WB_THREADS * sizeof(Ext);
    if (smem > 48 * 1024)
      TC_TRY(func_smem(ctx, (const void*)k_wsum_block, (int)smem));
    const bool prescale = P.off[P.nwin - 1] <= 32;
    k_wsum_block<<<nw_total, WB_THREADS, smem, st>>>(buckets, P, wsum, prescale ? 1 : 0);
    TC_LAUNCHED(ctx);
    if (prescale && ctx->defer_req) {
      // the caller (commit + tree) sums the windows and converts to affine inside its own
      // fused tail kernel: hand over the prescaled window sums instead of the points
      ctx->defer_wsum = wsum;
      ctx->defer_nwin = P.nwin;
      ctx->defer_L = L;
      return TC_OK;
    }
    if (prescale)
      k_final_sum<<<blocks_for((uint64_t)L * 32, 128), 128, 0, st>>>(wsum, (uint32_t)L, P.nwin, d_out);
    else
      k_final<<<blocks_for(L, 32), 32, 0, st>>>(wsum, (uint32_t)L, P, d_out);
    TC_LAUNCHED(ctx);
    return TC_OK;
  }
  // recursive segmentation (k_wsum_level): host builds all level tables, one upload
  std::vector<uint32_t> wcnt(nw_total), off(nw_total);
  for (uint32_t g = 0; g < nw_total; g++) {
    const uint32_t l = g / P.nwin, w = g % P.nwin;
    wcnt[g] = P.base[w + 1] - P.base[w];
    off[g] = l * P.nbm + P.base[w];
  }
  std::vector<uint32_t> tabs;   // per level: in_off[ng], in_cnt[ng], out_off[ng+1]
  std::vector<uint32_t> totals;
  bool more = true;
  while (more) {
    std::vector<uint32_t> oo(nw_total + 1);
    uint32_t acc = 0;
    more = false;
    for (uint32_t g = 0; g < nw_total; g++) {
      oo[g] = acc;
      const uint32_t k = (wcnt[g] + SEG - 1) / SEG;
      acc += k;
      if (k > 1) more = true;
    }
    oo[nw_total] = acc;
    tabs.insert(tabs.end(), off.begin(), off.end());
    tabs.insert(tabs.end(), wcnt.begin(), wcnt.end());
    tabs.insert(tabs.end(), oo.begin(), oo.end());
    totals.push_back(acc);
    for (uint32_t g = 0; g < nw_total; g++) {
      off[g] = oo[g];
      wcnt[g] = oo[g + 1] - oo[g];
    }
  }
  const uint32_t R = (uint32_t)totals.size();
  if (R > 9) return fail(ctx, TC_ERR_VALUE, "msm: bucket window too large (%u levels)", R);   // SEG^R fits 32 bits
  const size_t tab_bytes = tabs.size() * sizeof(uint32_t);
  const size_t stage_off = 256 * 1024;
  uint32_t* d_tabs;
  TC_TRY(scratch_t(ctx, "msm.wtabs", tabs.size(), &d_tabs));
  if (tab_bytes + stage_off <= ctx->h_stage_bytes) {
    memcpy((char*)ctx->h_stage + stage_off, tabs.data(), tab_bytes);
    TC_CUDA(ctx, cudaMemcpyAsync(d_tabs, (char*)ctx->h_stage + stage_off, tab_bytes, cudaMemcpyHostToDevice, st));
  } else {   // very large batches: pageable, synchronous
    TC_CUDA(ctx, cudaMemcpy(d_tabs, tabs.data(), tab_bytes, cudaMemcpyHostToDevice));
  }
  Ext *TA, *TB, *DA, *DB, *wsum;
  TC_TRY(scratch_t(ctx, "msm.wTA", totals[0] + 1, &TA));
  TC_TRY(scratch_t(ctx, "msm.wTB", totals[0] + 1, &TB));
  TC_TRY(scratch_t(ctx, "msm.wDA", totals[0] + 1, &DA));
  TC_TRY(scratch_t(ctx, "msm.wDB", totals[0] + 1, &DB));
  TC_TRY(scratch_t(ctx, "msm.wsum", nw_total, &wsum));
  const uint32_t stride = 3 * nw_total + 1;
  const Ext* Tin = buckets;
  const Ext* Din = nullptr;
  for (uint32_t r = 0; r < R; r++) {
    GroupTab G{d_tabs + r * stride, d_tabs + r * stride + nw_total, d_tabs + r * stride + 2 * nw_total, nw_total};
    Ext* To = (r & 1) ? TB : TA;
    Ext* Do = (r & 1) ? DB : DA;
    k_wsum_level<<<blocks_for(totals[r], 128), 128, 0, st>>>(Tin, Din, G, totals[r], SEG_LG * r, SEG, To, Do);
    TC_LAUNCHED(ctx);
    Tin = To;
    Din = Do;
  }
  uint64_t p8 = 1;
  for (uint32_t r = 0; r < R; r++) p8 *= SEG;
  const uint32_t c = (uint32_t)((p8 - SEG) / (SEG - 1));
  k_wsum_final<<<blocks_for(nw_total, 64), 64, 0, st>>>(Tin, Din, nw_total, c, P, wsum);
  TC_LAUNCHED(ctx);
  k_final<<<blocks_for(L, 32), 32, 0, st>>>(wsum, (uint32_t)L, P, d_out);
  TC_LAUNCHED(ctx);
  // the table upload reads h_stage asynchronously: finish before it can be reused
  TC_CUDA(ctx, cudaStreamSynchronize(st));
  return TC_OK;
}

int msm_device(tc_ctx* ctx, ScalarKind kind, const void* d_scalars, const EdPk* d_bases, uint64_t n, Aff* d_out) {
  if (kind != SCALAR_FP_CANON) return fail(ctx, TC_ERR_ARGUMENT, "msm: scalar kind");
  const void* ptrs[1] = {d_scalars};
  return msm_batch_device(ctx, TC_DTYPE_FP_LIMBS, 0, ptrs, 1, d_bases, n, d_out);
}

}  // namespace tcrt
