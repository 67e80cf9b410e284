// K2 / K4: the polynomial side of the prover on the device.
//
// interpolate_device  — mvpoly.interpolate_lagrange (mvpoly.py:233-247): for each axis j the
//   d_j x d_j matrix B_j (column l = monomial coefficients of the l-th Lagrange basis
//   polynomial on nodes 1..d_j, mvpoly.py:193-218) is applied to every fibre along axis j
//   (mvpoly.py:168-186).  Axes with <= 128 nodes and enough fibres take the Newton form
//   instead (k_interp_newton / k_interp_newton_w: forward differences, d divisions by k!,
//   basis expansion by small-integer multiply-subtracts with the sparse-p fold) — the same
//   unique interpolant at ~8x fewer wide multiplies.  Otherwise (k_interp_axis) a block
//   stages FB whole fibres in shared memory; each output coefficient is a length-d_j dot
//   product accumulated as full 384-bit products and Montgomery-reduced ONCE
//   (sum < 4 d p^2 < p R for d < 2^28), so a MAC costs the 6x6 product only.  B_j is kept
//   in Montgomery form and the samples canonical, so the reduction lands directly on
//   canonical coefficients.
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

// a * s mod p for a < 2p, s < 2^20, canonical result.  p = 2^161 + 2^24 + 1 is sparse:
// t = hi 2^161 + lo  ==  lo - hi (2^24 + 1)  with lo < 2^161 < p and hi (2^24+1) < 2^45,
// so one borrow-corrected subtraction lands in [0, p) — 6 IMAD.WIDE and no Montgomery step.
__device__ __forceinline__ Fe fp_mul_u32(const Fe& a, uint32_t s) {
  uint32_t t[6];
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < 6; i++) {
    c += (uint64_t)a.v[i] * s;
    t[i] = (uint32_t)c;
    c >>= 32;
  }
  const uint32_t hi = t[5] >> 1;
  const uint64_t h = (uint64_t)hi * 0x1000001ull;
  Fe r;
  uint32_t br;
  asm("sub.cc.u32  %0, %7, %13;\n\t"
      "subc.cc.u32 %1, %8, %14;\n\t"
      "subc.cc.u32 %2, %9, 0;\n\t"
      "subc.cc.u32 %3, %10, 0;\n\t"
      "subc.cc.u32 %4, %11, 0;\n\t"
      "subc.cc.u32 %5, %12, 0;\n\t"
      "subc.u32    %6, 0, 0;\n\t"
      : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(br)
      : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5] & 1u), "r"((uint32_t)h),
        "r"((uint32_t)(h >> 32)));
  const uint32_t k0 = br ? FpParams::M0 : 0u, k5 = br ? FpParams::M5 : 0u;
  asm("add.cc.u32  %0, %0, %6;\n\t"
      "addc.cc.u32 %1, %1, 0;\n\t"
      "addc.cc.u32 %2, %2, 0;\n\t"
      "addc.cc.u32 %3, %3, 0;\n\t"
      "addc.cc.u32 %4, %4, 0;\n\t"
      "addc.u32    %5, %5, %7;\n\t"
      : "+r"(r.v[0]), "+r"(r.v[1]), "+r"(r.v[2]), "+r"(r.v[3]), "+r"(r.v[4]), "+r"(r.v[5])
      : "r"(k0), "r"(k5));
  return r;
}

// Newton-form interpolation on the nodes 1..d, one thread per fibre (d <= 32): forward
// differences (d^2/2 subtractions), c_k = Delta^k y_0 / k! (d Montgomery products), then
// the Newton basis prod_{j<k} (X - (j+1)) is expanded to monomials in place
// (d^2/2 multiply-by-small-integer subtractions, fp_mul_u32).  ~8x fewer IMAD.WIDE than
// the dense d x d matrix (k_interp_axis) and the same unique interpolant, so the output is
// bit-identical.  Fibres are staged in shared memory limb-major (SoA, padded pitch FB + 1)
// so the per-thread sweeps are bank-conflict free.
template <int FB>
__global__ void __launch_bounds__(FB) k_interp_newton(Fe* data, const Fe* invfact, uint32_t d, uint64_t stride,
                                                      uint64_t nfib) {
  extern __shared__ uint32_t sw[];
  constexpr uint32_t P = FB + 1;
  const uint64_t f0 = (uint64_t)blockIdx.x * FB;
  const uint32_t nloc = (nfib - f0 < FB) ? (uint32_t)(nfib - f0) : FB;
  const uint32_t tot = nloc * d;
  const bool contiguous = (stride == 1);
  for (uint32_t idx = threadIdx.x; idx < tot; idx += FB) {
    uint32_t fl, l;
    if (contiguous) {
      fl = idx / d;
      l = idx - fl * d;
    } else {
      l = idx / nloc;
      fl = idx - l * nloc;
    }
    const Fe x = data[fibre_addr(f0 + fl, l, d, stride)];
#pragma unroll
    for (int i = 0; i < 6; i++) sw[(l * 6 + i) * P + fl] = x.v[i];
  }
  __syncthreads();
  const uint32_t fl = threadIdx.x;
  auto LD = [&](uint32_t l) {
    Fe r;
#pragma unroll
    for (int i = 0; i < 6; i++) r.v[i] = sw[(l * 6 + i) * P + fl];
    return r;
  };
  auto ST = [&](uint32_t l, const Fe& x) {
#pragma unroll
    for (int i = 0; i < 6; i++) sw[(l * 6 + i) * P + fl] = x.v[i];
  };
  if (fl < nloc) {
    // v[k] <- Delta^k y_0 (descending sweeps keep v[j-1] un-updated when v[j] is)
    for (uint32_t k = 1; k < d; k++) {
      Fe hi = LD(d - 1);
#pragma unroll 4
      for (uint32_t j = d - 1; j >= k; j--) {
        const Fe lo = LD(j - 1);
        ST(j, Fp::sub(hi, lo));
        hi = lo;
      }
    }
    for (uint32_t k = 2; k < d; k++) ST(k, Fp::mul(LD(k), invfact[k]));
    // Horner on the Newton form: a <- a (X - (k+1)) + c_k, coefficients in v[k..d)
    for (int k = (int)d - 2; k >= 0; k--) {
      const uint32_t s = (uint32_t)k + 1;
      Fe cur = LD(k);
#pragma unroll 4
      for (uint32_t j = k; j + 1 < d; j++) {
        const Fe nx = LD(j + 1);
        ST(j, Fp::sub(cur, fp_mul_u32(nx, s)));
        cur = nx;
      }
    }
  }
  __syncthreads();
  for (uint32_t idx = threadIdx.x; idx < tot; idx += FB) {
    uint32_t f, l;
    if (contiguous) {
      f = idx / d;
      l = idx - f * d;
    } else {
      l = idx / nloc;
      f = idx - l * nloc;
    }
    Fe x;
#pragma unroll
    for (int i = 0; i < 6; i++) x.v[i] = sw[(l * 6 + i) * P + f];
    data[fibre_addr(f0 + f, l, d, stride)] = Fp::canon(x);
  }
}

// Two threads per fibre (adjacent lanes, same SMEM fibre layout as k_interp_newton): every
// sweep is split at its midpoint, the upper thread taking the upper half.  A sweep reads
// the OLD value across the split point, so that value is read before a __syncwarp and the
// halves then run concurrently — twice the resident threads for the same shared memory
// (the one-thread kernel is occupancy-limited by its fibres: 8 warps per SM).
template <int FB>
__global__ void __launch_bounds__(2 * FB) k_interp_newton2(Fe* data, const Fe* invfact, uint32_t d, uint64_t stride,
                                                           uint64_t nfib) {
  extern __shared__ uint32_t sw[];
  constexpr uint32_t P = FB + 1;
  const uint64_t f0 = (uint64_t)blockIdx.x * FB;
  const uint32_t nloc = (nfib - f0 < FB) ? (uint32_t)(nfib - f0) : FB;
  const uint32_t tot = nloc * d;
  const bool contiguous = (stride == 1);
  for (uint32_t idx = threadIdx.x; idx < tot; idx += 2 * FB) {
    uint32_t fl, l;
    if (contiguous) {
      fl = idx / d;
      l = idx - fl * d;
    } else {
      l = idx / nloc;
      fl = idx - l * nloc;
    }
    const Fe x = data[fibre_addr(f0 + fl, l, d, stride)];
#pragma unroll
    for (int i = 0; i < 6; i++) sw[(l * 6 + i) * P + fl] = x.v[i];
  }
  __syncthreads();
  // lanes past nloc sweep a stale column: harmless, never written back
  const uint32_t fl = threadIdx.x >> 1;
  const bool upper = (threadIdx.x & 1u) == 0;
  auto LD = [&](int l) {
    Fe r;
#pragma unroll
    for (int i = 0; i < 6; i++) r.v[i] = sw[(l * 6 + i) * P + fl];
    return r;
  };
  auto ST = [&](int l, const Fe& x) {
#pragma unroll
    for (int i = 0; i < 6; i++) sw[(l * 6 + i) * P + fl] = x.v[i];
  };
  const int D = (int)d;
  // both halves run the same code on their own range (no divergent branches inside a warp);
  // the value just outside a range is read before the __syncwarp that lets the other half
  // overwrite it.
  // forward differences: sweep k updates j = D-1 .. k (descending), v[j] -= v[j-1]
  for (int k = 1; k < D; k++) {
    const int mid = k + (D - k) / 2;
    const int lo = upper ? mid : k, hi = upper ? D - 1 : mid - 1;   // this half: j in [lo, hi]
    const Fe below = LD(lo - 1);
    __syncwarp();
    if (hi >= lo) {
      Fe top = LD(hi);
      for (int j = hi; j > lo; j--) {
        const Fe nx = LD(j - 1);
        ST(j, Fp::sub(top, nx));
        top = nx;
      }
      ST(lo, Fp::sub(top, below));
    }
    __syncwarp();
  }
  for (int k = 2 + (upper ? 0 : 1); k < D; k += 2) ST(k, Fp::mul(LD(k), invfact[k]));
  __syncwarp();
  // basis expansion: step k updates j = k .. D-2 (ascending), v[j] -= (k+1) v[j+1]
  for (int k = D - 2; k >= 0; k--) {
    const uint32_t sc = (uint32_t)k + 1;
    const int mid = k + (D - 1 - k) / 2;
    const int lo = upper ? mid : k, hi = upper ? D - 2 : mid - 1;   // j in [lo, hi]
    const Fe above = LD(hi + 1);
    __syncwarp();
    if (hi >= lo) {
      Fe cur = LD(lo);
      for (int j = lo; j < hi; j++) {
        const Fe nx = LD(j + 1);
        ST(j, Fp::sub(cur, fp_mul_u32(nx, sc)));
        cur = nx;
      }
      ST(hi, Fp::sub(cur, fp_mul_u32(above, sc)));
    }
    __syncwarp();
  }
  __syncthreads();
  for (uint32_t idx = threadIdx.x; idx < tot; idx += 2 * FB) {
    uint32_t f, l;
    if (contiguous) {
      f = idx / d;
      l = idx - f * d;
    } else {
      l = idx / nloc;
      f = idx - l * nloc;
    }
    Fe x;
#pragma unroll
    for (int i = 0; i < 6; i++) x.v[i] = sw[(l * 6 + i) * P + f];
    data[fibre_addr(f0 + f, l, d, stride)] = Fp::canon(x);
  }
}

// Warp-per-fibre variant of k_interp_newton (fibres longer than 32 nodes): element j = e*32 + lane
// of the fibre lives in lane `lane`, register slot e (E = ceil(d/32)); the difference and
// expansion sweeps shift the fibre by one node with warp shuffles, no shared memory.
__device__ __forceinline__ Fe shfl_fe(const Fe& a, int src) {
  Fe r;
#pragma unroll
  for (int i = 0; i < 6; i++) r.v[i] = __shfl_sync(0xffffffffu, a.v[i], src);
  return r;
}

template <int E>
__global__ void __launch_bounds__(256) k_interp_newton_w(Fe* data, const Fe* invfact, uint32_t d, uint64_t stride,
                                                         uint64_t nfib) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t f = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); f < nfib; f += nw) {
    Fe v[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
      const uint32_t j = e * 32 + lane;
      v[e] = (j < d) ? data[fibre_addr(f, j, d, stride)] : Fp::zero();
    }
    for (uint32_t k = 1; k < d; k++) {
      Fe prev[E];
#pragma unroll
      for (int e = 0; e < E; e++) {
        const Fe up = shfl_fe(v[e], (lane + 31) & 31);
        if (e == 0) {
          prev[e] = up;
        } else {
          const Fe top = shfl_fe(v[e > 0 ? e - 1 : 0], 31);
          prev[e] = lane ? up : top;
        }
      }
#pragma unroll
      for (int e = 0; e < E; e++) {
        const uint32_t j = e * 32 + lane;
        if (j >= k && j < d) v[e] = Fp::sub(v[e], prev[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < E; e++) {
      const uint32_t j = e * 32 + lane;
      if (j >= 2 && j < d) v[e] = Fp::mul(v[e], invfact[j]);
    }
    for (int k = (int)d - 2; k >= 0; k--) {
      Fe nx[E];
#pragma unroll
      for (int e = 0; e < E; e++) {
        const Fe dn = shfl_fe(v[e], (lane + 1) & 31);
        if (e + 1 == E) {
          nx[e] = dn;
        } else {
          const Fe bot = shfl_fe(v[e + 1 < E ? e + 1 : e], 0);
          nx[e] = (lane == 31) ? bot : dn;
        }
      }
#pragma unroll
      for (int e = 0; e < E; e++) {
        const uint32_t j = e * 32 + lane;
        if ((int)j >= k && j + 1 < d) v[e] = Fp::sub(v[e], fp_mul_u32(nx[e], (uint32_t)k + 1));
      }
    }
#pragma unroll
    for (int e = 0; e < E; e++) {
      const uint32_t j = e * 32 + lane;
      if (j < d) data[fibre_addr(f, j, d, stride)] = Fp::canon(v[e]);
    }
  }
}

// Register-blocked Newton interpolation (d a multiple of EPT, G = d / EPT <= 32): a block
// holds 32 fibres, lane = fibre; warp q keeps elements [q EPT, (q+1) EPT) of its lane's
// fibre in registers.  Each sweep step needs one neighbour element from the next-lower
// (differences) or next-higher (expansion) warp, exchanged through a double-buffered
// shared-memory slot with one barrier per step; a warp whose elements are all below the
// step's start skips the step (warp-uniform), so the triangular sweeps cost d^2/2 updates
// per fibre like the scalar form — without the shared-memory traffic of k_interp_newton2
// (12 words per update) or the lane masking of the warp-per-fibre k_interp_newton_w.
template <int EPT>
__global__ void __launch_bounds__(256) k_interp_newton_b(Fe* data, const Fe* __restrict__ invfact, uint32_t d,
                                                         uint64_t stride, uint64_t nfib) {
  extern __shared__ uint32_t sx[];   // [2][G][6][32]
  const uint32_t lane = threadIdx.x & 31, q = threadIdx.x >> 5, G = d / EPT;
  const uint64_t f = (uint64_t)blockIdx.x * 32 + lane;
  const bool live = f < nfib;
  const int j0 = (int)(q * EPT);
  Fe v[EPT];
#pragma unroll
  for (int e = 0; e < EPT; e++) v[e] = live ? data[fibre_addr(f, (uint32_t)(j0 + e), d, stride)] : Fp::zero();
  auto slot = [&](int b, uint32_t w, int i) -> uint32_t& { return sx[((b * G + w) * 6 + i) * 32 + lane]; };
  // forward differences: step k sets v[j] -= v[j-1] for j = d-1 .. k (descending)
  for (int k = 1; k < (int)d; k++) {
    const int b = k & 1;
    if (q + 1 < G && j0 + EPT >= k) {   // old top element, read by the next warp
#pragma unroll
      for (int i = 0; i < 6; i++) slot(b, q, i) = v[EPT - 1].v[i];
    }
    __syncthreads();
    if (j0 + EPT - 1 >= k) {
      Fe below;
      if (q > 0) {
#pragma unroll
        for (int i = 0; i < 6; i++) below.v[i] = slot(b, q - 1, i);
      }
      if (j0 >= k) {   // the whole range (every step but the EPT - 1 where k falls inside it)
#pragma unroll
        for (int e = EPT - 1; e >= 1; e--) v[e] = Fp::sub(v[e], v[e - 1]);
        v[0] = Fp::sub(v[0], below);
      } else {
#pragma unroll
        for (int e = EPT - 1; e >= 1; e--)
          if (j0 + e >= k) v[e] = Fp::sub(v[e], v[e - 1]);
      }
    }
  }
  // c_k = Delta^k y_0 / k!
#pragma unroll
  for (int e = 0; e < EPT; e++)
    if (j0 + e >= 2) v[e] = Fp::mul(v[e], invfact[j0 + e]);
  // Newton basis -> monomials: step k sets v[j] -= (k+1) v[j+1] for j = k .. d-2 (ascending)
  for (int k = (int)d - 2; k >= 0; k--) {
    const int b = k & 1;
    if (q > 0 && j0 - 1 >= k) {   // old bottom element, read by the previous warp
#pragma unroll
      for (int i = 0; i < 6; i++) slot(b, q, i) = v[0].v[i];
    }
    __syncthreads();
    if (j0 + EPT - 1 >= k) {
      Fe above;
      if (q + 1 < G) {
#pragma unroll
        for (int i = 0; i < 6; i++) above.v[i] = slot(b, q + 1, i);
      }
      const uint32_t sc = (uint32_t)k + 1;
      if (j0 >= k && q + 1 < G) {   // the whole range, not the fibre's top element
#pragma unroll
        for (int e = 0; e < EPT; e++) v[e] = Fp::sub(v[e], fp_mul_u32(e + 1 < EPT ? v[e + 1] : above, sc));
      } else {
#pragma unroll
        for (int e = 0; e < EPT; e++) {
          const int j = j0 + e;
          if (j >= k && j <= (int)d - 2) v[e] = Fp::sub(v[e], fp_mul_u32(e + 1 < EPT ? v[e + 1] : above, sc));
        }
      }
    }
  }
  if (live) {
#pragma unroll
    for (int e = 0; e < EPT; e++) data[fibre_addr(f, (uint32_t)(j0 + e), d, stride)] = Fp::canon(v[e]);
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
    const uint64_t nfib = n / d;
    // Newton form when there are enough fibres to fill the GPU one thread per fibre;
    // TC_INTERP_NEWTON_MIN_FIB overrides the threshold (tests force it to 1), TC_INTERP_DENSE
    // keeps the matrix kernel everywhere
    static const bool newton_off = getenv("TC_INTERP_DENSE") != nullptr;
    static const uint64_t newton_min =
        getenv("TC_INTERP_NEWTON_MIN_FIB") ? strtoull(getenv("TC_INTERP_NEWTON_MIN_FIB"), nullptr, 10) : 2048;
    if (!newton_off && d <= 128 && nfib >= newton_min) {
      std::string key = "interp.invfact." + std::to_string(d);
      Fe* dIf;
      bool have = ctx->scratch.count(key + ".ready") != 0;
      TC_TRY(scratch_t(ctx, key.c_str(), (uint64_t)d, &dIf));
      if (!have) {
        std::vector<Fe> h(d);
        Fe f = Fp::one();
        for (uint32_t k = 0; k < d; k++) {
          if (k > 1) f = Fp::mul(f, Fp::to_mont_small(k));
          h[k] = Fp::inv_fast(f);
        }
        TC_CUDA(ctx, cudaMemcpyAsync(dIf, h.data(), d * sizeof(Fe), cudaMemcpyHostToDevice, st));
        TC_CUDA(ctx, cudaStreamSynchronize(st));
        ctx->scratch[key + ".ready"] = tc_ctx::Buf{};
      }
      // d <= 32: one thread per fibre (measured 267 us vs 354 us per 2^21-element axis);
      // longer fibres: one warp per fibre (500 us vs 644 us at d = 64), the SMEM footprint of
      // the thread-per-fibre kernel caps it at 4 warps per SM there
      static const bool warp_all = getenv("TC_INTERP_WARP") != nullptr;
      static const bool no_blocked = getenv("TC_INTERP_NO_BLOCKED") != nullptr;
      if (!warp_all && !no_blocked && d % 8 == 0 && d <= 32) {
        // register-blocked kernel: 8 elements per thread, d / 8 warps per 32 fibres (config 3's
        // 32-node axes: 23.4 -> 19.4 ms per forward; 4 elements per thread measured the same;
        // at 64 nodes the warp-per-fibre kernel stays ahead, 15.9 vs 16.3 ms)
        const uint32_t G = d / 8;
        k_interp_newton_b<8><<<(unsigned)((nfib + 31) / 32), 32 * G, 2 * G * 6 * 32 * sizeof(uint32_t), st>>>(
            d_vals, dIf, d, stride, nfib);
        TC_LAUNCHED(ctx);
        continue;
      }
      if (warp_all || d > 32) {
        const unsigned grid = (unsigned)std::min<uint64_t>((nfib + 7) / 8, 148ull * 8);
        if (d <= 32) k_interp_newton_w<1><<<grid, 256, 0, st>>>(d_vals, dIf, d, stride, nfib);
        else if (d <= 64) k_interp_newton_w<2><<<grid, 256, 0, st>>>(d_vals, dIf, d, stride, nfib);
        else k_interp_newton_w<4><<<grid, 256, 0, st>>>(d_vals, dIf, d, stride, nfib);
        TC_LAUNCHED(ctx);
        continue;
      }
      constexpr int FB = 64;
      const size_t smem = (size_t)(FB + 1) * d * 6 * sizeof(uint32_t);
      static const bool one_thread = getenv("TC_INTERP_NEWTON1") != nullptr;
      if (!one_thread) {
        TC_TRY(func_smem(ctx, (const void*)k_interp_newton2<FB>, (int)((FB + 1) * 128 * 6 * sizeof(uint32_t))));
        k_interp_newton2<FB><<<(unsigned)((nfib + FB - 1) / FB), 2 * FB, smem, st>>>(d_vals, dIf, d, stride, nfib);
        TC_LAUNCHED(ctx);
        continue;
      }
      TC_TRY(func_smem(ctx, (const void*)k_interp_newton<FB>, (int)((FB + 1) * 128 * 6 * sizeof(uint32_t))));
      k_interp_newton<FB><<<(unsigned)((nfib + FB - 1) / FB), FB, smem, st>>>(d_vals, dIf, d, stride, nfib);
      TC_LAUNCHED(ctx);
      continue;
    }
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
    size_t smem = (size_t)FB * d * sizeof(Fe);
    if (smem > 48 * 1024)
      TC_TRY(func_smem(ctx, (const void*)k_interp_axis, (int)smem));
    unsigned grid = (unsigned)((nfib + FB - 1) / FB);
    k_interp_axis<<<grid, 256, smem, st>>>(d_vals, dB, d, stride, nfib, FB);
    TC_LAUNCHED(ctx);
  }
  return TC_OK;
}

// r (scratch copy of the coefficients) is consumed; quotients are m x n, zero outside
// their support.  omega canonical; returns y canonical on the host.
int open_quotients_device(tc_ctx* ctx, const Fe* d_coeffs, const uint32_t* shape, int m,
                          const Fe* omega_canon, Fe* d_quotients, Fe* h_y, Fe* d_y) {
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
  if (d_y) {   // batched openings: y stays on the device, no host round trip here
    TC_CUDA(ctx, cudaMemcpyAsync(d_y, r, sizeof(Fe), cudaMemcpyDeviceToDevice, st));
    return TC_OK;
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
