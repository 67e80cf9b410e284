// FP64-pipe F_q arithmetic (csrc/field_f64.cuh): exactness against the integer Montgomery
// product (host and device), and throughput of integer-only, FP64-only and mixed warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//      -I include -o tools/fp64_bench tools/fp64_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

#include <cuda_runtime.h>

#include "field_f64.cuh"

using namespace tc;

// float-Mont <-> int-Mont constants
TC_HD FeD c_i2f() {   // 2^144 mod q as 24-bit limbs (int-Mont x*2^192 -> x*2^168)
  // 2^144 < q, so its words are exact: bit 144 -> word 4 bit 16
  Fe t{{0, 0, 0, 0, 1u << 16, 0}};
  return FqD::from_words(t);
}
TC_HD FeD c_f2i() { return FqD::from_words(Fq::one()); }   // 2^192 mod q

TC_HD Fe roundtrip_mul(const Fe& a, const Fe& b) {
  FeD A = FqD::mul(FqD::from_words(a), c_i2f());
  FeD B = FqD::mul(FqD::from_words(b), c_i2f());
  FeD P = FqD::mul(A, B);
  // a few extra operations to exercise add/sub/sqr within the invariants
  FeD S = FqD::sqr(FqD::sub(P, A));     // (P - A)^2
  FeD T = FqD::mul(FqD::add(S, B), P);  // (S + B) * P
  FeD out = FqD::mul(T, c_f2i());
  return Fq::canon(FqD::to_words_lazy(out));
}
TC_HD Fe ref_mul(const Fe& a, const Fe& b) {
  Fe P = Fq::mul(a, b);
  Fe S = Fq::sqr(Fq::sub(P, a));
  Fe T = Fq::mul(Fq::add(S, b), P);
  return Fq::canon(T);
}

__global__ void k_check(const Fe* a, const Fe* b, int n, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Fe r = roundtrip_mul(a[i], b[i]), w = ref_mul(a[i], b[i]);
  for (int k = 0; k < 6; k++)
    if (r.v[k] != w.v[k]) {
      atomicAdd(bad, 1);
      break;
    }
}

// MODE 0: all warps integer; 1: all warps FP64; 2: even warps integer, odd warps FP64
template <int MODE>
__global__ void k_thr(uint32_t* out, uint32_t seed, int iters) {
  // warp w runs on SMSP w % 4: mix the two kinds WITHIN every SMSP (warps 4..7 of a block
  // of 256, or odd blocks for 128-thread blocks)
  const bool use_f = MODE == 1 || (MODE == 2 && (blockDim.x >= 256 ? ((threadIdx.x >> 7) & 1) : (blockIdx.x & 1)));
  Fe a[4];
  for (int j = 0; j < 4; j++)
    for (int i = 0; i < 6; i++) a[j].v[i] = (seed * (i + 7 * j + 1) + threadIdx.x) & (i == 5 ? 0x7fu : 0xffffffffu);
  uint32_t s = 0;
  if (use_f) {
    FeD x[4], b = FqD::from_words(a[0]);
    for (int j = 0; j < 4; j++) x[j] = FqD::from_words(a[j]);
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int j = 0; j < 4; j++) x[j] = FqD::mul(x[j], b);
    }
    for (int j = 0; j < 4; j++) s ^= __double2loint(x[j].v[0]);
  } else {
    Fe b = a[0];
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int j = 0; j < 4; j++) a[j] = Fq::mul(a[j], b);
    }
    for (int j = 0; j < 4; j++) s ^= a[j].v[0];
  }
  if (s == 0x12345678) out[0] = s;
}

static Fe rand_fe(std::mt19937_64& g) {
  // uniform-ish in [0, 2q): top word < 0x1E0
  Fe r;
  for (int i = 0; i < 5; i++) r.v[i] = (uint32_t)g();
  r.v[5] = (uint32_t)(g() % 0x1E0);
  return r;
}

int main() {
  std::mt19937_64 g(1);
  const int n = 1 << 16;
  Fe *ha = new Fe[n], *hb = new Fe[n];
  for (int i = 0; i < n; i++) ha[i] = rand_fe(g), hb[i] = rand_fe(g);
  // edge values
  ha[0] = Fe{{0, 0, 0, 0, 0, 0}};
  ha[1] = Fe{{0x78000077u - 1, 0, 0, 0, 0, 0xF0u}};   // q - 1
  ha[2] = Fe{{0xF00000EEu - 1, 0, 0, 0, 0, 0x1E0u}};  // 2q - 1 (lazy max)
  hb[2] = ha[2];
  int host_bad = 0;
  for (int i = 0; i < 4096; i++) {
    Fe r = roundtrip_mul(ha[i], hb[i]), w = ref_mul(ha[i], hb[i]);
    for (int k = 0; k < 6; k++)
      if (r.v[k] != w.v[k]) {
        host_bad++;
        break;
      }
  }
  printf("{\"check\": \"host\", \"n\": 4096, \"bad\": %d}\n", host_bad);
  Fe *da, *db;
  int* dbad;
  cudaMalloc(&da, n * sizeof(Fe));
  cudaMalloc(&db, n * sizeof(Fe));
  cudaMalloc(&dbad, 4);
  cudaMemset(dbad, 0, 4);
  cudaMemcpy(da, ha, n * sizeof(Fe), cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, n * sizeof(Fe), cudaMemcpyHostToDevice);
  k_check<<<n / 128, 128>>>(da, db, n, dbad);
  int dev_bad = -1;
  cudaMemcpy(&dev_bad, dbad, 4, cudaMemcpyDeviceToHost);
  printf("{\"check\": \"device\", \"n\": %d, \"bad\": %d}\n", n, dev_bad);

  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 4; r++) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    return best;
  };
  for (int tpb : {128, 256}) {
    for (int bps : {4, 8}) {
      const int it = 256;
      double nm = (double)sms * bps * tpb * it * 4;
      float t0 = timeit([&] { k_thr<0><<<sms * bps, tpb>>>(out, 11, it); });
      float t1 = timeit([&] { k_thr<1><<<sms * bps, tpb>>>(out, 11, it); });
      float t2 = timeit([&] { k_thr<2><<<sms * bps, tpb>>>(out, 11, it); });
      printf("{\"tpb\": %d, \"blocks_per_sm\": %d, \"Gmulmod_int\": %.1f, \"Gmulmod_f64\": %.1f, \"Gmulmod_mixed\": %.1f}\n",
             tpb, bps, nm / t0 / 1e6, nm / t1 / 1e6, nm / t2 / 1e6);
    }
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
