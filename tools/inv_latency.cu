// Latency of ONE thread's F_q inversion / product / Edwards add and doubling (clock64), B200.
// Measured: Fermat inversion 49.5k cycles, mulmod 260-265, ext_add 2.4-3.1k (a single warp
// is bound by its own IMAD.WIDE issue rate: interleaving independent products did not help).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/inv_latency tools/inv_latency.cu
#include <cstdio>
#include "../paper_2602_12630_b200/csrc/ec.cuh"
using namespace tc;

__global__ void k_lat(uint32_t* out, long long* cyc, uint32_t seed) {
  Fe a{{seed * 7919u + 1u, seed, 3u, 4u, 5u, 0x17u}};
  Ext e{a, Fq::add(a, a), Fq::one(), a};
  long long t0 = clock64();
  for (int i = 0; i < 8; i++) a = Fq::inv(a);
  long long t1 = clock64();
  for (int i = 0; i < 16; i++) e = ext_dbl(e);
  long long t2 = clock64();
  for (int i = 0; i < 64; i++) a = Fq::mul(a, a);
  long long t3 = clock64();
  for (int i = 0; i < 16; i++) ext_add(e, e);
  long long t4 = clock64();
  cyc[0] = (t1 - t0) / 8, cyc[1] = (t2 - t1) / 16, cyc[2] = (t3 - t2) / 64, cyc[3] = (t4 - t3) / 16;
  out[0] = a.v[0] ^ e.X.v[0];
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMallocManaged(&cyc, 4 * sizeof(long long));
  for (int r = 0; r < 3; r++) {
    k_lat<<<1, 1>>>(out, cyc, 5 + r);
    cudaDeviceSynchronize();
  }
  printf("{\"fermat_inv_cycles\": %lld, \"ext_dbl_latency_cycles\": %lld, \"mulmod_latency_cycles\": %lld, \"ext_add_latency_cycles\": %lld, \"err\": \"%s\"}\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
