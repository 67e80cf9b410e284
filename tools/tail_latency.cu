// Single-thread latency (clock64) of the pieces of the commit/tree tail on B200: F_q
// inversion, ext_to_aff, aff_encode43, hash_to_scalar (SHA-256 + mod p), ext_add.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/tail_latency tools/tail_latency.cu
#include <cstdio>
#include "../paper_2602_12630_b200/csrc/ec.cuh"
#include "../paper_2602_12630_b200/csrc/sha256.cuh"
using namespace tc;

__global__ void k_lat(uint32_t* out, long long* cyc, uint32_t seed) {
  Fe a{{seed * 7919u + 1u, seed, 3u, 4u, 5u, 0x17u}};
  Ext e{a, Fq::add(a, a), Fq::one(), a};
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < 4; i++) a = Fq::inv(a);
  long long t1 = clock64();
  Aff r;
  for (int i = 0; i < 4; i++) {
    r = ext_to_aff(e);
    e.X.v[0] ^= r.x.v[0] & 1u;
  }
  long long t2 = clock64();
  uint8_t enc[43];
  for (int i = 0; i < 4; i++) {
    aff_encode43(r, enc);
    r.x.v[1] ^= enc[5];
  }
  long long t3 = clock64();
  const uint8_t tag[] = {'t', 'e', 'r', 'k', 'l', 'e', '/', 'n', 'o', 'd', 'e'};
  Fe h{};
  for (int i = 0; i < 4; i++) {
    h = hash_to_scalar(enc, 43, tag, sizeof tag);
    enc[3] ^= (uint8_t)h.v[0];
  }
  long long t4 = clock64();
  for (int i = 0; i < 8; i++) ext_add(e, e);
  long long t5 = clock64();
  for (int i = 0; i < 4; i++) a = Fq::inv_bygcd(a);
  long long t6 = clock64();
  Fe hp{};
  for (int i = 0; i < 4; i++) {
    hp = hash_point_to_scalar(r, true);
    r.x.v[2] ^= hp.v[0] & 1u;
  }
  long long t7 = clock64();
  cyc[5] = (t6 - t5) / 4, cyc[6] = (t7 - t6) / 4;
  cyc[0] = (t1 - t0) / 4, cyc[1] = (t2 - t1) / 4, cyc[2] = (t3 - t2) / 4, cyc[3] = (t4 - t3) / 4, cyc[4] = (t5 - t4) / 8;
  out[0] = a.v[0] ^ e.X.v[0] ^ r.y.v[0] ^ h.v[1] ^ acc ^ hp.v[0];
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMallocManaged(&cyc, 7 * sizeof(long long));
  for (int r = 0; r < 3; r++) {
    k_lat<<<1, 1>>>(out, cyc, 5 + r);
    cudaDeviceSynchronize();
  }
  printf("{\"inv_fermat\": %lld, \"ext_to_aff\": %lld, \"encode43\": %lld, \"hash_to_scalar\": %lld, \"ext_add\": %lld, \"inv_safegcd\": %lld, \"hash_point\": %lld, \"err\": \"%s\"}\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
