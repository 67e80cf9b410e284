// Integer-pipe microbenchmarks on B200: mad.lo / mad.hi / mad.wide (64-bit accumulate)
// throughput, and the throughput of the library's F_q Montgomery product and XYZZ mixed add.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//      -I include -o tools/imad_peak tools/imad_peak.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "../paper_2602_12630_b200/csrc/ec.cuh"

using namespace tc;

template <int MODE>
__global__ void k_imad(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[16];
  uint64_t w[8];
  const uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = seed * (i + 1) + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) w[i] = a[i];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      if (MODE == 0) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b));
      if (MODE == 1) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b));
      if (MODE == 2 && i < 8) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"(a[i]), "r"(b));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s ^= a[i];
#pragma unroll
  for (int i = 0; i < 8; i++) s ^= w[i];
  if (s == 0x12345678) out[0] = (uint32_t)s;
}

__global__ void k_fqmul(uint32_t* out, uint32_t seed, int iters) {
  Fe a[4];
  for (int j = 0; j < 4; j++)
    for (int i = 0; i < 6; i++) a[j].v[i] = (seed * (i + 7 * j + 1) + threadIdx.x) & (i == 5 ? 0xffu : 0xffffffffu);
  Fe b = a[0];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++) a[j] = Fq::mul(a[j], b);
  }
  uint32_t s = 0;
  for (int j = 0; j < 4; j++) s ^= a[j].v[0];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_madd(uint32_t* out, const Aff* pts, int npts, int iters) {
  Xyzz acc = xyzz_inf();
  int idx = (blockIdx.x * blockDim.x + threadIdx.x) % npts;
  for (int it = 0; it < iters; it++) {
    xyzz_add_aff(acc, pts[idx]);
    idx = (idx + 1) % npts;
  }
  if (acc.X.v[0] == 0x12345678) out[0] = acc.X.v[1];
}

// FP64 pipe: independent DFMA chains; MODE 1 mixes 8 DFMA + 8 IMAD chains to see whether
// the two pipes issue concurrently (a hybrid integer/float multiprecision design needs it).
template <int MODE>
__global__ void k_dfma(uint32_t* out, double seed, int iters) {
  double d[16];
  uint32_t a[8];
  const double b = seed * 1.0000001 + threadIdx.x * 1e-9;
  const uint32_t bi = __double2uint_rz(seed) ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < 16; i++) d[i] = seed * (i + 1) + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = bi * (i + 3);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      if (MODE == 0 || (MODE < 4 && i < 8)) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(b));
      if (MODE == 4) {
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(a[i & 7]), "r"(bi), "l"((uint64_t)a[i & 7]));
        a[i & 7] = (uint32_t)(w >> 32) ^ (uint32_t)w;
      }
      if (MODE == 1 && i >= 8) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i - 8]) : "r"(bi));
      if (MODE == 2 && i >= 8) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[i - 8]) : "r"(bi));
      if (MODE == 3 && i >= 8) {   // dependent 32x32->64 multiply-add (IMAD.WIDE), not hoistable
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(a[i - 8]), "r"(bi), "l"((uint64_t)a[i - 8]));
        a[i - 8] = (uint32_t)(w >> 32) ^ (uint32_t)w;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += d[i];
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) t ^= a[i];
  if (s == 1.2345 || t == 0x12345678) out[0] = t;
}

int main() {
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
  const int threads = 512, blocks = sms * 4, iters = 4096;
  double n16 = (double)blocks * threads * iters * 16, n8 = n16 / 2;
  float t0 = timeit([&] { k_imad<0><<<blocks, threads>>>(out, 7, iters); });
  float t1 = timeit([&] { k_imad<1><<<blocks, threads>>>(out, 7, iters); });
  float t2 = timeit([&] { k_imad<2><<<blocks, threads>>>(out, 7, iters); });
  printf("{\"op\": \"mad.lo.u32\", \"Tops\": %.3f}\n", n16 / t0 / 1e9);
  printf("{\"op\": \"mad.hi.u32\", \"Tops\": %.3f}\n", n16 / t1 / 1e9);
  printf("{\"op\": \"mad.wide.u32 (64-bit acc)\", \"Tops\": %.3f}\n", n8 / t2 / 1e9);
  float td0 = timeit([&] { k_dfma<0><<<blocks, threads>>>(out, 0.5, iters); });
  float td1 = timeit([&] { k_dfma<1><<<blocks, threads>>>(out, 0.5, iters); });
  printf("{\"op\": \"fma.rn.f64\", \"Tops\": %.3f}\n", n16 / td0 / 1e9);
  float td2 = timeit([&] { k_dfma<2><<<blocks, threads>>>(out, 0.5, iters); });
  float td3 = timeit([&] { k_dfma<3><<<blocks, threads>>>(out, 0.5, iters); });
  float td4 = timeit([&] { k_dfma<4><<<blocks, threads>>>(out, 0.5, iters); });
  printf("{\"op\": \"8 fma.f64 + 8 mad.hi\", \"ms\": %.3f}\n", td2);
  printf("{\"op\": \"8 fma.f64 + 8 mad.wide(+xor)\", \"ms\": %.3f}\n", td3);
  printf("{\"op\": \"16 mad.wide(+xor)\", \"ms\": %.3f}\n", td4);
  printf("{\"op\": \"8 fma.f64 + 8 mad.lo chains\", \"ms\": %.3f, \"ms_imad16\": %.3f, \"ms_dfma16\": %.3f}\n", td1, t0, td0);
  for (int tpb : {128, 256, 384}) {
    int it = 512;
    float t = timeit([&] { k_fqmul<<<sms * 8, tpb>>>(out, 11, it); });
    printf("{\"op\": \"Fq::mul\", \"threads\": %d, \"Gmulmod_per_s\": %.2f}\n", tpb, (double)sms * 8 * tpb * it * 4 / t / 1e6);
  }
  // mixed adds over random-ish points (same curve points repeated; exercises the add path)
  const int npts = 1 << 16;
  Aff* d_pts;
  cudaMalloc(&d_pts, npts * sizeof(Aff));
  Aff* h = new Aff[npts];
  // point = (x, y) from k * g computed on the host via repeated affine-add-free doubling
  Xyzz acc = xyzz_inf();
  Fe gx{{0xbe9bb8c2u, 0x9f4698deu, 0x2e04a40bu, 0x96df9421u, 0xd6e0e406u, 0x000000abu}};
  Fe gy{{0xca83210eu, 0x0d3911f8u, 0x28e6ecd6u, 0xfcd508bdu, 0xc7320595u, 0x00000018u}};
  Aff g{Fq::to_mont(gx), Fq::to_mont(gy)};
  for (int i = 0; i < npts; i++) {
    xyzz_add_aff(acc, g);
    h[i] = xyzz_to_aff(acc);
    if (i > 64) {   // cheap: reuse earlier points for the rest
      for (int k = i; k < npts; k++) h[k] = h[k % 64 + 1];
      break;
    }
  }
  cudaMemcpy(d_pts, h, npts * sizeof(Aff), cudaMemcpyHostToDevice);
  for (int tpb : {128, 256}) {
    int it = 256;
    float t = timeit([&] { k_madd<<<sms * 8, tpb>>>(out, d_pts, npts, it); });
    printf("{\"op\": \"xyzz_add_aff\", \"threads\": %d, \"Gadd_per_s\": %.3f}\n", tpb, (double)sms * 8 * tpb * it / t / 1e6);
  }
  printf("{\"err\": \"%s\", \"sms\": %d}\n", cudaGetErrorString(cudaGetLastError()), sms);
  return 0;
}
