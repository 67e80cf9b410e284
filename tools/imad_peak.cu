// Integer-multiply pipe peak microbenchmark (IMAD / IMAD.HI / IMAD.WIDE) on B200.
// Used to fill the missing integer roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_imad(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[8], b = seed ^ threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = seed * (i + 1) + threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) {            // mad.lo: 1 IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b));
      } else if (MODE == 1) {     // mad.hi: IMAD.HI
        asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b));
      } else {                    // mad.wide: IMAD.WIDE.U32 (64-bit result)
        uint64_t r;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a[i]), "r"(b), "l"((uint64_t)a[i]));
        a[i] = (uint32_t)r ^ (uint32_t)(r >> 32);
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += a[i];
  if (s == 0x12345678) out[0] = s;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  uint32_t* out; cudaMalloc(&out, 4);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  const char* names[3] = {"mad.lo.u32", "mad.hi.u32", "mad.wide.u32"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; mode++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      if (mode == 0) k_imad<0><<<blocks, threads>>>(out, 7, iters);
      if (mode == 1) k_imad<1><<<blocks, threads>>>(out, 7, iters);
      if (mode == 2) k_imad<2><<<blocks, threads>>>(out, 7, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8;
      if (rep == 2) printf("{\"op\": \"%s\", \"sms\": %d, \"Tops_per_s\": %.3f, \"ms\": %.3f}\n", names[mode], sms, ops / ms / 1e9, ms);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
