// Throughput probe of the special-function unit on this GPU (attention roofline):
// tanh.approx.f32, ex2.approx.f32, rcp.approx, and FFMA, per SM per clock, many independent chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
  float x[8];
  unsigned long long v2[8];
  const unsigned long long c2 = 0x3F8000013F800001ull, d2 = 0x3A83126F3A83126Full;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = 0.001f * (threadIdx.x + i);
    v2[i] = ((unsigned long long)__float_as_uint(x[i]) << 32) | __float_as_uint(x[i]);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[i]));
      if (OP == 5) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v2[i]) : "l"(c2), "l"(d2));  // FFMA2
      if (OP == 6) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 4) {  // tanh.approx.bf16x2 on a packed pair
        unsigned v = __float_as_uint(x[i]);
        asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(v));
        x[i] = __uint_as_float(v);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + __uint_as_float((unsigned)v2[i]) + __uint_as_float((unsigned)(v2[i] >> 32));
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* o;
  cudaMalloc(&o, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"tanh.approx.f32", "ex2.approx.f32", "rcp.approx.f32", "ffma.f32", "tanh.approx.bf16x2",
                         "ffma2 (+fadd)", "rcp.approx.ftz"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int op = 0; op < 7; ++op) {
    const int iters = 4096, blocks = sms * 4, threads = 512;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (op) {
        case 0: k<0><<<blocks, threads>>>(o, iters); break;
        case 1: k<1><<<blocks, threads>>>(o, iters); break;
        case 2: k<2><<<blocks, threads>>>(o, iters); break;
        case 3: k<3><<<blocks, threads>>>(o, iters); break;
        case 4: k<4><<<blocks, threads>>>(o, iters); break;
        case 5: k<5><<<blocks, threads>>>(o, iters); break;
        case 6: k<6><<<blocks, threads>>>(o, iters); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)blocks * threads * iters * 8;
      if (rep) printf("%-20s %8.3f ms  %.3e op/s  %.1f op/clk/SM (at %d MHz nominal)\n", names[op], ms, ops / ms * 1e3,
                      ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
