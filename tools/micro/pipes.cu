// Pipe throughput micro-benchmark (dev tool): MUFU.EX2, FFMA2 (packed), FFMA, LDS.128
// broadcast, each in a long unrolled loop of independent chains, full occupancy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
// Prints warp-instructions / clk / SM for each pipe.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float s) {
  __shared__ float4 sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(s, s, s, s);
  __syncthreads();
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  unsigned long long a2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1,%2};" : "=l"(a2[i]) : "f"(x[i]), "f"(x[i] + 1.f));
  unsigned long long m2, c2;
  asm("mov.b64 %0, {%1,%2};" : "=l"(m2) : "f"(0.999f), "f"(0.998f));
  asm("mov.b64 %0, {%1,%2};" : "=l"(c2) : "f"(s), "f"(s));
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a2[i]) : "l"(m2), "l"(c2));
      if (MODE == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(0.999f), "f"(s));
      if (MODE == 3) {
        const float4 v = sm[(it + i) & 63];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
  }
  float r = acc.x + acc.y + acc.z + acc.w;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a2[i]));
    r += x[i] + lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name) {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, sizeof(float) * sms * 8 * 256);
  const int iters = 1 << 14;
  k<MODE><<<sms * 8, 256>>>(o, 16, 1.f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<sms * 8, 256>>>(o, iters, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  // SM clock from the driver attribute is the max; report per-ns rate and per-clk at that clock
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double warp_instr = (double)sms * 8 * 8 * iters * 8;  // blocks * warps/block * iters * 8 per iter
  const double per_ns_sm = warp_instr / sms / (ms * 1e6);
  printf("%-10s %.3f warp-instr/ns/SM  (= %.3f /clk/SM at %.0f MHz)\n", name, per_ns_sm,
         per_ns_sm / (clk_khz * 1e-6), clk_khz / 1e3);
  cudaFree(o);
}

int main() {
  run<0>("MUFU.EX2");
  run<1>("FFMA2");
  run<2>("FFMA");
  run<3>("LDS.128bc");
  return 0;
}
