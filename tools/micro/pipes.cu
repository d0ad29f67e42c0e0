// Pipe-rate microbenchmark (dev tool): FFMA2 / FFMA / MUFU.EX2 / mixed throughput per SM.
#include <cstdio>
#include <cuda_runtime.h>

struct __align__(8) f2 { float x, y; };
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm volatile("{.reg .b64 ra,rb,rc,rd;\n\tmov.b64 ra,{%2,%3}; mov.b64 rb,{%4,%5}; mov.b64 rc,{%6,%7};\n\t"
      "fma.rn.f32x2 rd,ra,rb,rc; mov.b64 {%0,%1},rd;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float ex2(float x) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

template <int MODE, int NACC>
__global__ void k(float* out, int iters, float s) {
  __shared__ float2 sm[256];
  if (threadIdx.x < 256) sm[threadIdx.x] = make_float2(threadIdx.x, 1.f);
  __syncthreads();
  float2 lacc = make_float2(0.f, 0.f);
  f2 acc[NACC];
  float e[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i] = f2{threadIdx.x * 1e-3f + i, 1.f}; e[i] = -0.001f * i; }
  const f2 m{0.999f, 0.998f}, c{s, s};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      if (MODE == 0) acc[i] = fma2(acc[i], m, c);                        // FFMA2 only
      if (MODE == 1) acc[i].x = fmaf(acc[i].x, m.x, c.x);               // FFMA only
      if (MODE == 2) e[i] = ex2(e[i]);                                   // MUFU only
      if (MODE == 3) { acc[i] = fma2(acc[i], m, c); acc[i] = fma2(acc[i], m, c); acc[i] = fma2(acc[i], m, c);
                       e[i] = ex2(e[i]); }                              // 3 FFMA2 : 1 EX2
      if (MODE == 4) { acc[i] = fma2(acc[i], m, c); e[i] = ex2(e[i]); }  // 1 FFMA2 : 1 EX2
      if (MODE == 5) { e[i] = ex2(e[i]); float2 v = sm[(it * 8 + i) & 255]; lacc.x += v.x; lacc.y += v.y; }  // EX2 + broadcast LDS.64
      if (MODE == 6) { float2 v = sm[(it * 8 + i) & 255]; lacc.x += v.x; lacc.y += v.y; }  // broadcast LDS.64 only
      if (MODE == 7) { e[i] = ex2(e[i]); float2 v = sm[(it * 8 + i) & 255]; float2 w = sm[(it * 8 + i + 1) & 255]; lacc.x += v.x + w.x; lacc.y += v.y * w.y; }  // EX2 + 2 LDS
    }
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) t += acc[i].x + acc[i].y + e[i];
  t += lacc.x + lacc.y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int MODE>
void run(const char* name, int ops_per_iter_per_acc, int threads, int blocks_per_sm) {
  float* out;
  cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
  int iters = 4096;
  dim3 g(148 * blocks_per_sm), b(threads);
  k<MODE, 8><<<g, b>>>(out, 16, 0.f);
  cudaEvent_t a, z; cudaEventCreate(&a); cudaEventCreate(&z);
  cudaEventRecord(a);
  k<MODE, 8><<<g, b>>>(out, iters, 0.f);
  cudaEventRecord(z); cudaEventSynchronize(z);
  float ms; cudaEventElapsedTime(&ms, a, z);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_instr = (double)g.x * threads / 32 * iters * 8 * ops_per_iter_per_acc;
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s threads=%4d bps=%d  %.3f ms  warp-instr/clk/SM = %.3f\n", name, threads, blocks_per_sm, ms,
         warp_instr / cyc / 148);
  cudaFree(out);
}

int main() {
  for (int bps : {4}) {
    run<5>("EX2+LDS.64 (2 instr)", 2, 256, bps);
    run<6>("LDS.64 bcast (1 instr)", 1, 256, bps);
    run<7>("EX2+2xLDS.64 (3 instr)", 3, 256, bps);
  }
  for (int bps : {1, 4}) {
    run<0>("FFMA2 (1 instr)", 1, 256, bps);
    run<1>("FFMA (1 instr)", 1, 256, bps);
    run<2>("MUFU.EX2 (1 instr)", 1, 256, bps);
    run<3>("3xFFMA2+EX2 (4 instr)", 4, 256, bps);
    run<4>("FFMA2+EX2 (2 instr)", 2, 256, bps);
  }
  return 0;
}
