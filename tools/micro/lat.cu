// Dependent-chain latency of FFMA2 / FFMA / MUFU.EX2 / SHFL (dev tool): one warp, one chain.
#include <cstdio>
#include <cuda_runtime.h>
struct __align__(8) f2 { float x, y; };
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm volatile("{.reg .b64 ra,rb,rc,rd;\n\tmov.b64 ra,{%2,%3}; mov.b64 rb,{%4,%5}; mov.b64 rc,{%6,%7};\n\t"
      "fma.rn.f32x2 rd,ra,rb,rc; mov.b64 {%0,%1},rd;}" : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
template <int MODE>
__global__ void k(float* out, int iters, float s, long long* cyc) {
  f2 a{threadIdx.x * 1e-3f, 1.f}; float x = threadIdx.x * 1e-3f;
  const f2 m{0.999f, 0.998f}, c{s, s};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (MODE == 0) a = fma2(a, m, c);
      if (MODE == 1) x = fmaf(x, m.x, s + x * 0.f);
      if (MODE == 2) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); x = r * -0.5f; }
      if (MODE == 3) x = __shfl_xor_sync(0xffffffffu, x, 1) + s;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = a.x + a.y + x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE> void run(const char* n) {
  float* o; long long* c; cudaMalloc(&o, 1024 * 4); cudaMalloc(&c, 8);
  k<MODE><<<1, 32>>>(o, 10, 0.f, c); cudaDeviceSynchronize();
  k<MODE><<<1, 32>>>(o, 1000, 0.f, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-10s %.2f cycles per dependent op\n", n, h / 16000.0);
}
int main() { run<0>("FFMA2"); run<1>("FFMA"); run<2>("EX2(+FMUL)"); run<3>("SHFL(+FADD)"); }
