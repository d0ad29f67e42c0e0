// RMSNorm with learned scale (nn.rms_norm, nn.py:55-58; eps 1e-6, no bias) —
// the first op of every LBVim block (block.py:170).  HBM-bound: one warp per
// token row, 16-byte vector loads/stores, fp32 accumulation.
#include "lbs_common.cuh"
#include "lbs_internal.h"

namespace lbs {

template <typename T, int VPL, int RPW>  // VPL = 16-byte vectors per lane; RPW rows per warp
__global__ void __launch_bounds__(256) rms_norm_kernel(const T* __restrict__ x, const float* __restrict__ scale,
                                                       T* __restrict__ out, long long rows, int D, float eps,
                                                       long long sx, long long so) {
  constexpr int EPV = 16 / sizeof(T);
  const long long row0 = ((long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * RPW;
  const int lane = threadIdx.x % 32;
  if (row0 >= rows) return;
  // all RPW rows' loads are in flight before the first reduction (memory-level parallelism)
  uint4 raw[RPW][VPL];
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c0 = (lane + 32 * k) * EPV;
      if (row0 + r < rows && c0 < D) raw[r][k] = *reinterpret_cast<const uint4*>(x + (row0 + r) * sx + c0);
      else raw[r][k] = make_uint4(0, 0, 0, 0);
    }
  // this lane's scale entries, loaded once per warp (16-byte loads)
  float sc[VPL][EPV];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c0 = (lane + 32 * k) * EPV;
#pragma unroll
    for (int i = 0; i < EPV; i += 4) {
      const float4 s4 = c0 < D ? __ldg(reinterpret_cast<const float4*>(scale + c0 + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
      sc[k][i] = s4.x;
      sc[k][i + 1] = s4.y;
      sc[k][i + 2] = s4.z;
      sc[k][i + 3] = s4.w;
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    if (row0 + r >= rows) break;
    float v[VPL][EPV];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const T* e = reinterpret_cast<const T*>(&raw[r][k]);
#pragma unroll
      for (int i = 0; i < EPV; ++i) {
        v[k][i] = to_f(e[i]);
        ss = fmaf(v[k][i], v[k][i], ss);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = rsqrtf(ss / (float)D + eps);
    T* orow = out + (row0 + r) * so;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c0 = (lane + 32 * k) * EPV;
      if (c0 < D) {
        uint4 o4;
        T* e = reinterpret_cast<T*>(&o4);
#pragma unroll
        for (int i = 0; i < EPV; ++i) {
          const float y = v[k][i] * inv * sc[k][i];
          if constexpr (sizeof(T) == 4) e[i] = y;
          else e[i] = __float2bfloat16_rn(y);
        }
        *reinterpret_cast<uint4*>(orow + c0) = o4;
      }
    }
  }
}

// G lanes per row (G | 32, 32/G rows per warp), VPL 16-byte vectors per lane:
// every lane busy and 32/G rows of loads in flight per warp (D = 192 bf16 is 24
// vectors: 8 lanes x 3 instead of 24 of 32 lanes x 1).
template <typename T, int G, int VPL, typename To = T>
__global__ void __launch_bounds__(256) rms_norm_group_kernel(const T* __restrict__ x, const float* __restrict__ scale,
                                                             To* __restrict__ out, long long rows, int D, float eps,
                                                             long long sx, long long so) {
  constexpr int EPV = 16 / sizeof(T);
  constexpr int RPWG = 32 / G;  // rows per warp per pass
  const int lane = threadIdx.x % 32;
  const int sub = lane % G;
  // grid-stride over row groups (the launcher sizes the grid to one resident wave);
  // the next group's loads are issued before this group is reduced and stored
  const long long warp0 = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const long long wstride = (long long)gridDim.x * (blockDim.x / 32) * RPWG;
  auto load = [&](long long row, uint4 (&raw)[VPL]) {
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c0 = (sub + G * k) * EPV;
      raw[k] = (row < rows && c0 < D) ? *reinterpret_cast<const uint4*>(x + row * sx + c0) : make_uint4(0, 0, 0, 0);
    }
  };
  long long wrow = warp0 * RPWG;  // first row of this warp's group (warp-uniform)
  uint4 raw[VPL];
  load(wrow + lane / G, raw);
  for (; wrow < rows; wrow += wstride) {
    const long long row = wrow + lane / G;
    uint4 nxt[VPL];
    load(wrow + wstride + lane / G, nxt);
    float v[VPL][EPV];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const T* e = reinterpret_cast<const T*>(&raw[k]);
#pragma unroll
      for (int i = 0; i < EPV; ++i) {
        v[k][i] = to_f(e[i]);
        ss = fmaf(v[k][i], v[k][i], ss);
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = rsqrtf(ss / (float)D + eps);
    if (row < rows) {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int c0 = (sub + G * k) * EPV;
        if (c0 < D) {
          // EPV outputs of To: 16 bytes (To == T), or 8 (fp32 in -> bf16 out)
          using OV = std::conditional_t<sizeof(To) == sizeof(T), uint4, uint2>;
          OV o4;
          To* e = reinterpret_cast<To*>(&o4);
#pragma unroll
          for (int i = 0; i < EPV; i += 4) {
            const float4 s4 = __ldg(reinterpret_cast<const float4*>(scale + c0 + i));
            const float sc[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) e[i + u] = from_f<To>(v[k][i + u] * inv * sc[u]);
          }
          *reinterpret_cast<OV*>(out + row * so + c0) = o4;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) raw[k] = nxt[k];
  }
}

// any D / alignment: one warp per row, scalar strided accesses
template <typename T, typename To = T>
__global__ void __launch_bounds__(256) rms_norm_scalar_kernel(const T* __restrict__ x, const float* __restrict__ scale,
                                                              To* __restrict__ out, long long rows, int D, float eps,
                                                              long long sx, long long so) {
  const long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  float ss = 0.f;
  for (int c = lane; c < D; c += 32) {
    const float v = to_f(x[row * sx + c]);
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / (float)D + eps);
  for (int c = lane; c < D; c += 32) st<To>(out + row * so + c, to_f(x[row * sx + c]) * inv * scale[c]);
}

template <typename T, typename To = T>
static cudaError_t launch_norm_t(const NormParams& p, cudaStream_t st) {
  constexpr int EPV = 16 / sizeof(T);
  constexpr int OVB = EPV * (int)sizeof(To);  // bytes of one output vector (16, or 8 for f32 -> bf16)
  const int vpl = (p.D + 32 * EPV - 1) / (32 * EPV);
  dim3 block(256), grid((unsigned)((p.rows + 7) / 8));
  const T* x = static_cast<const T*>(p.x);
  To* o = static_cast<To*>(p.out);
  const bool vec = p.D % EPV == 0 && (p.sx * (long long)sizeof(T)) % 16 == 0 &&
                   (p.so * (long long)sizeof(To)) % OVB == 0 && reinterpret_cast<uintptr_t>(p.x) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(p.out) % OVB == 0 && reinterpret_cast<uintptr_t>(p.scale) % 16 == 0 && vpl <= 4;
  if (!vec) {
    rms_norm_scalar_kernel<T, To><<<grid, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so);
    return cudaGetLastError();
  }
#ifndef LBS_NORM_RPW
#define LBS_NORM_RPW 1  // rows per warp (2, 4, 8 measured no better)
#endif
#ifndef LBS_NORM_PERSIST
#define LBS_NORM_PERSIST 1
#endif
#ifndef LBS_NORM_GROUP
#define LBS_NORM_GROUP 1
#endif
  if (LBS_NORM_GROUP) {
    // smallest power-of-two lane group with <= 3 vectors per lane
    const int nv = p.D / EPV;
    int G = 1;
    while (G < 32 && (nv + G - 1) / G > 3) G *= 2;
    const int vpl = (nv + G - 1) / G;
    if (vpl <= 3) {
      const long long rows_per_block = 8LL * (32 / G);
      static const int n_sms = [] {
        int d = 0, n = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
        return n;
      }();
      long long nb = (p.rows + rows_per_block - 1) / rows_per_block;
      if (LBS_NORM_PERSIST && nb > (long long)n_sms * 8) nb = (long long)n_sms * 8;  // one resident wave
      dim3 gg((unsigned)nb);
#define LBS_NORM_G(GG)                                                                                     \
  if (G == GG) {                                                                                           \
    if (vpl == 1) rms_norm_group_kernel<T, GG, 1, To><<<gg, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so); \
    else if (vpl == 2) rms_norm_group_kernel<T, GG, 2, To><<<gg, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so); \
    else rms_norm_group_kernel<T, GG, 3, To><<<gg, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so); \
    return cudaGetLastError();                                                                             \
  }
      LBS_NORM_G(1) LBS_NORM_G(2) LBS_NORM_G(4) LBS_NORM_G(8) LBS_NORM_G(16) LBS_NORM_G(32)
#undef LBS_NORM_G
    }
  }
  if constexpr (!std::is_same<T, To>::value) {
    // mixed dtypes have the lane-group and scalar kernels only
    rms_norm_scalar_kernel<T, To><<<grid, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so);
    return cudaGetLastError();
  } else {
    constexpr int RPW = LBS_NORM_RPW;
    dim3 gridv((unsigned)((p.rows + 8 * RPW - 1) / (8 * RPW)));
    if (vpl <= 1) rms_norm_kernel<T, 1, RPW><<<gridv, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so);
    else if (vpl <= 2) rms_norm_kernel<T, 2, RPW><<<gridv, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so);
    else if (vpl <= 4) rms_norm_kernel<T, 4, RPW><<<gridv, block, 0, st>>>(x, p.scale, o, p.rows, p.D, p.eps, p.sx, p.so);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
  }
}

// ---------------------------------------------------------------------------
// Backward.  One warp per row (grid-stride over a fixed set of warps), 16-byte
// vectors: r is recomputed from x, dot = sum(g x) with g = dout * scale, then
// dx = r g - x r^3 dot / D.  Each lane keeps its columns' dscale partials
// (sum of dout x r over the rows it visits) in registers and writes them once
// per warp; a second kernel adds the per-warp partials in fixed order.
constexpr int kNormBwdBlocks = 148 * 2;  // x 8 warps: one resident wave at 2 blocks/SM (the launch is independent of the device)
int norm_bwd_warps(long long rows) {
  const long long w = rows < (long long)kNormBwdBlocks * 8 ? rows : (long long)kNormBwdBlocks * 8;
  return (int)(w < 1 ? 1 : w);
}

template <typename T, int VPL>
__global__ void __launch_bounds__(256) rms_norm_bwd_kernel(NormBwdParams p) {
  constexpr int EPV = 16 / sizeof(T);
  const int lane = threadIdx.x % 32;
  const long long warp = (long long)blockIdx.x * 8 + threadIdx.x / 32;
  const int D = p.D;
  float sc[VPL][EPV], dsc[VPL][EPV];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c0 = (lane + 32 * k) * EPV;
#pragma unroll
    for (int i = 0; i < EPV; ++i) {
      sc[k][i] = c0 < D ? p.scale[c0 + i] : 0.f;
      dsc[k][i] = 0.f;
    }
  }
  const T* X = static_cast<const T*>(p.x);
  const T* G = static_cast<const T*>(p.dout);
  T* DX = static_cast<T*>(p.dx);
  // the next row's x / dout are loaded before this row is reduced (one row of
  // loads always in flight per warp)
  const T* R = static_cast<const T*>(p.dres);  // optional residual gradient: dx += dres
  auto load = [&](long long row, uint4 (&rx)[VPL], uint4 (&rg)[VPL]) {
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c0 = (lane + 32 * k) * EPV;
      const bool ok = row < p.rows && c0 < D;
      rx[k] = ok ? *reinterpret_cast<const uint4*>(X + row * p.sx + c0) : make_uint4(0, 0, 0, 0);
      rg[k] = ok ? *reinterpret_cast<const uint4*>(G + row * p.sg + c0) : make_uint4(0, 0, 0, 0);
    }
  };
  uint4 rx[VPL], rg[VPL];
  load(warp, rx, rg);
  for (long long row = warp; row < p.rows; row += p.n_warps) {
    uint4 nx[VPL], ng[VPL];
    load(row + p.n_warps, nx, ng);
    uint4 rr[VPL];
    if (R) {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int c0 = (lane + 32 * k) * EPV;
        rr[k] = c0 < D ? *reinterpret_cast<const uint4*>(R + row * p.sres + c0) : make_uint4(0, 0, 0, 0);
      }
    }
    float ss = 0.f, dot = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const T* ex = reinterpret_cast<const T*>(&rx[k]);
      const T* eg = reinterpret_cast<const T*>(&rg[k]);
#pragma unroll
      for (int i = 0; i < EPV; ++i) {
        const float xv = to_f(ex[i]);
        ss = fmaf(xv, xv, ss);
        dot = fmaf(to_f(eg[i]) * sc[k][i], xv, dot);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      dot += __shfl_xor_sync(0xffffffffu, dot, o);
    }
    const float r = rsqrtf(ss / (float)D + p.eps);
    const float c = r * r * r * dot / (float)D;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c0 = (lane + 32 * k) * EPV;
      if (c0 < D) {
        const T* ex = reinterpret_cast<const T*>(&rx[k]);
        const T* eg = reinterpret_cast<const T*>(&rg[k]);
        uint4 o4;
        T* e = reinterpret_cast<T*>(&o4);
        const T* er = reinterpret_cast<const T*>(&rr[k]);
#pragma unroll
        for (int i = 0; i < EPV; ++i) {
          const float xv = to_f(ex[i]), gv = to_f(eg[i]);
          float d = r * gv * sc[k][i] - xv * c;
          if (R) d += to_f(er[i]);
          e[i] = from_f<T>(d);
          dsc[k][i] = fmaf(gv, xv * r, dsc[k][i]);
        }
        *reinterpret_cast<uint4*>(DX + row * p.sdx + c0) = o4;
      }
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      rx[k] = nx[k];
      rg[k] = ng[k];
    }
  }
  if (p.part != nullptr && warp < p.n_warps) {
    float* pw = p.part + warp * D;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c0 = (lane + 32 * k) * EPV;
      if (c0 < D) {
#pragma unroll
        for (int i = 0; i < EPV; ++i) pw[c0 + i] = dsc[k][i];
      }
    }
  }
}

// Any D / alignment: one warp per row, scalar strided accesses; the warp's dscale
// partial row lives in the workspace (each warp owns its row: no races).
template <typename T>
__global__ void __launch_bounds__(256) rms_norm_bwd_scalar_kernel(NormBwdParams p) {
  const int lane = threadIdx.x % 32;
  const long long warp = (long long)blockIdx.x * 8 + threadIdx.x / 32;
  if (warp >= p.n_warps) return;
  const int D = p.D;
  const T* X = static_cast<const T*>(p.x);
  const T* G = static_cast<const T*>(p.dout);
  T* DX = static_cast<T*>(p.dx);
  float* pw = p.part ? p.part + warp * D : nullptr;
  if (pw)
    for (int c = lane; c < D; c += 32) pw[c] = 0.f;
  for (long long row = warp; row < p.rows; row += p.n_warps) {
    float ss = 0.f, dot = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float xv = to_f(X[row * p.sx + c]);
      ss = fmaf(xv, xv, ss);
      dot = fmaf(to_f(G[row * p.sg + c]) * p.scale[c], xv, dot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      dot += __shfl_xor_sync(0xffffffffu, dot, o);
    }
    const float r = rsqrtf(ss / (float)D + p.eps);
    const float cc = r * r * r * dot / (float)D;
    for (int c = lane; c < D; c += 32) {
      const float xv = to_f(X[row * p.sx + c]);
      const float gv = to_f(G[row * p.sg + c]);
      float d = r * gv * p.scale[c] - xv * cc;
      if (p.dres) d += to_f(static_cast<const T*>(p.dres)[row * p.sres + c]);
      DX[row * p.sdx + c] = from_f<T>(d);
      if (pw) pw[c] = fmaf(gv, xv * r, pw[c]);
    }
  }
}

// dscale[c] += sum over warps of part[w][c]: a 1024-thread block owns 32 columns,
// 32 slices each sum every 32nd warp's partial (fp64), then the slices are added
// in fixed order (deterministic; a serial per-column loop over ~4.7k partials was
// a 350 us load chain)
__global__ void __launch_bounds__(1024) rms_norm_bwd_reduce_kernel(const float* part, int n_warps, int D,
                                                                   float* dscale) {
  __shared__ double acc[32][33];
  const int lane = threadIdx.x % 32, slice = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (c < D) {
    int w = slice;
    for (; w + 96 < n_warps; w += 128) {
      const float a0 = part[(long long)w * D + c];
      const float a1 = part[(long long)(w + 32) * D + c];
      const float a2 = part[(long long)(w + 64) * D + c];
      const float a3 = part[(long long)(w + 96) * D + c];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; w < n_warps; w += 32) s += part[(long long)w * D + c];
  }
  acc[slice][lane] = s;
  __syncthreads();
  if (slice == 0 && c < D) {
    double t = 0.0;
    for (int k = 0; k < 32; ++k) t += acc[k][lane];
    dscale[c] += (float)t;
  }
}

template <typename T>
static cudaError_t launch_norm_bwd_t(const NormBwdParams& p, cudaStream_t st) {
  constexpr int EPV = 16 / sizeof(T);
  const int vpl = (p.D / EPV + 31) / 32;
  const unsigned blocks = (unsigned)((p.n_warps + 7) / 8);
  auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  const bool vec = p.D % EPV == 0 && p.sx % EPV == 0 && p.sg % EPV == 0 && p.sdx % EPV == 0 && al(p.x) &&
                   al(p.dout) && al(p.dx) && (!p.dres || (p.sres % EPV == 0 && al(p.dres))) && vpl <= 4;
  if (!vec) rms_norm_bwd_scalar_kernel<T><<<blocks, 256, 0, st>>>(p);
  else if (vpl <= 1) rms_norm_bwd_kernel<T, 1><<<blocks, 256, 0, st>>>(p);
  else if (vpl <= 2) rms_norm_bwd_kernel<T, 2><<<blocks, 256, 0, st>>>(p);
  else if (vpl <= 3) rms_norm_bwd_kernel<T, 3><<<blocks, 256, 0, st>>>(p);
  else rms_norm_bwd_kernel<T, 4><<<blocks, 256, 0, st>>>(p);
  if (p.dscale != nullptr) rms_norm_bwd_reduce_kernel<<<(p.D + 31) / 32, 1024, 0, st>>>(p.part, p.n_warps, p.D, p.dscale);
  return cudaGetLastError();
}

cudaError_t launch_rms_norm_bwd(const NormBwdParams& p, int dtype, cudaStream_t st) {
  if (dtype == LBS_F32) return launch_norm_bwd_t<float>(p, st);
  if (dtype == LBS_BF16) return launch_norm_bwd_t<__nv_bfloat16>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_rms_norm(const NormParams& p, int dtype, int out_dtype, cudaStream_t st) {
  if (dtype == LBS_F32 && out_dtype == LBS_F32) return launch_norm_t<float>(p, st);
  if (dtype == LBS_F32 && out_dtype == LBS_BF16) return launch_norm_t<float, __nv_bfloat16>(p, st);
  if (dtype == LBS_BF16 && out_dtype == LBS_BF16) return launch_norm_t<__nv_bfloat16>(p, st);
  return cudaErrorInvalidValue;
}

}  // namespace lbs
