// Depthwise causal conv1d (+ fused SiLU), channel-last, with flip-on-load.
//
// Forward replaces nn.causal_conv1d + nn.silu (nn.py:87-99,25-26):
//   xc[l] = sum_{q<K} w[e,q] x[l-q] (+ bias),  out = silu(xc)
// Backward replaces nn.causal_conv1d_grad + silu_grad (nn.py:102-114,29-31),
// recomputing xc instead of storing it:
//   g = dout * silu'(xc);  dx[l] = sum_q w[e,q] g[l+q];  dw[e,q] = sum_{b,l} g[l] x[l-q]
// "l" is the logical (scanned) index; with LBS_FLAG_REVERSE logical l reads
// physical L-1-l, so LBVim's reverse-direction layers need no flip copies
// (block.py:180-181, model.py:216-218).
//
// HBM-bound elementwise kernel: one thread per (b, e, chunk of kConvChunk
// steps) keeps the K-1 step history in registers; a warp covers 32
// consecutive channels, so every step is one contiguous row segment.
#include <algorithm>
#include <string>
#include <type_traits>

#include "lbs_common.cuh"
#include "lbs_internal.h"

namespace lbs {

#ifndef LBS_CONV_CTAS_PER_SM
#define LBS_CONV_CTAS_PER_SM 24  // target grid size of the streaming kernel (8/12/16/24 measured: 24 best)
#endif
static int conv_num_sms() {
  static int n = 0;
  if (n <= 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        n <= 0)
      n = 148;
  }
  return n;
}

constexpr int kConvThreads = 128;
constexpr int kConvChunk = 32;
constexpr int kMaxWidth = 8;

struct ConvParams {
  int Bt, L, E, K;
  uint32_t flags;
  View3D x, dout;
  void* out;
  long long so0, so1, so2;
  void* dx;
  long long sd0, sd1, sd2;
  const float* w;
  const float* bias;
  float* part;  // (n_part, E, K+1) dweight/dbias partials
  int n_chunks;
};

template <typename T, int KW>
__global__ void __launch_bounds__(kConvThreads) conv_fwd_kernel(ConvParams p) {
  const int e = blockIdx.x * kConvThreads + threadIdx.x;
  if (e >= p.E) return;
  const int chunk = blockIdx.y, b = blockIdx.z;
  const int L = p.L;
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool act = p.flags & LBS_CONV_SILU;
  float w[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) w[q] = q < p.K ? p.w[(long long)e * p.K + q] : 0.f;
  const float bias = p.bias ? p.bias[e] : 0.f;
  const T* xp = static_cast<const T*>(p.x.p) + (long long)b * p.x.s0 + (long long)e * p.x.s2;
  T* op = static_cast<T*>(p.out) + (long long)b * p.so0 + (long long)e * p.so2;
  const int l0 = chunk * kConvChunk;
  const int l1 = min(L, l0 + kConvChunk);
  auto phys = [&](int l) -> long long { return rev ? (L - 1 - l) : l; };
  float hist[KW];  // hist[q] = x[l - q]
  hist[0] = 0.f;
#pragma unroll
  for (int q = 1; q < KW; ++q) {
    const int l = l0 - q;
    hist[q] = (q < p.K && l >= 0) ? ld<T>(xp + phys(l) * p.x.s1) : 0.f;
  }
  // groups of 8 steps: all 8 loads are issued before any use (memory-level
  // parallelism), then the window slides through them in registers
  const long long xs = rev ? -p.x.s1 : p.x.s1;
  const long long os = rev ? -p.so1 : p.so1;
  const T* xl = xp + phys(l0) * p.x.s1;
  T* ol = op + phys(l0) * p.so1;
  for (int l = l0; l < l1; l += 8) {
    float xv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = (l + i < l1) ? ld<T>(xl + (long long)(l - l0 + i) * xs) : 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hist[0] = xv[i];
      float acc = bias;
#pragma unroll
      for (int q = KW - 1; q >= 0; --q) acc = fmaf(w[q], hist[q], acc);
      if (l + i < l1) st<T>(ol + (long long)(l - l0 + i) * os, act ? silu_f(acc) : acc);
#pragma unroll
      for (int q = KW - 1; q >= 1; --q) hist[q] = hist[q - 1];
    }
  }
}

__device__ __forceinline__ void cp_async16_conv(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// Tile-staged forward (default for 16-byte aligned rows): a 128-thread CTA owns
// (b, kConvTT steps, 128 channels).  The (kConvTT + K - 1) input rows arrive by
// cp.async 16-byte pieces, each thread sweeps its channel through shared memory
// (K-1 history in registers) into an output tile, and the tile leaves as
// coalesced 16-byte stores -- every HBM access is a whole 16-byte piece.
// Flip-on-load: logical row l is physical L-1-l for both the input and output.
constexpr int kConvTT = 32;
constexpr int kConvTE = 128;

template <typename T, int KW>
__global__ void __launch_bounds__(kConvTE) conv_fwd_tile_kernel(ConvParams p) {
  constexpr int V = 16 / sizeof(T);
  constexpr int ROWS = kConvTT + KW - 1;
  __shared__ __align__(16) T xin[ROWS][kConvTE];
  __shared__ __align__(16) T yout[kConvTT][kConvTE];
  const int e0 = blockIdx.x * kConvTE;
  const int l0 = blockIdx.y * kConvTT;
  const int b = blockIdx.z;
  const int L = p.L;
  const int EC = min(kConvTE, p.E - e0);
  const int TT = min(kConvTT, L - l0);
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool act = p.flags & LBS_CONV_SILU;
  const int ppr = EC / V;  // 16-byte pieces per row
  const T* xb = static_cast<const T*>(p.x.p) + (long long)b * p.x.s0 + e0;
  for (int i = threadIdx.x; i < ROWS * ppr; i += kConvTE) {
    const int r = i / ppr, pc = i - r * ppr;
    const int l = l0 - (KW - 1) + r;
    T* dst = &xin[r][pc * V];
    if (l >= 0 && l < L) {
      cp_async16_conv(dst, xb + (long long)(rev ? L - 1 - l : l) * p.x.s1 + pc * V);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int c = threadIdx.x;
  if (c < EC) {
    const int e = e0 + c;
    float w[KW];
#pragma unroll
    for (int q = 0; q < KW; ++q) w[q] = q < p.K ? p.w[(long long)e * p.K + q] : 0.f;
    const float bias = p.bias ? p.bias[e] : 0.f;
    float hist[KW];  // hist[q] = x[l - q]
#pragma unroll
    for (int q = 1; q < KW; ++q) hist[q] = to_f(xin[KW - 1 - q][c]);
    if (TT == kConvTT) {
#pragma unroll 8
      for (int j = 0; j < kConvTT; ++j) {
        hist[0] = to_f(xin[KW - 1 + j][c]);
        float acc = bias;
#pragma unroll
        for (int q = KW - 1; q >= 0; --q) acc = fmaf(w[q], hist[q], acc);
        yout[j][c] = from_f<T>(act ? silu_f(acc) : acc);
#pragma unroll
        for (int q = KW - 1; q >= 1; --q) hist[q] = hist[q - 1];
      }
    } else {
      for (int j = 0; j < TT; ++j) {
        hist[0] = to_f(xin[KW - 1 + j][c]);
        float acc = bias;
#pragma unroll
        for (int q = KW - 1; q >= 0; --q) acc = fmaf(w[q], hist[q], acc);
        yout[j][c] = from_f<T>(act ? silu_f(acc) : acc);
#pragma unroll
        for (int q = KW - 1; q >= 1; --q) hist[q] = hist[q - 1];
      }
    }
  }
  __syncthreads();
  T* ob = static_cast<T*>(p.out) + (long long)b * p.so0 + e0;
  for (int i = threadIdx.x; i < TT * ppr; i += kConvTE) {
    const int j = i / ppr, pc = i - j * ppr;
    const int l = l0 + j;
    *reinterpret_cast<uint4*>(ob + (long long)(rev ? L - 1 - l : l) * p.so1 + pc * V) =
        *reinterpret_cast<const uint4*>(&yout[j][pc * V]);
  }
}

template <typename T, int KW>
__global__ void __launch_bounds__(kConvThreads) conv_bwd_kernel(ConvParams p) {
  const int e = blockIdx.x * kConvThreads + threadIdx.x;
  const int chunk = blockIdx.y, b = blockIdx.z;
  if (e >= p.E) return;
  const int L = p.L, K = p.K;
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool act = p.flags & LBS_CONV_SILU;
  float w[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) w[q] = q < K ? p.w[(long long)e * K + q] : 0.f;
  const float bias = p.bias ? p.bias[e] : 0.f;
  const T* xp = static_cast<const T*>(p.x.p) + (long long)b * p.x.s0 + (long long)e * p.x.s2;
  const T* gp = static_cast<const T*>(p.dout.p) + (long long)b * p.dout.s0 + (long long)e * p.dout.s2;
  T* dxp = static_cast<T*>(p.dx) + (long long)b * p.sd0 + (long long)e * p.sd2;
  auto phys = [&](int l) -> long long { return rev ? (L - 1 - l) : l; };
  auto X = [&](int l) -> float { return (l >= 0 && l < L) ? ld<T>(xp + phys(l) * p.x.s1) : 0.f; };
  // g[l] = dout[l] * silu'(xc[l]); xc recomputed from x
  auto G = [&](int l) -> float {
    if (l < 0 || l >= L) return 0.f;
    float gv = ld<T>(gp + phys(l) * p.dout.s1);
    if (act) {
      float xc = bias;
#pragma unroll
      for (int q = 0; q < KW; ++q)
        if (q < K) xc = fmaf(w[q], X(l - q), xc);
      const float s = sigmoid_f(xc);
      gv *= s * (1.f + xc * (1.f - s));
    }
    return gv;
  };
  const int l0 = chunk * kConvChunk;
  const int l1 = min(L, l0 + kConvChunk);
  float dw[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) dw[q] = 0.f;
  float db = 0.f;
  // sliding window of future g: fut[q] = g[l + q]
  float fut[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) fut[q] = (q < K) ? G(l0 + q) : 0.f;
  for (int l = l0; l < l1; ++l) {
    float acc = 0.f;
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) acc = fmaf(w[q], fut[q], acc);
    st<T>(dxp + phys(l) * p.sd1, acc);
    const float g0 = fut[0];
    db += g0;
#pragma unroll
    for (int q = 0; q < KW; ++q)
      if (q < K) dw[q] = fmaf(g0, X(l - q), dw[q]);
#pragma unroll
    for (int q = 0; q < KW - 1; ++q) fut[q] = fut[q + 1];
    fut[KW - 1] = 0.f;
    if (K >= 1) {
      // fill slot K-1 with g[l + K]
      float nxt = G(l + K);
#pragma unroll
      for (int q = 0; q < KW; ++q)
        if (q == K - 1) fut[q] = nxt;
    }
  }
  float* part = p.part + (((long long)b * p.n_chunks + chunk) * p.E + e) * (K + 1);
  for (int q = 0; q < K; ++q) part[q] = dw[q];
  part[K] = db;
}

// Tile-staged backward (16-byte aligned rows): a 64-thread CTA owns (b, 32-step
// chunk, 64 channels).  x rows [l0-(K-1), l0+32+K-1) and dout rows [l0, l0+32+K-1)
// arrive by cp.async 16-byte pieces; each thread recomputes g = dout * silu'(xc)
// for its channel from shared memory and slides the K-step window exactly as
// conv_bwd_kernel does (same operation order: identical dx and partials); dx
// leaves through a shared-memory tile as 16-byte stores.  The scalar kernel
// re-read x K+1 times per step through L1 (0.2 of HBM at the LBVim-S shape).
constexpr int kConvBE = 64;
template <typename T, int KW>
__global__ void __launch_bounds__(kConvBE) conv_bwd_tile_kernel(ConvParams p) {
  constexpr int V = 16 / sizeof(T);
  constexpr int TT = kConvChunk;
  constexpr int XR = TT + 2 * KW;  // x rows: l0-(KW-1) .. l0+TT+KW (the register window reads 2 past)
  constexpr int GR = TT + KW;            // dout rows: l0 .. l0+TT+KW-1 (the window's last, unused, lookahead reads row TT+K-1)
  __shared__ __align__(16) T xs[XR][kConvBE];
  __shared__ __align__(16) T gs[GR][kConvBE];
  // dx row j overwrites dout row j: this thread last read its column of that row
  // K steps earlier (the g window lives in registers)
  T (*dxo)[kConvBE] = gs;
  const int e0 = blockIdx.x * kConvBE;
  const int chunk = blockIdx.y, b = blockIdx.z;
  const int l0 = chunk * TT;
  const int L = p.L;
  constexpr int K = KW;  // launched only for K == KW (exact window: no predicated copies)
  const int EC = min(kConvBE, p.E - e0);
  const int ppr = EC / V;
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool act = p.flags & LBS_CONV_SILU;
  const T* xb = static_cast<const T*>(p.x.p) + (long long)b * p.x.s0 + e0;
  const T* gb = static_cast<const T*>(p.dout.p) + (long long)b * p.dout.s0 + e0;
  for (int i = threadIdx.x; i < (XR + GR) * ppr; i += kConvBE) {
    const int r = i / ppr, pc = i - r * ppr;
    const bool isx = r < XR;
    const int l = isx ? l0 - (KW - 1) + r : l0 + (r - XR);
    T* dst = isx ? &xs[r][pc * V] : &gs[r - XR][pc * V];
    if (l >= 0 && l < L) {
      const long long ph = rev ? L - 1 - l : l;
      cp_async16_conv(dst, isx ? xb + ph * p.x.s1 + pc * V : gb + ph * p.dout.s1 + pc * V);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int c = threadIdx.x;
  const int l1 = min(L, l0 + TT);
  if (c < EC) {
    const int e = e0 + c;
    float w[KW];
#pragma unroll
    for (int q = 0; q < KW; ++q) w[q] = q < K ? p.w[(long long)e * K + q] : 0.f;
    const float bias = p.bias ? p.bias[e] : 0.f;
    auto X = [&](int l) -> float { return to_f(xs[l - l0 + (KW - 1)][c]); };  // zero-padded rows
    // x in a register window: xw[i] = x[l - (KW-1) + i], i < 2 KW (one new row per step)
    float xw[2 * KW];
#pragma unroll
    for (int i = 0; i < 2 * KW; ++i) xw[i] = X(l0 - (KW - 1) + i);
    // g = dout * silu'(xc) at l + off, from the window (off in [0, KW])
    auto Gw = [&](int l, int off) -> float {
      if (l + off >= L) return 0.f;
      float gv = to_f(gs[l + off - l0][c]);
      if (act) {
        float xc = bias;
#pragma unroll
        for (int q = 0; q < KW; ++q)
          if (q < K) xc = fmaf(w[q], xw[KW - 1 + off - q], xc);
        const float sg = sigmoid_f(xc);
        gv *= sg * (1.f + xc * (1.f - sg));
      }
      return gv;
    };
    float dw[KW];
#pragma unroll
    for (int q = 0; q < KW; ++q) dw[q] = 0.f;
    float db = 0.f;
    float fut[KW];  // fut[q] = g[l + q]
#pragma unroll
    for (int q = 0; q < KW; ++q) fut[q] = (q < K) ? Gw(l0, q) : 0.f;
#pragma unroll 4
    for (int l = l0; l < l1; ++l) {
      float acc = 0.f;
#pragma unroll
      for (int q = KW - 1; q >= 0; --q) acc = fmaf(w[q], fut[q], acc);
      dxo[l - l0][c] = from_f<T>(acc);
      const float g0 = fut[0];
      db += g0;
#pragma unroll
      for (int q = 0; q < KW; ++q)
        if (q < K) dw[q] = fmaf(g0, xw[KW - 1 - q], dw[q]);
#pragma unroll
      for (int q = 0; q < KW - 1; ++q) fut[q] = fut[q + 1];
      fut[KW - 1] = 0.f;
      fut[K - 1] = Gw(l, K);
      // slide the x window one step
#pragma unroll
      for (int i = 0; i < 2 * KW - 1; ++i) xw[i] = xw[i + 1];
      xw[2 * KW - 1] = X(l + KW + 1);
    }
    float* part = p.part + (((long long)b * p.n_chunks + chunk) * p.E + e) * (K + 1);
    for (int q = 0; q < K; ++q) part[q] = dw[q];
    part[K] = db;
  }
  __syncthreads();
  T* ob = static_cast<T*>(p.dx) + (long long)b * p.sd0 + e0;
  for (int i = threadIdx.x; i < (l1 - l0) * ppr; i += kConvBE) {
    const int j = i / ppr, pc = i - j * ppr;
    const int l = l0 + j;
    *reinterpret_cast<uint4*>(ob + (long long)(rev ? L - 1 - l : l) * p.sd1 + pc * V) =
        *reinterpret_cast<const uint4*>(&dxo[j][pc * V]);
  }
}

// Two-channel variant of the tile backward (whole 128-channel tiles, K = 4, fp32 /
// bf16): 64 threads, each a channel PAIR with packed taps (FFMA2) and 4-/8-byte
// shared-memory accesses; per channel the same operation order as
// conv_bwd_tile_kernel (identical dx and partials).  The one-channel kernel is
// issue-bound (74 % issue-active, ncu) on per-element index math.
template <typename T>
__global__ void __launch_bounds__(64) conv_bwd_tile2_kernel(ConvParams p) {
  constexpr int KW = 4, K = 4;
  constexpr int V = 16 / sizeof(T);
  constexpr int TE = 128, NT = 64, PPR = TE / V;
  constexpr int TT = kConvChunk;
  constexpr int XR = TT + 2 * KW;
  constexpr int GR = TT + KW;
  __shared__ __align__(16) T xs[XR][TE];
  __shared__ __align__(16) T gs[GR][TE];
  T (*dxo)[TE] = gs;  // dx row j overwrites dout row j (consumed K steps earlier)
  const int e0 = blockIdx.x * TE;
  const int chunk = blockIdx.y, b = blockIdx.z;
  const int l0 = chunk * TT;
  const int L = p.L;
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool act = p.flags & LBS_CONV_SILU;
  const T* xb = static_cast<const T*>(p.x.p) + (long long)b * p.x.s0 + e0;
  const T* gb = static_cast<const T*>(p.dout.p) + (long long)b * p.dout.s0 + e0;
#pragma unroll 4
  for (int i0 = 0; i0 < (XR + GR) * PPR; i0 += NT) {
    const int i = i0 + threadIdx.x;
    const int r = i / PPR, pc = i % PPR;
    const bool isx = r < XR;
    const int l = isx ? l0 - (KW - 1) + r : l0 + (r - XR);
    T* dst = isx ? &xs[r][pc * V] : &gs[r - XR][pc * V];
    if (l >= 0 && l < L) {
      const long long ph = rev ? L - 1 - l : l;
      cp_async16_conv(dst, isx ? xb + ph * p.x.s1 + pc * V : gb + ph * p.dout.s1 + pc * V);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int c = 2 * threadIdx.x;
  const int e = e0 + c;
  const int l1 = min(L, l0 + TT);
  auto ld2 = [&](const T* row) -> f2 {
    if constexpr (sizeof(T) == 4) {
      const float2 v = *reinterpret_cast<const float2*>(row + c);
      return mk2(v.x, v.y);
    } else {
      const unsigned u = *reinterpret_cast<const unsigned*>(row + c);
      return mk2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
    }
  };
  f2 w[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) w[q] = mk2(p.w[(long long)e * K + q], p.w[(long long)(e + 1) * K + q]);
  const f2 bias = p.bias ? mk2(p.bias[e], p.bias[e + 1]) : mk2(0.f, 0.f);
  f2 xw[2 * KW];  // xw[i] = x[l - (KW-1) + i]
#pragma unroll
  for (int i = 0; i < 2 * KW; ++i) xw[i] = ld2(xs[i]);  // rows l0-(KW-1)+i -> xs row i
  auto Gw = [&](int l, int off) -> f2 {
    if (l + off >= L) return mk2(0.f, 0.f);
    f2 gv = ld2(gs[l + off - l0]);
    if (act) {
      f2 xc = bias;
#pragma unroll
      for (int q = 0; q < KW; ++q) xc = fma2(w[q], xw[KW - 1 + off - q], xc);
      const float s0 = sigmoid_f(xc.x), s1 = sigmoid_f(xc.y);
      gv.x *= s0 * (1.f + xc.x * (1.f - s0));
      gv.y *= s1 * (1.f + xc.y * (1.f - s1));
    }
    return gv;
  };
  f2 dw[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) dw[q] = mk2(0.f, 0.f);
  f2 db = mk2(0.f, 0.f);
  f2 fut[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q) fut[q] = Gw(l0, q);
#pragma unroll 4
  for (int l = l0; l < l1; ++l) {
    f2 acc = mk2(0.f, 0.f);
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) acc = fma2(w[q], fut[q], acc);
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float2*>(&dxo[l - l0][c]) = make_float2(acc.x, acc.y);
    } else {
      *reinterpret_cast<__nv_bfloat162*>(&dxo[l - l0][c]) = __floats2bfloat162_rn(acc.x, acc.y);
    }
    const f2 g0 = fut[0];
    db = add2(db, g0);
#pragma unroll
    for (int q = 0; q < KW; ++q) dw[q] = fma2(g0, xw[KW - 1 - q], dw[q]);
#pragma unroll
    for (int q = 0; q < KW - 1; ++q) fut[q] = fut[q + 1];
    fut[K - 1] = Gw(l, K);
#pragma unroll
    for (int i = 0; i < 2 * KW - 1; ++i) xw[i] = xw[i + 1];
    xw[2 * KW - 1] = ld2(xs[l + KW + 1 - l0 + (KW - 1)]);
  }
  float* part = p.part + (((long long)b * p.n_chunks + chunk) * p.E + e) * (K + 1);
#pragma unroll
  for (int q = 0; q < K; ++q) {
    part[q] = dw[q].x;
    part[(K + 1) + q] = dw[q].y;
  }
  part[K] = db.x;
  part[(K + 1) + K] = db.y;
  __syncthreads();
  T* ob = static_cast<T*>(p.dx) + (long long)b * p.sd0 + e0;
  for (int i = threadIdx.x; i < (l1 - l0) * PPR; i += NT) {
    const int j = i / PPR, pc = i % PPR;
    const int l = l0 + j;
    *reinterpret_cast<uint4*>(ob + (long long)(rev ? L - 1 - l : l) * p.sd1 + pc * V) =
        *reinterpret_cast<const uint4*>(&dxo[j][pc * V]);
  }
}

// deterministic reduction of the (B * n_chunks) partials -> dweight, dbias (+=).
// A 1024-thread block owns 32 consecutive (e, q) outputs: 32 slices of threads
// each sum every 32nd partial (fp64, fixed order, 4 loads in flight), then the
// 32 slice sums are added in fixed order.  (One thread per output walking all
// partials serially was a ~900-deep load chain: 134 us at the LBVim-S shape.)
constexpr int kRedSlices = 32;
__global__ void __launch_bounds__(32 * kRedSlices) conv_reduce_kernel(const float* part, int n_part, int E, int K,
                                                                       float* dw, float* db) {
  __shared__ double acc[kRedSlices][33];
  const int lane = threadIdx.x % 32, slice = threadIdx.x / 32;
  const int idx = blockIdx.x * 32 + lane;
  const int n = E * (K + 1);
  double s = 0.0;
  if (idx < n) {
    const long long stride = (long long)n;
    int i = slice;
    for (; i + 3 * kRedSlices < n_part; i += 4 * kRedSlices) {
      const float a0 = part[(long long)i * stride + idx];
      const float a1 = part[(long long)(i + kRedSlices) * stride + idx];
      const float a2 = part[(long long)(i + 2 * kRedSlices) * stride + idx];
      const float a3 = part[(long long)(i + 3 * kRedSlices) * stride + idx];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; i < n_part; i += kRedSlices) s += part[(long long)i * stride + idx];
  }
  acc[slice][lane] = s;
  __syncthreads();
  if (slice == 0 && idx < n) {
    double t = 0.0;
#pragma unroll 8
    for (int k = 0; k < kRedSlices; ++k) t += acc[k][lane];
    const int e = idx / (K + 1), q = idx - e * (K + 1);
    if (q < K) dw[(long long)e * K + q] += (float)t;
    else if (db) db[e] += (float)t;
  }
}

// Streaming forward (16-byte aligned rows, E % 128 == 0): a 64-thread CTA owns
// 128 channels (two per thread) of one batch row over a range of `rows` logical
// steps and streams it through a 2-stage cp.async ring of kConvST rows -- the
// next chunk's loads are in flight while the current chunk is computed, the
// K-1 history stays in registers across chunks (no halo reload), and each
// thread stores its channel pair per step (a warp writes 128 contiguous bytes).
// Replaces the one-shot tile kernel (load -> barrier -> compute -> barrier ->
// store per 32-step tile), whose per-CTA fill and drain left the LBVim-Ti
// layer shape at 0.46 of HBM (tools/convbench.py).
constexpr int kConvST = 32;
template <typename T, int KW>
__global__ void __launch_bounds__(64) conv_fwd_stream_kernel(ConvParams p, int rows) {
  constexpr int TE = 128, NT = 64;
  constexpr int V = 16 / sizeof(T);
  constexpr int PPR = TE / V;  // 16-byte pieces per row
  __shared__ __align__(16) T ring[2][kConvST][TE];
  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * TE;
  const int b = blockIdx.z;
  const int L = p.L;
  const int lb = blockIdx.y * rows;
  const int le = min(L, lb + rows);
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool act = p.flags & LBS_CONV_SILU;
  const T* xb = static_cast<const T*>(p.x.p) + (long long)b * p.x.s0 + e0;
  T* ob = static_cast<T*>(p.out) + (long long)b * p.so0 + e0;
  auto phys = [&](int l) -> long long { return rev ? (long long)(L - 1 - l) : (long long)l; };
  auto issue = [&](int stg, int l0) {
#pragma unroll
    for (int i0 = 0; i0 < kConvST * PPR; i0 += NT) {
      const int i = i0 + tid;
      const int r = i / PPR, pc = i % PPR;
      if (l0 + r < le) cp_async16_conv(&ring[stg][r][pc * V], xb + phys(l0 + r) * p.x.s1 + pc * V);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if (lb >= le) return;
  issue(0, lb);
  const int c = 2 * tid;
  const int e = e0 + c;
  f2 w[KW];
#pragma unroll
  for (int q = 0; q < KW; ++q)
    w[q] = q < p.K ? mk2(p.w[(long long)e * p.K + q], p.w[(long long)(e + 1) * p.K + q]) : mk2(0.f, 0.f);
  const f2 bias = p.bias ? mk2(p.bias[e], p.bias[e + 1]) : mk2(0.f, 0.f);
  f2 hist[KW];  // hist[q] = x[l - q] for the two channels
  hist[0] = mk2(0.f, 0.f);
#pragma unroll
  for (int q = 1; q < KW; ++q) {
    const int l = lb - q;
    hist[q] = (q < p.K && l >= 0) ? mk2(ld<T>(xb + phys(l) * p.x.s1 + c), ld<T>(xb + phys(l) * p.x.s1 + c + 1))
                                  : mk2(0.f, 0.f);
  }
  const long long os = rev ? -p.so1 : p.so1;
  T* op = ob + phys(lb) * p.so1 + c;
  for (int l0 = lb, k = 0; l0 < le; l0 += kConvST, ++k) {
    const int stg = k & 1;
    if (l0 + kConvST < le) issue(stg ^ 1, l0 + kConvST);
    else asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();  // chunk k visible to all threads
    const int n = min(kConvST, le - l0);
#pragma unroll 8
    for (int j = 0; j < n; ++j) {
      if constexpr (sizeof(T) == 4) {
        const float2 v = *reinterpret_cast<const float2*>(&ring[stg][j][c]);
        hist[0] = mk2(v.x, v.y);
      } else {
        const unsigned u = *reinterpret_cast<const unsigned*>(&ring[stg][j][c]);
        hist[0] = mk2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
      }
      f2 acc = bias;
#pragma unroll
      for (int q = KW - 1; q >= 0; --q) acc = fma2(w[q], hist[q], acc);
      if (act) acc = mk2(silu_f(acc.x), silu_f(acc.y));
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float2*>(op) = make_float2(acc.x, acc.y);
      } else {
        *reinterpret_cast<__nv_bfloat162*>(op) = __floats2bfloat162_rn(acc.x, acc.y);
      }
      op += os;
#pragma unroll
      for (int q = KW - 1; q >= 1; --q) hist[q] = hist[q - 1];
    }
    __syncthreads();  // all reads of stage stg done before it is refilled
  }
}

template <typename T>
static bool conv_vec_ok(const ConvParams& p) {
  constexpr int V = 16 / sizeof(T);
  auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  return p.E % V == 0 && p.x.s2 == 1 && p.so2 == 1 && al(p.x.p) && al(p.out) && p.x.s0 % V == 0 &&
         p.x.s1 % V == 0 && p.so0 % V == 0 && p.so1 % V == 0;
}

template <typename T>
static bool conv_bwd_vec_ok(const ConvParams& p) {
  constexpr int V = 16 / sizeof(T);
  auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  return p.E % V == 0 && p.x.s2 == 1 && p.dout.s2 == 1 && p.sd2 == 1 && al(p.x.p) && al(p.dout.p) && al(p.dx) &&
         p.x.s0 % V == 0 && p.x.s1 % V == 0 && p.dout.s0 % V == 0 && p.dout.s1 % V == 0 && p.sd0 % V == 0 &&
         p.sd1 % V == 0;
}

template <typename T>
static cudaError_t conv_fwd_t(const ConvParams& p, cudaStream_t st) {
  if constexpr (std::is_same<T, float>::value || std::is_same<T, __nv_bfloat16>::value) {
    if (conv_vec_ok<T>(p) && p.E % kConvTE == 0) {
      // rows per CTA: split L so that ~8 CTAs per SM are resident over the grid
      const long long units = (long long)(p.E / kConvTE) * p.Bt;
      long long splits = ((long long)LBS_CONV_CTAS_PER_SM * conv_num_sms() + units - 1) / units;
      const long long max_splits = (p.L + kConvST - 1) / kConvST;
      if (splits > max_splits) splits = max_splits;
      if (splits < 1) splits = 1;
      int rows = (int)((p.L + splits - 1) / splits);
      dim3 grid(p.E / kConvTE, (unsigned)((p.L + rows - 1) / rows), p.Bt);
      if (p.K <= 4) conv_fwd_stream_kernel<T, 4><<<grid, 64, 0, st>>>(p, rows);
      else conv_fwd_stream_kernel<T, kMaxWidth><<<grid, 64, 0, st>>>(p, rows);
      return cudaGetLastError();
    }
  }
  if (conv_vec_ok<T>(p)) {
    dim3 grid((p.E + kConvTE - 1) / kConvTE, (p.L + kConvTT - 1) / kConvTT, p.Bt);
    if (p.K <= 4) conv_fwd_tile_kernel<T, 4><<<grid, kConvTE, 0, st>>>(p);
    else conv_fwd_tile_kernel<T, kMaxWidth><<<grid, kConvTE, 0, st>>>(p);
    return cudaGetLastError();
  }
  dim3 grid((p.E + kConvThreads - 1) / kConvThreads, (p.L + kConvChunk - 1) / kConvChunk, p.Bt);
  if (p.K <= 4) conv_fwd_kernel<T, 4><<<grid, kConvThreads, 0, st>>>(p);
  else conv_fwd_kernel<T, kMaxWidth><<<grid, kConvThreads, 0, st>>>(p);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t conv_bwd_t(const ConvParams& p, float* dw, float* db, cudaStream_t st) {
  dim3 grid((p.E + kConvThreads - 1) / kConvThreads, (p.L + kConvChunk - 1) / kConvChunk, p.Bt);
  bool done = false;
  if constexpr (std::is_same<T, float>::value || std::is_same<T, __nv_bfloat16>::value) {
    if (conv_bwd_vec_ok<T>(p) && p.K == 4 && p.E % 128 == 0) {
      dim3 gt(p.E / 128, (p.L + kConvChunk - 1) / kConvChunk, p.Bt);
      conv_bwd_tile2_kernel<T><<<gt, 64, 0, st>>>(p);
      done = true;
    }
  }
  if (done) {
  } else if (conv_bwd_vec_ok<T>(p) && p.K == 4) {
    dim3 gt((p.E + kConvBE - 1) / kConvBE, (p.L + kConvChunk - 1) / kConvChunk, p.Bt);
    conv_bwd_tile_kernel<T, 4><<<gt, kConvBE, 0, st>>>(p);
  } else if (p.K <= 4) {
    conv_bwd_kernel<T, 4><<<grid, kConvThreads, 0, st>>>(p);
  } else {
    conv_bwd_kernel<T, kMaxWidth><<<grid, kConvThreads, 0, st>>>(p);
  }
  const int n = p.E * (p.K + 1);
  conv_reduce_kernel<<<(n + 31) / 32, 32 * kRedSlices, 0, st>>>(p.part, p.Bt * p.n_chunks, p.E, p.K, dw, db);
  return cudaGetLastError();
}

cudaError_t launch_conv_fwd(const ConvParams& p, int dtype, cudaStream_t st) {
  if (dtype == LBS_F32) return conv_fwd_t<float>(p, st);
  if (dtype == LBS_BF16) return conv_fwd_t<__nv_bfloat16>(p, st);
  return conv_fwd_t<__half>(p, st);
}

cudaError_t launch_conv_bwd(const ConvParams& p, int dtype, float* dw, float* db, cudaStream_t st) {
  if (dtype == LBS_F32) return conv_bwd_t<float>(p, dw, db, st);
  if (dtype == LBS_BF16) return conv_bwd_t<__nv_bfloat16>(p, dw, db, st);
  return conv_bwd_t<__half>(p, dw, db, st);
}

}  // namespace lbs

// ---------------------------------------------------------------------------
// C ABI

namespace {
int conv_validate(const lbs_conv_args* a, bool bwd, std::string* err) {
  if (!a) { *err = "null args"; return LBS_ERR_INVALID; }
  if (a->batch < 1 || a->seqlen < 1 || a->dim < 1 || a->width < 1) {
    *err = "all dimensions must be >= 1";
    return LBS_ERR_INVALID;
  }
  if (a->width > lbs::kMaxWidth) { *err = "conv width > 8 unsupported"; return LBS_ERR_UNSUPPORTED; }
  if (a->io_dtype != LBS_F32 && a->io_dtype != LBS_BF16 && a->io_dtype != LBS_F16) {
    *err = "bad dtype";
    return LBS_ERR_INVALID;
  }
  if (a->batch > 65535) { *err = "batch > 65535"; return LBS_ERR_UNSUPPORTED; }
  if (!a->x || !a->weight) { *err = "x and weight must be non-null"; return LBS_ERR_INVALID; }
  if (!bwd && !a->out) { *err = "out must be non-null"; return LBS_ERR_INVALID; }
  if (bwd && (!a->dout || !a->dx || !a->dweight)) { *err = "dout, dx, dweight must be non-null"; return LBS_ERR_INVALID; }
  return LBS_OK;
}

lbs::ConvParams conv_params(const lbs_conv_args* a) {
  lbs::ConvParams p{};
  p.Bt = (int)a->batch;
  p.L = (int)a->seqlen;
  p.E = (int)a->dim;
  p.K = (int)a->width;
  p.flags = a->flags;
  p.x = lbs::View3D{a->x, a->x_stride[0], a->x_stride[1], a->x_stride[2]};
  p.dout = lbs::View3D{a->dout, a->dout_stride[0], a->dout_stride[1], a->dout_stride[2]};
  p.out = a->out;
  p.so0 = a->out_stride[0]; p.so1 = a->out_stride[1]; p.so2 = a->out_stride[2];
  p.dx = a->dx;
  p.sd0 = a->dx_stride[0]; p.sd1 = a->dx_stride[1]; p.sd2 = a->dx_stride[2];
  p.w = a->weight;
  p.bias = a->bias;
  p.n_chunks = (int)((a->seqlen + lbs::kConvChunk - 1) / lbs::kConvChunk);
  return p;
}
}  // namespace

extern "C" int lbs_set_error(int code, const char* msg);

extern "C" size_t lbs_causal_conv1d_bwd_workspace_bytes(const lbs_conv_args* a) {
  std::string err;
  if (conv_validate(a, true, &err) != LBS_OK) return 0;
  const size_t nch = (a->seqlen + lbs::kConvChunk - 1) / lbs::kConvChunk;
  return (size_t)a->batch * nch * a->dim * (a->width + 1) * sizeof(float);
}

extern "C" int lbs_causal_conv1d_fwd(const lbs_conv_args* a, void* stream) {
  std::string err;
  int rc = conv_validate(a, false, &err);
  if (rc != LBS_OK) return lbs_set_error(rc, err.c_str());
  lbs::ConvParams p = conv_params(a);
  cudaError_t e = lbs::launch_conv_fwd(p, a->io_dtype, (cudaStream_t)stream);
  if (e != cudaSuccess) return lbs_set_error(LBS_ERR_CUDA, cudaGetErrorString(e));
  return LBS_OK;
}

extern "C" int lbs_causal_conv1d_bwd(const lbs_conv_args* a, void* ws, size_t ws_bytes, void* stream) {
  std::string err;
  int rc = conv_validate(a, true, &err);
  if (rc != LBS_OK) return lbs_set_error(rc, err.c_str());
  const size_t need = lbs_causal_conv1d_bwd_workspace_bytes(a);
  if (!ws || ws_bytes < need) return lbs_set_error(LBS_ERR_INVALID, "conv bwd workspace too small");
  lbs::ConvParams p = conv_params(a);
  p.part = static_cast<float*>(ws);
  cudaError_t e = lbs::launch_conv_bwd(p, a->io_dtype, a->dweight, a->dbias, (cudaStream_t)stream);
  if (e != cudaSuccess) return lbs_set_error(LBS_ERR_CUDA, cudaGetErrorString(e));
  return LBS_OK;
}
