// Internal (host+device) parameter blocks shared by the kernels and the C ABI layer.
#pragma once

#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>
#include <stdint.h>

namespace lbs {

// TMA tensor maps of the forward's staged inputs (u, delta, z, B, C), each 3-D
// (inner dim, L, B), encoded on the host per call (lbs_capi.cu) and passed to
// the kernel as a __grid_constant__ parameter.
struct alignas(64) FwdTmaMaps {
  CUtensorMap tm[5];
};

constexpr int kFwdThreads = 128;  // channels per CTA
constexpr int kFwdChunk = 64;     // steps of B/C staged in shared memory per chunk

struct View3D {
  const void* p;
  long long s0, s1, s2;
};

struct FwdParams {
  int Bt, L, E, N, m;
  uint32_t flags;
  View3D u, delta, z, Bm, Cm;
  void* out;
  long long so0, so1, so2;
  const float* A;
  const float* D;
  const float* bias;
  float* last_state;
  // CTA width (128, or 64 for low channel parallelism) and sequence split
  int cta;
  int n_seg, seg_len;
  float* seg_agg;  // (Bt, n_seg, E, 2*NS) fp32 workspace
  // training checkpoints (state entering each ckpt chunk)
  float* ckpt;
  int ckpt_len, n_ckpt;
  // TMA staging (host pointer, read by the launcher only; nullptr: cp.async staging)
  const FwdTmaMaps* tma_maps;
};
// whether the forward's TMA staging is compiled in (LBS_FWD_TMA)
bool fwd_tma_enabled();

cudaError_t launch_fwd(const FwdParams& p, int io_dtype, int bc_dtype, cudaStream_t st);
int fwd_padded_states(int N);  // NS used by the kernels for a given N

struct OutView {
  void* p;
  long long s0, s1, s2;
};

// Backward: the forward's parameters (f.out unused) plus gradients.
// f.ckpt must hold the checkpoints (state entering every bwd chunk of
// f.ckpt_len steps) — written by the forward or by a checkpoint-only sweep.
struct BwdParams {
  FwdParams f;
  View3D dout;
  OutView du, ddelta, dz;  // io dtype; dz.p == nullptr iff no gate
  float* part_bc;          // [n_eblk][Bt][L][2][NS] dB/dC partials per channel block
  float* part_w;           // [Bt*n_seg][NS+2][E] per-(row, segment) dA (NS), dD, ddelta_bias partials
  // sequence split (few channels): segment s = chunks [s*seg_chunks, (s+1)*seg_chunks);
  // bagg[(b*n_seg + s)*E + e][2*NS] = (P, M) of segment s: the carry mu = a*lam leaving
  // the segment to the left is mu_out = P*mu_in + M (P = prod a over the segment)
  int n_seg, seg_chunks;
  float* bagg;
  // final outputs (reduction kernel)
  float* dA;               // (E, N)  +=
  float* dD;               // (E) or nullptr, +=
  float* dbias;            // (E) or nullptr, +=
  float* dB;
  long long sb0, sb1, sb2;
  float* dC;
  long long sc0, sc1, sc2;
};

cudaError_t launch_bwd(const BwdParams& p, int io_dtype, int bc_dtype, cudaStream_t st);
int bwd_chunk_len(int m);  // steps per backward chunk (= checkpoint spacing) for window m

// Generic fused path (lbs_generic.cu): windows min(M, L) > 16 or N > 16.
size_t gen_fwd_workspace_floats(int Bt, int L, int E);
size_t gen_bwd_workspace_floats(int Bt, int L, int E, int N);
cudaError_t launch_fwd_generic(const FwdParams& p, float* ws, int io_dtype, int bc_dtype, cudaStream_t st);
// BwdParams.part_w must point at gen_bwd_workspace_floats - 7 B L E floats past ws
cudaError_t launch_bwd_generic(const BwdParams& P, float* ws, int io_dtype, int bc_dtype, cudaStream_t st);

struct PreParams {
  int Bt, L, E, N, m;
  uint32_t flags;
  const void* abar;
  const void* bx;
  const void* c;
  const void* dx;
  void* y;
  void* h_final;
};
cudaError_t launch_prediscretized(const PreParams& p, bool f64, cudaStream_t st);

struct NormParams {
  long long rows;
  int D;
  float eps;
  const void* x;
  long long sx;
  const float* scale;
  void* out;
  long long so;
};
cudaError_t launch_rms_norm(const NormParams& p, int dtype, int out_dtype, cudaStream_t st);

struct NormBwdParams {
  long long rows;
  int D;
  float eps;
  const void* x;
  long long sx;
  const float* scale;
  const void* dout;
  long long sg;
  void* dx;
  long long sdx;
  float* dscale;
  float* part;  // (n_warps, D) fp32 dscale partials
  int n_warps;
  const void* dres;  // optional residual gradient added to dx (io dtype)
  long long sres;
};
int norm_bwd_warps(long long rows);
cudaError_t launch_rms_norm_bwd(const NormBwdParams& p, int dtype, cudaStream_t st);

}  // namespace lbs
