/*
 * lbscan_b200 — C ABI of the B200-native locally bi-directional (LB) selective scan.
 *
 * One shared library (paper_2506_15976_b200/liblbscan_b200.so).  Plain pointers,
 * sizes and element strides; no torch types.  Every entry point is
 * stream-ordered: it validates arguments on the host, enqueues kernels on the
 * caller's stream and returns without synchronising.  The caller owns every
 * buffer (outputs and workspace); the library keeps no global device state and
 * is re-entrant per stream.  Errors are returned, never thrown:
 *   LBS_OK (0) | LBS_ERR_INVALID (1, maps to the reference's ShapeError)
 *   | LBS_ERR_CUDA (2, RuntimeError) | LBS_ERR_UNSUPPORTED (3).
 * lbs_last_error() returns a thread-local message for the last failure.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/lbscan):
 *   lbs_scan_fwd            <- block._run_scan (block.py:132-138) + engine.lbm_scan_par
 *                              (engine.py:299-302) with block._discretize_cached
 *                              (block.py:87-103) and the gate (block.py:177-178) fused;
 *                              LBS_FLAG_REVERSE replaces the reverse copies
 *                              (block.py:180-181) by flip-on-load (engine.py:133,183).
 *                              Without LBS_FLAG_LB it is engine.forward_scan_par (engine.py:294).
 *   lbs_scan_bwd            <- autodiff.lbm_scan_grad (autodiff.py:192-195) chained through
 *                              block._discretize_backward (block.py:106-129) and the gate
 *                              adjoint (block.py:199-200).
 *   lbs_prediscretized_fwd  <- engine.lbm_scan_par / forward_scan_par on (abar, bx, c, dx)
 *                              (engine.py:294-302) — debug/parity entry.
 *   lbs_causal_conv1d_silu_fwd/bwd <- nn.causal_conv1d + nn.silu (nn.py:87-99,25-26) and
 *                              nn.causal_conv1d_grad + silu_grad (nn.py:102-114,29-31).
 *   lbs_select_tile_len     <- engine.select_tile_len (engine.py:54-62).
 *   lbs_rms_norm_fwd        <- nn.rms_norm (nn.py:55-58), the block's first op (block.py:170).
 *   lbs_rms_norm_bwd        <- its adjoint in block_backward (block.py:193-220).
 *
 * Layout: sequence tensors are addressed as element (b, l, e) at
 *   base + b*stride[0] + l*stride[1] + e*stride[2]      (reference: channel-last (B,L,E))
 * and the per-step projections B, C as (b, l, n).  A is (E, N) fp32 row-major;
 * D and delta_bias are (E) fp32.  States are (B, E, N) fp32.
 */
#ifndef LBSCAN_B200_H
#define LBSCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBS_ABI_VERSION 2

enum lbs_status { LBS_OK = 0, LBS_ERR_INVALID = 1, LBS_ERR_CUDA = 2, LBS_ERR_UNSUPPORTED = 3 };
enum lbs_dtype { LBS_F32 = 0, LBS_BF16 = 1, LBS_F16 = 2, LBS_F64 = 3 };

/* flags */
#define LBS_FLAG_REVERSE   (1u << 0) /* scan right-to-left, tiles aligned from the right end   */
#define LBS_FLAG_SOFTPLUS  (1u << 1) /* delta := softplus(delta + delta_bias)                  */
#define LBS_FLAG_LB        (1u << 2) /* add the tile-local backward record (LBMamba); else fwd */
#define LBS_FLAG_LINEAR    (1u << 3) /* discretize_mode="linear": abar = delta*A (block.py:94)  */
#define LBS_FLAG_NO_TMA    (1u << 6) /* testing: stage the forward's inputs with cp.async rows
                                        instead of TMA tensor copies (bitwise-equal results) */
#define LBS_FLAG_ACCUM     (1u << 5) /* out += result (second sweep of the global-bidirectional
                                        baseline, engine.global_bidir_par, engine.py:305-327);
                                        forward-only scans (not with LBS_FLAG_LB)              */

/* Fused LB selective scan, forward.
 * out[b,l,e] = (sum_n C[b,l,n] (h + r)[b,l,e,n] + D[e] u[b,l,e]) * silu(z[b,l,e])
 * with h the forward state and r the exclusive tile-local backward record over
 * tiles of `window` steps (SURVEY.md §8 "exact math").                                   */
typedef struct lbs_scan_fwd_args {
  int64_t batch, seqlen, dim, dstate, window;
  int32_t io_dtype;      /* dtype of u, delta, z, out            */
  int32_t bc_dtype;      /* dtype of B, C                        */
  uint32_t flags;
  int32_t seg_hint;      /* 0 = auto; >0 forces that many sequence segments (testing)    */
  const void* u;      int64_t u_stride[3];
  const void* delta;  int64_t delta_stride[3];
  const float* A;                             /* (E, N) fp32          */
  const void* B;      int64_t B_stride[3];    /* (b, l, n)            */
  const void* C;      int64_t C_stride[3];    /* (b, l, n)            */
  const float* D;                             /* (E) or NULL          */
  const float* delta_bias;                    /* (E) or NULL          */
  const void* z;      int64_t z_stride[3];    /* or NULL: no gate     */
  void* out;          int64_t out_stride[3];
  float* last_state;                          /* (B, E, N) or NULL    */
  /* Training checkpoints for lbs_scan_bwd: NULL, or lbs_scan_ckpt_bytes() of fp32
   * (opaque layout: the state entering every backward chunk).  ckpt_len must equal
   * lbs_scan_ckpt_len(seqlen, window).  With checkpoints != NULL, out may be NULL
   * (checkpoint-only sweep).                                                       */
  float* checkpoints;
  int64_t ckpt_len;
} lbs_scan_fwd_args;

/* Fused LB selective scan, backward (autodiff.lbm_scan_grad chained through
 * block._discretize_backward and the gate).  Inputs as in the forward plus dout;
 * fwd.checkpoints from the training forward (or NULL: a checkpoint-only forward
 * sweep runs first, into the workspace).  fwd.out / fwd.last_state are ignored.
 * Outputs: du, ddelta, dz in the io dtype (dz given iff z is), flip-on-store for
 * LBS_FLAG_REVERSE; dA (E,N), dD (E), ddelta_bias (E) fp32, ACCUMULATED (+=) so
 * several calls can share one gradient buffer (dD / ddelta_bias may be NULL);
 * dB, dC (b,l,n) fp32, written.  Deterministic: all reductions are fixed-order
 * partial sums (no atomics).                                                       */
typedef struct lbs_scan_bwd_args {
  lbs_scan_fwd_args fwd;   /* fwd.out / fwd.last_state are ignored */
  const void* dout;   int64_t dout_stride[3];
  void* du;           int64_t du_stride[3];
  void* ddelta;       int64_t ddelta_stride[3];
  void* dz;           int64_t dz_stride[3];
  float* dA;
  float* dD;
  float* ddelta_bias;
  float* dB;          int64_t dB_stride[3];
  float* dC;          int64_t dC_stride[3];
} lbs_scan_bwd_args;

/* Pre-discretised scan (engine.lbm_scan_par / forward_scan_par): abar, bx (B,L,E,N);
 * c (B,L,N); dx (B,L,E); y (B,L,E); h_final (B,E,N).  Contiguous, dtype LBS_F32 or
 * LBS_F64 (fp64 runs the reference's 1e-12 structural tests on the GPU).  N <= 64.    */
typedef struct lbs_prediscretized_args {
  int64_t batch, seqlen, dim, dstate, window;
  uint32_t flags;          /* LBS_FLAG_LB, LBS_FLAG_REVERSE */
  int32_t dtype;
  const void* abar; const void* bx; const void* c; const void* dx;
  void* y; void* h_final;
} lbs_prediscretized_args;

/* Depthwise causal conv1d (+ optional SiLU), channel-last.  weight is (E, K) in the
 * reference's tap order: out[l] = sum_q w[e,q] x[l-q] (q counts back in time).
 * REVERSE flips time on load/store so a reverse-direction layer needs no copy.        */
typedef struct lbs_conv_args {
  int64_t batch, seqlen, dim, width;
  int32_t io_dtype;
  uint32_t flags;          /* LBS_FLAG_REVERSE; bit 4 = apply SiLU */
  const void* x;   int64_t x_stride[3];
  const float* weight;     /* (E, K) fp32 */
  const float* bias;       /* (E) or NULL */
  void* out;       int64_t out_stride[3];
  /* backward only */
  const void* dout; int64_t dout_stride[3];
  void* dx;         int64_t dx_stride[3];
  float* dweight;          /* (E, K) fp32, accumulated (+=) */
  float* dbias;            /* (E) fp32 or NULL, accumulated */
} lbs_conv_args;
#define LBS_CONV_SILU (1u << 4)

/* RMSNorm with learned scale (nn.rms_norm, nn.py:55-58): out = x / sqrt(mean(x^2) + eps) * scale,
 * over rows of `dim` contiguous elements.  dim % (16/sizeof(elem)) == 0, rows 16-byte aligned. */
typedef struct lbs_norm_args {
  int64_t rows, dim;
  int32_t io_dtype;
  float eps;
  const void* x;   int64_t x_row_stride;
  const float* scale;       /* (dim) fp32 */
  void* out;       int64_t out_row_stride;
  int32_t out_dtype;        /* ABI 2: dtype of out (LBS_F32 / LBS_BF16); may differ from io_dtype
                               only as f32 in -> bf16 out (the bf16 GEMM input of an fp32
                               residual stream, no separate cast)                              */
} lbs_norm_args;

int lbs_abi_version(void);
const char* lbs_last_error(void);
int64_t lbs_select_tile_len(int64_t seqlen);

/* Steps between training checkpoints (= the backward's chunk) for a window, and the
 * checkpoint buffer size for a forward call; -1 / 0 when the window is unsupported. */
int64_t lbs_scan_ckpt_len(int64_t seqlen, int64_t window);
size_t lbs_scan_ckpt_bytes(const lbs_scan_fwd_args* args);

size_t lbs_scan_fwd_workspace_bytes(const lbs_scan_fwd_args* args);
int lbs_scan_fwd(const lbs_scan_fwd_args* args, void* workspace, size_t workspace_bytes,
                 void* cuda_stream);

size_t lbs_scan_bwd_workspace_bytes(const lbs_scan_bwd_args* args);
int lbs_scan_bwd(const lbs_scan_bwd_args* args, void* workspace, size_t workspace_bytes,
                 void* cuda_stream);

int lbs_prediscretized_fwd(const lbs_prediscretized_args* args, void* cuda_stream);

int lbs_rms_norm_fwd(const lbs_norm_args* args, void* cuda_stream);

/* RMSNorm backward (the adjoint of nn.rms_norm, nn.py:55-58, as the reference's
 * block_backward chains it, block.py:193-220): with r = 1/sqrt(mean(x^2) + eps) and
 * g = dout * scale per row, dx = r g - x r^3 mean(g x); dscale += sum over rows of
 * dout x r (fp32, fixed-order reduction through the workspace: deterministic).
 * Any row stride; 16-byte aligned rows with dim <= 128 * (16 / sizeof(elem)) take the
 * vector kernel. */
typedef struct lbs_norm_bwd_args {
  int64_t rows, dim;
  int32_t io_dtype;
  float eps;
  const void* x;     int64_t x_row_stride;
  const float* scale;         /* (dim) fp32 */
  const void* dout;  int64_t dout_row_stride;
  void* dx;          int64_t dx_row_stride;
  float* dscale;              /* (dim) fp32, accumulated (+=); NULL to skip */
  const void* dres;  int64_t dres_row_stride;  /* ABI 2: optional residual gradient (io dtype)
                                                  added to dx: dx = norm adjoint + dres */
} lbs_norm_bwd_args;
size_t lbs_rms_norm_bwd_workspace_bytes(const lbs_norm_bwd_args* args);
int lbs_rms_norm_bwd(const lbs_norm_bwd_args* args, void* workspace, size_t workspace_bytes,
                     void* cuda_stream);

size_t lbs_causal_conv1d_bwd_workspace_bytes(const lbs_conv_args* args);
int lbs_causal_conv1d_fwd(const lbs_conv_args* args, void* cuda_stream);
int lbs_causal_conv1d_bwd(const lbs_conv_args* args, void* workspace, size_t workspace_bytes,
                          void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* LBSCAN_B200_H */
