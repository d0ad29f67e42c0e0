// C ABI layer: argument validation (host), sequence-split planning, dispatch.
// Error behaviour mirrors the reference: shape/plan problems are
// LBS_ERR_INVALID, which the Python host maps to lbscan's ShapeError
// (core.py:24-25, engine.py:56-57,221-243); the hot path does not scan for
// NaN (the reference engine does not either, engine.py:221-236).
#include <cstdarg>
#include <cstdio>
#include <string>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#ifndef LBS_FWD_TMA_BF16
#define LBS_FWD_TMA_BF16 0
#endif

#include "lbs_common.cuh"
#include "lbs_internal.h"

extern "C" int64_t lbs_scan_ckpt_len(int64_t seqlen, int64_t window);
extern "C" size_t lbs_scan_ckpt_bytes(const lbs_scan_fwd_args* a);

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return LBS_OK;
  return fail(LBS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool io_dtype_ok(int d) { return d == LBS_F32 || d == LBS_BF16 || d == LBS_F16; }

// SM count of the current device (148 on B200; MIG slices and other SKUs
// differ), queried once per device ordinal
int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int n = cache[dev];
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return n;
}

// states padded per thread (kernels instantiate NS in {4, 16})
int padded_states(int64_t N) { return N <= 4 ? 4 : 16; }

// Launch plan of the forward.
//  * CTA width: 128 channels, or 64 when channels are scarce (E <= 64, or fewer
//    than two 128-wide CTAs per SM) — no idle threads, finer balance over SMs.
//  * Sequence split: cut L into S segments (multiples of the window) only when
//    B*E alone cannot fill the machine (~8 resident warps per SM); each extra
//    segment costs one aggregate pass over its steps, so S stays minimal.  The
//    segments are stitched by a parallel prefix over their aggregates.
void plan_fwd(const lbs_scan_fwd_args* a, int* cta, int* n_seg, int* seg_len) {
  const int64_t L = a->seqlen, m = a->window < a->seqlen ? a->window : a->seqlen;
  const int64_t ctas128 = ((a->dim + 127) / 128) * a->batch;
  const int sms = num_sms();
  *cta = (a->dim <= 64 || ctas128 < 2 * sms) ? 64 : 128;
  const int64_t warps = ((a->dim + 31) / 32) * a->batch;
  int64_t S = 1;
  if (a->seg_hint > 0) {
    S = a->seg_hint;
  } else if (warps < 4 * sms && L >= 1024) {
    // few channels, long L: the serial per-channel sweep leaves the SMs
    // latency-bound; split L so ~8 warps per SM run (segments >= 128 steps)
    S = (8 * sms + warps - 1) / warps;
    const int64_t max_s = L / 128;
    if (S > max_s) S = max_s;
    if (S > 2048) S = 2048;
    if (S < 1) S = 1;
  } else if (4 * warps < sms) {
    // short L and less than one warp per SM sub-partition (configs[0]): a few
    // segments (each costs an aggregate pass over its steps; measured best at
    // 8 for configs[0], 49 -> 31 us; at a few warps per SM no split pays,
    // tools/segsweep.py)
    S = 8;
    const int64_t max_s = (L + 2 * m - 1) / (2 * m);  // >= 2 tiles per segment
    if (S > max_s) S = max_s;
    if (S < 1) S = 1;
  }
  int64_t len = (L + S - 1) / S;
  len = ((len + m - 1) / m) * m;  // segment boundaries on tile boundaries
  S = (L + len - 1) / len;
  *n_seg = (int)S;
  *seg_len = (int)len;
}

void plan_segments(const lbs_scan_fwd_args* a, int* n_seg, int* seg_len) {
  int cta;
  plan_fwd(a, &cta, n_seg, seg_len);
}

// Shapes outside the register-resident kernels (N > 16 or an effective window
// > 16) take the state-outer generic path (lbs_generic.cu).
bool is_generic(const lbs_scan_fwd_args* a) {
  const int64_t m = a->window < a->seqlen ? a->window : a->seqlen;
  return a->dstate > 16 || m > 16;
}

int validate_fwd(const lbs_scan_fwd_args* a) {
  if (!a) return fail(LBS_ERR_INVALID, "null args");
  if (a->batch < 1 || a->seqlen < 1 || a->dim < 1 || a->dstate < 1)
    return fail(LBS_ERR_INVALID, "all dimensions must be >= 1 (B=%lld L=%lld E=%lld N=%lld)",
                (long long)a->batch, (long long)a->seqlen, (long long)a->dim, (long long)a->dstate);
  if (a->window < 1) return fail(LBS_ERR_INVALID, "tile length must be >= 1, got %lld", (long long)a->window);
  if (a->batch > 65535) return fail(LBS_ERR_UNSUPPORTED, "batch > 65535");
  if (a->seqlen > (int64_t)1 << 30 || a->dim > (int64_t)1 << 24)
    return fail(LBS_ERR_UNSUPPORTED, "sequence or channel count too large");
  if (!io_dtype_ok(a->io_dtype)) return fail(LBS_ERR_INVALID, "bad io dtype %d", a->io_dtype);
  if (!io_dtype_ok(a->bc_dtype)) return fail(LBS_ERR_INVALID, "bad B/C dtype %d", a->bc_dtype);
  {
    const bool ok = (a->io_dtype == LBS_F32 && a->bc_dtype == LBS_F32) ||
                    (a->io_dtype == LBS_BF16 && (a->bc_dtype == LBS_BF16 || a->bc_dtype == LBS_F32));
    if (!ok)
      return fail(LBS_ERR_UNSUPPORTED, "dtype combination io=%d bc=%d not instantiated (f32/f32, bf16/bf16, bf16/f32)",
                  a->io_dtype, a->bc_dtype);
  }
  if (!a->u || !a->delta || !a->A || !a->B || !a->C)
    return fail(LBS_ERR_INVALID, "u, delta, A, B and C must be non-null");
  if (a->dstate > 4096) return fail(LBS_ERR_UNSUPPORTED, "dstate %lld > 4096", (long long)a->dstate);
  if ((a->flags & LBS_FLAG_ACCUM) && (a->flags & LBS_FLAG_LB))
    return fail(LBS_ERR_UNSUPPORTED, "LBS_FLAG_ACCUM is supported for the forward-only scan (no LBS_FLAG_LB)");
  if (a->checkpoints && is_generic(a))
    return fail(LBS_ERR_UNSUPPORTED, "training checkpoints are not used for N > 16 or windows > 16 "
                "(the generic path recomputes; pass NULL)");
  if (a->checkpoints && a->ckpt_len != lbs_scan_ckpt_len(a->seqlen, a->window))
    return fail(LBS_ERR_INVALID, "ckpt_len %lld != lbs_scan_ckpt_len(L, window) = %lld", (long long)a->ckpt_len,
                (long long)lbs_scan_ckpt_len(a->seqlen, a->window));
  return LBS_OK;
}

lbs::View3D view(const void* p, const int64_t* s) { return lbs::View3D{p, s[0], s[1], s[2]}; }

// ---------------------------------------------------------------------------
// TMA tensor maps for the forward's staged inputs.  The driver's encoder is
// reached through the runtime (no libcuda link); encoding is a host-only call.
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// (inner, L, B) view with element strides s[0] (batch), s[1] (step), s[2] == 1
bool encode_view(CUtensorMap* m, const void* base, const int64_t* s, int64_t inner, int64_t L, int64_t B,
                 size_t es, int dtype, unsigned box_inner, unsigned box_rows) {
  auto enc = tma_encoder();
  if (!enc || !base || s[2] != 1) return false;
  const uint64_t a = reinterpret_cast<uint64_t>(base);
  const int64_t s1 = s[1] * (int64_t)es, s0 = s[0] * (int64_t)es;
  if (a % 16 || s1 % 16 || s0 % 16 || s1 <= 0 || s0 <= 0 || s1 < inner * (int64_t)es || (B > 1 && s0 < L * s1))
    return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)s1, (cuuint64_t)(B > 1 ? s0 : L * s1)};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t el[3] = {1, 1, 1};
  const CUtensorMapDataType dt = dtype == LBS_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  return enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Maps for u, delta, z, B, C when every view qualifies (16-byte aligned rows of
// whole pieces, N a full state tile of whole 16-byte rows); else false (cp.async).
bool encode_fwd_maps(const lbs_scan_fwd_args* a, int cta, lbs::FwdTmaMaps* m) {
  if (!lbs::fwd_tma_enabled() || (a->flags & LBS_FLAG_NO_TMA)) return false;
  const int ns = padded_states(a->dstate);
  const size_t es = a->io_dtype == LBS_F32 ? 4 : 2, eb = a->bc_dtype == LBS_F32 ? 4 : 2;
  if (a->dstate != ns || (ns * eb) % 16 || (a->dim * es) % 16) return false;
  if (a->B_stride[1] != a->C_stride[1]) return false;
  const unsigned CL = 16;  // fwd_chunk(window <= 16)
  return encode_view(&m->tm[0], a->u, a->u_stride, a->dim, a->seqlen, a->batch, es, a->io_dtype, cta, CL) &&
         encode_view(&m->tm[1], a->delta, a->delta_stride, a->dim, a->seqlen, a->batch, es, a->io_dtype, cta, CL) &&
         (!a->z || encode_view(&m->tm[2], a->z, a->z_stride, a->dim, a->seqlen, a->batch, es, a->io_dtype, cta, CL)) &&
         encode_view(&m->tm[3], a->B, a->B_stride, ns, a->seqlen, a->batch, eb, a->bc_dtype, ns, CL) &&
         encode_view(&m->tm[4], a->C, a->C_stride, ns, a->seqlen, a->batch, eb, a->bc_dtype, ns, CL);
}

void fill_fwd_params(const lbs_scan_fwd_args* a, lbs::FwdParams* p) {
  p->Bt = (int)a->batch;
  p->L = (int)a->seqlen;
  p->E = (int)a->dim;
  p->N = (int)a->dstate;
  // a window longer than the sequence is one (ragged) tile (test_oracle.py:247-252)
  p->m = (int)(a->window > a->seqlen ? a->seqlen : a->window);
  p->flags = a->flags;
  p->u = view(a->u, a->u_stride);
  p->delta = view(a->delta, a->delta_stride);
  p->z = view(a->z, a->z_stride);
  p->Bm = view(a->B, a->B_stride);
  p->Cm = view(a->C, a->C_stride);
  p->out = a->out;
  p->so0 = a->out_stride[0];
  p->so1 = a->out_stride[1];
  p->so2 = a->out_stride[2];
  p->A = a->A;
  p->D = a->D;
  p->bias = a->delta_bias;
  p->last_state = a->last_state;
  p->ckpt = a->checkpoints;
  p->ckpt_len = (int)a->ckpt_len;
  p->n_ckpt = a->checkpoints ? (int)((a->seqlen + a->ckpt_len - 1) / a->ckpt_len) : 0;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct BwdLayout {
  int64_t ckpt_len, n_ckpt;
  int n_seg, seg_chunks;
  size_t off_ckpt, off_seg, off_bc, off_w, off_bagg, total;
};

// Sequence split of the backward: when the (128-channel block, batch row) CTAs
// cannot fill one wave at 2 CTAs per SM, cut the chunk range into segments
// (whole checkpoint chunks) so the CTAs do; the carry of the global adjoint
// across segments comes from bwd_segment_adjoint_kernel (folded inside the
// main pass for <= 32 segments, by the parallel segment prefix beyond).  Each
// extra segment costs one light adjoint sweep over its steps.
constexpr int64_t kBwdMaxSeg = 2048;
void plan_bwd(const lbs_scan_fwd_args* f, int64_t nck, int* n_seg, int* seg_chunks) {
  const int64_t ctas = ((f->dim + lbs::kFwdThreads - 1) / lbs::kFwdThreads) * f->batch;
  const int64_t slots = 2 * (int64_t)num_sms();
  int64_t S = 1;
  if (f->seg_hint > 0) S = f->seg_hint;
  else if (ctas < slots) S = slots / ctas;
  if (S > kBwdMaxSeg) S = kBwdMaxSeg;
  if (S > nck) S = nck;
  if (S < 1) S = 1;
  const int64_t per = (nck + S - 1) / S;
  *seg_chunks = (int)per;
  *n_seg = (int)((nck + per - 1) / per);
}

int validate_bwd(const lbs_scan_bwd_args* a) {
  const lbs_scan_fwd_args* f = &a->fwd;
  if (!a->dout || !a->du || !a->ddelta)
    return fail(LBS_ERR_INVALID, "dout, du and ddelta must be non-null");
  if ((a->dz == nullptr) != (f->z == nullptr))
    return fail(LBS_ERR_INVALID, "dz must be given exactly when z is");
  if (!a->dA || !a->dB || !a->dC) return fail(LBS_ERR_INVALID, "dA, dB and dC must be non-null");
  if (a->dD && !f->D) return fail(LBS_ERR_INVALID, "dD given without D");
  if (a->ddelta_bias && !f->delta_bias) return fail(LBS_ERR_INVALID, "ddelta_bias given without delta_bias");
  return LBS_OK;
}

// workspace: [checkpoints (if not supplied)][forward segment aggregates][dB/dC partials][dA/dD/dbias partials]
int bwd_layout(const lbs_scan_bwd_args* a, BwdLayout* lay) {
  if (!a) return fail(LBS_ERR_INVALID, "null args");
  const lbs_scan_fwd_args* f = &a->fwd;
  int rc = validate_fwd(f);
  if (rc != LBS_OK) return rc;
  if (is_generic(f)) {
    lay->ckpt_len = lay->n_ckpt = 0;
    lay->n_seg = 1;
    lay->seg_chunks = 0;
    lay->off_ckpt = lay->off_seg = lay->off_bc = lay->off_w = lay->off_bagg = 0;
    lay->total = lbs::gen_bwd_workspace_floats((int)f->batch, (int)f->seqlen, (int)f->dim, (int)f->dstate) *
                 sizeof(float);
    return LBS_OK;
  }
  const int64_t K = lbs_scan_ckpt_len(f->seqlen, f->window);
  const int64_t nck = (f->seqlen + K - 1) / K;
  const int NS = padded_states(f->dstate);
  lay->ckpt_len = K;
  lay->n_ckpt = nck;
  size_t off = 0;
  lay->off_ckpt = off;
  lay->off_seg = off;
  if (!f->checkpoints) {
    off += align256(lbs_scan_ckpt_bytes(f));
    lay->off_seg = off;
    lbs_scan_fwd_args b2 = *f;
    if (b2.window > b2.seqlen) b2.window = b2.seqlen;
    int S, len;
    plan_segments(&b2, &S, &len);
    if (S > 1) off += align256((size_t)f->batch * S * f->dim * 2 * NS * sizeof(float));
  }
  plan_bwd(f, nck, &lay->n_seg, &lay->seg_chunks);
  const int64_t n_eblk = (f->dim + lbs::kFwdThreads - 1) / lbs::kFwdThreads;
  lay->off_bc = off;
  off += align256((size_t)n_eblk * f->batch * f->seqlen * 2 * NS * sizeof(float));
  lay->off_w = off;
  off += align256((size_t)f->batch * lay->n_seg * (NS + 2) * f->dim * sizeof(float));
  lay->off_bagg = off;
  if (lay->n_seg > 1) off += align256((size_t)f->batch * lay->n_seg * f->dim * 2 * NS * sizeof(float));
  lay->total = off;
  return LBS_OK;
}

}  // namespace

namespace lbs {
int fwd_padded_states(int N) { return padded_states(N); }
}  // namespace lbs

extern "C" {

int lbs_set_error(int code, const char* msg) { return fail(code, "%s", msg); }

int lbs_abi_version(void) { return LBS_ABI_VERSION; }

const char* lbs_last_error(void) { return g_err.c_str(); }

int64_t lbs_select_tile_len(int64_t L) {
  // engine.py:54-62
  if (L < 1) return -1;
  if (L > 256) return 16;
  if (L > 128) return 8;
  return 4;
}

size_t lbs_scan_fwd_workspace_bytes(const lbs_scan_fwd_args* a) {
  if (validate_fwd(a) != LBS_OK) return 0;
  if (is_generic(a)) return lbs::gen_fwd_workspace_floats((int)a->batch, (int)a->seqlen, (int)a->dim) * sizeof(float);
  lbs_scan_fwd_args b = *a;
  if (b.window > b.seqlen) b.window = b.seqlen;
  int S, len;
  plan_segments(&b, &S, &len);
  if (S <= 1) return 0;
  return (size_t)a->batch * S * a->dim * 2 * padded_states(a->dstate) * sizeof(float);
}

int64_t lbs_scan_ckpt_len(int64_t seqlen, int64_t window) {
  if (seqlen < 1 || window < 1) return -1;
  const int64_t m = window < seqlen ? window : seqlen;
  if (m > 16) return -1;
  return lbs::bwd_chunk_len((int)m);
}

size_t lbs_scan_ckpt_bytes(const lbs_scan_fwd_args* a) {
  if (!a || a->batch < 1 || a->seqlen < 1 || a->dim < 1 || a->dstate < 1) return 0;
  if (is_generic(a)) return 0;  // the generic backward recomputes its states
  const int64_t K = lbs_scan_ckpt_len(a->seqlen, a->window);
  if (K < 1) return 0;
  const int64_t nck = (a->seqlen + K - 1) / K;
  return (size_t)a->batch * nck * a->dim * padded_states(a->dstate) * sizeof(float);
}

int lbs_scan_fwd(const lbs_scan_fwd_args* a, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate_fwd(a);
  if (rc != LBS_OK) return rc;
  if (!a->out && !a->checkpoints) return fail(LBS_ERR_INVALID, "out must be non-null");
  lbs::FwdParams p{};
  fill_fwd_params(a, &p);
  if (is_generic(a)) {
    if (!a->out) return fail(LBS_ERR_INVALID, "out must be non-null");
    const size_t need = lbs_scan_fwd_workspace_bytes(a);
    if (!ws || ws_bytes < need) return fail(LBS_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return cuda_status(lbs::launch_fwd_generic(p, static_cast<float*>(ws), a->io_dtype, a->bc_dtype, (cudaStream_t)stream),
                       "lbs_scan_fwd (generic)");
  }
  lbs_scan_fwd_args b = *a;
  b.window = p.m;
  plan_fwd(&b, &p.cta, &p.n_seg, &p.seg_len);
  if (p.n_seg > 1) {
    const size_t need = (size_t)a->batch * p.n_seg * a->dim * 2 * padded_states(a->dstate) * sizeof(float);
    if (!ws || ws_bytes < need)
      return fail(LBS_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    p.seg_agg = static_cast<float*>(ws);
  }
  // TMA tensor-copy staging where it measured faster (round 2, tools/kbench.py and
  // bench.py A/B): unsplit launches with fp32 I/O (configs[2] -1 %, its 8-GPU
  // shard -4 %).  bf16 I/O stays on cp.async (LBVim-Ti layer +2 % with TMA), as do
  // split launches (configs[0] +14 %).
  lbs::FwdTmaMaps maps;
  if (p.n_seg == 1 && (a->io_dtype == LBS_F32 || LBS_FWD_TMA_BF16) && encode_fwd_maps(a, p.cta, &maps))
    p.tma_maps = &maps;
  return cuda_status(lbs::launch_fwd(p, a->io_dtype, a->bc_dtype, (cudaStream_t)stream), "lbs_scan_fwd");
}

int lbs_prediscretized_fwd(const lbs_prediscretized_args* a, void* stream) {
  if (!a) return fail(LBS_ERR_INVALID, "null args");
  if (a->batch < 1 || a->seqlen < 1 || a->dim < 1 || a->dstate < 1)
    return fail(LBS_ERR_INVALID, "all dimensions must be >= 1");
  if (a->window < 1) return fail(LBS_ERR_INVALID, "tile length must be >= 1, got %lld", (long long)a->window);
  if (a->dstate > 64) return fail(LBS_ERR_UNSUPPORTED, "dstate > 64");
  if (a->dtype != LBS_F32 && a->dtype != LBS_F64) return fail(LBS_ERR_INVALID, "dtype must be f32 or f64");
  if (!a->abar || !a->bx || !a->c || !a->dx || !a->y || !a->h_final)
    return fail(LBS_ERR_INVALID, "null tensor");
  if (a->batch > 65535) return fail(LBS_ERR_UNSUPPORTED, "batch > 65535");
  lbs::PreParams p{};
  p.Bt = (int)a->batch;
  p.L = (int)a->seqlen;
  p.E = (int)a->dim;
  p.N = (int)a->dstate;
  p.m = (int)(a->window > a->seqlen ? a->seqlen : a->window);
  p.flags = a->flags;
  p.abar = a->abar;
  p.bx = a->bx;
  p.c = a->c;
  p.dx = a->dx;
  p.y = a->y;
  p.h_final = a->h_final;
  return cuda_status(lbs::launch_prediscretized(p, a->dtype == LBS_F64, (cudaStream_t)stream),
                     "lbs_prediscretized_fwd");
}

int lbs_rms_norm_fwd(const lbs_norm_args* a, void* stream) {
  if (!a) return fail(LBS_ERR_INVALID, "null args");
  if (a->rows < 1 || a->dim < 1) return fail(LBS_ERR_INVALID, "rows and dim must be >= 1");
  if (a->io_dtype != LBS_F32 && a->io_dtype != LBS_BF16) return fail(LBS_ERR_INVALID, "dtype must be f32 or bf16");
  if (!a->x || !a->scale || !a->out) return fail(LBS_ERR_INVALID, "null tensor");
  if (a->rows > (int64_t)1 << 34) return fail(LBS_ERR_UNSUPPORTED, "too many rows");
  if (a->out_dtype != a->io_dtype && !(a->io_dtype == LBS_F32 && a->out_dtype == LBS_BF16))
    return fail(LBS_ERR_INVALID, "out_dtype must equal io_dtype, or be bf16 for f32 input");
  lbs::NormParams p{a->rows, (int)a->dim, a->eps, a->x, a->x_row_stride, a->scale, a->out, a->out_row_stride};
  return cuda_status(lbs::launch_rms_norm(p, a->io_dtype, a->out_dtype, (cudaStream_t)stream), "lbs_rms_norm_fwd");
}

namespace {
int validate_norm_bwd(const lbs_norm_bwd_args* a) {
  if (!a) return fail(LBS_ERR_INVALID, "null args");
  if (a->rows < 1 || a->dim < 1) return fail(LBS_ERR_INVALID, "rows and dim must be >= 1");
  if (a->io_dtype != LBS_F32 && a->io_dtype != LBS_BF16) return fail(LBS_ERR_INVALID, "dtype must be f32 or bf16");
  if (!a->x || !a->scale || !a->dout || !a->dx) return fail(LBS_ERR_INVALID, "null tensor");
  if (a->dim > (int64_t)1 << 20) return fail(LBS_ERR_UNSUPPORTED, "dim too large");
  if (a->rows > (int64_t)1 << 34) return fail(LBS_ERR_UNSUPPORTED, "too many rows");
  return LBS_OK;
}
}  // namespace

size_t lbs_rms_norm_bwd_workspace_bytes(const lbs_norm_bwd_args* a) {
  if (!a || a->rows < 1 || a->dim < 1) return 0;
  return a->dscale ? (size_t)lbs::norm_bwd_warps(a->rows) * (size_t)a->dim * sizeof(float) : 0;
}

int lbs_rms_norm_bwd(const lbs_norm_bwd_args* a, void* ws, size_t ws_bytes, void* stream) {
  const int rc = validate_norm_bwd(a);
  if (rc != LBS_OK) return rc;
  const size_t need = lbs_rms_norm_bwd_workspace_bytes(a);
  if (need && (!ws || ws_bytes < need))
    return fail(LBS_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need, ws_bytes);
  lbs::NormBwdParams p{a->rows, (int)a->dim, a->eps, a->x, a->x_row_stride, a->scale, a->dout,
                       a->dout_row_stride, a->dx, a->dx_row_stride, a->dscale, static_cast<float*>(ws),
                       lbs::norm_bwd_warps(a->rows), a->dres, a->dres_row_stride};
  return cuda_status(lbs::launch_rms_norm_bwd(p, a->io_dtype, (cudaStream_t)stream), "lbs_rms_norm_bwd");
}

size_t lbs_scan_bwd_workspace_bytes(const lbs_scan_bwd_args* a) {
  BwdLayout lay;
  if (bwd_layout(a, &lay) != LBS_OK) return 0;
  return lay.total;
}

int lbs_scan_bwd(const lbs_scan_bwd_args* a, void* ws, size_t ws_bytes, void* stream) {
  BwdLayout lay;
  int rc = bwd_layout(a, &lay);
  if (rc != LBS_OK) return rc;
  rc = validate_bwd(a);
  if (rc != LBS_OK) return rc;
  if (lay.total && (!ws || ws_bytes < lay.total))
    return fail(LBS_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", lay.total, ws_bytes);
  char* w = static_cast<char*>(ws);
  cudaStream_t st = (cudaStream_t)stream;
  const lbs_scan_fwd_args* f = &a->fwd;
  lbs::BwdParams P{};
  fill_fwd_params(f, &P.f);
  if (is_generic(f)) {
    P.dout = view(a->dout, a->dout_stride);
    P.du = lbs::OutView{a->du, a->du_stride[0], a->du_stride[1], a->du_stride[2]};
    P.ddelta = lbs::OutView{a->ddelta, a->ddelta_stride[0], a->ddelta_stride[1], a->ddelta_stride[2]};
    P.dz = lbs::OutView{a->dz, a->dz_stride[0], a->dz_stride[1], a->dz_stride[2]};
    P.dA = a->dA;
    P.dD = a->dD;
    P.dbias = a->ddelta_bias;
    P.dB = a->dB;
    P.sb0 = a->dB_stride[0];
    P.sb1 = a->dB_stride[1];
    P.sb2 = a->dB_stride[2];
    P.dC = a->dC;
    P.sc0 = a->dC_stride[0];
    P.sc1 = a->dC_stride[1];
    P.sc2 = a->dC_stride[2];
    P.part_w = reinterpret_cast<float*>(w) + 7 * (size_t)f->batch * f->seqlen * f->dim;
    return cuda_status(lbs::launch_bwd_generic(P, reinterpret_cast<float*>(w), f->io_dtype, f->bc_dtype, st),
                       "lbs_scan_bwd (generic)");
  }
  P.f.out = nullptr;
  P.f.last_state = nullptr;
  P.f.n_seg = 1;
  P.f.seg_len = P.f.L;
  P.f.seg_agg = nullptr;
  P.f.ckpt_len = (int)lay.ckpt_len;
  P.f.n_ckpt = (int)lay.n_ckpt;
  if (f->checkpoints) {
    P.f.ckpt = f->checkpoints;
  } else {
    // checkpoint-only forward sweep (no LB pass, no output) into the workspace
    P.f.ckpt = reinterpret_cast<float*>(w + lay.off_ckpt);
    lbs::FwdParams fp = P.f;
    fp.flags &= ~LBS_FLAG_LB;
    fp.z = lbs::View3D{nullptr, 0, 0, 0};
    lbs_scan_fwd_args b2 = *f;
    b2.window = fp.m;
    plan_fwd(&b2, &fp.cta, &fp.n_seg, &fp.seg_len);
    if (fp.n_seg > 1) fp.seg_agg = reinterpret_cast<float*>(w + lay.off_seg);
    rc = cuda_status(lbs::launch_fwd(fp, f->io_dtype, f->bc_dtype, st), "lbs_scan_bwd (recompute)");
    if (rc != LBS_OK) return rc;
  }
  P.dout = view(a->dout, a->dout_stride);
  P.du = lbs::OutView{a->du, a->du_stride[0], a->du_stride[1], a->du_stride[2]};
  P.ddelta = lbs::OutView{a->ddelta, a->ddelta_stride[0], a->ddelta_stride[1], a->ddelta_stride[2]};
  P.dz = lbs::OutView{a->dz, a->dz_stride[0], a->dz_stride[1], a->dz_stride[2]};
  P.part_bc = reinterpret_cast<float*>(w + lay.off_bc);
  P.part_w = reinterpret_cast<float*>(w + lay.off_w);
  P.n_seg = lay.n_seg;
  P.seg_chunks = lay.seg_chunks;
  P.bagg = lay.n_seg > 1 ? reinterpret_cast<float*>(w + lay.off_bagg) : nullptr;
  P.dA = a->dA;
  P.dD = a->dD;
  P.dbias = a->ddelta_bias;
  P.dB = a->dB;
  P.sb0 = a->dB_stride[0];
  P.sb1 = a->dB_stride[1];
  P.sb2 = a->dB_stride[2];
  P.dC = a->dC;
  P.sc0 = a->dC_stride[0];
  P.sc1 = a->dC_stride[1];
  P.sc2 = a->dC_stride[2];
  return cuda_status(lbs::launch_bwd(P, f->io_dtype, f->bc_dtype, st), "lbs_scan_bwd");
}

}  // extern "C"
