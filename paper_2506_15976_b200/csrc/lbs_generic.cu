// Fused LB selective scan for shapes outside the register-resident kernels'
// range: windows min(M, L) > 16 and state sizes N > 16 (the reference accepts
// any M >= 1 and any N: engine.py:65-85, test_oracle.py:221-226).
//
// Same semantics and C ABI as lbs_scan_fwd / lbs_scan_bwd (discretisation,
// LB record, D skip, SiLU gate, flip-on-load reverse, exp / linear modes), but
// state-outer: one thread per (b, e) channel sweeps the sequence once per
// state n, so neither the window nor N has to fit in registers.  Per-step
// accumulators over n live in fp32 workspace rows [b][t][e] (coalesced across
// the CTA's channels).  The forward is one launch; the backward is one launch
// per state (ascending pass: h, LB adjoint v; descending pass: global adjoint
// lam, LB record Q, all chain terms) plus a fixed-order E-reduction of that
// state's dB/dC terms, then a finishing launch (du, ddelta, dz, dD/dbias
// partials) and the shared dA/dD/dbias reduction.  Deterministic (no atomics).
// These shapes are off the benchmarked path; the kernels favour simplicity.
#include "lbs_common.cuh"
#include "lbs_internal.h"

namespace lbs {
namespace {

constexpr int kGT = 128;

struct Col {
  const void* p;
  long long base, step;  // element offset of logical step 0, signed stride per logical step
};

__device__ __forceinline__ Col col(const View3D& v, int b, int e, int L, bool rev) {
  return Col{v.p, (long long)b * v.s0 + (long long)e * v.s2 + (rev ? (long long)(L - 1) * v.s1 : 0),
             rev ? -v.s1 : v.s1};
}
template <typename T>
__device__ __forceinline__ float at(const Col& c, int t) {
  return to_f(static_cast<const T*>(c.p)[c.base + (long long)t * c.step]);
}

struct Step {
  float dl, du, a, b, C;
};

template <typename Tio, typename Tbc>
__device__ __forceinline__ Step load_step(const FwdParams& p, const Col& cu, const Col& cd, const Col& cB,
                                          const Col& cC, int t, float bias, float An, bool softplus,
                                          bool linear) {
  Step s;
  const float x = at<Tio>(cd, t) + bias;
  s.dl = softplus ? softplus_f(x) : x;
  s.du = s.dl * at<Tio>(cu, t);
  s.a = linear ? s.dl * An : ex2(s.dl * An * kLog2e);
  s.b = s.du * at<Tbc>(cB, t);
  s.C = at<Tbc>(cC, t);
  return s;
}

// ---------------------------------------------------------------------------
// forward: yacc[b][t][e] = sum_n C (h + r); out = (yacc + D u) silu(z)
template <typename Tio, typename Tbc>
__global__ void __launch_bounds__(kGT) gen_fwd_kernel(FwdParams p, float* yacc) {
  const int e = blockIdx.x * kGT + threadIdx.x, b = blockIdx.y;
  if (e >= p.E) return;
  const int L = p.L, N = p.N, m = p.m;
  const bool rev = p.flags & LBS_FLAG_REVERSE, lb = p.flags & LBS_FLAG_LB;
  const bool softplus = p.flags & LBS_FLAG_SOFTPLUS, linear = p.flags & LBS_FLAG_LINEAR;
  const Col cu = col(p.u, b, e, L, rev), cd = col(p.delta, b, e, L, rev);
  const Col cB = col(p.Bm, b, 0, L, rev), cC = col(p.Cm, b, 0, L, rev);
  const float bias = p.bias ? p.bias[e] : 0.f;
  float* y = yacc + (long long)b * L * p.E + e;
  for (int n = 0; n < N; ++n) {
    const float An = p.A[(long long)e * N + n];
    const Col cBn{cB.p, cB.base + (long long)n * p.Bm.s2, cB.step};
    const Col cCn{cC.p, cC.base + (long long)n * p.Cm.s2, cC.step};
    float h = 0.f;
    for (int t0 = 0; t0 < L; t0 += m) {
      const int te = min(t0 + m, L) - 1;
      if (lb) {  // exclusive tile-local record r_t = a_t (r_{t+1} + b_{t+1}), right to left
        float s = 0.f;
        for (int t = te; t >= t0; --t) {
          const Step st = load_step<Tio, Tbc>(p, cu, cd, cBn, cCn, t, bias, An, softplus, linear);
          float c = 0.f;
          if (t < te) {
            const float r = st.a * s;
            c = st.C * r;
            s = r + st.b;
          } else {
            s = st.b;
          }
          float* yt = y + (long long)t * p.E;
          *yt = n == 0 ? c : *yt + c;
        }
      }
      for (int t = t0; t <= te; ++t) {
        const Step st = load_step<Tio, Tbc>(p, cu, cd, cBn, cCn, t, bias, An, softplus, linear);
        h = st.a * h + st.b;
        float* yt = y + (long long)t * p.E;
        *yt = (n == 0 && !lb) ? st.C * h : *yt + st.C * h;
      }
    }
    if (p.last_state) p.last_state[((long long)b * p.E + e) * N + n] = h;
  }
  // D skip + gate (block.py:177-178), flip-on-store
  const Col cz = col(p.z, b, e, L, rev);
  Tio* op = static_cast<Tio*>(p.out) + (long long)b * p.so0 + (long long)e * p.so2 + (rev ? (long long)(L - 1) * p.so1 : 0);
  const long long ostep = rev ? -p.so1 : p.so1;
  const float Dv = p.D ? p.D[e] : 0.f;
  const bool accum = p.flags & LBS_FLAG_ACCUM;
  for (int t = 0; t < L; ++t) {
    float v = y[(long long)t * p.E] + Dv * at<Tio>(cu, t);
    if (p.z.p) v *= silu_f(at<Tio>(cz, t));
    Tio* o = op + (long long)t * ostep;
    st<Tio>(o, accum ? to_f(*o) + v : v);
  }
}

// ---------------------------------------------------------------------------
// backward, one launch per state n (see the file comment; autodiff.py:48-195,
// block.py:106-129).  Scratch rows are [b][t][e] fp32, logical t.
struct GenBwdScratch {
  float *hbuf, *vbuf, *pacc, *sacc, *yacc, *pb, *pc;
};

template <typename Tio, typename Tbc>
__global__ void __launch_bounds__(kGT) gen_bwd_state_kernel(BwdParams P, GenBwdScratch w, int n) {
  const FwdParams& p = P.f;
  const int e = blockIdx.x * kGT + threadIdx.x, b = blockIdx.y;
  if (e >= p.E) return;
  const int L = p.L, N = p.N, m = p.m;
  const bool rev = p.flags & LBS_FLAG_REVERSE, lb = p.flags & LBS_FLAG_LB;
  const bool softplus = p.flags & LBS_FLAG_SOFTPLUS, linear = p.flags & LBS_FLAG_LINEAR;
  const Col cu = col(p.u, b, e, L, rev), cd = col(p.delta, b, e, L, rev);
  const Col cB0 = col(p.Bm, b, 0, L, rev), cC0 = col(p.Cm, b, 0, L, rev);
  const Col cBn{cB0.p, cB0.base + (long long)n * p.Bm.s2, cB0.step};
  const Col cCn{cC0.p, cC0.base + (long long)n * p.Cm.s2, cC0.step};
  const Col cg = col(P.dout, b, e, L, rev), cz = col(p.z, b, e, L, rev);
  const float bias = p.bias ? p.bias[e] : 0.f;
  const float An = p.A[(long long)e * N + n];
  const long long row = (long long)b * L * p.E + e;
  auto gy_at = [&](int t) {
    float g = at<Tio>(cg, t);
    if (p.z.p) g *= silu_f(at<Tio>(cz, t));
    return g;
  };
  // ascending: h_t and the tile-local adjoint v_i = g_i + a_{i-1} v_{i-1}
  float h = 0.f, v = 0.f, a_prev = 0.f;
  for (int t = 0; t < L; ++t) {
    const Step st = load_step<Tio, Tbc>(p, cu, cd, cBn, cCn, t, bias, An, softplus, linear);
    h = st.a * h + st.b;
    const float g = st.C * gy_at(t);
    v = (t % m == 0) ? g : a_prev * v + g;
    w.hbuf[row + (long long)t * p.E] = h;
    w.vbuf[row + (long long)t * p.E] = v;
    a_prev = st.a;
  }
  // descending: lam_t = g_t + a_{t+1} lam_{t+1}; Q_t = r_t + b_t = a_t Q_{t+1} + b_t
  float lam = 0.f, a_next = 0.f, Qn = 0.f, dA = 0.f;
  Step cur = load_step<Tio, Tbc>(p, cu, cd, cBn, cCn, L - 1, bias, An, softplus, linear);
  for (int t = L - 1; t >= 0; --t) {
    Step prv{};
    if (t > 0) prv = load_step<Tio, Tbc>(p, cu, cd, cBn, cCn, t - 1, bias, An, softplus, linear);
    const float gyt = gy_at(t);
    const float g = cur.C * gyt;
    const bool rec = lb && !(((t + 1) % m == 0) || t == L - 1);  // t is not a tile end
    const bool not_start = lb && (t % m != 0);                    // t is not a tile start
    lam = g + (t < L - 1 ? a_next * lam : 0.f);
    const float ht = w.hbuf[row + (long long)t * p.E];
    const float hprev = t > 0 ? w.hbuf[row + (long long)(t - 1) * p.E] : 0.f;
    float hr = ht, Q = cur.b, dab = lam * hprev;
    if (rec) {
      hr = ht + cur.a * Qn;
      Q = cur.a * Qn + cur.b;
      dab += w.vbuf[row + (long long)t * p.E] * Qn;
    }
    float dbx = lam;
    if (not_start) dbx += prv.a * w.vbuf[row + (long long)(t - 1) * p.E];
    const float da = linear ? dab : dab * cur.a;
    const long long i = row + (long long)t * p.E;
    const float pa = da * An, sa = dbx * at<Tbc>(cBn, t), ya = cur.C * hr;
    w.pacc[i] = n == 0 ? pa : w.pacc[i] + pa;
    w.sacc[i] = n == 0 ? sa : w.sacc[i] + sa;
    w.yacc[i] = n == 0 ? ya : w.yacc[i] + ya;
    w.pb[i] = dbx * cur.du;  // dB[b,t,n] = sum_e dbx dl u
    w.pc[i] = gyt * hr;      // dC[b,t,n] = sum_e gy (h + r)
    dA += da * cur.dl;
    Qn = Q;
    a_next = cur.a;
    cur = prv;
  }
  P.part_w[((long long)b * (N + 2) + n) * p.E + e] = dA;
}

// dB / dC of state n: fixed-order sums over e of the pb / pc rows (one warp per (b, t))
__global__ void gen_bwd_reduce_bc_kernel(BwdParams P, GenBwdScratch w, int n) {
  const FwdParams& p = P.f;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (wid >= (long long)p.Bt * p.L) return;
  const int b = (int)(wid / p.L), t = (int)(wid % p.L);
  const float* rb = w.pb + ((long long)b * p.L + t) * p.E;
  const float* rc = w.pc + ((long long)b * p.L + t) * p.E;
  float sb = 0.f, sc = 0.f;
  for (int e = lane; e < p.E; e += 32) {
    sb += rb[e];
    sc += rc[e];
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
  }
  if (lane == 0) {
    const bool rev = p.flags & LBS_FLAG_REVERSE;
    const long long tp = rev ? (p.L - 1 - t) : t;
    P.dB[b * P.sb0 + tp * P.sb1 + n * P.sb2] = sb;
    P.dC[b * P.sc0 + tp * P.sc1 + n * P.sc2] = sc;
  }
}

// du, ddelta, dz and the dD / dbias partials from the per-step accumulators
template <typename Tio, typename Tbc>
__global__ void __launch_bounds__(kGT) gen_bwd_finish_kernel(BwdParams P, GenBwdScratch w) {
  const FwdParams& p = P.f;
  const int e = blockIdx.x * kGT + threadIdx.x, b = blockIdx.y;
  if (e >= p.E) return;
  const int L = p.L, N = p.N;
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool softplus = p.flags & LBS_FLAG_SOFTPLUS;
  const Col cu = col(p.u, b, e, L, rev), cd = col(p.delta, b, e, L, rev);
  const Col cg = col(P.dout, b, e, L, rev), cz = col(p.z, b, e, L, rev);
  const float bias = p.bias ? p.bias[e] : 0.f, Dv = p.D ? p.D[e] : 0.f;
  const long long row = (long long)b * L * p.E + e;
  auto obase = [&](const OutView& o) -> Tio* {
    return o.p ? static_cast<Tio*>(o.p) + (long long)b * o.s0 + (long long)e * o.s2 + (rev ? (long long)(L - 1) * o.s1 : 0)
               : nullptr;
  };
  Tio *dup = obase(P.du), *ddp = obase(P.ddelta), *dzp = obase(P.dz);
  const long long sdu = rev ? -P.du.s1 : P.du.s1, sdd = rev ? -P.ddelta.s1 : P.ddelta.s1,
                  sdz = rev ? -P.dz.s1 : P.dz.s1;
  float dD = 0.f, dbias = 0.f;
  for (int t = 0; t < L; ++t) {
    const float x = at<Tio>(cd, t) + bias;
    const float dl = softplus ? softplus_f(x) : x;
    const float uv = at<Tio>(cu, t), go = at<Tio>(cg, t);
    float gy = go, zv = 0.f, sz = 0.f;
    if (p.z.p) {
      zv = at<Tio>(cz, t);
      sz = sigmoid_f(zv);
      gy *= zv * sz;
    }
    const long long i = row + (long long)t * p.E;
    const float s = w.sacc[i];
    const float ddl = w.pacc[i] + uv * s;
    const float ddv = softplus ? ddl * sigmoid_f(x) : ddl;
    st<Tio>(dup + (long long)t * sdu, Dv * gy + dl * s);
    st<Tio>(ddp + (long long)t * sdd, ddv);
    if (dzp) {
      const float y = w.yacc[i] + Dv * uv;
      st<Tio>(dzp + (long long)t * sdz, go * y * sz * (1.f + zv * (1.f - sz)));
    }
    dD += gy * uv;
    dbias += ddv;
  }
  P.part_w[((long long)b * (N + 2) + N) * p.E + e] = dD;
  P.part_w[((long long)b * (N + 2) + N + 1) * p.E + e] = dbias;
}

// dA (E, N), dD, dbias (E) += fixed-order sums over b of part_w
__global__ void gen_bwd_reduce_w_kernel(BwdParams P) {
  const FwdParams& p = P.f;
  const int total = p.E * (p.N + 2);
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int e = idx % p.E, i = idx / p.E;
  double s = 0.0;
  for (int b = 0; b < p.Bt; ++b) s += P.part_w[((long long)b * (p.N + 2) + i) * p.E + e];
  if (i < p.N) P.dA[(long long)e * p.N + i] += (float)s;
  else if (i == p.N) {
    if (P.dD) P.dD[e] += (float)s;
  } else if (P.dbias) {
    P.dbias[e] += (float)s;
  }
}

template <typename Tio, typename Tbc>
cudaError_t fwd_t(const FwdParams& p, float* yacc, cudaStream_t st) {
  gen_fwd_kernel<Tio, Tbc><<<dim3((p.E + kGT - 1) / kGT, p.Bt), kGT, 0, st>>>(p, yacc);
  return cudaGetLastError();
}

template <typename Tio, typename Tbc>
cudaError_t bwd_t(const BwdParams& P, float* scratch, cudaStream_t st) {
  const FwdParams& p = P.f;
  const size_t rows = (size_t)p.Bt * p.L * p.E;
  GenBwdScratch w{scratch, scratch + rows, scratch + 2 * rows, scratch + 3 * rows, scratch + 4 * rows,
                  scratch + 5 * rows, scratch + 6 * rows};
  const dim3 grid((p.E + kGT - 1) / kGT, p.Bt);
  const long long warps = (long long)p.Bt * p.L;
  for (int n = 0; n < p.N; ++n) {
    gen_bwd_state_kernel<Tio, Tbc><<<grid, kGT, 0, st>>>(P, w, n);
    gen_bwd_reduce_bc_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(P, w, n);
  }
  gen_bwd_finish_kernel<Tio, Tbc><<<grid, kGT, 0, st>>>(P, w);
  const int nw = p.E * (p.N + 2);
  gen_bwd_reduce_w_kernel<<<(nw + 255) / 256, 256, 0, st>>>(P);
  return cudaGetLastError();
}

}  // namespace

size_t gen_fwd_workspace_floats(int Bt, int L, int E) { return (size_t)Bt * L * E; }
size_t gen_bwd_workspace_floats(int Bt, int L, int E, int N) {
  return 7 * (size_t)Bt * L * E + (size_t)Bt * (N + 2) * E;
}

cudaError_t launch_fwd_generic(const FwdParams& p, float* ws, int io_dtype, int bc_dtype, cudaStream_t st) {
  if (io_dtype == LBS_F32 && bc_dtype == LBS_F32) return fwd_t<float, float>(p, ws, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_BF16) return fwd_t<__nv_bfloat16, __nv_bfloat16>(p, ws, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_F32) return fwd_t<__nv_bfloat16, float>(p, ws, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_generic(const BwdParams& P, float* ws, int io_dtype, int bc_dtype, cudaStream_t st) {
  if (io_dtype == LBS_F32 && bc_dtype == LBS_F32) return bwd_t<float, float>(P, ws, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_BF16) return bwd_t<__nv_bfloat16, __nv_bfloat16>(P, ws, st);
  if (io_dtype == LBS_BF16 && bc_dtype == LBS_F32) return bwd_t<__nv_bfloat16, float>(P, ws, st);
  return cudaErrorInvalidValue;
}

}  // namespace lbs
