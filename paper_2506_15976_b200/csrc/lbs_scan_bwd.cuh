// Fused LB selective scan — backward (sm_100a).
//
// Replaces the reference's adjoint kernel autodiff._scan_grad_kernel
// (autodiff.py:48-159, restated in oracle/lbscan_oracle.py:lbm_scan_grad),
// chained in the same launch through block._discretize_backward
// (block.py:106-129) and the gate adjoint (block.py:199-200).  Nothing of
// size (B,L,E,N) touches HBM: per (b,l) the kernel reads u, delta, z, dout (E
// each) and B, C (N each) and writes du, ddelta, dz (E each) plus fp32 dB/dC
// partial sums (2N per channel block).
//
// Math per lane (b,e,n), t in scanned order (a = exp(dl*A), b = dl*u*B,
// g = C*gy, gy = dout*silu(z)):
//   forward adjoint  lam_t = g_t + a_{t+1} lam_{t+1}      -> dbx_t = lam_t, dabar_t = lam_t h_{t-1}
//   tile-local LB    v_i = g_i + a_{i-1} v_{i-1} (ascending in a tile, v_lo = g_lo)
//                    dabar_i += v_i (r_{i+1} + b_{i+1})     (i not a tile end)
//                    dbx_{i+1} += a_i v_i                  (i+1 not a tile start)
//   chain            ddl = sum_n dabar a A + u sum_n dbx B;  du = D gy + dl sum_n dbx B
//                    dA += dabar a dl;  dB = sum_e dbx dl u;  dC = sum_e gy (h + r)
//                    ddelta = ddl * sigmoid(delta + bias);   dz = dout y silu'(z)
//
// Execution model: one thread owns one (b, e) channel (128 channels per CTA,
// like the forward) and walks the sequence BACKWARDS in chunks of K steps
// (K = whole LB tiles, K <= KT registers).  The state entering every chunk
// comes from checkpoints (written by the training forward, or by a
// checkpoint-only forward sweep), staged into shared memory with cp.async one
// chunk ahead together with u/delta/z/dout rows and B/C.  Inside a chunk the
// loop runs state-pair-outer: for each pair (n, n+1) an ascending pass
// recomputes a, h and the LB adjoint v in registers, and a descending pass
// runs the LB record r (as Q = r + b), the global adjoint lam and all chain
// terms with packed FFMA2.  lam crosses chunk boundaries through shared
// memory.  The E-reductions for dB/dC are a per-warp shared-memory transpose
// (one 16-byte store per step, fixed-order lane sums) + a 4-warp sum, written as per-CTA partials and
// reduced deterministically by a second kernel (no atomics: the reference's
// partial-then-reduce order, autodiff.py:182,188).
#pragma once
#include "lbs_scan_fwd.cuh"

namespace lbs {

constexpr int kBwdThreads = kFwdThreads;  // BcPrefetch assumes 128 threads
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}


template <typename Tio, int NS, int KT>
struct BwdSmem {
  static constexpr int NP = NS / 2;
  static constexpr size_t seq_bytes = 2ull * 4 * KT * kBwdThreads * sizeof(Tio);  // u, delta, z, dout
  static constexpr size_t bc_bytes = (size_t)KT * 2 * NS * sizeof(float);
  static constexpr size_t ck_bytes = 2ull * NP * kBwdThreads * sizeof(f2);
  static constexpr size_t pq_bytes = (size_t)NP * kBwdThreads * sizeof(f2);  // a2s, mu, dA each
  static constexpr size_t red_bytes = 4ull * KT * 2 * NS * sizeof(float);
  static constexpr size_t raw_bytes = 2ull * KT * 2 * NS * 4;  // B|C rows as loaded (<= fp32)
  static constexpr size_t off_bc = seq_bytes;
  static constexpr size_t off_ck = off_bc + bc_bytes;
  static constexpr size_t off_a2 = off_ck + ck_bytes;
  static constexpr size_t off_mu = off_a2 + pq_bytes;
  static constexpr size_t off_da = off_mu + pq_bytes;
  static constexpr size_t off_red = off_da + pq_bytes;
  static constexpr size_t off_raw = off_red + red_bytes;
  static constexpr size_t tr_bytes = 4ull * 32 * (KT * 4 + 4) * sizeof(float);  // per-warp transpose [lane][v]
  static constexpr size_t off_tr = off_raw + raw_bytes;
  // sigmoid(delta_pre) and sigmoid(z) of the chunk's steps, kept from the
  // prologue (which already has e^x / computes silu(z)) for the epilogue
  static constexpr size_t sig_bytes = 2ull * KT * kBwdThreads * sizeof(float);
  static constexpr size_t off_sig = off_tr + tr_bytes;
  // 16-step chunks run as two 8-step halves (bwd_chunk16): the record value Q and the
  // adjoint carry a*lam crossing from the right half to the left, per state pair
  static constexpr size_t car_bytes = KT > 8 ? 2ull * NP * kBwdThreads * sizeof(f2) : 0;
  static constexpr size_t off_car = off_sig + sig_bytes;
  static constexpr size_t total = off_car + car_bytes;
};

// u / delta / z / dout rows of one chunk -> ring stage (see SeqStager).
template <typename Tio, bool kVec, int KT>
struct BwdStager {
  static constexpr int PPR = kBwdThreads * sizeof(Tio) / 16;
  static constexpr int EPP = 16 / sizeof(Tio);
  static constexpr int RS = kBwdThreads / PPR;
  static constexpr int KP = (KT + RS - 1) / RS;
  const Tio* base[4];
  long long step[4];
  int row0, col;
  bool ok;
  __device__ __forceinline__ void init(const View3D (&v)[4], int L, bool rev, int b, int e0, int E) {
    if constexpr (kVec) {
      row0 = threadIdx.x / PPR;
      col = (threadIdx.x % PPR) * EPP;
    } else {
      row0 = 0;
      col = threadIdx.x;
    }
    ok = e0 + col < E;
    const int ec = ok ? e0 + col : 0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const View3D w = v[a];
      base[a] = w.p ? static_cast<const Tio*>(w.p) + (long long)b * w.s0 + (long long)ec * w.s2 +
                          (rev ? (long long)(L - 1) * w.s1 : 0)
                    : nullptr;
      step[a] = rev ? -w.s1 : w.s1;
    }
  }
  __device__ __forceinline__ void issue(Tio* seq, int stg, int c, int clen) const {
    if (!ok) return;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (base[a] == nullptr) continue;
      Tio* dst = seq + ((size_t)(stg * 4 + a) * KT) * kBwdThreads + col;
      if constexpr (kVec) {
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int t = row0 + k * RS;
          if (t < clen) cp_async16(dst + t * kBwdThreads, base[a] + (long long)(c + t) * step[a]);
        }
      } else {
        for (int t = 0; t < clen; ++t) dst[t * kBwdThreads] = base[a][(long long)(c + t) * step[a]];
      }
    }
  }
};

struct BwdChunkCtx {
  int c, clen, L, m, stg;
  unsigned tstart, tend;  // bit j: step j starts / ends an LB tile
  bool active, has_z, softplus, linear;
  float Dv, bias;
};

template <typename Tio, int NS, int KT, bool kLB, bool kFull, bool kOneTile>
__device__ __forceinline__ void bwd_chunk(const BwdParams& P, const BwdChunkCtx& x, const Tio* su,
                                          const Tio* sd, const Tio* sz, const Tio* sg,
                                          const float* bcf, const f2* ck, const f2* a2s, f2* mu,
                                          f2* dAs, float* red, float* tr, float* sig, float& dD_acc, float& dbias_acc,
                                          Tio* dup, Tio* ddp, Tio* dzp, long long sdu, long long sdd,
                                          long long sdz) {
  constexpr int NP = NS / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int clen = x.clen;
  float dl[KT], dlu[KT], gy[KT];
  f2 Y[KT], Pacc[KT], S[KT];
  float uvs[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    const bool on = kFull || j < clen;
    dl[j] = on ? to_f(sd[j * kBwdThreads + tid]) + x.bias : 0.f;
    uvs[j] = on ? to_f(su[j * kBwdThreads + tid]) : 0.f;
    gy[j] = (on && x.active) ? to_f(sg[j * kBwdThreads + tid]) : 0.f;
    Y[j] = mk2(0.f, 0.f);
    Pacc[j] = mk2(0.f, 0.f);
    S[j] = mk2(0.f, 0.f);
  }
  // one uniform branch per chunk for each of softplus and the gate: the
  // per-step MUFU chains are independent and interleave
  float* sig_d = sig;                      // [KT][128]: sigmoid(delta + bias)
  float* sig_z = sig + KT * kBwdThreads;   // [KT][128]: sigmoid(z)
  if (x.softplus) {
    // softplus and its derivative from one e^x: 3 MUFU instead of 4
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const float xv = dl[j];
      const float t = ex2(xv * kLog2e);
      const float opt = 1.0f + t;
      float sp = lg2(opt) * (1.0f / kLog2e);
      sp = (xv > 15.0f) ? xv : sp;
      dl[j] = (xv < -15.0f) ? t : sp;
      const float r = rcp(opt);
      sig_d[j * kBwdThreads + tid] = (xv > 15.0f) ? 1.0f - r : t * r;  // t/(1+t) without inf*0
    }
  }
  if (x.has_z) {
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (kFull || j < clen) {
        const float zv = to_f(sz[j * kBwdThreads + tid]);
        const float sg = sigmoid_f(zv);
        sig_z[j * kBwdThreads + tid] = sg;
        gy[j] *= zv * sg;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    if (!(kFull || j < clen)) dl[j] = 0.f;
    dlu[j] = dl[j] * uvs[j];
  }
  const int jlast = kFull ? KT - 1 : clen - 1;

  // tile boundaries: compile-time when the chunk is exactly one tile (M == KT, the
  // LBVim / cfg-3 case), else the per-chunk masks
  auto is_start = [&](int j) -> bool { return kOneTile ? j == 0 : (j == 0 || ((x.tstart >> j) & 1u)); };
  auto is_end = [&](int j) -> bool {
    return kOneTile ? (kFull ? j == KT - 1 : j == clen - 1) : ((x.tend >> j) & 1u);
  };
#pragma unroll 1
  for (int q = 0; q < NP; ++q) {
    const f2 A2 = a2s[q * kBwdThreads + tid];
    const f2 h0 = ck[q * kBwdThreads + tid];
    const f2 mu_in = mu[q * kBwdThreads + tid];
    const float* bq = bcf + 4 * q;  // interleaved table: [t][q][B0 B1 C0 C1]
    auto BC = [&](int j) -> float4 { return *reinterpret_cast<const float4*>(bq + j * 2 * NS); };
    f2 a[KT], h[KT], v[KT];
    // ---- ascending: a, h (state recompute from the checkpoint), LB adjoint v
    f2 hp = h0;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (kFull || j < clen) {
        const float4 bc = BC(j);
        const f2 xa = mul2(bc2(dl[j]), A2);
        a[j] = x.linear ? xa : mk2(ex2(xa.x), ex2(xa.y));
        hp = fma2(a[j], hp, mul2(bc2(dlu[j]), mk2(bc.x, bc.y)));
        h[j] = hp;
        if (kLB) {
          const f2 g = mul2(bc2(gy[j]), mk2(bc.z, bc.w));
          v[j] = is_start(j) ? g : fma2(a[j > 0 ? j - 1 : 0], v[j > 0 ? j - 1 : 0], g);
        }
      } else {
        a[j] = mk2(0.f, 0.f);
        h[j] = mk2(0.f, 0.f);
        v[j] = mk2(0.f, 0.f);
      }
    }
    // ---- descending: LB record Q = r + b, adjoint lam, chain terms
    f2 Qn = mk2(0.f, 0.f), lam = mk2(0.f, 0.f), dAq = mk2(0.f, 0.f);
#pragma unroll
    for (int j = KT - 1; j >= 0; --j) {
      f2 dBv = mk2(0.f, 0.f), dCv = mk2(0.f, 0.f);
      if (kFull || j < clen) {
        const float4 bc = BC(j);
        const f2 Bv = mk2(bc.x, bc.y);
        const f2 Cv = mk2(bc.z, bc.w);
        const f2 bj = mul2(bc2(dlu[j]), Bv);
        const f2 g = mul2(bc2(gy[j]), Cv);
        const bool tend = is_end(j);
        const bool tstart = is_start(j);
        f2 hr = h[j], Qc = bj;
        if (kLB && !tend) {
          hr = fma2(a[j], Qn, h[j]);
          Qc = fma2(a[j], Qn, bj);
        }
        const f2 lamj = (j == jlast) ? add2(g, mu_in) : fma2(a[j < KT - 1 ? j + 1 : j], lam, g);
        const f2 hprev = j > 0 ? h[j > 0 ? j - 1 : 0] : h0;
        f2 dab = mul2(lamj, hprev);
        if (kLB && !tend) dab = fma2(v[j], Qn, dab);
        f2 dbx = lamj;
        if (kLB && !tstart) dbx = fma2(a[j > 0 ? j - 1 : 0], v[j > 0 ? j - 1 : 0], dbx);
        const f2 da = x.linear ? dab : mul2(dab, a[j]);
        Pacc[j] = fma2(da, A2, Pacc[j]);
        dAq = fma2(da, bc2(dl[j]), dAq);
        S[j] = fma2(dbx, Bv, S[j]);
        if (x.has_z) Y[j] = fma2(Cv, hr, Y[j]);
        // threads past the last channel (E % 128 != 0) run on unstaged shared-memory
        // rows: their terms must not enter the block's dB/dC sums (0 * NaN = NaN)
        dBv = x.active ? mul2(dbx, bc2(dlu[j])) : mk2(0.f, 0.f);
        dCv = x.active ? mul2(hr, bc2(gy[j])) : mk2(0.f, 0.f);
        lam = lamj;
        Qn = Qc;
      }
      // this lane's row [lane][v] of the warp's transpose buffer, row stride KT*4+4
      // (= 4 mod 32: the 16-byte stores of a quarter-warp hit distinct banks)
      float* tw = tr + (size_t)warp * 32 * (KT * 4 + 4);
      *reinterpret_cast<float4*>(&tw[lane * (KT * 4 + 4) + j * 4]) = make_float4(dBv.x, dBv.y, dCv.x, dCv.y);
    }
    // warp sum of each of the KT*4 values: lane l owns values l, l+32, ...
    __syncwarp();
    {
      const float* tw = tr + (size_t)warp * 32 * (KT * 4 + 4);
#pragma unroll
      for (int v0 = 0; v0 < KT * 4; v0 += 32) {
        const int vv = v0 + lane;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          s0 += tw[k * (KT * 4 + 4) + vv];
          s1 += tw[(k + 1) * (KT * 4 + 4) + vv];
          s2 += tw[(k + 2) * (KT * 4 + 4) + vv];
          s3 += tw[(k + 3) * (KT * 4 + 4) + vv];
        }
        const int jj = vv >> 2, kind = vv & 3;
        red[((warp * KT + jj) * 2 + (kind >> 1)) * NS + 2 * q + (kind & 1)] = (s0 + s1) + (s2 + s3);
      }
    }
    __syncwarp();
    // carry into the previous chunk: a_{c} * lam_{c}
    mu[q * kBwdThreads + tid] = mul2(a[0], lam);
    dAs[q * kBwdThreads + tid] = add2(dAs[q * kBwdThreads + tid], dAq);
  }

  // ---- per-step outputs: du, ddelta, dz
  if (x.active) {
    Tio* dupj = dup + (long long)x.c * sdu;
    Tio* ddpj = ddp + (long long)x.c * sdd;
    Tio* dzpj = dzp + (long long)x.c * sdz;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (kFull || j < clen) {
        const float uv = uvs[j];
        const float s = S[j].x + S[j].y;
        const float duv = x.Dv * gy[j] + dl[j] * s;
        const float pp = (Pacc[j].x + Pacc[j].y) * (x.linear ? 1.f : kLn2);
        const float ddl = pp + uv * s;
        const float ddv = x.softplus ? ddl * sig_d[j * kBwdThreads + tid] : ddl;
        dbias_acc += ddv;
        dD_acc += gy[j] * uv;
        st<Tio>(dupj, duv);
        st<Tio>(ddpj, ddv);
        if (x.has_z) {
          const float y = Y[j].x + Y[j].y + x.Dv * uv;
          const float zv = to_f(sz[j * kBwdThreads + tid]);
          const float sgm = sig_z[j * kBwdThreads + tid];
          const float go = to_f(sg[j * kBwdThreads + tid]);
          st<Tio>(dzpj, go * y * sgm * (1.f + zv * (1.f - sgm)));
        }
      }
      dupj += sdu;
      ddpj += sdd;
      dzpj += sdz;
    }
  }
}

// A 16-step chunk (windows 9..16: the chunk is exactly one tile, possibly the
// ragged last one) processed as two 8-step halves, step-half outer and state pair
// inner, so only one half's per-step accumulators (Y, Pacc, S) and per-pair
// arrays (a, h, v) are live — the one-pass form needs both halves' and spills
// (1.2-1.8 KB per thread).  Right half first (the adjoint runs backwards): per
// pair an ascending pass over the left half keeps only its end values (h_7,
// v_7, a_7), the right half's descending pass leaves the record Q_8 and the
// carry a_8 lam_8 in shared memory, and the left half then recomputes its decays
// (+50 % exps on 16-step windows) and finishes the tile.  Same terms and order
// per step as bwd_chunk.
template <typename Tio, int NS, bool kLB, bool kFull>
__device__ __forceinline__ void bwd_chunk16(const BwdParams& P, const BwdChunkCtx& x, const Tio* su,
                                            const Tio* sd, const Tio* sz, const Tio* sg, const float* bcf,
                                            const f2* ck, const f2* a2s, f2* mu, f2* dAs, float* red, float* tr,
                                            float* sig, f2* car, float& dD_acc, float& dbias_acc, Tio* dup, Tio* ddp,
                                            Tio* dzp, long long sdu, long long sdd, long long sdz) {
  constexpr int KT = 16, H = 8;
  constexpr int NP = NS / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int clen = kFull ? KT : x.clen;
  const int nL = kFull ? H : min(H, clen), nR = kFull ? H : max(0, clen - H);
  float dl[KT], dlu[KT], gy[KT];
  float* sig_d = sig;
  float* sig_z = sig + KT * kBwdThreads;
  f2* qcar = car;                        // [NP][128]: Q_8
  f2* lcar = car + NP * kBwdThreads;     // [NP][128]: a_8 lam_8
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    const bool on = kFull || j < clen;
    dl[j] = on ? to_f(sd[j * kBwdThreads + tid]) + x.bias : 0.f;
    gy[j] = (on && x.active) ? to_f(sg[j * kBwdThreads + tid]) : 0.f;
  }
  if (x.softplus) {
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const float xv = dl[j];
      const float t = ex2(xv * kLog2e);
      const float opt = 1.0f + t;
      float sp = lg2(opt) * (1.0f / kLog2e);
      sp = (xv > 15.0f) ? xv : sp;
      dl[j] = (xv < -15.0f) ? t : sp;
      const float r = rcp(opt);
      sig_d[j * kBwdThreads + tid] = (xv > 15.0f) ? 1.0f - r : t * r;
    }
  }
  if (x.has_z) {
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (kFull || j < clen) {
        const float zv = to_f(sz[j * kBwdThreads + tid]);
        const float sgm = sigmoid_f(zv);
        sig_z[j * kBwdThreads + tid] = sgm;
        gy[j] *= zv * sgm;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    if (!(kFull || j < clen)) dl[j] = 0.f;
    dlu[j] = dl[j] * ((kFull || j < clen) ? to_f(su[j * kBwdThreads + tid]) : 0.f);
  }

#pragma unroll
  for (int half = 1; half >= 0; --half) {
    const int o = half * H;            // chunk step of the half's first step
    const int n = half ? nR : nL;      // steps in this half
    if (n <= 0) continue;              // uniform: the chunk is one half long
    f2 Y[H], Pacc[H], S[H];
#pragma unroll
    for (int jj = 0; jj < H; ++jj) Y[jj] = Pacc[jj] = S[jj] = mk2(0.f, 0.f);
#pragma unroll 1
    for (int q = 0; q < NP; ++q) {
      const f2 A2 = a2s[q * kBwdThreads + tid];
      const f2 h0 = ck[q * kBwdThreads + tid];
      const float* bq = bcf + 4 * q;
      auto BC = [&](int j) -> float4 { return *reinterpret_cast<const float4*>(bq + j * 2 * NS); };
      auto decay = [&](int j) -> f2 {
        const f2 xa = mul2(bc2(dl[j]), A2);
        return x.linear ? xa : mk2(ex2(xa.x), ex2(xa.y));
      };
      // entering the half: state, LB adjoint and decay of the step before it
      f2 hin = h0, vin = mk2(0.f, 0.f), ain = mk2(0.f, 0.f);
      if (half) {
        f2 hp = h0, vv = mk2(0.f, 0.f), ap = mk2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const float4 bc = BC(j);
          const f2 aj = decay(j);
          hp = fma2(aj, hp, mul2(bc2(dlu[j]), mk2(bc.x, bc.y)));
          if (kLB) {
            const f2 g = mul2(bc2(gy[j]), mk2(bc.z, bc.w));
            vv = j == 0 ? g : fma2(ap, vv, g);
          }
          ap = aj;
        }
        hin = hp;
        vin = vv;
        ain = ap;
      }
      f2 a[H], h[H], v[H];
      f2 hp = hin;
#pragma unroll
      for (int jj = 0; jj < H; ++jj) {
        const int j = o + jj;
        if (jj < n) {
          const float4 bc = BC(j);
          a[jj] = decay(j);
          hp = fma2(a[jj], hp, mul2(bc2(dlu[j]), mk2(bc.x, bc.y)));
          h[jj] = hp;
          if (kLB) {
            const f2 g = mul2(bc2(gy[j]), mk2(bc.z, bc.w));
            const f2 ap = jj > 0 ? a[jj > 0 ? jj - 1 : 0] : ain;
            const f2 vp = jj > 0 ? v[jj > 0 ? jj - 1 : 0] : vin;
            v[jj] = (!half && jj == 0) ? g : fma2(ap, vp, g);  // the tile starts at chunk step 0
          }
        } else {
          a[jj] = h[jj] = v[jj] = mk2(0.f, 0.f);
        }
      }
      // descending; the tile ends at chunk step clen - 1 (in the right half unless
      // the chunk is at most one half long)
      const bool end_here = half || nR == 0;
      f2 Qn = (!half && nR > 0) ? qcar[q * kBwdThreads + tid] : mk2(0.f, 0.f);
      const f2 lin = (!half && nR > 0) ? lcar[q * kBwdThreads + tid] : mu[q * kBwdThreads + tid];
      f2 lam = mk2(0.f, 0.f), dAq = mk2(0.f, 0.f);
      float* tw = tr + (size_t)warp * 32 * (KT * 4 + 4);
#pragma unroll
      for (int jj = H - 1; jj >= 0; --jj) {
        const int j = o + jj;
        f2 dBv = mk2(0.f, 0.f), dCv = mk2(0.f, 0.f);
        if (jj < n) {
          const float4 bc = BC(j);
          const f2 Bv = mk2(bc.x, bc.y);
          const f2 Cv = mk2(bc.z, bc.w);
          const f2 bj = mul2(bc2(dlu[j]), Bv);
          const f2 g = mul2(bc2(gy[j]), Cv);
          const bool tend = end_here && jj == n - 1;
          const bool tstart = !half && jj == 0;
          f2 hr = h[jj], Qc = bj;
          if (kLB && !tend) {
            hr = fma2(a[jj], Qn, h[jj]);
            Qc = fma2(a[jj], Qn, bj);
          }
          const f2 lamj = (jj == n - 1) ? add2(g, lin) : fma2(a[jj < H - 1 ? jj + 1 : jj], lam, g);
          const f2 hprev = jj > 0 ? h[jj > 0 ? jj - 1 : 0] : hin;
          f2 dab = mul2(lamj, hprev);
          if (kLB && !tend) dab = fma2(v[jj], Qn, dab);
          f2 dbx = lamj;
          if (kLB && !tstart) {
            const f2 ap = jj > 0 ? a[jj > 0 ? jj - 1 : 0] : ain;
            const f2 vp = jj > 0 ? v[jj > 0 ? jj - 1 : 0] : vin;
            dbx = fma2(ap, vp, dbx);
          }
          const f2 da = x.linear ? dab : mul2(dab, a[jj]);
          Pacc[jj] = fma2(da, A2, Pacc[jj]);
          dAq = fma2(da, bc2(dl[j]), dAq);
          S[jj] = fma2(dbx, Bv, S[jj]);
          if (x.has_z) Y[jj] = fma2(Cv, hr, Y[jj]);
          dBv = x.active ? mul2(dbx, bc2(dlu[j])) : mk2(0.f, 0.f);
          dCv = x.active ? mul2(hr, bc2(gy[j])) : mk2(0.f, 0.f);
          lam = lamj;
          Qn = Qc;
        }
        *reinterpret_cast<float4*>(&tw[lane * (KT * 4 + 4) + j * 4]) = make_float4(dBv.x, dBv.y, dCv.x, dCv.y);
      }
      // warp sums of the half's 8 steps x 4 values: lane l owns value o*4 + l
      __syncwarp();
      {
        const int vv = o * 4 + lane;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          s0 += tw[k * (KT * 4 + 4) + vv];
          s1 += tw[(k + 1) * (KT * 4 + 4) + vv];
          s2 += tw[(k + 2) * (KT * 4 + 4) + vv];
          s3 += tw[(k + 3) * (KT * 4 + 4) + vv];
        }
        const int jj = vv >> 2, kind = vv & 3;
        red[((warp * KT + jj) * 2 + (kind >> 1)) * NS + 2 * q + (kind & 1)] = (s0 + s1) + (s2 + s3);
      }
      __syncwarp();
      if (half) {
        qcar[q * kBwdThreads + tid] = Qn;               // Q_8
        lcar[q * kBwdThreads + tid] = mul2(a[0], lam);  // a_8 lam_8
      } else {
        mu[q * kBwdThreads + tid] = mul2(a[0], lam);    // carry into the previous chunk
      }
      dAs[q * kBwdThreads + tid] = add2(dAs[q * kBwdThreads + tid], dAq);
    }
    // ---- per-step outputs of the half: du, ddelta, dz
    if (x.active) {
#pragma unroll
      for (int jj = 0; jj < H; ++jj) {
        const int j = o + jj;
        if (jj < n) {
          const float uv = to_f(su[j * kBwdThreads + tid]);
          const float s = S[jj].x + S[jj].y;
          const float duv = x.Dv * gy[j] + dl[j] * s;
          const float pp = (Pacc[jj].x + Pacc[jj].y) * (x.linear ? 1.f : kLn2);
          const float ddl = pp + uv * s;
          const float ddv = x.softplus ? ddl * sig_d[j * kBwdThreads + tid] : ddl;
          dbias_acc += ddv;
          dD_acc += gy[j] * uv;
          st<Tio>(dup + (long long)(x.c + j) * sdu, duv);
          st<Tio>(ddp + (long long)(x.c + j) * sdd, ddv);
          if (x.has_z) {
            const float y = Y[jj].x + Y[jj].y + x.Dv * uv;
            const float zv = to_f(sz[j * kBwdThreads + tid]);
            const float sgm = sig_z[j * kBwdThreads + tid];
            const float go = to_f(sg[j * kBwdThreads + tid]);
            st<Tio>(dzp + (long long)(x.c + j) * sdz, go * y * sgm * (1.f + zv * (1.f - sgm)));
          }
        }
      }
    }
  }
}

#ifndef LBS_BWD_MINB
#define LBS_BWD_MINB 2
#endif

template <typename Tio, typename Tbc, int NS, int KT, bool kLB, bool kVec>
__global__ void __launch_bounds__(kBwdThreads, LBS_BWD_MINB) bwd_kernel(BwdParams P) {
  constexpr int NP = NS / 2;
  using Sm = BwdSmem<Tio, NS, KT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tio* seq = reinterpret_cast<Tio*>(smem_raw);
  float* bcf = reinterpret_cast<float*>(smem_raw + Sm::off_bc);
  f2* cks = reinterpret_cast<f2*>(smem_raw + Sm::off_ck);
  f2* a2s = reinterpret_cast<f2*>(smem_raw + Sm::off_a2);
  f2* mus = reinterpret_cast<f2*>(smem_raw + Sm::off_mu);
  f2* dAs = reinterpret_cast<f2*>(smem_raw + Sm::off_da);
  float* red = reinterpret_cast<float*>(smem_raw + Sm::off_red);
  Tbc* bcraw = reinterpret_cast<Tbc*>(smem_raw + Sm::off_raw);
  float* trs = reinterpret_cast<float*>(smem_raw + Sm::off_tr);
  float* sigs = reinterpret_cast<float*>(smem_raw + Sm::off_sig);

  const FwdParams& p = P.f;
  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * kBwdThreads;
  const int e = e0 + tid;
  const int b = blockIdx.y;
  const bool active = e < p.E;
  const int ec = active ? e : p.E - 1;
  const int L = p.L, N = p.N, m = p.m, K = p.ckpt_len, nck = p.n_ckpt;
  const int seg = blockIdx.z;
  const int k_lo = seg * P.seg_chunks;
  const int k_hi = min(nck, k_lo + P.seg_chunks);
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool linear = p.flags & LBS_FLAG_LINEAR;
  const bool has_z = p.z.p != nullptr;

#pragma unroll
  for (int q = 0; q < NP; ++q) {
    float a0 = 2 * q < N ? p.A[(long long)ec * N + 2 * q] : 0.f;
    float a1 = 2 * q + 1 < N ? p.A[(long long)ec * N + 2 * q + 1] : 0.f;
    if (!linear) { a0 *= kLog2e; a1 *= kLog2e; }
    a2s[q * kBwdThreads + tid] = mk2(a0, a1);
    // carry entering from the right: fold the maps of segments n_seg-1 .. seg+1
    f2 mu = mk2(0.f, 0.f);
    if (seg + 1 < P.n_seg) {
      const f2* agg = reinterpret_cast<const f2*>(P.bagg) + ((long long)b * P.n_seg * p.E + ec) * NS + q;
      const long long sstride = (long long)p.E * NS;
      if (P.n_seg <= kFoldMax) {
#pragma unroll 8
        for (int s = P.n_seg - 1; s > seg; --s) mu = fma2(agg[s * sstride], mu, agg[s * sstride + NP]);
      } else {
        // maps stored right to left and folded by segment_prefix_kernel: the H slot of
        // reversed segment r holds the carry entering reversed segment r + 1
        mu = agg[(long long)(P.n_seg - 2 - seg) * sstride + NP];
      }
    }
    mus[q * kBwdThreads + tid] = mu;
    dAs[q * kBwdThreads + tid] = mk2(0.f, 0.f);
  }
  BwdChunkCtx x;
  x.L = L;
  x.m = m;
  x.active = active;
  x.has_z = has_z;
  x.softplus = p.flags & LBS_FLAG_SOFTPLUS;
  x.linear = linear;
  x.Dv = p.D ? p.D[ec] : 0.f;
  x.bias = p.bias ? p.bias[ec] : 0.f;
  float dD_acc = 0.f, dbias_acc = 0.f;

  // output row bases (flip-on-store for the reverse direction)
  auto obase = [&](const OutView& o) -> Tio* {
    if (o.p == nullptr) return nullptr;
    return static_cast<Tio*>(o.p) + (long long)b * o.s0 + (long long)ec * o.s2 + (rev ? (long long)(L - 1) * o.s1 : 0);
  };
  Tio* dup = obase(P.du);
  Tio* ddp = obase(P.ddelta);
  Tio* dzp = obase(P.dz);
  const long long sdu = rev ? -P.du.s1 : P.du.s1;
  const long long sdd = rev ? -P.ddelta.s1 : P.ddelta.s1;
  const long long sdz = rev ? -P.dz.s1 : P.dz.s1;

  const View3D zv = has_z ? p.z : View3D{nullptr, 0, 0, 0};
  const View3D views[4] = {p.u, p.delta, zv, P.dout};
  BwdStager<Tio, kVec, KT> stager;
  stager.init(views, L, rev, b, e0, p.E);
  // interleaved fp32 table, cp.async when aligned; the scalar table build (the vectorised
  // one measured +1.8 % on the configs[2] backward)
  BcStage<Tbc, NS, KT, kVec && bc_async_ok<Tbc, NS>(), true, kBwdThreads, false> bcs;
  bcs.init(p, b);
  const bool one_tile = m == KT;
  const f2* ckg = reinterpret_cast<const f2*>(p.ckpt) + (long long)b * nck * NP * p.E + ec;
  auto ck_issue = [&](int stg, int k) {
#pragma unroll
    for (int q = 0; q < NP; ++q)
      cp_async8(&cks[(stg * NP + q) * kBwdThreads + tid], ckg + ((long long)k * NP + q) * p.E);
  };

  int k = k_hi - 1;
  int c = k * K;
  int clen = min(K, L - c);
  stager.issue(seq, 0, c, clen);
  ck_issue(0, k);
  bcs.issue(bcraw, 0, c, clen);
  cp_async_commit();
  const int eblk = blockIdx.x;
  for (int it = 0; k >= k_lo; ++it, --k) {
    const int stg = it & 1;
    cp_async_wait_all();
    __syncthreads();  // chunk k landed; chunk k+1 compute (and its partial write) done
    bcs.publish(bcf, bcraw, stg, clen);
    if (k > k_lo) {
      stager.issue(seq, stg ^ 1, c - K, K);
      ck_issue(stg ^ 1, k - 1);
      bcs.issue(bcraw, stg ^ 1, c - K, K);
    }
    cp_async_commit();
    __syncthreads();  // bcf visible

    x.c = c;
    x.clen = clen;
    x.stg = stg;
    // tile start / end bits of this chunk's steps (only needed when a chunk holds
    // several tiles); one division per chunk, the phase then steps without any
    // (16 runtime modulos per chunk were 12 % of the kernel's stall samples)
    unsigned ts = 0u, te = 0u;
    if (!one_tile) {
      int ph = c % m;
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        if (j < clen) {
          if (ph == 0) ts |= 1u << j;
          if (ph == m - 1 || c + j == L - 1) te |= 1u << j;
          ph = ph + 1 == m ? 0 : ph + 1;
        }
      }
    }
    x.tstart = ts;
    x.tend = te;
    const Tio* base = seq + (size_t)stg * 4 * KT * kBwdThreads;
    const Tio* su = base;
    const Tio* sd = base + KT * kBwdThreads;
    const Tio* sz = base + 2 * KT * kBwdThreads;
    const Tio* sg = base + 3 * KT * kBwdThreads;
    const f2* ck = cks + stg * NP * kBwdThreads;
#define LBS_BWD_CHUNK(FULL, ONE)                                                                     \
  bwd_chunk<Tio, NS, KT, kLB, FULL, ONE>(P, x, su, sd, sz, sg, bcf, ck, a2s, mus, dAs, red, trs, sigs, dD_acc, dbias_acc, \
                                         dup, ddp, dzp, sdu, sdd, sdz)
    if constexpr (KT == 16) {
      // windows 9..16: the chunk is one tile (bwd_chunk_len), run as two halves
      f2* cars = reinterpret_cast<f2*>(smem_raw + Sm::off_car);
      if (clen == KT)
        bwd_chunk16<Tio, NS, kLB, true>(P, x, su, sd, sz, sg, bcf, ck, a2s, mus, dAs, red, trs, sigs, cars, dD_acc,
                                        dbias_acc, dup, ddp, dzp, sdu, sdd, sdz);
      else
        bwd_chunk16<Tio, NS, kLB, false>(P, x, su, sd, sz, sg, bcf, ck, a2s, mus, dAs, red, trs, sigs, cars, dD_acc,
                                         dbias_acc, dup, ddp, dzp, sdu, sdd, sdz);
    } else if (one_tile) {
      if (clen == KT) LBS_BWD_CHUNK(true, true);
      else LBS_BWD_CHUNK(false, true);
    } else {
      if (clen == KT) LBS_BWD_CHUNK(true, false);
      else LBS_BWD_CHUNK(false, false);
    }
#undef LBS_BWD_CHUNK
    __syncthreads();  // red complete
    // dB / dC partials of this channel block: sum the 4 warps
    for (int i = tid; i < KT * 2 * NS; i += kBwdThreads) {
      const int j = i / (2 * NS);
      if (j < clen) {
        const float s = red[i] + red[KT * 2 * NS + i] + red[2 * KT * 2 * NS + i] + red[3 * KT * 2 * NS + i];
        P.part_bc[(((long long)eblk * p.Bt + b) * L + (c + j)) * (2 * NS) + (i - j * 2 * NS)] = s;
      }
    }
    c -= K;
    clen = K;
  }
  if (active) {
    float* pw = P.part_w + ((long long)b * P.n_seg + seg) * (NS + 2) * p.E + e;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const f2 d = dAs[q * kBwdThreads + tid];
      pw[(long long)(2 * q) * p.E] = d.x;
      pw[(long long)(2 * q + 1) * p.E] = d.y;
    }
    pw[(long long)NS * p.E] = dD_acc;
    pw[(long long)(NS + 1) * p.E] = dbias_acc;
  }
}

// Pass 1 of the backward's sequence split.  Segment s (steps [lo, hi)) hands
// its left neighbour the carry mu_out = a_lo lam_lo of the global adjoint
// lam_t = g_t + a_{t+1} lam_{t+1} (autodiff.py:125-137), g = C gy.  As a map
// of the carry entering from the right, mu_in = a_hi lam_hi, it is affine:
// mu_out = P mu_in + M with P = prod_{t in seg} a_t = exp(A sum dl) and M the
// carry computed from mu_in = 0 — both per lane, computed here by one sweep
// over the segment from the right.  (The LB record and its adjoint are
// tile-local and segments are whole chunks of whole tiles, so nothing else
// crosses a segment boundary; the states come from the checkpoints.)
// p.u is the upstream gradient dout (staged in u's slot).  Segment 0's map is
// never needed: blockIdx.z = s - 1.
template <typename Tio, typename Tbc, int NS, bool kVec>
__global__ void __launch_bounds__(kBwdThreads) bwd_segment_adjoint_kernel(FwdParams p, int seg_steps, float* bagg,
                                                                          bool reversed) {
  constexpr int NP = NS / 2;
  constexpr int CL = LBS_FWD_CL;
  constexpr int CT = kBwdThreads;
  using Sm = FwdSmem<Tio, Tbc, NS, CL, CT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tio* seq = reinterpret_cast<Tio*>(smem_raw);
  float* bcf = reinterpret_cast<float*>(smem_raw + Sm::seq_bytes);
  f2* a2s = reinterpret_cast<f2*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes);
  Tbc* bcraw = reinterpret_cast<Tbc*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes + Sm::a2_bytes);

  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * CT;
  const int e = e0 + tid;
  const int b = blockIdx.y;
  const int seg = blockIdx.z + 1;
  const int n_seg = gridDim.z + 1;
  const bool active = e < p.E;
  const int ec = active ? e : p.E - 1;
  const int N = p.N;
  const bool softplus = p.flags & LBS_FLAG_SOFTPLUS;
  const bool linear = p.flags & LBS_FLAG_LINEAR;
  const bool has_z = p.z.p != nullptr;
  const int lo = seg * seg_steps;
  const int hi = min(p.L, lo + seg_steps);

#pragma unroll
  for (int q = 0; q < NP; ++q) {
    float a0 = 2 * q < N ? p.A[(long long)ec * N + 2 * q] : 0.f;
    float a1 = 2 * q + 1 < N ? p.A[(long long)ec * N + 2 * q + 1] : 0.f;
    if (!linear) { a0 *= kLog2e; a1 *= kLog2e; }
    a2s[q * CT + tid] = mk2(a0, a1);
  }
  const float bias = p.bias ? p.bias[ec] : 0.f;
  f2 mu[NP], P[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) { mu[q] = mk2(0.f, 0.f); P[q] = mk2(1.f, 1.f); }
  float dsum = 0.f;

  SeqStager<Tio, kVec, CL, CT> stager;
  stager.init(p, b, e0, has_z);
  BcStage<Tbc, NS, CL, kVec && bc_async_ok<Tbc, NS>(), kBcIL, CT> bcs;
  bcs.init(p, b);
  // chunks of the segment, right to left
  const int nch = (hi - lo + CL - 1) / CL;
  int k = nch - 1;
  int c = lo + k * CL;
  int clen = hi - c;
  stager.issue(seq, 0, c, clen);
  bcs.issue(bcraw, 0, c, clen);
  cp_async_commit();
  for (int it = 0; k >= 0; ++it, --k) {
    const int stg = it & 1;
    cp_async_wait_all();
    __syncthreads();
    bcs.publish(bcf, bcraw, stg, clen);
    if (k > 0) {
      stager.issue(seq, stg ^ 1, c - CL, CL);
      bcs.issue(bcraw, stg ^ 1, c - CL, CL);
    }
    cp_async_commit();
    __syncthreads();
    const Tio* sg = seq + ((size_t)stg * 3 + 0) * CL * CT;  // dout (u's slot)
    const Tio* sd = seq + ((size_t)stg * 3 + 1) * CL * CT;
    const Tio* sz = seq + ((size_t)stg * 3 + 2) * CL * CT;
    for (int t = clen - 1; t >= 0; --t) {
      float dl = to_f(sd[t * CT + tid]) + bias;
      if (softplus) dl = softplus_f(dl);
      float gy = to_f(sg[t * CT + tid]);
      if (has_z) gy *= silu_f(to_f(sz[t * CT + tid]));
      dsum += dl;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const f2 x = mul2(bc2(dl), a2s[q * CT + tid]);
        const f2 a = linear ? x : mk2(ex2(x.x), ex2(x.y));
        const f2 Cv = *reinterpret_cast<const f2*>(&bcf[bc_index<NS, kBcIL>(t, 1, 2 * q)]);
        const f2 lam = fma2(bc2(gy), Cv, mu[q]);  // lam_t = g_t + a_{t+1} lam_{t+1}
        mu[q] = mul2(a, lam);                     // carry a_t lam_t to step t-1
        if (linear) P[q] = mul2(P[q], a);
      }
    }
    c -= CL;
    clen = CL;
  }
  if (!linear) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const f2 x = mul2(bc2(dsum), a2s[q * CT + tid]);
      P[q] = mk2(ex2(x.x), ex2(x.y));
    }
  }
  if (active) {
    // reversed: segments stored right to left, so segment_prefix_kernel's left-to-right
    // fold yields the carry entering each segment from the right
    const int slot = reversed ? n_seg - 1 - seg : seg;
    f2* out = reinterpret_cast<f2*>(bagg + ((((long long)b * n_seg + slot) * p.E + e) * (2 * NS)));
#pragma unroll
    for (int q = 0; q < NP; ++q) { out[q] = P[q]; out[NP + q] = mu[q]; }
  }
}

// Deterministic reductions of the partials (fixed order, fp64 accumulate).
template <int NS>
__device__ __forceinline__ void bwd_reduce_bc(const BwdParams& P, int n_eblk, long long idx) {
  const FwdParams& p = P.f;
  const long long total = (long long)p.Bt * p.L * 2 * p.N;
  if (idx >= total) return;
  const int n = idx % p.N;
  const int which = (idx / p.N) % 2;
  const long long bt = idx / (2 * p.N);
  const int t = bt % p.L;
  const int b = bt / p.L;
  double s = 0.0;
  for (int k = 0; k < n_eblk; ++k)
    s += P.part_bc[(((long long)k * p.Bt + b) * p.L + t) * (2 * NS) + which * NS + n];
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const long long tp = rev ? (p.L - 1 - t) : t;
  if (which == 0)
    P.dB[b * P.sb0 + tp * P.sb1 + n * P.sb2] = (float)s;
  else
    P.dC[b * P.sc0 + tp * P.sc1 + n * P.sc2] = (float)s;
}

// dA[e, n], dD[e], dbias[e]: one 256-thread block per (output row, 32 channels); the
// lanes are 32 consecutive channels (coalesced 128-byte reads of the [row][e] partial
// rows), the 8 warps sum fixed contiguous ranges of the (batch row, segment) partials
// in order, then warp 0 adds the 8 warp sums in order -- deterministic, and no long
// serial chain when the backward was split into hundreds of segments.  (The round-1
// form, a warp per output with the lanes striding the partials, read one 32-byte
// sector per 4-byte value: 21 us of the configs[2] backward.)
template <int NS>
__device__ __forceinline__ void bwd_reduce_w(const BwdParams& P, int blk) {
  const FwdParams& p = P.f;
  const int n_eb = (p.E + 31) / 32;
  const int i = blk / n_eb;
  if (i >= p.N + 2) return;  // block-uniform
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = (blk % n_eb) * 32 + lane;
  const int row = i < p.N ? i : NS + (i - p.N);
  const int rows = p.Bt * P.n_seg;  // (batch row, segment) partials
  const int per = (rows + 7) / 8;
  const int r0 = min(rows, warp * per), r1 = min(rows, r0 + per);
  double s = 0.0;
  if (e < p.E) {
    const float* src = P.part_w + (long long)row * p.E + e;
    const long long rstride = (long long)(NS + 2) * p.E;
#pragma unroll 8
    for (int r = r0; r < r1; ++r) s += src[r * rstride];
  }
  __shared__ double wsum[8][32];
  wsum[warp][lane] = s;
  __syncthreads();
  if (warp != 0 || e >= p.E) return;
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += wsum[w][lane];
  if (i < p.N)
    P.dA[(long long)e * p.N + i] += (float)t;
  else if (i == p.N) {
    if (P.dD) P.dD[e] += (float)t;
  } else if (P.dbias) {
    P.dbias[e] += (float)t;
  }
}

// both fixed-order reductions in one launch: blocks [0, nbc_blocks) reduce dB/dC over
// the channel blocks, the rest dA/dD/dbias over the batch rows and segments
template <int NS>
__global__ void __launch_bounds__(256) bwd_reduce_kernel(BwdParams P, int n_eblk, int nbc_blocks) {
  if ((int)blockIdx.x < nbc_blocks)
    bwd_reduce_bc<NS>(P, n_eblk, (long long)blockIdx.x * blockDim.x + threadIdx.x);
  else
    bwd_reduce_w<NS>(P, (int)blockIdx.x - nbc_blocks);
}

template <typename Tio, typename Tbc, int NS, int KT, bool kVec>
inline cudaError_t launch_bwd_t(const BwdParams& P, cudaStream_t st) {
  const size_t smem = BwdSmem<Tio, NS, KT>::total;
  const FwdParams& p = P.f;
  const int n_eblk = (p.E + kBwdThreads - 1) / kBwdThreads;
  if (P.n_seg > 1) {
    FwdParams pa = p;
    pa.u = P.dout;  // the adjoint sweep stages dout in u's slot
    const size_t smem1 = FwdSmem<Tio, Tbc, NS, LBS_FWD_CL, kBwdThreads>::total;
    auto k1 = bwd_segment_adjoint_kernel<Tio, Tbc, NS, kVec>;
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    const bool many = P.n_seg > kFoldMax;
    k1<<<dim3(n_eblk, p.Bt, P.n_seg - 1), kBwdThreads, smem1, st>>>(pa, P.seg_chunks * p.ckpt_len, P.bagg, many);
    if (many) {
      FwdParams pp = p;
      pp.n_seg = P.n_seg;
      pp.seg_agg = P.bagg;
      const long long lanes = (long long)p.Bt * p.E * (NS / 2);  // one warp each
      segment_prefix_kernel<NS><<<(unsigned)((lanes * 32 + 127) / 128), 128, 0, st>>>(pp);
    }
  }
  dim3 grid(n_eblk, p.Bt, P.n_seg);
  auto k = (p.flags & LBS_FLAG_LB) ? bwd_kernel<Tio, Tbc, NS, KT, true, kVec>
                                   : bwd_kernel<Tio, Tbc, NS, KT, false, kVec>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, kBwdThreads, smem, st>>>(P);
  const long long nbc = (long long)p.Bt * p.L * 2 * p.N;
  const int nbc_blocks = (int)((nbc + 255) / 256);
  const int nw_blocks = ((p.E + 31) / 32) * (p.N + 2);  // one block per (output row, 32 channels)
  bwd_reduce_kernel<NS><<<(unsigned)(nbc_blocks + nw_blocks), 256, 0, st>>>(P, n_eblk, nbc_blocks);
  return cudaGetLastError();
}

template <typename Tio, typename Tbc, int NS, bool kVec>
inline cudaError_t launch_bwd_m(const BwdParams& P, cudaStream_t st) {
  if (P.f.m <= 8) return launch_bwd_t<Tio, Tbc, NS, 8, kVec>(P, st);
  return launch_bwd_t<Tio, Tbc, NS, 16, kVec>(P, st);
}

template <typename Tio, typename Tbc, bool kVec>
inline cudaError_t launch_bwd_n(const BwdParams& P, cudaStream_t st) {
  if (P.f.N <= 4) return launch_bwd_m<Tio, Tbc, 4, kVec>(P, st);
  return launch_bwd_m<Tio, Tbc, 16, kVec>(P, st);
}

template <typename Tio, typename Tbc>
inline cudaError_t launch_bwd_v(const BwdParams& P, cudaStream_t st) {
  const size_t es = sizeof(Tio);
  const int epp = 16 / (int)es;
  auto ok = [&](const View3D& v) {
    if (!v.p) return true;
    return v.s2 == 1 && (reinterpret_cast<uintptr_t>(v.p) % 16) == 0 && (v.s0 * es) % 16 == 0 &&
           (v.s1 * es) % 16 == 0;
  };
  const bool bc = bc_vec_ok<Tbc>(P.f);
  const bool vec = P.f.E % epp == 0 && ok(P.f.u) && ok(P.f.delta) && ok(P.f.z) && ok(P.dout) && bc;
  return vec ? launch_bwd_n<Tio, Tbc, true>(P, st) : launch_bwd_n<Tio, Tbc, false>(P, st);
}

}  // namespace lbs
