// Fused LB selective scan — forward (sm_100a).
//
// Replaces, in one launch, the reference's numpy discretisation
// (block._discretize_cached, block.py:87-103 — materialises two (B,L,E,N)
// tensors), the numba tiled scan (engine._scan_kernel, engine.py:88-218), the
// D-skip and the SiLU(z) gate (block.py:177-178).  Nothing of size (B,L,E,N)
// ever touches HBM: per (b,l) the kernel reads u, delta, z (E each) and B, C
// (N each) and writes out (E).
//
// Execution model (B200-first, not the reference's 3-phase tile scan):
//  * one thread owns one (b, e) channel and ALL its N states, and sweeps the
//    sequence serially: the forward recurrence costs 1 FFMA per state-step
//    (no in-tile aggregate + rescan as in engine.py:128-154).  The LB window
//    of M steps lives in registers: per tile the thread first runs the
//    tile-local backward recurrence r_i = a_i (r_{i+1} + b_{i+1})
//    (oracle.py:80-112) accumulating C_i·r_i into the outputs, then the
//    forward recurrence h_i = a_i h_{i-1} + b_i accumulating C_i·h_i.
//  * state pairs (n, n+1) use packed FFMA2/FMUL2/FADD2; exp(delta*A) is one
//    MUFU.EX2 per state-step — the kernel is MUFU/issue-bound.
//  * a CTA owns 128 consecutive channels of one batch row.  Chunks of CL steps
//    of u/delta/z are staged into a 2-stage shared-memory ring one chunk ahead
//    of the compute: by TMA (one cp.async.bulk.tensor box per array per chunk
//    from host-encoded 3-D tensor maps, issued by one thread, completing on a
//    per-stage mbarrier, one CTA barrier per chunk) for aligned unsplit fp32
//    launches, else by cp.async (16-byte LDGSTS, coalesced rows); B and C
//    of the chunk (shared by all channels) are prefetched into registers one
//    chunk ahead and published to shared memory as fp32, so the warp reads
//    them as broadcast LDS.64.  Global-memory latency is off the critical path.
//  * reverse direction = flip-on-load: the stager copies physical row
//    L-1-t into ring row t, so the compute loop is direction-agnostic and
//    tiles are aligned from logical 0 (engine.py:133,183).
//  * optional sequence split (long L, few channels): pass 1
//    (segment_state_kernel) computes each segment's affine aggregate
//    h -> P h + H per lane; the main pass enters segment s with the exact
//    state folded from segments < s.  Segment boundaries are tile boundaries.
#pragma once
#include "lbs_common.cuh"
#include "lbs_internal.h"

namespace lbs {

// ---------------------------------------------------------------------------
// cp.async helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// up to this many segments the main pass folds the segment aggregates itself
// (a short sequential fold per thread beats a separate prefix launch)
constexpr int kFoldMax = 32;

// ---------------------------------------------------------------------------
// kernel parameter of the instantiations without TMA staging (no 640-byte maps)
struct NoMaps {
  int unused;
};

// TMA (cp.async.bulk.tensor) staging: one 3-D box copy per array per chunk,
// issued by one thread, completing on the stage's mbarrier
#ifndef LBS_FWD_TMA
#define LBS_FWD_TMA 1
#endif
#ifndef LBS_FWD_TMA_BF16
#define LBS_FWD_TMA_BF16 0  // TMA staging for bf16 I/O as well (measured: see lbs_capi.cu)
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LBS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LBS_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

#ifndef LBS_FWD_CL
#define LBS_FWD_CL 16  // steps per staged chunk (raised to the tile length for long windows)
#endif
#ifndef LBS_FWD_ONEBAR
#define LBS_FWD_ONEBAR 1  // 16-step windows, 16-bit I/O: B/C two chunks ahead, one barrier per chunk
#endif

template <typename Tio, int CLv = LBS_FWD_CL, int CT = kFwdThreads>
struct FwdCfg {
  static constexpr int CL = CLv;                               // max steps per chunk
  static constexpr int PPR = CT * sizeof(Tio) / 16;  // 16-byte pieces per ring row
  static constexpr int EPP = 16 / sizeof(Tio);                // elements per piece
  static constexpr int RS = CT / PPR;                 // ring rows covered per pass
  static constexpr int KP = (CL + RS - 1) / RS;                // pieces per thread per array
};

// Shared-memory layout (dynamic):
//   seq[2 stages][3 arrays][CL][128]  (Tio)   u, delta, z
//   bcf[CL][2*NS]                      (f32)   B then C per step, zero padded
//   a2s[NS/2][128]                     (f2)    A*log2(e) per channel pair
//   bcraw[2 stages][CL][2*NS]           (Tbc)   B|C rows as loaded (cp.async path)
template <typename Tio, typename Tbc, int NS, int CLv = LBS_FWD_CL, int CT = kFwdThreads>
struct FwdSmem {
  static constexpr int CL = CLv;
  static constexpr size_t seq_bytes = 2ull * 3 * CL * CT * sizeof(Tio);
  static constexpr size_t bc_bytes = (size_t)CL * 2 * NS * sizeof(float);
  static constexpr size_t a2_bytes = (size_t)(NS / 2) * CT * sizeof(f2);
  static constexpr size_t raw_bytes = 2ull * CL * 2 * NS * sizeof(Tbc);
  static constexpr size_t hs_bytes = (size_t)(NS / 2) * CT * sizeof(f2);  // state spill area
  static constexpr size_t total = seq_bytes + bc_bytes + a2_bytes + raw_bytes + hs_bytes;
};

// Per-thread staging plan for u/delta/z rows.  With 16-byte pieces each
// thread owns one fixed piece column and rows t = row0 + k*RS, so all index
// math is hoisted out of the chunk loop; "logical step l" addresses
// base + l*step (step < 0 for the reverse direction = flip-on-load).
template <typename Tio, bool kVec, int CLv = LBS_FWD_CL, int CT = kFwdThreads>
struct SeqStager {
  using C = FwdCfg<Tio, CLv, CT>;
  const Tio* base[3];
  long long step[3];
  int narr, row0, col;
  bool ok;
  __device__ __forceinline__ void init(const FwdParams& p, int b, int e0, bool has_z) {
    const bool rev = p.flags & LBS_FLAG_REVERSE;
    narr = has_z ? 3 : 2;
    if constexpr (kVec) {
      row0 = threadIdx.x / C::PPR;
      col = (threadIdx.x % C::PPR) * C::EPP;
    } else {
      row0 = 0;
      col = threadIdx.x;
    }
    ok = e0 + col < p.E;
    const int ec = ok ? e0 + col : 0;
    auto setup = [&](int a, const View3D v) {
      base[a] = v.p ? static_cast<const Tio*>(v.p) + (long long)b * v.s0 + (long long)ec * v.s2 +
                          (rev ? (long long)(p.L - 1) * v.s1 : 0)
                    : nullptr;
      step[a] = rev ? -v.s1 : v.s1;
    };
    setup(0, p.u);
    setup(1, p.delta);
    setup(2, p.z);
  }
  __device__ __forceinline__ void issue(Tio* seq, int stg, int c, int clen) const {
    if (!ok) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= narr) break;
      Tio* dst = seq + ((size_t)(stg * 3 + a) * C::CL) * CT + col;
      if constexpr (kVec) {
#pragma unroll
        for (int k = 0; k < C::KP; ++k) {
          const int t = row0 + k * C::RS;
          if (t < clen) cp_async16(dst + t * CT, base[a] + (long long)(c + t) * step[a]);
        }
      } else {
        for (int t = 0; t < clen; ++t) dst[t * CT] = base[a][(long long)(c + t) * step[a]];
      }
    }
  }
};

// B/C of one chunk: each thread owns one fixed (B|C, n) column and rows
// t = row0 + k*RS; values are prefetched into registers one chunk ahead and
// published to shared memory as fp32 (zero for n >= N).
// forward B/C table layout: [t][pair q][B0 B1 C0 C1] (one LDS.128 per pair-step)
constexpr bool kBcIL = true;
// index of (step t, B|C = w, state n) in the fp32 broadcast table
template <int NS, bool kIL>
__host__ __device__ constexpr int bc_index(int t, int w, int n) {
  return kIL ? t * 2 * NS + (n >> 1) * 4 + w * 2 + (n & 1) : t * 2 * NS + w * NS + n;
}

template <typename Tbc, int NS, int CL, bool kIL = false, int CT = kFwdThreads>
struct BcPrefetch {
  static constexpr int W = 2 * NS;                  // values per step
  static constexpr int RS = CT / W;        // rows per pass
  static constexpr int BCR = (CL + RS - 1) / RS;    // values per thread
  float v[BCR];
  const Tbc* base;
  long long step;
  int row0, kk;
  bool ok;
  __device__ __forceinline__ void init(const FwdParams& p, int b) {
    const bool rev = p.flags & LBS_FLAG_REVERSE;
    kk = threadIdx.x % W;
    row0 = threadIdx.x / W;
    const int which = kk / NS, n = kk % NS;
    ok = n < p.N;
    // select by value (a reference to a runtime-chosen kernel parameter would
    // force a local-memory copy of the whole parameter block)
    const void* vp = which == 0 ? p.Bm.p : p.Cm.p;
    const long long s0 = which == 0 ? p.Bm.s0 : p.Cm.s0;
    const long long s1 = which == 0 ? p.Bm.s1 : p.Cm.s1;
    const long long s2 = which == 0 ? p.Bm.s2 : p.Cm.s2;
    base = static_cast<const Tbc*>(vp) + (long long)b * s0 + (long long)(ok ? n : 0) * s2 +
           (rev ? (long long)(p.L - 1) * s1 : 0);
    step = rev ? -s1 : s1;
  }
  __device__ __forceinline__ void load(int c, int clen) {
#pragma unroll
    for (int k = 0; k < BCR; ++k) {
      const int t = row0 + k * RS;
      v[k] = (ok && t < clen) ? ld<Tbc>(base + (long long)(c + t) * step) : 0.f;
    }
  }
  __device__ __forceinline__ void publish(float* bcf) const {
#pragma unroll
    for (int k = 0; k < BCR; ++k) {
      const int t = row0 + k * RS;
      if (t < CL) bcf[bc_index<NS, kIL>(t, kk / NS, kk % NS)] = v[k];
    }
  }
};

// B/C rows can go through 16-byte cp.async only when a row of NS elements is
// whole 16-byte pieces (not bf16 with NS = 4: 8 bytes per row)
template <typename Tbc, int NS>
__host__ __device__ constexpr bool bc_async_ok() { return (NS * sizeof(Tbc)) % 16 == 0; }

#ifndef LBS_BC_PUBLISH_VEC
#define LBS_BC_PUBLISH_VEC 1
#endif
// B/C staging for one chunk.  kAsync (N == NS, rows of 16-byte pieces): the
// raw rows are copied by cp.async into a 2-stage shared-memory ring together
// with u/delta/z — a global load the compiler cannot sink to its use — and
// converted to the fp32 broadcast table at publish.  Otherwise: BcPrefetch.
template <typename Tbc, int NS, int CL, bool kAsync, bool kIL = false, int CT = kFwdThreads, bool kVecPub = true>
struct BcStage {
  static constexpr int EPB = 16 / sizeof(Tbc);   // elements per 16-byte piece
  static constexpr int PB = NS / EPB;            // pieces per B (or C) row
  static_assert(!kAsync || (PB >= 1 && PB * EPB == NS), "async B/C rows must be whole 16-byte pieces");
  BcPrefetch<Tbc, NS, CL, kIL, CT> pre;
  const Tbc* base[2];
  long long step;
  __device__ __forceinline__ void init(const FwdParams& p, int b) {
    if constexpr (kAsync) {
      const bool rev = p.flags & LBS_FLAG_REVERSE;
      base[0] = static_cast<const Tbc*>(p.Bm.p) + (long long)b * p.Bm.s0 + (rev ? (long long)(p.L - 1) * p.Bm.s1 : 0);
      base[1] = static_cast<const Tbc*>(p.Cm.p) + (long long)b * p.Cm.s0 + (rev ? (long long)(p.L - 1) * p.Cm.s1 : 0);
      step = rev ? -p.Bm.s1 : p.Bm.s1;  // kAsync requires equal B/C row strides
    } else {
      pre.init(p, b);
    }
  }
  __device__ __forceinline__ void issue(Tbc* raw, int stg, int c, int clen) {
    if constexpr (kAsync) {
      static_assert(CL * 2 * PB <= CT || (CL * 2 * PB) % CT == 0, "piece split");
#pragma unroll
      for (int i0 = 0; i0 < CL * 2 * PB; i0 += CT) {
        const int i = i0 + threadIdx.x;
        const int t = i / (2 * PB), r = i % (2 * PB);
        const int w = r / PB, piece = r % PB;
        if (i < CL * 2 * PB && t < clen)
          cp_async16(raw + ((size_t)(stg * CL + t) * 2 * NS + w * NS + piece * EPB),
                     (w ? base[1] : base[0]) + (long long)(c + t) * step + piece * EPB);
      }
    } else {
      pre.load(c, clen);
    }
  }
  __device__ __forceinline__ void publish(float* bcf, const Tbc* raw, int stg, int clen) {
    if constexpr (kAsync && kIL && kVecPub && LBS_BC_PUBLISH_VEC) {
      // one 16-byte piece per (step, B|C, piece): a 16-byte shared load, the state pairs
      // (n, n+1) converted with bit moves and written as the table's 8-byte pair slots
      // (the scalar form was a load -> convert -> store chain per value with a branch,
      // 13 % of the stall samples at configs[3])
      constexpr int UNITS = CL * 2 * PB;
#pragma unroll
      for (int u0 = 0; u0 < UNITS; u0 += CT) {
        const int u = u0 + threadIdx.x;
        if (UNITS % CT == 0 || u < UNITS) {
          const int t = u / (2 * PB), rr = u % (2 * PB);
          const int w = rr / PB, pc = rr % PB;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (t < clen)
            v = *reinterpret_cast<const uint4*>(raw + ((size_t)(stg * CL + t) * 2 * NS + w * NS + pc * EPB));
          float* row = bcf + t * 2 * NS + w * 2;  // pair q at row[q * 4]
          const unsigned wd[4] = {v.x, v.y, v.z, v.w};
          if constexpr (sizeof(Tbc) == 2) {
#pragma unroll
            for (int j = 0; j < 4; ++j)  // word j: states pc*8 + 2j (low half), + 2j + 1 (high half)
              *reinterpret_cast<float2*>(row + (pc * 4 + j) * 4) =
                  make_float2(__uint_as_float(wd[j] << 16), __uint_as_float(wd[j] & 0xffff0000u));
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j)  // states pc*4 + 2j, + 2j + 1
              *reinterpret_cast<float2*>(row + (pc * 2 + j) * 4) =
                  make_float2(__uint_as_float(wd[2 * j]), __uint_as_float(wd[2 * j + 1]));
          }
        }
      }
    } else if constexpr (kAsync) {
#pragma unroll
      for (int i0 = 0; i0 < CL * 2 * NS; i0 += CT) {
        const int i = i0 + threadIdx.x;
        const int t = i / (2 * NS), kk = i % (2 * NS);
        if (i < CL * 2 * NS)  // (CL * 2 * NS may be < the 128 threads, e.g. N = 4 in the backward)
          bcf[bc_index<NS, kIL>(t, kk / NS, kk % NS)] = t < clen ? to_f(raw[(size_t)stg * CL * 2 * NS + i]) : 0.f;
      }
    } else {
      pre.publish(bcf);
    }
  }
};

// One LB tile of r steps at ring rows [t0, t0+r): all state pairs, then the
// D-skip + gate + store.  For MT > 8 the injections b_j are recomputed in the
// forward sweep instead of held (keeps the 16-step window under 168 regs).
struct TileOut {
  void* op;        // address of logical step 0 for this channel
  long long step;  // signed element stride per logical step
  int c;
  bool active, has_z;
  float Dv;
  bool accum;      // out += y (LBS_FLAG_ACCUM)
};

#ifndef LBS_RAGGED_QU
#define LBS_RAGGED_QU 2  // state pairs per unrolled group in the LB ragged-tile path (-2..4 % vs 1)
#endif
#ifndef LBS_QUNROLL16
#define LBS_QUNROLL16 2  // the same for 16-step tiles
#endif
#ifndef LBS_QUNROLL
#define LBS_QUNROLL 2  // state pairs per unrolled group in a full tile; 0 = all (state in registers)
#endif

// One state pair (n, n+1) through one tile: exps, tile-local record, forward
// recurrence, accumulation of C (h + r) into the per-step outputs.
template <int NS, int MT, bool kLB, bool kFull, bool kIL = kBcIL>
__device__ __forceinline__ void pair_tile(f2& hq, const f2 A2, int q, const float (&dl)[MT], const float (&du)[MT],
                                          f2 (&yacc)[MT], const float* bcf, int t0, int r, bool linear) {
  constexpr bool kHoldB = MT <= 8;
  constexpr bool kHoldC = kIL && kHoldB;  // interleaved table: one LDS.128 per pair-step, C held
  f2 a[MT], bb[kHoldB ? MT : 1], cc[kHoldC ? MT : 1];
#pragma unroll
  for (int j = 0; j < MT; ++j) {
    const f2 x = mul2(bc2(dl[j]), A2);
    a[j] = linear ? x : mk2(ex2(x.x), ex2(x.y));
    if constexpr (kHoldC) {
      const float4 v = *reinterpret_cast<const float4*>(&bcf[bc_index<NS, true>(t0 + j, 0, 2 * q)]);
      bb[j] = mul2(bc2(du[j]), mk2(v.x, v.y));
      cc[j] = mk2(v.z, v.w);
    } else if constexpr (kHoldB) {
      const f2 Bv = *reinterpret_cast<const f2*>(&bcf[bc_index<NS, kIL>(t0 + j, 0, 2 * q)]);
      bb[j] = mul2(bc2(du[j]), Bv);
    }
  }
  auto binj = [&](int j) -> f2 {
    if constexpr (kHoldB) {
      return bb[j];
    } else {
      const f2 Bv = *reinterpret_cast<const f2*>(&bcf[bc_index<NS, kIL>(t0 + j, 0, 2 * q)]);
      return mul2(bc2(du[j]), Bv);
    }
  };
  auto cinj = [&](int j) -> f2 {
    if constexpr (kHoldC) {
      return cc[j];
    } else {
      return *reinterpret_cast<const f2*>(&bcf[bc_index<NS, kIL>(t0 + j, 1, 2 * q)]);
    }
  };
  if (kLB) {
    // exclusive tile-local backward record: r_{end} = 0, r_i = a_i (r_{i+1} + b_{i+1})
    f2 s = mk2(0.f, 0.f);
#pragma unroll
    for (int j = MT - 1; j >= 0; --j) {
      if (kFull) {
        if (j == MT - 1) {
          s = binj(j);
        } else {
          const f2 rr = mul2(a[j], s);
          yacc[j] = fma2(cinj(j), rr, yacc[j]);
          s = add2(rr, binj(j));
        }
      } else if (j < r) {
        // ragged tile: selects on the (runtime) tile end instead of a branch
        // chain, which the compiler turns into a local-memory lookup b[r-1]
        const bool end = j == r - 1;
        const f2 rr = mul2(a[j], s);
        if (!end) yacc[j] = fma2(cinj(j), rr, yacc[j]);
        const f2 bj = binj(j);
        const f2 sn = add2(rr, bj);
        s = end ? bj : sn;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MT; ++j) {
    if (kFull || j < r) {
      hq = fma2(a[j], hq, binj(j));
      yacc[j] = fma2(cinj(j), hq, yacc[j]);
    }
  }
}

// Fixed-size state store of a thread: registers (QU == NP: every loop over q is
// unrolled) or this thread's column of a shared-memory array [NP][128] (QU < NP:
// the pair loop stays rolled, which keeps the kernel's code in the I-cache).
template <int NP, bool kRegs, int CT = kFwdThreads>
struct StateStore {
  f2 r[kRegs ? NP : 1];
  f2* s;
  __device__ __forceinline__ f2 get(int q) const { return kRegs ? r[kRegs ? q : 0] : s[q * CT + threadIdx.x]; }
  __device__ __forceinline__ void set(int q, f2 v) {
    if constexpr (kRegs) r[q] = v;
    else s[q * CT + threadIdx.x] = v;
  }
};

// kFull: a whole tile (r == MT) through the MT-step unrolled code; else a
// ragged tile (once per segment).  Measured: an extra unrolled instantiation
// for ragged tiles (masked steps) costs 4-10 % on every config even where it
// never runs, and so does a runtime step count inside the full-tile code
// (ragged tiles padded with delta = -inf) -- r must stay a compile-time MT here.
template <typename Tio, int NS, int MT, bool kLB, bool kFull, int QU, bool kRegs, bool kAccum = false,
          int CT = kFwdThreads>
__device__ __forceinline__ void tile_compute(const Tio* su, const Tio* sd, const Tio* sz,
                                             const float* bcf, const f2* a2s, StateStore<NS / 2, kRegs, CT>& h,
                                             int t0, int r_, float bias, bool softplus, bool linear,
                                             const TileOut& o, int rs = CT) {
  // rs: elements between the ring rows of consecutive logical steps (-CT when a
  // TMA-staged chunk of the reverse direction holds its rows in physical order)
  constexpr int NP = NS / 2;
  const int r = kFull ? MT : r_;
  const int tid = threadIdx.x;
  float dl[MT], du[MT];
  f2 yacc[MT];
  // LBS_FLAG_ACCUM: the previous outputs of this tile are loaded before the
  // pair loop so the read latency hides under the tile's compute
  float prev[kAccum ? MT : 1];
  if (kAccum && o.active) {
    const Tio* opp = static_cast<const Tio*>(o.op);
#pragma unroll
    for (int j = 0; j < MT; ++j) prev[j] = (j < r) ? to_f(opp[(long long)(o.c + t0 + j) * o.step]) : 0.f;
  }
  float uv[MT];
#pragma unroll
  for (int j = 0; j < MT; ++j) {
    const bool on = kFull || j < r;
    dl[j] = on ? to_f(sd[(t0 + j) * rs + tid]) + bias : 0.f;
    uv[j] = on ? to_f(su[(t0 + j) * rs + tid]) : 0.f;
  }
  // one uniform branch per tile: the MT softplus chains (EX2 -> LG2) are
  // independent and interleave
  if (softplus) {
#pragma unroll
    for (int j = 0; j < MT; ++j) dl[j] = softplus_f(dl[j]);
  }
#pragma unroll
  for (int j = 0; j < MT; ++j) {
    du[j] = dl[j] * uv[j];
    yacc[j] = mk2(o.Dv * uv[j], 0.f);  // D-skip folded into the accumulator
  }
  if constexpr (kRegs) {
#pragma unroll
    for (int q = 0; q < NP; ++q)
      pair_tile<NS, MT, kLB, kFull>(h.r[q], a2s[q * CT + tid], q, dl, du, yacc, bcf, t0, r, linear);
  } else {
#pragma unroll 1
    for (int q0 = 0; q0 < NP; q0 += QU) {
#pragma unroll
      for (int qq = 0; qq < QU; ++qq) {
        const int q = q0 + qq;
        f2 hq = h.get(q);
        pair_tile<NS, MT, kLB, kFull>(hq, a2s[q * CT + tid], q, dl, du, yacc, bcf, t0, r, linear);
        h.set(q, hq);
      }
    }
  }
  if (o.active) {
    Tio* dst = static_cast<Tio*>(o.op) + (long long)(o.c + t0) * o.step;
#pragma unroll
    for (int j = 0; j < MT; ++j) {
      if (j < r) {
        float y = yacc[j].x + yacc[j].y;
        if (o.has_z) y *= silu_out<Tio>(to_f(sz[(t0 + j) * rs + tid]));
        if constexpr (kAccum) y += prev[j];
        st<Tio>(dst, y);
      }
      dst += o.step;
    }
  }
}

// chunk length of the main kernel: LBS_FWD_CL, but at least one whole tile
#ifndef LBS_FWD_CL16
#define LBS_FWD_CL16 32  // 16-step windows with 16-bit I/O: steps per staged chunk
#endif
constexpr int fwd_chunk(int mt, int io_bytes = 4) {
  return (mt > 8 && io_bytes == 2) ? LBS_FWD_CL16 : (mt > LBS_FWD_CL ? mt : LBS_FWD_CL);
}

#ifndef LBS_FWD_MINB
#define LBS_FWD_MINB 4
#endif
#ifndef LBS_FWD_MINB16
#define LBS_FWD_MINB16 2
#endif

template <typename Tio, typename Tbc, int NS, int MT, bool kLB, bool kVec, bool kAccum = false, int CT = kFwdThreads,
          bool kTma = false>
__global__ void __launch_bounds__(CT, (MT <= 8 ? LBS_FWD_MINB : LBS_FWD_MINB16) * (kFwdThreads / CT))
    fwd_kernel(FwdParams p, const __grid_constant__ std::conditional_t<kTma, FwdTmaMaps, NoMaps> tmaps) {
  constexpr int NP = NS / 2;
  constexpr int CL = fwd_chunk(MT, sizeof(Tio));
  using Sm = FwdSmem<Tio, Tbc, NS, CL, CT>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tio* seq = reinterpret_cast<Tio*>(smem_raw);
  float* bcf = reinterpret_cast<float*>(smem_raw + Sm::seq_bytes);
  f2* a2s = reinterpret_cast<f2*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes);
  Tbc* bcraw = reinterpret_cast<Tbc*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes + Sm::a2_bytes);
  f2* hsm = reinterpret_cast<f2*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes + Sm::a2_bytes + Sm::raw_bytes);
  constexpr int QU = MT > 8 ? LBS_QUNROLL16 : (LBS_QUNROLL == 0 ? NP : LBS_QUNROLL);
  constexpr bool kRegs = QU >= NP;

  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * CT;
  const int e = e0 + tid;
  const int b = blockIdx.y;
  const int seg = blockIdx.z;
  const bool active = e < p.E;
  const int ec = active ? e : p.E - 1;
  const int L = p.L, N = p.N, m = p.m;
  const bool rev = p.flags & LBS_FLAG_REVERSE;
  const bool softplus = p.flags & LBS_FLAG_SOFTPLUS;
  const bool linear = p.flags & LBS_FLAG_LINEAR;
  const bool has_z = p.z.p != nullptr;
  const int CLm = (CL / m) * m;  // steps per chunk: whole tiles
  const int seg_lo = seg * p.seg_len;
  const int seg_hi = min(L, seg_lo + p.seg_len);

#pragma unroll
  for (int q = 0; q < NP; ++q) {
    float a0 = 2 * q < N ? p.A[(long long)ec * N + 2 * q] : 0.f;
    float a1 = 2 * q + 1 < N ? p.A[(long long)ec * N + 2 * q + 1] : 0.f;
    if (!linear) { a0 *= kLog2e; a1 *= kLog2e; }
    a2s[q * CT + tid] = mk2(a0, a1);
  }
  const float Dv = p.D ? p.D[ec] : 0.f;
  const float bias = p.bias ? p.bias[ec] : 0.f;

  StateStore<NP, kRegs, CT> h;
  h.s = hsm;
#pragma unroll
  for (int q = 0; q < NP; ++q) h.set(q, mk2(0.f, 0.f));
  if (seg > 0) {
    const f2* agg = reinterpret_cast<const f2*>(p.seg_agg) + ((long long)b * p.n_seg * p.E + ec) * NS;
    const long long sstride = (long long)p.E * NS;  // f2 per segment
    if (p.n_seg <= kFoldMax) {
      // few segments: fold the raw aggregates h -> P h + H of segments 0..seg-1
      // here (core.py:48-55 combine, left to right), no prefix kernel
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        f2 hq = mk2(0.f, 0.f);
#pragma unroll 8
        for (int s = 0; s < seg; ++s) hq = fma2(agg[s * sstride + q], hq, agg[s * sstride + NP + q]);
        h.set(q, hq);
      }
    } else {
      // state entering this segment, folded by segment_prefix_kernel
#pragma unroll
      for (int q = 0; q < NP; ++q) h.set(q, agg[(seg - 1) * sstride + NP + q]);
    }
  }

  // p.out == nullptr: checkpoint-only sweep (the backward's recompute pass)
  Tio* op = p.out == nullptr ? nullptr
                             : static_cast<Tio*>(p.out) + (long long)b * p.so0 + (long long)ec * p.so2 +
                                   (rev ? (long long)(L - 1) * p.so1 : 0);
  const long long ostep = rev ? -p.so1 : p.so1;

  // TMA staging (aligned views, host-encoded tensor maps): thread 0 issues one box
  // copy per array per chunk; an mbarrier per ring stage; the B/C fp32 table is
  // double-buffered so ONE CTA barrier per chunk suffices.  Else cp.async rows.
  static_assert(!kTma || (kVec && bc_async_ok<Tbc, NS>()), "TMA staging needs aligned rows of whole pieces");
  SeqStager<Tio, kVec, CL, CT> stager;
  BcStage<Tbc, NS, CL, kVec && bc_async_ok<Tbc, NS>(), kBcIL, CT> bcs;
  __shared__ __align__(8) uint64_t bars[2];
  float* bcf2 = reinterpret_cast<float*>(smem_raw + Sm::total);  // second B/C table (TMA; kOneBar)
  // kOneBar (16-step windows, 16-bit I/O, cp.async): the B/C rows of chunk k+1 are staged
  // two chunks ahead (3-stage raw ring) and converted into the other half of a
  // double-buffered table while chunk k computes, so a chunk needs ONE CTA barrier (the
  // table of chunk k was built before it); the third raw stage follows the second table.
  // Measured: configs[3] LB scan -2.6 %, bitwise equal; the forward-only scan (+1.5 %) and
  // 8-step windows (LBVim-Ti, +1 %) keep two barriers (profiles/r02_fwd_experiments.txt)
  constexpr bool kOneBar =
      LBS_FWD_ONEBAR && kLB && MT > 8 && sizeof(Tio) == 2 && kVec && bc_async_ok<Tbc, NS>() && !kTma;
  Tbc* raw3 = reinterpret_cast<Tbc*>(smem_raw + Sm::total + Sm::bc_bytes);
  auto raw_stage = [&](int s3) -> Tbc* { return s3 < 2 ? bcraw + (size_t)s3 * CL * 2 * NS : raw3; };
  auto table = [&](int s2) -> float* { return s2 ? bcf2 : bcf; };
  Tbc* rawB = bcraw;                                              // TMA: [2][CL][NS] B rows
  Tbc* rawC = bcraw + 2 * CL * NS;                                //      [2][CL][NS] C rows
  const int narr = has_z ? 3 : 2;
  const unsigned tma_bytes = (unsigned)(narr * CL * CT * sizeof(Tio) + 2 * CL * NS * sizeof(Tbc));
  auto tma_issue = [&](int stg, int cc, int len) {
    if constexpr (kTma) {
    // logical steps [cc, cc + len): physical rows [cc, ...) forward, [L - cc - len, ...) reverse
    const int l0 = rev ? L - cc - len : cc;
    mbar_expect_tx(&bars[stg], tma_bytes);
    for (int a = 0; a < narr; ++a)
      tma_load_3d(seq + ((size_t)stg * 3 + a) * CL * CT, &tmaps.tm[a], e0, l0, b, &bars[stg]);
    tma_load_3d(rawB + (size_t)stg * CL * NS, &tmaps.tm[3], 0, l0, b, &bars[stg]);
    tma_load_3d(rawC + (size_t)stg * CL * NS, &tmaps.tm[4], 0, l0, b, &bars[stg]);
    }
  };
  // prologue: chunk 0
  int c = seg_lo;
  int clen = min(CLm, seg_hi - c);
  if constexpr (kTma) {
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_fence_init();
      tma_issue(0, c, clen);
    }
    __syncthreads();
  } else if constexpr (kOneBar) {
    stager.init(p, b, e0, has_z);
    bcs.init(p, b);
    stager.issue(seq, 0, c, clen);
    bcs.issue(raw_stage(0), 0, c, clen);
    const int c1 = c + clen;
    if (c1 < seg_hi) bcs.issue(raw_stage(1), 0, c1, min(CLm, seg_hi - c1));
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    bcs.publish(table(0), raw_stage(0), 0, clen);  // visible after iteration 0's barrier
  } else {
    stager.init(p, b, e0, has_z);
    bcs.init(p, b);
    stager.issue(seq, 0, c, clen);
    bcs.issue(bcraw, 0, c, clen);
    cp_async_commit();
  }

  for (int k = 0; c < seg_hi; ++k) {
    const int stg = k & 1;
    const int cn = c + clen;
    const int clen_n = cn < seg_hi ? min(CLm, seg_hi - cn) : 0;
    const float* bcfk = bcf;
    int rs = CT, rb = 0;  // ring row of logical step t = rb + t * rs / CT
    if constexpr (kTma) {
      mbar_wait(&bars[stg], (k >> 1) & 1);
      float* bt = stg ? bcf2 : bcf;
      if (rev) { rs = -CT; rb = clen - 1; }
      // B/C rows -> fp32 broadcast table in logical order: one 16-byte piece per
      // (step, B|C, piece), pairs written as the table's 8-byte slots (as BcStage::publish)
      {
        constexpr int EPB = 16 / sizeof(Tbc), PB = NS / EPB;
        for (int u = tid; u < CL * 2 * PB; u += CT) {
          const int t = u / (2 * PB), rr = u % (2 * PB);
          const int w = rr / PB, pc = rr % PB;
          const int row = rev ? clen - 1 - t : t;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (t < clen)
            v = *reinterpret_cast<const uint4*>((w ? rawC : rawB) + ((size_t)stg * CL + row) * NS + pc * EPB);
          float* trow = bt + t * 2 * NS + w * 2;
          const unsigned wd[4] = {v.x, v.y, v.z, v.w};
          if constexpr (sizeof(Tbc) == 2) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<float2*>(trow + (pc * 4 + j) * 4) =
                  make_float2(__uint_as_float(wd[j] << 16), __uint_as_float(wd[j] & 0xffff0000u));
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              *reinterpret_cast<float2*>(trow + (pc * 2 + j) * 4) =
                  make_float2(__uint_as_float(wd[2 * j]), __uint_as_float(wd[2 * j + 1]));
          }
        }
      }
      bcfk = bt;
      __syncthreads();  // table visible; chunk k-1 done with ring stage stg ^ 1
      if (tid == 0 && clen_n > 0) tma_issue(stg ^ 1, cn, clen_n);
    } else if constexpr (kOneBar) {
      cp_async_wait_all();
      __syncthreads();  // seq rows of chunk k, B/C rows of chunk k+1 landed; table k visible;
                        // compute of chunk k-1 done (its seq stage and table half are free)
      bcfk = table(stg);
      if (clen_n > 0) {
        bcs.publish(table(stg ^ 1), raw_stage((k + 1) % 3), 0, clen_n);
        stager.issue(seq, stg ^ 1, cn, clen_n);
        const int c2 = cn + clen_n;
        if (c2 < seg_hi) bcs.issue(raw_stage((k + 2) % 3), 0, c2, min(CLm, seg_hi - c2));
      }
      cp_async_commit();
    } else {
      cp_async_wait_all();
      __syncthreads();  // chunk k landed (all threads); compute of chunk k-1 done
      bcs.publish(bcf, bcraw, stg, clen);
      if (clen_n > 0) {
        stager.issue(seq, stg ^ 1, cn, clen_n);
        bcs.issue(bcraw, stg ^ 1, cn, clen_n);
      }
      cp_async_commit();
      __syncthreads();  // bcf visible
    }

    const Tio* su = seq + ((size_t)stg * 3 + 0) * CL * CT + rb * CT;
    const Tio* sd = seq + ((size_t)stg * 3 + 1) * CL * CT + rb * CT;
    const Tio* sz = seq + ((size_t)stg * 3 + 2) * CL * CT + rb * CT;
    const TileOut o{op, ostep, c, active && p.out != nullptr, has_z, Dv, (p.flags & LBS_FLAG_ACCUM) != 0};
    for (int t0 = 0; t0 < clen; t0 += m) {
      const int r = min(m, clen - t0);
      if (p.ckpt != nullptr && active && (c + t0) % p.ckpt_len == 0) {
        // training checkpoint: state entering backward chunk (c+t0)/ckpt_len,
        // layout [b][chunk][pair q][e] (f2) — coalesced across the warp
        f2* ck = reinterpret_cast<f2*>(p.ckpt) +
                 (((long long)b * p.n_ckpt + (c + t0) / p.ckpt_len) * NP) * p.E + e;
#pragma unroll
        for (int q = 0; q < NP; ++q) ck[(long long)q * p.E] = h.get(q);
      }
      if (r == MT)
        tile_compute<Tio, NS, MT, kLB, true, QU, kRegs, kAccum, CT>(su, sd, sz, bcfk, a2s, h, t0, r, bias, softplus, linear, o, rs);
      else {
        // ragged tile (at most once per segment): rolled pair loop on the smem state
        StateStore<NP, false, CT> hp;
        hp.s = hsm;
        if constexpr (kRegs) {
#pragma unroll
          for (int q = 0; q < NP; ++q) hp.set(q, h.get(q));
        }
        tile_compute<Tio, NS, MT, kLB, false, (kLB ? LBS_RAGGED_QU : 1), false, kAccum, CT>(su, sd, sz, bcfk, a2s, hp, t0, r, bias, softplus, linear, o, rs);
        if constexpr (kRegs) {
#pragma unroll
          for (int q = 0; q < NP; ++q) h.set(q, hp.get(q));
        }
      }
    }
    c = cn;
    clen = clen_n;
  }

  if (active && p.last_state && seg_hi == L) {
    float* hs = p.last_state + ((long long)b * p.E + e) * N;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const f2 hv = h.get(q);
      if (2 * q < N) hs[2 * q] = hv.x;
      if (2 * q + 1 < N) hs[2 * q + 1] = hv.y;
    }
  }
}

// Pass 1 of the sequence split: per (b, segment, e, n) the segment's
// aggregate affine map h -> P*h + H with P = prod a = exp(A * sum delta) and
// H the local end state from zero (core.py:48-55 combine, applied serially).
template <typename Tio, typename Tbc, int NS, bool kVec, int CT = kFwdThreads>
__global__ void __launch_bounds__(CT) segment_state_kernel(FwdParams p) {
  constexpr int NP = NS / 2;
  constexpr int CL = LBS_FWD_CL;
  using Sm = FwdSmem<Tio, Tbc, NS, CL, CT>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tio* seq = reinterpret_cast<Tio*>(smem_raw);
  float* bcf = reinterpret_cast<float*>(smem_raw + Sm::seq_bytes);
  f2* a2s = reinterpret_cast<f2*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes);
  Tbc* bcraw = reinterpret_cast<Tbc*>(smem_raw + Sm::seq_bytes + Sm::bc_bytes + Sm::a2_bytes);

  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * CT;
  const int e = e0 + tid;
  const int b = blockIdx.y;
  const int seg = blockIdx.z;
  const bool active = e < p.E;
  const int ec = active ? e : p.E - 1;
  const int L = p.L, N = p.N;
  const bool softplus = p.flags & LBS_FLAG_SOFTPLUS;
  const bool linear = p.flags & LBS_FLAG_LINEAR;
  const int seg_lo = seg * p.seg_len;
  const int seg_hi = min(L, seg_lo + p.seg_len);
  (void)L;

#pragma unroll
  for (int q = 0; q < NP; ++q) {
    float a0 = 2 * q < N ? p.A[(long long)ec * N + 2 * q] : 0.f;
    float a1 = 2 * q + 1 < N ? p.A[(long long)ec * N + 2 * q + 1] : 0.f;
    if (!linear) { a0 *= kLog2e; a1 *= kLog2e; }
    a2s[q * CT + tid] = mk2(a0, a1);
  }
  const float bias = p.bias ? p.bias[ec] : 0.f;
  f2 H[NP], P[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) { H[q] = mk2(0.f, 0.f); P[q] = mk2(1.f, 1.f); }
  float dsum = 0.f;

  SeqStager<Tio, kVec, LBS_FWD_CL, CT> stager;
  stager.init(p, b, e0, false);
  BcStage<Tbc, NS, CL, kVec && bc_async_ok<Tbc, NS>(), kBcIL, CT> bcs;
  bcs.init(p, b);
  int c = seg_lo;
  int clen = min(CL, seg_hi - c);
  stager.issue(seq, 0, c, clen);
  bcs.issue(bcraw, 0, c, clen);
  cp_async_commit();
  for (int k = 0; c < seg_hi; ++k) {
    const int stg = k & 1;
    const int cn = c + clen;
    const int clen_n = cn < seg_hi ? min(CL, seg_hi - cn) : 0;
    cp_async_wait_all();
    __syncthreads();
    bcs.publish(bcf, bcraw, stg, clen);
    if (clen_n > 0) {
      stager.issue(seq, stg ^ 1, cn, clen_n);
      bcs.issue(bcraw, stg ^ 1, cn, clen_n);
    }
    cp_async_commit();
    __syncthreads();
    const Tio* su = seq + ((size_t)stg * 3 + 0) * CL * CT;
    const Tio* sd = seq + ((size_t)stg * 3 + 1) * CL * CT;
    for (int t = 0; t < clen; ++t) {
      float dl = to_f(sd[t * CT + tid]) + bias;
      if (softplus) dl = softplus_f(dl);
      const float du = dl * to_f(su[t * CT + tid]);
      dsum += dl;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const f2 x = mul2(bc2(dl), a2s[q * CT + tid]);
        const f2 a = linear ? x : mk2(ex2(x.x), ex2(x.y));
        const f2 Bv = *reinterpret_cast<const f2*>(&bcf[bc_index<NS, kBcIL>(t, 0, 2 * q)]);
        H[q] = fma2(a, H[q], mul2(bc2(du), Bv));
        if (linear) P[q] = mul2(P[q], a);
      }
    }
    c = cn;
    clen = clen_n;
  }
  if (!linear) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const f2 x = mul2(bc2(dsum), a2s[q * CT + tid]);
      P[q] = mk2(ex2(x.x), ex2(x.y));
    }
  }
  if (active) {
    f2* out = reinterpret_cast<f2*>(p.seg_agg + ((((long long)b * p.n_seg + seg) * p.E + e) * (2 * NS)));
#pragma unroll
    for (int q = 0; q < NP; ++q) { out[q] = P[q]; out[NP + q] = H[q]; }
  }
}

// ---------------------------------------------------------------------------
// Pass 2 of the sequence split: for every lane (b, e, state pair) the states
// entering segments 1..S-1, h_{s+1} = P_s h_s + H_s with h_0 = 0, written into
// the H slot of segment s.  One warp per lane, a parallel scan of the affine
// maps (P, H) (core.py:48-55 combine): each thread composes up to 16
// consecutive segment maps (loads all in flight), the warp scans the 32
// composed maps with shuffles, then each thread replays its segments from the
// scanned carry-in and stores the entering states.  Rounds of 512 segments
// carry the state across.
template <int NS>
__global__ void __launch_bounds__(128) segment_prefix_kernel(FwdParams p) {
  constexpr int NP = NS / 2;
  constexpr int K = 16;  // segments per thread per round
  const long long wid = ((long long)blockIdx.x * 128 + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const long long total = (long long)p.Bt * p.E * NP;
  if (wid >= total) return;
  const int q = (int)(wid % NP);
  const int e = (int)((wid / NP) % p.E);
  const int b = (int)(wid / ((long long)NP * p.E));
  f2* base = reinterpret_cast<f2*>(p.seg_agg) + (((long long)b * p.n_seg) * p.E + e) * NS;
  const long long sstride = (long long)p.E * NS;  // f2 units per segment
  const int nmaps = p.n_seg - 1;                  // aggregates of segments 0..S-2
  f2 carry = mk2(0.f, 0.f);
  for (int r0 = 0; r0 < nmaps; r0 += 32 * K) {
    const int s0 = r0 + lane * K;
    f2 P[K], H[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (s0 + k < nmaps) {
        P[k] = base[(s0 + k) * sstride + q];
        H[k] = base[(s0 + k) * sstride + NP + q];
      } else {
        P[k] = mk2(1.f, 1.f);
        H[k] = mk2(0.f, 0.f);
      }
    }
    // compose this thread's maps: x -> Pc x + Hc
    f2 Pc = mk2(1.f, 1.f), Hc = mk2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      Hc = fma2(P[k], Hc, H[k]);
      Pc = mul2(P[k], Pc);
    }
    // inclusive warp scan of the composed maps (earlier lanes applied first)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float px = __shfl_up_sync(0xffffffffu, Pc.x, o), py = __shfl_up_sync(0xffffffffu, Pc.y, o);
      const float hx = __shfl_up_sync(0xffffffffu, Hc.x, o), hy = __shfl_up_sync(0xffffffffu, Hc.y, o);
      if (lane >= o) {
        Hc = fma2(Pc, mk2(hx, hy), Hc);
        Pc = mul2(Pc, mk2(px, py));
      }
    }
    // exclusive prefix applied to the round's carry-in = state entering segment s0
    float epx = __shfl_up_sync(0xffffffffu, Pc.x, 1), epy = __shfl_up_sync(0xffffffffu, Pc.y, 1);
    float ehx = __shfl_up_sync(0xffffffffu, Hc.x, 1), ehy = __shfl_up_sync(0xffffffffu, Hc.y, 1);
    if (lane == 0) { epx = epy = 1.f; ehx = ehy = 0.f; }
    f2 h = fma2(mk2(epx, epy), carry, mk2(ehx, ehy));
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (s0 + k < nmaps) {
        h = fma2(P[k], h, H[k]);
        base[(s0 + k) * sstride + NP + q] = h;  // state entering segment s0 + k + 1
      }
    }
    // carry = state after the round's last map (inclusive scan of lane 31 applied to carry)
    const f2 last = fma2(Pc, carry, Hc);
    carry = mk2(__shfl_sync(0xffffffffu, last.x, 31), __shfl_sync(0xffffffffu, last.y, 31));
  }
}

// launcher

template <typename Tio, typename Tbc, int NS, int MT, bool kVec, int CT>
inline cudaError_t launch_fwd_t(const FwdParams& p, cudaStream_t st) {
  using SmT = FwdSmem<Tio, Tbc, NS, fwd_chunk(MT, sizeof(Tio)), CT>;
  // TMA-staged instantiations exist for fp32 I/O only (the launch policy, lbs_capi.cu)
  constexpr bool kTmaOk = LBS_FWD_TMA && kVec && bc_async_ok<Tbc, NS>() && (sizeof(Tio) == 4 || LBS_FWD_TMA_BF16);
  // + the second B/C table and the third raw B/C stage for the one-barrier (16-bit, aligned) kernels
  constexpr bool kOneBarL = LBS_FWD_ONEBAR && MT > 8 && sizeof(Tio) == 2 && kVec && bc_async_ok<Tbc, NS>();
  const size_t smem = SmT::total + (kOneBarL ? SmT::bc_bytes + (size_t)fwd_chunk(MT, sizeof(Tio)) * 2 * NS * sizeof(Tbc) : 0);
  FwdParams pk = p;
  if (!kTmaOk) pk.tma_maps = nullptr;
  dim3 block(CT);
  if (p.n_seg > 1) {
    const size_t smem1 = FwdSmem<Tio, Tbc, NS, LBS_FWD_CL, CT>::total;
    auto k1 = segment_state_kernel<Tio, Tbc, NS, kVec, CT>;
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    dim3 g1((p.E + CT - 1) / CT, p.Bt, p.n_seg - 1);
    k1<<<g1, block, smem1, st>>>(p);
    if (p.n_seg > kFoldMax) {
      const long long lanes = (long long)p.Bt * p.E * (NS / 2);  // one warp each
      segment_prefix_kernel<NS><<<(unsigned)((lanes * 32 + 127) / 128), 128, 0, st>>>(p);
    }
  }
  dim3 grid((p.E + CT - 1) / CT, p.Bt, p.n_seg);
  // LBS_FLAG_ACCUM is instantiated for the forward-only scan (the global-bidir
  // baseline's second sweep); the C ABI rejects ACCUM together with LB
  if constexpr (kTmaOk) {
    if (pk.tma_maps) {
      auto k = (p.flags & LBS_FLAG_LB)      ? fwd_kernel<Tio, Tbc, NS, MT, true, kVec, false, CT, true>
               : (p.flags & LBS_FLAG_ACCUM) ? fwd_kernel<Tio, Tbc, NS, MT, false, kVec, true, CT, true>
                                            : fwd_kernel<Tio, Tbc, NS, MT, false, kVec, false, CT, true>;
      const size_t smem_tma = smem + SmT::bc_bytes;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tma);
      k<<<grid, block, smem_tma, st>>>(pk, *pk.tma_maps);
      return cudaGetLastError();
    }
  }
  auto k = (p.flags & LBS_FLAG_LB)      ? fwd_kernel<Tio, Tbc, NS, MT, true, kVec, false, CT>
           : (p.flags & LBS_FLAG_ACCUM) ? fwd_kernel<Tio, Tbc, NS, MT, false, kVec, true, CT>
                                        : fwd_kernel<Tio, Tbc, NS, MT, false, kVec, false, CT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, block, smem, st>>>(pk, NoMaps{0});
  return cudaGetLastError();
}

// CTA width: 128 channels, or 64 when channels are scarce (p.cta == 64: no idle
// threads for E <= 64, finer load balance and twice the resident segments)
template <typename Tio, typename Tbc, int NS, int MT, bool kVec>
inline cudaError_t launch_fwd_c(const FwdParams& p, cudaStream_t st) {
  if (p.cta == 64) return launch_fwd_t<Tio, Tbc, NS, MT, kVec, 64>(p, st);
  return launch_fwd_t<Tio, Tbc, NS, MT, kVec, kFwdThreads>(p, st);
}

template <typename Tio, typename Tbc, int NS, bool kVec>
inline cudaError_t launch_fwd_m(const FwdParams& p, cudaStream_t st) {
  if (p.m <= 1) return launch_fwd_c<Tio, Tbc, NS, 1, kVec>(p, st);
  if (p.m <= 4) return launch_fwd_c<Tio, Tbc, NS, 4, kVec>(p, st);
  if (p.m <= 8) return launch_fwd_c<Tio, Tbc, NS, 8, kVec>(p, st);
  return launch_fwd_c<Tio, Tbc, NS, 16, kVec>(p, st);
}

template <typename Tio, typename Tbc, bool kVec>
inline cudaError_t launch_fwd_n(const FwdParams& p, cudaStream_t st) {
  if (p.N <= 4) return launch_fwd_m<Tio, Tbc, 4, kVec>(p, st);
  return launch_fwd_m<Tio, Tbc, 16, kVec>(p, st);
}

// 16-byte cp.async staging needs 16-byte aligned rows of whole pieces
// (and B/C rows of N elements as whole 16-byte pieces with equal row strides)
inline bool view_vec_ok(const View3D& v, size_t es) {
  if (!v.p) return true;
  return v.s2 == 1 && (reinterpret_cast<uintptr_t>(v.p) % 16) == 0 && (v.s0 * es) % 16 == 0 &&
         (v.s1 * es) % 16 == 0;
}

// kVec also selects cp.async B/C staging when bc_async_ok<Tbc, NS>(); the B/C
// rows must then be N == NS aligned pieces with equal row strides (else the
// register-prefetch B/C path, which takes any layout, runs with kVec rows)
template <typename Tbc>
inline bool bc_vec_ok(const FwdParams& p) {
  const size_t eb = sizeof(Tbc);
  const int NS = p.N <= 4 ? 4 : 16;
  const bool async = NS == 4 ? bc_async_ok<Tbc, 4>() : bc_async_ok<Tbc, 16>();
  if (!async) return true;
  return p.N == NS && view_vec_ok(p.Bm, eb) && view_vec_ok(p.Cm, eb) && p.Bm.s1 == p.Cm.s1;
}

template <typename Tio, typename Tbc>
static bool vec_ok(const FwdParams& p) {
  const size_t es = sizeof(Tio);
  const int epp = 16 / (int)es;
  return p.E % epp == 0 && view_vec_ok(p.u, es) && view_vec_ok(p.delta, es) && view_vec_ok(p.z, es) &&
         bc_vec_ok<Tbc>(p);
}

template <typename Tio, typename Tbc>
inline cudaError_t launch_fwd_v(const FwdParams& p, cudaStream_t st) {
  return vec_ok<Tio, Tbc>(p) ? launch_fwd_n<Tio, Tbc, true>(p, st) : launch_fwd_n<Tio, Tbc, false>(p, st);
}

}  // namespace lbs
