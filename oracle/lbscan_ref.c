/*
 * CPU restatement of the reference's tiled LB scan engine — TEST / BASELINE
 * INFRASTRUCTURE ONLY (the CPU baseline leg of bench.py and the parity tests).
 *
 * Follows engine._scan_kernel (/root/reference/pkg/src/lbscan/engine.py:88-218)
 * phase by phase: per (batch, channel-block) work item and per tile of m
 * steps, (1) in-tile inclusive pair scan keeping the tile aggregate
 * (engine.py:128-142), (3) rescan seeded by the float64 running prefix
 * (:144-154), (2) float64 serial exchange of the aggregate (:156-165), the
 * in-tile exclusive reverse pass for the LB variant (:167-179) and the output
 * stage with 4-way split accumulators (:181-205); h_final is the last rescan
 * state (:207-209).  `reverse` indexes the sequence right-to-left (:133,183).
 * Work items run in parallel with OpenMP like numba's prange (:94); every
 * lane's arithmetic is independent of the partition.
 *
 * fp32 data with fp64 carries, exactly as the reference's single-precision
 * path.  Layouts: a2, b2 (B, L, E*N); c (B, L, N); dx, y (B, L, E);
 * hfin (B, E*N).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EBLOCK 16 /* engine.py:48 _EBLOCK for float32 */

int lbs_ref_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void lbs_ref_scan_f32(const float* a2, const float* b2, const float* c, const float* dx, int64_t B,
                      int64_t L, int64_t E, int64_t N, int64_t m, int do_backward, int reverse,
                      float* y_out, float* hfin2, int nthreads) {
  const int64_t EN = E * N;
  const int64_t T = (L + m - 1) / m;
  const int64_t eblk = E < EBLOCK ? E : EBLOCK;
  const int64_t nblk = (E + eblk - 1) / eblk;
  const int64_t items = B * nblk;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t item = 0; item < items; ++item) {
    const int64_t b = item / nblk;
    const int64_t e0 = (item % nblk) * eblk;
    const int64_t e1 = (e0 + eblk < E) ? e0 + eblk : E;
    const int64_t w0 = e0 * N;
    const int64_t W = e1 * N - w0;
    double* pfx_a = (double*)malloc(sizeof(double) * W);
    double* pfx_b = (double*)malloc(sizeof(double) * W);
    float* sa = (float*)malloc(sizeof(float) * W);
    float* sb = (float*)malloc(sizeof(float) * W);
    float* ra = (float*)malloc(sizeof(float) * W);
    float* rb = (float*)malloc(sizeof(float) * W);
    float* hb = (float*)malloc(sizeof(float) * W);
    float* abuf = (float*)malloc(sizeof(float) * m * W);
    float* bbuf = (float*)malloc(sizeof(float) * m * W);
    float* hbuf = (float*)malloc(sizeof(float) * m * W);
    for (int64_t w = 0; w < W; ++w) { pfx_a[w] = 1.0; pfx_b[w] = 0.0; }
    for (int64_t t = 0; t < T; ++t) {
      const int64_t lo = t * m;
      const int64_t hi = (lo + m < L) ? lo + m : L;
      const int64_t r = hi - lo;
      /* phase 1: in-tile inclusive pair scan */
      for (int64_t w = 0; w < W; ++w) { sa[w] = 1.0f; sb[w] = 0.0f; }
      for (int64_t j = 0; j < r; ++j) {
        const int64_t src = reverse ? L - 1 - (lo + j) : lo + j;
        const float* ap = a2 + (b * L + src) * EN + w0;
        const float* bp = b2 + (b * L + src) * EN + w0;
        float* ab = abuf + j * W;
        float* bb = bbuf + j * W;
        for (int64_t w = 0; w < W; ++w) {
          const float a = ap[w], v = bp[w];
          ab[w] = a;
          bb[w] = v;
          sa[w] = sa[w] * a;
          sb[w] = a * sb[w] + v;
        }
      }
      /* phase 3: rescan seeded with this tile's prefix */
      for (int64_t w = 0; w < W; ++w) { ra[w] = (float)pfx_a[w]; rb[w] = (float)pfx_b[w]; }
      for (int64_t j = 0; j < r; ++j) {
        const float* ab = abuf + j * W;
        const float* bb = bbuf + j * W;
        float* hh = hbuf + j * W;
        for (int64_t w = 0; w < W; ++w) {
          const float a = ab[w];
          ra[w] = ra[w] * a;
          rb[w] = a * rb[w] + bb[w];
          hh[w] = rb[w];
        }
      }
      /* phase 2: float64 exchange of the tile aggregate */
      if (t < T - 1) {
        for (int64_t w = 0; w < W; ++w) {
          const double ag = (double)sa[w];
          pfx_b[w] = ag * pfx_b[w] + (double)sb[w];
          pfx_a[w] = ag * pfx_a[w];
        }
      }
      /* in-tile backward pass (LB only) */
      if (do_backward && r > 1) {
        for (int64_t w = 0; w < W; ++w) hb[w] = bbuf[(r - 1) * W + w];
        for (int64_t j = r - 2; j >= 1; --j) {
          for (int64_t w = 0; w < W; ++w) {
            const float dec = abuf[j * W + w] * hb[w];
            hbuf[j * W + w] = hbuf[j * W + w] + dec;
            hb[w] = dec + bbuf[j * W + w];
          }
        }
        for (int64_t w = 0; w < W; ++w) hbuf[w] = hbuf[w] + abuf[w] * hb[w];
      }
      /* output stage */
      for (int64_t j = 0; j < r; ++j) {
        const int64_t src = reverse ? L - 1 - (lo + j) : lo + j;
        const float* cc = c + (b * L + src) * N;
        for (int64_t ee = e0; ee < e1; ++ee) {
          const float* hh = hbuf + j * W + (ee - e0) * N;
          float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
          int64_t n = 0;
          for (; n + 4 <= N; n += 4) {
            q0 = q0 + cc[n] * hh[n];
            q1 = q1 + cc[n + 1] * hh[n + 1];
            q2 = q2 + cc[n + 2] * hh[n + 2];
            q3 = q3 + cc[n + 3] * hh[n + 3];
          }
          for (; n < N; ++n) q0 = q0 + cc[n] * hh[n];
          y_out[(b * L + src) * E + ee] = ((q0 + q1) + (q2 + q3)) + dx[(b * L + src) * E + ee];
        }
      }
    }
    for (int64_t w = 0; w < W; ++w) hfin2[b * EN + w0 + w] = rb[w];
    free(pfx_a); free(pfx_b); free(sa); free(sb); free(ra); free(rb); free(hb);
    free(abuf); free(bbuf); free(hbuf);
  }
}
