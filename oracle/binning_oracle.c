/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the per-Gaussian projection, conic tile binning
 * and tile|depth ordering that the CUDA path computes in
 * paper_2603_02887_b200/csrc/project.cu, used as the bit-exact checker for
 * "projection and binning plus a radix sort keyed on tile|depth".  The
 * reference has no binning (it tests every Gaussian against every pixel,
 * reference pkg/src/nexsplat/render.py:109-138); what it does define, and
 * what this file follows, is:
 *   - the global order: stable argsort of the float64 view depth
 *     (μ - o)·forward, reference render.py:350-358 (evaluated as a
 *     compensated dot product: numpy's `@` goes through OpenBLAS with a
 *     CPU-dependent FMA order, so the reference's last bit is not
 *     machine-independent; see test_binning_oracle.py for the tie rule);
 *   - the per-Gaussian frame: normalised quaternion -> R
 *     (primitives.py:45-64), A = R diag(s^-2) R^T, b = μ - o
 *     (render.py:116-121);
 *   - validity alpha >= cutoff <=> m2 <= 2 ln(opacity/cutoff)
 *     (render.py:130-134), whose silhouette conic bounds the tile set.
 * The camera-frame conic algebra and the op order are the
 * normative definition shared with the CUDA kernel; this file is built with
 * -O2 -ffp-contract=off so every double op is one IEEE op, like the kernel
 * (nvcc --fmad=false).  Sorting here is a plain stable merge sort and a
 * stable counting sort — independent of the device's radix sorts.
 *
 * Build: see oracle/Makefile (output oracle/build/libnxs_oracle.so).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16
#define RF_CONIC 1

static double ln_series(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0.70710678118654752440) {
    m = m * 2.0;
    e = e - 1;
  }
  double z = (m - 1.0) / (m + 1.0);
  double z2 = z * z;
  static const double inv_odd[12] = {1.0 / 23.0, 1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0,
                                     1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0, 1.0 / 9.0,
                                     1.0 / 7.0,  1.0 / 5.0,  1.0 / 3.0,  1.0};
  double s = inv_odd[0];
  for (int k = 1; k < 12; ++k) s = s * z2 + inv_odd[k];
  return (double)e * 0.69314718055994530942 + 2.0 * z * s;
}

/* compensated dot product (Dot2), same op sequence as the device's K0 */
static double dot3_compensated(double a0, double a1, double a2, double b0, double b1, double b2) {
  double p = a0 * b0;
  double s = fma(a0, b0, -p);
  double h = a1 * b1, r = fma(a1, b1, -h);
  double t = p + h, bb = t - p, q = (p - (t - bb)) + (h - bb);
  p = t;
  s = s + (q + r);
  h = a2 * b2;
  r = fma(a2, b2, -h);
  t = p + h;
  bb = t - p;
  q = (p - (t - bb)) + (h - bb);
  p = t;
  s = s + (q + r);
  return p + s;
}

static uint64_t depth_key(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

/* stable merge sort of idx by key */
static void msort(uint32_t* idx, uint32_t* tmp, const uint64_t* key, int64_t n) {
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = (key[idx[b]] < key[idx[a]]) ? idx[b++] : idx[a++];
      while (a < mid) tmp[o++] = idx[a++];
      while (b < hi) tmp[o++] = idx[b++];
    }
    memcpy(idx, tmp, (size_t)n * sizeof(uint32_t));
  }
}

/* Exact tile culling (csrc/project.cu tile_hit): does the silhouette
 * ellipse q(X, Y) = Hᵀ Q H <= 0 meet the tile's pixel-centre rectangle?
 * t = (q00, q01, q11, q02, q12, q22, c0, c1), c = the projected centre (inside). */
static int tile_hit(const double* t, int tx, int ty, double cx, double cy, double f, int W,
                    int H) {
  const double q00 = t[0];
  if (!(q00 == q00)) return 1;
  const double q01 = t[1], q11 = t[2], q02 = t[3], q12 = t[4], q22 = t[5];
  const double c0 = t[6], c1 = t[7], h00 = t[8], h11 = t[9];
  const int jx0 = tx * TILE, iy0 = ty * TILE;
  const int jx1 = jx0 + TILE - 1 < W - 1 ? jx0 + TILE - 1 : W - 1;
  const int iy1 = iy0 + TILE - 1 < H - 1 ? iy0 + TILE - 1 : H - 1;
  const double inv_f = 1.0 / f;
  const double x0 = (((double)jx0 + 0.5) - cx) * inv_f, x1 = (((double)jx1 + 0.5) - cx) * inv_f;
  const double y0 = (((double)iy0 + 0.5) - cy) * inv_f, y1 = (((double)iy1 + 0.5) - cy) * inv_f;
  if (c0 >= x0 && c0 <= x1 && c1 >= y0 && c1 <= y1) return 1;
  for (int k = 0; k < 2; ++k) {
    const double xe = k ? x1 : x0;
    const double b = 2.0 * (q01 * xe + q12);
    const double c = (q00 * xe * xe + 2.0 * q02 * xe) + q22;
    double yv = -b * h11;
    yv = yv < y0 ? y0 : (yv > y1 ? y1 : yv);
    if ((q11 * yv + b) * yv + c <= 0.0) return 1;
  }
  for (int k = 0; k < 2; ++k) {
    const double ye = k ? y1 : y0;
    const double b = 2.0 * (q01 * ye + q02);
    const double c = (q11 * ye * ye + 2.0 * q12 * ye) + q22;
    double xv = -b * h00;
    xv = xv < x0 ? x0 : (xv > x1 ? x1 : xv);
    if ((q00 * xv + b) * xv + c <= 0.0) return 1;
  }
  return 0;
}

/*
 * Outputs (caller-allocated):
 *   order[P]       rank -> Gaussian index
 *   records[P*32]  per-rank record floats (layout of csrc/nxs_internal.cuh)
 *   rects[P*4]     tx0, ty0, tx1, ty1 per rank (-1 when culled)
 *   ranges[T*2]    per-tile [start, end) in the pair list
 *   pairs          per-tile rank lists; pass NULL to only get n_pairs
 * Returns the number of pairs, or -1 if a Gaussian straddles the near plane.
 */
int64_t nxs_oracle_binning(int64_t P, const float* centers, const float* scales,
                           const float* quats, const float* opacities, const double* cam_o,
                           const double* cam_R, double f, double cx, double cy, int W, int H,
                           double cutoff, double near_plane, int32_t* order, float* records,
                           int32_t* rects, int32_t* ranges, int32_t* pairs, int64_t pair_cap) {
  const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
  const int T = tiles_x * tiles_y;
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(P > 0 ? P : 1));
  uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(P > 0 ? P : 1));
  uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(P > 0 ? P : 1));
  int64_t straddle = 0;
  for (int64_t i = 0; i < P; ++i) {
    double b0 = (double)centers[3 * i + 0] - cam_o[0];
    double b1 = (double)centers[3 * i + 1] - cam_o[1];
    double b2 = (double)centers[3 * i + 2] - cam_o[2];
    double depth = dot3_compensated(b0, b1, b2, cam_R[2], cam_R[5], cam_R[8]);
    key[i] = depth_key(depth);
    idx[i] = (uint32_t)i;
  }
  msort(idx, tmp, key, P);
  int64_t* count = (int64_t*)calloc((size_t)(P > 0 ? P : 1), sizeof(int64_t));
  double* tq = (double*)malloc(sizeof(double) * 10 * (size_t)(P > 0 ? P : 1));
  for (int64_t r = 0; r < P; ++r) {
    const int64_t g = idx[r];
    order[r] = (int32_t)g;
    double qw = quats[4 * g + 0], qx = quats[4 * g + 1], qy = quats[4 * g + 2],
           qz = quats[4 * g + 3];
    double nq = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
    double inq = 1.0 / nq;
    double w = qw * inq, x = qx * inq, y = qy * inq, z = qz * inq;
    double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                   2.0 * (x * y + w * z),       1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                   2.0 * (x * z - w * y),       2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    double M[9], Ap[9], bp[3], Ab[3], N[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        M[3 * i + j] = (cam_R[0 + i] * R[0 + j] + cam_R[3 + i] * R[3 + j]) + cam_R[6 + i] * R[6 + j];
    double s0 = scales[3 * g + 0], s1 = scales[3 * g + 1], s2 = scales[3 * g + 2];
    double is0 = 1.0 / (s0 * s0), is1 = 1.0 / (s1 * s1), is2 = 1.0 / (s2 * s2);
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        double v = ((M[3 * i + 0] * is0) * M[3 * j + 0] + (M[3 * i + 1] * is1) * M[3 * j + 1]) +
                   (M[3 * i + 2] * is2) * M[3 * j + 2];
        Ap[3 * i + j] = v;
        Ap[3 * j + i] = v;
      }
    double b0 = (double)centers[3 * g + 0] - cam_o[0];
    double b1 = (double)centers[3 * g + 1] - cam_o[1];
    double b2 = (double)centers[3 * g + 2] - cam_o[2];
    for (int i = 0; i < 3; ++i) bp[i] = (cam_R[0 + i] * b0 + cam_R[3 + i] * b1) + cam_R[6 + i] * b2;
    for (int i = 0; i < 3; ++i)
      Ab[i] = (Ap[3 * i + 0] * bp[0] + Ap[3 * i + 1] * bp[1]) + Ap[3 * i + 2] * bp[2];
    double bAb = (bp[0] * Ab[0] + bp[1] * Ab[1]) + bp[2] * Ab[2];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) N[3 * i + j] = bAb * Ap[3 * i + j] - Ab[i] * Ab[j];

    int32_t rect[4] = {-1, -1, -1, -1};
    int64_t ntile = 0;
    double opac = (double)opacities[g];
    int live = opac >= cutoff;
    double r2 = live ? 2.0 * ln_series(opac / cutoff) : 0.0;
    double r2m = r2 * (1.0 + 1e-4) + 1e-4;
    double rm = sqrt(r2m);
    double m20 = M[6] * s0, m21 = M[7] * s1, m22 = M[8] * s2;
    double sz = sqrt((m20 * m20 + m21 * m21) + m22 * m22);
    double zmin = bp[2] - rm * sz, zmax = bp[2] + rm * sz;
    if (live && zmax <= 0.0) live = 0;
    if (live && zmin <= near_plane * 1.001) {
      ++straddle;
      live = 0;
    }
    double f2 = f * f;
    double if2 = 1.0 / f2;
    double Np00 = N[0] * if2, Np01 = N[1] * if2, Np11 = N[4] * if2;
    double n0 = Np00, kk = Np01 / Np00, n1 = Np11 - Np01 * kk;
    double ibz = 1.0 / bp[2];
    double ccx = cx + f * (bp[0] * ibz);
    double ccy = cy + f * (bp[1] * ibz);
    float cxh = (float)ccx, cyh = (float)ccy;
    float cxl = (float)(ccx - (double)cxh), cyl = (float)(ccy - (double)cyh);
    double a = Ap[0], ia = 1.0 / a, bb = Ap[1] * ia, cc = Ap[2] * ia;
    double A11s = Ap[4] - Ap[1] * bb, A12s = Ap[5] - Ap[1] * cc, A22s = Ap[8] - Ap[2] * cc;
    double d = A11s, e = A12s / d, gg = A22s - A12s * e;
    if (live) {
      double Q[9];
      for (int i = 0; i < 9; ++i) Q[i] = N[i] - r2m * Ap[i];
      double S00 = Q[4] * Q[8] - Q[5] * Q[5];
      double S11 = Q[0] * Q[8] - Q[2] * Q[2];
      double S22 = Q[0] * Q[4] - Q[1] * Q[1];
      double S02 = Q[1] * Q[5] - Q[2] * Q[4];
      double S12 = Q[1] * Q[2] - Q[0] * Q[5];
      double dx = S02 * S02 - S00 * S22;
      double dy = S12 * S12 - S11 * S22;
      double jlo = 0.0, jhi = (double)(W - 1), ilo = 0.0, ihi = (double)(H - 1);
      const int ok = (dx >= 0.0) && (dy >= 0.0) && (S22 != 0.0);
      if (ok) {
        double sx = sqrt(dx), sy = sqrt(dy);
        double iS = 1.0 / S22;
        double x1 = (S02 - sx) * iS, x2 = (S02 + sx) * iS;
        double y1 = (S12 - sy) * iS, y2 = (S12 + sy) * iS;
        double xl = x1 < x2 ? x1 : x2, xh = x1 < x2 ? x2 : x1;
        double yl = y1 < y2 ? y1 : y2, yh = y1 < y2 ? y2 : y1;
        double pjl = ceil((cx + f * xl) - 0.5), pjh = floor((cx + f * xh) - 0.5);
        double pil = ceil((cy + f * yl) - 0.5), pih = floor((cy + f * yh) - 0.5);
        if (pjl > jlo) jlo = pjl;
        if (pjh < jhi) jhi = pjh;
        if (pil > ilo) ilo = pil;
        if (pih < ihi) ihi = pih;
      }
      tq[10 * r] = NAN;
      if (jlo <= jhi && ilo <= ihi) {
        int j0 = (int)jlo, j1 = (int)jhi, i0 = (int)ilo, i1 = (int)ihi;
        rect[0] = j0 / TILE;
        rect[1] = i0 / TILE;
        rect[2] = j1 / TILE;
        rect[3] = i1 / TILE;
        if (ok) {
          double* t = tq + 10 * r;
          t[0] = Q[0];
          t[1] = Q[1];
          t[2] = Q[4];
          t[3] = Q[2];
          t[4] = Q[5];
          t[5] = Q[8];
          t[6] = bp[0] * ibz;
          t[7] = bp[1] * ibz;
          t[8] = 0.5 / Q[0];
          t[9] = 0.5 / Q[4];
        }
        for (int ty = rect[1]; ty <= rect[3]; ++ty)
          for (int tx = rect[0]; tx <= rect[2]; ++tx)
            ntile += tile_hit(tq + 10 * r, tx, ty, cx, cy, f, W, H);
      }
    }
    float* rec = records + r * 32;
    rec[0] = cxh; rec[1] = cyh; rec[2] = cxl; rec[3] = cyl;
    rec[4] = (float)n0; rec[5] = (float)kk; rec[6] = (float)n1; rec[7] = (float)r2m;
    rec[8] = (float)a; rec[9] = (float)bb; rec[10] = (float)cc; rec[11] = (float)d;
    rec[12] = (float)e; rec[13] = (float)gg; rec[14] = (float)opac;
    {
      int32_t fl = RF_CONIC;
      memcpy(&rec[15], &fl, 4);
    }
    /* rec[16..27]: sh copy, rec[28..31]: A'b', zmin (not checked here) */
    for (int k = 16; k < 32; ++k) rec[k] = 0.0f;
    rec[28] = (float)Ab[0]; rec[29] = (float)Ab[1]; rec[30] = (float)Ab[2]; rec[31] = (float)zmin;
    memcpy(rects + 4 * r, rect, sizeof rect);
    count[r] = ntile;
  }
  /* stable counting sort of (tile, rank) pairs by tile, emitted in rank order */
  int64_t n_pairs = 0;
  for (int64_t r = 0; r < P; ++r) n_pairs += count[r];
  int64_t* tcount = (int64_t*)calloc((size_t)T + 1, sizeof(int64_t));
  for (int64_t r = 0; r < P; ++r) {
    const int32_t* rc = rects + 4 * r;
    if (rc[0] < 0) continue;
    for (int ty = rc[1]; ty <= rc[3]; ++ty)
      for (int tx = rc[0]; tx <= rc[2]; ++tx)
        if (tile_hit(tq + 10 * r, tx, ty, cx, cy, f, W, H)) tcount[ty * tiles_x + tx + 1]++;
  }
  for (int t = 0; t < T; ++t) tcount[t + 1] += tcount[t];
  for (int t = 0; t < T; ++t) {
    /* the device leaves untouched (empty) tiles at [0, 0) */
    int64_t s0 = tcount[t], s1 = tcount[t + 1];
    ranges[2 * t + 0] = s1 > s0 ? (int32_t)s0 : 0;
    ranges[2 * t + 1] = s1 > s0 ? (int32_t)s1 : 0;
  }
  if (pairs && pair_cap >= n_pairs) {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
    for (int t = 0; t < T; ++t) fill[t] = tcount[t];
    for (int64_t r = 0; r < P; ++r) {
      const int32_t* rc = rects + 4 * r;
      if (rc[0] < 0) continue;
      for (int ty = rc[1]; ty <= rc[3]; ++ty)
        for (int tx = rc[0]; tx <= rc[2]; ++tx)
          if (tile_hit(tq + 10 * r, tx, ty, cx, cy, f, W, H))
            pairs[fill[ty * tiles_x + tx]++] = (int32_t)r;
    }
    free(fill);
  }
  free(tcount);
  free(count);
  free(tq);
  free(key);
  free(idx);
  free(tmp);
  return straddle ? -1 : n_pairs;
}
