// Per-pixel ray-peak test and emission shared by the forward (K3) and the
// backward (K4) blend kernels.
//
// Every float operation is an explicit round-to-nearest intrinsic, so the
// compiler cannot contract or reorder differently in the two kernels: the
// backward replays exactly the validity decisions and alphas of the forward.
//
// Restates, per (Gaussian, pixel) (reference pkg/src/nexsplat/render.py):
//   t, m2, alpha, valid     _chunk_geometry, render.py:122-134
//   emission E, E>0 mask    _sh_basis/_emission, render.py:97-106, 141-144
// via the centred-conic form of SURVEY §8.0.5: m2 = Δᵀ N' Δ / hᵀA'h with
// Δ the pixel offset from the fp32 (hi, lo) projected centre.
#pragma once
#include "nxs_internal.cuh"

namespace nxs {

// Packed f32x2 arithmetic (Blackwell FFMA2/FADD2/FMUL2): lane x and lane y
// are each the IEEE round-to-nearest scalar op, so packed and scalar code
// give bit-identical results; scalar operands broadcast without moves.
struct F2 {
  float x, y;
};
__device__ __forceinline__ F2 f2(float a) { return F2{a, a}; }
#define NXS_F2OP3(name, op)                                                                  \
  __device__ __forceinline__ F2 name(F2 a, F2 b) {                                          \
    F2 d;                                                                                    \
    asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n " op        \
        " rd, ra, rb;\n mov.b64 {%0,%1}, rd;}"                                              \
        : "=f"(d.x), "=f"(d.y)                                                               \
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                           \
    return d;                                                                                \
  }
NXS_F2OP3(add2, "add.rn.f32x2")
NXS_F2OP3(sub2, "sub.rn.f32x2")
NXS_F2OP3(mul2, "mul.rn.f32x2")
#undef NXS_F2OP3
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n"
      " mov.b64 rc, {%6,%7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ F2 sel2(bool qa, bool qb, F2 v) {
  return F2{qa ? v.x : 0.f, qb ? v.y : 0.f};
}
// packed df_add: (hi, lo) += a per lane, exactly (nxs_internal.cuh df_add)
__device__ __forceinline__ void df_add2(F2& hi, F2& lo, F2 a) {
  const F2 s = add2(hi, a);
  const F2 bb = sub2(s, hi);
  const F2 e = add2(sub2(hi, sub2(s, bb)), sub2(a, bb));
  const F2 el = add2(e, lo);
  const F2 s2 = add2(s, el);
  lo = sub2(el, sub2(s2, s));
  hi = s2;
}

struct PixelConst {
  float pxc, pyc;  // pixel centre (j + 0.5, i + 0.5)
  float hx, hy;    // normalised image coordinates ((j+0.5-cx)/f, (i+0.5-cy)/f)
  float Y1, Y2, Y3;  // SH band-1 basis; Y0 = C0
};

__device__ __forceinline__ PixelConst pixel_setup(const CamDev& cam, int px, int py) {
  PixelConst pc;
  const double inv_f = cam.inv_f;  // = 1.0 / cam.f, correctly rounded on the host
  const double hxd = ((double)px + 0.5 - cam.cx) * inv_f;
  const double hyd = ((double)py + 0.5 - cam.cy) * inv_f;
  pc.pxc = (float)px + 0.5f;
  pc.pyc = (float)py + 0.5f;
  pc.hx = (float)hxd;
  pc.hy = (float)hyd;
  // world direction = R (hx, hy, 1), normalised (primitives.py:192-203); the
  // SH basis only needs it to fp32 accuracy
  const float dx = __fmaf_rn(cam.Rf[0], pc.hx, __fmaf_rn(cam.Rf[1], pc.hy, cam.Rf[2]));
  const float dy = __fmaf_rn(cam.Rf[3], pc.hx, __fmaf_rn(cam.Rf[4], pc.hy, cam.Rf[5]));
  const float dz = __fmaf_rn(cam.Rf[6], pc.hx, __fmaf_rn(cam.Rf[7], pc.hy, cam.Rf[8]));
  const float inv = rsqrtf(__fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz))));
  pc.Y1 = (float)(-SH_C1) * (dy * inv);
  pc.Y2 = (float)SH_C1 * (dz * inv);
  pc.Y3 = (float)(-SH_C1) * (dx * inv);
  return pc;
}

struct TestOut {
  float ddx, ddy;  // Δ in pixels
  float D;         // hᵀ A' h
  float rD;        // rcp.approx(D), shared by m2 and the backward's ε
  float u, v;      // D = a·u² + d·v² + g  (so (A'h)_x = a·u, (A'h)_y = a·b·u + d·v)
  float m2;        // Mahalanobis distance² at the ray peak
  float kern;      // exp(-m2/2)
  float araw;      // opacity·kern (unclamped)
  float alpha;     // min(araw, ALPHA_MAX)
};

// r0 = (cxh, cyh, cxl, cyl); r1 = (n0, k, n1, r2m); r2 = (a, b, c, d); r3 = (e, g, opac, flags)
__device__ __forceinline__ bool ray_peak_test(const float4& r0, const float4& r1, const float4& r2,
                                              const float4& r3, const PixelConst& pc, float cutoff,
                                              TestOut& o) {
  o.ddx = __fsub_rn(__fsub_rn(pc.pxc, r0.x), r0.z);
  o.ddy = __fsub_rn(__fsub_rn(pc.pyc, r0.y), r0.w);
  float w = __fmaf_rn(r1.y, o.ddy, o.ddx);
  float num = __fmaf_rn(__fmul_rn(r1.x, w), w, __fmul_rn(__fmul_rn(r1.z, o.ddy), o.ddy));
  const float u = __fadd_rn(__fmaf_rn(r2.y, pc.hy, r2.z), pc.hx);
  const float v = __fadd_rn(pc.hy, r3.x);
  o.u = u;
  o.v = v;
  o.D = __fmaf_rn(__fmul_rn(r2.x, u), u, __fmaf_rn(__fmul_rn(r2.w, v), v, r3.y));
  // cheap reject against the cutoff ellipse (r2m carries a 1e-4 margin)
  if (num > __fmul_rn(r1.w, o.D)) return false;
  o.rD = rcp_approx(o.D);
  o.m2 = __fmul_rn(num, o.rD);
  o.kern = ex2_approx(__fmul_rn(-0.72134752044448170368f, o.m2));  // e^{-m2/2}
  o.araw = __fmul_rn(r3.z, o.kern);
  o.alpha = fminf(o.araw, ALPHA_MAX_F);
  return o.alpha >= cutoff;
}

// General path (records flagged RF_GENERAL: the cutoff ellipsoid reaches
// the near region, so the conic form and its implied t > near do not hold):
// the reference's per-(Gaussian, pixel) formula, render.py:122-134, in fp64
// with explicit IEEE ops (identical in the forward and backward kernels).
// Outputs the world-frame peak offset diff = t·d - b for the chain.
__device__ __forceinline__ bool general_test(const float4* rec, const CamDev& cam, int px, int py,
                                             float cutoff, double near_plane, TestOut& o,
                                             float& gdx, float& gdy, float& gdz, float& tpk) {
  const double* dp = reinterpret_cast<const double*>(rec);
  const double b0 = dp[0], b1 = dp[1], b2 = dp[2];
  const double A00 = dp[3], A01 = dp[4], A02 = dp[5], A11 = dp[6], A12 = dp[14], A22 = dp[15];
  const float opac = reinterpret_cast<const float*>(rec)[14];
  // unit world direction through the pixel centre (primitives.py:192-203)
  const double hx = __ddiv_rn(__dsub_rn(__dadd_rn((double)px, 0.5), cam.cx), cam.f);
  const double hy = __ddiv_rn(__dsub_rn(__dadd_rn((double)py, 0.5), cam.cy), cam.f);
  double d0 = __dadd_rn(__dadd_rn(__dmul_rn(hx, cam.R[0]), __dmul_rn(hy, cam.R[1])), cam.R[2]);
  double d1 = __dadd_rn(__dadd_rn(__dmul_rn(hx, cam.R[3]), __dmul_rn(hy, cam.R[4])), cam.R[5]);
  double d2 = __dadd_rn(__dadd_rn(__dmul_rn(hx, cam.R[6]), __dmul_rn(hy, cam.R[7])), cam.R[8]);
  const double nd = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)),
                                         __dmul_rn(d2, d2)));
  d0 = __ddiv_rn(d0, nd);
  d1 = __ddiv_rn(d1, nd);
  d2 = __ddiv_rn(d2, nd);
#define NXS_DOT3(a0, a1, a2, c0, c1, c2) \
  __dadd_rn(__dadd_rn(__dmul_rn(a0, c0), __dmul_rn(a1, c1)), __dmul_rn(a2, c2))
  const double Ad0 = NXS_DOT3(A00, A01, A02, d0, d1, d2);
  const double Ad1 = NXS_DOT3(A01, A11, A12, d0, d1, d2);
  const double Ad2 = NXS_DOT3(A02, A12, A22, d0, d1, d2);
  const double dAd = NXS_DOT3(Ad0, Ad1, Ad2, d0, d1, d2);
  const double bAd = NXS_DOT3(b0, b1, b2, Ad0, Ad1, Ad2);
  const double t = __ddiv_rn(bAd, dAd);
  const double x0 = __dsub_rn(__dmul_rn(t, d0), b0);
  const double x1 = __dsub_rn(__dmul_rn(t, d1), b1);
  const double x2 = __dsub_rn(__dmul_rn(t, d2), b2);
  const double m2 = NXS_DOT3(x0, x1, x2, NXS_DOT3(A00, A01, A02, x0, x1, x2),
                             NXS_DOT3(A01, A11, A12, x0, x1, x2), NXS_DOT3(A02, A12, A22, x0, x1, x2));
#undef NXS_DOT3
  o.m2 = (float)m2;
  o.rD = 0.f;
  o.kern = ex2_approx(__fmul_rn(-0.72134752044448170368f, o.m2));
  o.araw = __fmul_rn(opac, o.kern);
  o.alpha = fminf(o.araw, ALPHA_MAX_F);
  gdx = (float)x0;
  gdy = (float)x1;
  gdz = (float)x2;
  tpk = (float)t;
  return (t > near_plane) && (o.alpha >= cutoff);
}

// E_c = max(Σ_k sh[c][k] Y_k, 0); returns the positivity mask bits.  The
// record holds sh[c][0]·Y0 pre-multiplied (project.cu).
__device__ __forceinline__ int emission(const float4& s0, const float4& s1, const float4& s2,
                                        const PixelConst& pc, float& E0, float& E1, float& E2) {
  float e0 = __fmaf_rn(s0.w, pc.Y3, __fmaf_rn(s0.z, pc.Y2, __fmaf_rn(s0.y, pc.Y1, s0.x)));
  float e1 = __fmaf_rn(s1.w, pc.Y3, __fmaf_rn(s1.z, pc.Y2, __fmaf_rn(s1.y, pc.Y1, s1.x)));
  float e2 = __fmaf_rn(s2.w, pc.Y3, __fmaf_rn(s2.z, pc.Y2, __fmaf_rn(s2.y, pc.Y1, s2.x)));
  int mask = (e0 > 0.f ? 1 : 0) | (e1 > 0.f ? 2 : 0) | (e2 > 0.f ? 4 : 0);
  E0 = fmaxf(e0, 0.f);
  E1 = fmaxf(e1, 0.f);
  E2 = fmaxf(e2, 0.f);
  return mask;
}

// Packed ray-peak test of one record for a column's two pixels (a: lane x,
// b: lane y; same px, so Δx is shared): the same rounded ops as
// ray_peak_test, lane by lane.  ok_a/ok_b enter as "pixel still replays"
// and leave as "pixel passes the test".
struct TestOut2 {
  float ddx;
  F2 ddy, u, v, rD, kern, araw, alpha;
};
__device__ __forceinline__ void ray_peak_test2(const float4& r0, const float4& r1, const float4& r2,
                                               const float4& r3, const PixelConst& pa,
                                               const PixelConst& pb, float cutoff, TestOut2& o,
                                               bool& ok_a, bool& ok_b) {
  o.ddx = __fsub_rn(__fsub_rn(pa.pxc, r0.x), r0.z);
  const F2 hy{pa.hy, pb.hy};
  o.ddy = sub2(sub2(F2{pa.pyc, pb.pyc}, f2(r0.y)), f2(r0.w));
  const F2 w = fma2(f2(r1.y), o.ddy, f2(o.ddx));
  const F2 num = fma2(mul2(f2(r1.x), w), w, mul2(mul2(f2(r1.z), o.ddy), o.ddy));
  o.u = add2(fma2(f2(r2.y), hy, f2(r2.z)), f2(pa.hx));
  o.v = add2(hy, f2(r3.x));
  const F2 D = fma2(mul2(f2(r2.x), o.u), o.u, fma2(mul2(f2(r2.w), o.v), o.v, f2(r3.y)));
  const F2 lim = mul2(f2(r1.w), D);
  ok_a = ok_a && !(num.x > lim.x);
  ok_b = ok_b && !(num.y > lim.y);
  if (!(ok_a || ok_b)) return;
  o.rD = F2{rcp_approx(D.x), rcp_approx(D.y)};
  const F2 ek = mul2(f2(-0.72134752044448170368f), mul2(num, o.rD));
  o.kern = F2{ex2_approx(ek.x), ex2_approx(ek.y)};
  o.araw = mul2(f2(r3.z), o.kern);
  o.alpha = F2{fminf(o.araw.x, ALPHA_MAX_F), fminf(o.araw.y, ALPHA_MAX_F)};
  ok_a = ok_a && o.alpha.x >= cutoff;
  ok_b = ok_b && o.alpha.y >= cutoff;
}

// Packed emission (same rounded ops as emission); c = the unclamped sums.
__device__ __forceinline__ void emission2(const float4& s0, const float4& s1, const float4& s2,
                                          const PixelConst& pa, const PixelConst& pb, F2& c0,
                                          F2& c1, F2& c2) {
  const F2 Y1{pa.Y1, pb.Y1}, Y2{pa.Y2, pb.Y2}, Y3{pa.Y3, pb.Y3};
  c0 = fma2(f2(s0.w), Y3, fma2(f2(s0.z), Y2, fma2(f2(s0.y), Y1, f2(s0.x))));
  c1 = fma2(f2(s1.w), Y3, fma2(f2(s1.z), Y2, fma2(f2(s1.y), Y1, f2(s1.x))));
  c2 = fma2(f2(s2.w), Y3, fma2(f2(s2.z), Y2, fma2(f2(s2.y), Y1, f2(s2.x))));
}

}  // namespace nxs
