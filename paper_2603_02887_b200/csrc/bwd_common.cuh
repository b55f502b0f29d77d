// Per-pixel back-to-front adjoint step shared by the global-order (K4) and
// exact-order (K4x) backward kernels.
#pragma once
#include "blend_common.cuh"

namespace nxs {

// per-pixel back-to-front replay state
struct BwdPix {
  PixelConst pc;
  int px, py, last, ck;
  bool sat;
  float tk, thi, tlo, P, Pck, s0, s1, s2, ek0, ek1, ek2, carry;
};

// one pixel's contribution of list entry (records rec, B frame bf) at
// virtual position idx; returns false (and leaves the outputs at zero) when
// the pixel does not replay this entry
template <int FAM>
__device__ __forceinline__ bool bwd_pixel(BwdPix& st, const float4* rec, const float4* bf, int idx,
                                          const CamDev& cam, const ModelDev& m, float cutoff,
                                          double near_plane, float inv_f, float gam, float& dm2,
                                          float& ux, float& uy, float& uz, float& dak, float& e0,
                                          float& e1, float& e2, unsigned long long& ntest,
                                          bool count) {
  if (idx > st.last) return false;
  if (count) ++ntest;
  TestOut t;
  const bool gen = (__float_as_int(rec[3].w) & RF_GENERAL) != 0;  // block-uniform
  float gx = 0.f, gy = 0.f, gz = 0.f;
  float tpk;
  const bool ok = gen ? general_test(rec, cam, st.px, st.py, cutoff, near_plane, t, gx, gy, gz, tpk)
                      : ray_peak_test(rec[0], rec[1], rec[2], rec[3], st.pc, cutoff, t);
  if (!ok) return false;
  const float alpha = t.alpha;
  float E0, E1, E2;
  const int mask = emission(rec[4], rec[5], rec[6], st.pc, E0, E1, E2);
  float dE0, dE1, dE2;
  if (st.sat && idx == st.last) {
    // saturating splat: moves the loss only through its emission (render.py:313-314)
    st.ek0 = E0;
    st.ek1 = E1;
    st.ek2 = E2;
    dE0 = st.s0 * st.tk;
    dE1 = st.s1 * st.tk;
    dE2 = st.s2 * st.tk;
  } else {
    // state in front of splat i, recovered back to front
    if constexpr (FAM != FAM_EXP) df_add(st.thi, st.tlo, -alpha);
    if constexpr (IsPFam<FAM>::value) {
      st.P = (idx == st.ck) ? st.Pck : div_newton(st.P, __fsub_rn(1.0f, alpha));
    }
    float fp;
    const float g = weight_g<FAM>(m, st.thi, st.tlo, st.P, fp);
    const float w = alpha * g;
    const float sdE = fmaf(st.s0, E0 - st.ek0, fmaf(st.s1, E1 - st.ek1, st.s2 * (E2 - st.ek2)));
    float da;
    if constexpr (IsPFam<FAM>::value) {
      da = fmaf(sdE, g, -gam * st.P * st.carry);
      st.carry = fmaf(1.0f - alpha, st.carry, sdE * alpha);
    } else {
      da = fmaf(sdE, g, st.carry);
      st.carry = fmaf(sdE * alpha, fp, st.carry);
    }
    dE0 = st.s0 * w;
    dE1 = st.s1 * w;
    dE2 = st.s2 * w;
    // chain moments (render.py:326-339): by the envelope theorem the
    // kernel-peak offset u = Rᵀ(t·d - b) carries the whole chain
    // (∂m2/∂μ = -2RΛu, ∂m2/∂s_k = -2u_k²/s_k³, ∂m2/∂R = 2 diff (Λu)ᵀ)
    const float dae = (t.araw >= ALPHA_MAX_F) ? 0.f : da;
    dm2 = -0.5f * alpha * dae;
    dak = dae * t.kern;
    // Whitened Gaussian-frame peak offset y = Λ^{1/2} u (u = Rᵀ diff; the
    // chain rescales by s in fp64), with the whitened B̃ = Λ^{1/2} B of K1.
    // Conic records: y = B̃ e with the stable conic offset e = δ - ε h
    // (δ = Δ/f, ε = δᵀA'h/D, all O(|δ|)).  For a thin Gaussian the
    // thin-axis component of B̃ e cancels (error ~1e-7 x the aspect ratio);
    // those records (RF_ANISO) use the cross-product form
    // y = b'_z (a × v)/|a|², a = B̃ h, v_k = s_k² [B̃ (Δ × c)]_k / (s0 s1 s2),
    // c = the centre's normalised image point: every input is O(1)-accurate.
    const int rflags = __float_as_int(rec[3].w);
    if (!gen && (rflags & RF_ANISO)) {
      const float dxn = t.ddx * inv_f, dyn = t.ddy * inv_f;
      const float ccx = st.pc.hx - dxn, ccy = st.pc.hy - dyn;
      const float w0 = dyn, w1 = -dxn, w2 = fmaf(dxn, ccy, -dyn * ccx);  // Δ × c
      const float ax = fmaf(bf[0].x, st.pc.hx, fmaf(bf[0].y, st.pc.hy, bf[0].z));
      const float ay = fmaf(bf[1].x, st.pc.hx, fmaf(bf[1].y, st.pc.hy, bf[1].z));
      const float az = fmaf(bf[2].x, st.pc.hx, fmaf(bf[2].y, st.pc.hy, bf[2].z));
      const float ip3 = 1.0f / (bf[0].w * bf[1].w * bf[2].w);
      const float v0 = fmaf(bf[0].x, w0, fmaf(bf[0].y, w1, bf[0].z * w2)) * (bf[0].w * bf[0].w * ip3);
      const float v1 = fmaf(bf[1].x, w0, fmaf(bf[1].y, w1, bf[1].z * w2)) * (bf[1].w * bf[1].w * ip3);
      const float v2 = fmaf(bf[2].x, w0, fmaf(bf[2].y, w1, bf[2].z * w2)) * (bf[2].w * bf[2].w * ip3);
      const float sc = rec[7].w / fmaf(ax, ax, fmaf(ay, ay, az * az));
      ux = fmaf(ay, v2, -az * v1) * sc;
      uy = fmaf(az, v0, -ax * v2) * sc;
      uz = fmaf(ax, v1, -ay * v0) * sc;
    } else {
      float qx, qy, qz;  // peak offset e (conic: diff'/b'_z; general: diff)
      if (gen) {
        qx = gx;
        qy = gy;
        qz = gz;
      } else {
        const float4 r2 = rec[2];
        const float dxn = t.ddx * inv_f, dyn = t.ddy * inv_f;
        const float Ahx = r2.x * t.u;
        const float Ahy = fmaf(r2.x * r2.y, t.u, r2.w * t.v);
        const float eps = fmaf(dxn, Ahx, dyn * Ahy) * t.rD;
        qx = fmaf(-eps, st.pc.hx, dxn);
        qy = fmaf(-eps, st.pc.hy, dyn);
        qz = -eps;
      }
      ux = fmaf(bf[0].x, qx, fmaf(bf[0].y, qy, bf[0].z * qz));
      uy = fmaf(bf[1].x, qx, fmaf(bf[1].y, qy, bf[1].z * qz));
      uz = fmaf(bf[2].x, qx, fmaf(bf[2].y, qy, bf[2].z * qz));
    }
  }
  // SH moments use dE_c·[E_c > 0] (render.py:340-341)
  e0 = (mask & 1) ? dE0 : 0.f;
  e1 = (mask & 2) ? dE1 : 0.f;
  e2 = (mask & 4) ? dE2 : 0.f;
  return true;
}

__device__ __forceinline__ void bwd_load(BwdPix& st, const CamDev& cam, int px, int py,
                                         const PixCache& cache, const float* __restrict__ seed,
                                         float bg0, float bg1, float bg2) {
  st.px = px;
  st.py = py;
  st.pc = pixel_setup(cam, px, py);
  st.last = -1;
  st.sat = false;
  st.tk = st.thi = st.tlo = st.Pck = 0.f;
  st.P = 1.f;
  st.ck = -1;
  st.s0 = st.s1 = st.s2 = 0.f;
  if (px < cam.W && py < cam.H) {
    const int pix = py * cam.W + px;
    st.last = cache.last[pix];
    st.sat = cache.sat[pix] != 0;
    st.tk = cache.t_k[pix];
    st.thi = cache.tau_hi[pix];
    st.tlo = cache.tau_lo[pix];
    st.P = cache.P_end[pix];
    st.ck = cache.ck_idx[pix];
    st.Pck = cache.P_ck[pix];
    st.s0 = seed[3 * pix + 0];
    st.s1 = seed[3 * pix + 1];
    st.s2 = seed[3 * pix + 2];
  }
  st.ek0 = bg0;
  st.ek1 = bg1;
  st.ek2 = bg2;
  st.carry = 0.f;  // Θ (τ-family) or U (P-family), seed-contracted
}

}  // namespace nxs
