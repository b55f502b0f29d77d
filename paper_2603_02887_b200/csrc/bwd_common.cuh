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

// ---------------------------------------------------------------------------
// Packed two-pixel step (Blackwell FFMA2/FADD2/FMUL2).  The global-order
// backward gives each thread two pixels of the same column (adjacent rows), so
// every per-pixel fp32 operation of the common record kind (conic, not thin)
// runs as one f32x2 instruction on the pair; record values enter as scalar
// broadcast operands.  Each lane of an f32x2 op is the IEEE round-to-nearest
// scalar op, so the ray-peak test and the emission stay bit-identical to the
// forward's scalar code (blend_common.cuh); MUFU ops stay scalar.
// ---------------------------------------------------------------------------

// Outputs of one entry for the thread's two pixels (lane x: pixel a, y: b),
// zero where a pixel does not replay the entry.
struct PairOut {
  F2 dm2, ux, uy, uz, dak, e0, e1, e2;
};

// Both pixels' contributions of a conic, non-thin record (rec[3].w flags
// clear of RF_GENERAL | RF_ANISO); same results as two bwd_pixel calls.
template <int FAM>
__device__ __forceinline__ bool bwd_pair(BwdPix& A, BwdPix& B, const float4* rec, const float4* bf,
                                         int idx, const ModelDev& m, float cutoff, float inv_f,
                                         float gam, PairOut& o, unsigned long long& ntest,
                                         bool count) {
  const bool actA = idx <= A.last, actB = idx <= B.last;
  if (!(actA || actB)) {
    o = PairOut{};  // zero contributions (the warp's moments may still be formed)
    return false;
  }
  if (count) ntest += (unsigned)actA + (unsigned)actB;
  TestOut2 t;
  bool okA = actA, okB = actB;
  ray_peak_test2(rec[0], rec[1], rec[2], rec[3], A.pc, B.pc, cutoff, t, okA, okB);
  if (!(okA || okB)) {
    o = PairOut{};
    return false;
  }
  const F2 alpha = t.alpha, kern = t.kern, araw = t.araw, rD = t.rD, u = t.u, v = t.v;
  const F2 ddy = t.ddy, hy{A.pc.hy, B.pc.hy};
  const float ddx = t.ddx;
  const float4 r2 = rec[2];
  F2 c0, c1, c2;
  emission2(rec[4], rec[5], rec[6], A.pc, B.pc, c0, c1, c2);
  const F2 E0{fmaxf(c0.x, 0.f), fmaxf(c0.y, 0.f)};
  const F2 E1{fmaxf(c1.x, 0.f), fmaxf(c1.y, 0.f)};
  const F2 E2{fmaxf(c2.x, 0.f), fmaxf(c2.y, 0.f)};
  // the saturating splat moves the loss only through its emission
  const bool satA = okA && A.sat && idx == A.last, satB = okB && B.sat && idx == B.last;
  const bool nA = okA && !satA, nB = okB && !satB;
  const F2 s_0{A.s0, B.s0}, s_1{A.s1, B.s1}, s_2{A.s2, B.s2};
  // E_k (the saturating splat's emission, else the background) comes from
  // the forward's cache, bit-identical to this entry's emission on the
  // saturating one (same rounded ops), so no per-entry update is needed
  const F2 ek0{A.ek0, B.ek0}, ek1{A.ek1, B.ek1}, ek2{A.ek2, B.ek2};
  const F2 sdE = fma2(s_0, sub2(E0, ek0), fma2(s_1, sub2(E1, ek1), mul2(s_2, sub2(E2, ek2))));
  // state in front of splat i, recovered back to front (normal pixels only)
  F2 thi{A.thi, B.thi}, tlo{A.tlo, B.tlo};
  if constexpr (FAM != FAM_EXP) {
    F2 h = thi, l = tlo;
    df_add2(h, l, F2{-alpha.x, -alpha.y});
    if (nA) { A.thi = h.x; A.tlo = l.x; }
    if (nB) { B.thi = h.y; B.tlo = l.y; }
  }
  if constexpr (IsPFam<FAM>::value) {
    if (nA) A.P = (idx == A.ck) ? A.Pck : div_newton(A.P, __fsub_rn(1.0f, alpha.x));
    if (nB) B.P = (idx == B.ck) ? B.Pck : div_newton(B.P, __fsub_rn(1.0f, alpha.y));
  }
  F2 fp, g;
  if constexpr (FAM == FAM_SOFT) {
    // weight_g<FAM_SOFT> on the pair (σ split by sign; MUFU ops per lane)
    const F2 x = mul2(f2(m.c), sub2(sub2(f2(1.0f), F2{A.thi, B.thi}), F2{A.tlo, B.tlo}));
    const F2 nx = mul2(F2{-fabsf(x.x), -fabsf(x.y)}, f2(1.4426950408889634f));
    const F2 t{ex2_approx(nx.x), ex2_approx(nx.y)};
    const F2 op = add2(f2(1.0f), t);
    const F2 r{__fdividef(1.0f, op.x), __fdividef(1.0f, op.y)};
    const F2 tr = mul2(t, r);
    const F2 sig{x.x >= 0.f ? r.x : tr.x, x.y >= 0.f ? r.y : tr.y};
    const F2 oms{x.x >= 0.f ? tr.x : r.x, x.y >= 0.f ? tr.y : r.y};
    g = mul2(f2(m.K), sig);
    fp = mul2(mul2(f2(-m.c), g), oms);
  } else {
    g = F2{weight_g<FAM>(m, A.thi, A.tlo, A.P, fp.x), weight_g<FAM>(m, B.thi, B.tlo, B.P, fp.y)};
  }
  const F2 wgt = mul2(alpha, g);
  const F2 carry{A.carry, B.carry};
  F2 da, nc;
  if constexpr (IsPFam<FAM>::value) {
    const F2 P{A.P, B.P};
    da = fma2(sdE, g, mul2(mul2(f2(-gam), P), carry));
    nc = fma2(sub2(f2(1.0f), alpha), carry, mul2(sdE, alpha));
  } else {
    da = fma2(sdE, g, carry);
    nc = fma2(mul2(sdE, alpha), fp, carry);
  }
  if (nA) A.carry = nc.x;
  if (nB) B.carry = nc.y;
  // dE = s·w for normal pixels, s·T̄_k for the saturating one
  // (zero for a pixel that does not replay the entry: its dE vanish)
  const F2 wt{satA ? A.tk : (okA ? wgt.x : 0.f), satB ? B.tk : (okB ? wgt.y : 0.f)};
  const F2 dE0 = mul2(s_0, wt), dE1 = mul2(s_1, wt), dE2 = mul2(s_2, wt);
  // zero for a clamped alpha (render.py:329) and for a pixel that does not
  // contribute (kern and alpha are finite there), so dm2 and dak need no mask
  const F2 dae{(!nA || araw.x >= ALPHA_MAX_F) ? 0.f : da.x,
               (!nB || araw.y >= ALPHA_MAX_F) ? 0.f : da.y};
  o.dm2 = mul2(mul2(f2(-0.5f), alpha), dae);
  o.dak = mul2(dae, kern);
  // whitened peak offset y = B̃ e, e = δ − ε h (bwd_pixel's conic branch)
  const float dxn = ddx * inv_f;
  const F2 dyn = mul2(ddy, f2(inv_f));
  const F2 Ahx = mul2(f2(r2.x), u);
  const F2 Ahy = fma2(f2(r2.x * r2.y), u, mul2(f2(r2.w), v));
  const F2 eps = mul2(fma2(f2(dxn), Ahx, mul2(dyn, Ahy)), rD);
  const F2 qx = fma2(eps, f2(-A.pc.hx), f2(dxn));
  const F2 qy = fma2(eps, F2{-hy.x, -hy.y}, dyn);
  // qz = −ε: the B̃ z-column enters negated.  Not masked: every moment of
  // the offset carries the factor dm2, zero for a pixel that does not
  // contribute, and the offset itself is finite (D > 0 for any pixel).
  o.ux = fma2(f2(bf[0].x), qx, fma2(f2(bf[0].y), qy, mul2(f2(-bf[0].z), eps)));
  o.uy = fma2(f2(bf[1].x), qx, fma2(f2(bf[1].y), qy, mul2(f2(-bf[1].z), eps)));
  o.uz = fma2(f2(bf[2].x), qx, fma2(f2(bf[2].y), qy, mul2(f2(-bf[2].z), eps)));
  // SH moments use dE_c·[E_c > 0] (render.py:340-341)
  o.e0 = sel2(c0.x > 0.f, c0.y > 0.f, dE0);
  o.e1 = sel2(c1.x > 0.f, c1.y > 0.f, dE1);
  o.e2 = sel2(c2.x > 0.f, c2.y > 0.f, dE2);
  return true;
}

// Warp transpose-reduce scratch: 12 moment-pair rows of 72 floats per warp
// (row p = moments (2p, 2p+1) of all 32 lanes; lanes 16-31 shifted by 4
// banks so the 8-byte pair stores and the 16-byte row loads are conflict free)
constexpr int RED_HALF = 36;                    // lanes 16-31's pairs start here (bank shift)
constexpr int RED_ROW = 2 * RED_HALF;           // one row per moment pair
constexpr int RED_WARP = (NMOM / 2) * RED_ROW;  // floats per warp

// Per list entry: each thread adds its two pixels' 24 moments, the warp
// transposes them through `red` (12 moment-pair rows) and lane m < NMOM
// returns moment m summed over the warp's 64 pixels.
__device__ __forceinline__ float warp_moments(const PairOut& po, const PixelConst& pa,
                                              const PixelConst& pb, float* red, int lane,
                                              float Y0) {
  // warp transpose-reduce through shared memory (moment-pair rows)
  const F2 a = mul2(po.dm2, po.ux), b = mul2(po.dm2, po.uy), c = mul2(po.dm2, po.uz);
  // moment pairs (2p, 2p+1) as one 8-byte store; rows 9 and 10 are unused
  float v[NMOM];
  v[0] = fmaf(a.x, po.ux.x, a.y * po.ux.y);
  v[1] = fmaf(a.x, po.uy.x, a.y * po.uy.y);
  v[2] = fmaf(a.x, po.uz.x, a.y * po.uz.y);
  v[3] = fmaf(b.x, po.uy.x, b.y * po.uy.y);
  v[4] = fmaf(b.x, po.uz.x, b.y * po.uz.y);
  v[5] = fmaf(c.x, po.uz.x, c.y * po.uz.y);
  v[6] = a.x + a.y;
  v[7] = b.x + b.y;
  v[8] = c.x + c.y;
  v[9] = 0.f;
  v[10] = 0.f;
  v[11] = po.dak.x + po.dak.y;
  v[12] = (po.e0.x + po.e0.y) * Y0;
  v[13] = fmaf(po.e0.x, pa.Y1, po.e0.y * pb.Y1);
  v[14] = fmaf(po.e0.x, pa.Y2, po.e0.y * pb.Y2);
  v[15] = fmaf(po.e0.x, pa.Y3, po.e0.y * pb.Y3);
  v[16] = (po.e1.x + po.e1.y) * Y0;
  v[17] = fmaf(po.e1.x, pa.Y1, po.e1.y * pb.Y1);
  v[18] = fmaf(po.e1.x, pa.Y2, po.e1.y * pb.Y2);
  v[19] = fmaf(po.e1.x, pa.Y3, po.e1.y * pb.Y3);
  v[20] = (po.e2.x + po.e2.y) * Y0;
  v[21] = fmaf(po.e2.x, pa.Y1, po.e2.y * pb.Y1);
  v[22] = fmaf(po.e2.x, pa.Y2, po.e2.y * pb.Y2);
  v[23] = fmaf(po.e2.x, pa.Y3, po.e2.y * pb.Y3);
  float2* col = reinterpret_cast<float2*>(red + (lane < 16 ? 2 * lane : RED_HALF + 2 * (lane - 16)));
#pragma unroll
  for (int q = 0; q < NMOM / 2; ++q) col[q * (RED_ROW / 2)] = make_float2(v[2 * q], v[2 * q + 1]);
  __syncwarp();
  // lane 2p sums moments (2p, 2p+1) over lanes 0-15, lane 2p+1 over
  // lanes 16-31 (packed adds), then each keeps its own moment and
  // takes the partner's half of it
  F2 part = f2(0.f);
  if (lane < NMOM) {
    const float4* row =
        reinterpret_cast<const float4*>(red + (lane >> 1) * RED_ROW + (lane & 1) * RED_HALF);
    F2 t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 r = row[i];
      t[i] = add2(F2{r.x, r.y}, F2{r.z, r.w});
    }
    part = add2(add2(add2(t[0], t[1]), add2(t[2], t[3])), add2(add2(t[4], t[5]), add2(t[6], t[7])));
  }
  const float other = __shfl_xor_sync(0xffffffffu, (lane & 1) ? part.x : part.y, 1);
  const float sum = ((lane & 1) ? part.y : part.x) + other;
  return sum;
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
  st.ek0 = bg0;
  st.ek1 = bg1;
  st.ek2 = bg2;
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
    st.ek0 = cache.e_k[3 * pix + 0];  // saturating splat's emission, else the background
    st.ek1 = cache.e_k[3 * pix + 1];
    st.ek2 = cache.e_k[3 * pix + 2];
  }
  st.carry = 0.f;  // Θ (τ-family) or U (P-family), seed-contracted
}

}  // namespace nxs
