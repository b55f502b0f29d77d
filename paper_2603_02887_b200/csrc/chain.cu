// K5: per-Gaussian moments -> parameter gradients, fp64.
//
// Replaces the reference chain (pkg/src/nexsplat/render.py:326-341, with
// quat_rot_jacobian primitives.py:67-93).  With m2 = ΔᵀN'Δ / hᵀA'h
// (SURVEY §8.0.5/§8.0.7), for any parameter direction θ̇:
//   Σ_px dm2 ∂m2/∂θ = Σ_ij Ṅ'_ij S_ij − 2 Σ_ij N'_ij ċ_i S_j − Σ_kl Ȧ'_kl H_kl
// where S_ij = Σ dm2 Δ_iΔ_j/D, S_i = Σ dm2 Δ_i/D, H_kl = Σ dm2 m2 h_k h_l/D
// are the moments K4 accumulated (dm2 = -½·α·dα).  Each parameter (μ 3,
// s 3, q 4) is one forward-mode tangent through (A', b') -> (N', c).  The
// quaternion gradient is projected orthogonally to the unit quaternion
// without a 1/|q| factor, exactly as render.py:339 does.
#include "nxs_internal.cuh"

namespace nxs {

struct ChainGeo {
  double M[9];    // Rc^T R
  double Ap[9];   // camera-frame inverse covariance
  double bp[3];   // camera-frame centre offset
  double Ab[3];   // A' b'
  double bAb;
  double Np[3];   // N'00, N'01, N'11 (pixel units)
};

struct Mom {
  double S00, S01, S11, Sx, Sy, H00, H01, H02, H11, H12, H22;
};

// contribution of one tangent (dAp symmetric 3x3, dbp 3-vector)
__device__ __forceinline__ double tangent_contract(const ChainGeo& G, const Mom& mo,
                                                   const double* dAp, const double* dbp,
                                                   double f) {
  double dAb[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    dAb[i] = dAp[3 * i + 0] * G.bp[0] + dAp[3 * i + 1] * G.bp[1] + dAp[3 * i + 2] * G.bp[2] +
             G.Ap[3 * i + 0] * dbp[0] + G.Ap[3 * i + 1] * dbp[1] + G.Ap[3 * i + 2] * dbp[2];
  const double dbAb = dbp[0] * G.Ab[0] + dbp[1] * G.Ab[1] + dbp[2] * G.Ab[2] +
                      G.bp[0] * dAb[0] + G.bp[1] * dAb[1] + G.bp[2] * dAb[2];
  const double if2 = 1.0 / (f * f);
  const double dN00 = (dbAb * G.Ap[0] + G.bAb * dAp[0] - 2.0 * dAb[0] * G.Ab[0]) * if2;
  const double dN01 =
      (dbAb * G.Ap[1] + G.bAb * dAp[1] - dAb[0] * G.Ab[1] - G.Ab[0] * dAb[1]) * if2;
  const double dN11 = (dbAb * G.Ap[4] + G.bAb * dAp[4] - 2.0 * dAb[1] * G.Ab[1]) * if2;
  const double bz = G.bp[2];
  const double dcx = f * (dbp[0] * bz - G.bp[0] * dbp[2]) / (bz * bz);
  const double dcy = f * (dbp[1] * bz - G.bp[1] * dbp[2]) / (bz * bz);
  double acc = dN00 * mo.S00 + 2.0 * dN01 * mo.S01 + dN11 * mo.S11;
  acc -= 2.0 * ((G.Np[0] * dcx + G.Np[1] * dcy) * mo.Sx + (G.Np[1] * dcx + G.Np[2] * dcy) * mo.Sy);
  acc -= dAp[0] * mo.H00 + 2.0 * dAp[1] * mo.H01 + 2.0 * dAp[2] * mo.H02 + dAp[4] * mo.H11 +
         2.0 * dAp[5] * mo.H12 + dAp[8] * mo.H22;
  return acc;
}

__global__ void k_chain(const float* __restrict__ centers, const float* __restrict__ scales,
                        const float* __restrict__ quats, int C, int64_t P,
                        const uint32_t* __restrict__ order, CamDev cam,
                        const double* __restrict__ moments, float* __restrict__ g_centers,
                        float* __restrict__ g_scales, float* __restrict__ g_quats,
                        float* __restrict__ g_opac, float* __restrict__ g_sh) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P) return;
  const double* mm = moments + r * NMOM;
  double mv[NMOM];
  bool any = false;
#pragma unroll
  for (int k = 0; k < NMOM; ++k) {
    mv[k] = mm[k];
    any |= (mv[k] != 0.0);
  }
  if (!any) return;
  const int64_t g = order[r];

  // SH and opacity need no geometry
  g_opac[g] += (float)mv[11];
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < C; ++k) g_sh[(g * 3 + c) * C + k] += (float)mv[12 + 4 * c + k];

  const Mom mo{mv[0], mv[1], mv[2], mv[3], mv[4], mv[5], mv[6], mv[7], mv[8], mv[9], mv[10]};
  if (mo.S00 == 0.0 && mo.S01 == 0.0 && mo.S11 == 0.0 && mo.Sx == 0.0 && mo.Sy == 0.0 &&
      mo.H22 == 0.0)
    return;

  double qw = quats[4 * g + 0], qx = quats[4 * g + 1], qy = quats[4 * g + 2], qz = quats[4 * g + 3];
  const double nq = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  const double w = qw / nq, x = qx / nq, y = qy / nq, z = qz / nq;
  double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                 2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                 2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
  const double s[3] = {scales[3 * g + 0], scales[3 * g + 1], scales[3 * g + 2]};
  const double is[3] = {1.0 / (s[0] * s[0]), 1.0 / (s[1] * s[1]), 1.0 / (s[2] * s[2])};
  ChainGeo G;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      G.M[3 * i + j] = cam.R[0 + i] * R[0 + j] + cam.R[3 + i] * R[3 + j] + cam.R[6 + i] * R[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      G.Ap[3 * i + j] = G.M[3 * i + 0] * is[0] * G.M[3 * j + 0] +
                        G.M[3 * i + 1] * is[1] * G.M[3 * j + 1] +
                        G.M[3 * i + 2] * is[2] * G.M[3 * j + 2];
  const double b[3] = {(double)centers[3 * g + 0] - cam.o[0], (double)centers[3 * g + 1] - cam.o[1],
                       (double)centers[3 * g + 2] - cam.o[2]};
  for (int i = 0; i < 3; ++i) G.bp[i] = cam.R[0 + i] * b[0] + cam.R[3 + i] * b[1] + cam.R[6 + i] * b[2];
  for (int i = 0; i < 3; ++i)
    G.Ab[i] = G.Ap[3 * i + 0] * G.bp[0] + G.Ap[3 * i + 1] * G.bp[1] + G.Ap[3 * i + 2] * G.bp[2];
  G.bAb = G.bp[0] * G.Ab[0] + G.bp[1] * G.Ab[1] + G.bp[2] * G.Ab[2];
  const double f = cam.f, if2 = 1.0 / (f * f);
  G.Np[0] = (G.bAb * G.Ap[0] - G.Ab[0] * G.Ab[0]) * if2;
  G.Np[1] = (G.bAb * G.Ap[1] - G.Ab[0] * G.Ab[1]) * if2;
  G.Np[2] = (G.bAb * G.Ap[4] - G.Ab[1] * G.Ab[1]) * if2;

  const double zero3[3] = {0.0, 0.0, 0.0};
  double dAp[9];
  // μ_k: b' moves along row k of Rc (b' = Rc^T (μ - o))
  for (int k = 0; k < 3; ++k) {
    for (int i = 0; i < 9; ++i) dAp[i] = 0.0;
    const double dbp[3] = {cam.R[3 * k + 0], cam.R[3 * k + 1], cam.R[3 * k + 2]};
    g_centers[3 * g + k] += (float)tangent_contract(G, mo, dAp, dbp, f);
  }
  // s_k: A' += -2/s_k^3 M[:,k] M[:,k]^T
  for (int k = 0; k < 3; ++k) {
    const double coef = -2.0 / (s[k] * s[k] * s[k]);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) dAp[3 * i + j] = coef * G.M[3 * i + k] * G.M[3 * j + k];
    g_scales[3 * g + k] += (float)tangent_contract(G, mo, dAp, zero3, f);
  }
  // q_k: dR = J_k (primitives.py:67-93), dM = Rc^T dR, dA' = dM Λ M^T + M Λ dM^T
  double gq[4];
  for (int k = 0; k < 4; ++k) {
    double J[9];
    if (k == 0) {
      const double t[9] = {0, -z, y, z, 0, -x, -y, x, 0};
      for (int i = 0; i < 9; ++i) J[i] = 2.0 * t[i];
    } else if (k == 1) {
      const double t[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
      for (int i = 0; i < 9; ++i) J[i] = 2.0 * t[i];
    } else if (k == 2) {
      const double t[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
      for (int i = 0; i < 9; ++i) J[i] = 2.0 * t[i];
    } else {
      const double t[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
      for (int i = 0; i < 9; ++i) J[i] = 2.0 * t[i];
    }
    double dM[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        dM[3 * i + j] = cam.R[0 + i] * J[0 + j] + cam.R[3 + i] * J[3 + j] + cam.R[6 + i] * J[6 + j];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double v = 0.0;
        for (int l = 0; l < 3; ++l)
          v += is[l] * (dM[3 * i + l] * G.M[3 * j + l] + G.M[3 * i + l] * dM[3 * j + l]);
        dAp[3 * i + j] = v;
      }
    gq[k] = tangent_contract(G, mo, dAp, zero3, f);
  }
  const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
  g_quats[4 * g + 0] += (float)(gq[0] - w * dot);
  g_quats[4 * g + 1] += (float)(gq[1] - x * dot);
  g_quats[4 * g + 2] += (float)(gq[2] - y * dot);
  g_quats[4 * g + 3] += (float)(gq[3] - z * dot);
}

void launch_chain(const float* centers, const float* scales, const float* quats, int C, int64_t P,
                  const uint32_t* order, const CamDev& cam, const double* moments,
                  float* g_centers, float* g_scales, float* g_quats, float* g_opac, float* g_sh,
                  cudaStream_t s) {
  if (P == 0) return;
  k_chain<<<(unsigned)((P + 127) / 128), 128, 0, s>>>(centers, scales, quats, C, P, order, cam,
                                                      moments, g_centers, g_scales, g_quats,
                                                      g_opac, g_sh);
}

}  // namespace nxs
