// K5: per-Gaussian moments -> parameter gradients, fp64.
//
// Replaces the reference chain (pkg/src/nexsplat/render.py:326-341, with
// quat_rot_jacobian primitives.py:67-93).  K4 accumulated, in the camera
// frame and per rank,
//     X = Σ_px dm2 · e eᵀ   (6 values, symmetric 3x3)
//     Y = Σ_px dm2 · e      (3 values)
// with dm2 = -½·α·dα (dα zeroed where α is clamped, render.py:327) and
// e = diff'/b'_z the kernel-peak offset.  By the envelope theorem (the peak
// depth's own dependence drops out, primitives.py:245-249)
//     ∂m2/∂A' = diff' diff'ᵀ,   ∂m2/∂b' = -2 A' diff',
// so for any parameter tangent (Ȧ', ḃ')
//     Σ_px dm2 ∂m2/∂θ = b'_z² Σ_kl Ȧ'_kl X_kl − 2 b'_z ḃ'ᵀ A' Y.
// μ moves b' (= Rcᵀ(μ − o)); s and q move A' (= Rcᵀ R diag(s⁻²) Rᵀ Rc).
// The quaternion gradient is projected orthogonally to the unit quaternion
// without a 1/|q| factor, exactly as render.py:339 does.
#include "nxs_internal.cuh"

namespace nxs {

__global__ void k_chain(const float* __restrict__ centers, const float* __restrict__ scales,
                        const float* __restrict__ quats, int C, int64_t P,
                        const uint32_t* __restrict__ order,
                        const float4* __restrict__ records, CamDev cam,
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

  // opacity and SH need no geometry
  g_opac[g] += (float)mv[11];
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < C; ++k) g_sh[(g * 3 + c) * C + k] += (float)mv[12 + 4 * c + k];

  bool geo = false;
#pragma unroll
  for (int k = 0; k < 9; ++k) geo |= (mv[k] != 0.0);
  if (!geo) return;
  // symmetric X, vector Y
  const double X[9] = {mv[0], mv[1], mv[2], mv[1], mv[3], mv[4], mv[2], mv[4], mv[5]};
  const double Y[3] = {mv[6], mv[7], mv[8]};

  const double qw = quats[4 * g + 0], qx = quats[4 * g + 1], qy = quats[4 * g + 2],
               qz = quats[4 * g + 3];
  const double nq = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  const double w = qw / nq, x = qx / nq, y = qy / nq, z = qz / nq;
  const double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                       2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                       2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
  const double s[3] = {scales[3 * g + 0], scales[3 * g + 1], scales[3 * g + 2]};
  const double is[3] = {1.0 / (s[0] * s[0]), 1.0 / (s[1] * s[1]), 1.0 / (s[2] * s[2])};
  // conic records: camera frame (F = Rc, M = Rcᵀ R, κ = b'_z);
  // general records: world frame (F = I, M = R, κ = 1), moments of diff itself
  const bool gen = (__float_as_int(records[r * REC_F4 + 3].w) & RF_GENERAL) != 0;
  double F[9];
  for (int i = 0; i < 9; ++i) F[i] = gen ? ((i % 4 == 0) ? 1.0 : 0.0) : cam.R[i];
  double M[9], Ap[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = F[0 + i] * R[0 + j] + F[3 + i] * R[3 + j] + F[6 + i] * R[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      Ap[3 * i + j] = M[3 * i + 0] * is[0] * M[3 * j + 0] + M[3 * i + 1] * is[1] * M[3 * j + 1] +
                      M[3 * i + 2] * is[2] * M[3 * j + 2];
  const double b[3] = {(double)centers[3 * g + 0] - cam.o[0],
                       (double)centers[3 * g + 1] - cam.o[1],
                       (double)centers[3 * g + 2] - cam.o[2]};
  const double bz = gen ? 1.0 : cam.R[2] * b[0] + cam.R[5] * b[1] + cam.R[8] * b[2];
  const double bz2 = bz * bz;

  // μ: ∂L/∂b' = -2 b'_z A'Y, ∂L/∂μ = Rc ∂L/∂b'
  double AY[3];
  for (int i = 0; i < 3; ++i) AY[i] = Ap[3 * i + 0] * Y[0] + Ap[3 * i + 1] * Y[1] + Ap[3 * i + 2] * Y[2];
  for (int k = 0; k < 3; ++k)
    g_centers[3 * g + k] +=
        (float)(-2.0 * bz * (F[3 * k + 0] * AY[0] + F[3 * k + 1] * AY[1] + F[3 * k + 2] * AY[2]));

  // s_k: Ȧ' = -2/s_k³ M_k M_kᵀ  ->  b'_z² (-2/s_k³) M_kᵀ X M_k
  for (int k = 0; k < 3; ++k) {
    double Xm[3];
    for (int i = 0; i < 3; ++i)
      Xm[i] = X[3 * i + 0] * M[0 + k] + X[3 * i + 1] * M[3 + k] + X[3 * i + 2] * M[6 + k];
    const double mXm = M[0 + k] * Xm[0] + M[3 + k] * Xm[1] + M[6 + k] * Xm[2];
    g_scales[3 * g + k] += (float)(bz2 * (-2.0 / (s[k] * s[k] * s[k])) * mXm);
  }

  // q_k: Ṙ = J_k (primitives.py:67-93), Ṁ = Rcᵀ Ṙ, Ȧ' = Ṁ Λ Mᵀ + M Λ Ṁᵀ
  //      Σ Ȧ'⊙X = 2 Σ_l is_l (Ṁ_{:,l})ᵀ X M_{:,l}
  double XM[9];  // X M, column l = X M_{:,l}
  for (int i = 0; i < 3; ++i)
    for (int l = 0; l < 3; ++l)
      XM[3 * i + l] = X[3 * i + 0] * M[0 + l] + X[3 * i + 1] * M[3 + l] + X[3 * i + 2] * M[6 + l];
  double gq[4];
  for (int k = 0; k < 4; ++k) {
    double t[9];
    if (k == 0) {
      const double v[9] = {0, -z, y, z, 0, -x, -y, x, 0};
      for (int i = 0; i < 9; ++i) t[i] = 2.0 * v[i];
    } else if (k == 1) {
      const double v[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
      for (int i = 0; i < 9; ++i) t[i] = 2.0 * v[i];
    } else if (k == 2) {
      const double v[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
      for (int i = 0; i < 9; ++i) t[i] = 2.0 * v[i];
    } else {
      const double v[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
      for (int i = 0; i < 9; ++i) t[i] = 2.0 * v[i];
    }
    double acc = 0.0;
    for (int l = 0; l < 3; ++l) {
      double col = 0.0;  // (Ṁ_{:,l})ᵀ (X M)_{:,l}, Ṁ_il = Σ_k Rc_ki J_kl
      for (int i = 0; i < 3; ++i) {
        const double dMil = F[0 + i] * t[0 + l] + F[3 + i] * t[3 + l] + F[6 + i] * t[6 + l];
        col += dMil * XM[3 * i + l];
      }
      acc += is[l] * col;
    }
    gq[k] = bz2 * 2.0 * acc;
  }
  const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
  g_quats[4 * g + 0] += (float)(gq[0] - w * dot);
  g_quats[4 * g + 1] += (float)(gq[1] - x * dot);
  g_quats[4 * g + 2] += (float)(gq[2] - y * dot);
  g_quats[4 * g + 3] += (float)(gq[3] - z * dot);
}

void launch_chain(const float* centers, const float* scales, const float* quats, int C, int64_t P,
                  const uint32_t* order, const float4* records, const CamDev& cam,
                  const double* moments,
                  float* g_centers, float* g_scales, float* g_quats, float* g_opac, float* g_sh,
                  cudaStream_t s) {
  if (P == 0) return;
  k_chain<<<(unsigned)((P + 127) / 128), 128, 0, s>>>(centers, scales, quats, C, P, order,
                                                      records, cam, moments, g_centers, g_scales, g_quats,
                                                      g_opac, g_sh);
}

}  // namespace nxs
