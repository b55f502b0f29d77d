// K5: per-Gaussian moments -> parameter gradients, fp64.  Only ranks the
// backward touched are read; their moments are re-zeroed here, so the
// buffer is clean for the next backward without a separate clear.
//
// Replaces the reference chain (pkg/src/nexsplat/render.py:326-341, with
// quat_rot_jacobian primitives.py:67-93).  K4 accumulated per rank, in the
// Gaussian's own whitened frame (y = Λ^{1/2} u, u = Rᵀ(t·d − b) the
// kernel-peak offset), U' = Σ_px dm2 · y yᵀ and V' = Σ_px dm2 · y; here
//     U = S U' S = Σ_px dm2 · u uᵀ   (6 values, symmetric 3x3)
//     V = S V'   = Σ_px dm2 · u      (3 values)
// with dm2 = -½·α·dα (dα zeroed where α is clamped, render.py:327).  By the
// envelope theorem (primitives.py:245-249) m2 = diffᵀ A diff differentiated
// at fixed peak depth, so with Λ = diag(s⁻²):
//     ∂L/∂μ   = Σ dm2 · (−2 A diff) = −2 R Λ V                (render.py:331)
//     ∂L/∂s_k = Σ dm2 · (−2 u_k² / s_k³) = −2 U_kk / s_k³     (render.py:332-334)
//     ∂L/∂q_k = Σ dm2 · 2 diffᵀ J_k Λ u = 2 Σ_ab (RᵀJ_k)_ab Λ_b U_ab
//               then projected orthogonally to the unit quaternion without a
//               1/|q| factor, exactly as render.py:336-339 does.
#include "nxs_internal.cuh"

namespace nxs {

__global__ void k_chain(const float* __restrict__ scales, const float* __restrict__ quats, int C,
                        int64_t P, const uint32_t* __restrict__ order,
                        double* __restrict__ moments, uint8_t* __restrict__ touched,
                        float* __restrict__ g_centers,
                        float* __restrict__ g_scales, float* __restrict__ g_quats,
                        float* __restrict__ g_opac, float* __restrict__ g_sh,
                        uint32_t* __restrict__ tlist, unsigned long long* __restrict__ tcount) {
  nxs_pdl_enter();
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = r < P && touched[r];
  const int64_t g = act ? (int64_t)order[r] : 0;
  if (tlist && g_centers) {
    // the Gaussians this backward wrote (any order): the touched-row export,
    // appended one atomic per warp (a per-Gaussian atomic on the one
    // counter serialised the kernel)
    const unsigned m = __ballot_sync(0xffffffffu, act);
    if (m) {
      const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
      unsigned long long at = 0;
      if (lane == leader) at = atomicAdd(tcount, (unsigned long long)__popc(m));
      at = __shfl_sync(0xffffffffu, at, leader);
      if (act) tlist[at + __popc(m & ((1u << lane) - 1u))] = (uint32_t)g;
    }
  }
  if (!act) return;
  // read this rank's moments and leave the buffer zeroed for the next backward
  double* mm = moments + r * NMOM;
  double mv[NMOM];
#pragma unroll
  for (int k = 0; k < NMOM; ++k) {
    mv[k] = mm[k];
    mm[k] = 0.0;
  }
  touched[r] = 0;
  if (!g_centers) return;  // clear only (a discarded speculative backward)

  // Gradients accumulate atomically: views sharing one gradient buffer may
  // run their chains concurrently on different streams (include/nxs.h).
  // opacity and SH need no geometry
  atomicAdd(g_opac + g, (float)mv[11]);
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < C; ++k) atomicAdd(g_sh + (g * 3 + c) * C + k, (float)mv[12 + 4 * c + k]);

  bool geo = false;
#pragma unroll
  for (int k = 0; k < 9; ++k) geo |= (mv[k] != 0.0);
  if (!geo) return;
  // K4 accumulated the whitened offset y = Λ^{1/2} u: U = S U' S, V = S V'
  const double s[3] = {scales[3 * g + 0], scales[3 * g + 1], scales[3 * g + 2]};
  const double U[9] = {mv[0] * s[0] * s[0], mv[1] * s[0] * s[1], mv[2] * s[0] * s[2],
                       mv[1] * s[0] * s[1], mv[3] * s[1] * s[1], mv[4] * s[1] * s[2],
                       mv[2] * s[0] * s[2], mv[4] * s[1] * s[2], mv[5] * s[2] * s[2]};
  const double V[3] = {mv[6] * s[0], mv[7] * s[1], mv[8] * s[2]};

  const double qw = quats[4 * g + 0], qx = quats[4 * g + 1], qy = quats[4 * g + 2],
               qz = quats[4 * g + 3];
  const double nq = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  const double w = qw / nq, x = qx / nq, y = qy / nq, z = qz / nq;
  const double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                       2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                       2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
  const double L[3] = {1.0 / (s[0] * s[0]), 1.0 / (s[1] * s[1]), 1.0 / (s[2] * s[2])};

  const double LV[3] = {L[0] * V[0], L[1] * V[1], L[2] * V[2]};
  for (int i = 0; i < 3; ++i)
    atomicAdd(g_centers + 3 * g + i,
              (float)(-2.0 * (R[3 * i + 0] * LV[0] + R[3 * i + 1] * LV[1] + R[3 * i + 2] * LV[2])));
  for (int k = 0; k < 3; ++k)
    atomicAdd(g_scales + 3 * g + k, (float)(-2.0 * U[4 * k] / (s[k] * s[k] * s[k])));

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
    double acc = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        const double om = R[0 + a] * J[0 + b] + R[3 + a] * J[3 + b] + R[6 + a] * J[6 + b];
        acc += om * L[b] * U[3 * a + b];
      }
    gq[k] = 2.0 * acc;
  }
  const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
  atomicAdd(g_quats + 4 * g + 0, (float)(gq[0] - w * dot));
  atomicAdd(g_quats + 4 * g + 1, (float)(gq[1] - x * dot));
  atomicAdd(g_quats + 4 * g + 2, (float)(gq[2] - y * dot));
  atomicAdd(g_quats + 4 * g + 3, (float)(gq[3] - z * dot));
}

void launch_chain(const float* scales, const float* quats, int C, int64_t P, const uint32_t* order,
                  double* moments, uint8_t* touched, float* g_centers, float* g_scales,
                  float* g_quats, float* g_opac, float* g_sh, uint32_t* tlist,
                  unsigned long long* tcount, cudaStream_t s) {
  if (P == 0) return;
  // touched ranks lie below the processed ranks (P here): small blocks
  // spread their fp64 work over every SM
  nxs_launch(k_chain, (unsigned)((P + 63) / 64), 64, 0, s, scales, quats, C, P, order, moments, touched,
                                                    g_centers, g_scales, g_quats, g_opac, g_sh,
                                                    tlist, tcount);
}

}  // namespace nxs
