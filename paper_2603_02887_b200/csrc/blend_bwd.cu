// K4: path-replay backward, one 16x16 tile per 256-thread block.
//
// Replaces the reference replay and closed-form adjoints
// (pkg/src/nexsplat/render.py:_backward_sweep 220-324) and produces the
// per-Gaussian moments the parameter chain (render.py:326-341, done by K5
// in chain.cu) needs.
//
// Each pixel walks its tile list BACK TO FRONT from the last live splat the
// forward cached, with O(1) state (unified adjoint):
//   τ-family (linear, quadratic, softplus, power law):
//       dα_i = s·ΔE_i g_i + Θ,      Θ += s·ΔE_i α_i f'(τ̄_i)
//   P-family (exponential γ=1, blended/vicini γ):
//       dα_i = s·ΔE_i g_i − γ P_i U, U = s·ΔE_i α_i + (1−α_i) U
// with s the adjoint seed, ΔE_i = E_i − E_k (E_k: saturating splat's
// emission, else background), τ̄_i recovered exactly from the double-float
// cache and P_i = P_{i+1}/(1−α_i) (checkpointed where P underflows).  The
// saturating splat only receives dE = s·T̄_k (render.py:313-314).  No
// per-sample state is stored.
//
// Reduction: per list entry each warp reduces its 32 pixels' 24 moments
// with a transpose-reduce (31 shuffles), lanes 0..23 add into a per-entry
// shared accumulator, and after each batch the block flushes the non-zero
// sums with one fp64 atomic each into the per-rank moment buffer.
#include "blend_common.cuh"

namespace nxs {

constexpr int BWD_BATCH = 128;  // list entries staged per batch

// v[32] per lane -> returns Σ_lanes v[lane]
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const bool upper = (lane & step) != 0;
#pragma unroll
    for (int k = 0; k < step; ++k) {
      const float send = upper ? v[k] : v[k + step];
      const float keep = upper ? v[k + step] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, step);
    }
  }
  return v[0];
}

template <int FAM, bool COUNT>
__global__ void __launch_bounds__(TILE_PIX)
    k_blend_bwd(const float4* __restrict__ records, const uint32_t* __restrict__ pairs,
                const int2* __restrict__ ranges, CamDev cam, ModelDev m, float cutoff,
                double near_plane, float bg0, float bg1, float bg2,
                const float* __restrict__ seed, PixCache cache,
                double* __restrict__ moments, Counters* __restrict__ cnt) {
  __shared__ float4 s_rec[BWD_BATCH][REC_F4];
  __shared__ uint32_t s_rank[BWD_BATCH];
  __shared__ float s_acc[BWD_BATCH * NMOM];
  __shared__ int s_maxlast;

  const int tile = blockIdx.x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int px = tx * TILE + (tid & (TILE - 1)), py = ty * TILE + (tid >> 4);
  const bool inside = px < cam.W && py < cam.H;
  const PixelConst pc = pixel_setup(cam, px, py);
  const int pix = py * cam.W + px;

  int last = -1;
  bool sat = false;
  float tk = 0.f, thi = 0.f, tlo = 0.f, P = 1.f, Pck = 0.f;
  int ck = -1;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
  if (inside) {
    last = cache.last[pix];
    sat = cache.sat[pix] != 0;
    tk = cache.t_k[pix];
    thi = cache.tau_hi[pix];
    tlo = cache.tau_lo[pix];
    P = cache.P_end[pix];
    ck = cache.ck_idx[pix];
    Pck = cache.P_ck[pix];
    s0 = seed[3 * pix + 0];
    s1 = seed[3 * pix + 1];
    s2 = seed[3 * pix + 2];
  }
  float ek0 = bg0, ek1 = bg1, ek2 = bg2;
  float carry = 0.f;  // Θ (τ-family) or U (P-family), seed-contracted
  const float gam = (FAM == FAM_EXP) ? 1.0f : m.c;
  const float inv_f = (float)(1.0 / cam.f);
  unsigned long long ntest = 0, nent = 0;

  if (tid == 0) s_maxlast = -1;
  __syncthreads();
  if (last >= 0) atomicMax(&s_maxlast, last);
  __syncthreads();
  const int2 rg = ranges[tile];
  const int hi_end = s_maxlast + 1;

  for (int hi = hi_end; hi > rg.x; hi -= BWD_BATCH) {
    const int base = max(rg.x, hi - BWD_BATCH);
    const int n = hi - base;
    __syncthreads();
    if (tid < n) s_rank[tid] = pairs[base + tid];
    for (int k = tid; k < n * NMOM; k += TILE_PIX) s_acc[k] = 0.f;
    __syncthreads();
    for (int k = tid; k < n * 8; k += TILE_PIX) {
      const int e = k >> 3, part = k & 7;
      s_rec[e][part] = records[(size_t)s_rank[e] * REC_F4 + part];
    }
    __syncthreads();
    if (COUNT) nent += n;

    for (int j = n - 1; j >= 0; --j) {
      const int idx = base + j;
      float v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = 0.f;
      bool contrib = false;
      if (idx <= last) {
        if (COUNT) ++ntest;
        TestOut t;
        const bool gen = (__float_as_int(s_rec[j][3].w) & RF_GENERAL) != 0;  // block-uniform
        float gx = 0.f, gy = 0.f, gz = 0.f;
        bool ok;
        if (gen)
          ok = general_test(s_rec[j], cam, px, py, cutoff, near_plane, t, gx, gy, gz);
        else
          ok = ray_peak_test(s_rec[j][0], s_rec[j][1], s_rec[j][2], s_rec[j][3], pc, cutoff, t);
        if (ok) {
          contrib = true;
          const float alpha = t.alpha;
          float E0, E1, E2;
          const int mask = emission(s_rec[j][4], s_rec[j][5], s_rec[j][6], pc, E0, E1, E2);
          float dE0, dE1, dE2;
          if (sat && idx == last) {
            // saturating splat: moves the loss only through its emission
            ek0 = E0;
            ek1 = E1;
            ek2 = E2;
            dE0 = s0 * tk;
            dE1 = s1 * tk;
            dE2 = s2 * tk;
          } else {
            // state in front of splat i, recovered back to front
            if constexpr (FAM != FAM_EXP) df_add(thi, tlo, -alpha);
            if constexpr (IsPFam<FAM>::value) {
              P = (idx == ck) ? Pck : __fdiv_rn(P, __fsub_rn(1.0f, alpha));
            }
            float fp;
            const float g = weight_g<FAM>(m, thi, tlo, P, fp);
            const float w = alpha * g;
            const float sdE = fmaf(s0, E0 - ek0, fmaf(s1, E1 - ek1, s2 * (E2 - ek2)));
            float da;
            if constexpr (IsPFam<FAM>::value) {
              da = fmaf(sdE, g, -gam * P * carry);
              carry = fmaf(1.0f - alpha, carry, sdE * alpha);
            } else {
              da = fmaf(sdE, g, carry);
              carry = fmaf(sdE * alpha, fp, carry);
            }
            dE0 = s0 * w;
            dE1 = s1 * w;
            dE2 = s2 * w;
            // chain moments (render.py:326-339 in the camera frame): by the
            // envelope theorem ∂m2/∂A' = diff'diff'ᵀ and ∂m2/∂b' = -2A'diff',
            // with the peak offset diff' = b'_z·e, e = δ - ε h, δ = Δ/f,
            // ε = δᵀA'h / D — all O(|δ|) terms, no cancellation against b'
            const float dae = (t.araw >= ALPHA_MAX_F) ? 0.f : da;
            const float dm2 = -0.5f * alpha * dae;
            float ex, ey, ez;
            if (gen) {  // world-frame diff (K5 knows the record kind)
              ex = gx;
              ey = gy;
              ez = gz;
            } else {
              const float4 r2 = s_rec[j][2];
              const float dxn = t.ddx * inv_f, dyn = t.ddy * inv_f;
              const float Ahx = r2.x * t.u;
              const float Ahy = fmaf(r2.x * r2.y, t.u, r2.w * t.v);
              const float eps = __fdividef(fmaf(dxn, Ahx, dyn * Ahy), t.D);
              ex = fmaf(-eps, pc.hx, dxn);
              ey = fmaf(-eps, pc.hy, dyn);
              ez = -eps;
            }
            const float wx = dm2 * ex, wy = dm2 * ey, wz = dm2 * ez;
            v[0] = wx * ex;
            v[1] = wx * ey;
            v[2] = wx * ez;
            v[3] = wy * ey;
            v[4] = wy * ez;
            v[5] = wz * ez;
            v[6] = wx;
            v[7] = wy;
            v[8] = wz;
            v[11] = dae * t.kern;
          }
          // SH moments dE_c·[E_c > 0]·Y_k (render.py:340-341)
          const float Y0 = (float)SH_C0;
          const float e0 = (mask & 1) ? dE0 : 0.f;
          const float e1 = (mask & 2) ? dE1 : 0.f;
          const float e2 = (mask & 4) ? dE2 : 0.f;
          v[12] = e0 * Y0;
          v[13] = e0 * pc.Y1;
          v[14] = e0 * pc.Y2;
          v[15] = e0 * pc.Y3;
          v[16] = e1 * Y0;
          v[17] = e1 * pc.Y1;
          v[18] = e1 * pc.Y2;
          v[19] = e1 * pc.Y3;
          v[20] = e2 * Y0;
          v[21] = e2 * pc.Y1;
          v[22] = e2 * pc.Y2;
          v[23] = e2 * pc.Y3;
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        const float r = transpose_reduce32(v, lane);
        if (lane < NMOM && r != 0.f) atomicAdd(&s_acc[j * NMOM + lane], r);
      }
    }
    __syncthreads();
    for (int k = tid; k < n * NMOM; k += TILE_PIX) {
      const float val = s_acc[k];
      if (val != 0.f) {
        const int e = k / NMOM;
        atomicAdd(&moments[(size_t)s_rank[e] * NMOM + (k - e * NMOM)], (double)val);
      }
    }
  }

  if (COUNT) {
    __shared__ unsigned long long s_cnt[2];
    __syncthreads();
    if (tid == 0) s_cnt[0] = s_cnt[1] = 0;
    __syncthreads();
    atomicAdd(&s_cnt[0], ntest);
    __syncthreads();
    if (tid == 0) {
      atomicAdd(&cnt->tests_bwd, s_cnt[0]);
      atomicAdd(&cnt->entries_bwd, nent);
    }
  }
}

template <int FAM>
static void launch_bwd_fam(bool count, int n_tiles, const float4* records, const uint32_t* pairs,
                           const int2* ranges, const CamDev& cam, const ModelDev& m,
                           float cutoff, double near_plane, const float* bg, const float* seed,
                           const PixCache& cache, double* moments, Counters* cnt,
                           cudaStream_t s) {
  if (count)
    k_blend_bwd<FAM, true><<<n_tiles, TILE_PIX, 0, s>>>(records, pairs, ranges, cam, m, cutoff,
                                                         near_plane, bg[0], bg[1], bg[2], seed,
                                                         cache, moments, cnt);
  else
    k_blend_bwd<FAM, false><<<n_tiles, TILE_PIX, 0, s>>>(records, pairs, ranges, cam, m, cutoff,
                                                          near_plane, bg[0], bg[1], bg[2], seed,
                                                          cache, moments, cnt);
}

void launch_blend_bwd(bool count, int n_tiles, const float4* records, const uint32_t* pairs,
                      const int2* ranges, const CamDev& cam, const ModelDev& m, float cutoff,
                      double near_plane, const float* bg, const float* seed,
                      const PixCache& cache, double* moments, Counters* cnt, cudaStream_t s) {
  if (n_tiles == 0) return;
#define NXS_BWD(F) \
  launch_bwd_fam<F>(count, n_tiles, records, pairs, ranges, cam, m, cutoff, near_plane, bg, seed, \
                    cache, moments, cnt, s)
  switch (m.fam) {
    case FAM_EXP: NXS_BWD(FAM_EXP); break;
    case FAM_LIN: NXS_BWD(FAM_LIN); break;
    case FAM_QUAD: NXS_BWD(FAM_QUAD); break;
    case FAM_BLEND: NXS_BWD(FAM_BLEND); break;
    case FAM_POW: NXS_BWD(FAM_POW); break;
    default: NXS_BWD(FAM_SOFT); break;
  }
#undef NXS_BWD
}

}  // namespace nxs
