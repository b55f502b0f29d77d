// K3: forward compositing, one 16x16 tile per 256-thread block.
//
// Replaces the reference per-pixel loop (pkg/src/nexsplat/render.py:
// _forward_sweep 147-217: live/sat_now/go, clamp, overdraw, finalize) for
// the global depth order (reference chunk_size=1, SURVEY §8.0.6 Mode G).
//
// Per batch of 64 list entries the block stages the projected records
// (8 threads per 128-B record, coalesced 16-B cp.async copies, double
// buffered so the next batch loads while this one is composited);
// every thread then walks the batch front to back for its pixel with the
// carry in registers and leaves once saturated or capped; the block leaves
// when all its pixels have.  Numerics (SURVEY R10 + §8.0.4):
//   * remaining transmittance T_rem is carried instead of cum (exp: P;
//     blended: closed form; others: T_rem -= w) and saturation is w >= T_rem;
//   * the optical depth τ̄ is an exact double-float sum, so the backward can
//     subtract its way back to every τ̄_i bit-exactly;
//   * the per-pixel cache (last live position, τ̄_end, P_end, t_k, P
//     checkpoint) is all the back-to-front backward needs.
#include <type_traits>

#include "blend_common.cuh"

namespace nxs {

#ifndef NXS_FWD_BATCH
#define NXS_FWD_BATCH 128
#endif
constexpr int FWD_BATCH = NXS_FWD_BATCH;  // list entries per staged batch
#ifndef NXS_FWD_MINB
#define NXS_FWD_MINB 3
#endif

template <int FAM, bool COUNT, bool THETA>
__global__ void __launch_bounds__(TILE_PIX, NXS_FWD_MINB)
    k_blend_fwd(const float4* __restrict__ records, const uint32_t* __restrict__ pairs,
                const int2* __restrict__ ranges, const int32_t* __restrict__ cum_in,
                int32_t* __restrict__ cum_out, uint8_t* __restrict__ active,
                unsigned int* __restrict__ n_active, bool resume, bool save, CamDev cam,
                ModelDev m,
                int max_splats, float cutoff, double near_plane, float bg0, float bg1, float bg2,
                float* __restrict__ rgb, int32_t* __restrict__ overdraw,
                float* __restrict__ residual, PixCache cache, PixResume rs,
                unsigned long long* __restrict__ need_rank, int32_t* __restrict__ tile_last,
                Counters* __restrict__ cnt) {
  nxs_pdl_enter();
  const int tile = blockIdx.x;
  if (!active[tile]) return;  // every pixel of the tile finished in an earlier phase
  // two 64-entry record buffers: the next batch streams in (cp.async)
  // while the current one is composited
  __shared__ float4 s_rec[2][FWD_BATCH][REC_F4];

  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int tid = threadIdx.x;
  // warp footprint: 16x2 rows, or a compact 8x4 block for the exponential
  // family, whose pixels walk long lists (8x4: exponential fwd -3.5 %,
  // softplus +1 %)
  const bool w8 = FAM == FAM_EXP;
  const int px = tx * TILE + (w8 ? ((tid >> 5) & 1) * 8 + (tid & 7) : (tid & (TILE - 1)));
  const int py = ty * TILE + (w8 ? (tid >> 6) * 4 + ((tid >> 3) & 3) : (tid >> 4));
  const bool inside = px < cam.W && py < cam.H;
  const PixelConst pc = pixel_setup(cam, px, py);

  float rad0 = 0.f, rad1 = 0.f, rad2 = 0.f;
  float thi = 0.f, tlo = 0.f;  // exact τ̄
  float P = 1.f;               // transparency product Π(1-α)
  float Trem = 1.f;            // 1 - cum
  int count = 0, last = -1;
  bool sat = false;
  float ek0 = bg0, ek1 = bg1, ek2 = bg2, tk = 0.f;
  float sea0 = 0.f, sea1 = 0.f, sea2 = 0.f, sa = 0.f;  // reference theta0 sums
  int ck = -1;
  float Pck = 0.f;
  unsigned long long ntest = 0;
  const int pix = py * cam.W + px;
  if (resume && inside) {  // carry of the previous depth phase
    rad0 = rs.rad[3 * pix + 0];
    rad1 = rs.rad[3 * pix + 1];
    rad2 = rs.rad[3 * pix + 2];
    Trem = rs.trem[pix];
    count = rs.count[pix];
    if (THETA) {
      sea0 = rs.sea[3 * pix + 0];
      sea1 = rs.sea[3 * pix + 1];
      sea2 = rs.sea[3 * pix + 2];
      sa = rs.sa[pix];
    }
    last = cache.last[pix];
    sat = cache.sat[pix] != 0;
    tk = cache.t_k[pix];
    thi = cache.tau_hi[pix];
    tlo = cache.tau_lo[pix];
    P = cache.P_end[pix];
    ck = cache.ck_idx[pix];
    Pck = cache.P_ck[pix];
    ek0 = cache.e_k[3 * pix + 0];
    ek1 = cache.e_k[3 * pix + 1];
    ek2 = cache.e_k[3 * pix + 2];
  }
  bool done = !inside || sat || count >= max_splats;
  const int count0 = count;

  const int2 rg = ranges[tile];
  const int vbase = cum_in[tile] - rg.x;  // list position -> virtual per-tile index
  auto stage = [&](int buf, int base) {
    const int n = min(FWD_BATCH, rg.y - base);
    NXS_CHECK(n > 0 && n <= FWD_BATCH && base >= rg.x);
    for (int k = tid; k < n * REC_F4; k += TILE_PIX) {
      const int e = k >> 3, part = k & 7;
      cp_async16(&s_rec[buf][e][part], records + (size_t)pairs[base + e] * REC_F4 + part);
    }
    cp_async_commit();
  };
  int dpos = -1;  // list position of the entry that finished this pixel
  // One list entry (record rj at list position lpos): the ray-peak test and,
  // on a hit, the composite.  Returns true when the pixel is finished.
  auto entry = [&](const float4* rj, int lpos, auto gen_tag) -> bool {
    constexpr bool GEN = decltype(gen_tag)::value;
    if (COUNT) ++ntest;
    TestOut tn;
    bool ok;
    if (GEN && (__float_as_int(rj[3].w) & RF_GENERAL)) {  // (uniform over the block)
      float gx, gy, gz, tpk;
      ok = general_test(rj, cam, px, py, cutoff, near_plane, tn, gx, gy, gz, tpk);
    } else {
      ok = ray_peak_test(rj[0], rj[1], rj[2], rj[3], pc, cutoff, tn);
    }
    if (!ok) return false;
    float E0, E1, E2;
    emission(rj[4], rj[5], rj[6], pc, E0, E1, E2);
    const float alpha = tn.alpha;
    const int idx = vbase + lpos;
    float fp;
    const float g = weight_g<FAM>(m, thi, tlo, P, fp);
    const float wr = alpha * g;
    const bool satnow = (FAM == FAM_EXP) ? false : (wr >= Trem);
    const int cb = count;
    ++count;
    last = idx;
    if (satnow) {
      rad0 = fmaf(Trem, E0, rad0);
      rad1 = fmaf(Trem, E1, rad1);
      rad2 = fmaf(Trem, E2, rad2);
      ek0 = E0;
      ek1 = E1;
      ek2 = E2;
      tk = Trem;
      sat = true;
      done = true;
      dpos = lpos;
      return true;
    }
    rad0 = fmaf(wr, E0, rad0);
    rad1 = fmaf(wr, E1, rad1);
    rad2 = fmaf(wr, E2, rad2);
    if (THETA && cb >= 1) {
      sea0 = fmaf(alpha, E0, sea0);
      sea1 = fmaf(alpha, E1, sea1);
      sea2 = fmaf(alpha, E2, sea2);
      sa += alpha;
    }
    if constexpr (FAM != FAM_EXP) df_add(thi, tlo, alpha);
    if constexpr (IsPFam<FAM>::value) {
      const float Pn = __fmul_rn(P, __fsub_rn(1.0f, alpha));
      if (Pn < P_FLOOR && ck < 0) {
        ck = idx;
        Pck = P;
      }
      P = Pn;
    }
    if constexpr (FAM == FAM_EXP) {
      Trem = P;
    } else if constexpr (FAM == FAM_BLEND) {
      Trem = fmaf(1.0f - m.c, __fsub_rn(__fsub_rn(1.0f, thi), tlo), m.c * P);
    } else {
      Trem = __fsub_rn(Trem, wr);
    }
    if (count >= max_splats) {
      done = true;
      dpos = lpos;
      return true;
    }
    return false;
  };
  {
  if (rg.x < rg.y) stage(0, rg.x);
  int buf = 0;
  for (int base = rg.x; base < rg.y; base += FWD_BATCH, buf ^= 1) {
    const int n = min(FWD_BATCH, rg.y - base);
    if (base + FWD_BATCH < rg.y) {
      stage(buf ^ 1, base + FWD_BATCH);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    // (the barrier also tells whether this batch holds a near-plane record:
    // almost never, so the common walk carries no per-entry flag test)
    const bool gen_batch =
        __syncthreads_or(tid < n && (__float_as_int(s_rec[buf][tid][3].w) & RF_GENERAL));
    float4(*s_cur)[REC_F4] = s_rec[buf];
    if (!done) {
      if (gen_batch) {
        for (int j = 0; j < n; ++j)
          if (entry(s_cur[j], base + j, std::true_type{})) break;
      } else {
        for (int j = 0; j < n; ++j)
          if (entry(s_cur[j], base + j, std::false_type{})) break;
      }
    }
    // all threads are past buffer `buf` before the next iteration refills it
    if (__syncthreads_count(!done) == 0) break;
  }
  }
  cp_async_wait<0>();
  __shared__ int s_dpos, s_last;
  if (tid == 0) s_dpos = s_last = -1;
  const int still = __syncthreads_count(!done);
  if (still == 0 && need_rank && dpos >= 0) atomicMax(&s_dpos, dpos);
  {  // the tile's last replayed position: K4 sizes its batches from it
    const int wl = __reduce_max_sync(0xffffffffu, last);
    if ((tid & 31) == 0 && wl >= 0) atomicMax(&s_last, wl);
  }
  __syncthreads();
  if (tid == 0) {
    tile_last[tile] = s_last;
    active[tile] = still > 0 ? 1 : 0;
    cum_out[tile] = cum_in[tile] + (rg.y - rg.x);
    if (still > 0) atomicAdd(n_active, 1u);
    // the last rank this finished tile needed (the list is in rank order)
    else if (need_rank && s_dpos >= 0) atomicMax(need_rank, (unsigned long long)pairs[s_dpos]);
  }

  if (COUNT) {
    __shared__ unsigned long long s_cnt[2];
    if (tid == 0) s_cnt[0] = s_cnt[1] = 0;
    __syncthreads();
    atomicAdd(&s_cnt[0], ntest);
    atomicAdd(&s_cnt[1], (unsigned long long)(count - count0));
    __syncthreads();
    if (tid == 0) {
      atomicAdd(&cnt->tests_fwd, s_cnt[0]);
      atomicAdd(&cnt->composited, s_cnt[1]);
    }
  }

  if (!inside) return;
  const float res = sat ? 0.f : Trem;  // render.py:210
  rgb[3 * pix + 0] = fmaf(bg0, res, rad0);
  rgb[3 * pix + 1] = fmaf(bg1, res, rad1);
  rgb[3 * pix + 2] = fmaf(bg2, res, rad2);
  overdraw[pix] = count;
  residual[pix] = res;
  cache.last[pix] = last;
  cache.sat[pix] = sat ? 1 : 0;
  cache.t_k[pix] = sat ? tk : res;  // render.py:212
  cache.tau_hi[pix] = thi;
  cache.tau_lo[pix] = tlo;
  cache.P_end[pix] = P;
  cache.ck_idx[pix] = ck;
  cache.P_ck[pix] = Pck;
  cache.e_k[3 * pix + 0] = ek0;
  cache.e_k[3 * pix + 1] = ek1;
  cache.e_k[3 * pix + 2] = ek2;
  if (THETA) {
    cache.theta0[3 * pix + 0] = sea0 - ek0 * sa;  // render.py:213
    cache.theta0[3 * pix + 1] = sea1 - ek1 * sa;
    cache.theta0[3 * pix + 2] = sea2 - ek2 * sa;
  }
  if (save && still > 0) {  // the tile continues in the next depth phase
    rs.rad[3 * pix + 0] = rad0;
    rs.rad[3 * pix + 1] = rad1;
    rs.rad[3 * pix + 2] = rad2;
    rs.trem[pix] = Trem;
    rs.count[pix] = count;
    if (THETA) {
      rs.sea[3 * pix + 0] = sea0;
      rs.sea[3 * pix + 1] = sea1;
      rs.sea[3 * pix + 2] = sea2;
      rs.sa[pix] = sa;
    }
  }
}


template <int FAM>
static void launch_fwd_fam(bool count, int n_tiles, const FwdArgs& a, const CamDev& cam,
                           const ModelDev& m, const PixCache& cache, const PixResume& rs,
                           Counters* cnt, cudaStream_t s) {
  auto k = count ? (a.theta0 ? k_blend_fwd<FAM, true, true> : k_blend_fwd<FAM, true, false>)
                 : (a.theta0 ? k_blend_fwd<FAM, false, true> : k_blend_fwd<FAM, false, false>);
  nxs_launch(k, n_tiles, TILE_PIX, 0, s, a.records, a.pairs, a.ranges, a.cum_in, a.cum_out, a.active,
                                 a.n_active, a.resume, a.save, cam, m, a.max_splats, a.cutoff,
                                 a.near_plane, a.bg[0], a.bg[1], a.bg[2], a.rgb, a.overdraw,
                                 a.residual, cache, rs, a.need_rank, a.tile_last, cnt);
}

void launch_blend_fwd(bool count, int n_tiles, const FwdArgs& a, const CamDev& cam,
                      const ModelDev& m, const PixCache& cache, const PixResume& rs,
                      Counters* cnt, cudaStream_t s) {
  if (n_tiles == 0) return;
  switch (m.fam) {
    case FAM_EXP: launch_fwd_fam<FAM_EXP>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_LIN: launch_fwd_fam<FAM_LIN>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_QUAD: launch_fwd_fam<FAM_QUAD>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_BLEND: launch_fwd_fam<FAM_BLEND>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_POW: launch_fwd_fam<FAM_POW>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    default: launch_fwd_fam<FAM_SOFT>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
  }
}

}  // namespace nxs
