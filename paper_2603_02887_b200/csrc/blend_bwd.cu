// K4: path-replay backward, one 16x16 tile per 128-thread block (2 pixels per thread).
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
// Reduction: per list entry each warp transposes its 32 lanes' 24 moments
// (each lane's two pixels already summed) through shared memory as 12
// moment-pair rows (12 eight-byte stores per lane); lanes 2p and 2p+1 sum
// pair row p over lanes 0-15 and 16-31 with packed adds (8 row loads, 15
// FADD2), swap halves with one shuffle, and add their moment into a
// per-entry shared accumulator.  After each batch the block flushes the
// non-zero sums with one fp64 atomic each into the per-rank moment buffer.
#include "bwd_common.cuh"

namespace nxs {

// list entries staged per batch: 64, or 32 in deterministic mode (its four
// per-warp accumulator rows would otherwise cost a block per SM)
__host__ __device__ constexpr int bwd_batch(bool det) { return det ? 32 : 64; }

// Two pixels per thread: a 128-thread block covers the 16x16 tile, thread t
// owning pixels t (rows 0-7) and t+128 (rows 8-15).  Each thread sums its
// two pixels' moments in registers before the warp reduction, halving the
// per-entry reductions, and the two independent pixel chains add ILP.
constexpr int BWD_THREADS = TILE_PIX / 2;
constexpr int BWD_WARPS = BWD_THREADS / 32;

// Shared-memory layout of one block (dynamic): staged records + B frames,
// their ranks, per-entry moment accumulators, and one 12x72-float transpose
// scratch per warp (row p = moment pair (2p, 2p+1) of all 32 lanes, lanes
// 16-31 shifted by 4 banks so the pair stores and the 16-B row loads are
// conflict free).
// Records, B frames and ranks are double-buffered: the next batch streams
// in with cp.async while the current one is replayed.
// Deterministic mode keeps one accumulator row per warp (summed in warp order
// at the flush) instead of shared float atomics from the four warps.
__host__ __device__ constexpr int acc_rows(bool det) { return det ? BWD_WARPS : 1; }
constexpr size_t bwd_smem(bool det) {
  return 2 * (sizeof(float4) * bwd_batch(det) * (REC_F4 + 3) + sizeof(uint32_t) * bwd_batch(det)) +
         sizeof(float) * bwd_batch(det) * NMOM * acc_rows(det) + sizeof(float) * RED_WARP * BWD_WARPS;
}


// Both pixels' contributions of list entry idx (lane x: pixel a, y: b), zero
// where a pixel does not contribute, so the moments need no separate
// masking: the packed pair step for conic non-thin records (uniform over the
// warp: every lane reads the same record), else the scalar per-pixel path.
template <int FAM, bool COUNT>
__device__ __forceinline__ bool entry_step(BwdPix (&st)[2], const float4* rec, const float4* bf,
                                           int idx, const CamDev& cam, const ModelDev& m,
                                           float cutoff, double near_plane, float inv_f,
                                           float gam, PairOut& po, unsigned long long& ntest) {
  if ((__float_as_int(rec[3].w) & (RF_GENERAL | RF_ANISO)) == 0)
    return bwd_pair<FAM>(st[0], st[1], rec, bf, idx, m, cutoff, inv_f, gam, po, ntest, COUNT);
  float dm2[2] = {0.f, 0.f}, ux[2] = {0.f, 0.f}, uy[2] = {0.f, 0.f}, uz[2] = {0.f, 0.f};
  float dak[2] = {0.f, 0.f}, e0[2] = {0.f, 0.f}, e1[2] = {0.f, 0.f}, e2[2] = {0.f, 0.f};
  bool contrib = false;
#pragma unroll
  for (int q = 0; q < 2; ++q)
    contrib |= bwd_pixel<FAM>(st[q], rec, bf, idx, cam, m, cutoff, near_plane, inv_f, gam, dm2[q],
                              ux[q], uy[q], uz[q], dak[q], e0[q], e1[q], e2[q], ntest, COUNT);
  po.dm2 = F2{dm2[0], dm2[1]};
  po.ux = F2{ux[0], ux[1]};
  po.uy = F2{uy[0], uy[1]};
  po.uz = F2{uz[0], uz[1]};
  po.dak = F2{dak[0], dak[1]};
  po.e0 = F2{e0[0], e0[1]};
  po.e1 = F2{e1[0], e1[1]};
  po.e2 = F2{e2[0], e2[1]};
  return contrib;
}

#ifndef NXS_BWD_MINB
#define NXS_BWD_MINB 4
#endif
template <int FAM, bool COUNT, bool DET>
__global__ void __launch_bounds__(BWD_THREADS, NXS_BWD_MINB)
    k_blend_bwd(const float4* __restrict__ records, const float4* __restrict__ bframe,
                PhaseLists lists, CamDev cam, ModelDev m, float cutoff, double near_plane,
                float bg0, float bg1, float bg2, const float* __restrict__ seed, PixCache cache,
                double* __restrict__ moments, uint8_t* __restrict__ touched,
                Counters* __restrict__ cnt) {
  nxs_pdl_enter();
  constexpr int BWD_BATCH = bwd_batch(DET);
  extern __shared__ float4 smem_dyn[];
  // [buffer][entry][part]
  float4(*s_rec2)[BWD_BATCH][REC_F4] = reinterpret_cast<float4(*)[BWD_BATCH][REC_F4]>(smem_dyn);
  float4(*s_bf2)[BWD_BATCH][3] =
      reinterpret_cast<float4(*)[BWD_BATCH][3]>(smem_dyn + 2 * BWD_BATCH * REC_F4);
  uint32_t(*s_rank2)[BWD_BATCH] =
      reinterpret_cast<uint32_t(*)[BWD_BATCH]>(smem_dyn + 2 * BWD_BATCH * (REC_F4 + 3));
  float* s_acc = reinterpret_cast<float*>(s_rank2 + 2);
  float* s_red = s_acc + BWD_BATCH * NMOM * acc_rows(DET);
#ifdef NXS_CHECKS
  __shared__ int s_maxlast;  // (checks the forward's per-tile last position)
#endif

  const int tile = blockIdx.x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int tid = threadIdx.x, lane = tid & 31;
  // a warp = one 8x8 pixel block (warps 2 across, 2 down), the thread's two
  // pixels on adjacent rows: the most compact warp footprint, so a warp's
  // live entries and their lanes overlap most (16x4 rows r, r+8: bwd +7 %)
  const int px = tx * TILE + ((tid >> 5) & 1) * 8 + (tid & 7);
  const int py0 = ty * TILE + (tid >> 6) * 8 + 2 * ((tid >> 3) & 3);
  BwdPix st[2];
  float* red = s_red + (tid >> 5) * RED_WARP;
  const float gam = (FAM == FAM_EXP) ? 1.0f : m.c;
  const float inv_f = (float)cam.inv_f;
  const float Y0 = (float)SH_C0;
  unsigned long long ntest = 0, nent = 0;

  // virtual per-tile list positions [0, vmax) are replayed: the forward
  // recorded the tile's largest, so the first batch streams in while the
  // pixels' cache loads are in flight, with no block-wide max
  const int vmax = lists.tile_last[tile] + 1;

  // phases back to front, each phase's segment back to front, in batches of
  // BWD_BATCH virtual positions [base, hi); batch (ph, hi) -> the next one
  auto seg_end = [&](int ph) {  // first batch end of phase ph (<= c0: empty)
    const int2 seg = lists.ranges[ph][tile];
    const int c0 = lists.cum[ph][tile];
    return seg.y > seg.x ? min(c0 + (seg.y - seg.x), vmax) : c0;
  };
  auto next_batch = [&](int& ph, int& hi) -> bool {  // from (ph, hi) (hi: current end)
    const int c0 = lists.cum[ph][tile];
    const int base = max(c0, hi - BWD_BATCH);
    if (base > c0) {
      hi = base;
      return true;
    }
    for (--ph; ph >= 0; --ph) {
      hi = seg_end(ph);
      if (hi > lists.cum[ph][tile]) return true;
    }
    return false;
  };
  auto stage = [&](int b, int ph, int hi) {
    const int c0 = lists.cum[ph][tile];
    const int base = max(c0, hi - BWD_BATCH);
    const int n = hi - base;
    const uint32_t* __restrict__ pr = lists.pairs[ph] + lists.ranges[ph][tile].x + (base - c0);
    for (int k = tid; k < n * 8; k += BWD_THREADS) {
      const int e = k >> 3, part = k & 7;
      const uint32_t rk = __ldg(pr + e);
      if (part == 0) s_rank2[b][e] = rk;
      cp_async16(&s_rec2[b][e][part], records + (size_t)rk * REC_F4 + part);
    }
    for (int k = tid; k < n * 3; k += BWD_THREADS) {
      const int e = k / 3, part = k - 3 * (k / 3);
      cp_async16(&s_bf2[b][e][part], bframe + (size_t)__ldg(pr + e) * 3 + part);
    }
    cp_async_commit();
  };

  int ph = lists.n - 1, hi = 0;
  bool have = false;
  for (; ph >= 0; --ph) {
    hi = seg_end(ph);
    if (hi > lists.cum[ph][tile]) {
      have = true;
      break;
    }
  }
  if (have) stage(0, ph, hi);
  bwd_load(st[0], cam, px, py0, cache, seed, bg0, bg1, bg2);
  bwd_load(st[1], cam, px, py0 + 1, cache, seed, bg0, bg1, bg2);
  const int mylast = max(st[0].last, st[1].last);
  // this warp's last live entry: the entries behind it skip the warp
  const int wlast = __reduce_max_sync(0xffffffffu, mylast);
#ifdef NXS_CHECKS
  if (tid == 0) s_maxlast = -1;
  __syncthreads();
  if (mylast >= 0) atomicMax(&s_maxlast, mylast);
  __syncthreads();
  NXS_CHECK(s_maxlast + 1 == vmax);
#endif
  int buf = 0;
  while (have) {
    const int c0 = lists.cum[ph][tile];
    const int base = max(c0, hi - BWD_BATCH);  // virtual
    const int n = hi - base;
    NXS_CHECK(n > 0 && n <= BWD_BATCH && base >= c0);
    int nph = ph, nhi = hi;
    const bool more = next_batch(nph, nhi);
    __syncthreads();  // every thread is past the previous batch's flush
    if (more) stage(buf ^ 1, nph, nhi);
    if (DET) {
      for (int w = 0; w < BWD_WARPS; ++w)
        for (int k = tid; k < n * NMOM; k += BWD_THREADS) s_acc[w * BWD_BATCH * NMOM + k] = 0.f;
    } else {
      for (int k = tid; k < n * NMOM; k += BWD_THREADS) s_acc[k] = 0.f;
    }
    if (more) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    float4(*s_rec)[REC_F4] = s_rec2[buf];
    float4(*s_bf)[3] = s_bf2[buf];
    const uint32_t* s_rank = s_rank2[buf];
    if (COUNT) nent += n;

      for (int j = min(n - 1, wlast - base); j >= 0; --j) {
        const int idx = base + j;
        NXS_CHECK(j >= 0 && j < n);
        // both pixels' contributions (lane x: pixel a, y: b), zero where a
        // pixel does not contribute, so the moments need no separate masking
        PairOut po;
        const bool contrib = entry_step<FAM, COUNT>(st, s_rec[j], s_bf[j], idx, cam, m, cutoff,
                                                    near_plane, inv_f, gam, po, ntest);
        if (__any_sync(0xffffffffu, contrib)) {
          const float sum = warp_moments(po, st[0].pc, st[1].pc, red, lane, Y0);
          if (lane < NMOM && sum != 0.f) {
            if (DET)  // this warp's own row: one writer per (entry, moment)
              s_acc[((tid >> 5) * BWD_BATCH + j) * NMOM + lane] = sum;
            else
              atomicAdd(&s_acc[j * NMOM + lane], sum);
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (DET) {
        // fixed-order sum over the warps; one partial per (tile, entry):
        // k_det_reduce adds them per rank in tile order
        const int64_t slot0 = lists.poff[ph] + lists.ranges[ph][tile].x + (base - c0);
        NXS_CHECK(lists.ranges[ph][tile].x + (base - c0) + n <= lists.ranges[ph][tile].y);
        for (int k = tid; k < n * NMOM; k += BWD_THREADS) {
          float val = s_acc[k];
#pragma unroll
          for (int w = 1; w < BWD_WARPS; ++w) val += s_acc[w * BWD_BATCH * NMOM + k];
          const int e = k / NMOM;
          // every replayed entry's row is written (zeros too): k_det_reduce
          // reads only positions below the tile's last, so no memset
          lists.partial[(slot0 + e) * NMOM + (k - e * NMOM)] = val;
          if (val != 0.f) touched[s_rank[e]] = 1;
        }
      } else {
        for (int k = tid; k < n * NMOM; k += BWD_THREADS) {
          const float val = s_acc[k];
          if (val != 0.f) {
            const int e = k / NMOM;
            atomicAdd(&moments[(size_t)s_rank[e] * NMOM + (k - e * NMOM)], (double)val);
            touched[s_rank[e]] = 1;  // K5 reads (and re-zeroes) touched ranks only
          }
        }
      }
    ph = nph;
    hi = nhi;
    have = more;
    buf ^= 1;
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

template <int FAM, bool DET>
static void launch_bwd_fam(bool count, int n_tiles, const float4* records, const float4* bframe,
                           const PhaseLists& lists, const CamDev& cam, const ModelDev& m,
                           float cutoff, double near_plane, const float* bg, const float* seed,
                           const PixCache& cache, double* moments, uint8_t* touched,
                           Counters* cnt, cudaStream_t s) {
  static unsigned long long attr_dev = 0;  // per instantiation and device
  once_per_device(attr_dev, [] {
    for (auto k : {k_blend_bwd<FAM, true, DET>, k_blend_bwd<FAM, false, DET>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd_smem(DET));
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared);
    }
  });
  auto k = count ? k_blend_bwd<FAM, true, DET> : k_blend_bwd<FAM, false, DET>;
  nxs_launch(k, n_tiles, BWD_THREADS, bwd_smem(DET), s, records, bframe, lists, cam, m, cutoff, near_plane,
                                               bg[0], bg[1], bg[2], seed, cache, moments, touched,
                                               cnt);
}

// Deterministic moments: per touched rank, the (tile, entry) partials of
// every tile of its rectangle, summed in fp64 in a fixed order: one warp per
// rank, lane l takes the rect's tiles l, l+32, ... (row-major; each found by
// binary search in that tile's rank-sorted list, phases in order), then a
// fixed shuffle tree adds the lanes.
__global__ void __launch_bounds__(256)
    k_det_reduce(int64_t P, const uint32_t* __restrict__ order, const int4* __restrict__ rects,
                 int tiles_x, PhaseLists lists, const uint8_t* __restrict__ touched,
                 double* __restrict__ moments) {
  nxs_pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= P || !touched[r]) return;  // (warp-uniform)
  const int4 rc = rects[order[r]];
  const int w = rc.z - rc.x + 1, nt = w * (rc.w - rc.y + 1);
  double acc[NMOM];
#pragma unroll
  for (int m = 0; m < NMOM; ++m) acc[m] = 0.0;
  for (int p = 0; p < lists.n; ++p)
    for (int k = lane; k < nt; k += 32) {
      const int2 rg = lists.ranges[p][(rc.y + k / w) * tiles_x + rc.x + k % w];
      int lo = rg.x, hi = rg.y;  // first position with rank >= r
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lists.pairs[p][mid] < (uint32_t)r) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= rg.y || lists.pairs[p][lo] != (uint32_t)r) continue;
      // entries past the tile's last replayed position were not written
      const int tile = (rc.y + k / w) * tiles_x + rc.x + k % w;
      if (lists.cum[p][tile] + (lo - rg.x) > lists.tile_last[tile]) continue;
      const float4* q = reinterpret_cast<const float4*>(lists.partial + (lists.poff[p] + lo) * NMOM);
#pragma unroll
      for (int i = 0; i < NMOM / 4; ++i) {
        const float4 v = q[i];
        acc[4 * i + 0] += (double)v.x;
        acc[4 * i + 1] += (double)v.y;
        acc[4 * i + 2] += (double)v.z;
        acc[4 * i + 3] += (double)v.w;
      }
    }
#pragma unroll
  for (int m = 0; m < NMOM; ++m)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[m] += __shfl_xor_sync(0xffffffffu, acc[m], o);
  if (lane < NMOM) {
    double v = acc[0];
#pragma unroll
    for (int m = 1; m < NMOM; ++m)
      if (lane == m) v = acc[m];
    moments[r * NMOM + lane] = v;
  }
}

void launch_det_reduce(int64_t P, const uint32_t* order, const int4* rects, int tiles_x,
                       const PhaseLists& lists, const uint8_t* touched, double* moments,
                       cudaStream_t s) {
  if (P <= 0) return;
  nxs_launch(k_det_reduce, (unsigned)((P * 32 + 255) / 256), 256, 0, s, P, order, rects, tiles_x, lists,
                                                               touched, moments);
}

void launch_blend_bwd(bool count, int n_tiles, const float4* records, const float4* bframe,
                      const PhaseLists& lists, const CamDev& cam, const ModelDev& m,
                      float cutoff, double near_plane, const float* bg, const float* seed,
                      const PixCache& cache, double* moments, uint8_t* touched, Counters* cnt,
                      cudaStream_t s) {
  if (n_tiles == 0) return;
#define NXS_BWD(F)                                                                            \
  (lists.partial ? launch_bwd_fam<F, true>(count, n_tiles, records, bframe, lists, cam, m, cutoff, \
                                           near_plane, bg, seed, cache, moments, touched, cnt, s) \
                 : launch_bwd_fam<F, false>(count, n_tiles, records, bframe, lists, cam, m,      \
                                            cutoff, near_plane, bg, seed, cache, moments, touched, \
                                            cnt, s))
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
