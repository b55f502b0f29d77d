// K3x / K4x: exact per-pixel order — the reference's default traversal
// (render(..., chunk_size=None): one chunk, every pixel stable-sorts its
// valid splats by peak depth t, ties by storage index; reference
// pkg/src/nexsplat/render.py:171, primitives.py:299).
//
// Tile lists are ordered by z_lo, a lower bound of t over every pixel where a
// Gaussian can be valid (min camera-z of its cutoff ellipsoid; t >= z_lo·|h|).
// K3x walks the list keeping, per pixel, a pending buffer of valid entries
// sorted by (t, index) in shared memory: before testing the next entry it
// commits (composites) every pending entry whose t is below that entry's
// bound z_lo·|h| — no later entry can precede it — and at the end of the
// list it commits the rest.  A full buffer is an overflow:
// counted and reported by the API, never silently accepted.  Each pixel's
// commit sequence (list positions) is stored for the backward.
//
// K4x replays every pixel's sequence back to front with the same unified
// adjoint as K4 (bwd_common.cuh).  Lanes of a warp step together through
// list positions (the warp processes the largest pending position each
// step, pixels whose next entry it is take part), so the 24 moments still
// reduce per warp through the shared-memory transpose before one fp64
// atomic per moment.
#include "bwd_common.cuh"

namespace nxs {

#ifdef NXS_XSTATS
// debug statistics of the exact-order forward (variant build only):
// [0] inserts, [1] shifted entries, [2] sum of pending count at insert,
// [3] commits, [4] list entries tested, [5..36] histogram of pending at insert
__device__ unsigned long long g_xstats[40];
#endif

#ifndef NXS_X_DEFER
#define NXS_X_DEFER 32  // commit once every active lane of the warp has one due (32/32)
#endif

// pending entries per pixel: 16 for the chunked order (a chunk flush empties
// the buffer; an overflow reruns with 32), 32 for the exact order
// list entries staged per batch: 64 with the 16-entry buffer, 32 with the
// 32-entry one (so that its alpha column still leaves two blocks per SM)
__host__ __device__ constexpr int xbatch(int xb) { return xb <= 16 ? 64 : 32; }
// records of the current and the previous batch stay staged (a ring of
// 2 batches): most commits are of recently tested entries
// the 16-entry buffer also keeps each pending entry's alpha (no re-test at
// commit); the 32-entry one re-tests so that two blocks still fit an SM
__host__ __device__ constexpr bool keeps_alpha(int xb) { return xb <= 32; }
constexpr size_t fwdx_smem(int xb) {
  return sizeof(float4) * 2 * xbatch(xb) * REC_F4 + sizeof(uint32_t) * 2 * xbatch(xb) +
         (sizeof(uint32_t) + sizeof(float) + sizeof(uint32_t)) * xbatch(xb) +
         (sizeof(float) + sizeof(int) + (keeps_alpha(xb) ? sizeof(float) : 0)) * xb * TILE_PIX;
}

struct FwdXPix {
  float rad0, rad1, rad2, thi, tlo, P, Trem, ek0, ek1, ek2, tk, sea0, sea1, sea2, sa, Pck;
  int count, ck;
  bool sat, done;
};

// one front-to-back compositing step (reference render.py:181-203) for the
// entry committed as the pixel's `count`-th live splat
template <int FAM>
__device__ __forceinline__ void composite(FwdXPix& s, const ModelDev& m, int max_splats,
                                          float alpha, float E0, float E1, float E2) {
  float fp;
  const float g = weight_g<FAM>(m, s.thi, s.tlo, s.P, fp);
  const float wr = alpha * g;
  const bool satnow = (FAM == FAM_EXP) ? false : (wr >= s.Trem);
  const int cb = s.count;
  ++s.count;
  if (satnow) {
    s.rad0 = fmaf(s.Trem, E0, s.rad0);
    s.rad1 = fmaf(s.Trem, E1, s.rad1);
    s.rad2 = fmaf(s.Trem, E2, s.rad2);
    s.ek0 = E0;
    s.ek1 = E1;
    s.ek2 = E2;
    s.tk = s.Trem;
    s.sat = true;
    s.done = true;
    return;
  }
  s.rad0 = fmaf(wr, E0, s.rad0);
  s.rad1 = fmaf(wr, E1, s.rad1);
  s.rad2 = fmaf(wr, E2, s.rad2);
  if (cb >= 1) {
    s.sea0 = fmaf(alpha, E0, s.sea0);
    s.sea1 = fmaf(alpha, E1, s.sea1);
    s.sea2 = fmaf(alpha, E2, s.sea2);
    s.sa += alpha;
  }
  if constexpr (FAM != FAM_EXP) df_add(s.thi, s.tlo, alpha);
  if constexpr (IsPFam<FAM>::value) {
    const float Pn = __fmul_rn(s.P, __fsub_rn(1.0f, alpha));
    if (Pn < P_FLOOR && s.ck < 0) {
      s.ck = cb;
      s.Pck = s.P;
    }
    s.P = Pn;
  }
  if constexpr (FAM == FAM_EXP) {
    s.Trem = s.P;
  } else if constexpr (FAM == FAM_BLEND) {
    s.Trem = fmaf(1.0f - m.c, __fsub_rn(__fsub_rn(1.0f, s.thi), s.tlo), m.c * s.P);
  } else {
    s.Trem = __fsub_rn(s.Trem, wr);
  }
  if (s.count >= max_splats) s.done = true;
}

// ray-peak test of one record for this pixel, with the peak depth t
__device__ __forceinline__ bool test_with_t(const float4* rec, const CamDev& cam, int px, int py,
                                            const PixelConst& pc, float hnorm, float cutoff,
                                            double near_plane, TestOut& t, float& tpk) {
  if (__float_as_int(rec[3].w) & RF_GENERAL) {
    float gx, gy, gz;
    return general_test(rec, cam, px, py, cutoff, near_plane, t, gx, gy, gz, tpk);
  }
  if (!ray_peak_test(rec[0], rec[1], rec[2], rec[3], pc, cutoff, t)) return false;
  // t = |h| (A'b')·h / hᵀA'h  (rec[7].xyz = A'b')
  const float4 ab = rec[7];
  tpk = hnorm * (__fmaf_rn(ab.x, pc.hx, __fmaf_rn(ab.y, pc.hy, ab.z)) * t.rD);
  return true;
}

template <int FAM, bool COUNT, int XBUF, bool CH>
__global__ void __launch_bounds__(TILE_PIX, XBUF <= 16 ? 3 : 2)
    k_blend_fwd_x(const float4* __restrict__ records, const uint32_t* __restrict__ pairs,
                  const int2* __restrict__ ranges, const float* __restrict__ zlo_rank,
                  const uint32_t* __restrict__ order, const uint32_t* __restrict__ rank_c,
                  int chunk, CamDev cam, ModelDev m, int max_splats,
                  float cutoff, double near_plane, float bg0, float bg1, float bg2,
                  float* __restrict__ rgb, int32_t* __restrict__ overdraw,
                  float* __restrict__ residual, PixCache cache, PixResume rs,
                  int32_t* __restrict__ seq, unsigned long long* __restrict__ overflow,
                  uint8_t* __restrict__ active, unsigned int* __restrict__ n_active, bool resume,
                  bool save, float* __restrict__ carry_t, int32_t* __restrict__ carry_r,
                  int32_t* __restrict__ carry_n, const float* __restrict__ end_bound,
                  unsigned long long* __restrict__ need_rank, Counters* __restrict__ cnt) {
  nxs_pdl_enter();
  constexpr int XBT = xbatch(XBUF);
  const int tile = blockIdx.x;
  if (active && !active[tile]) return;  // finished in an earlier depth phase
  extern __shared__ float4 smem_dyn[];
  float4(*s_ring)[REC_F4] = reinterpret_cast<float4(*)[REC_F4]>(smem_dyn);  // [2*XBT]
  uint32_t* s_ring_rank = reinterpret_cast<uint32_t*>(smem_dyn + 2 * XBT * REC_F4);
  uint32_t* s_rank = s_ring_rank + 2 * XBT;
  float* s_zlo = reinterpret_cast<float*>(s_rank + XBT);
  uint32_t* s_chunk = reinterpret_cast<uint32_t*>(s_zlo + XBT);
  // pending entries, [XBUF][TILE_PIX]: (t, list position) pairs moved as one
  // 8-byte word, and alpha; each thread addresses its own column
  float2* bq = reinterpret_cast<float2*>(s_chunk + XBT);
  float* ba = reinterpret_cast<float*>(bq + XBUF * TILE_PIX);

  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int tid = threadIdx.x;
  // a warp = one 8x4 pixel block (warps 2 across, 4 down): compact, so the
  // lanes' pending buffers fill alike (16x2: exact-order fwd +5 %)
  const int px = tx * TILE + ((tid >> 5) & 1) * 8 + (tid & 7),
            py = ty * TILE + (tid >> 6) * 4 + ((tid >> 3) & 3);
  const bool inside = px < cam.W && py < cam.H;
  const PixelConst pc = pixel_setup(cam, px, py);
  const float hnorm = sqrtf(__fmaf_rn(pc.hx, pc.hx, __fmaf_rn(pc.hy, pc.hy, 1.0f)));
  const int pix = py * cam.W + px;
  const size_t npix = (size_t)cam.W * cam.H;
  int32_t* myseq = seq + (inside ? pix : 0);  // [slot][pixel]: lanes read/write contiguously
  float2* myq = bq + tid;
  float* mya = ba + tid;

  FwdXPix s{};
  s.P = 1.f;
  s.Trem = 1.f;
  s.ek0 = bg0;
  s.ek1 = bg1;
  s.ek2 = bg2;
  s.ck = -1;
  if (resume && inside) {  // carry of the previous depth phase
    s.rad0 = rs.rad[3 * pix + 0];
    s.rad1 = rs.rad[3 * pix + 1];
    s.rad2 = rs.rad[3 * pix + 2];
    s.Trem = rs.trem[pix];
    s.count = rs.count[pix];
    s.sea0 = rs.sea[3 * pix + 0];
    s.sea1 = rs.sea[3 * pix + 1];
    s.sea2 = rs.sea[3 * pix + 2];
    s.sa = rs.sa[pix];
    s.sat = cache.sat[pix] != 0;
    s.tk = cache.t_k[pix];
    s.thi = cache.tau_hi[pix];
    s.tlo = cache.tau_lo[pix];
    s.P = cache.P_end[pix];
    s.ck = cache.ck_idx[pix];
    s.Pck = cache.P_ck[pix];
    s.ek0 = cache.e_k[3 * pix + 0];
    s.ek1 = cache.e_k[3 * pix + 1];
    s.ek2 = cache.e_k[3 * pix + 2];
  }
  s.done = !inside || s.sat || s.count >= max_splats;
  const bool done0 = s.done;
  int dpos = -1;  // list position being examined when the pixel finished
  const int count0 = s.count;
  // pending entries: a ring of XBUF slots, ascending by (t, index) from the
  // head; new entries (lists are in z_lo order) usually append at the tail
  int nb = 0, head = 0;
  float thead = __int_as_float(0x7f800000);  // t of the head entry (+inf when empty)
  if (resume && inside && carry_n && !s.done) {
    // pending entries carried over the phase end: list positions encode
    // ranks as -1 - rank (their records are read from global memory)
    nb = carry_n[pix];
    for (int i = 0; i < nb; ++i) {
      const int32_t rk = carry_r[(size_t)i * npix + pix];
      myq[i * TILE_PIX] = make_float2(carry_t[(size_t)i * npix + pix], __int_as_float(-1 - rk));
      if constexpr (keeps_alpha(XBUF)) {  // (the carry keeps t and rank only)
        float4 r[REC_F4];
        const float4* rec = records + (size_t)rk * REC_F4;
#pragma unroll
        for (int k = 0; k < REC_F4; ++k) r[k] = __ldg(rec + k);
        TestOut t;
        float tpk;
        test_with_t(r, cam, px, py, pc, hnorm, cutoff, near_plane, t, tpk);  // valid when carried
        mya[i * TILE_PIX] = t.alpha;
      }
    }
    if (nb > 0) thead = myq[0].x;
  }
  uint32_t cur_chunk = 0;  // chunk of the pending entries (chunked order)
  unsigned long long ntest = 0;
  // ties in t: storage index (one chunk, reference argsort over arange(n)) or
  // the centre-depth rank (chunked: stable argsort within the chunk's ids)
  auto tie_key = [&](uint32_t rank) -> uint32_t {
    const uint32_t g = order[rank];
    return rank_c ? rank_c[g] : g;
  };

  // commit the smallest pending entry: its alpha was kept at insertion, the
  // emission re-reads the record's SH words (staged ring, else L1/L2)
  int ring_lo = 0;  // list positions [ring_lo, current batch end) are staged
  // where a list position's rank is read: the pair list, or (exact order)
  // the tile's ranks staged in shared memory, indexed from lbase
  const uint32_t* lpairs = pairs;
  int lbase = 0;
  auto commit_front = [&]() {
    NXS_CHECK(nb > 0 && head >= 0 && head < XBUF);
    const int pos = __float_as_int(myq[head * TILE_PIX].y);
    const float alpha_kept = mya[head * TILE_PIX];
    head = (head + 1) & (XBUF - 1);
    --nb;
    thead = nb > 0 ? myq[head * TILE_PIX].x : __int_as_float(0x7f800000);
    // explicit shared / global branches (no generic loads)
    float4 r[REC_F4];
    constexpr int K0 = keeps_alpha(XBUF) ? 4 : 0, K1 = keeps_alpha(XBUF) ? 7 : REC_F4;
    uint32_t rank;
    if (pos >= ring_lo) {  // (carried entries have pos < 0 and take the global path)
      NXS_CHECK(pos >= ring_lo && pos < ring_lo + 2 * XBT);
      const float4* rec = s_ring[pos % (2 * XBT)];
      rank = s_ring_rank[pos % (2 * XBT)];
#pragma unroll
      for (int k = K0; k < K1; ++k) r[k] = rec[k];
    } else {
      rank = pos < 0 ? (uint32_t)(-1 - pos) : lpairs[pos - lbase];
      const float4* rec = records + (size_t)rank * REC_F4;
#pragma unroll
      for (int k = K0; k < K1; ++k) r[k] = __ldg(rec + k);
    }
    float alpha;
    if constexpr (keeps_alpha(XBUF)) {
      alpha = alpha_kept;
    } else {
      TestOut t;
      float tpk;
      test_with_t(r, cam, px, py, pc, hnorm, cutoff, near_plane, t, tpk);  // valid by construction
      alpha = t.alpha;
    }
    float E0, E1, E2;
    emission(r[4], r[5], r[6], pc, E0, E1, E2);
    NXS_CHECK(s.count >= 0 && s.count < max_splats);
    myseq[(size_t)s.count * npix] = (int32_t)rank;
#ifdef NXS_XSTATS
    atomicAdd(&g_xstats[3], 1ull);
#endif
    composite<FAM>(s, m, max_splats, alpha, E0, E1, E2);
  };

  const int2 rg = ranges[tile];
  if constexpr (!CH) {
  // exact order: every warp walks the tile list on its own, reading each
  // entry's rank, z_lo and test words through L1 (the block's 8 warps share
  // the lines), software-pipelined in registers (ranks two entries ahead,
  // the test words one ahead) — no staged batches, so no block barrier
  // between entries: the warps' pending-buffer work is uneven, and the
  // barriers made every warp wait for the slowest (softplus fwd 0.825 ->
  // 0.745 ms, exponential 10.56 -> 5.94 ms at C3; unstaged without the
  // prefetch was 12 % slower than staged for the saturating models)
  ring_lo = 0x7fffffff;  // (commits re-read their records the same way)
  {
    // the tile's ranks in shared memory (the staged ring's space, unused in
    // this order) when they fit: one barrier, then every read is an LDS
    constexpr int LIST_CAP = 2 * XBT * REC_F4 * 4;
    const int nlist = rg.y - rg.x;
    if (nlist <= LIST_CAP) {  // (block-uniform)
      uint32_t* s_list = reinterpret_cast<uint32_t*>(smem_dyn);
      for (int k = threadIdx.x; k < nlist; k += blockDim.x) s_list[k] = __ldg(pairs + rg.x + k);
      __syncthreads();
      lpairs = s_list;
      lbase = rg.x;
    }
  }
  if (!s.done) {
    // software pipeline: ranks two entries ahead, the test words and z_lo
    // of the next entry one ahead (in registers)
    auto ldrank = [&](int q) { return q < rg.y ? lpairs[q - lbase] : 0u; };
    uint32_t rk_cur = ldrank(rg.x), rk_n1 = ldrank(rg.x + 1);
    float4 c0, c1, c2, c3, c7;
    float zc;
    auto ldrec = [&](uint32_t r, float4& w0, float4& w1, float4& w2, float4& w3, float4& w7,
                     float& z) {
      const float4* g = records + (size_t)r * REC_F4;
      w0 = __ldg(g + 0); w1 = __ldg(g + 1); w2 = __ldg(g + 2); w3 = __ldg(g + 3);
      w7 = __ldg(g + 7);
      z = __ldg(zlo_rank + r);
    };
    ldrec(rk_cur, c0, c1, c2, c3, c7, zc);
    for (int pos = rg.x; pos < rg.y; ++pos) {
      const uint32_t rk = rk_cur;
      const float4 t0 = c0, t1 = c1, t2 = c2, t3 = c3, t7 = c7;
      const float bound = zc * hnorm;
      const uint32_t rk_n2 = ldrank(pos + 2);
      if (pos + 1 < rg.y) ldrec(rk_n1, c0, c1, c2, c3, c7, zc);
      rk_cur = rk_n1;
      rk_n1 = rk_n2;
      const float4* rec = records + (size_t)rk * REC_F4;  // (general records only)
#if NXS_X_DEFER > 0
      bool go_commit;
      {
        const unsigned am = __activemask();
        const unsigned want = __ballot_sync(am, nb > 0 && thead < bound);
        go_commit = (NXS_X_DEFER >= 32 ? want == am : __popc(want) * 32 >= NXS_X_DEFER * __popc(am)) ||
                    nb >= XBUF - 4;
      }
      while (go_commit && nb > 0 && thead < bound) {
#else
      while (nb > 0 && thead < bound) {
#endif
        commit_front();
        if (s.done) break;
      }
      if (s.done) {
        dpos = pos;
        break;
      }
      if (COUNT) ++ntest;
      TestOut t;
      float tpk;
      bool okt;
      if (__float_as_int(t3.w) & RF_GENERAL) {
        okt = test_with_t(rec, cam, px, py, pc, hnorm, cutoff, near_plane, t, tpk);
      } else {
        okt = ray_peak_test(t0, t1, t2, t3, pc, cutoff, t);
        tpk = hnorm * (__fmaf_rn(t7.x, pc.hx, __fmaf_rn(t7.y, pc.hy, t7.z)) * t.rD);
      }
      if (!okt) continue;
      if (nb == XBUF) {
        atomicAdd(overflow, 1ull);
        commit_front();
        if (s.done) {
          dpos = pos;
          break;
        }
      }
      int i = nb;
      uint32_t gid_new = 0xffffffffu;
      // slot pointers walked down the ring (no index arithmetic per shift)
      int f = (head + nb) & (XBUF - 1);
      while (i > 0) {
        const int e = (f - 1) & (XBUF - 1);
        const float2 qe = myq[e * TILE_PIX];
        if (!(qe.x >= tpk)) break;  // (NaN: stop, as before)
        if (qe.x == tpk) {
          if (gid_new == 0xffffffffu) gid_new = tie_key(rk);
          const int pe = __float_as_int(qe.y);
          if (!(tie_key(pe < 0 ? (uint32_t)(-1 - pe) : lpairs[pe - lbase]) > gid_new)) break;
        }
        myq[f * TILE_PIX] = qe;
        if constexpr (keeps_alpha(XBUF)) mya[f * TILE_PIX] = mya[e * TILE_PIX];
        f = e;
        --i;
      }
      NXS_CHECK(nb < XBUF && i >= 0 && i <= nb);
      myq[f * TILE_PIX] = make_float2(tpk, __int_as_float(pos));
      if constexpr (keeps_alpha(XBUF)) mya[f * TILE_PIX] = t.alpha;
      if (i == 0) thead = tpk;
      ++nb;
    }
  }
  } else {
    for (int base = rg.x; base < rg.y; base += XBT) {
      const int n = min(XBT, rg.y - base);
      NXS_CHECK(n > 0 && n <= XBT);
      __syncthreads();
      if (tid < n) {
        const uint32_t rk = pairs[base + tid];
        s_rank[tid] = rk;
        s_ring_rank[(base + tid) % (2 * XBT)] = rk;
        s_zlo[tid] = zlo_rank[rk];
        if (CH) s_chunk[tid] = rank_c[order[rk]] / (uint32_t)chunk;
      }
      __syncthreads();
      // stage this batch into the ring slot it maps to (positions are consecutive)
      for (int k = tid; k < n * REC_F4; k += TILE_PIX) {
        const int e = k >> 3, part = k & 7;
        s_ring[(base + e) % (2 * XBT)][part] = records[(size_t)s_rank[e] * REC_F4 + part];
      }
      ring_lo = max(rg.x, base - XBT);
      __syncthreads();
      if (!s.done) {
        for (int j = 0; j < n; ++j) {
          const float4* s_rec_j = s_ring[(base + j) % (2 * XBT)];
          // every remaining entry has t >= bound: pending entries below it are
          // final; a new chunk makes every pending entry final
          const bool next_chunk = CH && s_chunk[j] != cur_chunk;  // (exact order: one chunk)
          const float bound = s_zlo[j] * hnorm;
  #if NXS_X_DEFER > 0
          // Committable entries stay committable (every later entry's t is above
          // this bound), so the exact order may defer them until enough lanes of
          // the warp have one: the composite then runs with most lanes active.
          // (a new chunk commits everything pending at once: never deferred)
          bool go_commit = next_chunk;
          if (!go_commit) {
            const unsigned am = __activemask();
            const unsigned want = __ballot_sync(am, nb > 0 && thead < bound);
            go_commit = (NXS_X_DEFER >= 32 ? want == am : __popc(want) * 32 >= NXS_X_DEFER * __popc(am)) ||
                    nb >= XBUF - 4;
          }
          while (go_commit && nb > 0 && (next_chunk || thead < bound)) {
  #else
          while (nb > 0 && (next_chunk || thead < bound)) {
  #endif
            commit_front();
            if (s.done) break;
          }
          if (s.done) {
            dpos = base + j;
            break;
          }
          if (CH) cur_chunk = s_chunk[j];
          if (COUNT) ++ntest;
          TestOut t;
          float tpk;
          if (!test_with_t(s_rec_j, cam, px, py, pc, hnorm, cutoff, near_plane, t, tpk)) continue;
          if (nb == XBUF) {
            // overflow: the order is no longer guaranteed for this pixel
            atomicAdd(overflow, 1ull);
            commit_front();
            if (s.done) {
              dpos = base + j;
              break;
            }
          }
          // insert (t, index) keeping the ring ascending from the head
          const int pos = base + j;
          int i = nb;
          uint32_t gid_new = 0xffffffffu;
          // slot index walked down the ring (no index arithmetic per shift)
          int f = (head + nb) & (XBUF - 1);
          while (i > 0) {
            const int e = (f - 1) & (XBUF - 1);
            const float2 qe = myq[e * TILE_PIX];
            // the pending entry commits after the new one: shift it
            if (!(qe.x >= tpk)) break;
            if (qe.x == tpk) {
              if (gid_new == 0xffffffffu) gid_new = tie_key(s_rank[j]);
              const int pe = __float_as_int(qe.y);
              if (!(tie_key(pe < 0 ? (uint32_t)(-1 - pe) : pairs[pe]) > gid_new)) break;
            }
            myq[f * TILE_PIX] = qe;
            if constexpr (keeps_alpha(XBUF)) mya[f * TILE_PIX] = mya[e * TILE_PIX];
            f = e;
            --i;
          }
          NXS_CHECK(nb < XBUF && i >= 0 && i <= nb);
  #ifdef NXS_XSTATS
          atomicAdd(&g_xstats[0], 1ull);
          atomicAdd(&g_xstats[1], (unsigned long long)(nb - i));
          atomicAdd(&g_xstats[2], (unsigned long long)nb);
          atomicAdd(&g_xstats[5 + min(nb, 31)], 1ull);
  #endif
          myq[f * TILE_PIX] = make_float2(tpk, __int_as_float(pos));
          if constexpr (keeps_alpha(XBUF)) mya[f * TILE_PIX] = t.alpha;
          if (i == 0) thead = tpk;
          ++nb;
        }
      }
      if (__syncthreads_count(!s.done) == 0) break;
    }
  }
  // end of the list: everything pending is final, in order (one chunk, the
  // end of a chunk, or the last depth phase) — or, with a later phase, only
  // what lies in front of that phase's first z_lo; the rest is carried
  if (end_bound && save) {
    const float bound = *end_bound * hnorm;
    while (nb > 0 && !s.done && thead < bound) commit_front();
    if (inside && !s.done) {
      carry_n[pix] = nb;
      for (int i = 0; i < nb; ++i) {
        const int e = (head + i) & (XBUF - 1);
        const float2 qe = myq[e * TILE_PIX];
        const int pe = __float_as_int(qe.y);
        carry_t[(size_t)i * npix + pix] = qe.x;
        carry_r[(size_t)i * npix + pix] = pe < 0 ? -1 - pe : (int32_t)pairs[pe];
      }
    }
  } else {
    while (nb > 0 && !s.done) commit_front();
  }
  // finished by the commits at the list end: it needed the whole list
  if (s.done && !done0 && dpos < 0 && rg.y > rg.x) dpos = rg.y - 1;
  __shared__ int s_dpos;
  if (tid == 0) s_dpos = -1;
  const int still = __syncthreads_count(!s.done);
  if (still == 0 && need_rank && dpos >= 0) atomicMax(&s_dpos, dpos);
  __syncthreads();
  if (tid == 0) {
    if (active) {
      active[tile] = still > 0 ? 1 : 0;
      if (still > 0) atomicAdd(n_active, 1u);
    }
    // the last rank this finished tile needed (lists are in rank order)
    if (still == 0 && need_rank && s_dpos >= 0)
      atomicMax(need_rank, (unsigned long long)pairs[s_dpos]);
  }

  if (COUNT) {
    __shared__ unsigned long long s_cnt[2];
    __syncthreads();
    if (tid == 0) s_cnt[0] = s_cnt[1] = 0;
    __syncthreads();
    atomicAdd(&s_cnt[0], ntest);
    atomicAdd(&s_cnt[1], (unsigned long long)(s.count - count0));
    __syncthreads();
    if (tid == 0) {
      atomicAdd(&cnt->tests_fwd, s_cnt[0]);
      atomicAdd(&cnt->composited, s_cnt[1]);
    }
  }
  if (!inside) return;
  if (save && still > 0) {  // the tile continues in the next depth phase
    rs.rad[3 * pix + 0] = s.rad0;
    rs.rad[3 * pix + 1] = s.rad1;
    rs.rad[3 * pix + 2] = s.rad2;
    rs.trem[pix] = s.Trem;
    rs.count[pix] = s.count;
    rs.sea[3 * pix + 0] = s.sea0;
    rs.sea[3 * pix + 1] = s.sea1;
    rs.sea[3 * pix + 2] = s.sea2;
    rs.sa[pix] = s.sa;
  }
  const float res = s.sat ? 0.f : s.Trem;  // render.py:210
  rgb[3 * pix + 0] = fmaf(bg0, res, s.rad0);
  rgb[3 * pix + 1] = fmaf(bg1, res, s.rad1);
  rgb[3 * pix + 2] = fmaf(bg2, res, s.rad2);
  overdraw[pix] = s.count;
  residual[pix] = res;
  cache.last[pix] = s.count - 1;  // index into the commit sequence
  cache.sat[pix] = s.sat ? 1 : 0;
  cache.t_k[pix] = s.sat ? s.tk : res;
  cache.tau_hi[pix] = s.thi;
  cache.tau_lo[pix] = s.tlo;
  cache.P_end[pix] = s.P;
  cache.ck_idx[pix] = s.ck;
  cache.P_ck[pix] = s.Pck;
  cache.e_k[3 * pix + 0] = s.ek0;
  cache.e_k[3 * pix + 1] = s.ek1;
  cache.e_k[3 * pix + 2] = s.ek2;
  cache.theta0[3 * pix + 0] = s.sea0 - s.ek0 * s.sa;
  cache.theta0[3 * pix + 1] = s.sea1 - s.ek1 * s.sa;
  cache.theta0[3 * pix + 2] = s.sea2 - s.ek2 * s.sa;
}

// ---------------------------------------------------------------------------
// K4x
// ---------------------------------------------------------------------------
constexpr int XRED_STRIDE = 36;
// per warp: the transpose scratch, then two record slots (record + B frame,
// 11 float4) — the next step's record streams in while this one is replayed
constexpr int XREC_F4 = REC_F4 + 3;
constexpr size_t BWDX_WARP_FLOATS = NMOM * XRED_STRIDE + 2 * XREC_F4 * 4;
// (per block: one warp slot per warp; NP pixels per thread)
constexpr size_t bwdx_smem(int np) { return sizeof(float) * BWDX_WARP_FLOATS * (np == 1 ? 1 : TILE_PIX / np / 32); }

// Each warp step serves the largest pending rank over the warp's pixels; the
// pixels whose entry it is take part, and the warp reduces their moments.
// Chunked order (k_blend_bwd_x2): two pixels per thread (adjacent rows, a
// warp = one 8x8 block, a 128-thread block per tile, as K4), a thread adding
// both pixels' moments before the warp reduction.  Exact order
// (k_blend_bwd_x1): one pixel per thread (a warp = an 8x4 block: smaller
// footprints take fewer lock-step steps) and one warp per block, so a warp
// that finishes its steps frees its slot at once (the warps of a tile share
// nothing): exact-order bwd 0.715 -> 0.616 ms, 0.566 with 20 blocks per SM
// (NXS_X1_MINB); the chunked order's warps
// finish together and keep the two-pixel, four-warp blocks.

template <int FAM, bool COUNT, int XNP>
__device__ __forceinline__ void bwd_x_body(const float4* __restrict__ records, const float4* __restrict__ bframe,
                  const uint32_t* __restrict__ pairs, const int32_t* __restrict__ seq,
                  int max_splats, CamDev cam, ModelDev m, float cutoff, double near_plane,
                  float bg0, float bg1, float bg2, const float* __restrict__ seed,
                  PixCache cache, double* __restrict__ moments, uint8_t* __restrict__ touched,
                  Counters* __restrict__ cnt, int tile, int wid) {
  nxs_pdl_enter();
  extern __shared__ float smem_red[];
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  // (tid: the thread's index within the tile; its warp's shared slot is
  // threadIdx.x >> 5 of this block)
  const int lane = threadIdx.x & 31, tid = wid * 32 + lane;
  // a warp = one 8x8 pixel block, the thread's pixels on adjacent rows (as
  // K4); with one pixel per thread an 8x4 block (as K3x)
  const int px = tx * TILE + ((tid >> 5) & 1) * 8 + (tid & 7),
            py0 = XNP == 2 ? ty * TILE + (tid >> 6) * 8 + 2 * ((tid >> 3) & 3)
                           : ty * TILE + (tid >> 6) * 4 + ((tid >> 3) & 3);
  BwdPix st[XNP];
  const int32_t* myseq[XNP];
  int ptr[XNP];
  const size_t npix = (size_t)cam.W * cam.H;
#pragma unroll
  for (int q = 0; q < XNP; ++q) {
    const int py = py0 + q;
    bwd_load(st[q], cam, px, py, cache, seed, bg0, bg1, bg2);
    const bool inside = px < cam.W && py < cam.H;
    myseq[q] = seq + (inside ? (size_t)py * cam.W + px : 0);  // [slot][pixel]
    ptr[q] = st[q].last;  // commit index, back to front
  }
  float* red = smem_red + (threadIdx.x >> 5) * BWDX_WARP_FLOATS;
  float4* wrec = reinterpret_cast<float4*>(red + NMOM * XRED_STRIDE);  // [2][XREC_F4]
  const float gam = (FAM == FAM_EXP) ? 1.0f : m.c;
  const float inv_f = (float)cam.inv_f;
  const float Y0 = (float)SH_C0;
  unsigned long long ntest = 0, nent = 0;
  // each pixel's next commit (cur) and the one after it (nxt, prefetched a
  // step ahead so its load latency hides behind a whole step)
  int cur[XNP], nxt[XNP];
#pragma unroll
  for (int q = 0; q < XNP; ++q) {
    NXS_CHECK(ptr[q] < max_splats);
    cur[q] = ptr[q] >= 0 ? myseq[q][(size_t)ptr[q] * npix] : -1;
    nxt[q] = ptr[q] >= 1 ? myseq[q][(size_t)(ptr[q] - 1) * npix] : -1;
  }
  // lanes 0..10 copy one float4 each of a rank's record + B frame
  auto fetch = [&](int rank, int b) {
    if (lane < XREC_F4) {
      const float4* src = lane < REC_F4 ? records + (size_t)rank * REC_F4 + lane
                                        : bframe + (size_t)rank * 3 + (lane - REC_F4);
      cp_async16(&wrec[b * XREC_F4 + lane], src);
    }
    cp_async_commit();
  };
  int wcur = __reduce_max_sync(0xffffffffu, XNP == 2 ? max(cur[0], cur[XNP - 1]) : cur[0]);
  int b = 0;
  if (wcur >= 0) fetch(wcur, 0);

  while (wcur >= 0) {
    if (COUNT && lane == 0) ++nent;
    const uint32_t rank = (uint32_t)wcur;  // warp-uniform
    // this step's pixels advance; the next step's rank is known at once
    bool mine[XNP];
    int idx[XNP];
#pragma unroll
    for (int q = 0; q < XNP; ++q) {
      mine[q] = cur[q] == wcur;
      idx[q] = ptr[q];
      if (mine[q]) {
        --ptr[q];
        cur[q] = nxt[q];
        nxt[q] = ptr[q] >= 1 ? myseq[q][(size_t)(ptr[q] - 1) * npix] : -1;
      }
    }
    const int wnext = __reduce_max_sync(0xffffffffu, XNP == 2 ? max(cur[0], cur[XNP - 1]) : cur[0]);
    if (wnext >= 0) {
      fetch(wnext, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const float4* rec = wrec + b * XREC_F4;
    const float4* bf = rec + REC_F4;
    float dm2[XNP], ux[XNP], uy[XNP], uz[XNP], dak[XNP], e0[XNP], e1[XNP], e2[XNP];
#pragma unroll
    for (int q = 0; q < XNP; ++q)
      dm2[q] = ux[q] = uy[q] = uz[q] = dak[q] = e0[q] = e1[q] = e2[q] = 0.f;
#pragma unroll
    for (int q = 0; q < XNP; ++q) {
      if (mine[q])
        bwd_pixel<FAM>(st[q], rec, bf, idx[q], cam, m, cutoff, near_plane, inv_f, gam, dm2[q],
                       ux[q], uy[q], uz[q], dak[q], e0[q], e1[q], e2[q], ntest, COUNT);
    }
    float* col = red + lane;
    if constexpr (XNP == 1) {
      const PixelConst& pa = st[0].pc;
      const float ax = dm2[0] * ux[0], ay = dm2[0] * uy[0], az = dm2[0] * uz[0];
      col[0 * XRED_STRIDE] = ax * ux[0];
      col[1 * XRED_STRIDE] = ax * uy[0];
      col[2 * XRED_STRIDE] = ax * uz[0];
      col[3 * XRED_STRIDE] = ay * uy[0];
      col[4 * XRED_STRIDE] = ay * uz[0];
      col[5 * XRED_STRIDE] = az * uz[0];
      col[6 * XRED_STRIDE] = ax;
      col[7 * XRED_STRIDE] = ay;
      col[8 * XRED_STRIDE] = az;
      col[11 * XRED_STRIDE] = dak[0];
      col[12 * XRED_STRIDE] = e0[0] * Y0;
      col[13 * XRED_STRIDE] = e0[0] * pa.Y1;
      col[14 * XRED_STRIDE] = e0[0] * pa.Y2;
      col[15 * XRED_STRIDE] = e0[0] * pa.Y3;
      col[16 * XRED_STRIDE] = e1[0] * Y0;
      col[17 * XRED_STRIDE] = e1[0] * pa.Y1;
      col[18 * XRED_STRIDE] = e1[0] * pa.Y2;
      col[19 * XRED_STRIDE] = e1[0] * pa.Y3;
      col[20 * XRED_STRIDE] = e2[0] * Y0;
      col[21 * XRED_STRIDE] = e2[0] * pa.Y1;
      col[22 * XRED_STRIDE] = e2[0] * pa.Y2;
      col[23 * XRED_STRIDE] = e2[0] * pa.Y3;
    } else {
    const PixelConst& pa = st[0].pc;
    const PixelConst& pb = st[XNP - 1].pc;
    const float ax = dm2[0] * ux[0], ay = dm2[0] * uy[0], az = dm2[0] * uz[0];
    const float bx = dm2[XNP - 1] * ux[XNP - 1], by = dm2[XNP - 1] * uy[XNP - 1],
                bz = dm2[XNP - 1] * uz[XNP - 1];
    col[0 * XRED_STRIDE] = fmaf(ax, ux[0], bx * ux[XNP - 1]);
    col[1 * XRED_STRIDE] = fmaf(ax, uy[0], bx * uy[XNP - 1]);
    col[2 * XRED_STRIDE] = fmaf(ax, uz[0], bx * uz[XNP - 1]);
    col[3 * XRED_STRIDE] = fmaf(ay, uy[0], by * uy[XNP - 1]);
    col[4 * XRED_STRIDE] = fmaf(ay, uz[0], by * uz[XNP - 1]);
    col[5 * XRED_STRIDE] = fmaf(az, uz[0], bz * uz[XNP - 1]);
    col[6 * XRED_STRIDE] = ax + bx;
    col[7 * XRED_STRIDE] = ay + by;
    col[8 * XRED_STRIDE] = az + bz;
    col[11 * XRED_STRIDE] = dak[0] + dak[XNP - 1];
    col[12 * XRED_STRIDE] = (e0[0] + e0[XNP - 1]) * Y0;
    col[13 * XRED_STRIDE] = fmaf(e0[0], pa.Y1, e0[XNP - 1] * pb.Y1);
    col[14 * XRED_STRIDE] = fmaf(e0[0], pa.Y2, e0[XNP - 1] * pb.Y2);
    col[15 * XRED_STRIDE] = fmaf(e0[0], pa.Y3, e0[XNP - 1] * pb.Y3);
    col[16 * XRED_STRIDE] = (e1[0] + e1[XNP - 1]) * Y0;
    col[17 * XRED_STRIDE] = fmaf(e1[0], pa.Y1, e1[XNP - 1] * pb.Y1);
    col[18 * XRED_STRIDE] = fmaf(e1[0], pa.Y2, e1[XNP - 1] * pb.Y2);
    col[19 * XRED_STRIDE] = fmaf(e1[0], pa.Y3, e1[XNP - 1] * pb.Y3);
    col[20 * XRED_STRIDE] = (e2[0] + e2[XNP - 1]) * Y0;
    col[21 * XRED_STRIDE] = fmaf(e2[0], pa.Y1, e2[XNP - 1] * pb.Y1);
    col[22 * XRED_STRIDE] = fmaf(e2[0], pa.Y2, e2[XNP - 1] * pb.Y2);
    col[23 * XRED_STRIDE] = fmaf(e2[0], pa.Y3, e2[XNP - 1] * pb.Y3);
    }
    __syncwarp();
    if (lane < NMOM && lane != 9 && lane != 10) {
      const float4* row = reinterpret_cast<const float4*>(red + lane * XRED_STRIDE);
      const float4 a = row[0], b = row[1], c = row[2], d = row[3];
      const float4 e = row[4], f = row[5], g = row[6], h = row[7];
      const float sum = (((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w))) +
                        (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w))) +
                        ((((e.x + e.y) + (e.z + e.w)) + ((f.x + f.y) + (f.z + f.w))) +
                         (((g.x + g.y) + (g.z + g.w)) + ((h.x + h.y) + (h.z + h.w))));
      if (sum != 0.f) {
        atomicAdd(&moments[(size_t)rank * NMOM + lane], (double)sum);
        touched[rank] = 1;
      }
    }
    __syncwarp();
    wcur = wnext;
    b ^= 1;
  }

  if (COUNT) {  // (per warp: the warps of a tile may be separate blocks)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ntest += __shfl_xor_sync(0xffffffffu, ntest, o);
    if (lane == 0) {
      atomicAdd(&cnt->tests_bwd, ntest);
      atomicAdd(&cnt->entries_bwd, nent);
    }
  }
}

// (the two block shapes as separate kernels so each gets its own register
// budget: 91-103 registers at one pixel per thread, 128 at two)
template <int FAM, bool COUNT>
#ifndef NXS_X1_MINB
#define NXS_X1_MINB 20  // (96 registers: 21 one-warp blocks per SM; 22+ spills)
#endif
__global__ void __launch_bounds__(32, NXS_X1_MINB) k_blend_bwd_x1(const float4* __restrict__ records, const float4* __restrict__ bframe,
                  const uint32_t* __restrict__ pairs, const int32_t* __restrict__ seq,
                  int max_splats, CamDev cam, ModelDev m, float cutoff, double near_plane,
                  float bg0, float bg1, float bg2, const float* __restrict__ seed,
                  PixCache cache, double* __restrict__ moments, uint8_t* __restrict__ touched,
                  Counters* __restrict__ cnt) {
  // one warp per block (8 per tile): a warp that finishes its steps frees
  // its slot at once instead of idling until its tile's slowest warp is done
  bwd_x_body<FAM, COUNT, 1>(records, bframe, pairs, seq, max_splats, cam, m, cutoff, near_plane, bg0, bg1, bg2, seed, cache, moments, touched, cnt, blockIdx.x >> 3, blockIdx.x & 7);
}
template <int FAM, bool COUNT>
__global__ void __launch_bounds__(TILE_PIX / 2) k_blend_bwd_x2(const float4* __restrict__ records, const float4* __restrict__ bframe,
                  const uint32_t* __restrict__ pairs, const int32_t* __restrict__ seq,
                  int max_splats, CamDev cam, ModelDev m, float cutoff, double near_plane,
                  float bg0, float bg1, float bg2, const float* __restrict__ seed,
                  PixCache cache, double* __restrict__ moments, uint8_t* __restrict__ touched,
                  Counters* __restrict__ cnt) {
  bwd_x_body<FAM, COUNT, 2>(records, bframe, pairs, seq, max_splats, cam, m, cutoff, near_plane, bg0, bg1, bg2, seed, cache, moments, touched, cnt, blockIdx.x, threadIdx.x >> 5);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <class K>
static void set_smem(K k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
}

template <int FAM, int XB>
static void launch_fwd_x_xb(bool count, int n_tiles, const FwdXArgs& a, const CamDev& cam,
                            const ModelDev& m, const PixCache& cache, const PixResume& rs,
                            Counters* cnt, cudaStream_t s) {
  static unsigned long long attr_dev = 0;
  once_per_device(attr_dev, [] {
    set_smem(k_blend_fwd_x<FAM, true, XB, true>, fwdx_smem(XB));
    set_smem(k_blend_fwd_x<FAM, false, XB, true>, fwdx_smem(XB));
    set_smem(k_blend_fwd_x<FAM, true, XB, false>, fwdx_smem(XB));
    set_smem(k_blend_fwd_x<FAM, false, XB, false>, fwdx_smem(XB));
  });
  // (CH: chunked order; the exact order carries no chunk ids)
  auto k = a.chunk > 0 ? (count ? k_blend_fwd_x<FAM, true, XB, true> : k_blend_fwd_x<FAM, false, XB, true>)
                       : (count ? k_blend_fwd_x<FAM, true, XB, false> : k_blend_fwd_x<FAM, false, XB, false>);
  nxs_launch(k, n_tiles, TILE_PIX, fwdx_smem(XB), s, 
      a.records, a.pairs, a.ranges, a.zlo_rank, a.order, a.rank_c, a.chunk, cam, m, a.max_splats,
      a.cutoff, a.near_plane, a.bg[0], a.bg[1], a.bg[2], a.rgb, a.overdraw, a.residual, cache, rs,
      a.seq, a.overflow, a.active, a.n_active, a.resume, a.save, a.carry_t, a.carry_r,
      a.carry_n, a.end_bound, a.need_rank, cnt);
}

template <int FAM>
static void launch_fwd_x_fam(bool count, int n_tiles, const FwdXArgs& a, const CamDev& cam,
                             const ModelDev& m, const PixCache& cache, const PixResume& rs,
                             Counters* cnt, cudaStream_t s) {
  if (a.xbuf <= 16)
    launch_fwd_x_xb<FAM, 16>(count, n_tiles, a, cam, m, cache, rs, cnt, s);
  else
    launch_fwd_x_xb<FAM, 32>(count, n_tiles, a, cam, m, cache, rs, cnt, s);
}

void launch_blend_fwd_x(bool count, int n_tiles, const FwdXArgs& a, const CamDev& cam,
                        const ModelDev& m, const PixCache& cache, const PixResume& rs,
                        Counters* cnt, cudaStream_t s) {
  if (n_tiles == 0) return;
  switch (m.fam) {
    case FAM_EXP: launch_fwd_x_fam<FAM_EXP>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_LIN: launch_fwd_x_fam<FAM_LIN>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_QUAD: launch_fwd_x_fam<FAM_QUAD>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_BLEND: launch_fwd_x_fam<FAM_BLEND>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    case FAM_POW: launch_fwd_x_fam<FAM_POW>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
    default: launch_fwd_x_fam<FAM_SOFT>(count, n_tiles, a, cam, m, cache, rs, cnt, s); break;
  }
}

template <int FAM>
static void launch_bwd_x_fam(bool count, int n_tiles, const BwdXArgs& a, const CamDev& cam,
                             const ModelDev& m, const PixCache& cache, Counters* cnt,
                             cudaStream_t s) {
  static unsigned long long attr_dev = 0;
  once_per_device(attr_dev, [] {
    set_smem(k_blend_bwd_x1<FAM, true>, bwdx_smem(1));
    set_smem(k_blend_bwd_x1<FAM, false>, bwdx_smem(1));
    set_smem(k_blend_bwd_x2<FAM, true>, bwdx_smem(2));
    set_smem(k_blend_bwd_x2<FAM, false>, bwdx_smem(2));
  });
  const int np = a.exact ? 1 : 2;
  auto k = a.exact ? (count ? k_blend_bwd_x1<FAM, true> : k_blend_bwd_x1<FAM, false>)
                   : (count ? k_blend_bwd_x2<FAM, true> : k_blend_bwd_x2<FAM, false>);
  nxs_launch(k, np == 1 ? 8 * n_tiles : n_tiles, np == 1 ? 32 : TILE_PIX / 2, bwdx_smem(np), s,
             a.records, a.bframe, a.pairs, a.seq,
             a.max_splats, cam, m, a.cutoff, a.near_plane, a.bg[0], a.bg[1], a.bg[2], a.seed,
             cache, a.moments, a.touched, cnt);
}

void launch_blend_bwd_x(bool count, int n_tiles, const BwdXArgs& a, const CamDev& cam,
                        const ModelDev& m, const PixCache& cache, Counters* cnt, cudaStream_t s) {
  if (n_tiles == 0) return;
  switch (m.fam) {
    case FAM_EXP: launch_bwd_x_fam<FAM_EXP>(count, n_tiles, a, cam, m, cache, cnt, s); break;
    case FAM_LIN: launch_bwd_x_fam<FAM_LIN>(count, n_tiles, a, cam, m, cache, cnt, s); break;
    case FAM_QUAD: launch_bwd_x_fam<FAM_QUAD>(count, n_tiles, a, cam, m, cache, cnt, s); break;
    case FAM_BLEND: launch_bwd_x_fam<FAM_BLEND>(count, n_tiles, a, cam, m, cache, cnt, s); break;
    case FAM_POW: launch_bwd_x_fam<FAM_POW>(count, n_tiles, a, cam, m, cache, cnt, s); break;
    default: launch_bwd_x_fam<FAM_SOFT>(count, n_tiles, a, cam, m, cache, cnt, s); break;
  }
}

}  // namespace nxs

#ifdef NXS_XSTATS
extern "C" int nxs_debug_xstats(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, nxs::g_xstats, sizeof(nxs::g_xstats)) == cudaSuccess ? 0 : -3;
}
#endif
