// K0 depth keys, K1 per-Gaussian projection + conic tile bbox, K2 pair
// emission and tile ranges.
//
// Compiled with --fmad=false: every fp64 operation here is a correctly
// rounded IEEE add/sub/mul/div/sqrt (plus exact floor/ceil/frexp), in the
// order written, so oracle/binning_oracle.c (gcc -ffp-contract=off)
// reproduces the records, rectangles, ranks and pair lists bit for bit.
// The operation order below is normative for that restatement.
//
// Replaces (reference pkg/src/nexsplat/):
//   _depth_chunks ordering           render.py:350-358
//   per-Gaussian part of _chunk_geometry (quat_to_rot, A, b)
//                                    render.py:116-121, primitives.py:45-64
// The per-pixel test those records feed is in blend_fwd.cu.
#include <algorithm>
#include <cstdlib>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "nxs_internal.cuh"

namespace nxs {

// ln(x) for x > 0 with only IEEE basic ops: x = m·2^e, m in [√½, √2),
// ln m = 2·atanh((m-1)/(m+1)) as an 11-term odd series (|z| <= 0.1716,
// truncation < 1e-18).  Deterministic across nvcc and gcc.
__device__ __forceinline__ double ln_det(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0.70710678118654752440) {
    m = m * 2.0;
    e = e - 1;
  }
  double z = (m - 1.0) / (m + 1.0);
  double z2 = z * z;
  double s = 1.0 / 23.0;
  s = s * z2 + 1.0 / 21.0;
  s = s * z2 + 1.0 / 19.0;
  s = s * z2 + 1.0 / 17.0;
  s = s * z2 + 1.0 / 15.0;
  s = s * z2 + 1.0 / 13.0;
  s = s * z2 + 1.0 / 11.0;
  s = s * z2 + 1.0 / 9.0;
  s = s * z2 + 1.0 / 7.0;
  s = s * z2 + 1.0 / 5.0;
  s = s * z2 + 1.0 / 3.0;
  s = s * z2 + 1.0;
  return (double)e * 0.69314718055994530942 + 2.0 * z * s;
}

// Compensated 3-term dot product (Ogita-Rump-Oishi Dot2: TwoProd via fma,
// TwoSum cascade).  The reference computes the depth with numpy's `@`,
// which runs through OpenBLAS with a CPU-dependent FMA/summation order, so
// its last bit is not machine-independent; Dot2 is as accurate as a
// double-double evaluation rounded once, and deterministic on both nvcc and
// gcc.  Orders can then differ from the reference only between Gaussians
// whose depths agree to a few ulps (true ties up to rounding).
__device__ __forceinline__ double dot3_compensated(double a0, double a1, double a2, double b0,
                                                   double b1, double b2) {
  double p = a0 * b0;
  double s = __fma_rn(a0, b0, -p);
  double h = a1 * b1, r = __fma_rn(a1, b1, -h);
  double t = p + h, bb = t - p, q = (p - (t - bb)) + (h - bb);
  p = t;
  s = s + (q + r);
  h = a2 * b2;
  r = __fma_rn(a2, b2, -h);
  t = p + h;
  bb = t - p;
  q = (p - (t - bb)) + (h - bb);
  p = t;
  s = s + (q + r);
  return p + s;
}

__device__ __forceinline__ unsigned long long dkey(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Lower bound of the camera depth of the ray-peak point over every pixel where
// the Gaussian can be valid; since x'_z = t·d'_z with d'_z = 1/|h|, every valid
// pixel has t >= z_lo·|h| (exact-order mode).
// Peak points x satisfy (x - b')ᵀA'x = 0: in A'-whitened coordinates y = Lx
// they lie on the sphere |y - c| = |c|, c = Lb'/2, and validity (m2 <= r²)
// keeps them within distance r of the sphere point 2c — a spherical cap.  The
// depth x'_z = wᵀy (w = L⁻ᵀe_z, |w| = σ_z) is minimised over that cap in
// closed form: z_lo = b'_z/2 + R σ_z cos(min(π, α + φ)), R = |c| = √(bᵀAb)/2,
// cos α = (b'_z/2)/(R σ_z), cos φ = 1 - r²/(2R²).  Far tighter than the
// ellipsoid's own minimum depth b'_z - r σ_z (used when R degenerates).
__device__ __forceinline__ double z_lower(const float* __restrict__ centers,
                                          const float* __restrict__ scales,
                                          const float* __restrict__ quats,
                                          const float* __restrict__ opacities, int64_t g,
                                          const CamDev& cam, double cutoff) {
  const float4 q4 = reinterpret_cast<const float4*>(quats)[g];
  double qw = q4.x, qx = q4.y, qy = q4.z, qz = q4.w;
  double nq = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
  double inq = 1.0 / nq;
  double w = qw * inq, x = qx * inq, y = qy * inq, z = qz * inq;
  const double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                       2.0 * (x * y + w * z),       1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                       2.0 * (x * z - w * y),       2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
  const double s[3] = {(double)scales[3 * g + 0], (double)scales[3 * g + 1],
                       (double)scales[3 * g + 2]};
  const double b0 = (double)centers[3 * g + 0] - cam.o[0];
  const double b1 = (double)centers[3 * g + 1] - cam.o[1];
  const double b2 = (double)centers[3 * g + 2] - cam.o[2];
  double szz = 0.0, bAb = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // camera z of Gaussian axis k, and the offset's component along it
    const double mk = (cam.R[2] * R[0 + k] + cam.R[5] * R[3 + k]) + cam.R[8] * R[6 + k];
    const double uk = (b0 * R[0 + k] + b1 * R[3 + k]) + b2 * R[6 + k];
    szz += (mk * s[k]) * (mk * s[k]);
    bAb += (uk / s[k]) * (uk / s[k]);
  }
  const double sz = sqrt(szz);
  const double op = (double)opacities[g];
  const double r2 = (op >= cutoff ? 2.0 * ln_det(op / cutoff) : 0.0) * (1.0 + 1e-4) + 1e-4;
  const double bz = (cam.R[2] * b0 + cam.R[5] * b1) + cam.R[8] * b2;
  const double zell = bz - sqrt(r2) * sz;  // the ellipsoid's own minimum depth
  const double Rs = 0.5 * sqrt(bAb);
  if (!(Rs > 0.0) || !(sz > 0.0)) return zell;
  double ca = (0.5 * bz) / (Rs * sz);
  ca = ca > 1.0 ? 1.0 : (ca < -1.0 ? -1.0 : ca);
  const double cf = 1.0 - r2 / (2.0 * Rs * Rs);
  double caf;
  if (cf <= -ca) {
    caf = -1.0;  // the cap reaches the sphere's deepest point against w
  } else {
    const double sa = sqrt(fmax(0.0, 1.0 - ca * ca)), sf = sqrt(fmax(0.0, 1.0 - cf * cf));
    caf = ca * cf - sa * sf;
  }
  const double zc = 0.5 * bz + Rs * sz * caf;
  // guard rounding: never above the true bound by more than a few ulps
  const double zlo = zc - 1e-9 * fabs(bz) - 1e-12;
  return (zlo == zlo) ? fmax(zlo, zell) : zell;
}

// K0: fp64 view depth (μ - o)·forward (compensated), its order-preserving
// u64 key (64-bit fallback sort), and the NaN-free min/max key of the batch.
// With `zmode` (exact-order mode) the sort key is z_lo instead of the
// centre depth.
__global__ void k_depth(const float* __restrict__ centers, const float* __restrict__ scales,
                        const float* __restrict__ quats, const float* __restrict__ opacities,
                        int64_t P, CamDev cam, double cutoff, int zmode,
                        double* __restrict__ depth, unsigned long long* __restrict__ key64,
                        uint32_t* __restrict__ idx, unsigned long long* __restrict__ kminmax) {
  nxs_pdl_enter();
  __shared__ unsigned long long s_min[8], s_max[8];
  unsigned long long kmin = ~0ull, kmax = 0ull;
  // grid-stride: few blocks, so few atomics on the two min/max words
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    double b0 = (double)centers[3 * i + 0] - cam.o[0];
    double b1 = (double)centers[3 * i + 1] - cam.o[1];
    double b2 = (double)centers[3 * i + 2] - cam.o[2];
    // forward = third column of the camera rotation
    const double d = zmode ? z_lower(centers, scales, quats, opacities, i, cam, cutoff)
                           : dot3_compensated(b0, b1, b2, cam.R[2], cam.R[5], cam.R[8]);
    depth[i] = d;
    const unsigned long long k = dkey(d);
    if (key64) {  // (the 64-bit sort's keys and values; lazy phases need neither)
      key64[i] = k;
      idx[i] = (uint32_t)i;
    }
    if (d == d) {
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_min[w] = kmin;
    s_max[w] = kmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      kmin = min(kmin, s_min[k]);
      kmax = max(kmax, s_max[k]);
    }
    if (kmin <= kmax) {
      atomicMin(&kminmax[0], kmin);
      atomicMax(&kminmax[1], kmax);
    }
  }
}

// K0, the centre-depth case (global and chunked orders): four Gaussians per
// thread from three 16-byte loads of their centres, so every thread has its
// whole input in flight at once (the one-per-thread grid-stride form waited
// out a DRAM round trip per element: 11.9 -> 8.2 us at 1M).  Same values as
// k_depth.
__global__ void k_depth4(const float4* __restrict__ centers4, int64_t P, CamDev cam,
                         double* __restrict__ depth, unsigned long long* __restrict__ key64,
                         uint32_t* __restrict__ idx, unsigned long long* __restrict__ kminmax) {
  nxs_pdl_enter();
  __shared__ unsigned long long s_min[8], s_max[8];
  unsigned long long kmin = ~0ull, kmax = 0ull;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = 4 * t;
  if (i0 < P) {
    float c[12];
    const float* cf = reinterpret_cast<const float*>(centers4);
    if (i0 + 4 <= P) {
      const float4 a = centers4[3 * t], b = centers4[3 * t + 1], e = centers4[3 * t + 2];
      c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
      c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
      c[8] = e.x; c[9] = e.y; c[10] = e.z; c[11] = e.w;
    } else {
#pragma unroll
      for (int k = 0; k < 12; ++k) c[k] = i0 * 3 + k < 3 * P ? cf[i0 * 3 + k] : 0.f;
    }
    double d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double b0 = (double)c[3 * q + 0] - cam.o[0];
      const double b1 = (double)c[3 * q + 1] - cam.o[1];
      const double b2 = (double)c[3 * q + 2] - cam.o[2];
      d[q] = dot3_compensated(b0, b1, b2, cam.R[2], cam.R[5], cam.R[8]);
    }
    if (i0 + 4 <= P) {
      double2* d2 = reinterpret_cast<double2*>(depth + i0);
      d2[0] = make_double2(d[0], d[1]);
      d2[1] = make_double2(d[2], d[3]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i0 + q >= P) break;
      if (i0 + 4 > P) depth[i0 + q] = d[q];
      const unsigned long long k = dkey(d[q]);
      if (key64) {
        key64[i0 + q] = k;
        idx[i0 + q] = (uint32_t)(i0 + q);
      }
      if (d[q] == d[q]) {
        kmin = min(kmin, k);
        kmax = max(kmax, k);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_min[w] = kmin;
    s_max[w] = kmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      kmin = min(kmin, s_min[k]);
      kmax = max(kmax, s_max[k]);
    }
    if (kmin <= kmax) {
      atomicMin(&kminmax[0], kmin);
      atomicMax(&kminmax[1], kmax);
    }
  }
}

// 32-bit monotone key: floor((d - dmin) * (2^32 - 2) / (dmax - dmin)); NaN last.
// d1 < d2 implies key(d1) <= key(d2); equal keys are re-ordered by k_key_fixup.
__device__ __forceinline__ uint32_t key32_of(double d, double lo, double scale, bool spread) {
  if (!(d == d)) return 0xffffffffu;
  if (!spread) return 0u;
  double x = (d - lo) * scale;
  x = x < 0.0 ? 0.0 : (x > 4294967294.0 ? 4294967294.0 : x);
  return (uint32_t)x;
}
__global__ void k_key32(const double* __restrict__ depth, int64_t P,
                        const unsigned long long* __restrict__ kminmax,
                        uint32_t* __restrict__ key) {
  nxs_pdl_enter();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const bool spread = kminmax[0] < kminmax[1];
  const double lo = dkey_inv(kminmax[0]), hi = dkey_inv(kminmax[1]);
  key[i] = key32_of(depth[i], lo, 4294967294.0 / (hi - lo), spread);
}
// 64-bit keys of the fallback sort from the depths (lazy phases skip them in K0)
__global__ void k_dkeys(const double* __restrict__ depth, int64_t P,
                        unsigned long long* __restrict__ key64) {
  nxs_pdl_enter();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) key64[i] = dkey(depth[i]);
}

// Runs of equal 32-bit keys come out of the stable sort in index order;
// re-sort each run by (fp64 depth, index) — exactly the 64-bit order.
// Runs longer than 256 raise `overflow` (the host then redoes the 64-bit sort).
// With `shift`, the keys were sorted on their bits >= shift only: runs are
// equal key >> shift, and the same re-sort makes the order exact.
__global__ void k_key_fixup(const uint32_t* __restrict__ key, uint32_t* __restrict__ idx,
                            const double* __restrict__ depth, int64_t P, int shift,
                            unsigned long long* __restrict__ overflow,
                            const int* __restrict__ nd) {
  nxs_pdl_enter();
  if (nd) P = min(P, (int64_t)*nd);  // device-sized phase: real items only
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const uint32_t k = key[i] >> shift;
  if (i > 0 && (key[i - 1] >> shift) == k) return;         // not a run start
  if (i + 1 >= P || (key[i + 1] >> shift) != k) return;    // singleton
  int64_t e = i + 1;
  while (e < P && (key[e] >> shift) == k && e - i <= 256) ++e;
  if (e - i > 256) {
    atomicAdd(overflow, 1ull);
    return;
  }
  for (int64_t a = i + 1; a < e; ++a) {  // insertion sort, stable by index
    const uint32_t v = idx[a];
    const double dv = depth[v];
    int64_t b = a - 1;
    while (b >= i) {
      const uint32_t w = idx[b];
      const double dw = depth[w];
      if (dw > dv || (dw == dv && w > v) || (!(dw == dw) && (dv == dv))) {
        idx[b + 1] = w;
        --b;
      } else {
        break;
      }
    }
    idx[b + 1] = v;
  }
}

__global__ void k_rank_of(const uint32_t* __restrict__ order, int64_t r0, int64_t r1,
                          uint32_t* __restrict__ rank_of, const int* __restrict__ nd) {
  nxs_pdl_enter();
  if (nd) r1 = min(r1, r0 + (int64_t)*nd);
  int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < r1) rank_of[order[r]] = (uint32_t)r;
}

// ---- lazy depth phases (global order): only the ranks a phase needs are
// sorted and projected.  The 32-bit keys are histogrammed by their top 12
// bits; phase p takes the bins up to the first one whose cumulative count
// reaches its target rank, so phases are unions of whole key bins (ties
// never straddle a boundary) and concatenating the phases' sorted ranks is
// exactly the full order.
constexpr int PH_BINS = 4096;
constexpr int BIN_STRIDE = 32;  // bin cursors, one per 128-byte line


// one block: inclusive scan of the histogram; for each target rank T_p the
// first bin whose cumulative count reaches it.  out[2p] = last bin of phase
// p, out[2p+1] = its end rank; the last phase ends at bin PH_BINS-1, rank P.
// (run by the last block of k_key32_hist_select; `hist` is read through L2:
// the other blocks wrote it)
__device__ __forceinline__ void phase_select_body(const unsigned int* __restrict__ hist,
                                                  const int64_t* __restrict__ targets,
                                                  int n_targets, int64_t P,
                                                  long long* __restrict__ out, int max_bin0,
                                                  unsigned long long* __restrict__ overflow,
                                                  unsigned int* __restrict__ bin_pos,
                                                  int* __restrict__ n_sel,
                                                  unsigned long long* cum, unsigned long long* wsum) {
  constexpr int PER = PH_BINS / 1024;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  unsigned long long loc[PER], run = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    run += __ldcg(hist + t * PER + k);
    loc[k] = run;
  }
  unsigned long long x = run;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long v = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  const unsigned long long base = x - run + (w > 0 ? wsum[w - 1] : 0ull);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    cum[t * PER + k] = base + loc[k];
    // each bin's first rank: the scatter's cursor (k_bin_scatter), one
    // counter per 128-byte line so the scatter's atomics spread over L2
    if (bin_pos)
      bin_pos[(t * PER + k) * BIN_STRIDE] = (unsigned int)(base + loc[k] - __ldcg(hist + t * PER + k));
  }
  __syncthreads();
  if (t < n_targets) {
    const unsigned long long T = (unsigned long long)targets[t];
    int lo = 0, hi = PH_BINS - 1;  // first bin with cum >= T
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cum[mid] >= T) hi = mid; else lo = mid + 1;
    }
    out[2 * t] = lo;
    out[2 * t + 1] = (long long)cum[lo];
    // device-sized phase 0 sorted only the key bits below max_bin0's
    if (t == 0 && max_bin0 >= 0 && lo > max_bin0) atomicAdd(overflow, 1ull);
  }
  if (t == 0) {
    out[2 * n_targets] = PH_BINS - 1;
    out[2 * n_targets + 1] = P;
    if (n_targets == 0 && max_bin0 >= 0 && max_bin0 < PH_BINS - 1) atomicAdd(overflow, 1ull);
    if (n_sel) *n_sel = (int)out[1];  // Gaussians of phase 0
  }
}

// The 32-bit keys (key32_of), their histogram over the top 12 bits and the
// phase selection in one launch: every block adds its shared
// histogram into `hist`, takes a ticket (hist[PH_BINS], zeroed by
// k_call_init) and the last block runs the phase selection — one kernel
// boundary and one single-block launch fewer on the pipeline's critical path.
__global__ void __launch_bounds__(1024)
    k_key32_hist_select(const double* __restrict__ depth, int64_t P,
                        const unsigned long long* __restrict__ kminmax, uint32_t* __restrict__ key,
                        unsigned int* __restrict__ hist, const int64_t* __restrict__ targets,
                        int n_targets, long long* __restrict__ out, int max_bin0,
                        unsigned long long* __restrict__ overflow,
                        unsigned int* __restrict__ bin_pos, int* __restrict__ n_sel) {
  nxs_pdl_enter();
  __shared__ unsigned long long smem[PH_BINS];  // histogram (u32 view), then the scan
  __shared__ unsigned long long wsum[32];
  __shared__ bool s_last;
  unsigned int* sh = reinterpret_cast<unsigned int*>(smem);
  for (int b = threadIdx.x; b < PH_BINS; b += blockDim.x) sh[b] = 0u;
  const bool spread = kminmax[0] < kminmax[1];
  const double lo = dkey_inv(kminmax[0]), hi = dkey_inv(kminmax[1]);
  const double scale = 4294967294.0 / (hi - lo);
  __syncthreads();
  // four Gaussians per thread: two 16-B depth loads in flight, one 16-B key store
  for (int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i0 < P;
       i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    if (i0 + 4 <= P) {
      const double2 a = reinterpret_cast<const double2*>(depth + i0)[0];
      const double2 b = reinterpret_cast<const double2*>(depth + i0)[1];
      uint4 k;
      k.x = key32_of(a.x, lo, scale, spread);
      k.y = key32_of(a.y, lo, scale, spread);
      k.z = key32_of(b.x, lo, scale, spread);
      k.w = key32_of(b.y, lo, scale, spread);
      *reinterpret_cast<uint4*>(key + i0) = k;
      atomicAdd(&sh[k.x >> 20], 1u);
      atomicAdd(&sh[k.y >> 20], 1u);
      atomicAdd(&sh[k.z >> 20], 1u);
      atomicAdd(&sh[k.w >> 20], 1u);
    } else {
      for (int64_t i = i0; i < P; ++i) {
        const uint32_t k = key32_of(depth[i], lo, scale, spread);
        key[i] = k;
        atomicAdd(&sh[k >> 20], 1u);
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < PH_BINS; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&hist[PH_BINS], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  phase_select_body(hist, targets, n_targets, P, out, max_bin0, overflow, bin_pos, n_sel, smem,
                    wsum);
}

// ---- one depth phase in exact order without a global sort: the phase's
// key bins are contiguous rank ranges (the phase selection's bin_pos), each
// Gaussian is scattered into its bin (any order), then each bin is sorted
// exactly by (depth, index) — NaN last — in shared memory, which is the
// order the 32-bit sort + fix-up produces.  Ranks are written alongside.
__global__ void k_bin_scatter(const uint32_t* __restrict__ key, int64_t P, int lo, int hi,
                              const long long* __restrict__ hi_dev,
                              unsigned int* __restrict__ bin_pos, uint32_t* __restrict__ order) {
  nxs_pdl_enter();
  if (hi_dev) hi = (int)hi_dev[0];
  // four keys per thread from one 16-B load (key is 16-B aligned)
  for (int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i0 < P;
       i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    uint32_t k[4];
    if (i0 + 4 <= P) {
      const uint4 v = *reinterpret_cast<const uint4*>(key + i0);
      k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) k[q] = i0 + q < P ? key[i0 + q] : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int b = (int)(k[q] >> 20);
      if (i0 + q < P && b >= lo && b <= hi)
        order[atomicAdd(&bin_pos[b * BIN_STRIDE], 1u)] = (uint32_t)(i0 + q);
    }
  }
}

// exact depth order as one integer: monotone in the depth, -0 = +0, every
// NaN last; ties (equal keys) go by index
__device__ __forceinline__ unsigned long long depth_sortkey(double d) {
  if (!(d == d)) return ~0ull;
  return dkey(d == 0.0 ? 0.0 : d);
}

constexpr int BIN_THREADS = 512;
constexpr int BIN_MAX = 2048;  // longest bin sorted in shared memory
__global__ void __launch_bounds__(BIN_THREADS)
    k_bin_sort(uint32_t* __restrict__ order, const double* __restrict__ depth,
               const unsigned int* __restrict__ hist, const unsigned int* __restrict__ bin_end,
               int lo, int hi, const long long* __restrict__ hi_dev,
               uint32_t* __restrict__ rank_out, unsigned long long* __restrict__ overflow) {
  nxs_pdl_enter();
  __shared__ unsigned long long s_k[BIN_MAX];
  __shared__ uint32_t s_i[BIN_MAX];
  if (hi_dev) hi = (int)hi_dev[0];
  const int b = lo + blockIdx.x, tid = threadIdx.x;
  if (b > hi) return;
  const int n = (int)hist[b];
  if (n == 0) return;
  const int start = (int)bin_end[b * BIN_STRIDE] - n;
  uint32_t* v = order + start;
  if (n > BIN_MAX) {
    if (tid == 0) atomicAdd(overflow, 1ull);
    return;
  }
  for (int i = tid; i < n; i += BIN_THREADS) {
    const uint32_t g = v[i];
    s_i[i] = g;
    s_k[i] = depth_sortkey(depth[g]);
  }
  if (n <= BIN_THREADS / 4) {
    // short bins, rank counting: two threads per element (halves of the bin)
    __syncthreads();
    const int e = tid >> 1, h = tid & 1;
    const bool live = e < n;
    const unsigned long long mk = live ? s_k[e] : 0ull;
    const uint32_t mi = live ? s_i[e] : 0u;
    int pos = 0;
    if (live) {
#pragma unroll 4
      for (int j = h; j < n; j += 2) {
        const unsigned long long kj = s_k[j];
        pos += (kj < mk || (kj == mk && s_i[j] < mi)) ? 1 : 0;
      }
    }
    pos += __shfl_xor_sync(0xffffffffu, pos, 1);
    if (live && h == 0) {
      v[pos] = mi;
      if (rank_out) rank_out[mi] = (uint32_t)(start + pos);
    }
    return;
  }
  if (n <= BIN_THREADS) {
    // one element per thread: a bitonic network whose strides below 32 run
    // on registers with shuffles inside the warp; only the 10 stages with
    // stride >= 32 exchange through shared memory (two barriers each),
    // instead of 45 barrier-separated shared-memory stages
    __syncthreads();
    unsigned long long k = tid < n ? s_k[tid] : ~0ull;
    uint32_t id = tid < n ? s_i[tid] : 0xffffffffu;
    for (int size = 2; size <= BIN_THREADS; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        unsigned long long ok;
        uint32_t oi;
        if (stride >= 32) {  // (block-uniform)
          __syncthreads();
          s_k[tid] = k;
          s_i[tid] = id;
          __syncthreads();
          ok = s_k[tid ^ stride];
          oi = s_i[tid ^ stride];
        } else {
          ok = __shfl_xor_sync(0xffffffffu, k, stride);
          oi = __shfl_xor_sync(0xffffffffu, id, stride);
        }
        const bool take_min = ((tid & size) == 0) == ((tid & stride) == 0);
        const bool o_first = ok < k || (ok == k && oi < id);
        if (take_min == o_first) {
          k = ok;
          id = oi;
        }
      }
    }
    if (tid < n) {
      v[tid] = id;
      if (rank_out) rank_out[id] = (uint32_t)(start + tid);
    }
    return;
  }
  int p2 = 2 * BIN_THREADS;
  while (p2 < n) p2 <<= 1;
  for (int i = n + tid; i < p2; i += BIN_THREADS) {
    s_i[i] = 0xffffffffu;
    s_k[i] = ~0ull;
  }
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < (p2 >> 1); i += BIN_THREADS) {
        const int a = 2 * i - (i & (stride - 1)), c = a + stride;
        const bool up = (a & size) == 0;
        const unsigned long long ka = s_k[a], kc = s_k[c];
        const uint32_t ia = s_i[a], ic = s_i[c];
        const bool c_first = kc < ka || (kc == ka && ic < ia);
        if (c_first == up) {
          s_k[a] = kc;
          s_k[c] = ka;
          s_i[a] = ic;
          s_i[c] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < n; i += BIN_THREADS) {
    v[i] = s_i[i];
    if (rank_out) rank_out[s_i[i]] = (uint32_t)(start + i);
  }
}

// Chunked order (reference chunk_size = C > 1, render.py:350-358): the
// chunks are consecutive runs of C Gaussians in centre-depth order; tile
// lists are ordered by (chunk, z_lo) so the exact-order blend can commit per
// chunk.  Keys are the monotone bits of float_rd(z_lo) — the value the blend
// bounds with — and ties need no fix-up: any order of equal z_lo within a
// chunk is a valid list order (the per-pixel order comes from t and the
// centre-depth rank).
__device__ __forceinline__ uint32_t zlo_key(double z) {
  const float zf = __double2float_rd(z);
  const uint32_t b = __float_as_uint(zf);
  return (zf == zf) ? ((b & 0x80000000u) ? ~b : (b | 0x80000000u)) : 0xffffffffu;
}

// z_lo per Gaussian; with key64 also the (chunk << 32 | z_lo key) sort key
// of the global fallback for chunks too large for one block
__global__ void k_chunk_key(const float* __restrict__ centers, const float* __restrict__ scales,
                            const float* __restrict__ quats, const float* __restrict__ opacities,
                            int64_t P, CamDev cam, double cutoff,
                            const uint32_t* __restrict__ rank_c, int chunk,
                            double* __restrict__ zlo, unsigned long long* __restrict__ key64,
                            uint32_t* __restrict__ idx) {
  nxs_pdl_enter();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P) return;
  const double z = z_lower(centers, scales, quats, opacities, g, cam, cutoff);
  zlo[g] = z;
  if (key64) {
    key64[g] = ((unsigned long long)(rank_c[g] / (uint32_t)chunk) << 32) | zlo_key(z);
    idx[g] = (uint32_t)g;
  }
}

// one block per chunk: stable block radix sort of the chunk's Gaussians
// (centre-depth order in, (z_lo, centre rank) order out)
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
    k_chunk_sort(const uint32_t* __restrict__ order_c, const double* __restrict__ zlo, int64_t P,
                 int chunk, uint32_t* __restrict__ order_out, const int* __restrict__ nd) {
  nxs_pdl_enter();
  if (nd) P = min(P, (int64_t)*nd);  // (a device-sized phase: its chunk-aligned rank count)
  if ((int64_t)blockIdx.x * chunk >= P) return;
  using Sort = cub::BlockRadixSort<uint32_t, THREADS, ITEMS, uint32_t>;
  __shared__ typename Sort::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * chunk;
  const int n = (int)((P - base) < (int64_t)chunk ? (P - base) : (int64_t)chunk);
  uint32_t keys[ITEMS], vals[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int k = threadIdx.x * ITEMS + i;  // blocked: padding sorts after equal real keys
    if (k < n) {
      const uint32_t g = order_c[base + k];
      keys[i] = zlo_key(zlo[g]);
      vals[i] = g;
    } else {
      keys[i] = 0xffffffffu;
      vals[i] = 0xffffffffu;
    }
  }
  Sort(tmp).Sort(keys, vals);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int k = threadIdx.x * ITEMS + i;
    if (k < n) order_out[base + k] = vals[i];
  }
}

struct ProjOut {
  const double* zlo;            // exact-order mode: z_lo per Gaussian (sort key), else null
  float* zlo_rank;              // exact-order mode: z_lo per rank, rounded down
  int4* rects;                  // per Gaussian tile rectangle
  float4* records;              // per rank 8 x float4
  float4* bframe;               // per rank 3 x float4: rows of B (backward only)
  unsigned long long* straddle; // counter
  double* tq;                   // per RANK: silhouette conic + an inside point, tile rect (TQ_STRIDE)
  // optional: the ranks with a tile rectangle, appended (any order), and
  // their count — the emission then visits only those
  uint32_t* live;
  unsigned long long* n_live;
};
// per-rank tile-test slot: 10 doubles (conic, centre, 1/(2 Q00), 1/(2 Q11)),
// then the tile rectangle as an int4 — the binning reads rank r's rect and
// test data from one slot, without the order[r] -> rects[g] gather
constexpr int TQ_STRIDE = 12;
__device__ __forceinline__ int4 tq_rect(const double* tq, int64_t r) {
  return *reinterpret_cast<const int4*>(tq + TQ_STRIDE * r + 10);
}

// K1: per rank r (Gaussian g = order[r]).
// Per-Gaussian projection (g = storage index, r = depth rank), parameters
// already in registers.
struct GParams {
  float4 q;
  float c0, c1, c2, s0, s1, s2, op;
  float shv[12];
};

__device__ __forceinline__ int4 project_one(const GParams& prm, int64_t g, int64_t rk, const CamDev& cam,
                                            double cutoff, double near_plane, const ProjOut& out,
                                            float4* rec, float4* bf) {
  const float cx0 = prm.c0, cx1 = prm.c1, cx2 = prm.c2;
  const float sc0 = prm.s0, sc1 = prm.s1, sc2 = prm.s2;
  const float op = prm.op;
  const float* shv = prm.shv;
  const float4 q4 = prm.q;

  // --- rotation from the normalised quaternion (primitives.py:45-64)
  double qw = q4.x, qx = q4.y, qy = q4.z, qz = q4.w;
  double nq = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
  double inq = 1.0 / nq;
  double w = qw * inq, x = qx * inq, y = qy * inq, z = qz * inq;
  double R[9];
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);

  // M = Rc^T R  (Gaussian axes in camera frame)
  double M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = (cam.R[0 + i] * R[0 + j] + cam.R[3 + i] * R[3 + j]) + cam.R[6 + i] * R[6 + j];

  double s0 = sc0, s1 = sc1, s2 = sc2;
  double is0 = 1.0 / (s0 * s0), is1 = 1.0 / (s1 * s1), is2 = 1.0 / (s2 * s2);
  // A' = M diag(1/s^2) M^T  (camera-frame inverse covariance)
  double Ap[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      double v = ((M[3 * i + 0] * is0) * M[3 * j + 0] + (M[3 * i + 1] * is1) * M[3 * j + 1]) +
                 (M[3 * i + 2] * is2) * M[3 * j + 2];
      Ap[3 * i + j] = v;
      Ap[3 * j + i] = v;
    }

  // b' = Rc^T (μ - o)
  double b0 = (double)cx0 - cam.o[0];
  double b1 = (double)cx1 - cam.o[1];
  double b2 = (double)cx2 - cam.o[2];
  double bp[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) bp[i] = (cam.R[0 + i] * b0 + cam.R[3 + i] * b1) + cam.R[6 + i] * b2;
  double Ab[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    Ab[i] = (Ap[3 * i + 0] * bp[0] + Ap[3 * i + 1] * bp[1]) + Ap[3 * i + 2] * bp[2];
  double bAb = (bp[0] * Ab[0] + bp[1] * Ab[1]) + bp[2] * Ab[2];
  // N = (b'A'b') A' - (A'b')(A'b')^T, null vector b'
  double N[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) N[3 * i + j] = bAb * Ap[3 * i + j] - Ab[i] * Ab[j];

  int4 rect = make_int4(-1, -1, -1, -1);

  double opac = (double)op;
  bool live = opac >= cutoff;
  // cutoff ellipsoid radius (Mahalanobis), with the bbox/pre-test margin
  double r2 = live ? 2.0 * ln_det(opac / cutoff) : 0.0;
  double r2m = r2 * (1.0 + 1e-4) + 1e-4;
  double rm = sqrt(r2m);
  double m20 = M[6] * s0, m21 = M[7] * s1, m22 = M[8] * s2;
  double sz = sqrt((m20 * m20 + m21 * m21) + m22 * m22);
  double zmin = bp[2] - rm * sz;
  double zmax = bp[2] + rm * sz;
  if (live && zmax <= 0.0) live = false;  // entirely behind the camera plane
  bool general = false;
  if (live && zmin <= near_plane * 1.001) {
    // crosses the near region: the conic form (and its implied t > near)
    // does not apply; evaluate the reference formula in fp64 per pixel over
    // the whole screen
    atomicAdd(out.straddle, 1ull);
    general = true;
  }

  // --- per-pixel test coefficients (Cholesky-style forms)
  double f = cam.f, f2 = f * f;
  double if2 = 1.0 / f2;
  double Np00 = N[0] * if2, Np01 = N[1] * if2, Np11 = N[4] * if2;
  double n0 = Np00, kk = Np01 / Np00, n1 = Np11 - Np01 * kk;
  double ibz = 1.0 / bp[2];
  double ccx = cam.cx + f * (bp[0] * ibz);
  double ccy = cam.cy + f * (bp[1] * ibz);
  float cxh = (float)ccx, cyh = (float)ccy;
  float cxl = (float)(ccx - (double)cxh), cyl = (float)(ccy - (double)cyh);
  double a = Ap[0], ia = 1.0 / a, bb = Ap[1] * ia, cc = Ap[2] * ia;
  double A11s = Ap[4] - Ap[1] * bb, A12s = Ap[5] - Ap[1] * cc, A22s = Ap[8] - Ap[2] * cc;
  double d = A11s, e = A12s / d, gg = A22s - A12s * e;

  if (live && !general) {
    // --- silhouette conic Q = N - r2m A' and its dual: tile bbox
    double Q[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Q[i] = N[i] - r2m * Ap[i];
    double S00 = Q[4] * Q[8] - Q[5] * Q[5];
    double S11 = Q[0] * Q[8] - Q[2] * Q[2];
    double S22 = Q[0] * Q[4] - Q[1] * Q[1];
    double S02 = Q[1] * Q[5] - Q[2] * Q[4];
    double S12 = Q[1] * Q[2] - Q[0] * Q[5];
    double dx = S02 * S02 - S00 * S22;
    double dy = S12 * S12 - S11 * S22;
    double jlo = 0.0, jhi = (double)(cam.W - 1), ilo = 0.0, ihi = (double)(cam.H - 1);
    bool ok = (dx >= 0.0) && (dy >= 0.0) && (S22 != 0.0);
    if (ok) {
      double sx = sqrt(dx), sy = sqrt(dy);
      double iS = 1.0 / S22;
      double x1 = (S02 - sx) * iS, x2 = (S02 + sx) * iS;
      double y1 = (S12 - sy) * iS, y2 = (S12 + sy) * iS;
      double xl = x1 < x2 ? x1 : x2, xh = x1 < x2 ? x2 : x1;
      double yl = y1 < y2 ? y1 : y2, yh = y1 < y2 ? y2 : y1;
      double pjl = ceil((cam.cx + f * xl) - 0.5), pjh = floor((cam.cx + f * xh) - 0.5);
      double pil = ceil((cam.cy + f * yl) - 0.5), pih = floor((cam.cy + f * yh) - 0.5);
      // NaN-safe clamps (a NaN bound keeps the full range)
      if (pjl > jlo) jlo = pjl;
      if (pjh < jhi) jhi = pjh;
      if (pil > ilo) ilo = pil;
      if (pih < ihi) ihi = pih;
    }
    if (jlo <= jhi && ilo <= ihi) {
      int j0 = (int)jlo, j1 = (int)jhi, i0 = (int)ilo, i1 = (int)ihi;
      rect = make_int4(j0 / TILE, i0 / TILE, j1 / TILE, i1 / TILE);
      if (ok && out.tq) {
        // exact tile test data: the silhouette conic q(X, Y) = Hᵀ Q H and
        // the projected centre (inside it: q = -r2m·D there)
        double* t = out.tq + TQ_STRIDE * rk;
        t[0] = Q[0];
        t[1] = Q[1];
        t[2] = Q[4];
        t[3] = Q[2];
        t[4] = Q[5];
        t[5] = Q[8];
        t[6] = bp[0] * ibz;
        t[7] = bp[1] * ibz;
        t[8] = 0.5 / Q[0];
        t[9] = 0.5 / Q[4];
      } else if (out.tq) {
        out.tq[TQ_STRIDE * rk] = __longlong_as_double(0x7ff8000000000000ll);  // NaN: no exact test
      }
    }
  }

  if (general) {
    rect = make_int4(0, 0, cam.tiles_x - 1, cam.tiles_y - 1);
    if (out.tq) out.tq[TQ_STRIDE * rk] = __longlong_as_double(0x7ff8000000000000ll);  // every tile
    // world-frame A = R diag(s^-2) R^T, b = μ - o (render.py:116-121)
    double A[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j)
        A[3 * i + j] = ((R[3 * i + 0] * is0) * R[3 * j + 0] + (R[3 * i + 1] * is1) * R[3 * j + 1]) +
                       (R[3 * i + 2] * is2) * R[3 * j + 2];
    double* dp = reinterpret_cast<double*>(rec);
    dp[0] = b0;
    dp[1] = b1;
    dp[2] = b2;
    dp[3] = A[0];
    dp[4] = A[1];
    dp[5] = A[2];
    dp[6] = A[4];
    dp[14] = A[5];
    dp[15] = A[8];
    float* fw = reinterpret_cast<float*>(rec);
    fw[14] = (float)opac;
    fw[15] = __int_as_float(RF_GENERAL);
  } else {
    rec[0] = make_float4(cxh, cyh, cxl, cyl);
    rec[1] = make_float4((float)n0, (float)kk, (float)n1, (float)r2m);
    rec[2] = make_float4((float)a, (float)bb, (float)cc, (float)d);
    const double smx = fmax(s0, fmax(s1, s2)), smn = fmin(s0, fmin(s1, s2));
    rec[3] = make_float4((float)e, (float)gg, (float)opac,
                         __int_as_float(RF_CONIC | (smx > 4.0 * smn ? RF_ANISO : 0)));
  }
  // SH per channel; the DC coefficient is stored pre-multiplied by Y0 = C0
  // (rounded once from fp64), so the per-pixel emission starts from it
  rec[4] = make_float4((float)((double)shv[0] * SH_C0), shv[1], shv[2], shv[3]);
  rec[5] = make_float4((float)((double)shv[4] * SH_C0), shv[5], shv[6], shv[7]);
  rec[6] = make_float4((float)((double)shv[8] * SH_C0), shv[9], shv[10], shv[11]);
  // conic: t coefficients (A'b')·h of the exact-order mode, and b'_z (the
  // backward's cancellation-free peak offset)
  if (!general) rec[7] = make_float4((float)Ab[0], (float)Ab[1], (float)Ab[2], (float)bp[2]);
  // B maps the per-pixel peak offset e (conic: camera-frame diff'/b'_z;
  // general: world-frame diff) to the Gaussian frame, u = Rᵀ diff = B e:
  // conic B = b'_z Mᵀ, general B = Rᵀ; stored whitened (row k / s_k, so
  // B̃ e = Λ^{1/2} u directly) with .w = s_k (used by the backward only)
  const double sk[3] = {s0, s1, s2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double ik = 1.0 / sk[k];
    if (general)
      bf[k] = make_float4((float)(R[0 + k] * ik), (float)(R[3 + k] * ik), (float)(R[6 + k] * ik),
                          (float)sk[k]);
    else
      bf[k] = make_float4((float)(bp[2] * M[0 + k] * ik), (float)(bp[2] * M[3 + k] * ik),
                          (float)(bp[2] * M[6 + k] * ik), (float)sk[k]);
  }
  out.rects[g] = rect;  // storage order (coalesced; exports, the exact order's binning)
  if (out.tq) *reinterpret_cast<int4*>(out.tq + TQ_STRIDE * rk + 10) = rect;
  return rect;
}

// K1: persistent blocks of 128 threads stream chunks of 128 Gaussians'
// parameters (~12 KB) into shared memory with 16-B cp.async copies, double
// buffered, so the fp64 projection of one chunk overlaps the loads of the
// next; the 128-B records land at their depth-rank slots.
constexpr int PROJ_CHUNK = 128;

struct ProjStage {  // one chunk of parameters in shared memory
  float4 q[PROJ_CHUNK];
  float c[PROJ_CHUNK * 3];
  float s[PROJ_CHUNK * 3];
  float sh[PROJ_CHUNK * 12];
  float op[PROJ_CHUNK];
  uint32_t rank[PROJ_CHUNK];
};

struct ProjOutStage {  // one chunk of finished records, written out per warp
  float4 rec[PROJ_CHUNK][REC_F4];
  float4 bf[PROJ_CHUNK][3];
  int64_t rank[PROJ_CHUNK];
};

__global__ void __launch_bounds__(PROJ_CHUNK)
    k_project(const float* __restrict__ centers, const float* __restrict__ scales,
              const float* __restrict__ quats, const float* __restrict__ opacities,
              const float* __restrict__ sh, int C, int64_t P,
              const uint32_t* __restrict__ rank_of, CamDev cam, double cutoff,
              double near_plane, ProjOut out) {
  nxs_pdl_enter();
  __shared__ ProjStage st[2];
  __shared__ ProjOutStage so;
  const int tid = threadIdx.x, lane = tid & 31, wbase = tid & ~31;
  const int64_t n_chunks = (P + PROJ_CHUNK - 1) / PROJ_CHUNK;
  // full chunks stream through cp.async; a partial last chunk uses plain loads
  auto stage = [&](int buf, int64_t ch) {
    const int64_t g0 = ch * PROJ_CHUNK;
    if (g0 + PROJ_CHUNK <= P) {
      ProjStage& S = st[buf];
      const char* src_q = reinterpret_cast<const char*>(quats + 4 * g0);
      const char* src_c = reinterpret_cast<const char*>(centers + 3 * g0);
      const char* src_s = reinterpret_cast<const char*>(scales + 3 * g0);
      const char* src_o = reinterpret_cast<const char*>(opacities + g0);
      const char* src_r = reinterpret_cast<const char*>(rank_of + g0);
      const char* src_h = reinterpret_cast<const char*>(sh + (int64_t)3 * C * g0);
      for (int k = tid; k < PROJ_CHUNK * 16 / 16; k += PROJ_CHUNK)
        cp_async16(reinterpret_cast<char*>(S.q) + 16 * k, src_q + 16 * k);
      for (int k = tid; k < PROJ_CHUNK * 12 / 16; k += PROJ_CHUNK) {
        cp_async16(reinterpret_cast<char*>(S.c) + 16 * k, src_c + 16 * k);
        cp_async16(reinterpret_cast<char*>(S.s) + 16 * k, src_s + 16 * k);
      }
      for (int k = tid; k < PROJ_CHUNK * 4 / 16; k += PROJ_CHUNK) {
        cp_async16(reinterpret_cast<char*>(S.op) + 16 * k, src_o + 16 * k);
        cp_async16(reinterpret_cast<char*>(S.rank) + 16 * k, src_r + 16 * k);
      }
      for (int k = tid; k < PROJ_CHUNK * 3 * C * 4 / 16; k += PROJ_CHUNK)  // 3*C floats each
        cp_async16(reinterpret_cast<char*>(S.sh) + 16 * k, src_h + 16 * k);
    }
    cp_async_commit();
  };
  int buf = 0;
  int64_t ch = blockIdx.x;
  if (ch < n_chunks) stage(0, ch);
  for (; ch < n_chunks; ch += gridDim.x, buf ^= 1) {
    const int64_t nxt = ch + gridDim.x;
    if (nxt < n_chunks) {
      stage(buf ^ 1, nxt);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t g = ch * PROJ_CHUNK + tid;
    if (g < P) {
      GParams prm;
      int64_t r;
      const bool full = ch * PROJ_CHUNK + PROJ_CHUNK <= P;
      if (full) {
        const ProjStage& S = st[buf];
        prm.q = S.q[tid];
        prm.c0 = S.c[3 * tid + 0];
        prm.c1 = S.c[3 * tid + 1];
        prm.c2 = S.c[3 * tid + 2];
        prm.s0 = S.s[3 * tid + 0];
        prm.s1 = S.s[3 * tid + 1];
        prm.s2 = S.s[3 * tid + 2];
        prm.op = S.op[tid];
        r = S.rank[tid];
        if (C == 4) {
#pragma unroll
          for (int k = 0; k < 12; ++k) prm.shv[k] = S.sh[12 * tid + k];
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            prm.shv[4 * c] = S.sh[3 * tid + c];
            prm.shv[4 * c + 1] = prm.shv[4 * c + 2] = prm.shv[4 * c + 3] = 0.0f;
          }
        }
      } else {
        prm.q = reinterpret_cast<const float4*>(quats)[g];
        prm.c0 = centers[3 * g + 0];
        prm.c1 = centers[3 * g + 1];
        prm.c2 = centers[3 * g + 2];
        prm.s0 = scales[3 * g + 0];
        prm.s1 = scales[3 * g + 1];
        prm.s2 = scales[3 * g + 2];
        prm.op = opacities[g];
        r = rank_of[g];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) prm.shv[4 * c + k] = (k < C) ? sh[(g * 3 + c) * C + k] : 0.0f;
      }
      project_one(prm, g, r, cam, cutoff, near_plane, out, so.rec[tid], so.bf[tid]);
      so.rank[tid] = r;
      if (out.zlo_rank) out.zlo_rank[r] = __double2float_rd(out.zlo[g]);
    } else {
      so.rank[tid] = -1;
    }
    __syncwarp();
    // each store instruction writes 4 complete 128-B records (full lines)
#pragma unroll
    for (int i = 0; i < REC_F4; ++i) {
      const int k = i * 32 + lane, t = wbase + (k >> 3), part = k & 7;
      const int64_t rr = so.rank[t];
      if (rr >= 0) out.records[rr * REC_F4 + part] = so.rec[t][part];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int k = i * 32 + lane, t = wbase + k / 3, part = k - 3 * (k / 3);
      const int64_t rr = so.rank[t];
      if (rr >= 0) out.bframe[rr * 3 + part] = so.bf[t][part];
    }
    __syncthreads();  // everyone is done with `buf` and `so` before they are refilled
  }
  cp_async_wait<0>();
}

// K1 for one lazy depth phase: ranks [r0, r1) in rank order (Gaussian
// g = order[r], parameters gathered), records written as full lines at
// consecutive ranks.
__global__ void __launch_bounds__(PROJ_CHUNK)
    k_project_ranks(const float* __restrict__ centers, const float* __restrict__ scales,
                    const float* __restrict__ quats, const float* __restrict__ opacities,
                    const float* __restrict__ sh, int C, int64_t r0, int64_t r1,
                    const uint32_t* __restrict__ order, CamDev cam, double cutoff,
                    double near_plane, ProjOut out, const int* __restrict__ nd) {
  nxs_pdl_enter();
  __shared__ ProjOutStage so;
  if (nd) r1 = min(r1, r0 + (int64_t)*nd);
  const int tid = threadIdx.x, lane = tid & 31, wbase = tid & ~31;
  const int64_t r = r0 + (int64_t)blockIdx.x * PROJ_CHUNK + tid;
  bool has_rect = false;
  if (r < r1) {
    const int64_t g = order[r];
    GParams prm;
    prm.q = reinterpret_cast<const float4*>(quats)[g];
    prm.c0 = centers[3 * g + 0];
    prm.c1 = centers[3 * g + 1];
    prm.c2 = centers[3 * g + 2];
    prm.s0 = scales[3 * g + 0];
    prm.s1 = scales[3 * g + 1];
    prm.s2 = scales[3 * g + 2];
    prm.op = opacities[g];
    if (C == 4) {
      const float4* h = reinterpret_cast<const float4*>(sh + g * 12);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float4 v = h[c];
        prm.shv[4 * c] = v.x;
        prm.shv[4 * c + 1] = v.y;
        prm.shv[4 * c + 2] = v.z;
        prm.shv[4 * c + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        prm.shv[4 * c] = sh[g * 3 + c];
        prm.shv[4 * c + 1] = prm.shv[4 * c + 2] = prm.shv[4 * c + 3] = 0.0f;
      }
    }
    const int4 rect = project_one(prm, g, r, cam, cutoff, near_plane, out, so.rec[tid], so.bf[tid]);
    if (out.zlo_rank) out.zlo_rank[r] = __double2float_rd(out.zlo[g]);
    so.rank[tid] = r;
    has_rect = rect.x >= 0;
  } else {
    so.rank[tid] = -1;
  }
  if (out.live) {  // warp-aggregated append of the ranks with a rectangle
    const unsigned m = __ballot_sync(0xffffffffu, has_rect);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned long long at = 0;
      if (lane == leader) at = atomicAdd(out.n_live, (unsigned long long)__popc(m));
      at = __shfl_sync(0xffffffffu, at, leader);
      if (has_rect) out.live[at + __popc(m & ((1u << lane) - 1u))] = (uint32_t)r;
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < REC_F4; ++i) {
    const int k = i * 32 + lane, t = wbase + (k >> 3), part = k & 7;
    const int64_t rr = so.rank[t];
    if (rr >= 0) out.records[rr * REC_F4 + part] = so.rec[t][part];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int k = i * 32 + lane, t = wbase + k / 3, part = k - 3 * (k / 3);
    const int64_t rr = so.rank[t];
    if (rr >= 0) out.bframe[rr * 3 + part] = so.bf[t][part];
  }
}

// Exact tile culling: does the silhouette ellipse q <= 0 meet the tile's
// pixel-centre rectangle (normalised coordinates)?  The projected centre is
// inside the ellipse, so it meets the (convex) rectangle iff the centre is
// in it or q <= 0 somewhere on one of its edges (the minimum of q along an
// edge line is the clamped vertex of a convex quadratic).  Conservative:
// every valid pixel lies strictly inside the margin ellipse (r2m).  fp64,
// IEEE op by op (this file is built with --fmad=false), restated in
// oracle/binning_oracle.c.
__device__ __forceinline__ bool tile_hit(const double* __restrict__ tq, int64_t r, int tx, int ty,
                                         const CamDev& cam, double inv_f) {
  if (!tq) return true;  // culling off (exact order: full binning, bbox tiles)
  const double* t = tq + TQ_STRIDE * r;
  const double q00 = t[0];
  if (!(q00 == q00)) return true;  // no exact test for this Gaussian
  const double q01 = t[1], q11 = t[2], q02 = t[3], q12 = t[4], q22 = t[5];
  const double c0 = t[6], c1 = t[7], h00 = t[8], h11 = t[9];
  const int jx0 = tx * TILE, iy0 = ty * TILE;
  const int jx1 = min(jx0 + TILE - 1, cam.W - 1), iy1 = min(iy0 + TILE - 1, cam.H - 1);
  const double x0 = (((double)jx0 + 0.5) - cam.cx) * inv_f, x1 = (((double)jx1 + 0.5) - cam.cx) * inv_f;
  const double y0 = (((double)iy0 + 0.5) - cam.cy) * inv_f, y1 = (((double)iy1 + 0.5) - cam.cy) * inv_f;
  if (c0 >= x0 && c0 <= x1 && c1 >= y0 && c1 <= y1) return true;
  for (int k = 0; k < 2; ++k) {  // vertical edges X = xe: q(Y) = q11 Y² + b Y + c
    const double xe = k ? x1 : x0;
    const double b = 2.0 * (q01 * xe + q12);
    const double c = (q00 * xe * xe + 2.0 * q02 * xe) + q22;
    double yv = -b * h11;
    yv = yv < y0 ? y0 : (yv > y1 ? y1 : yv);
    if ((q11 * yv + b) * yv + c <= 0.0) return true;
  }
  for (int k = 0; k < 2; ++k) {  // horizontal edges Y = ye: q(X) = q00 X² + b X + c
    const double ye = k ? y1 : y0;
    const double b = 2.0 * (q01 * ye + q02);
    const double c = (q11 * ye * ye + 2.0 * q12 * ye) + q22;
    double xv = -b * h00;
    xv = xv < x0 ? x0 : (xv > x1 ? x1 : xv);
    if ((q00 * xv + b) * xv + c <= 0.0) return true;
  }
  return false;
}

// K2a: per rank of [r0, r1), the number of still-active tiles in its rect.
// KSUB lanes per rank: lanes stride over the candidate tiles of the rect,
// so the fp64 exact tile tests of big rects run in parallel.  A depth phase
// of a few 10^4 near (big) Gaussians uses a warp per rank; a full binning of
// all ranks (mostly small rects) eight lanes.
template <int KSUB>
__global__ void __launch_bounds__(256)
    k_count_active(const int4* __restrict__ rects, const uint32_t* __restrict__ order,
                   int64_t r0, int64_t r1, int tiles_x, const uint8_t* __restrict__ active,
                   const unsigned int* __restrict__ gate, unsigned long long* __restrict__ counts,
                   const int* __restrict__ nd, const double* __restrict__ tq, CamDev cam) {
  nxs_pdl_enter();
  // later phases: nothing to count when the previous forward left no tile
  // active (the host then stops before reading the counts)
  if (gate && *gate == 0u) return;
  const int lane = threadIdx.x & 31, sl = lane & (KSUB - 1);
  const int64_t r = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / KSUB;
  const int64_t rn = nd ? min(r1, r0 + (int64_t)*nd) : r1;
  const bool live = r < rn;
  unsigned n = 0;
  if (live) {
    const int4 rc = tq ? tq_rect(tq, r) : rects[order[r]];
    if (rc.x >= 0) {
      const double inv_f = cam.inv_f;  // = 1.0 / cam.f (host, IEEE)
      const int w = rc.z - rc.x + 1, nt = w * (rc.w - rc.y + 1);
      for (int k = sl; k < nt; k += KSUB) {
        const int tx = rc.x + k % w, ty = rc.y + k / w;
        n += (active[ty * tiles_x + tx] && tile_hit(tq, r, tx, ty, cam, inv_f)) ? 1u : 0u;
      }
    }
  }
  for (int o = KSUB / 2; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if (sl == 0 && r < r1) counts[r - r0] = live ? n : 0ull;  // padding ranks count 0
}

// K2b: emit (tile, rank) pairs of active tiles at the exclusive-scan
// offsets, in rank order (so a stable sort by tile keeps ranks ascending);
// KSUB lanes per rank, a ballot orders each KSUB-tile group.
template <int KSUB>
__global__ void __launch_bounds__(256)
    k_emit_pairs(const int4* __restrict__ rects, const uint32_t* __restrict__ order,
                 const unsigned long long* __restrict__ offsets, int64_t r0, int64_t r1,
                 int tiles_x, const uint8_t* __restrict__ active, uint32_t* __restrict__ keys,
                 uint32_t* __restrict__ vals, const int* __restrict__ nd, unsigned long long cap,
                 const double* __restrict__ tq, CamDev cam) {
  nxs_pdl_enter();
  if (nd) r1 = min(r1, r0 + (int64_t)*nd);
  const int lane = threadIdx.x & 31, sl = lane & (KSUB - 1), grp = lane / KSUB;
  const int64_t r = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / KSUB;
  int4 rc = make_int4(-1, -1, -1, -1);
  if (r < r1) rc = tq ? tq_rect(tq, r) : rects[order[r]];
  const int w = rc.z - rc.x + 1;
  const int nt = rc.x >= 0 ? w * (rc.w - rc.y + 1) : 0;
  int nmax = nt;  // the warp loops to its largest rect (ballots need every lane)
  for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
  const double inv_f = cam.inv_f;  // = 1.0 / cam.f (host, IEEE)
  unsigned long long o = nt > 0 ? offsets[r - r0] : 0ull;
  for (int base = 0; base < nmax; base += KSUB) {
    const int k = base + sl;
    const int tx = rc.x + (w > 0 ? k % w : 0), ty = rc.y + (w > 0 ? k / w : 0);
    const int t = ty * tiles_x + tx;
    const bool hit = k < nt && active[t] && tile_hit(tq, r, tx, ty, cam, inv_f);
    const unsigned m = KSUB == 32 ? __ballot_sync(0xffffffffu, hit)
                                  : (__ballot_sync(0xffffffffu, hit) >> (grp * KSUB)) &
                                        ((1u << KSUB) - 1u);
    if (hit) {
      const unsigned long long q = o + __popc(m & ((1u << sl) - 1u));
      if (q < cap) {  // (the legacy path sizes the buffer exactly)
        keys[q] = (uint32_t)t;
        vals[q] = (uint32_t)r;
      }
    }
    o += __popc(m);
  }
}

// ---------------------------------------------------------------------------
// Tile-major binning (counting sort by tile): per-tile hit counts, one scan
// over the tiles (ranges, total, largest list), emission at per-tile atomic
// cursors, and a per-tile sort of each list by rank.  Replaces the per-rank
// scan + the radix sort of (tile, rank) pairs by tile: a rank order is
// unique, so the sorted lists equal the stable sort's bit for bit.
// ---------------------------------------------------------------------------
template <int KSUB>
__global__ void __launch_bounds__(256)
    k_count_tiles(const int4* __restrict__ rects, const uint32_t* __restrict__ order,
                  int64_t r0, int64_t r1, int tiles_x, const uint8_t* __restrict__ active,
                  const unsigned int* __restrict__ gate, unsigned int* __restrict__ tile_cnt,
                  const int* __restrict__ nd, const double* __restrict__ tq, CamDev cam) {
  nxs_pdl_enter();
  if (gate && *gate == 0u) return;
  const int sl = threadIdx.x & (KSUB - 1);
  const int64_t r = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / KSUB;
  const int64_t rn = nd ? min(r1, r0 + (int64_t)*nd) : r1;
  if (r >= rn) return;
  const int4 rc = tq ? tq_rect(tq, r) : rects[order[r]];
  if (rc.x < 0) return;
  const double inv_f = cam.inv_f;  // = 1.0 / cam.f (host, IEEE)
  const int w = rc.z - rc.x + 1, nt = w * (rc.w - rc.y + 1);
  for (int k = sl; k < nt; k += KSUB) {
    const int tx = rc.x + k % w, ty = rc.y + k / w;
    const int t = ty * tiles_x + tx;
    if (active[t] && tile_hit(tq, r, tx, ty, cam, inv_f)) atomicAdd(&tile_cnt[t], 1u);
  }
}

// one block: exclusive scan of the tile counts -> ranges [off, off + cnt),
// the total (and whether it exceeds cap), the longest list; the counts are
// reset to zero to serve as the emission cursors
constexpr int TSCAN_THREADS = 1024;
constexpr int TSCAN_STAGED = 32768;  // tiles staged in shared memory (128 KB)
__global__ void __launch_bounds__(TSCAN_THREADS)
    k_tile_scan(unsigned int* __restrict__ tile_cnt, int n_tiles, int2* __restrict__ ranges,
                unsigned long long* __restrict__ total, unsigned long long* __restrict__ maxseg,
                unsigned long long cap, unsigned long long* __restrict__ overflow, int seg_max) {
  nxs_pdl_enter();
  typedef cub::BlockScan<unsigned long long, TSCAN_THREADS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned int s_max;
  extern __shared__ unsigned int s_c[];  // staged counts, then exclusive offsets
  const bool staged = n_tiles <= TSCAN_STAGED;
  const int tid = threadIdx.x;
  if (tid == 0) s_max = 0;
  if (staged) {  // coalesced in, counts reset (they are the emission cursors)
    for (int t = tid; t < n_tiles; t += TSCAN_THREADS) {
      s_c[t] = tile_cnt[t];
      tile_cnt[t] = 0u;
    }
    __syncthreads();
  }
  const int per = (n_tiles + TSCAN_THREADS - 1) / TSCAN_THREADS;
  const int lo = min(n_tiles, tid * per), hi = min(n_tiles, lo + per);
  unsigned long long sum = 0;
  unsigned int mx = 0;
  for (int t = lo; t < hi; ++t) {
    const unsigned int c = staged ? s_c[t] : tile_cnt[t];
    sum += c;
    mx = max(mx, c);
  }
  unsigned long long off, all;
  Scan(tmp).ExclusiveSum(sum, off, all);
  atomicMax(&s_max, mx);
  if (staged) {
    for (int t = lo; t < hi; ++t) {
      const unsigned int c = s_c[t];
      s_c[t] = (unsigned int)min(off, cap);
      off += c;
    }
    __syncthreads();
    // (a device-sized buffer too small: lists clamped to it, the pass is
    // flagged and redone — no list may reach past the buffer meanwhile)
    const unsigned int capped = (unsigned int)min(all, cap);
    for (int t = tid; t < n_tiles; t += TSCAN_THREADS)
      ranges[t] = make_int2((int)s_c[t], (int)(t + 1 < n_tiles ? s_c[t + 1] : capped));
  } else {
    __syncthreads();
    for (int t = lo; t < hi; ++t) {
      const unsigned int c = tile_cnt[t];
      ranges[t] = make_int2((int)min(off, cap), (int)min(off + c, cap));
      off += c;
      tile_cnt[t] = 0u;
    }
  }
  __syncthreads();
  if (tid == 0) {
    *total = all;
    *maxseg = s_max;
    if (overflow && (all > cap || (int)s_max > seg_max)) atomicAdd(overflow, 1ull);
  }
}

// per-tile list capacities for the view's next device-sized pass, from this
// pass's phase-0 lists: cap_t = n_t + n_t/8 + 8, base = exclusive scan
__global__ void __launch_bounds__(TSCAN_THREADS)
    k_make_bases(const int2* __restrict__ ranges, int n_tiles, unsigned int* __restrict__ base) {
  nxs_pdl_enter();
  typedef cub::BlockScan<unsigned long long, TSCAN_THREADS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int per = (n_tiles + TSCAN_THREADS - 1) / TSCAN_THREADS;
  const int lo = min(n_tiles, (int)threadIdx.x * per), hi = min(n_tiles, lo + per);
  auto cap_of = [&](int t) {
    const int2 rg = ranges[t];
    const unsigned int n = (unsigned int)(rg.y - rg.x);
    return n + n / 8 + 8u;
  };
  unsigned long long sum = 0;
  for (int t = lo; t < hi; ++t) sum += cap_of(t);
  unsigned long long off, all;
  Scan(tmp).ExclusiveSum(sum, off, all);
  for (int t = lo; t < hi; ++t) {
    base[t] = (unsigned int)off;
    off += cap_of(t);
  }
  if (threadIdx.x == 0) base[n_tiles] = (unsigned int)all;
}

template <int KSUB>
__global__ void __launch_bounds__(256)
    k_emit_tiles(const int4* __restrict__ rects, const uint32_t* __restrict__ order, int64_t r0,
                 int64_t r1, int tiles_x, const uint8_t* __restrict__ active,
                 const int2* __restrict__ ranges, unsigned int* __restrict__ cursor,
                 uint32_t* __restrict__ vals, const int* __restrict__ nd, unsigned long long cap,
                 const double* __restrict__ tq, CamDev cam, const unsigned int* __restrict__ base,
                 unsigned long long* __restrict__ overflow, const uint32_t* __restrict__ live,
                 const unsigned long long* __restrict__ n_live) {
  nxs_pdl_enter();
  const int sl = threadIdx.x & (KSUB - 1);
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / KSUB;
  int64_t r;
  if (live) {  // only the phase's ranks with a tile rectangle (k_project_ranks)
    if (i >= (int64_t)*n_live) return;
    r = live[i];
  } else {
    r = r0 + i;
    const int64_t rn = nd ? min(r1, r0 + (int64_t)*nd) : r1;
    if (r >= rn) return;
  }
  const int4 rc = tq ? tq_rect(tq, r) : rects[order[r]];
  if (rc.x < 0) return;
  const double inv_f = cam.inv_f;  // = 1.0 / cam.f (host, IEEE)
  const int w = rc.z - rc.x + 1, nt = w * (rc.w - rc.y + 1);
  for (int k = sl; k < nt; k += KSUB) {
    const int tx = rc.x + k % w, ty = rc.y + k / w;
    const int t = ty * tiles_x + tx;
    if (active[t] && tile_hit(tq, r, tx, ty, cam, inv_f)) {
      if (base) {  // per-tile capacities from the view's last call (no count pass)
        const unsigned int q = atomicAdd(&cursor[t], 1u);
        if (q < base[t + 1] - base[t]) vals[base[t] + q] = (uint32_t)r;
        else atomicAdd(overflow, 1ull);  // (the pass is redone with exact counts)
      } else {
        const unsigned long long q = (unsigned long long)ranges[t].x + atomicAdd(&cursor[t], 1u);
        if (q < cap) vals[q] = (uint32_t)r;  // (a device-sized buffer too small is flagged)
      }
    }
  }
}

// Sort v[0, n) (distinct ranks, n <= 32K) ascending with one warp: a
// bitonic network over 32K register keys (element i*32 + lane; pads
// 0xffffffff sort last).  Strides below 32 pair lanes (one shuffle per
// key), larger strides pair a lane's own registers.  O(log² n) steps
// against the O(n²/32) of rank counting (seg sort 13.6 -> 11.0 us at C3).
// (Fully unrolled: keep K small — a 16-key version of the bin sort blew
// the instruction cache, 15 -> 70 us.)
template <int K>
__device__ __forceinline__ void warp_bitonic(uint32_t* __restrict__ v, int n, int lane) {
  uint32_t k[K];
#pragma unroll
  for (int i = 0; i < K; ++i) k[i] = i * 32 + lane < n ? v[i * 32 + lane] : 0xffffffffu;
#pragma unroll
  for (int size = 2; size <= 32 * K; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int s = stride >> 5;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i & s) continue;
          const bool up = ((i * 32 + lane) & size) == 0;
          const uint32_t a = k[i], b = k[i | s];
          k[i] = up ? min(a, b) : max(a, b);
          k[i | s] = up ? max(a, b) : min(a, b);
        }
      } else {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, k[i], stride);
          const bool up = ((i * 32 + lane) & size) == 0;
          const bool lower = (lane & stride) == 0;
          k[i] = (up == lower) ? min(k[i], o) : max(k[i], o);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
    if (i * 32 + lane < n) v[i * 32 + lane] = k[i];
}

// one block per tile: sort its list (distinct ranks) ascending in shared
// memory — rank counting for short lists, a bitonic network up to SEG_MAX;
// zeroes the tile's cursor for the next phase
constexpr int SEG_THREADS = 256;
constexpr int SEG_WARP_MAX = 256;  // lists up to this long: one warp each
// one warp per tile: lists of up to SEG_WARP_MAX by a register bitonic
// network (warp_bitonic); zeroes every tile's cursor
__global__ void __launch_bounds__(256)
    k_seg_sort_warp(uint32_t* __restrict__ vals, int2* __restrict__ ranges,
                    unsigned int* __restrict__ cursor, int n_tiles, unsigned long long cap,
                    const unsigned int* __restrict__ base, unsigned long long* __restrict__ total,
                    unsigned long long* __restrict__ overflow) {
  nxs_pdl_enter();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + w;
  __shared__ unsigned long long s_tot;  // the block's pairs: one global atomic per block
  if (threadIdx.x == 0) s_tot = 0ull;
  __syncthreads();
  const bool valid = t < n_tiles;
  int2 rg = make_int2(0, 0);
  if (valid) {
    if (base) {  // lists emitted at per-tile capacities: the range is [base, base + count)
      const unsigned int b0 = base[t];
      const int n0 = (int)min(cursor[t], base[t + 1] - b0);
      rg = make_int2((int)b0, (int)b0 + n0);
      __syncwarp();
      if (lane == 0) {
        ranges[t] = rg;
        atomicAdd(&s_tot, (unsigned long long)n0);
        if (n0 > SEG_MAX) atomicAdd(overflow, 1ull);
      }
    } else {
      rg = ranges[t];
    }
    if (lane == 0) cursor[t] = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0 && base && s_tot) atomicAdd(total, s_tot);
  if (!valid) return;
  const int n = rg.y - rg.x;
  if (n <= 1 || n > SEG_WARP_MAX || (unsigned long long)rg.y > cap) return;
  uint32_t* v = vals + rg.x;
  // bitonic network in registers: K keys per lane, element i*32 + lane
  if (n <= 32) warp_bitonic<1>(v, n, lane);
  else if (n <= 64) warp_bitonic<2>(v, n, lane);
  else if (n <= 128) warp_bitonic<4>(v, n, lane);
  else warp_bitonic<8>(v, n, lane);
}
// one block per tile for the longer lists (bitonic up to SEG_MAX)
__global__ void __launch_bounds__(SEG_THREADS)
    k_seg_sort(uint32_t* __restrict__ vals, const int2* __restrict__ ranges, int n_tiles,
               unsigned long long cap) {
  nxs_pdl_enter();
  __shared__ uint32_t s_k[SEG_MAX];
  const int tid = threadIdx.x;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
  const int2 rg = ranges[t];
  const int n = rg.y - rg.x;
  if (n <= SEG_WARP_MAX || n > SEG_MAX || (unsigned long long)rg.y > cap) continue;
  uint32_t* v = vals + rg.x;
  if (n <= SEG_THREADS) {
    const uint32_t k = tid < n ? v[tid] : 0u;
    if (tid < n) s_k[tid] = k;
    __syncthreads();
    if (tid < n) {
      int pos = 0;
      for (int j = 0; j < n; ++j) pos += s_k[j] < k ? 1 : 0;
      v[pos] = k;
    }
    return;
  }
  int p2 = SEG_THREADS * 2;
  while (p2 < n) p2 <<= 1;
  for (int i = tid; i < p2; i += SEG_THREADS) s_k[i] = i < n ? v[i] : 0xffffffffu;
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < (p2 >> 1); i += SEG_THREADS) {
        const int a = 2 * i - (i & (stride - 1)), b = a + stride;
        const bool up = (a & size) == 0;
        const uint32_t x = s_k[a], y = s_k[b];
        if ((x > y) == up) {
          s_k[a] = y;
          s_k[b] = x;
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < n; i += SEG_THREADS) v[i] = s_k[i];
  __syncthreads();  // (s_k is reused by the block's next tile)
  }
}

void launch_count_tiles(const int4* rects, const uint32_t* order, int64_t r0, int64_t r1,
                        int tiles_x, const uint8_t* active, const unsigned int* gate,
                        unsigned int* tile_cnt, const double* tq, const CamDev& cam,
                        cudaStream_t s, const int* nd) {
  if (r1 <= r0) return;
  if (r1 - r0 <= 262144)
    nxs_launch(k_count_tiles<32>, (unsigned)((r1 - r0 + 7) / 8), 256, 0, s, 
        rects, order, r0, r1, tiles_x, active, gate, tile_cnt, nd, tq, cam);
  else
    nxs_launch(k_count_tiles<8>, (unsigned)((r1 - r0 + 31) / 32), 256, 0, s, 
        rects, order, r0, r1, tiles_x, active, gate, tile_cnt, nd, tq, cam);
}
void launch_tile_scan(unsigned int* tile_cnt, int n_tiles, int2* ranges, unsigned long long* total,
                      unsigned long long* maxseg, unsigned long long cap,
                      unsigned long long* overflow, cudaStream_t s) {
  static unsigned long long attr_dev = 0;
  once_per_device(attr_dev, [] {
    cudaFuncSetAttribute(k_tile_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TSCAN_STAGED * (int)sizeof(unsigned int));
  });
  const size_t dyn = n_tiles <= TSCAN_STAGED ? (size_t)n_tiles * sizeof(unsigned int) : 0;
  nxs_launch(k_tile_scan, 1, TSCAN_THREADS, dyn, s, tile_cnt, n_tiles, ranges, total, maxseg, cap,
                                            overflow, SEG_MAX);
}
void launch_emit_tiles(const int4* rects, const uint32_t* order, int64_t r0, int64_t r1,
                       int tiles_x, const uint8_t* active, const int2* ranges,
                       unsigned int* cursor, uint32_t* vals, const double* tq, const CamDev& cam,
                       cudaStream_t s, const int* nd, unsigned long long cap,
                       const unsigned int* base, unsigned long long* overflow,
                       const uint32_t* live, const unsigned long long* n_live) {
  if (r1 <= r0) return;
#ifndef NXS_EMIT_KSUB
#define NXS_EMIT_KSUB 32
#endif
  constexpr int KS = NXS_EMIT_KSUB;  // lanes per rank for a near phase (big rects)
  if (r1 - r0 <= 262144)
    nxs_launch(k_emit_tiles<KS>, (unsigned)((r1 - r0 + 256 / KS - 1) / (256 / KS)), 256, 0, s, 
        rects, order, r0, r1, tiles_x, active, ranges, cursor, vals, nd, cap, tq, cam, base,
        overflow, live, n_live);
  else
    nxs_launch(k_emit_tiles<8>, (unsigned)((r1 - r0 + 31) / 32), 256, 0, s, 
        rects, order, r0, r1, tiles_x, active, ranges, cursor, vals, nd, cap, tq, cam, base,
        overflow, live, n_live);
}
void launch_make_bases(const int2* ranges, int n_tiles, unsigned int* base, cudaStream_t s) {
  nxs_launch(k_make_bases, 1, TSCAN_THREADS, 0, s, ranges, n_tiles, base);
}

// After a device-sized pass: re-derive the per-tile capacities from the
// counts that pass found (a scene that moves between calls, e.g. under
// Adam, drifts away from the exact pass's counts), each capped at the
// host's longest-list bound and committed only when the total still fits
// the pair buffer the host sized (`bound`); otherwise the old bases stay.
__global__ void __launch_bounds__(TSCAN_THREADS)
    k_refresh_bases(const int2* __restrict__ ranges, int n_tiles, unsigned int* __restrict__ base,
                    unsigned long long bound, unsigned int maxcap) {
  nxs_pdl_enter();
  typedef cub::BlockScan<unsigned long long, TSCAN_THREADS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int per = (n_tiles + TSCAN_THREADS - 1) / TSCAN_THREADS;
  const int lo = min(n_tiles, (int)threadIdx.x * per), hi = min(n_tiles, lo + per);
  auto cap_of = [&](int t) {
    const int2 rg = ranges[t];
    const unsigned int n = (unsigned int)max(0, rg.y - rg.x);
    return min(n + n / 8 + 8u, maxcap);
  };
  unsigned long long sum = 0;
  for (int t = lo; t < hi; ++t) sum += cap_of(t);
  unsigned long long off, all;
  Scan(tmp).ExclusiveSum(sum, off, all);
  if (all > bound) return;  // (block-uniform)
  __syncthreads();          // every thread has read its ranges before base moves
  for (int t = lo; t < hi; ++t) {
    base[t] = (unsigned int)off;
    off += cap_of(t);
  }
  if (threadIdx.x == 0) base[n_tiles] = (unsigned int)all;
}
void launch_refresh_bases(const int2* ranges, int n_tiles, unsigned int* base,
                          unsigned long long bound, unsigned int maxcap, cudaStream_t s) {
  nxs_launch(k_refresh_bases, 1, TSCAN_THREADS, 0, s, ranges, n_tiles, base, bound, maxcap);
}

// Export: gather each tile's list [ranges[t].x, ranges[t].y) to the compact
// offset dst_off[t] (lists laid out at per-tile capacities have gaps).
__global__ void k_compact_lists(const uint32_t* __restrict__ src, const int2* __restrict__ ranges,
                                const int* __restrict__ dst_off, int n_tiles,
                                uint32_t* __restrict__ dst, int2* __restrict__ dst_ranges) {
  nxs_pdl_enter();
  const int t = blockIdx.x;
  if (t >= n_tiles) return;
  const int2 r = ranges[t];
  const int o = dst_off[t], n = max(0, r.y - r.x);
  if (threadIdx.x == 0 && dst_ranges) dst_ranges[t] = make_int2(o, o + n);
  if (dst)
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[o + i] = src[r.x + i];
}
void launch_compact_lists(const uint32_t* src, const int2* ranges, const int* dst_off,
                          int n_tiles, uint32_t* dst, int2* dst_ranges, cudaStream_t s) {
  if (n_tiles > 0)
    nxs_launch(k_compact_lists, n_tiles, 128, 0, s, src, ranges, dst_off, n_tiles, dst, dst_ranges);
}
void launch_seg_sort(uint32_t* vals, int2* ranges, unsigned int* cursor, int n_tiles,
                     unsigned long long cap, cudaStream_t s, long long max_seg,
                     const unsigned int* base, unsigned long long* total,
                     unsigned long long* overflow) {
  if (n_tiles <= 0) return;
  nxs_launch(k_seg_sort_warp, (n_tiles + 7) / 8, 256, 0, s, vals, ranges, cursor, n_tiles, cap, base,
                                                    total, overflow);
  // (max_seg < 0: unknown on the host)
  if (max_seg < 0 || max_seg > SEG_WARP_MAX) {  // a persistent grid: most tiles are short
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    nxs_launch(k_seg_sort, std::min(n_tiles, sms * 4), SEG_THREADS, 0, s, vals, ranges, n_tiles, cap);
  }
}

__global__ void k_tile_ranges(const uint32_t* __restrict__ keys, int64_t n,
                              int2* __restrict__ ranges) {
  nxs_pdl_enter();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t t = keys[i];
  if (t == 0xffffffffu) return;  // padding of a device-sized pair buffer (sorted last)
  if (i == 0 || keys[i - 1] != t) ranges[t].x = (int)i;
  if (i == n - 1 || keys[i + 1] != t) ranges[t].y = (int)(i + 1);
}

// host launchers
void launch_depth(const float* centers, const float* scales, const float* quats,
                  const float* opacities, int64_t P, const CamDev& cam, double cutoff, int zmode,
                  double* depth, unsigned long long* key64, uint32_t* idx,
                  unsigned long long* kminmax, cudaStream_t s) {
  if (P == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!zmode && (reinterpret_cast<uintptr_t>(centers) & 15) == 0) {
    const int64_t nt = (P + 3) / 4;
    nxs_launch(k_depth4, (unsigned)((nt + 255) / 256), 256, 0, s,
               reinterpret_cast<const float4*>(centers), P, cam, depth, key64, idx, kminmax);
    return;
  }
  const unsigned grid = (unsigned)std::min<int64_t>((P + 255) / 256, (int64_t)sms * 8);
  nxs_launch(k_depth, grid, 256, 0, s, centers, scales, quats, opacities, P, cam, cutoff, zmode, depth,
                               key64, idx, kminmax);
}
void launch_key32(const double* depth, int64_t P, const unsigned long long* kminmax,
                  uint32_t* key, cudaStream_t s) {
  if (P == 0) return;
  nxs_launch(k_key32, (unsigned)((P + 255) / 256), 256, 0, s, depth, P, kminmax, key);
}
void launch_dkeys(const double* depth, int64_t P, unsigned long long* key64, cudaStream_t s) {
  if (P == 0) return;
  nxs_launch(k_dkeys, (unsigned)((P + 255) / 256), 256, 0, s, depth, P, key64);
}
void launch_key_fixup(const uint32_t* key, uint32_t* idx, const double* depth, int64_t P,
                      unsigned long long* overflow, cudaStream_t s, int shift, const int* nd) {
  if (P == 0) return;
  nxs_launch(k_key_fixup, (unsigned)((P + 255) / 256), 256, 0, s, key, idx, depth, P, shift, overflow,
                                                          nd);
}
void launch_chunk_key(const float* centers, const float* scales, const float* quats,
                      const float* opacities, int64_t P, const CamDev& cam, double cutoff,
                      const uint32_t* rank_c, int chunk, double* zlo, unsigned long long* key64,
                      uint32_t* idx, cudaStream_t s) {
  if (P == 0) return;
  nxs_launch(k_chunk_key, (unsigned)((P + 255) / 256), 256, 0, s, centers, scales, quats, opacities, P,
                                                          cam, cutoff, rank_c, chunk, zlo, key64,
                                                          idx);
}
// false when the chunk is too large for one block (use the global sort)
bool launch_chunk_sort(const uint32_t* order_c, const double* zlo, int64_t P, int chunk,
                       uint32_t* order_out, cudaStream_t s, const int* nd) {
  if (P == 0) return true;
  const unsigned grid = (unsigned)((P + chunk - 1) / chunk);
  if (chunk <= 128)
    nxs_launch(k_chunk_sort<128, 1>, grid, 128, 0, s, order_c, zlo, P, chunk, order_out, nd);
  else if (chunk <= 512)
    nxs_launch(k_chunk_sort<128, 4>, grid, 128, 0, s, order_c, zlo, P, chunk, order_out, nd);
  else if (chunk <= 2048)
    nxs_launch(k_chunk_sort<256, 8>, grid, 256, 0, s, order_c, zlo, P, chunk, order_out, nd);
  else
    return false;
  return true;
}
void launch_rank_of(const uint32_t* order, int64_t P, uint32_t* rank_of, cudaStream_t s) {
  if (P == 0) return;
  nxs_launch(k_rank_of, (unsigned)((P + 255) / 256), 256, 0, s, order, 0, P, rank_of, nullptr);
}
void launch_rank_of_range(const uint32_t* order, int64_t r0, int64_t r1, uint32_t* rank_of,
                          cudaStream_t s, const int* nd) {
  if (r1 <= r0) return;
  nxs_launch(k_rank_of, (unsigned)((r1 - r0 + 255) / 256), 256, 0, s, order, r0, r1, rank_of, nd);
}
__global__ void k_gather_keys(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ key,
                              int64_t n, uint32_t* __restrict__ out) {
  nxs_pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = key[idx[i]];
}
__global__ void k_clear_rects(const uint32_t* __restrict__ order, int64_t r0, int64_t r1,
                              int4* __restrict__ rects) {
  nxs_pdl_enter();
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < r1) rects[order[r]] = make_int4(-1, -1, -1, -1);
}
__global__ void k_iota(uint32_t* __restrict__ a, int64_t n) {
  nxs_pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (uint32_t)i;
}
// the device-sized phase-0 check, packed in host_small's layout:
// [2] straddle, [3] active tiles, [16..) phase bounds, [24] phase-0
// Gaussians, [25] overflow flags, [26] pair total
__global__ void k_pack_check(const unsigned long long* __restrict__ dsmall,
                             const long long* __restrict__ dsel, int n_ph,
                             unsigned long long* __restrict__ out) {
  nxs_pdl_enter();
  const int i = threadIdx.x;
  if (i >= 27) return;
  unsigned long long v = 0ull;
  if (i == 2) v = dsmall[0];
  else if (i == 3) v = (unsigned int)(dsmall[5] & 0xffffffffull);
  else if (i >= 16 && i < 16 + 2 * n_ph) v = (unsigned long long)dsel[i - 16];
  else if (i == 24) v = (unsigned int)*reinterpret_cast<const int*>(dsel + 48);
  else if (i == 25) v = dsmall[10];
  else if (i == 26) v = dsmall[11];
  out[i] = v;
}
// start of a forward: the small counters (dsmall; [6] = min-key init), every
// tile active, the phase-0 carry/ranges cleared and the phase targets — one
// launch instead of a string of memsets and a host copy
struct PhaseTargets {
  long long v[4];
};
__global__ void k_call_init(unsigned long long* __restrict__ dsmall, uint8_t* __restrict__ active,
                            int32_t* __restrict__ cum0, int2* __restrict__ ranges0,
                            unsigned int* __restrict__ tile_cnt, int n_tiles,
                            long long* __restrict__ dtgt, PhaseTargets tgt, int n_tgt,
                            unsigned int* __restrict__ hist) {
  nxs_pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (hist && i <= 4096) hist[i] = 0u;  // (bins and the k_key32_hist_select ticket)
  if (i < 16) dsmall[i] = (i == 6) ? ~0ull : 0ull;
  if (dtgt && i < n_tgt) dtgt[i] = tgt.v[i];
  if (i < n_tiles) {
    active[i] = 1;
    cum0[i] = 0;
    ranges0[i] = make_int2(0, 0);
    tile_cnt[i] = 0u;
  }
}
void launch_call_init(unsigned long long* dsmall, uint8_t* active, int32_t* cum0, int2* ranges0,
                      unsigned int* tile_cnt, int n_tiles, long long* dtgt, const int64_t* tgt,
                      int n_tgt, unsigned int* hist, cudaStream_t s) {
  PhaseTargets t{};
  for (int i = 0; i < n_tgt && i < 4; ++i) t.v[i] = tgt[i];
  const int n = std::max(n_tiles, 4097);
  nxs_launch(k_call_init, (n + 255) / 256, 256, 0, s, dsmall, active, cum0, ranges0, tile_cnt, n_tiles, dtgt, t,
                                              std::min(n_tgt, 4), hist);
}
void launch_pack_check(const unsigned long long* dsmall, const long long* dsel, int n_ph,
                       unsigned long long* out, cudaStream_t s) {
  nxs_launch(k_pack_check, 1, 32, 0, s, dsmall, dsel, n_ph, out);
}
// exact order over depth phases: a lower bound of the depth key (z_lo) of
// every Gaussian in the key bins after `bin` (the k_key32 map inverted, with
// a relative safety margin; smaller is always safe), as float rounded down
__global__ void k_phase_bound(const unsigned long long* __restrict__ kminmax, int bin,
                              float* __restrict__ out, const long long* __restrict__ dbin) {
  nxs_pdl_enter();
  if (dbin) bin = (int)dbin[0];  // (a device-sized phase: its last bin from the selection)
  if (kminmax[0] < kminmax[1]) {
    const double lo = dkey_inv(kminmax[0]), hi = dkey_inv(kminmax[1]);
    const double step = (double)((unsigned long long)(bin + 1) << 20) / (4294967294.0 / (hi - lo));
    const double b = (lo + step) - 1e-6 * (fabs(lo) + fabs(step));
    *out = __double2float_rd(b);
  } else {
    *out = __int_as_float(0xff800000);  // -inf: nothing is final at the phase end
  }
}
void launch_phase_bound(const unsigned long long* kminmax, int bin, float* out, cudaStream_t s,
                        const long long* dbin) {
  nxs_launch(k_phase_bound, 1, 1, 0, s, kminmax, bin, out, dbin);
}
void launch_iota(uint32_t* a, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  nxs_launch(k_iota, (unsigned)((n + 255) / 256), 256, 0, s, a, n);
}
void launch_gather_keys(const uint32_t* idx, const uint32_t* key, int64_t n, uint32_t* out,
                        cudaStream_t s) {
  if (n <= 0) return;
  nxs_launch(k_gather_keys, (unsigned)((n + 255) / 256), 256, 0, s, idx, key, n, out);
}
// chunked lazy phases: z_lo of the Gaussians at ranks [r0, r1)
__global__ void k_zlo_ranks(const float* __restrict__ centers, const float* __restrict__ scales,
                            const float* __restrict__ quats, const float* __restrict__ opacities,
                            const uint32_t* __restrict__ order, int64_t r0, int64_t r1,
                            CamDev cam, double cutoff, double* __restrict__ zlo,
                            const int* __restrict__ nd) {
  nxs_pdl_enter();
  if (nd) r1 = min(r1, r0 + (int64_t)*nd);
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  const int64_t g = order[r];
  zlo[g] = z_lower(centers, scales, quats, opacities, g, cam, cutoff);
}
// device-sized chunked phase 0: its chunk-aligned rank count (whole chunks of
// the selected n Gaussians, or all P) and a copy of that many ranks
__global__ void k_chunk_count(const int* __restrict__ n_sel, int64_t P, int chunk,
                              int* __restrict__ out) {
  const int64_t n = *n_sel;
  *out = (int)(n >= P ? P : (n / chunk) * (int64_t)chunk);
}
__global__ void k_copy_u32(const uint32_t* __restrict__ src, int64_t n,
                           const int* __restrict__ nd, uint32_t* __restrict__ dst) {
  nxs_pdl_enter();
  if (nd) n = min(n, (int64_t)*nd);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
void launch_chunk_count(const int* n_sel, int64_t P, int chunk, int* out, cudaStream_t s) {
  nxs_launch(k_chunk_count, 1, 1, 0, s, n_sel, P, chunk, out);
}
void launch_copy_u32(const uint32_t* src, int64_t n, const int* nd, uint32_t* dst,
                     cudaStream_t s) {
  if (n <= 0) return;
  nxs_launch(k_copy_u32, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s, src,
             n, nd, dst);
}
void launch_zlo_ranks(const float* centers, const float* scales, const float* quats,
                      const float* opacities, const uint32_t* order, int64_t r0, int64_t r1,
                      const CamDev& cam, double cutoff, double* zlo, cudaStream_t s,
                      const int* nd) {
  if (r1 <= r0) return;
  nxs_launch(k_zlo_ranks, (unsigned)((r1 - r0 + 255) / 256), 256, 0, s, centers, scales, quats,
                                                                opacities, order, r0, r1, cam,
                                                                cutoff, zlo, nd);
}
void launch_project_ranks_z(const float* centers, const float* scales, const float* quats,
                            const float* opacities, const float* sh, int C, int64_t r0,
                            int64_t r1, const uint32_t* order, const CamDev& cam, double cutoff,
                            double near_plane, const double* zlo, float* zlo_rank, int4* rects,
                            float4* records, float4* bframe, unsigned long long* straddle,
                            double* tq, cudaStream_t s, const int* nd) {
  if (r1 <= r0) return;
  ProjOut o{zlo, zlo_rank, rects, records, bframe, straddle, tq};
  nxs_launch(k_project_ranks, (unsigned)((r1 - r0 + PROJ_CHUNK - 1) / PROJ_CHUNK), PROJ_CHUNK, 0, s, 
      centers, scales, quats, opacities, sh, C, r0, r1, order, cam, cutoff, near_plane, o, nd);
}
void launch_clear_rects(const uint32_t* order, int64_t r0, int64_t r1, int4* rects,
                        cudaStream_t s) {
  if (r1 <= r0) return;
  nxs_launch(k_clear_rects, (unsigned)((r1 - r0 + 255) / 256), 256, 0, s, order, r0, r1, rects);
}
void launch_key32_hist_select(const double* depth, int64_t P, const unsigned long long* kminmax,
                              uint32_t* key, unsigned int* hist, const int64_t* targets,
                              int n_targets, long long* out, int max_bin0,
                              unsigned long long* overflow, unsigned int* bin_pos, int* n_sel,
                              cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifndef NXS_HIST_GRID_DIV
#define NXS_HIST_GRID_DIV 2
#endif
  // (each block flushes its whole shared histogram with global atomics:
  // fewer, longer blocks trade key-pass parallelism for fewer flushes)
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((P + 4095) / 4096, (int64_t)sms * 2 / NXS_HIST_GRID_DIV));
  nxs_launch(k_key32_hist_select, grid, 1024, 0, s, depth, P, kminmax, key, hist, targets,
             n_targets, out, max_bin0, overflow, bin_pos, n_sel);
}
void launch_bin_scatter(const uint32_t* key, int64_t P, int lo, int hi, const long long* hi_dev,
                        unsigned int* bin_pos, uint32_t* order, cudaStream_t s) {
  if (P <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>((P + 1023) / 1024, (int64_t)sms * 8);
  nxs_launch(k_bin_scatter, grid, 256, 0, s, key, P, lo, hi, hi_dev, bin_pos, order);
}
void launch_bin_sort(uint32_t* order, const double* depth, const unsigned int* hist,
                     const unsigned int* bin_end, int lo, int hi, const long long* hi_dev,
                     uint32_t* rank_out, unsigned long long* overflow, cudaStream_t s) {
  if (hi < lo) return;
  nxs_launch(k_bin_sort, hi - lo + 1, BIN_THREADS, 0, s, order, depth, hist, bin_end, lo, hi, hi_dev,
                                                 rank_out, overflow);
}
void launch_project_ranks(const float* centers, const float* scales, const float* quats,
                          const float* opacities, const float* sh, int C, int64_t r0, int64_t r1,
                          const uint32_t* order, const CamDev& cam, double cutoff,
                          double near_plane, int4* rects, float4* records, float4* bframe,
                          unsigned long long* straddle, double* tq, cudaStream_t s,
                          const int* nd, uint32_t* live, unsigned long long* n_live) {
  if (r1 <= r0) return;
  ProjOut o{nullptr, nullptr, rects, records, bframe, straddle, tq, live, n_live};
  nxs_launch(k_project_ranks, (unsigned)((r1 - r0 + PROJ_CHUNK - 1) / PROJ_CHUNK), PROJ_CHUNK, 0, s, 
      centers, scales, quats, opacities, sh, C, r0, r1, order, cam, cutoff, near_plane, o, nd);
}

void launch_project(const float* centers, const float* scales, const float* quats,
                    const float* opacities, const float* sh, int C, int64_t P,
                    const uint32_t* rank_of, const CamDev& cam, double cutoff, double near_plane,
                    const double* zlo, float* zlo_rank, int4* rects, float4* records,
                    float4* bframe, unsigned long long* straddle, double* tq, cudaStream_t s) {
  if (P == 0) return;
  ProjOut o{zlo, zlo_rank, rects, records, bframe, straddle, tq};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_chunks = (P + PROJ_CHUNK - 1) / PROJ_CHUNK;
  const unsigned grid = (unsigned)std::min<int64_t>(n_chunks, (int64_t)sms * 8);
  nxs_launch(k_project, grid, PROJ_CHUNK, 0, s, centers, scales, quats, opacities, sh, C, P, rank_of, cam,
                                         cutoff, near_plane, o);
}

void launch_count_active(const int4* rects, const uint32_t* order, int64_t r0, int64_t r1,
                         int tiles_x, const uint8_t* active, const unsigned int* gate,
                         unsigned long long* counts, const double* tq, const CamDev& cam,
                         cudaStream_t s, const int* nd) {
  if (r1 <= r0) return;
  if (r1 - r0 <= 262144)
    nxs_launch(k_count_active<32>, (unsigned)((r1 - r0 + 7) / 8), 256, 0, s, 
        rects, order, r0, r1, tiles_x, active, gate, counts, nd, tq, cam);
  else
    nxs_launch(k_count_active<8>, (unsigned)((r1 - r0 + 31) / 32), 256, 0, s, 
        rects, order, r0, r1, tiles_x, active, gate, counts, nd, tq, cam);
}

void launch_emit_pairs(const int4* rects, const uint32_t* order, const unsigned long long* offsets,
                       int64_t r0, int64_t r1, int tiles_x, const uint8_t* active, uint32_t* keys,
                       uint32_t* vals, const double* tq, const CamDev& cam, cudaStream_t s,
                       const int* nd, unsigned long long cap) {
  if (r1 <= r0) return;
  if (r1 - r0 <= 262144)
    nxs_launch(k_emit_pairs<32>, (unsigned)((r1 - r0 + 7) / 8), 256, 0, s, 
        rects, order, offsets, r0, r1, tiles_x, active, keys, vals, nd, cap, tq, cam);
  else
    nxs_launch(k_emit_pairs<8>, (unsigned)((r1 - r0 + 31) / 32), 256, 0, s, 
        rects, order, offsets, r0, r1, tiles_x, active, keys, vals, nd, cap, tq, cam);
}

void launch_tile_ranges(const uint32_t* keys, int64_t n, int2* ranges, cudaStream_t s) {
  if (n == 0) return;
  nxs_launch(k_tile_ranges, (unsigned)((n + 255) / 256), 256, 0, s, keys, n, ranges);
}

}  // namespace nxs
