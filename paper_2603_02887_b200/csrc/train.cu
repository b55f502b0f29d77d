// Train-step neighbours of the render path on the device:
// the image loss with its adjoint seed, and the bounded Adam step.
//
//   nxs_image_loss   reference pkg/src/nexsplat/optimizer.py:128-152 loss(),
//                    :68-111 ssim(), :114-125 mse(); images.py:31-50 sRGB
//   nxs_adam_step    reference optimizer.py:173-204 bounded_adam_step()
//
// Loss: everything after the fp32 inputs is fp64 (the reference computes in
// float64; SSIM's E[x²] − μ² cancels).  Two tiled passes over 32×32 output
// tiles with a 5-pixel halo, per channel:
//   L1  sRGB conversion, the five separable 11-tap window sums (μx, μy,
//       E[x²], E[y²], E[xy]; zero padding = scipy correlate1d mode
//       "constant"), the SSIM map and the three gradient maps
//       m·(∂s/∂μ − 2μx ∂s/∂σxx − μy ∂s/∂σxy), m·∂s/∂σxx, m·∂s/∂σxy
//       (m = interior mask / (n_valid·3)), plus per-block sums of the SSIM
//       map, |x − y| and the clipped-sRGB squared error;
//   L2  the window filter of the three maps, the SSIM gradient
//       F(a) + 2x·F(b) + y·F(c), and the seed
//       ((1−λ)·sign(x−y)/size − λ·∂S/∂x)·dsRGB/dlinear.
// A one-block pass reduces the block sums in a fixed order (deterministic).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nxs.h"
#include "nxs_internal.cuh"

namespace nxs {
int set_last_error(int code, const char* msg);  // api.cu
}

namespace nxs_train {

constexpr int LT = 32;            // output tile
constexpr int HALO = 5;           // SSIM_WINDOW // 2
constexpr int LS = LT + 2 * HALO; // staged tile side (42)
constexpr int LTHREADS = 256;
constexpr int PREP_BLOCKS = 148 * 4;
constexpr double SRGB_T = 0.0031308;
constexpr double SRGB_SLOPE1 = 1.055 / 2.4;
constexpr double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;

// 11-tap Gaussian window, sigma 1.5, normalised (optimizer.py:56-60)
__constant__ double c_win[11];

// x^(1/2.4) as exp2(log2(x)/2.4) (fp64, a few ulp; x in (T, 1])
__device__ __forceinline__ double root24(double x) { return exp2(log2(x) * (1.0 / 2.4)); }
__device__ __forceinline__ double to_srgb(double x) {  // images.py:31-36
  if (x <= SRGB_T) return 12.92 * x;
  if (x <= 1.0) return 1.055 * root24(x) - 0.055;
  return 1.0 + SRGB_SLOPE1 * (x - 1.0);
}
// images.py:47-50 from the value s = to_srgb(x): on (T, 1]
// (1.055/2.4)·x^(1/2.4 - 1) = (s + 0.055) / (2.4·x)
__device__ __forceinline__ double dsrgb_of(double x, double s) {
  if (x <= SRGB_T) return 12.92;
  if (x <= 1.0) return (s + 0.055) / (2.4 * x);
  return SRGB_SLOPE1;
}

struct LossArgs {
  const float* rendered;
  const float* target;
  int H, W;
  double lam;
  bool srgb_in;   // inputs already sRGB (ssim() semantics)
  bool with_ssim; // lam > 0
  // internal planes are channel-planar [c][H][W]
  double* maps;   // 3 gradient maps x 3 channels
  double* xs;     // sRGB render
  double* ys;     // sRGB target
  double* ds;     // dsRGB/dlinear of the render
  double* part;   // per block: ssim, l1, mse
};

// block-wide fp64 sum in a fixed order (thread 0 returns the total)
__device__ double block_sum(double v, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += scratch[k];
  return t;
}

// pass 0: sRGB planes (one transfer evaluation per element), per-block L1
// and clipped-sRGB squared-error sums
__global__ void __launch_bounds__(LTHREADS) k_loss_prep(LossArgs a) {
  __shared__ double scratch[LTHREADS / 32];
  const int64_t n = (int64_t)a.H * a.W * 3;
  double s_l1 = 0.0, s_mse = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * LTHREADS + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * LTHREADS) {
    const double xr = a.rendered[i], yr = a.target[i];
    const double xv = a.srgb_in ? xr : to_srgb(xr), yv = a.srgb_in ? yr : to_srgb(yr);
    const int64_t pix = i / 3, c = i - 3 * pix;
    const int64_t j = c * (n / 3) + pix;  // channel-planar
    a.xs[j] = xv;
    a.ys[j] = yv;
    a.ds[j] = a.srgb_in ? 1.0 : dsrgb_of(xr, xv);
    s_l1 += fabs(xv - yv);
    // optimizer.py:114-118: clip(linear_to_srgb(clip(a, 0)), 0, 1); equal to
    // the clipped plane value when the inputs are linear
    const double xa = a.srgb_in ? to_srgb(fmax(xr, 0.0)) : (xr < 0.0 ? 0.0 : xv);
    const double xb = a.srgb_in ? to_srgb(fmax(yr, 0.0)) : (yr < 0.0 ? 0.0 : yv);
    const double ca = fmin(fmax(xa, 0.0), 1.0), cb = fmin(fmax(xb, 0.0), 1.0);
    s_mse += (ca - cb) * (ca - cb);
  }
  const double t1 = block_sum(s_l1, scratch);
  const double t2 = block_sum(s_mse, scratch);
  if (threadIdx.x == 0) {
    a.part[3 * blockIdx.x + 1] = t1;
    a.part[3 * blockIdx.x + 2] = t2;
  }
}

// planar tile staging: [LS][LS] window of channel plane p (zero outside),
// asynchronous 8-byte copies (zero-filled out of the image) so every
// thread's loads are in flight together; the caller commits and waits
__device__ __forceinline__ void stage_tile(const LossArgs& a, const double* __restrict__ p,
                                           int x0, int y0, double* dst) {
  for (int k = threadIdx.x; k < LS * LS; k += LTHREADS) {
    const int gy = y0 - HALO + k / LS, gx = x0 - HALO + k % LS;
    const bool in = gy >= 0 && gy < a.H && gx >= 0 && gx < a.W;
    const double* src = in ? p + (size_t)gy * a.W + gx : p;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + k);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src),
                 "r"(in ? 8 : 0));
  }
}
__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
}

// horizontal 11-tap pass, register-blocked: each work item filters 4
// consecutive columns of one row for NQ products of the staged planes
template <int NQ, class Prod>
__device__ __forceinline__ void hpass(const double* const* src, double* hs, Prod prod) {
  for (int item = threadIdx.x; item < LS * (LT / 4); item += LTHREADS) {
    const int r = item / (LT / 4), q0 = (item % (LT / 4)) * 4;
    double acc[4][NQ];
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
      for (int j = 0; j < NQ; ++j) acc[o][j] = 0.0;
#pragma unroll
    for (int t = 0; t < 14; ++t) {
      double v[NQ];
      prod(src, r * LS + q0 + t, v);
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int tap = t - o;
        if (tap >= 0 && tap < 11)
#pragma unroll
          for (int j = 0; j < NQ; ++j) acc[o][j] = fma(c_win[tap], v[j], acc[o][j]);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
      for (int j = 0; j < NQ; ++j) hs[(j * LS + r) * LT + q0 + o] = acc[o][j];
  }
}

// vertical 11-tap pass: thread (column q, rows 4rb..4rb+3) of the tile
template <int NQ>
__device__ __forceinline__ void vpass(const double* hs, double (&f)[4][NQ]) {
  const int q = threadIdx.x % LT, rb = threadIdx.x / LT;
#pragma unroll
  for (int o = 0; o < 4; ++o)
#pragma unroll
    for (int j = 0; j < NQ; ++j) f[o][j] = 0.0;
#pragma unroll
  for (int t = 0; t < 14; ++t) {
    double v[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) v[j] = hs[(j * LS + 4 * rb + t) * LT + q];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int tap = t - o;
      if (tap >= 0 && tap < 11)
#pragma unroll
        for (int j = 0; j < NQ; ++j) f[o][j] = fma(c_win[tap], v[j], f[o][j]);
    }
  }
}

struct ProdStats {  // x, y, x², y², xy
  __device__ void operator()(const double* const* src, int k, double* v) const {
    const double x = src[0][k], y = src[1][k];
    v[0] = x;
    v[1] = y;
    v[2] = x * x;
    v[3] = y * y;
    v[4] = x * y;
  }
};
struct ProdMaps {  // the three gradient maps
  __device__ void operator()(const double* const* src, int k, double* v) const {
    v[0] = src[0][k];
    v[1] = src[1][k];
    v[2] = src[2][k];
  }
};

static_assert(LTHREADS == LT * LT / 4, "vertical pass: 4 output rows per thread");

// pass 1: SSIM window statistics, the SSIM map sum and the gradient maps
__global__ void __launch_bounds__(LTHREADS) k_loss_stats(LossArgs a, double* __restrict__ psum) {
  extern __shared__ double sm[];
  double* xs = sm;                  // [LS][LS]
  double* ys = xs + LS * LS;        // [LS][LS]
  double* hs = ys + LS * LS;        // [5][LS][LT] horizontal window sums
  __shared__ double scratch[LTHREADS / 32];
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const size_t hw = (size_t)a.H * a.W;
  const double m = 1.0 / ((double)(a.H - 2 * HALO) * (a.W - 2 * HALO) * 3.0);
  const int q = threadIdx.x % LT, rb = threadIdx.x / LT;
  double s_ssim = 0.0;
  for (int c = 0; c < 3; ++c) {
    __syncthreads();
    stage_tile(a, a.xs + c * hw, x0, y0, xs);
    stage_tile(a, a.ys + c * hw, x0, y0, ys);
    stage_wait();
    const double* src[2] = {xs, ys};
    hpass<5>(src, hs, ProdStats{});
    __syncthreads();
    double f[4][5];
    vpass<5>(hs, f);
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int gy = y0 + 4 * rb + o, gx = x0 + q;
      if (gy >= a.H || gx >= a.W) continue;
      const double mux = f[o][0], muy = f[o][1];
      const double vxx = f[o][2] - mux * mux, vyy = f[o][3] - muy * muy;
      const double vxy = f[o][4] - mux * muy;
      const double a1 = 2 * mux * muy + C1, a2 = 2 * vxy + C2;
      const double b1 = mux * mux + muy * muy + C1, b2 = vxx + vyy + C2;
      const double smap = (a1 * a2) / (b1 * b2);
      const bool in = gy >= HALO && gy < a.H - HALO && gx >= HALO && gx < a.W - HALO;
      const size_t i = c * hw + (size_t)gy * a.W + gx;
      double g0 = 0.0, g1 = 0.0, g2 = 0.0;
      if (in) {
        s_ssim += smap;
        // optimizer.py:103-106
        const double ds_dmu = 2 * (muy * a2 * b1 - mux * a1 * a2) / (b1 * b1 * b2);
        const double ds_dsxx = -smap / b2;
        const double ds_dsxy = 2 * a1 / (b1 * b2);
        g0 = m * (ds_dmu - 2 * mux * ds_dsxx - muy * ds_dsxy);
        g1 = m * ds_dsxx;
        g2 = m * ds_dsxy;
      }
      a.maps[i] = g0;
      a.maps[3 * hw + i] = g1;
      a.maps[6 * hw + i] = g2;
    }
  }
  const double t0 = block_sum(s_ssim, scratch);
  if (threadIdx.x == 0) psum[blockIdx.y * gridDim.x + blockIdx.x] = t0;
}

// pass 2: window filter of the gradient maps and the seed
__global__ void __launch_bounds__(LTHREADS) k_loss_seed(LossArgs a, float* __restrict__ seed) {
  extern __shared__ double sm[];
  double* ms = sm;                 // [3][LS][LS]
  double* hs = ms + 3 * LS * LS;   // [3][LS][LT]
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const size_t hw = (size_t)a.H * a.W;
  const double inv_size = 1.0 / (double)(3 * hw);
  const int q = threadIdx.x % LT, rb = threadIdx.x / LT;
  for (int c = 0; c < 3; ++c) {
    double f[4][3];
    if (a.with_ssim) {
      __syncthreads();
      for (int j = 0; j < 3; ++j) stage_tile(a, a.maps + (3 * j + c) * hw, x0, y0, ms + j * LS * LS);
      stage_wait();
      const double* src[3] = {ms, ms + LS * LS, ms + 2 * LS * LS};
      hpass<3>(src, hs, ProdMaps{});
      __syncthreads();
      vpass<3>(hs, f);
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int gy = y0 + 4 * rb + o, gx = x0 + q;
      if (gy >= a.H || gx >= a.W) continue;
      const size_t pi = (size_t)gy * a.W + gx, i = c * hw + pi;
      const double xv = a.xs[i], yv = a.ys[i];
      const double diff = xv - yv;
      const double sgn = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
      double d = (a.with_ssim ? (1.0 - a.lam) : 1.0) * sgn * inv_size;
      if (a.with_ssim) d -= a.lam * (f[o][0] + 2 * xv * f[o][1] + yv * f[o][2]);  // :107-109
      seed[3 * pi + c] = (float)(d * a.ds[i]);
    }
  }
}

__global__ void k_loss_final(const double* __restrict__ part, int nprep,
                             const double* __restrict__ psum, int nstat, int H, int W, double lam,
                             bool with_ssim, double* __restrict__ out) {
  __shared__ double scratch[32];
  double v[3] = {0, 0, 0};
  for (int b = threadIdx.x; b < nprep; b += blockDim.x) {
    v[1] += part[3 * b + 1];
    v[2] += part[3 * b + 2];
  }
  if (with_ssim)
    for (int b = threadIdx.x; b < nstat; b += blockDim.x) v[0] += psum[b];
  double t[3];
  for (int j = 0; j < 3; ++j) t[j] = block_sum(v[j], scratch);
  if (threadIdx.x == 0) {
    const double size = (double)H * W * 3;
    const double l1 = t[1] / size;
    const double s = with_ssim ? t[0] / ((double)(H - 2 * HALO) * (W - 2 * HALO) * 3.0) : 0.0;
    out[0] = with_ssim ? (1.0 - lam) * l1 + lam * (1.0 - s) : l1;
    out[1] = l1;
    out[2] = s;
    out[3] = t[2] / size;
  }
}

// ---------------------------------------------------------------------------
// bounded Adam (optimizer.py:173-204): groups centers, scales, quats,
// opacities, sh; non-finite gradients are dropped and counted
// ---------------------------------------------------------------------------
template <class T>
struct AdamGroupT {
  T* param;
  const T* grad;
  T* m;
  T* v;
  int64_t count;
  double lr;
};

template <class T>
struct AdamArgs {
  AdamGroupT<T> g[5];
  T b1, b2, omb1, omb2, inv_bc1, inv_bc2, eps, lr_mult;
  unsigned long long* nan_skips;
};

template <class T>
__device__ __forceinline__ T adam_one(const AdamArgs<T>& a, T p, T gr, T& m, T& v, T lr,
                                      unsigned& bad) {
  if (!isfinite(gr)) {
    ++bad;
    gr = T(0);
  }
  m = a.b1 * m + a.omb1 * gr;
  v = a.b2 * v + a.omb2 * gr * gr;
  return p - lr * (m * a.inv_bc1) / (sqrt(v * a.inv_bc2) + a.eps);
}

template <class T>
__device__ __forceinline__ T clamp_group(int gi, T p) {
  if (gi == 1) return p < T(1e-6) ? T(1e-6) : p;  // SCALE_MIN
  if (gi == 3) {                                   // opacity bounds
    const T hi = (T)(1.0 - 1e-6);
    return p < T(1e-4) ? T(1e-4) : (p > hi ? hi : p);
  }
  return p;
}

// one group per blockIdx.y; fp32: 16-B vectors (a quaternion row is one
// vector, renormalised after its update), scalar tail; fp64 (the numpy
// drop-in's float64 parameters, updated without an fp32 round trip): scalar
template <class T>
__global__ void __launch_bounds__(256) k_adam(AdamArgs<T> a) {
  const int gi = blockIdx.y;
  const AdamGroupT<T>& g = a.g[gi];
  if (!g.param || g.count <= 0) return;
  const T lr = (T)g.lr * a.lr_mult;
  unsigned bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool vec = false;
  int64_t n4 = 0;
  if constexpr (sizeof(T) == 4) {
    vec = ((reinterpret_cast<uintptr_t>(g.param) | reinterpret_cast<uintptr_t>(g.grad) |
            reinterpret_cast<uintptr_t>(g.m) | reinterpret_cast<uintptr_t>(g.v)) & 15) == 0;
    n4 = vec ? g.count / 4 : 0;
    for (int64_t r = t0; r < n4; r += stride) {
      float4 p = reinterpret_cast<const float4*>(g.param)[r];
      const float4 gr = __ldcs(reinterpret_cast<const float4*>(g.grad) + r);
      float4 m = reinterpret_cast<const float4*>(g.m)[r];
      float4 v = reinterpret_cast<const float4*>(g.v)[r];
      p.x = clamp_group<T>(gi, adam_one<T>(a, p.x, gr.x, m.x, v.x, lr, bad));
      p.y = clamp_group<T>(gi, adam_one<T>(a, p.y, gr.y, m.y, v.y, lr, bad));
      p.z = clamp_group<T>(gi, adam_one<T>(a, p.z, gr.z, m.z, v.z, lr, bad));
      p.w = clamp_group<T>(gi, adam_one<T>(a, p.w, gr.w, m.w, v.w, lr, bad));
      if (gi == 2) {  // quaternion row
        const float n = sqrtf(p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w);
        p.x /= n;
        p.y /= n;
        p.z /= n;
        p.w /= n;
      }
      reinterpret_cast<float4*>(g.param)[r] = p;
      reinterpret_cast<float4*>(g.m)[r] = m;
      reinterpret_cast<float4*>(g.v)[r] = v;
    }
  }
  if (gi == 2 && !vec) {  // quaternions row by row
    for (int64_t r = t0; r < g.count / 4; r += stride) {
      T q[4];
      for (int k = 0; k < 4; ++k) {
        const int64_t i = 4 * r + k;
        q[k] = adam_one<T>(a, g.param[i], g.grad[i], g.m[i], g.v[i], lr, bad);
      }
      const T n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      for (int k = 0; k < 4; ++k) g.param[4 * r + k] = q[k] / n;
    }
  } else if (gi != 2) {
    for (int64_t i = 4 * n4 + t0; i < g.count; i += stride)
      g.param[i] = clamp_group<T>(gi, adam_one<T>(a, g.param[i], g.grad[i], g.m[i], g.v[i], lr,
                                                  bad));
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(a.nan_skips, (unsigned long long)bad);
}

template <class T, class G>
int adam_step(const G* groups, int64_t step, double lr_mult, unsigned long long* nan_skips,
              void* stream) {
  if (!groups || !nan_skips || step < 1)
    return nxs::set_last_error(NXS_ERR_INVALID, "null argument or step < 1");
  AdamArgs<T> a;
  int64_t most = 0;
  for (int k = 0; k < 5; ++k) {
    a.g[k] = AdamGroupT<T>{groups[k].param, groups[k].grad, groups[k].m, groups[k].v,
                           groups[k].count, groups[k].lr};
    if (a.g[k].param && (!a.g[k].grad || !a.g[k].m || !a.g[k].v))
      return nxs::set_last_error(NXS_ERR_INVALID, "adam group without grad/m/v");
    if (k == 2 && a.g[k].count % 4 != 0)
      return nxs::set_last_error(NXS_ERR_INVALID, "quaternion count not a multiple of 4");
    most = std::max<int64_t>(most, a.g[k].param ? a.g[k].count : 0);
  }
  const double b1 = 0.9, b2 = 0.999;  // ADAM_BETA1/2, optimizer.py:42-44
  a.b1 = (T)b1;
  a.b2 = (T)b2;
  a.omb1 = (T)(1.0 - b1);
  a.omb2 = (T)(1.0 - b2);
  a.inv_bc1 = (T)(1.0 / (1.0 - std::pow(b1, (double)step)));
  a.inv_bc2 = (T)(1.0 / (1.0 - std::pow(b2, (double)step)));
  a.eps = (T)1e-8;
  a.lr_mult = (T)lr_mult;
  a.nan_skips = nan_skips;
  if (most == 0) return NXS_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (most / 4 + 255) / 256;
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8)), 5);
  k_adam<T><<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : nxs::set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

unsigned long long g_win_dev = 0;  // devices with the window and attributes set

}  // namespace nxs_train

using namespace nxs_train;

extern "C" {

int64_t nxs_loss_workspace_bytes(int32_t height, int32_t width) {
  if (height <= 0 || width <= 0) return 0;
  const int64_t nblk = (int64_t)((width + LT - 1) / LT) * ((height + LT - 1) / LT);
  return (int64_t)6 * height * width * 3 * 8 + (PREP_BLOCKS * 3 + nblk) * 8 + 256;
}

int nxs_image_loss(const float* rendered, const float* target, int32_t height, int32_t width,
                   double lam, int32_t flags, double* out, float* seed, void* workspace,
                   void* stream) {
  using nxs::set_last_error;
  if (!rendered || !target || !out || !workspace)
    return set_last_error(NXS_ERR_INVALID, "null argument");
  if (height <= 0 || width <= 0) return set_last_error(NXS_ERR_INVALID, "empty image");
  if (!(lam >= 0.0 && lam <= 1.0))
    return set_last_error(NXS_ERR_INVALID, "ssim weight must be in [0, 1]");
  const bool with_ssim = lam > 0.0;
  if (with_ssim && (height < 2 * HALO + 1 || width < 2 * HALO + 1))
    return set_last_error(NXS_ERR_INVALID, "images must be at least 11 pixels on each side");
  cudaStream_t s = (cudaStream_t)stream;
  bool win_ok = true;
  nxs::once_per_device(g_win_dev, [&] {
    double w[11], sum = 0.0;
    for (int i = 0; i < 11; ++i) {
      const double r = (i - 5) / 1.5;
      w[i] = std::exp(-0.5 * r * r);
      sum += w[i];
    }
    for (double& x : w) x /= sum;
    win_ok = cudaMemcpyToSymbol(c_win, w, sizeof(w)) == cudaSuccess;
    const size_t sm1 = sizeof(double) * (2 * LS * LS + 5 * LS * LT);
    const size_t sm2 = sizeof(double) * (3 * LS * LS + 3 * LS * LT);
    cudaFuncSetAttribute(k_loss_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    cudaFuncSetAttribute(k_loss_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  });
  if (!win_ok) {
    g_win_dev = 0;
    return nxs::set_last_error(NXS_ERR_CUDA, "window upload failed");
  }
  const dim3 grid((width + LT - 1) / LT, (height + LT - 1) / LT);
  const int nblk = (int)(grid.x * grid.y);
  const size_t plane = (size_t)height * width * 3;
  double* ws = static_cast<double*>(workspace);
  LossArgs a{rendered, target, height, width, lam, (flags & NXS_LOSS_SRGB_INPUT) != 0,
             with_ssim, ws, ws + 3 * plane, ws + 4 * plane, ws + 5 * plane, ws + 6 * plane};
  double* psum = a.part + 3 * PREP_BLOCKS;
  const int nprep = (int)std::min<int64_t>(PREP_BLOCKS, ((int64_t)plane + LTHREADS - 1) / LTHREADS);
  const size_t sm1 = sizeof(double) * (2 * LS * LS + 5 * LS * LT);
  const size_t sm2 = sizeof(double) * (3 * LS * LS + 3 * LS * LT);
  k_loss_prep<<<nprep, LTHREADS, 0, s>>>(a);
  if (with_ssim) k_loss_stats<<<grid, LTHREADS, sm1, s>>>(a, psum);
  if (seed) k_loss_seed<<<grid, LTHREADS, sm2, s>>>(a, seed);
  k_loss_final<<<1, 256, 0, s>>>(a.part, nprep, psum, nblk, height, width, lam, with_ssim, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

int nxs_adam_step(const nxs_adam_group* groups, int64_t step, double lr_mult,
                  unsigned long long* nan_skips, void* stream) {
  return adam_step<float>(groups, step, lr_mult, nan_skips, stream);
}

int nxs_adam_step_f64(const nxs_adam_group_f64* groups, int64_t step, double lr_mult,
                      unsigned long long* nan_skips, void* stream) {
  return adam_step<double>(groups, step, lr_mult, nan_skips, stream);
}

}  // extern "C"
