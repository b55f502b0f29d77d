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

namespace nxs {
int set_last_error(int code, const char* msg);  // api.cu
}

namespace nxs_train {

constexpr int LT = 32;            // output tile
constexpr int HALO = 5;           // SSIM_WINDOW // 2
constexpr int LS = LT + 2 * HALO; // staged tile side (42)
constexpr int LTHREADS = 256;
constexpr double SRGB_T = 0.0031308;
constexpr double SRGB_SLOPE1 = 1.055 / 2.4;
constexpr double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;

// 11-tap Gaussian window, sigma 1.5, normalised (optimizer.py:56-60)
__constant__ double c_win[11];

__device__ __forceinline__ double to_srgb(double x) {  // images.py:31-36
  if (x <= SRGB_T) return 12.92 * x;
  if (x <= 1.0) return 1.055 * pow(fmax(x, SRGB_T), 1.0 / 2.4) - 0.055;
  return 1.0 + SRGB_SLOPE1 * (x - 1.0);
}
__device__ __forceinline__ double dsrgb(double x) {  // images.py:47-50
  if (x <= SRGB_T) return 12.92;
  if (x <= 1.0) return SRGB_SLOPE1 * pow(fmin(fmax(x, SRGB_T), 1.0), 1.0 / 2.4 - 1.0);
  return SRGB_SLOPE1;
}

struct LossArgs {
  const float* rendered;
  const float* target;
  int H, W;
  double lam;
  bool srgb_in;   // inputs already sRGB (ssim() semantics)
  bool with_ssim; // lam > 0
  double* maps;   // 3 x (H*W*3) gradient maps
  double* part;   // per block: ssim, l1, mse
};

__device__ __forceinline__ double xval(const LossArgs& a, const float* img, int gy, int gx, int c) {
  if (gy < 0 || gy >= a.H || gx < 0 || gx >= a.W) return 0.0;  // constant-0 padding
  const double v = (double)img[((size_t)gy * a.W + gx) * 3 + c];
  return a.srgb_in ? v : to_srgb(v);
}

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

__global__ void __launch_bounds__(LTHREADS) k_loss_stats(LossArgs a) {
  extern __shared__ double sm[];
  double* xs = sm;                  // [LS][LS]
  double* ys = xs + LS * LS;        // [LS][LS]
  double* hs = ys + LS * LS;        // [5][LS][LT] horizontal window sums
  __shared__ double scratch[LTHREADS / 32];
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const int tid = threadIdx.x;
  const size_t plane = (size_t)a.H * a.W * 3;
  double s_ssim = 0.0, s_l1 = 0.0, s_mse = 0.0;

  // L1 and clipped-sRGB MSE over this tile's own pixels
  for (int k = tid; k < LT * LT * 3; k += LTHREADS) {
    const int c = k % 3, q = (k / 3) % LT, r = k / (3 * LT);
    const int gy = y0 + r, gx = x0 + q;
    if (gy >= a.H || gx >= a.W) continue;
    const size_t i = ((size_t)gy * a.W + gx) * 3 + c;
    const double xr = a.rendered[i], yr = a.target[i];
    const double xsv = a.srgb_in ? xr : to_srgb(xr), ysv = a.srgb_in ? yr : to_srgb(yr);
    s_l1 += fabs(xsv - ysv);
    // optimizer.py:114-118: clip(linear_to_srgb(clip(a, 0)), 0, 1)
    const double xa = fmin(fmax(to_srgb(fmax(xr, 0.0)), 0.0), 1.0);
    const double xb = fmin(fmax(to_srgb(fmax(yr, 0.0)), 0.0), 1.0);
    s_mse += (xa - xb) * (xa - xb);
  }

  if (a.with_ssim) {
    const int nvy = a.H - 2 * HALO, nvx = a.W - 2 * HALO;
    const double m = 1.0 / ((double)nvy * nvx * 3.0);
    for (int c = 0; c < 3; ++c) {
      __syncthreads();
      for (int k = tid; k < LS * LS; k += LTHREADS) {
        const int r = k / LS, q = k % LS;
        xs[k] = xval(a, a.rendered, y0 - HALO + r, x0 - HALO + q, c);
        ys[k] = xval(a, a.target, y0 - HALO + r, x0 - HALO + q, c);
      }
      __syncthreads();
      for (int k = tid; k < LS * LT; k += LTHREADS) {
        const int r = k / LT, q = k % LT;
        double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
        for (int t = 0; t < 11; ++t) {
          const double w = c_win[t], xv = xs[r * LS + q + t], yv = ys[r * LS + q + t];
          sx += w * xv;
          sy += w * yv;
          sxx += w * (xv * xv);
          syy += w * (yv * yv);
          sxy += w * (xv * yv);
        }
        hs[0 * LS * LT + k] = sx;
        hs[1 * LS * LT + k] = sy;
        hs[2 * LS * LT + k] = sxx;
        hs[3 * LS * LT + k] = syy;
        hs[4 * LS * LT + k] = sxy;
      }
      __syncthreads();
      for (int k = tid; k < LT * LT; k += LTHREADS) {
        const int r = k / LT, q = k % LT;
        const int gy = y0 + r, gx = x0 + q;
        if (gy >= a.H || gx >= a.W) continue;
        double f[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < 11; ++t) {
          const double w = c_win[t];
#pragma unroll
          for (int j = 0; j < 5; ++j) f[j] += w * hs[j * LS * LT + (r + t) * LT + q];
        }
        const double mux = f[0], muy = f[1];
        const double vxx = f[2] - mux * mux, vyy = f[3] - muy * muy, vxy = f[4] - mux * muy;
        const double a1 = 2 * mux * muy + C1, a2 = 2 * vxy + C2;
        const double b1 = mux * mux + muy * muy + C1, b2 = vxx + vyy + C2;
        const double smap = (a1 * a2) / (b1 * b2);
        const bool in = gy >= HALO && gy < a.H - HALO && gx >= HALO && gx < a.W - HALO;
        const size_t i = ((size_t)gy * a.W + gx) * 3 + c;
        if (in) {
          s_ssim += smap;
          // optimizer.py:103-106
          const double ds_dmu = 2 * (muy * a2 * b1 - mux * a1 * a2) / (b1 * b1 * b2);
          const double ds_dsxx = -smap / b2;
          const double ds_dsxy = 2 * a1 / (b1 * b2);
          a.maps[i] = m * (ds_dmu - 2 * mux * ds_dsxx - muy * ds_dsxy);
          a.maps[plane + i] = m * ds_dsxx;
          a.maps[2 * plane + i] = m * ds_dsxy;
        } else {
          a.maps[i] = 0.0;
          a.maps[plane + i] = 0.0;
          a.maps[2 * plane + i] = 0.0;
        }
      }
    }
  }
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  const double t0 = block_sum(s_ssim, scratch);
  const double t1 = block_sum(s_l1, scratch);
  const double t2 = block_sum(s_mse, scratch);
  if (tid == 0) {
    a.part[3 * blk + 0] = t0;
    a.part[3 * blk + 1] = t1;
    a.part[3 * blk + 2] = t2;
  }
}

__global__ void __launch_bounds__(LTHREADS) k_loss_seed(LossArgs a, float* __restrict__ seed) {
  extern __shared__ double sm[];
  double* ms = sm;                 // [3][LS][LS]
  double* hs = ms + 3 * LS * LS;   // [3][LS][LT]
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const int tid = threadIdx.x;
  const size_t plane = (size_t)a.H * a.W * 3;
  const double inv_size = 1.0 / (double)plane;
  for (int c = 0; c < 3; ++c) {
    if (a.with_ssim) {
      __syncthreads();
      for (int k = tid; k < LS * LS; k += LTHREADS) {
        const int gy = y0 - HALO + k / LS, gx = x0 - HALO + k % LS;
        const bool ok = gy >= 0 && gy < a.H && gx >= 0 && gx < a.W;
        const size_t i = ((size_t)gy * a.W + gx) * 3 + c;
#pragma unroll
        for (int j = 0; j < 3; ++j) ms[j * LS * LS + k] = ok ? a.maps[j * plane + i] : 0.0;
      }
      __syncthreads();
      for (int k = tid; k < LS * LT; k += LTHREADS) {
        const int r = k / LT, q = k % LT;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
#pragma unroll
          for (int t = 0; t < 11; ++t) s += c_win[t] * ms[j * LS * LS + r * LS + q + t];
          hs[j * LS * LT + k] = s;
        }
      }
      __syncthreads();
    }
    for (int k = tid; k < LT * LT; k += LTHREADS) {
      const int r = k / LT, q = k % LT;
      const int gy = y0 + r, gx = x0 + q;
      if (gy >= a.H || gx >= a.W) continue;
      const size_t i = ((size_t)gy * a.W + gx) * 3 + c;
      const double xr = a.rendered[i], yr = a.target[i];
      const double xv = a.srgb_in ? xr : to_srgb(xr), yv = a.srgb_in ? yr : to_srgb(yr);
      const double diff = xv - yv;
      const double sgn = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
      double d = (a.with_ssim ? (1.0 - a.lam) : 1.0) * sgn * inv_size;
      if (a.with_ssim) {
        double f[3] = {0, 0, 0};
#pragma unroll
        for (int t = 0; t < 11; ++t)
#pragma unroll
          for (int j = 0; j < 3; ++j) f[j] += c_win[t] * hs[j * LS * LT + (r + t) * LT + q];
        const double ds = f[0] + 2 * xv * f[1] + yv * f[2];  // optimizer.py:107-109
        d -= a.lam * ds;
      }
      seed[i] = (float)(a.srgb_in ? d : d * dsrgb(xr));
    }
  }
}

__global__ void k_loss_final(const double* __restrict__ part, int nblk, int H, int W, double lam,
                             bool with_ssim, double* __restrict__ out) {
  __shared__ double scratch[32];
  double v[3] = {0, 0, 0};
  for (int b = threadIdx.x; b < nblk; b += blockDim.x)
    for (int j = 0; j < 3; ++j) v[j] += part[3 * b + j];
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
struct AdamArgs {
  nxs_adam_group g[5];
  float b1, b2, omb1, omb2, inv_bc1, inv_bc2, eps, lr_mult;
  unsigned long long* nan_skips;
};

__device__ __forceinline__ void adam_elem(const AdamArgs& a, const nxs_adam_group& g, int64_t i,
                                          float lr, unsigned& bad) {
  float gr = g.grad[i];
  if (!isfinite(gr)) {
    ++bad;
    gr = 0.f;
  }
  const float m = a.b1 * g.m[i] + a.omb1 * gr;
  const float v = a.b2 * g.v[i] + a.omb2 * gr * gr;
  g.m[i] = m;
  g.v[i] = v;
  const float mh = m * a.inv_bc1, vh = v * a.inv_bc2;
  g.param[i] -= lr * mh / (sqrtf(vh) + a.eps);
}

__global__ void k_adam(AdamArgs a) {
  const int gi = blockIdx.y;
  const nxs_adam_group& g = a.g[gi];
  if (!g.param || g.count <= 0) return;
  const float lr = (float)g.lr * a.lr_mult;
  unsigned bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi == 2) {  // quaternions: update a row, then renormalise it
    for (int64_t r = t0; r < g.count / 4; r += stride) {
      for (int k = 0; k < 4; ++k) adam_elem(a, g, 4 * r + k, lr, bad);
      const float q0 = g.param[4 * r], q1 = g.param[4 * r + 1], q2 = g.param[4 * r + 2],
                  q3 = g.param[4 * r + 3];
      const float n = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
      g.param[4 * r] = q0 / n;
      g.param[4 * r + 1] = q1 / n;
      g.param[4 * r + 2] = q2 / n;
      g.param[4 * r + 3] = q3 / n;
    }
  } else {
    for (int64_t i = t0; i < g.count; i += stride) {
      adam_elem(a, g, i, lr, bad);
      if (gi == 1) g.param[i] = fmaxf(g.param[i], 1e-6f);  // SCALE_MIN
      if (gi == 3)                                         // [OPACITY_MIN, ALPHA_MAX]
        g.param[i] = fminf(fmaxf(g.param[i], 1e-4f), (float)(1.0 - 1e-6));
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(a.nan_skips, (unsigned long long)bad);
}

bool g_win_ready = false;

}  // namespace nxs_train

using namespace nxs_train;

extern "C" {

int64_t nxs_loss_workspace_bytes(int32_t height, int32_t width) {
  if (height <= 0 || width <= 0) return 0;
  const int64_t nblk = (int64_t)((width + LT - 1) / LT) * ((height + LT - 1) / LT);
  return (int64_t)3 * height * width * 3 * 8 + nblk * 3 * 8 + 256;
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
  if (!g_win_ready) {
    double w[11], sum = 0.0;
    for (int i = 0; i < 11; ++i) {
      const double r = (i - 5) / 1.5;
      w[i] = std::exp(-0.5 * r * r);
      sum += w[i];
    }
    for (double& x : w) x /= sum;
    if (cudaMemcpyToSymbol(c_win, w, sizeof(w)) != cudaSuccess)
      return nxs::set_last_error(NXS_ERR_CUDA, "window upload failed");
    static const size_t sm1 = sizeof(double) * (2 * LS * LS + 5 * LS * LT);
    static const size_t sm2 = sizeof(double) * (3 * LS * LS + 3 * LS * LT);
    cudaFuncSetAttribute(k_loss_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    cudaFuncSetAttribute(k_loss_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    g_win_ready = true;
  }
  const dim3 grid((width + LT - 1) / LT, (height + LT - 1) / LT);
  const int nblk = (int)(grid.x * grid.y);
  LossArgs a{rendered, target, height, width, lam, (flags & NXS_LOSS_SRGB_INPUT) != 0,
             with_ssim, static_cast<double*>(workspace),
             static_cast<double*>(workspace) + (size_t)3 * height * width * 3};
  const size_t sm1 = sizeof(double) * (2 * LS * LS + 5 * LS * LT);
  const size_t sm2 = sizeof(double) * (3 * LS * LS + 3 * LS * LT);
  k_loss_stats<<<grid, LTHREADS, sm1, s>>>(a);
  if (seed) k_loss_seed<<<grid, LTHREADS, sm2, s>>>(a, seed);
  k_loss_final<<<1, 256, 0, s>>>(a.part, nblk, height, width, lam, with_ssim, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

int nxs_adam_step(const nxs_adam_group* groups, int64_t step, double lr_mult,
                  unsigned long long* nan_skips, void* stream) {
  if (!groups || !nan_skips || step < 1)
    return nxs::set_last_error(NXS_ERR_INVALID, "null argument or step < 1");
  AdamArgs a;
  int64_t most = 0;
  for (int k = 0; k < 5; ++k) {
    a.g[k] = groups[k];
    if (a.g[k].param && (!a.g[k].grad || !a.g[k].m || !a.g[k].v))
      return nxs::set_last_error(NXS_ERR_INVALID, "adam group without grad/m/v");
    if (k == 2 && a.g[k].count % 4 != 0)
      return nxs::set_last_error(NXS_ERR_INVALID, "quaternion count not a multiple of 4");
    most = std::max<int64_t>(most, a.g[k].param ? a.g[k].count : 0);
  }
  const double b1 = 0.9, b2 = 0.999;  // ADAM_BETA1/2, optimizer.py:42-44
  a.b1 = (float)b1;
  a.b2 = (float)b2;
  a.omb1 = (float)(1.0 - b1);
  a.omb2 = (float)(1.0 - b2);
  a.inv_bc1 = (float)(1.0 / (1.0 - std::pow(b1, (double)step)));
  a.inv_bc2 = (float)(1.0 / (1.0 - std::pow(b2, (double)step)));
  a.eps = 1e-8f;
  a.lr_mult = (float)lr_mult;
  a.nan_skips = nan_skips;
  if (most == 0) return NXS_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (most + 255) / 256;
  const dim3 grid((unsigned)std::min<int64_t>(want, (int64_t)sms * 8), 5);
  k_adam<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : nxs::set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
