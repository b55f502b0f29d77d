// Per-ray batched compositing on the device: the
// reference's composite_batch (pkg/src/nexsplat/compositor.py:84-171) — R
// rays of N front-to-back samples — as one fp64 scan per ray.  It backs the
// finite-difference gradient oracle (adjoint.py:195-222), gradcheck and the
// per-ray studies, which perturb thousands of copies of one ray.
//
// One thread per ray walks its N samples once, keeping the running sums the
// reference builds with cumsum / cumprod (same order of fp64 additions and
// products): τ̄ (sum of alphas in front), Π(1-α) in front, and the
// cumulative unclamped weight; the saturating sample gets 1 - cum_before.
// Weights are written as they are produced; the per-ray outputs (radiance,
// residual, k0, overdraw, e_k, θ₀, t_k) at the end.  HBM-bound: 33 B read
// (+1 B valid) and 8 B written per sample.
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nxs.h"

namespace nxs {
int set_last_error(int code, const char* msg);  // api.cu
}

namespace nxs_batch {

struct Model64 {
  int variant;
  double p;      // model parameter
  double K;      // softplus: κ / softplus(κ)
  double ex;     // power law: -(1 + w) / w
};

// discrete_extinction (reference transmittance.py:215-265), fp64
__device__ __forceinline__ double extinction(const Model64& m, double a, double tb, double prod) {
  switch (m.variant) {
    case NXS_MODEL_EXPONENTIAL: return a * prod;
    case NXS_MODEL_LINEAR: return a;
    case NXS_MODEL_QUADRATIC: return a * (1.0 + m.p * tb);
    case NXS_MODEL_BLENDED: return a * (1.0 - m.p * (1.0 - prod));
    case NXS_MODEL_VICINI: {
      const double ex = a * prod;
      return a + m.p * (ex - a);
    }
    case NXS_MODEL_POWER_LAW: {
      if (m.p == -1.0) return a;
      if (fabs(m.p) < 1e-4) return a * exp(-tb);
      const double base = 1.0 + tb * m.p;
      return base > 0.0 ? a * pow(base, m.ex) : 0.0;
    }
    default: {  // softplus: a K expit(κ(1 - τ̄))
      const double x = m.p * (1.0 - tb);
      const double e = exp(-fabs(x));
      const double sig = x >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
      return a * m.K * sig;
    }
  }
}

struct BatchArgs {
  const double* alpha;     // R*N
  const double* emission;  // R*N*3
  const uint8_t* valid;    // R*N or null
  int64_t R, N;
  double bg[3];
  double* weights;         // R*N or null
  double* radiance;        // R*3
  double* residual;        // R or null
  int64_t* k0;             // R or null
  int64_t* overdraw;       // R or null
  double* e_k;             // R*3 or null
  double* theta0;          // R*3 or null
  double* t_k;             // R or null
};

__global__ void __launch_bounds__(128) k_composite_batch(Model64 m, BatchArgs b) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= b.R) return;
  const double* al = b.alpha + r * b.N;
  const double* em = b.emission + r * b.N * 3;
  const uint8_t* va = b.valid ? b.valid + r * b.N : nullptr;
  double* wt = b.weights ? b.weights + r * b.N : nullptr;
  double tau = 0.0, prod = 1.0, cum = 0.0;
  double rad0 = 0.0, rad1 = 0.0, rad2 = 0.0;
  double sa = 0.0, sea0 = 0.0, sea1 = 0.0, sea2 = 0.0;  // θ₀ sums (tail ahead of saturation)
  int64_t k0 = b.N, nvalid = 0;
  double tk = 0.0, ek0 = b.bg[0], ek1 = b.bg[1], ek2 = b.bg[2];
  for (int64_t i = 0; i < b.N; ++i) {
    const bool v = va ? va[i] != 0 : true;
    nvalid += v;
    const double a = v ? __ldg(al + i) : 0.0;
    if (k0 < b.N) {  // past saturation: zero weight (compositor.py:137-140)
      if (wt) wt[i] = 0.0;
      continue;
    }
    const double raw = v ? extinction(m, a, tau, prod) : 0.0;
    const double cum_before = cum;
    cum += raw;
    const double e0 = __ldg(em + 3 * i), e1 = __ldg(em + 3 * i + 1), e2 = __ldg(em + 3 * i + 2);
    double w;
    if (cum >= 1.0) {  // the saturating sample
      k0 = i;
      w = 1.0 - cum_before;
      tk = w;
      ek0 = e0;
      ek1 = e1;
      ek2 = e2;
    } else {
      w = raw;
      if (i >= 1 && v) {
        sa += a;
        sea0 += a * e0;
        sea1 += a * e1;
        sea2 += a * e2;
      }
    }
    if (wt) wt[i] = w;
    rad0 += w * e0;
    rad1 += w * e1;
    rad2 += w * e2;
    tau += a;
    prod *= 1.0 - a;
  }
  const bool sat = k0 < b.N;
  const double res = sat ? 0.0 : 1.0 - cum;
  b.radiance[3 * r + 0] = rad0 + b.bg[0] * res;
  b.radiance[3 * r + 1] = rad1 + b.bg[1] * res;
  b.radiance[3 * r + 2] = rad2 + b.bg[2] * res;
  if (b.residual) b.residual[r] = res;
  if (b.k0) b.k0[r] = k0;
  if (b.overdraw) b.overdraw[r] = sat ? k0 + 1 : nvalid;
  if (b.e_k) {
    b.e_k[3 * r + 0] = ek0;
    b.e_k[3 * r + 1] = ek1;
    b.e_k[3 * r + 2] = ek2;
  }
  if (b.theta0) {
    b.theta0[3 * r + 0] = sea0 - ek0 * sa;
    b.theta0[3 * r + 1] = sea1 - ek1 * sa;
    b.theta0[3 * r + 2] = sea2 - ek2 * sa;
  }
  if (b.t_k) b.t_k[r] = sat ? tk : res;
}

}  // namespace nxs_batch

using namespace nxs_batch;

extern "C" int nxs_composite_batch(const nxs_model* model, const double* alpha,
                                   const double* emission, const uint8_t* valid, int64_t rays,
                                   int64_t samples, const double background[3], double* weights,
                                   double* radiance, double* residual, int64_t* k0,
                                   int64_t* overdraw, double* e_k, double* theta0, double* t_k,
                                   void* stream) {
  using nxs::set_last_error;
  if (!model || !background || !radiance || rays < 0 || samples < 0)
    return set_last_error(NXS_ERR_INVALID, "null argument or negative size");
  if (rays > 0 && samples > 0 && (!alpha || !emission))
    return set_last_error(NXS_ERR_INVALID, "null sample arrays");
  Model64 m{model->variant, model->param, 0.0, 0.0};
  const double p = model->param;
  switch (model->variant) {
    case NXS_MODEL_EXPONENTIAL:
    case NXS_MODEL_LINEAR: break;
    case NXS_MODEL_QUADRATIC:
      if (!(p >= -0.5)) return set_last_error(NXS_ERR_INVALID, "quadratic curvature must be >= -0.5");
      break;
    case NXS_MODEL_BLENDED:
    case NXS_MODEL_VICINI:
      if (!(p >= 0.0 && p <= 1.0)) return set_last_error(NXS_ERR_INVALID, "mix weight must be in [0, 1]");
      break;
    case NXS_MODEL_POWER_LAW:
      if (!(p >= -1.0)) return set_last_error(NXS_ERR_INVALID, "power-law exponent must be >= -1");
      if (p != -1.0 && std::fabs(p) >= 1e-4) m.ex = -(1.0 + p) / p;
      break;
    case NXS_MODEL_SOFTPLUS:
      if (!(p >= 10.0)) return set_last_error(NXS_ERR_INVALID, "softplus sharpness must be >= 10");
      m.K = p / (p + std::log1p(std::exp(-p)));  // κ / logaddexp(0, κ)
      break;
    default: return set_last_error(NXS_ERR_INVALID, "unknown transmittance variant");
  }
  if (rays == 0) return NXS_OK;
  BatchArgs b{alpha, emission, valid, rays, samples, {background[0], background[1], background[2]},
              weights, radiance, residual, k0, overdraw, e_k, theta0, t_k};
  k_composite_batch<<<(unsigned)((rays + 127) / 128), 128, 0, (cudaStream_t)stream>>>(m, b);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}
