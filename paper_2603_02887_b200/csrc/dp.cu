// Data-parallel gradient plumbing: the per-rank gradient
// buffer, its touched-row mask, and the pack / scatter of the rows a
// sparse all-reduce moves.  The reference has no data parallelism (it
// renders one view per optimizer iteration, optimizer.py:393-408); this is
// the B200 layer around the renderer's C-ABI.
//
// Gradient buffer layout (paper_2603_02887_b200/dp.py GradBuffer): one
// float32 array of n Gaussians, field after field,
//     [centers (n,3) | scales (n,3) | quats (n,4) | opacities (n) | sh (n,3,C)],
// so a Gaussian's row is 11 + 3C floats spread over five segments.
#include <algorithm>

#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "../../include/nxs.h"
#include "nxs_internal.cuh"

namespace nxs {
int set_last_error(int code, const char* msg);  // api.cu

namespace {

struct Layout {
  int64_t off[5];
  int w[5];
};
__host__ __device__ inline Layout layout_of(int64_t n, int C) {
  Layout L;
  const int w[5] = {3, 3, 4, 1, 3 * C};
  int64_t o = 0;
  for (int k = 0; k < 5; ++k) {
    L.off[k] = o;
    L.w[k] = w[k];
    o += (int64_t)w[k] * n;
  }
  return L;
}

// the Gaussians listed in a view's touched list -> mask bytes
__global__ void k_touched_mark(const uint32_t* __restrict__ list,
                               const unsigned long long* __restrict__ count, int64_t n,
                               uint8_t* __restrict__ mask) {
  nxs_pdl_enter();
  const unsigned long long m = *count;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t g = list[i];
    if (g < (uint64_t)n) mask[g] = 1;
  }
}

// zero every flagged Gaussian's row (all five segments) and clear its flag
__global__ void k_zero_masked(float* __restrict__ flat, int64_t n, int C,
                              uint8_t* __restrict__ mask) {
  nxs_pdl_enter();
  const Layout L = layout_of(n, C);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    if (!mask[g]) continue;
    mask[g] = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      float* row = flat + L.off[k] + g * L.w[k];
      for (int j = 0; j < L.w[k]; ++j) row[j] = 0.f;
    }
  }
}

// packed[i] = row of Gaussian index[i] (gather) or the reverse (scatter)
template <bool GATHER>
__global__ void k_rows(float* __restrict__ flat, int64_t n, int C,
                       const int32_t* __restrict__ index, int64_t m,
                       float* __restrict__ packed) {
  nxs_pdl_enter();
  const Layout L = layout_of(n, C);
  const int W = 11 + 3 * C;
  const int64_t total = m * W;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / W;
    int c = (int)(t - i * W);
    const int64_t g = index[i];
    int k = 0;
    while (c >= L.w[k]) c -= L.w[k++];
    float* p = flat + L.off[k] + g * L.w[k] + c;
    if (GATHER)
      packed[t] = *p;
    else
      *p = packed[t];
  }
}

unsigned grid_for(int64_t work, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

}  // namespace

void launch_touched_mark(const uint32_t* list, const unsigned long long* count, int64_t n,
                         uint8_t* mask, cudaStream_t s) {
  nxs_launch(k_touched_mark, grid_for(std::min<int64_t>(n, 1 << 20), 256), 256, 0, s, list, count, n,
                                                                               mask);
}

}  // namespace nxs

using namespace nxs;

extern "C" {

int nxs_grads_zero_masked(float* flat, int64_t n, int32_t sh_coeffs, uint8_t* mask,
                          void* stream) {
  if (!flat || !mask || n < 0 || (sh_coeffs != 1 && sh_coeffs != 4))
    return set_last_error(NXS_ERR_INVALID, "bad gradient buffer arguments");
  if (n == 0) return NXS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  nxs_launch(k_zero_masked, grid_for(n, 256), 256, 0, s, flat, n, sh_coeffs, mask);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

int nxs_grads_select(const uint8_t* mask, int64_t n, int32_t* index, int64_t* count,
                     void* stream) {
  if (!mask || !index || !count || n < 0 || n > 0x7fffffffll)
    return set_last_error(NXS_ERR_INVALID, "bad select arguments");
  *count = 0;
  if (n == 0) return NXS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  size_t bytes = 0;
  int* d_count = nullptr;
  void* temp = nullptr;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, bytes, cub::CountingInputIterator<int32_t>(0),
                                             mask, index, (int*)nullptr, (int)n, s);
  const size_t at = (bytes + 15) / 16 * 16;  // the count lives behind the CUB scratch
  if (e == cudaSuccess) e = cudaMallocAsync(&temp, at + 16, s);
  if (e == cudaSuccess) {
    d_count = reinterpret_cast<int*>(static_cast<char*>(temp) + at);
    e = cub::DeviceSelect::Flagged(temp, bytes, cub::CountingInputIterator<int32_t>(0), mask,
                                   index, d_count, (int)n, s);
  }
  int h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d_count, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (temp) cudaFreeAsync(temp, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
  *count = h;
  return NXS_OK;
}

int nxs_grads_gather(const float* flat, int64_t n, int32_t sh_coeffs, const int32_t* index,
                     int64_t count, float* packed, void* stream) {
  if (!flat || (count > 0 && (!index || !packed)) || (sh_coeffs != 1 && sh_coeffs != 4))
    return set_last_error(NXS_ERR_INVALID, "bad gather arguments");
  if (count <= 0) return NXS_OK;
  const int W = 11 + 3 * sh_coeffs;
  nxs_launch(k_rows<true>, grid_for(count * W, 256), 256, 0, (cudaStream_t)stream, 
      const_cast<float*>(flat), n, sh_coeffs, index, count, packed);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

int nxs_grads_scatter(float* flat, int64_t n, int32_t sh_coeffs, const int32_t* index,
                      int64_t count, const float* packed, void* stream) {
  if (!flat || (count > 0 && (!index || !packed)) || (sh_coeffs != 1 && sh_coeffs != 4))
    return set_last_error(NXS_ERR_INVALID, "bad scatter arguments");
  if (count <= 0) return NXS_OK;
  const int W = 11 + 3 * sh_coeffs;
  nxs_launch(k_rows<false>, grid_for(count * W, 256), 256, 0, (cudaStream_t)stream, 
      flat, n, sh_coeffs, index, count, const_cast<float*>(packed));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NXS_OK : set_last_error(NXS_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
