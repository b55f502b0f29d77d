// Micro-benchmark: per-tile ordering of (tile, rank) pairs.
//  (a) CUB DeviceRadixSort::SortPairs on 13-bit tile keys (current binning)
//  (b) per-tile scatter (atomic cursors) + cub::DeviceSegmentedSort::SortKeys
// Synthetic segment sizes (mean ~55, heavy tail), 8160 tiles.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void scatter(const unsigned* tile_of, const unsigned* rank_of, int n, const int* off,
                        int* cur, unsigned* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned t = tile_of[i];
  int p = off[t] + atomicAdd(&cur[t], 1);
  out[p] = rank_of[i];
}

int main() {
  const int T = 8160;
  std::mt19937 rng(1);
  std::lognormal_distribution<double> ln(3.5, 0.9);
  std::vector<int> cnt(T);
  long n = 0;
  for (int t = 0; t < T; ++t) { cnt[t] = std::min(4000, (int)ln(rng)); n += cnt[t]; }
  printf("pairs %ld, max seg %d\n", n, *std::max_element(cnt.begin(), cnt.end()));
  // pairs emitted in rank order: rank r hits a few tiles
  std::vector<unsigned> tile(n), rank(n);
  { long k = 0; std::vector<int> left(cnt);
    std::vector<int> order; for (int t = 0; t < T; ++t) for (int j = 0; j < cnt[t]; ++j) order.push_back(t);
    std::shuffle(order.begin(), order.end(), rng);
    for (long i = 0; i < n; ++i) { tile[i] = order[i]; rank[i] = (unsigned)i; } (void)k; (void)left; }
  std::vector<int> off(T + 1, 0);
  for (int t = 0; t < T; ++t) off[t + 1] = off[t] + cnt[t];
  unsigned *dk, *dv, *dk2, *dv2, *dtile, *drank, *dsc;
  int *doff, *dcur;
  CK(cudaMalloc(&dk, n * 4)); CK(cudaMalloc(&dv, n * 4)); CK(cudaMalloc(&dk2, n * 4));
  CK(cudaMalloc(&dv2, n * 4)); CK(cudaMalloc(&dtile, n * 4)); CK(cudaMalloc(&drank, n * 4));
  CK(cudaMalloc(&dsc, n * 4)); CK(cudaMalloc(&doff, (T + 1) * 4)); CK(cudaMalloc(&dcur, T * 4));
  CK(cudaMemcpy(dtile, tile.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drank, rank.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(doff, off.data(), (T + 1) * 4, cudaMemcpyHostToDevice));
  size_t ta = 0, tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, ta, dk, dk2, dv, dv2, (int)n, 0, 13);
  cub::DeviceSegmentedSort::SortKeys(nullptr, tb, dsc, dv2, (int)n, T, doff, doff + 1);
  void* tmp; CK(cudaMalloc(&tmp, std::max(ta, tb)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    // (a)
    CK(cudaMemcpy(dk, dtile, n * 4, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(dv, drank, n * 4, cudaMemcpyDeviceToDevice));
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) { size_t t = ta; cub::DeviceRadixSort::SortPairs(tmp, t, dk, dk2, dv, dv2, (int)n, 0, 13); }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // (b)
    cudaEvent_t f0, f1; cudaEventCreate(&f0); cudaEventCreate(&f1);
    cudaEventRecord(f0);
    for (int i = 0; i < 10; ++i) {
      cudaMemsetAsync(dcur, 0, T * 4);
      scatter<<<(n + 255) / 256, 256>>>(dtile, drank, (int)n, doff, dcur, dsc);
      size_t t = tb; cub::DeviceSegmentedSort::SortKeys(tmp, t, dsc, dk2, (int)n, T, doff, doff + 1);
    }
    cudaEventRecord(f1); cudaEventSynchronize(f1);
    float ms2; cudaEventElapsedTime(&ms2, f0, f1);
    // check equality
    std::vector<unsigned> a(n), b(n);
    CK(cudaMemcpy(a.data(), dv2, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), dk2, n * 4, cudaMemcpyDeviceToHost));
    printf("radix sort %.1f us, scatter+segmented sort %.1f us, equal %d\n", ms * 100, ms2 * 100, (int)(a == b));
  }
  return 0;
}
