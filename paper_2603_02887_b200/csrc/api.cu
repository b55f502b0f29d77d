// C-ABI of libnxs (include/nxs.h): view workspace management and the
// per-view pipeline
//   K0 depth keys -> CUB stable radix sort (64-bit fp64 keys) -> order
//   K1 projection + conic tile bbox (per rank)
//   CUB exclusive scan of tile counts -> K2 pair emission (rank order)
//   CUB stable radix sort of pairs by tile id -> tile ranges
//   K3 forward blend                                  (nxs_forward)
//   K4 back-to-front replay -> moments -> K5 chain    (nxs_backward)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <chrono>
#include <thread>

// NXS_HOST_TIMING=1: host-side time between points of one fused call,
// printed to stderr (diagnostics only)
namespace {
struct HostTimer {
  bool on = std::getenv("NXS_HOST_TIMING") != nullptr;
  int n = 0;
  const char* lab[32];
  std::chrono::steady_clock::time_point t[32];
  void mark(const char* l) {
    if (!on || n >= 32) return;
    lab[n] = l;
    t[n++] = std::chrono::steady_clock::now();
  }
  void dump() {
    if (!on) return;
    for (int i = 1; i < n; ++i)
      std::fprintf(stderr, "%s %.1f | ", lab[i],
                   std::chrono::duration<double, std::micro>(t[i] - t[i - 1]).count());
    std::fprintf(stderr, "\n");
    n = 0;
  }
};
HostTimer g_ht;
}  // namespace

#include "../../include/nxs.h"
#include "nxs_internal.cuh"

namespace nxs {
void launch_depth(const float*, const float*, const float*, const float*, int64_t, const CamDev&,
                  double, int, double*, unsigned long long*, uint32_t*, unsigned long long*,
                  cudaStream_t);
void launch_key32(const double*, int64_t, const unsigned long long*, uint32_t*, cudaStream_t);
void launch_key_fixup(const uint32_t*, uint32_t*, const double*, int64_t, unsigned long long*,
                      cudaStream_t, int shift = 0, const int* nd = nullptr);
void launch_rank_of(const uint32_t*, int64_t, uint32_t*, cudaStream_t);
void launch_rank_of_range(const uint32_t*, int64_t, int64_t, uint32_t*, cudaStream_t,
                          const int* nd = nullptr);
void launch_key32_hist_select(const double*, int64_t, const unsigned long long*, uint32_t*,
                              unsigned int*, const int64_t*, int, long long*, int,
                              unsigned long long*, unsigned int*, int*, cudaStream_t);
void launch_bin_scatter(const uint32_t*, int64_t, int, int, const long long*, unsigned int*,
                        uint32_t*, cudaStream_t);
void launch_bin_sort(uint32_t*, const double*, const unsigned int*, const unsigned int*, int, int,
                     const long long*, uint32_t*, unsigned long long*, cudaStream_t);
void launch_project_ranks(const float*, const float*, const float*, const float*, const float*,
                          int, int64_t, int64_t, const uint32_t*, const CamDev&, double, double,
                          int4*, float4*, float4*, unsigned long long*, double*, cudaStream_t,
                          const int* nd = nullptr, uint32_t* live = nullptr,
                          unsigned long long* n_live = nullptr);
void launch_gather_keys(const uint32_t*, const uint32_t*, int64_t, uint32_t*, cudaStream_t);
void launch_clear_rects(const uint32_t*, int64_t, int64_t, int4*, cudaStream_t);
void launch_iota(uint32_t*, int64_t, cudaStream_t);
void launch_phase_bound(const unsigned long long*, int, float*, cudaStream_t,
                        const long long* dbin = nullptr);
void launch_zlo_ranks(const float*, const float*, const float*, const float*, const uint32_t*,
                      int64_t, int64_t, const CamDev&, double, double*, cudaStream_t,
                      const int* nd = nullptr);
void launch_project_ranks_z(const float*, const float*, const float*, const float*, const float*,
                            int, int64_t, int64_t, const uint32_t*, const CamDev&, double, double,
                            const double*, float*, int4*, float4*, float4*, unsigned long long*,
                            double*, cudaStream_t, const int* nd = nullptr);
void launch_pack_check(const unsigned long long*, const long long*, int, unsigned long long*,
                       cudaStream_t);
void launch_call_init(unsigned long long*, uint8_t*, int32_t*, int2*, unsigned int*, int,
                      long long*, const int64_t*, int, unsigned int*, cudaStream_t);
void launch_dkeys(const double*, int64_t, unsigned long long*, cudaStream_t);
void launch_count_tiles(const int4*, const uint32_t*, int64_t, int64_t, int, const uint8_t*,
                        const unsigned int*, unsigned int*, const double*, const CamDev&,
                        cudaStream_t, const int* nd = nullptr);
void launch_tile_scan(unsigned int*, int, int2*, unsigned long long*, unsigned long long*,
                      unsigned long long, unsigned long long*, cudaStream_t);
void launch_emit_tiles(const int4*, const uint32_t*, int64_t, int64_t, int, const uint8_t*,
                       const int2*, unsigned int*, uint32_t*, const double*, const CamDev&,
                       cudaStream_t, const int* nd, unsigned long long cap,
                       const unsigned int* base = nullptr, unsigned long long* overflow = nullptr,
                       const uint32_t* live = nullptr, const unsigned long long* n_live = nullptr);
void launch_seg_sort(uint32_t*, int2*, unsigned int*, int, unsigned long long, cudaStream_t,
                     long long max_seg = -1, const unsigned int* base = nullptr,
                     unsigned long long* total = nullptr, unsigned long long* overflow = nullptr);
void launch_make_bases(const int2*, int, unsigned int*, cudaStream_t);
void launch_refresh_bases(const int2*, int, unsigned int*, unsigned long long, unsigned int,
                          cudaStream_t);
void launch_compact_lists(const uint32_t*, const int2*, const int*, int, uint32_t*, int2*,
                          cudaStream_t);
void launch_chunk_key(const float*, const float*, const float*, const float*, int64_t,
                      const CamDev&, double, const uint32_t*, int, double*, unsigned long long*,
                      uint32_t*, cudaStream_t);
bool launch_chunk_sort(const uint32_t*, const double*, int64_t, int, uint32_t*, cudaStream_t,
                       const int* nd = nullptr);
void launch_chunk_count(const int*, int64_t, int, int*, cudaStream_t);
void launch_copy_u32(const uint32_t*, int64_t, const int*, uint32_t*, cudaStream_t);
void launch_project(const float*, const float*, const float*, const float*, const float*, int,
                    int64_t, const uint32_t*, const CamDev&, double, double, const double*,
                    float*, int4*, float4*, float4*, unsigned long long*, double*, cudaStream_t);
void launch_blend_fwd_x(bool, int, const FwdXArgs&, const CamDev&, const ModelDev&,
                        const PixCache&, const PixResume&, Counters*, cudaStream_t);
void launch_blend_bwd_x(bool, int, const BwdXArgs&, const CamDev&, const ModelDev&,
                        const PixCache&, Counters*, cudaStream_t);
void launch_count_active(const int4*, const uint32_t*, int64_t, int64_t, int, const uint8_t*,
                         const unsigned int*, unsigned long long*, const double*, const CamDev&,
                         cudaStream_t, const int* nd = nullptr);
void launch_emit_pairs(const int4*, const uint32_t*, const unsigned long long*, int64_t, int64_t,
                       int, const uint8_t*, uint32_t*, uint32_t*, const double*, const CamDev&,
                       cudaStream_t, const int* nd = nullptr, unsigned long long cap = ~0ull);
void launch_tile_ranges(const uint32_t*, int64_t, int2*, cudaStream_t);
void launch_blend_fwd(bool, int, const FwdArgs&, const CamDev&, const ModelDev&, const PixCache&,
                      const PixResume&, Counters*, cudaStream_t);
void launch_blend_bwd(bool, int, const float4*, const float4*, const PhaseLists&, const CamDev&,
                      const ModelDev&, float, double, const float*, const float*,
                      const PixCache&, double*, uint8_t*, Counters*, cudaStream_t);
void launch_touched_mark(const uint32_t*, const unsigned long long*, int64_t, uint8_t*,
                         cudaStream_t);
void launch_det_reduce(int64_t, const uint32_t*, const int4*, int, const PhaseLists&,
                       const uint8_t*, double*, cudaStream_t);
void launch_chain(const float*, const float*, int, int64_t, const uint32_t*, double*, uint8_t*,
                  float*, float*, float*, float*, float*, uint32_t*, unsigned long long*,
                  cudaStream_t);
}  // namespace nxs

using namespace nxs;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define NXS_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(_e == cudaErrorMemoryAllocation ? NXS_ERR_NOMEM : NXS_ERR_CUDA,      \
                  std::string(#call) + ": " + cudaGetErrorString(_e));                 \
  } while (0)

#define NXS_LAUNCHED(what)                                                             \
  do {                                                                                 \
    ++v->stats.n_launches;                                                             \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess)                                                             \
      return fail(NXS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(_e));    \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  cudaError_t ensure(size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 8;  // headroom against regrowth
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

int bits_for(uint32_t n) {
  int b = 1;
  while (b < 32 && (1u << b) < n) ++b;
  return b;
}

}  // namespace

namespace nxs {
// lazy depth phases: Gaussians whose 32-bit key falls in bins [lo, hi]
struct BinRange {
  const uint32_t* key;
  int lo, hi;
  const long long* dev_hi = nullptr;  // device-sized phase 0: last bin from k_phase_select
  __host__ __device__ bool operator()(const uint32_t& i) const {
    const int b = (int)(key[i] >> 20);
    return b >= lo && b <= (dev_hi ? (int)*dev_hi : hi);
  }
};
// error reporting for entry points defined in other translation units
int set_last_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace nxs

struct nxs_view {
  // per Gaussian
  Buf dkeys_in, dkeys_out, idx_in, idx_out, records, bframe, rects, ntiles, offsets, moments,
      touched, depth, k32a, k32b, k32c, rank_of, rank_c, zlo_rank, seq, ph_hist, ph_sel, tq, zlo64,
      xc_t, xc_r, xc_n;
  // per pair: sort scratch, and the sorted ranks of each depth phase
  Buf pk_in, pk_out, pv_in, pv_ph[MAX_PHASES];
  // per tile: phase ranges and virtual offsets, activity
  Buf ranges_ph[MAX_PHASES], cum_ph[MAX_PHASES + 1], active, tile_cnt;
  Buf tile_last;  // per tile: max over its pixels' last list position (K3 -> K4)
  Buf live;       // device-sized phase 0: its ranks with a tile rectangle (count: dsmall[15])
  Buf bin_pos;  // per depth-key bin: first rank, then the scatter cursor
  // per-tile list capacities for the device-sized first phase (from the
  // view's last exact phase 0): emission needs no count pass while they hold
  Buf tile_base;
  bool bases_valid = false;
  int bases_ntiles = 0;
  CamDev bases_cam{};  // the camera the capacities were derived for
  int64_t bases_bound = 0;  // >= base[n_tiles], the pair buffer it needs
  bool async_bases = false;  // this call's device-sized pass uses them
  int64_t bases_maxcap = 0;  // the largest per-tile capacity
  // per pixel: replay cache and the forward carry between phases
  Buf c_last, c_sat, c_tk, c_thi, c_tlo, c_P, c_ck, c_Pck, c_ek, c_th0;
  Buf r_rad, r_trem, r_count, r_sea, r_sa;
  Buf temp, dev_small;  // CUB temp; counters
  Buf tlist, tcount;     // Gaussians the last backward's chain wrote, and their number
  Buf partial;           // deterministic mode: per (tile, entry) moment partials
  bool tlist_valid = false;
  unsigned long long* host_small = nullptr;  // pinned
  // phase events: see NXS_PHASES in include/nxs.h
  cudaEvent_t ev[NXS_PHASES + 2] = {};
  // per depth phase: [0] start, [1] after sort+ranges, [2] after the forward kernel
  // [0] start, [1] after the phase's depth sort, [2] after its projection
  // (both lazy phases only), [3] after binning, [4] after the forward blend
  cudaEvent_t evp[MAX_PHASES][5] = {};
  bool ev_ok = false;
  bool timing = false;  // record the phase events (nxs_view_set_timing)
  bool ev_fwd = false, ev_bwd = false;
  cudaEvent_t ev_sync = nullptr;  // host-side polling for the in-pipeline syncs
  // state of the last forward
  bool have_fwd = false;
  CamDev cam{};
  ModelDev model{};
  nxs_opts opts{};
  float bg[3] = {0, 0, 0};
  int64_t P = 0;
  int32_t C = 1;
  int64_t n_pairs = 0;  // pairs emitted over all phases
  int64_t ph_pairs[MAX_PHASES] = {0, 0, 0, 0};
  int n_phases = 0;
  int n_tiles = 0;
  // lazy depth phases: ranks [0, sorted_end) are sorted (and, for processed
  // phases, projected); key bins [0, bin_done] are consumed
  bool lazy = false;
  // speculative fused forward+backward: the forward stopped before checking
  // whether depth phase `spec_phase` is needed (the previous call of this
  // view needed `phases_needed` phases)
  bool spec_pending = false;
  int phases_needed = 0;
  // device-sized first phase: sizes of this view's last call (ranks, pairs,
  // last key bin); valid after a call whose phase 0 was sized exactly
  int64_t est_n0 = 0, est_pairs = 0;
  int est_bin0 = -1;
  bool async_pending = false;  // phase 0 ran device-sized, not yet verified
  int64_t async_chunk = 0;     // its chunk size (chunked order: whole chunks were projected)
  // fused call, t-ordered modes: the forward's pending-buffer overflow count
  // (host_small[28]) is read behind the backward instead of before it
  bool defer_ovf = false, ovf_pending = false;
  cudaEvent_t ev_ovf = nullptr;
  cudaGraphExec_t gexec = nullptr;  // the device-sized phase 0, replayed as one graph
  cudaStream_t cap_stream = nullptr;  // capture happens on this (non-default) stream
  // small device->host reads that must not sit between two pipeline kernels
  // run on this stream, ordered after the work they read by ev_side
  cudaStream_t copy_stream = nullptr;
  // first-phase hint: host_small[30] lands behind a forward on the side
  // stream; the planner uses it only once ev_hint reports the copy complete
  cudaEvent_t ev_hint = nullptr;
  cudaEvent_t ev_bases = nullptr;  // the side-stream capacity refresh of the last call
  bool bases_pending = false;
  bool hint_pending = false;
  unsigned long long hint = 0;
  int device = 0;  // the CUDA device this view's workspace lives on
  cudaEvent_t ev_side = nullptr;
  bool capturing = false;
  int n_phases_plan = 0;       // planned depth phases of the last forward
  int64_t async_cap0 = 0, async_capp = 0;
  int64_t sorted_end = 0, proj_end = 0;
  int bin_done = -1;
  const float* scene_centers = nullptr;
  nxs_stats stats{};

  template <class F>
  void for_each_buf(F f) {
    Buf* all[] = {&dkeys_in, &dkeys_out, &idx_in,  &idx_out, &records, &bframe, &rects,
                  &ntiles,   &offsets,   &moments, &touched, &pk_in,   &pk_out,  &pv_in,  &active,
                  &tile_cnt, &tile_last, &live, &bin_pos, &tile_base,
                  &depth,    &k32a,      &k32b,    &k32c,    &rank_of, &rank_c, &zlo_rank, &seq, &ph_hist,
                  &ph_sel,   &tq,      &zlo64,  &xc_t, &xc_r, &xc_n,
                  &c_last,   &c_sat,     &c_tk,    &c_thi,   &c_tlo,   &c_P,    &c_ck,
                  &c_Pck,    &c_ek,      &c_th0,   &r_rad,   &r_trem,  &r_count, &r_sea,
                  &r_sa,     &temp,      &dev_small, &tlist, &tcount, &partial};
    for (Buf* b : all) f(*b);
    for (int p = 0; p < MAX_PHASES; ++p) {
      f(pv_ph[p]);
      f(ranges_ph[p]);
    }
    for (int p = 0; p <= MAX_PHASES; ++p) f(cum_ph[p]);
  }
  ~nxs_view() {
    // work of this view may still be queued (the caller's stream, the side
    // stream's readbacks into host_small): let it drain before freeing
    cudaDeviceSynchronize();
    cudaGetLastError();
    for_each_buf([](Buf& b) { b.release(); });
    if (host_small) cudaFreeHost(host_small);
    if (ev_sync) cudaEventDestroy(ev_sync);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (ev_hint) cudaEventDestroy(ev_hint);
    if (ev_ovf) cudaEventDestroy(ev_ovf);
    if (ev_bases) cudaEventDestroy(ev_bases);
    if (ev_side) cudaEventDestroy(ev_side);
    if (ev_ok) {
      for (auto& e : ev) cudaEventDestroy(e);
      for (auto& row : evp)
        for (auto& e : row) cudaEventDestroy(e);
    }
  }
  int64_t bytes() {
    int64_t s = 0;
    for_each_buf([&](Buf& b) { s += (int64_t)b.cap; });
    return s;
  }
  PixCache cache() const {
    return PixCache{c_last.as<int32_t>(), c_sat.as<uint8_t>(), c_tk.as<float>(),
                    c_thi.as<float>(), c_tlo.as<float>(), c_P.as<float>(),
                    c_ck.as<int32_t>(), c_Pck.as<float>(), c_ek.as<float>(),
                    c_th0.as<float>()};
  }
  PixResume resume() const {
    return PixResume{r_rad.as<float>(), r_trem.as<float>(), r_count.as<int32_t>(),
                     r_sea.as<float>(), r_sa.as<float>()};
  }
};

namespace {

int make_model(const nxs_model* m, ModelDev& md) {
  md = ModelDev{};
  const double p = m->param;
  switch (m->variant) {
    case NXS_MODEL_EXPONENTIAL: md.fam = FAM_EXP; break;
    case NXS_MODEL_LINEAR: md.fam = FAM_LIN; break;
    case NXS_MODEL_QUADRATIC:
      if (!(p >= -0.5)) return fail(NXS_ERR_INVALID, "quadratic curvature must be >= -0.5");
      md.fam = FAM_QUAD;
      md.c = (float)p;
      break;
    case NXS_MODEL_BLENDED:
    case NXS_MODEL_VICINI:
      if (!(p >= 0.0 && p <= 1.0)) return fail(NXS_ERR_INVALID, "mix weight must be in [0, 1]");
      md.fam = FAM_BLEND;
      md.c = (float)p;
      break;
    case NXS_MODEL_POWER_LAW:
      if (!(p >= -1.0)) return fail(NXS_ERR_INVALID, "power-law exponent must be >= -1");
      if (p == -1.0) {
        md.fam = FAM_LIN;
      } else {
        md.fam = FAM_POW;
        md.c = (float)p;
        md.powmode = std::fabs(p) < 1e-4 ? 2 : 0;
        md.ex = (float)(-(1.0 + p) / p);
      }
      break;
    case NXS_MODEL_SOFTPLUS:
      if (!(p >= 10.0)) return fail(NXS_ERR_INVALID, "softplus sharpness must be >= 10");
      md.fam = FAM_SOFT;
      md.c = (float)p;
      md.K = (float)(p / (p + std::log1p(std::exp(-p))));
      break;
    default:
      return fail(NXS_ERR_INVALID, "unknown transmittance variant");
  }
  return NXS_OK;
}

int make_camera(const nxs_camera* c, CamDev& cd) {
  if (!(c->focal > 0) || c->width <= 0 || c->height <= 0)
    return fail(NXS_ERR_INVALID, "focal length and image dimensions must be positive");
  for (int i = 0; i < 3; ++i) cd.o[i] = c->position[i];
  for (int i = 0; i < 9; ++i) cd.R[i] = c->rotation[i];
  cd.f = c->focal;
  cd.cx = c->cx;
  cd.cy = c->cy;
  cd.W = c->width;
  cd.H = c->height;
  cd.tiles_x = (c->width + TILE - 1) / TILE;
  cd.tiles_y = (c->height + TILE - 1) / TILE;
  cd.inv_f = 1.0 / c->focal;
  for (int i = 0; i < 9; ++i) cd.Rf[i] = (float)c->rotation[i];
  return NXS_OK;
}

// Stream capture of the device-sized first phase: its ~30 launches (sort,
// projection, binning, forward) run as one CUDA graph, which removes the
// per-launch gaps between the many short kernels.  The host code runs as
// usual every call (all host-side state stays current); only the launches
// are recorded, and the executable graph is updated in place.
struct CaptureGuard {
  cudaStream_t s = nullptr;
  bool on = false;
  bool* flag = nullptr;
  ~CaptureGuard() {  // an error path left the capture open: close and drop it
    if (flag) *flag = false;
    if (on) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
    }
  }
};

inline bool same_camera(const CamDev& a, const CamDev& b) {
  for (int i = 0; i < 3; ++i)
    if (a.o[i] != b.o[i]) return false;
  for (int i = 0; i < 9; ++i)
    if (a.R[i] != b.R[i]) return false;
  return a.f == b.f && a.cx == b.cx && a.cy == b.cy && a.W == b.W && a.H == b.H;
}

// Makes the view's device current for the duration of a call (a view's
// workspace, events and graph belong to the device it was created on) and
// restores the caller's device afterwards.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
      prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Wait for the stream by polling an event: the syncs inside the pipeline
// (pair counts, phase sizes) sit between kernels, and a blocking wait's
// wake-up latency would leave the GPU idle; fall back to blocking if no
// event could be created.
cudaError_t spin_sync(nxs_view* v, cudaStream_t s) {
  if (!v->ev_sync) return cudaStreamSynchronize(s);
  cudaError_t e = cudaEventRecord(v->ev_sync, s);
  if (e != cudaSuccess) return e;
  while ((e = cudaEventQuery(v->ev_sync)) == cudaErrorNotReady) std::this_thread::yield();
  return e;
}

// timing events: inside a stream capture they must be external event
// nodes to stay observable from the host
inline void rec_event(nxs_view* v, cudaEvent_t e, cudaStream_t s) {
  if (!v->timing) return;  // (an event node costs the pipeline a few us)
  if (v->capturing)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

inline void mark(nxs_view* v, int i, cudaStream_t s) {
  if (v->ev_ok && v->timing) rec_event(v, v->ev[i], s);
}

template <class T>
cudaError_t ensure_n(Buf& b, int64_t n) {
  return b.ensure((size_t)n * sizeof(T));
}

// Lazy depth phases leave the ranks past the last processed phase unsorted;
// the exports complete the order (sort + fix-up of the remaining key bins)
// and mark the unprojected Gaussians' tile rectangles empty.
int complete_order(nxs_view* v, cudaStream_t s) {
  if (!v->lazy || v->sorted_end >= v->P) return NXS_OK;
  const int64_t r0 = v->sorted_end, n = v->P - r0;
  unsigned long long* dsmall = v->dev_small.as<unsigned long long>();
  NXS_CUDA(ensure_n<uint32_t>(v->k32c, v->P));
  NXS_CUDA(ensure_n<uint32_t>(v->k32b, v->P));
  size_t tbs = v->temp.cap;
  NXS_CUDA(cub::DeviceSelect::If(v->temp.p, tbs, cub::CountingInputIterator<uint32_t>(0),
                                 v->idx_in.as<uint32_t>(),
                                 reinterpret_cast<int*>(v->ph_sel.as<long long>() + 48),
                                 (int)v->P, BinRange{v->k32a.as<uint32_t>(), v->bin_done + 1, 4095},
                                 s));
  launch_gather_keys(v->idx_in.as<uint32_t>(), v->k32a.as<uint32_t>(), n, v->k32c.as<uint32_t>(),
                     s);
  NXS_LAUNCHED("gather_keys");
  size_t tb = v->temp.cap;
  NXS_CUDA(cub::DeviceRadixSort::SortPairs(v->temp.p, tb, v->k32c.as<uint32_t>(),
                                           v->k32b.as<uint32_t>() + r0, v->idx_in.as<uint32_t>(),
                                           v->idx_out.as<uint32_t>() + r0, (int)n, 0, 32, s));
  NXS_CUDA(cudaMemsetAsync(dsmall + 8, 0, sizeof(unsigned long long), s));
  launch_key_fixup(v->k32b.as<uint32_t>() + r0, v->idx_out.as<uint32_t>() + r0,
                   v->depth.as<double>(), n, dsmall + 8, s);
  NXS_LAUNCHED("key_fixup");
  NXS_CUDA(cudaMemcpyAsync(v->host_small + 6, dsmall + 8, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
  NXS_CUDA(spin_sync(v, s));
  if (v->host_small[6] != 0) {
    // a long equal-key run in the tail: the 64-bit sort of everything (its
    // prefix is the order the processed phases already used)
    launch_iota(v->idx_in.as<uint32_t>(), v->P, s);
    NXS_LAUNCHED("iota");
    launch_dkeys(v->depth.as<double>(), v->P, v->dkeys_in.as<unsigned long long>(), s);
    NXS_LAUNCHED("dkeys");
    size_t tb64 = 0;
    NXS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb64, v->dkeys_in.as<unsigned long long>(),
                                             v->dkeys_out.as<unsigned long long>(),
                                             v->idx_in.as<uint32_t>(), v->idx_out.as<uint32_t>(),
                                             (int)v->P, 0, 64, s));
    NXS_CUDA(v->temp.ensure(tb64));
    tb64 = v->temp.cap;
    NXS_CUDA(cub::DeviceRadixSort::SortPairs(v->temp.p, tb64, v->dkeys_in.as<unsigned long long>(),
                                             v->dkeys_out.as<unsigned long long>(),
                                             v->idx_in.as<uint32_t>(), v->idx_out.as<uint32_t>(),
                                             (int)v->P, 0, 64, s));
  }
  launch_rank_of_range(v->idx_out.as<uint32_t>(), r0, v->P, v->rank_of.as<uint32_t>(), s);
  NXS_LAUNCHED("rank_of");
  launch_clear_rects(v->idx_out.as<uint32_t>(), v->proj_end, v->P, v->rects.as<int4>(), s);
  NXS_LAUNCHED("clear_rects");
  v->sorted_end = v->P;
  v->bin_done = 4095;
  return NXS_OK;
}

}  // namespace

extern "C" {

int nxs_abi_version(void) { return NXS_ABI_VERSION; }

const char* nxs_error_string(int code) {
  switch (code) {
    case NXS_OK: return "ok";
    case NXS_ERR_INVALID: return "invalid argument";
    case NXS_ERR_UNSUPPORTED: return "unsupported mode or model";
    case NXS_ERR_CUDA: return "CUDA error";
    case NXS_ERR_NOMEM: return "out of device memory";
    case NXS_ERR_STATE: return "backward without a matching forward";
    case NXS_ERR_GEOMETRY: return "unsupported geometry";
    case NXS_ERR_OVERFLOW: return "exact-order pending buffer overflow";
    default: return "unknown error";
  }
}

const char* nxs_last_error(void) { return g_last_error.c_str(); }

int nxs_view_create(nxs_view** out) {
  if (!out) return fail(NXS_ERR_INVALID, "null output pointer");
  nxs_view* v = new (std::nothrow) nxs_view();
  if (!v) return fail(NXS_ERR_NOMEM, "host allocation failed");
  if (cudaHostAlloc((void**)&v->host_small, 64 * sizeof(unsigned long long),
                    cudaHostAllocDefault) != cudaSuccess) {
    delete v;
    cudaGetLastError();
    return fail(NXS_ERR_CUDA, "cudaHostAlloc failed (no CUDA device?)");
  }
  std::memset(v->host_small, 0, 64 * sizeof(unsigned long long));
  cudaGetDevice(&v->device);
  v->ev_ok = true;
  for (auto& e : v->ev) v->ev_ok = v->ev_ok && cudaEventCreate(&e) == cudaSuccess;
  for (auto& row : v->evp)
    for (auto& e : row) v->ev_ok = v->ev_ok && cudaEventCreate(&e) == cudaSuccess;
  if (cudaEventCreateWithFlags(&v->ev_sync, cudaEventDisableTiming) != cudaSuccess)
    v->ev_sync = nullptr;
  *out = v;
  return NXS_OK;
}

int nxs_view_destroy(nxs_view* view) {
  if (!view) return NXS_OK;
  DevGuard dg(view->device);
  delete view;
  return NXS_OK;
}

int nxs_view_stats(const nxs_view* view, nxs_stats* out) {
  if (!view || !out) return fail(NXS_ERR_INVALID, "null pointer");
  *out = view->stats;
  return NXS_OK;
}

int64_t nxs_view_bytes(const nxs_view* view) {
  return view ? const_cast<nxs_view*>(view)->bytes() : 0;
}

namespace {
int forward_impl(nxs_view* v, const nxs_scene* scene, const nxs_camera* camera,
                 const nxs_model* model, const nxs_opts* opts, const float background[3],
                 float* rgb, int32_t* overdraw, float* residual, void* stream_, int spec_phase);
}

int nxs_forward(nxs_view* v, const nxs_scene* scene, const nxs_camera* camera,
                const nxs_model* model, const nxs_opts* opts, const float background[3],
                float* rgb, int32_t* overdraw, float* residual, void* stream_) {
  return forward_impl(v, scene, camera, model, opts, background, rgb, overdraw, residual, stream_,
                      0);
}

}  // extern "C"

namespace {
// Read back and check a device-sized phase 0 (behind its forward kernel):
// host_small[3] = active tiles, [16..) = phase bounds (bin, end rank) of
// k_phase_select, [24] = phase-0 Gaussians, [25] = overflow flags, [26] =
// pair total.  The copies are enqueued (and v->ev_sync recorded) by
// enqueue_async_check; finish_async_check waits for them: ok == false means
// some capacity was exceeded and the pass must be redone with exact sizes.
// the copy stream, ordered after everything enqueued on s so far (s itself
// when the side stream cannot be created)
cudaError_t side_after(nxs_view* v, cudaStream_t s, cudaStream_t& out) {
  out = s;
  if (v->capturing) return cudaSuccess;
  if (!v->copy_stream &&
      cudaStreamCreateWithFlags(&v->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    v->copy_stream = nullptr;
    return cudaGetLastError(), cudaSuccess;
  }
  if (!v->ev_side &&
      cudaEventCreateWithFlags(&v->ev_side, cudaEventDisableTiming) != cudaSuccess) {
    v->ev_side = nullptr;
    return cudaGetLastError(), cudaSuccess;
  }
  cudaError_t e = cudaEventRecord(v->ev_side, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(v->copy_stream, v->ev_side, 0);
  if (e == cudaSuccess) out = v->copy_stream;
  return e;
}

int enqueue_async_check(nxs_view* v, int n_ph, cudaStream_t s) {
  // one small kernel packs the values into host_small's layout (in the
  // pipeline, ahead of the backward that would hold every SM), one copy on
  // the side stream (the backward does not wait for it)
  unsigned long long* dsmall = v->dev_small.as<unsigned long long>();
  long long* dsel = v->ph_sel.as<long long>();
  unsigned long long* pack = reinterpret_cast<unsigned long long*>(dsel + 56);
  launch_pack_check(dsmall, dsel, n_ph, pack, s);
  NXS_LAUNCHED("pack_check");
  cudaStream_t cs;
  NXS_CUDA(side_after(v, s, cs));
  NXS_CUDA(cudaMemcpyAsync(v->host_small, pack, 27 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, cs));
  NXS_CUDA(cudaEventRecord(v->ev_sync, cs));
  return NXS_OK;
}

int finish_async_check(nxs_view* v, bool& ok) {
  cudaError_t e;
  while ((e = cudaEventQuery(v->ev_sync)) == cudaErrorNotReady) std::this_thread::yield();
  NXS_CUDA(e);
  const int64_t n0 = (int64_t)(int)(uint32_t)v->host_small[24];
  const uint64_t pairs = v->host_small[26];
  ok = v->host_small[25] == 0 && n0 <= v->async_cap0 && (int64_t)pairs <= v->async_capp;
  v->async_pending = false;
  if (!ok) {
    ++v->stats.n_redo;
    if (std::getenv("NXS_DEBUG_PLAN"))
      std::fprintf(stderr, "redo: device-sized pass flags=%llu n0=%lld/%lld pairs=%llu/%lld\n",
                   (unsigned long long)v->host_small[25], (long long)n0,
                   (long long)v->async_cap0, (unsigned long long)pairs,
                   (long long)v->async_capp);
    v->est_n0 = 0;  // the next pass sizes phase 0 exactly again
    return NXS_OK;
  }
  const long long* hsel = reinterpret_cast<const long long*>(v->host_small + 16);
  v->est_n0 = n0;
  v->est_pairs = (int64_t)pairs;
  v->est_bin0 = (int)hsel[0];
  v->ph_pairs[0] = (int64_t)pairs;
  v->n_pairs = (int64_t)pairs;
  v->stats.n_pairs = (int64_t)pairs;
  v->stats.n_straddling = (int64_t)v->host_small[2];
  v->sorted_end = v->proj_end = n0;
  if (v->async_chunk > 1 && n0 < v->P)  // (chunked: only whole chunks were projected)
    v->proj_end = n0 / v->async_chunk * v->async_chunk;
  v->bin_done = (int)hsel[0];
  return NXS_OK;
}
}  // namespace

namespace {
int forward_impl(nxs_view* v, const nxs_scene* scene, const nxs_camera* camera,
                 const nxs_model* model, const nxs_opts* opts, const float background[3],
                 float* rgb, int32_t* overdraw, float* residual, void* stream_, int spec_phase) {
  if (!v || !scene || !camera || !model || !opts || !background || !rgb || !overdraw ||
      !residual)
    return fail(NXS_ERR_INVALID, "null argument");
  DevGuard dg(v->device);
  cudaStream_t s = (cudaStream_t)stream_;
  if (v->bases_pending) {  // the last call's side-stream capacity refresh
    NXS_CUDA(cudaStreamWaitEvent(s, v->ev_bases, 0));
    v->bases_pending = false;
  }
  v->have_fwd = false;
  v->spec_pending = false;
  CamDev cam;
  ModelDev md;
  int rc;
  if ((rc = make_camera(camera, cam)) != NXS_OK) return rc;
  if ((rc = make_model(model, md)) != NXS_OK) return rc;
  const int64_t P = scene->count;
  const int C = scene->sh_coeffs;
  if (P < 0 || (C != 1 && C != 4)) return fail(NXS_ERR_INVALID, "bad scene size or sh_coeffs");
  if (P > 0 && (!scene->centers || !scene->scales || !scene->quats || !scene->opacities ||
                !scene->sh))
    return fail(NXS_ERR_INVALID, "null scene array");
  if (P >= (int64_t)1 << 31) return fail(NXS_ERR_INVALID, "more than 2^31 Gaussians");
  if (opts->chunk_size < 0) return fail(NXS_ERR_INVALID, "chunk_size must be >= 0");
  // per-pixel t order within chunks: one chunk (exact, 0, or C >= P) or
  // chunks of C > 1 in centre-depth order; chunk_size 1 is the global order
  const bool chunked = opts->chunk_size > 1 && (int64_t)opts->chunk_size < P;
  const bool exact = opts->chunk_size == NXS_CHUNK_EXACT || (opts->chunk_size > 1 && !chunked);
  const bool torder = exact || chunked;
  if (torder && opts->max_splats > 4096)
    return fail(NXS_ERR_INVALID, "t-ordered modes support max_splats <= 4096");
  if (!(opts->alpha_cutoff > 0.0) || !(opts->near_plane >= 0.0))
    return fail(NXS_ERR_INVALID, "alpha_cutoff must be > 0 and near >= 0");

  const int64_t npix = (int64_t)cam.W * cam.H;
  const int n_tiles = cam.tiles_x * cam.tiles_y;
  {
    const int64_t launched = v->stats.n_launches;  // (cumulative over calls)
    const int64_t redone = v->stats.n_redo;
    v->stats = nxs_stats{};
    v->stats.n_launches = launched;
    v->stats.n_redo = redone;
  }
  v->stats.n_gaussians = P;
  v->stats.n_tiles = n_tiles;
  const bool count = (opts->flags & NXS_FLAG_COUNT_EVENTS) != 0;

  // ---- workspace
  NXS_CUDA(ensure_n<unsigned long long>(v->dkeys_in, P));
  NXS_CUDA(ensure_n<unsigned long long>(v->dkeys_out, P));
  NXS_CUDA(ensure_n<double>(v->depth, P));
  NXS_CUDA(ensure_n<uint32_t>(v->k32a, P));
  NXS_CUDA(ensure_n<uint32_t>(v->k32b, P));
  NXS_CUDA(ensure_n<uint32_t>(v->rank_of, P));
  NXS_CUDA(ensure_n<uint32_t>(v->idx_in, P));
  NXS_CUDA(ensure_n<uint32_t>(v->idx_out, P));
  NXS_CUDA(ensure_n<float4>(v->records, P * REC_F4));
  NXS_CUDA(ensure_n<float4>(v->bframe, P * 3));
  NXS_CUDA(ensure_n<int4>(v->rects, P));
  NXS_CUDA(ensure_n<double>(v->tq, P * 12));  // per rank: tile test + rect (project.cu TQ_STRIDE)
  NXS_CUDA(ensure_n<unsigned long long>(v->ntiles, P));
  NXS_CUDA(ensure_n<unsigned long long>(v->offsets, P));
  NXS_CUDA(ensure_n<uint8_t>(v->active, n_tiles));
  NXS_CUDA(ensure_n<int32_t>(v->c_last, npix));
  NXS_CUDA(ensure_n<uint8_t>(v->c_sat, npix));
  NXS_CUDA(ensure_n<float>(v->c_tk, npix));
  NXS_CUDA(ensure_n<float>(v->c_thi, npix));
  NXS_CUDA(ensure_n<float>(v->c_tlo, npix));
  NXS_CUDA(ensure_n<float>(v->c_P, npix));
  NXS_CUDA(ensure_n<int32_t>(v->c_ck, npix));
  NXS_CUDA(ensure_n<float>(v->c_Pck, npix));
  NXS_CUDA(ensure_n<float>(v->c_ek, npix * 3));
  NXS_CUDA(ensure_n<float>(v->c_th0, npix * 3));
  NXS_CUDA(v->dev_small.ensure(16 * sizeof(unsigned long long)));
  // dsmall: [0] straddle count, [1..4] event counters, [5] active tiles (u32),
  // [6] min depth key, [7] max depth key, [8] key-run overflow, [9] pending
  // overflow, [10]/[11] device-sized overflow/pairs, [12] last rank the
  // finished tiles needed, [13]/[14] pair total / longest tile list, [15] ranks
  // with a tile rectangle (device-sized phase 0: the emission list)
  unsigned long long* dsmall = v->dev_small.as<unsigned long long>();
  Counters* cnt = reinterpret_cast<Counters*>(dsmall + 1);
  unsigned int* n_active = reinterpret_cast<unsigned int*>(dsmall + 5);
  NXS_CUDA(ensure_n<int2>(v->ranges_ph[0], n_tiles));
  NXS_CUDA(ensure_n<int32_t>(v->cum_ph[0], n_tiles));
  NXS_CUDA(ensure_n<uint32_t>(v->tile_cnt, n_tiles));
  NXS_CUDA(ensure_n<int32_t>(v->tile_last, n_tiles));
  NXS_CUDA(ensure_n<uint32_t>(v->bin_pos, 4096 * 32));  // (one cursor per 128-byte line)
  NXS_CUDA(v->ph_hist.ensure(4097 * sizeof(unsigned int)));  // bins + ticket
  NXS_CUDA(v->ph_sel.ensure(96 * sizeof(long long)));
  if (P == 0) {  // (P > 0: k_call_init below, in the pipeline)
    NXS_CUDA(cudaMemsetAsync(dsmall, 0, 16 * sizeof(unsigned long long), s));
    NXS_CUDA(cudaMemsetAsync(v->active.p, 1, (size_t)n_tiles, s));
    NXS_CUDA(cudaMemsetAsync(v->cum_ph[0].p, 0, (size_t)n_tiles * 4, s));
    NXS_CUDA(cudaMemsetAsync(v->ranges_ph[0].p, 0, (size_t)n_tiles * sizeof(int2), s));
    NXS_CUDA(cudaMemsetAsync(v->tile_cnt.p, 0, (size_t)n_tiles * 4, s));
  }

  // ---- depth phases [R_p, R_{p+1}): R_1 = first phase, then x8.  The
  // chunked order cuts phases on chunk boundaries (nothing is pending
  // there); the exact order keeps per-pixel pending state: one phase.
  // a view whose camera changed since its last call (a pooled workspace
  // cycling the views of a step) sizes its device-sized pass from a nearby
  // camera's counts: wider headroom (fewer redone passes)
  const bool cam_moved = !same_camera(v->cam, cam);
  const int64_t hdiv = cam_moved ? 4 : 8;
  int64_t R[MAX_PHASES + 1];
  int n_ph = 0;
  {
    int64_t r1;
    if (opts->flags & NXS_FLAG_FULL_BINNING)
      r1 = P;
    else if (opts->first_phase_ranks > 0)
      r1 = opts->first_phase_ranks;
    else  // measured at C3: saturating models finish every tile within P/32
          // ranks (P/16 by z_lo, the looser exact-order key); exp never
          // saturates and runs to the 128 cap
      r1 = (md.fam == FAM_EXP) ? P / 4 : (exact ? P / 16 : P / 32);
    if (!(opts->flags & NXS_FLAG_FULL_BINNING) && opts->first_phase_ranks <= 0) {
      // this view's previous call reported the last rank its finished tiles
      // needed (host_small[30], copied behind that forward);
      // a first phase covering it (plus headroom) avoids a second phase, and
      // one no larger spares sorting, projecting and binning ranks no tile reads.
      // The hint only moves phase boundaries, never the result.
      if (v->hint_pending && v->ev_hint && cudaEventQuery(v->ev_hint) == cudaSuccess) {
        v->hint = v->host_small[30];
        v->hint_pending = false;
      }
      const int64_t need = (int64_t)v->hint;
      if (need > 0 && need < P) {
        const int64_t target = cam_moved ? need + need / 4 + 4096 : need + 1 + need / 16 + 1024;
        // (a nearby camera's need is only a guess: never below the default)
        r1 = cam_moved ? std::max(r1, target) : need < r1 ? std::min(r1, target) : target;
      }
      // device-sized phase-0 estimates that fell short: size exactly again
      if (need > 0 && v->est_n0 > 0 && need >= v->est_n0) v->est_n0 = 0;
    }
    r1 = std::max<int64_t>(r1, 4096);
    const int64_t unit = chunked ? opts->chunk_size : 1;
    auto up = [&](int64_t r) { return std::min(P, (r + unit - 1) / unit * unit); };
    R[0] = 0;
    int64_t r = up(r1);
    while (true) {
      R[++n_ph] = r;
      if (r >= P || n_ph == MAX_PHASES - 1) break;
      r = up(r * 8);
    }
    if (R[n_ph] < P) R[++n_ph] = P;
  }

  // depth order: 32-bit monotone keys + exact fix-up of equal-key runs;
  // the 64-bit sort is the fallback when a run is too long (retry below).
  // The global order sorts and projects lazily, one depth phase at a time
  // (only the phases the image needs); the t-ordered modes, full binning
  // and the 64-bit fallback sort and project everything up front.
  bool sort64 = false;
  v->n_phases_plan = n_ph;
  int64_t Rplan[MAX_PHASES + 1];
  const int n_ph_plan = n_ph;
  for (int i = 0; i <= n_ph; ++i) Rplan[i] = R[i];
  int ph_bin[MAX_PHASES] = {0, 0, 0, 0};  // last key bin of each lazy phase
  CaptureGuard cap;
  cap.flag = &v->capturing;
  const cudaStream_t s_caller = s;
  // device-sized phase 0 (no host sync before the first forward): needs
  // estimates from this view's previous call and a later phase to verify at
  // (a new camera's depth-key histogram differs: its phase-0 bins and pair
  // count are sized exactly, with host reads, rather than risk a redo)
  bool async0 = v->est_n0 > 0 && v->est_pairs >= 0 && v->est_bin0 >= 0 && n_ph >= 2 &&
                spec_phase >= 0 && !cam_moved && (!chunked || opts->chunk_size <= 2048);
  if (std::getenv("NXS_DEBUG_PLAN"))
    std::fprintf(stderr, "plan P=%lld n_ph=%d R1=%lld async0=%d est_n0=%lld est_bin0=%d hint=%llu\n",
                 (long long)P, n_ph, (long long)R[1], (int)async0, (long long)v->est_n0,
                 v->est_bin0, (unsigned long long)v->hint);
  int64_t proc_end = 0;  // chunked lazy phases: ranks [0, proc_end) are processed
  bool phase_full[MAX_PHASES] = {false, false, false, false};  // lazy phase sorted on 32 bits
  int phase_shift[MAX_PHASES] = {0, 0, 0, 0};
  g_ht.mark("setup");
retry_sort:
  if (sort64) async0 = false;
  v->async_pending = false;
  if (async0) {
    // every buffer the device-sized phase 0 touches is sized up front: no
    // allocation may move a buffer once its pointer is in the captured graph
    // per-tile capacities are camera-specific: a workspace shared by several
    // views (dp.py pools them) falls back to the counting pass on a new camera
    v->async_bases = v->bases_valid && v->bases_ntiles == n_tiles && same_camera(v->bases_cam, cam) &&
                     !getenv("NXS_NO_BASES");
    const int64_t capp =
        v->async_bases ? v->bases_bound : v->est_pairs + v->est_pairs / hdiv + 8192 * (8 / hdiv);
    // (the scratch the generic setup below sizes for a full sort / scan)
    size_t t_scan = 0, t_sel = 0, t_full = 0;
    NXS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_full, v->k32a.as<uint32_t>(),
                                             v->k32b.as<uint32_t>(), v->idx_in.as<uint32_t>(),
                                             v->idx_out.as<uint32_t>(), (int)P, 0, 32, s));
    NXS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, v->ntiles.as<unsigned long long>(),
                                           v->offsets.as<unsigned long long>(), (int)P, s));
    NXS_CUDA(cub::DeviceSelect::If(nullptr, t_sel, cub::CountingInputIterator<uint32_t>(0),
                                   v->idx_in.as<uint32_t>(), v->ph_sel.as<int>(), (int)P,
                                   BinRange{nullptr, 0, 0}, s));
    NXS_CUDA(v->temp.ensure(std::max({t_full, t_scan, t_sel})));
    NXS_CUDA(v->ph_hist.ensure(4097 * sizeof(unsigned int)));  // bins + ticket
    NXS_CUDA(v->ph_sel.ensure(96 * sizeof(long long)));
    NXS_CUDA(ensure_n<uint32_t>(v->pv_ph[0], capp));
    NXS_CUDA(ensure_n<uint32_t>(v->live, P));
    NXS_CUDA(ensure_n<int2>(v->ranges_ph[0], n_tiles));
    NXS_CUDA(ensure_n<int32_t>(v->cum_ph[0], n_tiles));
    NXS_CUDA(ensure_n<int32_t>(v->cum_ph[1], n_tiles));
    NXS_CUDA(ensure_n<float>(v->r_rad, npix * 3));
    NXS_CUDA(ensure_n<float>(v->r_trem, npix));
    NXS_CUDA(ensure_n<int32_t>(v->r_count, npix));
    NXS_CUDA(ensure_n<float>(v->r_sea, npix * 3));
    NXS_CUDA(ensure_n<float>(v->r_sa, npix));
    if (torder) {  // t-ordered phase 0: sequences, z_lo per rank, pending carry
      NXS_CUDA(ensure_n<int32_t>(v->seq, npix * std::max(1, opts->max_splats)));
      NXS_CUDA(ensure_n<float>(v->zlo_rank, P));
    }
    if (chunked) {  // chunk ids (centre-depth ranks), z_lo per Gaussian
      NXS_CUDA(ensure_n<uint32_t>(v->rank_c, P));
      NXS_CUDA(ensure_n<double>(v->zlo64, P));
    }
    if (exact) {
      NXS_CUDA(ensure_n<float>(v->xc_t, (int64_t)32 * npix));
      NXS_CUDA(ensure_n<int32_t>(v->xc_r, (int64_t)32 * npix));
      NXS_CUDA(ensure_n<int32_t>(v->xc_n, npix));
    }
  }
  if (async0 && !getenv("NXS_NO_GRAPH")) {
    // record on the view's own stream (the caller's may be the legacy default
    // stream, which cannot capture); the graph is launched on the caller's
    if (!v->cap_stream) NXS_CUDA(cudaStreamCreateWithFlags(&v->cap_stream, cudaStreamNonBlocking));
    s = v->cap_stream;
    g_ht.mark("presize");
    NXS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    cap.s = s;
    cap.on = true;
    v->capturing = true;
  }
  n_ph = n_ph_plan;
  for (int i = 0; i <= n_ph; ++i) R[i] = Rplan[i];
  // lazy depth phases: the global order, and the chunked order (phases end
  // on chunk boundaries; each phase's chunks are z_lo-sorted when complete)
  v->lazy = (!torder || exact || (chunked && opts->chunk_size <= 2048)) && !sort64 &&
            !(opts->flags & NXS_FLAG_FULL_BINNING) && P > 0;
  v->sorted_end = 0;
  v->proj_end = 0;
  v->bin_done = -1;
  proc_end = 0;
  if (exact && !v->lazy) {  // the exact order phases only lazily (pending carry)
    n_ph = 1;
    R[1] = P;
  }
  mark(v, 0, s);
  if (P > 0) {
    size_t tmp_sort = 0, tmp_scan = 0;
    if (sort64)
      NXS_CUDA(cub::DeviceRadixSort::SortPairs(
          nullptr, tmp_sort, v->dkeys_in.as<unsigned long long>(),
          v->dkeys_out.as<unsigned long long>(), v->idx_in.as<uint32_t>(),
          v->idx_out.as<uint32_t>(), (int)P, 0, 64, s));
    else
      NXS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, v->k32a.as<uint32_t>(),
                                               v->k32b.as<uint32_t>(), v->idx_in.as<uint32_t>(),
                                               v->idx_out.as<uint32_t>(), (int)P, 0, 32, s));
    NXS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan,
                                           v->ntiles.as<unsigned long long>(),
                                           v->offsets.as<unsigned long long>(), (int)P, s));
    if (chunked && opts->chunk_size > 2048) {
      size_t tmp_chunk = 0;
      NXS_CUDA(cub::DeviceRadixSort::SortPairs(
          nullptr, tmp_chunk, v->dkeys_in.as<unsigned long long>(),
          v->dkeys_out.as<unsigned long long>(), v->idx_in.as<uint32_t>(),
          v->idx_out.as<uint32_t>(), (int)P, 0, 64, s));
      tmp_sort = std::max(tmp_sort, tmp_chunk);
    }
    if (v->lazy) {
      size_t tmp_sel = 0;
      NXS_CUDA(cub::DeviceSelect::If(nullptr, tmp_sel, cub::CountingInputIterator<uint32_t>(0),
                                     v->idx_in.as<uint32_t>(), v->ph_sel.as<int>(), (int)P,
                                     BinRange{nullptr, 0, 0}, s));
      tmp_sort = std::max(tmp_sort, tmp_sel);
    }
    NXS_CUDA(v->temp.ensure(std::max(tmp_sort, tmp_scan)));
    // ---- counters, tile flags, phase-0 ranges/carry and the phase targets
    {
      int64_t tgt[4] = {0, 0, 0, 0};
      for (int p = 1; p < n_ph && p <= 4; ++p) tgt[p - 1] = R[p];
      launch_call_init(dsmall, v->active.as<uint8_t>(), v->cum_ph[0].as<int32_t>(),
                       v->ranges_ph[0].as<int2>(), v->tile_cnt.as<uint32_t>(), n_tiles,
                       v->lazy ? v->ph_sel.as<long long>() + 32 : nullptr, tgt, n_ph - 1,
                       v->ph_hist.as<unsigned int>(), s);
      NXS_LAUNCHED("call_init");
    }
    // ---- K0 depth (+ min/max) and the stable depth sort
    const bool keys64 = sort64 || !v->lazy;  // lazy phases need only the depths
    launch_depth(scene->centers, scene->scales, scene->quats, scene->opacities, P, cam,
                 opts->alpha_cutoff, exact ? 1 : 0, v->depth.as<double>(),
                 keys64 ? v->dkeys_in.as<unsigned long long>() : nullptr,
                 keys64 ? v->idx_in.as<uint32_t>() : nullptr, dsmall + 6, s);
    NXS_LAUNCHED("depth");
    size_t tb = v->temp.cap;
    if (sort64) {
      NXS_CUDA(cub::DeviceRadixSort::SortPairs(
          v->temp.p, tb, v->dkeys_in.as<unsigned long long>(),
          v->dkeys_out.as<unsigned long long>(), v->idx_in.as<uint32_t>(),
          v->idx_out.as<uint32_t>(), (int)P, 0, 64, s));
    } else if (v->lazy) {
      // phase boundaries on whole key bins: one host sync for their ranks
      // keys, their histogram and (last block) the phase selection, one launch
      long long* dsel = v->ph_sel.as<long long>();  // [32..) phase targets (k_call_init)
      if (async0) {
        // phase 0 sized from the previous call; the last bin it may use is
        // checked on the device (phase selection) and verified later
        ph_bin[0] = std::min(4095, v->est_bin0 + (cam_moved ? 8 : 2));
      }
      launch_key32_hist_select(v->depth.as<double>(), P, dsmall + 6, v->k32a.as<uint32_t>(),
                               v->ph_hist.as<unsigned int>(), reinterpret_cast<int64_t*>(dsel + 32),
                               n_ph - 1, dsel, async0 ? ph_bin[0] : -1,
                               async0 ? dsmall + 10 : nullptr, v->bin_pos.as<uint32_t>(),
                               async0 ? reinterpret_cast<int*>(dsel + 48) : nullptr, s);
      NXS_LAUNCHED("key32_hist_select");
      if (async0) {
        v->async_cap0 = std::min<int64_t>(P, v->est_n0 + v->est_n0 / hdiv + 2048 * (8 / hdiv));
        v->async_capp =
            v->async_bases ? v->bases_bound : v->est_pairs + v->est_pairs / hdiv + 8192 * (8 / hdiv);
        R[0] = 0;
        R[1] = v->async_cap0;  // ranks phase 0 may occupy; later bounds come with the check
      }
    }
    if (v->lazy && !async0) {
      long long* dsel = v->ph_sel.as<long long>();  // (selected by k_key32_hist_select)
      long long* hsel = reinterpret_cast<long long*>(v->host_small + 16);
      NXS_CUDA(cudaMemcpyAsync(hsel, dsel, sizeof(long long) * 2 * n_ph, cudaMemcpyDeviceToHost,
                               s));
      NXS_CUDA(spin_sync(v, s));
      // phases = bins (prev, ph_bin]; drop phases that came out empty
      int m = 0;
      int64_t last = 0;
      for (int p = 0; p < n_ph; ++p) {
        const int64_t end = hsel[2 * p + 1];
        if (end <= last && m > 0) continue;
        ph_bin[m] = (int)hsel[2 * p];
        R[++m] = std::max(end, last);
        last = R[m];
      }
      n_ph = m;
      R[0] = 0;
    } else if (!v->lazy && !sort64) {
      launch_key32(v->depth.as<double>(), P, dsmall + 6, v->k32a.as<uint32_t>(), s);
      NXS_LAUNCHED("key32");
      NXS_CUDA(cub::DeviceRadixSort::SortPairs(v->temp.p, tb, v->k32a.as<uint32_t>(),
                                               v->k32b.as<uint32_t>(), v->idx_in.as<uint32_t>(),
                                               v->idx_out.as<uint32_t>(), (int)P, 0, 32, s));
      launch_key_fixup(v->k32b.as<uint32_t>(), v->idx_out.as<uint32_t>(), v->depth.as<double>(),
                       P, dsmall + 8, s);
      NXS_LAUNCHED("key_fixup");
    }
    if (chunked && !v->lazy) {
      // chunk = centre-depth rank / C; lists in (chunk, z_lo) order: one
      // block radix sort per chunk, or a global 64-bit sort for huge chunks
      NXS_CUDA(ensure_n<uint32_t>(v->rank_c, P));
      launch_rank_of(v->idx_out.as<uint32_t>(), P, v->rank_c.as<uint32_t>(), s);
      NXS_LAUNCHED("rank_of");
      const bool block_sort = opts->chunk_size <= 2048;
      launch_chunk_key(scene->centers, scene->scales, scene->quats, scene->opacities, P, cam,
                       opts->alpha_cutoff, v->rank_c.as<uint32_t>(), opts->chunk_size,
                       v->depth.as<double>(),
                       block_sort ? nullptr : v->dkeys_in.as<unsigned long long>(),
                       v->idx_in.as<uint32_t>(), s);
      NXS_LAUNCHED("chunk_key");
      if (block_sort) {
        // centre order (idx_out) -> per-chunk z_lo order (idx_in) -> idx_out
        launch_chunk_sort(v->idx_out.as<uint32_t>(), v->depth.as<double>(), P, opts->chunk_size,
                          v->idx_in.as<uint32_t>(), s);
        NXS_LAUNCHED("chunk_sort");
        NXS_CUDA(cudaMemcpyAsync(v->idx_out.p, v->idx_in.p, (size_t)P * 4,
                                 cudaMemcpyDeviceToDevice, s));
      } else {
        const int n_chunks = (int)((P + opts->chunk_size - 1) / opts->chunk_size);
        size_t tb = v->temp.cap;
        NXS_CUDA(cub::DeviceRadixSort::SortPairs(
            v->temp.p, tb, v->dkeys_in.as<unsigned long long>(),
            v->dkeys_out.as<unsigned long long>(), v->idx_in.as<uint32_t>(),
            v->idx_out.as<uint32_t>(), (int)P, 0,
            32 + bits_for((uint32_t)std::max(n_chunks, 2)), s));
      }
    }
    if (!v->lazy) {
      launch_rank_of(v->idx_out.as<uint32_t>(), P, v->rank_of.as<uint32_t>(), s);
      NXS_LAUNCHED("rank_of");
      v->sorted_end = v->proj_end = P;
    }
  }
  mark(v, 1, s);
  if (P > 0 && !v->lazy) {
    // ---- K1 projection (all Gaussians, storage order; records land at their rank)
    if (torder) NXS_CUDA(ensure_n<float>(v->zlo_rank, P));
    launch_project(scene->centers, scene->scales, scene->quats, scene->opacities, scene->sh, C, P,
                   v->rank_of.as<uint32_t>(), cam, opts->alpha_cutoff, opts->near_plane,
                   torder ? v->depth.as<double>() : nullptr,
                   torder ? v->zlo_rank.as<float>() : nullptr, v->rects.as<int4>(),
                   v->records.as<float4>(), v->bframe.as<float4>(), dsmall, v->tq.as<double>(), s);
    NXS_LAUNCHED("project");
  }
  mark(v, 2, s);

  const float bgf[3] = {background[0], background[1], background[2]};
  const int tbits = bits_for((uint32_t)std::max(n_tiles, 2));
  int64_t total_pairs = 0;
  int ph_done = 0;
  // end the phase-0 capture (after its forward kernel) and launch the graph
  auto end_capture = [&]() -> int {
    cudaGraph_t g = nullptr;
    cap.on = false;
    v->capturing = false;
    NXS_CUDA(cudaStreamEndCapture(s, &g));
    s = s_caller;
    cudaGraphExecUpdateResultInfo info;
    if (!v->gexec || cudaGraphExecUpdate(v->gexec, g, &info) != cudaSuccess) {
      cudaGetLastError();
      if (v->gexec) cudaGraphExecDestroy(v->gexec);
      v->gexec = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&v->gexec, g, 0);
      if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        v->gexec = nullptr;
        return fail(NXS_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
      }
    }
    cudaGraphDestroy(g);
    NXS_CUDA(cudaGraphLaunch(v->gexec, s));
    g_ht.mark("graph");
    return NXS_OK;
  };
  for (int ph = 0; ph < n_ph; ++ph) {
    int64_t r0 = R[ph], r1 = R[ph + 1], nr = r1 - r0;
    if (v->ev_ok) rec_event(v, v->evp[ph][0], s);
    if (v->async_pending && ph > 0 && ph != spec_phase) {
      // verify the device-sized phase 0 and learn the real phase bounds
      bool ok = false;
      int rc2;
      if ((rc2 = enqueue_async_check(v, n_ph, s))) return rc2;
      if ((rc2 = finish_async_check(v, ok))) return rc2;
      if (!ok) {
        async0 = false;
        NXS_CUDA(cudaMemsetAsync(dsmall, 0, 16 * sizeof(unsigned long long), s));
        NXS_CUDA(cudaMemsetAsync(v->active.p, 1, (size_t)n_tiles, s));
        goto retry_sort;
      }
      if (chunked) proc_end = v->proj_end;  // (the next phase starts at the partial chunk)
      total_pairs += v->ph_pairs[0];
      const long long* hsel = reinterpret_cast<const long long*>(v->host_small + 16);
      int m = 0;
      int64_t last = 0;
      for (int p = 0; p < n_ph; ++p) {
        const int64_t end = hsel[2 * p + 1];
        if (end <= last && m > 0) continue;
        ph_bin[m] = (int)hsel[2 * p];
        R[++m] = std::max(end, last);
        last = R[m];
      }
      n_ph = m;
      R[0] = 0;
      if ((unsigned)v->host_small[3] == 0 || ph >= n_ph) {  // every tile finished
        v->phases_needed = 1;
        break;
      }
      r0 = R[ph];
      r1 = R[ph + 1];
      nr = r1 - r0;
    }
    if (async0 && ph == 0) {
      // ---- device-sized phase 0: every size below is an upper bound from
      // this view's previous call; the real counts stay on the device
      // (n_sel, pair total) and are verified behind the forward
      const int64_t cap0 = v->async_cap0, capp = v->async_capp;
      int* n_sel = reinterpret_cast<int*>(v->ph_sel.as<long long>() + 48);  // (k_phase_select)
      long long* dsel = v->ph_sel.as<long long>();
      // exact order of phase 0's key bins [0, dsel[0]]: scatter into the
      // bins' rank ranges, per-bin sort by (depth, index), ranks
      launch_bin_scatter(v->k32a.as<uint32_t>(), P, 0, 0, dsel, v->bin_pos.as<uint32_t>(),
                         v->idx_out.as<uint32_t>(), s);
      NXS_LAUNCHED("bin_scatter");
      launch_bin_sort(v->idx_out.as<uint32_t>(), v->depth.as<double>(),
                      v->ph_hist.as<unsigned int>(), v->bin_pos.as<uint32_t>(), 0, ph_bin[0], dsel,
                      chunked ? v->rank_c.as<uint32_t>() : v->rank_of.as<uint32_t>(), dsmall + 10,
                      s);
      NXS_LAUNCHED("bin_sort");
      if (v->ev_ok) rec_event(v, v->evp[0][1], s);
      if (chunked) {
        // whole chunks of the selected Gaussians (the partial last one waits
        // for the next phase): z_lo, per-chunk z_lo sort, ranks, projection
        int* n_ch = reinterpret_cast<int*>(v->ph_sel.as<long long>() + 52);
        launch_chunk_count(n_sel, P, opts->chunk_size, n_ch, s);
        launch_zlo_ranks(scene->centers, scene->scales, scene->quats, scene->opacities,
                         v->idx_out.as<uint32_t>(), 0, cap0, cam, opts->alpha_cutoff,
                         v->zlo64.as<double>(), s, n_ch);
        NXS_LAUNCHED("zlo_ranks");
        launch_chunk_sort(v->idx_out.as<uint32_t>(), v->zlo64.as<double>(), cap0,
                          (int)opts->chunk_size, v->idx_in.as<uint32_t>(), s, n_ch);
        NXS_LAUNCHED("chunk_sort");
        launch_copy_u32(v->idx_in.as<uint32_t>(), cap0, n_ch, v->idx_out.as<uint32_t>(), s);
        launch_rank_of_range(v->idx_out.as<uint32_t>(), 0, cap0, v->rank_of.as<uint32_t>(), s,
                             n_ch);
        NXS_LAUNCHED("rank_of");
        launch_project_ranks_z(scene->centers, scene->scales, scene->quats, scene->opacities,
                               scene->sh, C, 0, cap0, v->idx_out.as<uint32_t>(), cam,
                               opts->alpha_cutoff, opts->near_plane, v->zlo64.as<double>(),
                               v->zlo_rank.as<float>(), v->rects.as<int4>(),
                               v->records.as<float4>(), v->bframe.as<float4>(), dsmall,
                               v->tq.as<double>(), s, n_ch);
        n_sel = n_ch;  // the binning below takes the processed (whole-chunk) ranks
      } else if (exact)  // (z_lo per rank too: the pending-buffer bounds)
        launch_project_ranks_z(scene->centers, scene->scales, scene->quats, scene->opacities,
                               scene->sh, C, 0, cap0, v->idx_out.as<uint32_t>(), cam,
                               opts->alpha_cutoff, opts->near_plane, v->depth.as<double>(),
                               v->zlo_rank.as<float>(), v->rects.as<int4>(),
                               v->records.as<float4>(), v->bframe.as<float4>(), dsmall,
                               v->tq.as<double>(), s, n_sel);
      else
        launch_project_ranks(scene->centers, scene->scales, scene->quats, scene->opacities,
                             scene->sh, C, 0, cap0, v->idx_out.as<uint32_t>(), cam,
                             opts->alpha_cutoff, opts->near_plane, v->rects.as<int4>(),
                             v->records.as<float4>(), v->bframe.as<float4>(), dsmall,
                             v->tq.as<double>(), s, n_sel,
                             v->async_bases ? v->live.as<uint32_t>() : nullptr, dsmall + 15);
      NXS_LAUNCHED("project_ranks");
      if (v->ev_ok) rec_event(v, v->evp[0][2], s);
      NXS_CUDA(ensure_n<int2>(v->ranges_ph[0], n_tiles));
      NXS_CUDA(ensure_n<int32_t>(v->cum_ph[1], n_tiles));
      NXS_CUDA(ensure_n<uint32_t>(v->pv_ph[0], capp));
      if (v->async_bases) {
        // ---- per-tile capacities of the view's last pass: emission at
        // base + cursor (an exceeded capacity is flagged and the pass redone),
        // the list sort writes the ranges and the pair total
        mark(v, 3, s);
        launch_emit_tiles(v->rects.as<int4>(), v->idx_out.as<uint32_t>(), 0, cap0, cam.tiles_x,
                          v->active.as<uint8_t>(), nullptr, v->tile_cnt.as<uint32_t>(),
                          v->pv_ph[0].as<uint32_t>(), v->tq.as<double>(), cam, s, n_sel,
                          (unsigned long long)capp, v->tile_base.as<uint32_t>(), dsmall + 10,
                          v->live.as<uint32_t>(), dsmall + 15);
        NXS_LAUNCHED("emit_tiles");
        mark(v, 4, s);
        launch_seg_sort(v->pv_ph[0].as<uint32_t>(), v->ranges_ph[0].as<int2>(),
                        v->tile_cnt.as<uint32_t>(), n_tiles, (unsigned long long)capp, s,
                        v->bases_maxcap, v->tile_base.as<uint32_t>(), dsmall + 11, dsmall + 10);
        NXS_LAUNCHED("seg_sort");
        if (v->bases_maxcap > 256) ++v->stats.n_launches;  // (long lists: a second kernel)
      } else {
        // ---- tile-major binning: per-tile counts, one scan over the tiles
        // (ranges, total vs capacity, longest list), emission at per-tile
        // cursors, per-tile sort by rank
        launch_count_tiles(v->rects.as<int4>(), v->idx_out.as<uint32_t>(), 0, cap0, cam.tiles_x,
                           v->active.as<uint8_t>(), nullptr, v->tile_cnt.as<uint32_t>(),
                           v->tq.as<double>(), cam, s, n_sel);
        NXS_LAUNCHED("count_tiles");
        mark(v, 3, s);
        launch_tile_scan(v->tile_cnt.as<uint32_t>(), n_tiles, v->ranges_ph[0].as<int2>(),
                         dsmall + 11, dsmall + 14, (unsigned long long)capp, dsmall + 10, s);
        NXS_LAUNCHED("tile_scan");
        launch_emit_tiles(v->rects.as<int4>(), v->idx_out.as<uint32_t>(), 0, cap0, cam.tiles_x,
                          v->active.as<uint8_t>(), v->ranges_ph[0].as<int2>(),
                          v->tile_cnt.as<uint32_t>(), v->pv_ph[0].as<uint32_t>(),
                          v->tq.as<double>(), cam, s, n_sel, (unsigned long long)capp);
        NXS_LAUNCHED("emit_tiles");
        mark(v, 4, s);
        launch_seg_sort(v->pv_ph[0].as<uint32_t>(), v->ranges_ph[0].as<int2>(),
                        v->tile_cnt.as<uint32_t>(), n_tiles, (unsigned long long)capp, s);
        NXS_LAUNCHED("seg_sort");
        ++v->stats.n_launches;  // (short and long lists: two kernels)
      }
      mark(v, 5, s);
      mark(v, 6, s);
      if (v->ev_ok) rec_event(v, v->evp[0][3], s);
      v->async_pending = true;
      v->async_chunk = chunked ? opts->chunk_size : 0;
      v->ph_pairs[0] = capp;  // capacity; the real count comes with the check
    } else {
      if (v->lazy) {
        if (ph > 0 && ph == spec_phase) {
          // fused call: the backward goes ahead and the check overlaps it
          v->spec_pending = true;
          break;
        }
        if (ph > 0 && !(ph == 1 && async0)) {
          // the previous phase's forward decides whether this one is needed
          NXS_CUDA(cudaMemcpyAsync(v->host_small + 3, n_active, sizeof(unsigned int),
                                   cudaMemcpyDeviceToHost, s));
          NXS_CUDA(spin_sync(v, s));
          if ((unsigned)v->host_small[3] == 0) {  // every tile finished
            v->phases_needed = ph;
            break;
          }
        }
        if (nr > 0) {
          // ---- this phase's Gaussians (key bins (prev, ph_bin]) in storage
          // order, 32-bit sort + fix-up into ranks [r0, r1), projection
          const int lo = ph == 0 ? 0 : ph_bin[ph - 1] + 1, hi = ph_bin[ph];
          if (!phase_full[ph]) {
            // scatter into the bins' rank ranges, per-bin exact sort, ranks
            // (a bin too long for one block redoes the phase with the sort)
            NXS_CUDA(ensure_n<uint32_t>(chunked ? v->rank_c : v->rank_of, P));
            launch_bin_scatter(v->k32a.as<uint32_t>(), P, lo, hi, nullptr,
                               v->bin_pos.as<uint32_t>(), v->idx_out.as<uint32_t>(), s);
            NXS_LAUNCHED("bin_scatter");
            launch_bin_sort(v->idx_out.as<uint32_t>(), v->depth.as<double>(),
                            v->ph_hist.as<unsigned int>(), v->bin_pos.as<uint32_t>(), lo, hi,
                            nullptr, chunked ? v->rank_c.as<uint32_t>() : v->rank_of.as<uint32_t>(),
                            dsmall + 8, s);
            NXS_LAUNCHED("bin_sort");
            phase_shift[ph] = 1;  // (an overflow redoes the phase with the radix sort)
          } else {
            size_t tbs = v->temp.cap;
            NXS_CUDA(cub::DeviceSelect::If(v->temp.p, tbs, cub::CountingInputIterator<uint32_t>(0),
                                           v->idx_in.as<uint32_t>(),
                                           reinterpret_cast<int*>(v->ph_sel.as<long long>() + 48),
                                           (int)P, BinRange{v->k32a.as<uint32_t>(), lo, hi}, s));
            NXS_CUDA(ensure_n<uint32_t>(v->k32c, P));
            launch_gather_keys(v->idx_in.as<uint32_t>(), v->k32a.as<uint32_t>(), nr,
                               v->k32c.as<uint32_t>(), s);
            NXS_LAUNCHED("gather_keys");
            // 32-bit radix sort; the fix-up re-sorts equal keys exactly (a
            // run over 256 falls back to the 64-bit sort)
            size_t tb = v->temp.cap;
            NXS_CUDA(cub::DeviceRadixSort::SortPairs(v->temp.p, tb, v->k32c.as<uint32_t>(),
                                                     v->k32b.as<uint32_t>() + r0,
                                                     v->idx_in.as<uint32_t>(),
                                                     v->idx_out.as<uint32_t>() + r0, (int)nr, 0,
                                                     32, s));
            launch_key_fixup(v->k32b.as<uint32_t>() + r0, v->idx_out.as<uint32_t>() + r0,
                             v->depth.as<double>(), nr, dsmall + 8, s, 0);
            NXS_LAUNCHED("key_fixup");
            phase_shift[ph] = 0;
            NXS_CUDA(ensure_n<uint32_t>(chunked ? v->rank_c : v->rank_of, P));
            launch_rank_of_range(v->idx_out.as<uint32_t>(), r0, r1,
                                 chunked ? v->rank_c.as<uint32_t>() : v->rank_of.as<uint32_t>(), s);
            NXS_LAUNCHED("rank_of");
          }
          v->sorted_end = r1;
          v->bin_done = hi;
          if (chunked) {
            // centre-depth ranks of this phase, then the complete chunks it
            // finishes, [proc_end, p1), sorted by z_lo and processed
            NXS_CUDA(ensure_n<uint32_t>(v->rank_c, P));
            NXS_CUDA(ensure_n<double>(v->zlo64, P));
            NXS_CUDA(ensure_n<float>(v->zlo_rank, P));
            // (rank_c of this phase was written with the sort)
            const int64_t Cc = opts->chunk_size;
            const int64_t p0 = proc_end, p1 = (r1 >= P) ? P : (r1 / Cc) * Cc;
            if (v->ev_ok) rec_event(v, v->evp[ph][1], s);
            if (p1 > p0) {
              launch_zlo_ranks(scene->centers, scene->scales, scene->quats, scene->opacities,
                               v->idx_out.as<uint32_t>(), p0, p1, cam, opts->alpha_cutoff,
                               v->zlo64.as<double>(), s);
              NXS_LAUNCHED("zlo_ranks");
              launch_chunk_sort(v->idx_out.as<uint32_t>() + p0, v->zlo64.as<double>(), p1 - p0,
                                (int)Cc, v->idx_in.as<uint32_t>() + p0, s);
              NXS_LAUNCHED("chunk_sort");
              NXS_CUDA(cudaMemcpyAsync(v->idx_out.as<uint32_t>() + p0,
                                       v->idx_in.as<uint32_t>() + p0, (size_t)(p1 - p0) * 4,
                                       cudaMemcpyDeviceToDevice, s));
              launch_rank_of_range(v->idx_out.as<uint32_t>(), p0, p1, v->rank_of.as<uint32_t>(), s);
              NXS_LAUNCHED("rank_of");
              launch_project_ranks_z(scene->centers, scene->scales, scene->quats,
                                     scene->opacities, scene->sh, C, p0, p1,
                                     v->idx_out.as<uint32_t>(), cam, opts->alpha_cutoff,
                                     opts->near_plane, v->zlo64.as<double>(),
                                     v->zlo_rank.as<float>(), v->rects.as<int4>(),
                                     v->records.as<float4>(), v->bframe.as<float4>(), dsmall,
                                     v->tq.as<double>(), s);
              NXS_LAUNCHED("project_ranks");
            }
            proc_end = p1;
            v->proj_end = p1;
            r0 = p0;  // the rest of the phase works on the processed ranks
            r1 = p1;
            nr = p1 - p0;
          } else {
            // (rank_of of this phase was written with the sort)
            if (v->ev_ok) rec_event(v, v->evp[ph][1], s);
            if (exact) {  // z_lo per rank for the pending-buffer bounds
              NXS_CUDA(ensure_n<float>(v->zlo_rank, P));
              launch_project_ranks_z(scene->centers, scene->scales, scene->quats,
                                     scene->opacities, scene->sh, C, r0, r1,
                                     v->idx_out.as<uint32_t>(), cam, opts->alpha_cutoff,
                                     opts->near_plane, v->depth.as<double>(),
                                     v->zlo_rank.as<float>(), v->rects.as<int4>(),
                                     v->records.as<float4>(), v->bframe.as<float4>(), dsmall,
                                     v->tq.as<double>(), s);
            } else {
              launch_project_ranks(scene->centers, scene->scales, scene->quats, scene->opacities,
                                   scene->sh, C, r0, r1, v->idx_out.as<uint32_t>(), cam,
                                   opts->alpha_cutoff, opts->near_plane, v->rects.as<int4>(),
                                   v->records.as<float4>(), v->bframe.as<float4>(), dsmall,
                                   v->tq.as<double>(), s);
            }
            NXS_LAUNCHED("project_ranks");
            v->proj_end = r1;
          }
        } else if (v->ev_ok) {
          rec_event(v, v->evp[ph][1], s);
        }
        if (v->ev_ok) rec_event(v, v->evp[ph][2], s);
      } else if (v->ev_ok) {
        rec_event(v, v->evp[ph][1], s);
        rec_event(v, v->evp[ph][2], s);
      }
      // ---- K2a counts over active tiles, scan, one host sync for the pair count
      NXS_CUDA(ensure_n<int2>(v->ranges_ph[ph], n_tiles));
      if (nr > 0) {
        // per-tile counts and one scan over the tiles: ranges, total, longest list
        launch_count_tiles(v->rects.as<int4>(), v->idx_out.as<uint32_t>(), r0, r1, cam.tiles_x,
                           v->active.as<uint8_t>(), ph > 0 ? n_active : nullptr,
                           v->tile_cnt.as<uint32_t>(), v->tq.as<double>(), cam,
                           s);
        NXS_LAUNCHED("count_tiles");
        launch_tile_scan(v->tile_cnt.as<uint32_t>(), n_tiles, v->ranges_ph[ph].as<int2>(),
                         dsmall + 13, dsmall + 14, ~0ull, nullptr, s);
        NXS_LAUNCHED("tile_scan");
      }
      // one copy of the small device counters (pair total and longest list,
      // straddle count, active tiles, key-run overflow) behind the counting
      unsigned long long* mirror = v->host_small + 32;
      NXS_CUDA(cudaMemcpyAsync(mirror, dsmall, 16 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
      NXS_CUDA(spin_sync(v, s));
      v->host_small[0] = nr > 0 ? mirror[13] : 0ull;
      v->host_small[1] = nr > 0 ? mirror[14] : 0ull;
      v->host_small[2] = mirror[0];
      v->host_small[3] = (unsigned int)mirror[5];
      if (ph == 0 || v->lazy) v->host_small[6] = mirror[8];
      if (v->lazy && v->host_small[6] != 0 && phase_shift[ph] > 0) {
        // a long run of equal truncated keys: redo this phase on all 32 bits
        phase_full[ph] = true;
        NXS_CUDA(cudaMemsetAsync(dsmall + 8, 0, sizeof(unsigned long long), s));
        --ph;
        continue;
      }
      if ((ph == 0 || v->lazy) && !sort64 && v->host_small[6] != 0) {
        // an equal-key run longer than the fix-up handles: redo with 64-bit keys
        sort64 = true;
        NXS_CUDA(cudaMemsetAsync(dsmall, 0, 16 * sizeof(unsigned long long), s));
        goto retry_sort;
      }
      if (ph == 0) mark(v, 3, s);
      const unsigned long long n_pairs = v->host_small[0];
      const unsigned long long max_seg = v->host_small[1];
      v->stats.n_straddling = (int64_t)v->host_small[2];
      if (ph > 0 && !v->lazy && (unsigned)v->host_small[3] == 0) break;  // every tile finished
      if (n_pairs >= (1ull << 31)) return fail(NXS_ERR_NOMEM, "more than 2^31 tile pairs");
      total_pairs += (int64_t)n_pairs;
      v->ph_pairs[ph] = (int64_t)n_pairs;

      NXS_CUDA(ensure_n<int32_t>(v->cum_ph[ph + 1], n_tiles));
      NXS_CUDA(ensure_n<uint32_t>(v->pv_ph[ph], std::max<int64_t>(1, (int64_t)n_pairs)));
      if (n_pairs > 0 && max_seg <= (unsigned long long)SEG_MAX) {
        // ---- K2b emission at the per-tile cursors, per-tile sort by rank
        launch_emit_tiles(v->rects.as<int4>(), v->idx_out.as<uint32_t>(), r0, r1, cam.tiles_x,
                          v->active.as<uint8_t>(), v->ranges_ph[ph].as<int2>(),
                          v->tile_cnt.as<uint32_t>(), v->pv_ph[ph].as<uint32_t>(),
                          v->tq.as<double>(), cam, s, nullptr, n_pairs);
        NXS_LAUNCHED("emit_tiles");
        if (ph == 0) mark(v, 4, s);
        launch_seg_sort(v->pv_ph[ph].as<uint32_t>(), v->ranges_ph[ph].as<int2>(),
                        v->tile_cnt.as<uint32_t>(), n_tiles, n_pairs, s, (long long)max_seg);
        NXS_LAUNCHED("seg_sort");
        if (max_seg > 256) ++v->stats.n_launches;  // (long lists: a second kernel)
        if (ph == 0 && v->lazy && !torder) {
          // per-tile capacities for this view's next device-sized pass
          NXS_CUDA(ensure_n<uint32_t>(v->tile_base, (int64_t)n_tiles + 1));
          launch_make_bases(v->ranges_ph[0].as<int2>(), n_tiles, v->tile_base.as<uint32_t>(), s);
          NXS_LAUNCHED("make_bases");
          v->bases_valid = true;
          v->bases_ntiles = n_tiles;
          v->bases_cam = cam;
          v->bases_bound = (int64_t)n_pairs + (int64_t)n_pairs / 8 + 8 * (int64_t)n_tiles + 1;
          v->bases_maxcap = (int64_t)max_seg + (int64_t)max_seg / 8 + 8;
        }
        if (ph == 0) mark(v, 5, s);
      } else if (n_pairs > 0) {
        // a tile list longer than the per-tile sort takes: per-rank counts,
        // emission in rank order and a stable radix sort by tile
        NXS_CUDA(cudaMemsetAsync(v->tile_cnt.p, 0, (size_t)n_tiles * 4, s));
        launch_count_active(v->rects.as<int4>(), v->idx_out.as<uint32_t>(), r0, r1, cam.tiles_x,
                            v->active.as<uint8_t>(), nullptr, v->ntiles.as<unsigned long long>(),
                            v->tq.as<double>(), cam, s);
        NXS_LAUNCHED("count_active");
        size_t tbo = v->temp.cap;
        NXS_CUDA(cub::DeviceScan::ExclusiveSum(v->temp.p, tbo, v->ntiles.as<unsigned long long>(),
                                               v->offsets.as<unsigned long long>(), (int)nr, s));
        NXS_CUDA(cudaMemsetAsync(v->ranges_ph[ph].p, 0, (size_t)n_tiles * sizeof(int2), s));
        NXS_CUDA(ensure_n<uint32_t>(v->pk_in, (int64_t)n_pairs));
        NXS_CUDA(ensure_n<uint32_t>(v->pk_out, (int64_t)n_pairs));
        NXS_CUDA(ensure_n<uint32_t>(v->pv_in, (int64_t)n_pairs));
        size_t tmp_pairs = 0;
        NXS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_pairs, v->pk_in.as<uint32_t>(),
                                                 v->pk_out.as<uint32_t>(), v->pv_in.as<uint32_t>(),
                                                 v->pv_ph[ph].as<uint32_t>(), (int)n_pairs, 0,
                                                 tbits, s));
        NXS_CUDA(v->temp.ensure(tmp_pairs));
        launch_emit_pairs(v->rects.as<int4>(), v->idx_out.as<uint32_t>(),
                          v->offsets.as<unsigned long long>(), r0, r1, cam.tiles_x,
                          v->active.as<uint8_t>(), v->pk_in.as<uint32_t>(), v->pv_in.as<uint32_t>(),
                          v->tq.as<double>(), cam, s);
        NXS_LAUNCHED("emit_pairs");
        if (ph == 0) mark(v, 4, s);
        size_t tb = v->temp.cap;
        NXS_CUDA(cub::DeviceRadixSort::SortPairs(v->temp.p, tb, v->pk_in.as<uint32_t>(),
                                                 v->pk_out.as<uint32_t>(), v->pv_in.as<uint32_t>(),
                                                 v->pv_ph[ph].as<uint32_t>(), (int)n_pairs, 0,
                                                 tbits, s));
        if (ph == 0) mark(v, 5, s);
        launch_tile_ranges(v->pk_out.as<uint32_t>(), (int64_t)n_pairs,
                           v->ranges_ph[ph].as<int2>(), s);
        NXS_LAUNCHED("tile_ranges");
      } else if (ph == 0) {
        mark(v, 4, s);
        mark(v, 5, s);
      }
      if (ph == 0) mark(v, 6, s);
      if (v->ev_ok) rec_event(v, v->evp[ph][3], s);
    }
    if (ph == 1 || (ph == 0 && n_ph > 1)) {
      // forward carry between phases (allocated only when a second phase exists)
      NXS_CUDA(ensure_n<float>(v->r_rad, npix * 3));
      NXS_CUDA(ensure_n<float>(v->r_trem, npix));
      NXS_CUDA(ensure_n<int32_t>(v->r_count, npix));
      NXS_CUDA(ensure_n<float>(v->r_sea, npix * 3));
      NXS_CUDA(ensure_n<float>(v->r_sa, npix));
    }
    if (torder) {
      // ---- K3x exact/chunked-order forward of this phase
      NXS_CUDA(ensure_n<int32_t>(v->seq, npix * std::max(1, opts->max_splats)));  // [slot][pixel]
      if (n_ph > 1 && ph > 0) NXS_CUDA(cudaMemsetAsync(n_active, 0, sizeof(unsigned int), s));
      // exact order over several phases: pending entries cross the phase end
      const bool xcarry = exact && n_ph > 1;
      float* ebound = nullptr;
      if (xcarry) {
        NXS_CUDA(ensure_n<float>(v->xc_t, (int64_t)32 * npix));
        NXS_CUDA(ensure_n<int32_t>(v->xc_r, (int64_t)32 * npix));
        NXS_CUDA(ensure_n<int32_t>(v->xc_n, npix));
        if (ph + 1 < n_ph) {
          ebound = reinterpret_cast<float*>(v->ph_sel.as<long long>() + 90);
          // (a device-sized phase 0 ends at the selection's bin, dsel[0])
          launch_phase_bound(dsmall + 6, ph_bin[ph], ebound, s,
                             (async0 && ph == 0) ? v->ph_sel.as<long long>() : nullptr);
          NXS_LAUNCHED("phase_bound");
        }
      }
      FwdXArgs xa{v->records.as<float4>(), v->pv_ph[ph].as<uint32_t>(),
                  v->ranges_ph[ph].as<int2>(), v->zlo_rank.as<float>(), v->idx_out.as<uint32_t>(),
                  chunked ? v->rank_c.as<uint32_t>() : nullptr, chunked ? opts->chunk_size : 0,
                  opts->max_splats, (float)opts->alpha_cutoff, opts->near_plane,
                  {bgf[0], bgf[1], bgf[2]}, rgb, overdraw, residual, v->seq.as<int32_t>(),
                  dsmall + 9, n_ph > 1 ? v->active.as<uint8_t>() : nullptr,
                  n_ph > 1 ? n_active : nullptr, ph > 0, ph + 1 < n_ph,
                  (chunked && !(opts->flags & NXS_FLAG_XBUF32)) ? 16 : 32,
                  xcarry ? v->xc_t.as<float>() : nullptr,
                  xcarry ? v->xc_r.as<int32_t>() : nullptr,
                  xcarry ? v->xc_n.as<int32_t>() : nullptr, ebound,
                  v->lazy ? dsmall + 12 : nullptr};
      launch_blend_fwd_x(count, n_tiles, xa, cam, md, v->cache(), v->resume(), cnt, s);
      NXS_LAUNCHED("blend_fwd_x");
      if (v->ev_ok) rec_event(v, v->evp[ph][4], s);
      ph_done = ph + 1;
      if (cap.on && ph == 0) {
        const int erc = end_capture();
        if (erc) return erc;
      }
      continue;
    }
    // ---- K3 forward blend of this phase (tiles still active; phase 0's
    // count was cleared by k_call_init)
    if (ph > 0) NXS_CUDA(cudaMemsetAsync(n_active, 0, sizeof(unsigned int), s));
    FwdArgs fa{v->records.as<float4>(), v->pv_ph[ph].as<uint32_t>(), v->ranges_ph[ph].as<int2>(),
               v->cum_ph[ph].as<int32_t>(), v->cum_ph[ph + 1].as<int32_t>(),
               v->active.as<uint8_t>(), n_active, ph > 0, ph + 1 < n_ph, opts->max_splats,
               (float)opts->alpha_cutoff, opts->near_plane, {bgf[0], bgf[1], bgf[2]},
               rgb, overdraw, residual, v->lazy ? dsmall + 12 : nullptr,
               (opts->flags & NXS_FLAG_THETA0) != 0, v->tile_last.as<int32_t>()};
    launch_blend_fwd(count, n_tiles, fa, cam, md, v->cache(), v->resume(), cnt, s);
    g_ht.mark("fwd_enq");
    NXS_LAUNCHED("blend_fwd");
    if (v->ev_ok) rec_event(v, v->evp[ph][4], s);
    ph_done = ph + 1;
    if (cap.on && ph == 0) {
      const int erc = end_capture();
      if (erc) return erc;
    }
  }
  mark(v, 7, s);
  if (v->lazy) {  // the next call's first-phase hint (read without a sync)
    cudaStream_t cs;
    NXS_CUDA(side_after(v, s, cs));
    if (v->async_bases) {
      // the next call's per-tile capacities follow this pass's counts (a
      // moving scene drifts from the exact pass's); one block on the side
      // stream, off the pipeline — the next call waits for it (ev_bases)
      launch_refresh_bases(v->ranges_ph[0].as<int2>(), n_tiles, v->tile_base.as<uint32_t>(),
                           (unsigned long long)v->bases_bound,
                           (unsigned int)std::min<int64_t>(v->bases_maxcap, 0xffffffffll), cs);
      NXS_LAUNCHED("refresh_bases");
      if (!v->ev_bases) NXS_CUDA(cudaEventCreateWithFlags(&v->ev_bases, cudaEventDisableTiming));
      NXS_CUDA(cudaEventRecord(v->ev_bases, cs));
      v->bases_pending = true;
    }
    NXS_CUDA(cudaMemcpyAsync(v->host_small + 30, dsmall + 12, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, cs));
    if (!v->ev_hint) NXS_CUDA(cudaEventCreateWithFlags(&v->ev_hint, cudaEventDisableTiming));
    NXS_CUDA(cudaEventRecord(v->ev_hint, cs));
    v->hint_pending = true;
  }
  v->ev_fwd = true;
  v->ev_bwd = false;
  v->stats.n_pairs = total_pairs;
  v->ovf_pending = false;
  if (torder && v->defer_ovf) {
    // (nxs_forward_backward enqueues the backward first and checks this
    // behind it: finish_ovf_check)
    cudaStream_t cs;
    NXS_CUDA(side_after(v, s, cs));
    NXS_CUDA(cudaMemcpyAsync(v->host_small + 28, dsmall + 9, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, cs));
    if (!v->ev_ovf) NXS_CUDA(cudaEventCreateWithFlags(&v->ev_ovf, cudaEventDisableTiming));
    NXS_CUDA(cudaEventRecord(v->ev_ovf, cs));
    v->ovf_pending = true;
  } else if (torder) {
    // pending-buffer overflow means the exact order was not guaranteed: report
    NXS_CUDA(cudaMemcpyAsync(v->host_small + 7, dsmall + 9, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    NXS_CUDA(spin_sync(v, s));
    v->stats.n_overflow = (int64_t)v->host_small[7];
    if (v->host_small[7] > 0 && chunked && !(opts->flags & NXS_FLAG_XBUF32)) {
      // the small pending buffer overflowed: redo the pass with the large one
      ++v->stats.n_redo;
      nxs_opts o2 = *opts;
      o2.flags |= NXS_FLAG_XBUF32;
      return nxs_forward(v, scene, camera, model, &o2, background, rgb, overdraw, residual,
                         stream_);
    }
    if (v->host_small[7] > 0)
      return fail(NXS_ERR_OVERFLOW, std::to_string(v->host_small[7]) +
                                        " pixel-entries overflowed the exact-order pending "
                                        "buffer; the per-pixel order is not guaranteed");
  }
  if (count) {
    NXS_CUDA(cudaMemcpyAsync(v->host_small + 4, cnt, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    NXS_CUDA(spin_sync(v, s));
    v->stats.n_tests_fwd = (int64_t)v->host_small[4];
    v->stats.n_composited = (int64_t)v->host_small[5];
  }

  v->have_fwd = true;
  v->tlist_valid = false;
  v->cam = cam;
  v->model = md;
  v->opts = *opts;
  for (int i = 0; i < 3; ++i) v->bg[i] = bgf[i];
  v->P = P;
  v->C = C;
  v->n_pairs = total_pairs;
  v->n_phases = ph_done;
  v->n_tiles = n_tiles;
  v->scene_centers = scene->centers;
  if (!v->spec_pending) v->phases_needed = ph_done;
  if (v->lazy && !async0 && ph_done >= 1) {  // exact phase 0: sizes for the next call
    v->est_n0 = R[1];
    v->est_pairs = v->ph_pairs[0];
    v->est_bin0 = ph_bin[0];
  }
  return NXS_OK;
}

// backward blend (K4/K4x) into the per-rank moments; the chain follows
int backward_blend(nxs_view* v, const float* seed, cudaStream_t s) {
  const int64_t P = v->P;
  mark(v, 8, s);
  {
    // moments/touched stay zero between backwards (K5 re-zeroes what it
    // reads); clear only freshly allocated buffers
    void* mp = v->moments.p;
    void* tp = v->touched.p;
    NXS_CUDA(ensure_n<double>(v->moments, P * NMOM));
    NXS_CUDA(ensure_n<uint8_t>(v->touched, P));
    if (v->moments.p != mp)
      NXS_CUDA(cudaMemsetAsync(v->moments.p, 0, v->moments.cap, s));
    if (v->touched.p != tp) NXS_CUDA(cudaMemsetAsync(v->touched.p, 0, v->touched.cap, s));
  }
  mark(v, 9, s);
  const bool count = (v->opts.flags & NXS_FLAG_COUNT_EVENTS) != 0;
  unsigned long long* dsmall = v->dev_small.as<unsigned long long>();
  Counters* cnt = reinterpret_cast<Counters*>(dsmall + 1);
  const bool det = (v->opts.flags & NXS_FLAG_DETERMINISTIC) != 0;
  if (det && v->opts.chunk_size != 1)
    return fail(NXS_ERR_UNSUPPORTED,
                "deterministic gradients: global depth order (chunk_size=1) only");
  if (v->opts.chunk_size != 1) {
    BwdXArgs xa{v->records.as<float4>(), v->bframe.as<float4>(), v->pv_ph[0].as<uint32_t>(),
                v->seq.as<int32_t>(), std::max(1, v->opts.max_splats),
                (float)v->opts.alpha_cutoff, v->opts.near_plane, {v->bg[0], v->bg[1], v->bg[2]},
                seed, v->moments.as<double>(), v->touched.as<uint8_t>(),
                !(v->opts.chunk_size > 1 && v->opts.chunk_size < v->P)};
    launch_blend_bwd_x(count, v->n_tiles, xa, v->cam, v->model, v->cache(), cnt, s);
  } else {
  PhaseLists lists{};
  lists.n = v->n_phases;
  for (int p = 0; p < v->n_phases; ++p) {
    lists.pairs[p] = v->pv_ph[p].as<uint32_t>();
    lists.ranges[p] = v->ranges_ph[p].as<int2>();
    lists.cum[p] = v->cum_ph[p].as<int32_t>();
  }
  lists.partial = nullptr;
  lists.tile_last = v->tile_last.as<int32_t>();  // written by every K3 pass of the tile
  if (det) {  // partials per (tile, entry), reduced per rank in a fixed order
    int64_t off = 0;
    for (int p = 0; p < v->n_phases; ++p) {
      lists.poff[p] = off;
      off += (int64_t)(v->pv_ph[p].cap / sizeof(uint32_t));
    }
    NXS_CUDA(ensure_n<float>(v->partial, std::max<int64_t>(off, 1) * NMOM));
    lists.partial = v->partial.as<float>();
  }
  launch_blend_bwd(count, v->n_tiles, v->records.as<float4>(), v->bframe.as<float4>(), lists,
                   v->cam, v->model, (float)v->opts.alpha_cutoff, v->opts.near_plane, v->bg, seed,
                   v->cache(), v->moments.as<double>(), v->touched.as<uint8_t>(), cnt, s);
  if (det) {
    NXS_LAUNCHED("blend_bwd");
    launch_det_reduce(v->proj_end > 0 ? std::min(v->proj_end, P) : P, v->idx_out.as<uint32_t>(),
                      v->rects.as<int4>(), v->cam.tiles_x, lists, v->touched.as<uint8_t>(),
                      v->moments.as<double>(), s);
    NXS_LAUNCHED("det_reduce");
    mark(v, 10, s);
    return NXS_OK;
  }
  }
  NXS_LAUNCHED("blend_bwd");
  mark(v, 10, s);
  return NXS_OK;
}

// K5: moments -> gradients (null gradients: only clear the moments)
int backward_chain(nxs_view* v, const nxs_scene* scene, float* g_centers, float* g_scales,
                   float* g_quats, float* g_opacities, float* g_sh, cudaStream_t s) {
  // (the backward touches only processed ranks: [0, proj_end))
  if (g_centers) {
    NXS_CUDA(ensure_n<uint32_t>(v->tlist, std::max<int64_t>(v->P, 1)));
    NXS_CUDA(v->tcount.ensure(sizeof(unsigned long long)));
    NXS_CUDA(cudaMemsetAsync(v->tcount.p, 0, sizeof(unsigned long long), s));
  }
  launch_chain(scene->scales, scene->quats, v->C,
               v->proj_end > 0 ? std::min(v->proj_end, v->P) : v->P, v->idx_out.as<uint32_t>(),
               v->moments.as<double>(), v->touched.as<uint8_t>(), g_centers, g_scales, g_quats,
               g_opacities, g_sh, g_centers ? v->tlist.as<uint32_t>() : nullptr,
               g_centers ? v->tcount.as<unsigned long long>() : nullptr, s);
  NXS_LAUNCHED("chain");
  if (!g_centers) return NXS_OK;
  v->tlist_valid = true;
  mark(v, 11, s);
  v->ev_bwd = true;
  const bool count = (v->opts.flags & NXS_FLAG_COUNT_EVENTS) != 0;
  unsigned long long* dsmall = v->dev_small.as<unsigned long long>();
  Counters* cnt = reinterpret_cast<Counters*>(dsmall + 1);
  if (count) {
    NXS_CUDA(cudaMemcpyAsync(v->host_small + 5, &cnt->tests_bwd, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    NXS_CUDA(spin_sync(v, s));
    v->stats.n_tests_bwd = (int64_t)v->host_small[5];
    v->stats.n_entries_bwd = (int64_t)v->host_small[6];
  }
  return NXS_OK;
}

int check_backward_args(nxs_view* v, const nxs_scene* scene, const float* seed, float* g_centers,
                        float* g_scales, float* g_quats, float* g_opacities, float* g_sh) {
  if (!v || !scene || !seed) return fail(NXS_ERR_INVALID, "null argument");
  if (v->P > 0 && (!g_centers || !g_scales || !g_quats || !g_opacities || !g_sh))
    return fail(NXS_ERR_INVALID, "null gradient buffer");
  return NXS_OK;
}

}  // namespace

extern "C" {

int nxs_backward(nxs_view* v, const nxs_scene* scene, const float* seed, float* g_centers,
                 float* g_scales, float* g_quats, float* g_opacities, float* g_sh, void* stream_) {
  if (!v) return fail(NXS_ERR_INVALID, "null view");
  DevGuard dg(v->device);
  int rc;
  if ((rc = check_backward_args(v, scene, seed, g_centers, g_scales, g_quats, g_opacities, g_sh)))
    return rc;
  if (!v->have_fwd) return fail(NXS_ERR_STATE, "no forward pass recorded in this view");
  if (scene->count != v->P || scene->sh_coeffs != v->C)
    return fail(NXS_ERR_STATE, "scene differs from the forward call");
  if (v->spec_pending) return fail(NXS_ERR_STATE, "internal: unresolved speculative forward");
  cudaStream_t s = (cudaStream_t)stream_;
  if (v->P == 0) return NXS_OK;
  if ((rc = backward_blend(v, seed, s))) return rc;
  return backward_chain(v, scene, g_centers, g_scales, g_quats, g_opacities, g_sh, s);
}

int nxs_forward_backward(nxs_view* v, const nxs_scene* scene, const nxs_camera* camera,
                         const nxs_model* model, const nxs_opts* opts, const float background[3],
                         float* rgb, int32_t* overdraw, float* residual, const float* seed,
                         float* g_centers, float* g_scales, float* g_quats, float* g_opacities,
                         float* g_sh, void* stream_) {
  if (!v) return fail(NXS_ERR_INVALID, "null view");
  DevGuard dg(v->device);
  int rc;
  if ((rc = check_backward_args(v, scene, seed, g_centers, g_scales, g_quats, g_opacities, g_sh)))
    return rc;
  cudaStream_t s = (cudaStream_t)stream_;
  g_ht.mark("start");
  // speculate that this view needs as many depth phases as its last call
  // and, in the t-ordered modes, that no pending buffer overflowed
  const int spec = (v->ev_sync && v->phases_needed > 0) ? v->phases_needed : 0;
  v->defer_ovf = true;
  rc = forward_impl(v, scene, camera, model, opts, background, rgb, overdraw, residual, stream_,
                    spec);
  v->defer_ovf = false;
  if (rc) return rc;
  if (v->P == 0) return NXS_OK;
  const bool spec_check = v->spec_pending;
  const bool async_check = v->async_pending;
  if (spec_check) {
    // the active-tile count of the last forward kernel (and, for a
    // device-sized phase 0, its sizes), read back right behind it; the host
    // waits for the forward only, not for the backward
    if (async_check) {
      if ((rc = enqueue_async_check(v, v->n_phases_plan, s))) return rc;
    } else {
      unsigned int* n_active =
          reinterpret_cast<unsigned int*>(v->dev_small.as<unsigned long long>() + 5);
      cudaStream_t cs;
      NXS_CUDA(side_after(v, s, cs));
      NXS_CUDA(cudaMemcpyAsync(v->host_small + 3, n_active, sizeof(unsigned int),
                               cudaMemcpyDeviceToHost, cs));
      NXS_CUDA(cudaEventRecord(v->ev_sync, cs));
    }
  }
  g_ht.mark("check_enq");
  if ((rc = backward_blend(v, seed, s))) return rc;
  g_ht.mark("bwd_enq");
  if (v->ovf_pending) {
    v->ovf_pending = false;
    NXS_CUDA(cudaEventSynchronize(v->ev_ovf));
    v->stats.n_overflow = (int64_t)v->host_small[28];
    if (v->host_small[28] > 0) {
      // the order was not guaranteed: drop the moments; the chunked order
      // reruns with the large buffer, the exact order reports (as nxs_forward)
      ++v->stats.n_redo;
      if ((rc = backward_chain(v, scene, nullptr, nullptr, nullptr, nullptr, nullptr, s)))
        return rc;
      if (spec_check) {  // (the check's copies land before the rerun reuses their slots)
        bool ok_unused = true;
        if (async_check) {
          if ((rc = finish_async_check(v, ok_unused))) return rc;
        } else {
          NXS_CUDA(cudaEventSynchronize(v->ev_sync));
        }
      }
      v->spec_pending = v->async_pending = false;
      v->phases_needed = 0;
      if ((rc = nxs_forward(v, scene, camera, model, opts, background, rgb, overdraw, residual,
                            stream_)))
        return rc;
      if ((rc = backward_blend(v, seed, s))) return rc;
      return backward_chain(v, scene, g_centers, g_scales, g_quats, g_opacities, g_sh, s);
    }
  }
  if (spec_check) {
    bool ok = true;
    if (async_check) {
      if ((rc = finish_async_check(v, ok))) return rc;
    } else {
      cudaError_t e;
      while ((e = cudaEventQuery(v->ev_sync)) == cudaErrorNotReady) std::this_thread::yield();
      NXS_CUDA(e);
    }
    v->spec_pending = false;
    g_ht.mark("spin");
    if (!ok || (unsigned)v->host_small[3] != 0) {
      // more depth phases were needed: drop the moments, redo both passes
      ++v->stats.n_redo;
      if (std::getenv("NXS_DEBUG_PLAN"))
        std::fprintf(stderr, "redo: speculation ok=%d active_tiles=%u phases_needed=%d\n",
                     (int)ok, (unsigned)v->host_small[3], v->phases_needed);
      if ((rc = backward_chain(v, scene, nullptr, nullptr, nullptr, nullptr, nullptr, s)))
        return rc;
      v->phases_needed = 0;
      if ((rc = forward_impl(v, scene, camera, model, opts, background, rgb, overdraw, residual,
                             stream_, 0)))
        return rc;
      if ((rc = backward_blend(v, seed, s))) return rc;
    }
  }
  rc = backward_chain(v, scene, g_centers, g_scales, g_quats, g_opacities, g_sh, s);
  g_ht.mark("chain_enq");
  g_ht.dump();
  return rc;
}

int nxs_view_set_timing(nxs_view* v, int on) {
  if (!v) return fail(NXS_ERR_INVALID, "null view");
  v->timing = on != 0;
  return NXS_OK;
}

int nxs_view_timings(nxs_view* v, float* ms, int n) {
  if (!v || !ms) return fail(NXS_ERR_INVALID, "null argument");
  if (!v->ev_ok) return fail(NXS_ERR_CUDA, "timing events unavailable");
  if (!v->timing)
    return fail(NXS_ERR_STATE, "phase timing is off for this view (nxs_view_set_timing)");
  float t[NXS_PHASES] = {0};
  auto el = [&](cudaEvent_t a, cudaEvent_t b, float& out) -> int {
    NXS_CUDA(cudaEventSynchronize(b));
    float x = 0.f;
    NXS_CUDA(cudaEventElapsedTime(&x, a, b));
    out += x;
    return NXS_OK;
  };
  int rc;
  if (v->ev_fwd) {
    if ((rc = el(v->ev[0], v->ev[1], t[0]))) return rc;  // depth keys + sort
    if ((rc = el(v->ev[1], v->ev[2], t[1]))) return rc;  // projection
    for (int p = 0; p < v->n_phases; ++p) {
      if ((rc = el(v->evp[p][0], v->evp[p][1], t[0]))) return rc;  // lazy phase: depth sort
      if ((rc = el(v->evp[p][1], v->evp[p][2], t[1]))) return rc;  // lazy phase: projection
      if ((rc = el(v->evp[p][2], v->evp[p][3], t[2]))) return rc;  // count+scan+sync+emit+sort+ranges
      if ((rc = el(v->evp[p][3], v->evp[p][4], t[3]))) return rc;  // forward blend (+carry)
    }
    t[4] = (float)v->n_phases;
  }
  if (v->ev_fwd && (rc = el(v->ev[0], v->ev[7], t[6]))) return rc;  // whole forward
  if (v->ev_fwd && v->ev_bwd && (rc = el(v->ev[7], v->ev[8], t[5]))) return rc;  // gap
  if (v->ev_bwd) {
    if ((rc = el(v->ev[8], v->ev[9], t[7]))) return rc;
    if ((rc = el(v->ev[9], v->ev[10], t[8]))) return rc;
    if ((rc = el(v->ev[10], v->ev[11], t[9]))) return rc;
  }
  for (int i = 0; i < n && i < NXS_PHASES; ++i) ms[i] = t[i];
  return NXS_OK;
}

int nxs_cache_export(nxs_view* v, uint8_t* sat, float* e_k, float* t_k, float* theta0,
                     void* stream_) {
  if (!v) return fail(NXS_ERR_INVALID, "null view");
  DevGuard dg(v->device);
  if (!v->have_fwd) return fail(NXS_ERR_STATE, "no forward pass recorded in this view");
  cudaStream_t s = (cudaStream_t)stream_;
  const size_t npix = (size_t)v->cam.W * v->cam.H;
  if (sat) NXS_CUDA(cudaMemcpyAsync(sat, v->c_sat.p, npix, cudaMemcpyDeviceToDevice, s));
  if (e_k) NXS_CUDA(cudaMemcpyAsync(e_k, v->c_ek.p, npix * 12, cudaMemcpyDeviceToDevice, s));
  if (t_k) NXS_CUDA(cudaMemcpyAsync(t_k, v->c_tk.p, npix * 4, cudaMemcpyDeviceToDevice, s));
  if (theta0) {
    if (v->opts.chunk_size == 1 && !(v->opts.flags & NXS_FLAG_THETA0))
      return fail(NXS_ERR_STATE, "theta0 was not accumulated: forward without NXS_FLAG_THETA0");
    NXS_CUDA(cudaMemcpyAsync(theta0, v->c_th0.p, npix * 12, cudaMemcpyDeviceToDevice, s));
  }
  return NXS_OK;
}

int nxs_depth_order(nxs_view* v, int32_t* order, void* stream_) {
  if (!v || !order) return fail(NXS_ERR_INVALID, "null argument");
  DevGuard dg(v->device);
  if (!v->have_fwd) return fail(NXS_ERR_STATE, "no forward pass recorded in this view");
  if (v->P == 0) return NXS_OK;
  int rc;
  if ((rc = complete_order(v, (cudaStream_t)stream_)) != NXS_OK) return rc;
  NXS_CUDA(cudaMemcpyAsync(order, v->idx_out.p, (size_t)v->P * 4, cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream_));
  return NXS_OK;
}

int nxs_binning_export(nxs_view* v, int32_t* rects, int32_t* ranges, int32_t* pair_ranks,
                       void* stream_) {
  if (!v) return fail(NXS_ERR_INVALID, "null view");
  DevGuard dg(v->device);
  if (!v->have_fwd) return fail(NXS_ERR_STATE, "no forward pass recorded in this view");
  cudaStream_t s = (cudaStream_t)stream_;
  int rc;
  if (v->P && (rc = complete_order(v, s)) != NXS_OK) return rc;
  if (rects && v->P)
    NXS_CUDA(cudaMemcpyAsync(rects, v->rects.p, (size_t)v->P * 16, cudaMemcpyDeviceToDevice, s));
  if (v->n_phases < 1 || (!ranges && !pair_ranks)) return NXS_OK;
  // The first phase's lists may sit at per-tile capacities (device-sized
  // pass) with gaps between them: export them compacted, tile after tile,
  // with the ranges rewritten to the compact offsets.  (Synchronises s.)
  const int T = v->n_tiles;
  std::vector<int2> hr(T);
  NXS_CUDA(cudaMemcpyAsync(hr.data(), v->ranges_ph[0].p, (size_t)T * sizeof(int2),
                           cudaMemcpyDeviceToHost, s));
  NXS_CUDA(cudaStreamSynchronize(s));
  std::vector<int> off(T);
  long long tot = 0;
  for (int t = 0; t < T; ++t) {
    off[t] = (int)tot;
    tot += std::max(0, hr[t].y - hr[t].x);
  }
  if (tot != v->ph_pairs[0])
    return fail(NXS_ERR_STATE, "tile lists do not add up to the phase's pair count");
  int* d_off = nullptr;
  NXS_CUDA(cudaMallocAsync((void**)&d_off, (size_t)std::max(T, 1) * sizeof(int), s));
  cudaError_t e = cudaMemcpyAsync(d_off, off.data(), (size_t)T * sizeof(int),
                                  cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    launch_compact_lists(v->pv_ph[0].as<uint32_t>(), v->ranges_ph[0].as<int2>(), d_off, T,
                         reinterpret_cast<uint32_t*>(pair_ranks), reinterpret_cast<int2*>(ranges),
                         s);
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_off, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // (off[] is host memory)
  if (e != cudaSuccess) return fail(NXS_ERR_CUDA, std::string("binning export: ") +
                                                      cudaGetErrorString(e));
  return NXS_OK;
}

int nxs_touched_export(nxs_view* v, int32_t* gids, int64_t* count, void* stream_) {
  if (!v || !count) return fail(NXS_ERR_INVALID, "null argument");
  DevGuard dg(v->device);
  if (!v->tlist_valid) return fail(NXS_ERR_STATE, "no backward recorded in this view");
  cudaStream_t s = (cudaStream_t)stream_;
  unsigned long long n = 0;
  NXS_CUDA(cudaMemcpyAsync(&n, v->tcount.p, sizeof(n), cudaMemcpyDeviceToHost, s));
  NXS_CUDA(cudaStreamSynchronize(s));
  *count = (int64_t)n;
  if (gids && n)
    NXS_CUDA(cudaMemcpyAsync(gids, v->tlist.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  return NXS_OK;
}

// sizing history of a view (the device-sized first phase's estimates), so a
// caller cycling many cameras through a few workspaces keeps each camera's
// sync-free device-sized first phase (nxs_view_history_save / _load)
struct ViewHistory {
  uint32_t magic;
  int32_t est_bin0, phases_needed, valid;
  int64_t est_n0, est_pairs;
  unsigned long long hint;
  CamDev cam;
};
constexpr uint32_t HIST_MAGIC = 0x4e585348u;

int64_t nxs_view_history_bytes(void) { return (int64_t)sizeof(ViewHistory); }

int nxs_view_history_save(nxs_view* v, void* blob) {
  if (!v || !blob) return fail(NXS_ERR_INVALID, "null argument");
  DevGuard dg(v->device);
  if (v->hint_pending && v->ev_hint) {  // the hint lands behind the last forward
    NXS_CUDA(cudaEventSynchronize(v->ev_hint));
    v->hint = v->host_small[30];
    v->hint_pending = false;
  }
  ViewHistory h{};
  h.magic = HIST_MAGIC;
  h.valid = v->have_fwd ? 1 : 0;
  h.est_n0 = v->est_n0;
  h.est_pairs = v->est_pairs;
  h.est_bin0 = v->est_bin0;
  h.phases_needed = v->phases_needed;
  h.hint = v->hint;
  h.cam = v->cam;
  std::memcpy(blob, &h, sizeof(h));
  return NXS_OK;
}

int nxs_view_history_load(nxs_view* v, const void* blob) {
  if (!v || !blob) return fail(NXS_ERR_INVALID, "null argument");
  ViewHistory h;
  std::memcpy(&h, blob, sizeof(h));
  if (h.magic != HIST_MAGIC) return fail(NXS_ERR_INVALID, "not a view history blob");
  DevGuard dg(v->device);
  if (v->hint_pending && v->ev_hint) NXS_CUDA(cudaEventSynchronize(v->ev_hint));
  v->hint_pending = false;
  // the workspace now serves another camera: its last forward is gone
  v->have_fwd = false;
  v->tlist_valid = false;
  if (!h.valid) {
    v->est_n0 = 0;
    v->hint = 0;
    v->phases_needed = 0;
    v->cam = CamDev{};
    return NXS_OK;
  }
  v->est_n0 = h.est_n0;
  v->est_pairs = h.est_pairs;
  v->est_bin0 = h.est_bin0;
  v->phases_needed = h.phases_needed;
  v->hint = h.hint;
  v->cam = h.cam;
  return NXS_OK;
}

int nxs_touched_mark(nxs_view* v, uint8_t* mask, void* stream_) {
  if (!v || !mask) return fail(NXS_ERR_INVALID, "null argument");
  if (!v->tlist_valid) return fail(NXS_ERR_STATE, "no backward recorded in this view");
  DevGuard dg(v->device);
  launch_touched_mark(v->tlist.as<uint32_t>(), v->tcount.as<unsigned long long>(), v->P, mask,
                      (cudaStream_t)stream_);
  NXS_LAUNCHED("touched_mark");
  return NXS_OK;
}

int nxs_records_export(nxs_view* v, float* records, void* stream_) {
  if (!v || !records) return fail(NXS_ERR_INVALID, "null argument");
  DevGuard dg(v->device);
  if (!v->have_fwd) return fail(NXS_ERR_STATE, "no forward pass recorded in this view");
  if (v->P == 0) return NXS_OK;
  NXS_CUDA(cudaMemcpyAsync(records, v->records.p, (size_t)v->P * REC_F4 * 16,
                           cudaMemcpyDeviceToDevice, (cudaStream_t)stream_));
  return NXS_OK;
}

}  // extern "C"
