// Internal device-side definitions shared by the kernels of libnxs.
//
// Layout in HBM (per view):
//   order    [P]      u32   rank -> Gaussian index (stable fp64 depth sort)
//   records  [P][8]   float4 per-rank projected record, 128 B, rank order
//   rects    [P]      int4  tile rectangle per rank (tx0,ty0,tx1,ty1)
//   pairs    [p][n]   u32   per depth phase p: ranks grouped by tile (stable,
//                          so rank-ascending); tiles still active only
//   ranges   [p][T]   int2  [start, end) of each tile's run in pairs[p]
//   cum      [p][T]   i32   virtual list index where tile's phase-p run starts
//   cache    [H*W]    per-pixel replay state (SoA, see PixCache)
//   moments  [P][24]  f64   per-rank gradient moments (backward)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <utility>

// NXS_CHECK(cond): device bounds checks of the blend kernels' shared-memory
// rings, staged batches, commit sequences and list indices, compiled in by
// the `checks` variant (python -m paper_2603_02887_b200.build --variant=checks
// -DNXS_CHECKS); the GPU tests run against it (tools/checks_gpu.sh), in
// place of compute-sanitizer, which this GPU pool does not allow.
#ifdef NXS_CHECKS
#include <cassert>
#define NXS_CHECK(cond) assert(cond)
#else
#define NXS_CHECK(cond) ((void)0)
#endif

namespace nxs {

// Programmatic dependent launch (Hopper+/Blackwell): every library kernel
// starts with nxs_pdl_enter() — it lets the next kernel of the stream begin
// launching once all of this grid's blocks are running, then waits for the
// previous kernel's completion (and memory) before touching anything — and
// is launched by nxs_launch with the programmatic-serialization attribute,
// so the launch latency and ramp of consecutive pipeline kernels overlap the
// previous kernel's tail.  Opt-in (NXS_PDL=1): measured at C3 it made the
// global-order step slower (0.530 -> 0.596 ms; the exact order 1 % faster),
// so plain launches are the default (griddepcontrol.wait is then a no-op).
__device__ __forceinline__ void nxs_pdl_enter() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

inline bool nxs_pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NXS_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void nxs_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  if (nxs_pdl_enabled()) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  } else {
    kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
  }
}

// Host: run `f` once per (call site, CUDA device) — kernel attributes and
// constant-memory uploads are per-device state.  `done` is the call site's
// bit set of devices (device ids >= 64 share bit 63 and re-run every time).
template <class F>
inline void once_per_device(unsigned long long& done, F&& f) {
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev < 63 ? dev : 63);
  std::lock_guard<std::mutex> lock(mu);
  if ((done & bit) && dev < 63) return;
  f();
  done |= bit;
}

constexpr int TILE = 16;
constexpr int TILE_PIX = TILE * TILE;  // 256 threads per tile block
constexpr int SEG_MAX = 4096;  // longest tile list the per-tile sort handles (else radix sort)
constexpr int REC_F4 = 8;              // float4 per record
constexpr int NMOM = 24;               // gradient moments per Gaussian

// reference compositor.py:30-31 (ALPHA_MAX = 1 - 1e-6), rounded to fp32
constexpr float ALPHA_MAX_F = 0.999999f;
// reference primitives.py:41-42
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
// P-family checkpoint: below this the transparency product is frozen for
// the backward's recovery (see blend kernels)
constexpr float P_FLOOR = 1e-30f;

// record flags (stored as int bits in rec[3].w)
constexpr int RF_CONIC = 1;    // centred-conic fp32 evaluation
constexpr int RF_GENERAL = 2;  // crosses the near region: fp64 reference diff-form
constexpr int RF_ANISO = 4;    // conic record of a Gaussian with max/min scale > 4: the
                               // backward uses the cancellation-free peak offset
// General-path record: fp64 world-frame b = μ - o and A = R diag(s⁻²) Rᵀ
// (upper triangle) packed as doubles 0..6 = b0 b1 b2 A00 A01 A02 A11 (float
// words 0..13) and doubles 14..15 = A12 A22 (float words 28..31); words 14
// (opacity), 15 (flags) and 16..27 (SH) keep their conic-record meaning.

struct CamDev {
  double o[3];
  double R[9];  // row-major, camera -> world
  double f, cx, cy;
  int W, H;
  int tiles_x, tiles_y;
  double inv_f;  // 1/f (IEEE, host): per-pixel setup without a double division
  float Rf[9];   // R rounded to fp32 (the SH basis direction)
};

// model families
enum Fam : int {
  FAM_EXP = 0,
  FAM_LIN = 1,
  FAM_QUAD = 2,
  FAM_BLEND = 3,  // blended and vicini (identical discrete weights)
  FAM_POW = 5,
  FAM_SOFT = 6,
};

struct ModelDev {
  int fam;
  float c;       // quad: c; blend: gamma; soft: kappa; pow: v
  float K;       // soft: kappa / log(1 + e^kappa)
  float ex;      // pow: -(1+v)/v
  int powmode;   // pow: 0 general, 1 linear (v == -1), 2 exponential limit
};

struct PixCache {
  int32_t* last;     // list position of the last live splat (-1: none)
  uint8_t* sat;      // saturated
  float* t_k;        // saturating weight, or residual
  float* tau_hi;     // exact double-float optical depth after the last go splat
  float* tau_lo;
  float* P_end;      // transparency product after the last go splat
  int32_t* ck_idx;   // list position where P fell below P_FLOOR (-1: never)
  float* P_ck;       // P before that splat
  float* e_k;        // [3] saturating emission (or background)
  float* theta0;     // [3] reference quadratic-adjoint cache (compat)
};

// Progressive binning: ranks are binned in depth phases [R_p, R_{p+1});
// phase p only emits pairs for tiles with a pixel still neither saturated
// nor capped, and the forward resumes its per-pixel carry across phases.
constexpr int MAX_PHASES = 4;

struct PixResume {  // forward carry kept between phases (besides PixCache)
  float* rad;       // [3]
  float* trem;
  int32_t* count;
  float* sea;       // [3]
  float* sa;
};

struct PhaseLists {  // the per-tile virtual list = phase segments in order
  const uint32_t* pairs[MAX_PHASES];  // sorted ranks of phase p
  const int2* ranges[MAX_PHASES];     // per tile [start, end) in pairs[p]
  const int32_t* cum[MAX_PHASES];     // per tile virtual index of the segment start
  int n;
  // deterministic gradients (NXS_FLAG_DETERMINISTIC): per (tile, entry)
  // moment partials at partial[(poff[p] + index in pairs[p]) * NMOM + m]
  float* partial;
  int64_t poff[MAX_PHASES];
  // per tile: the largest virtual position any pixel replays (K3 writes it)
  const int32_t* tile_last;
};

// arguments of one forward phase launch
struct FwdArgs {
  const float4* records;
  const uint32_t* pairs;
  const int2* ranges;
  const int32_t* cum_in;
  int32_t* cum_out;
  uint8_t* active;
  unsigned int* n_active;
  bool resume;  // load the carry of the previous phase
  bool save;    // another phase follows: keep the carry of unfinished tiles
  int max_splats;
  float cutoff;
  double near_plane;
  float bg[3];
  float* rgb;
  int32_t* overdraw;
  float* residual;
  // max over the tiles finishing in this pass of the last rank their list
  // needed (the view's first-phase hint for its next call), or null
  unsigned long long* need_rank;
  bool theta0;  // accumulate the reference cache's theta0 (NXS_FLAG_THETA0)
  int32_t* tile_last;  // per tile: max of its pixels' last (read by K4)
};

// exact-order mode (K3x/K4x)
struct FwdXArgs {
  const float4* records;
  const uint32_t* pairs;
  const int2* ranges;
  const float* zlo_rank;
  const uint32_t* order;
  const uint32_t* rank_c;  // chunked order: centre-depth rank per Gaussian, else null
  int chunk;               // chunked order: chunk size C, else 0 (one chunk)
  int max_splats;
  float cutoff;
  double near_plane;
  float bg[3];
  float* rgb;
  int32_t* overdraw;
  float* residual;
  int32_t* seq;                // commit sequence [slot][pixel]: ranks
  unsigned long long* overflow;
  // depth phases (chunked order; phases end on chunk boundaries, where no
  // entry is pending, so the carry is the global-order one)
  uint8_t* active;
  unsigned int* n_active;
  bool resume, save;
  int xbuf;  // pending entries per pixel (16 or 32)
  // exact order over depth phases: the pending entries of unfinished pixels
  // cross the phase end ([slot][pixel] t and rank, per-pixel count), and
  // *end_bound is a lower bound of every later phase's z_lo (null: commit all)
  float* carry_t;
  int32_t* carry_r;
  int32_t* carry_n;
  const float* end_bound;
  unsigned long long* need_rank;  // as FwdArgs::need_rank
};
struct BwdXArgs {
  const float4* records;
  const float4* bframe;
  const uint32_t* pairs;
  const int32_t* seq;
  int max_splats;
  float cutoff;
  double near_plane;
  float bg[3];
  const float* seed;
  double* moments;
  uint8_t* touched;
  bool exact;  // exact order (one chunk): one pixel per thread, else two
};

struct Counters {
  unsigned long long tests_fwd, composited, tests_bwd, entries_bwd;
};

// ---------------------------------------------------------------------------
// error-free float transforms (exact double-float optical depth)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void two_sum(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  float bb = __fsub_rn(s, a);
  e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
}
__device__ __forceinline__ void fast_two_sum(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  e = __fsub_rn(b, __fsub_rn(s, a));
}
// (hi, lo) += a, exactly (the partial sums of alphas >= 2^-8 need < 48 bits)
__device__ __forceinline__ void df_add(float& hi, float& lo, float a) {
  float s, e;
  two_sum(hi, a, s, e);
  fast_two_sum(s, __fadd_rn(e, lo), hi, lo);
}

// Ampere+ asynchronous global->shared copies (LDGSTS), 16 B each
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// a / b within ~1 ulp: approximate reciprocal plus one Newton step on the
// quotient (no IEEE-division slow path); b in normal range
__device__ __forceinline__ float div_newton(float a, float b) {
  const float r = rcp_approx(b);
  const float q = a * r;
  return fmaf(fmaf(-q, b, a), r, q);
}

// ---------------------------------------------------------------------------
// transmittance weights p̄ = α·g  (reference transmittance.py:234-262)
// τ-family: g = f(τ̄), fp = f'(τ̄).  P-family: g = (1-γ) + γP.
// ---------------------------------------------------------------------------
template <int FAM>
__device__ __forceinline__ float weight_g(const ModelDev& m, float thi, float tlo, float P,
                                          float& fp) {
  if constexpr (FAM == FAM_EXP) {
    fp = 0.f;
    return P;
  } else if constexpr (FAM == FAM_BLEND) {
    fp = 0.f;
    return fmaf(m.c, P - 1.0f, 1.0f);
  } else if constexpr (FAM == FAM_LIN) {
    fp = 0.f;
    return 1.0f;
  } else if constexpr (FAM == FAM_QUAD) {
    fp = m.c;
    return fmaf(m.c, thi, fmaf(m.c, tlo, 1.0f));
  } else if constexpr (FAM == FAM_SOFT) {
    // σ(x), x = κ(1 - τ̄), split by sign so neither exp overflows
    float x = m.c * __fsub_rn(__fsub_rn(1.0f, thi), tlo);
    float t = ex2_approx(-fabsf(x) * 1.4426950408889634f);  // e^{-|x|}
    float r = __fdividef(1.0f, 1.0f + t);
    float sig = x >= 0.f ? r : t * r;
    float oms = x >= 0.f ? t * r : r;  // 1 - σ
    float g = m.K * sig;
    fp = -m.c * g * oms;
    return g;
  } else {  // FAM_POW
    if (m.powmode == 1) {
      fp = 0.f;
      return 1.0f;
    }
    float tau = thi + tlo;
    if (m.powmode == 2) {
      float e = ex2_approx(-tau * 1.4426950408889634f);
      fp = -e;
      return e;
    }
    float base = fmaf(tau, m.c, 1.0f);
    if (!(base > 0.f)) {
      fp = 0.f;
      return 0.f;
    }
    float g = ex2_approx(m.ex * lg2_approx(base));
    fp = m.ex * m.c * __fdividef(g, base);
    return g;
  }
}

template <int FAM>
struct IsPFam {
  static constexpr bool value = (FAM == FAM_EXP || FAM == FAM_BLEND);
};

}  // namespace nxs
