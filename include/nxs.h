/*
 * nxs.h — C-ABI of the B200 generalized-transmittance splat renderer.
 *
 * Drop-in boundary for the reference's image renderer (reference
 * pkg/src/nexsplat/render.py, module `nexsplat.render`, __all__ at
 * render.py:34-41).  The reference is pure Python/numpy and has no FFI of
 * its own; these entry points are what its Python API binds to (the
 * ctypes binding is paper_2603_02887_b200/_native.py; INTEGRATION.md shows
 * the stub a nexsplat maintainer would add).  Plain C types only: no torch,
 * no CUDA types in the signatures (streams are passed as void*).
 *
 * Entry point  ->  reference interface it replaces
 *   nxs_forward        render_forward_cached / render      (render.py:361-425;
 *                      core _forward_sweep, render.py:147-217)
 *   nxs_backward       render_backward                      (render.py:428-442;
 *                      core _backward_sweep, render.py:220-347)
 *   nxs_cache_export   the cache dict of render_forward_cached
 *                      (render.py:214-217: sat, e_k, t_k, theta0)
 *   nxs_depth_order    _depth_chunks ordering               (render.py:350-358)
 *
 * Conventions
 *   - Status: 0 on success, negative NXS_ERR_* on failure; no exceptions
 *     cross the ABI.  nxs_error_string() / nxs_last_error() describe it.
 *   - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors) unless stated; the caller owns them.  Work is enqueued on
 *     `stream` (a cudaStream_t, NULL = legacy default stream).
 *   - Host waits: a view's first call (and any call whose sizes outgrow the
 *     previous one) reads phase and pair counts from the device between
 *     kernels; from the second call on, the first depth phase is sized from
 *     the view's history and runs without a host sync (its check is read
 *     behind the forward).  nxs_forward_backward returns once that check
 *     has been read; the waits poll an event (yielding the host thread).
 *   - A view (nxs_view) owns the per-view device workspace (projected
 *     records, tile lists, the per-pixel replay cache), allocated by the
 *     library with cudaMalloc on the device that was current at
 *     nxs_view_create; every call on the view makes that device current and
 *     restores the caller's.  It persists from nxs_forward to nxs_backward
 *     of the same view ("settings must match the forward call",
 *     render.py:435-436).  Distinct views are independent and may be used
 *     concurrently on distinct streams; nxs_view_destroy waits for the
 *     view's device to drain.
 *   - Gradients ACCUMULATE (+=, atomically) into the caller's buffers, so a
 *     rank's views sum into one buffer before the data-parallel all-reduce;
 *     views sharing a buffer may run concurrently on distinct streams (the
 *     float summation order then varies run to run).
 */
#ifndef NXS_H
#define NXS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NXS_ABI_VERSION 2

/* status codes */
#define NXS_OK 0
#define NXS_ERR_INVALID (-1)       /* bad argument (shape, pointer, option) */
#define NXS_ERR_UNSUPPORTED (-2)   /* mode/model combination not implemented */
#define NXS_ERR_CUDA (-3)          /* a CUDA call failed */
#define NXS_ERR_NOMEM (-4)         /* device allocation failed */
#define NXS_ERR_STATE (-5)         /* backward without a matching forward */
#define NXS_ERR_GEOMETRY (-6)      /* reserved: unsupported geometry */
#define NXS_ERR_OVERFLOW (-7)      /* exact order: a pixel's pending buffer overflowed */

/* transmittance variants: order of reference transmittance.py:32-40 */
#define NXS_MODEL_EXPONENTIAL 0
#define NXS_MODEL_LINEAR 1
#define NXS_MODEL_QUADRATIC 2
#define NXS_MODEL_BLENDED 3
#define NXS_MODEL_VICINI 4
#define NXS_MODEL_POWER_LAW 5
#define NXS_MODEL_SOFTPLUS 6

/* opts.flags */
#define NXS_FLAG_COUNT_EVENTS 1    /* count tests/composites (instrumented run) */
#define NXS_FLAG_FULL_BINNING 2    /* bin every rank in one phase (no progressive binning) */
#define NXS_FLAG_XBUF32 4          /* chunked order: start with the 32-entry pending buffer
                                      (default 16, rerun with 32 on overflow) */
#define NXS_FLAG_DETERMINISTIC 16  /* bit-reproducible gradients (SPEC "deterministic
                                      partitioned reduction"): per (tile, list entry)
                                      moment partials, summed per Gaussian in a fixed
                                      tile order instead of atomics; global depth order
                                      (chunk_size=1) only, else NXS_ERR_UNSUPPORTED at
                                      the backward.  Costs shared memory (occupancy). */
#define NXS_FLAG_THETA0 8          /* also accumulate the reference cache's theta0
                                      (render.py:213; only nxs_cache_export reads it, the
                                      backward does not: off by default on the global order) */

/* ordering: opts.chunk_size (reference render(..., chunk_size=), render.py:350-358)
 *   NXS_CHUNK_EXACT (None) or C >= count: one chunk, exact per-pixel t order
 *   1: global centre-depth order
 *   1 < C < count: chunks of C in centre-depth order, per-pixel t order within */
#define NXS_CHUNK_EXACT 0

/* TransmittanceModel (reference transmittance.py:54-79): variant + param */
typedef struct {
    int32_t variant;
    double param;
} nxs_model;

/* Camera (reference primitives.py:153-190): rotation maps camera axes
 * (right, down, forward) to world, row-major 3x3; pixel (row i, col j)
 * looks along rotation * ((j+0.5-cx)/focal, (i+0.5-cy)/focal, 1). */
typedef struct {
    double position[3];
    double rotation[9];
    double focal, cx, cy;
    int32_t width, height;
} nxs_camera;

/* render keyword arguments (reference render.py:361-364) */
typedef struct {
    int32_t max_splats;      /* default 128 */
    double alpha_cutoff;     /* default 1/255 */
    double near_plane;       /* default 1e-4 */
    int32_t chunk_size;      /* NXS_CHUNK_EXACT (None) or >= 1, see above */
    int32_t flags;           /* NXS_FLAG_* */
    int64_t first_phase_ranks; /* progressive binning: ranks in the first depth
                                  phase (0 = automatic); later phases grow x8 */
} nxs_opts;

/* SceneArrays (reference render.py:44-52), device float32, row-major:
 * centers (P,3), scales (P,3), quats (P,4) (w,x,y,z; normalised on use),
 * opacities (P), sh (P,3,C) with C in {1,4}. */
typedef struct {
    const float* centers;
    const float* scales;
    const float* quats;
    const float* opacities;
    const float* sh;
    int64_t count;
    int32_t sh_coeffs;
} nxs_scene;

/* per-view statistics of the last forward/backward */
typedef struct {
    int64_t n_gaussians;
    int64_t n_visible;        /* Gaussians with >= 1 tile */
    int64_t n_pairs;          /* (tile, Gaussian) pairs sorted */
    int64_t n_straddling;     /* Gaussians crossing the near plane */
    int64_t n_tiles;
    int64_t n_tests_fwd;      /* (pixel, list entry) pairs tested   [COUNT_EVENTS] */
    int64_t n_composited;     /* sum of overdraw                     [COUNT_EVENTS] */
    int64_t n_tests_bwd;      /* pairs re-tested by the backward     [COUNT_EVENTS] */
    int64_t n_entries_bwd;    /* (tile, entry) pairs replayed        [COUNT_EVENTS] */
    int64_t n_overflow;       /* exact order: pending-buffer overflows (must be 0) */
    int64_t n_launches;       /* kernels this view has launched so far (cumulative;
                                 the ones replayed from its CUDA graph included) */
    int64_t n_redo;           /* passes redone so far (cumulative): a device-sized
                                 first phase whose capacities were exceeded, a fused
                                 call that needed more depth phases than speculated,
                                 a chunked pass whose 16-entry buffer overflowed */
} nxs_stats;

typedef struct nxs_view nxs_view;

/* device-timed phases of the last forward + backward (CUDA events on the
 * call's stream), order of nxs_view_timings' output */
#define NXS_PHASES 10
/* 0 depth sort (K0 + radix sort), 1 projection (K1), 2 tile binning over
 * all depth phases (active-tile counts, scan + host sync, pair emission,
 * sort by tile, ranges), 3 forward blend over all phases (K3), 4 number of
 * depth phases run (a count, not ms), 5 device idle time between the end of
 * the forward and the start of the backward (host sync + caller), 6 the
 * whole forward, 7 moment clear, 8 backward blend (K4), 9 chain (K5) */

int nxs_abi_version(void);
const char* nxs_error_string(int code);
/* message of the last error on this thread (with CUDA detail if any) */
const char* nxs_last_error(void);

int nxs_view_create(nxs_view** out);
int nxs_view_destroy(nxs_view* view);
int nxs_view_stats(const nxs_view* view, nxs_stats* out);
/* bytes of device memory currently held by the view */
int64_t nxs_view_bytes(const nxs_view* view);

/* Phase timing (CUDA events between the pipeline's phases) is off by
 * default: each event costs the device pipeline a few microseconds.  on != 0
 * records them from the next call on. */
int nxs_view_set_timing(nxs_view* view, int on);
/* Milliseconds per phase (NXS_PHASES entries) of the last nxs_forward /
 * nxs_backward of this view (timing on); waits for those phases to finish. */
int nxs_view_timings(nxs_view* view, float* ms, int n);

/* Forward render (render_forward_cached).  background: 3 host floats.
 * rgb (H*W*3), overdraw (H*W), residual (H*W): device outputs, row-major
 * over (row, col).  Fills the view's replay cache. */
int nxs_forward(nxs_view* view, const nxs_scene* scene, const nxs_camera* camera,
                const nxs_model* model, const nxs_opts* opts, const float background[3],
                float* rgb, int32_t* overdraw, float* residual, void* stream);

/* Backward (render_backward) for adjoint seed d loss / d rgb (device,
 * H*W*3).  Replays the view's last forward; the scene must be unchanged.
 * Accumulates into g_centers (P,3), g_scales (P,3), g_quats (P,4),
 * g_opacities (P), g_sh (P,3,C) (device float32). */
int nxs_backward(nxs_view* view, const nxs_scene* scene, const float* seed,
                 float* g_centers, float* g_scales, float* g_quats,
                 float* g_opacities, float* g_sh, void* stream);

/* Forward + backward in one call (render_with_gradients, render.py:445-464):
 * nxs_forward then nxs_backward with the same arguments, but the depth-phase
 * check that ends the forward is overlapped with the backward (the view
 * speculates on the number of phases its previous call needed and redoes
 * both passes when more were needed). */
int nxs_forward_backward(nxs_view* view, const nxs_scene* scene, const nxs_camera* camera,
                         const nxs_model* model, const nxs_opts* opts, const float background[3],
                         float* rgb, int32_t* overdraw, float* residual, const float* seed,
                         float* g_centers, float* g_scales, float* g_quats, float* g_opacities,
                         float* g_sh, void* stream);

/* Reference cache fields of the last forward (device outputs, any may be
 * NULL): sat (H*W uint8), e_k (H*W*3), t_k (H*W), theta0 (H*W*3). */
int nxs_cache_export(nxs_view* view, uint8_t* sat, float* e_k, float* t_k,
                     float* theta0, void* stream);

/* Front-to-back depth order of the last forward: order (P int32, device),
 * order[rank] = Gaussian index, stable by fp64 view depth (render.py:355-357).
 * The global order sorts lazily (only the depth phases the image needed);
 * this call completes the order of the remaining ranks first.  (Chunked and
 * exact orders: the ranks of the list order the blend used.) */
int nxs_depth_order(nxs_view* view, int32_t* order, void* stream);

/* Binning of the last forward, for the bit-exact checks against the C
 * restatement (oracle/binning_oracle.c): tile rectangle per Gaussian in
 * storage order (P x int32[4] = tx0,ty0,tx1,ty1; empty = -1; Gaussians
 * outside the projected depth phases read empty), and the FIRST depth
 * phase's tile ranges (n_tiles x int32[2]) and sorted pair values, lists
 * compacted tile after tile (ranges index pair_ranks); with
 * NXS_FLAG_FULL_BINNING that phase holds every rank (n_pairs ranks).
 * Synchronises `stream` (an inspection call, not on the hot path). */
int nxs_binning_export(nxs_view* view, int32_t* rects, int32_t* ranges,
                       int32_t* pair_ranks, void* stream);

/* Projected per-rank records (P x 32 float32) of the last forward; only the
 * ranks of the processed depth phases are defined (NXS_FLAG_FULL_BINNING
 * projects every rank). */
int nxs_records_export(nxs_view* view, float* records, void* stream);

/* The Gaussians (storage indices, no particular order) whose gradients the
 * last backward of this view wrote: every other row of its gradient
 * contribution is zero.  *count (HOST pointer) receives their number; the
 * call synchronises `stream` to read it.  gids (device, capacity >= the
 * scene's count, or NULL to query the count only).  Used to move only the
 * touched gradient rows (render_with_gradients' download, the sparse
 * data-parallel reduction). */
int nxs_touched_export(nxs_view* view, int32_t* gids, int64_t* count, void* stream);

/* Sizing history of a view — the estimates its device-sized first depth
 * phase is planned from (ranks, pairs, key bins, the last rank its tiles
 * needed, the speculated phase count) and the camera they belong to — as an
 * opaque blob of nxs_view_history_bytes() bytes.  A caller that cycles many
 * cameras through a few workspaces saves each camera's history after its
 * call and loads it into the workspace before the next call of that camera,
 * so every camera keeps the sync-free path.  Loading ends the workspace's
 * last forward (no backward of it afterwards). */
int64_t nxs_view_history_bytes(void);
int nxs_view_history_save(nxs_view* view, void* blob);
int nxs_view_history_load(nxs_view* view, const void* blob);

/* ---- data-parallel gradient plumbing (no reference
 * counterpart: the reference renders one view per iteration,
 * optimizer.py:393-408) ------------------------------------------------
 * A rank's gradient buffer `flat` is float32, n Gaussians, field after
 * field: [centers (n,3) | scales (n,3) | quats (n,4) | opacities (n) |
 * sh (n,3,C)] (paper_2603_02887_b200/dp.py GradBuffer); a Gaussian's row is
 * 11 + 3C floats.  `mask` is one byte per Gaussian. */

/* mask[g] = 1 for every Gaussian the view's last backward wrote (async,
 * no host sync): the union over a rank's views is its touched set. */
int nxs_touched_mark(nxs_view* view, uint8_t* mask, void* stream);

/* Zero the rows of flagged Gaussians and clear their flags (the next step's
 * clear touches only last step's rows, instead of the whole buffer). */
int nxs_grads_zero_masked(float* flat, int64_t n, int32_t sh_coeffs, uint8_t* mask,
                          void* stream);

/* index[0..count) = flagged Gaussians, ascending; *count (HOST) — the call
 * synchronises `stream` to read it (the collective needs the size). */
int nxs_grads_select(const uint8_t* mask, int64_t n, int32_t* index, int64_t* count,
                     void* stream);

/* packed (count x (11+3C)) <- rows index[0..count) of flat, and back. */
int nxs_grads_gather(const float* flat, int64_t n, int32_t sh_coeffs, const int32_t* index,
                     int64_t count, float* packed, void* stream);
int nxs_grads_scatter(float* flat, int64_t n, int32_t sh_coeffs, const int32_t* index,
                      int64_t count, const float* packed, void* stream);

/* ---- train-step neighbours ---------------------------- */

/* Image loss (reference optimizer.py:128-152 loss(), :68-111 ssim(),
 * :114-118 mse()): (1 - lam) L1 + lam (1 - SSIM) in sRGB between the linear
 * render and target (device float32, H*W*3, row-major), 11x11 Gaussian
 * window (sigma 1.5) over fully-interior windows, computed in fp64.
 * out (device, 4 doubles): total, L1, mean SSIM (0 when lam == 0), MSE of
 * the clipped sRGB images.  seed (device H*W*3, may be NULL): d total /
 * d render, the adjoint seed for nxs_backward.  With NXS_LOSS_SRGB_INPUT the
 * inputs are already sRGB (the reference ssim(x, y) semantics) and seed is
 * d total / d x.  workspace: nxs_loss_workspace_bytes(H, W) device bytes.
 * lam > 0 needs H, W >= 11 (reference ValueError). */
#define NXS_LOSS_SRGB_INPUT 1
int64_t nxs_loss_workspace_bytes(int32_t height, int32_t width);
int nxs_image_loss(const float* rendered, const float* target, int32_t height, int32_t width,
                   double lam, int32_t flags, double* out, float* seed, void* workspace,
                   void* stream);

/* One bounded Adam step (reference optimizer.py:173-204 bounded_adam_step):
 * groups[5] in the order centers, scales, quats, opacities, sh (device
 * float32 param / grad / m / v of `count` elements; param NULL skips the
 * group).  Non-finite gradients are zeroed and counted into *nan_skips
 * (device u64); scales are floored at 1e-6, opacities clamped to
 * [1e-4, 1 - 1e-6], quaternion rows renormalised.  step = Adam step t >= 1
 * (after increment), betas 0.9 / 0.999, eps 1e-8. */
typedef struct {
    float* param;
    const float* grad;
    float* m;
    float* v;
    int64_t count;
    double lr;
} nxs_adam_group;
int nxs_adam_step(const nxs_adam_group* groups, int64_t step, double lr_mult,
                  unsigned long long* nan_skips, void* stream);
/* The same step in float64 (param / grad / m / v double): the numpy
 * drop-in's float64 parameters update without a float32 round trip, like
 * the reference optimizer (optimizer.py:173-204). */
typedef struct {
    double* param;
    const double* grad;
    double* m;
    double* v;
    int64_t count;
    double lr;
} nxs_adam_group_f64;
int nxs_adam_step_f64(const nxs_adam_group_f64* groups, int64_t step, double lr_mult,
                      unsigned long long* nan_skips, void* stream);

/* ---- per-ray batched compositing --------------------- */

/* composite_batch (reference compositor.py:84-171), fp64: R rays of N
 * front-to-back samples.  alpha (R*N), emission (R*N*3), valid (R*N uint8,
 * NULL = all valid; padding must be 0), background: 3 host doubles.
 * Device outputs (only radiance is required): weights (R*N clamped
 * extinction weights), radiance (R*3), residual (R), k0 (R, 0-based
 * saturation index, N when none), overdraw (R), e_k (R*3), theta0 (R*3),
 * t_k (R).  Backs finite_diff_gradients (adjoint.py:195-222). */
int nxs_composite_batch(const nxs_model* model, const double* alpha, const double* emission,
                        const uint8_t* valid, int64_t rays, int64_t samples,
                        const double background[3], double* weights, double* radiance,
                        double* residual, int64_t* k0, int64_t* overdraw, double* e_k,
                        double* theta0, double* t_k, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NXS_H */
