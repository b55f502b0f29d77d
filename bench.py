"""Benchmark: fwd+bwd megapixels/s of the splat renderer (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = forward + backward of the hot path for each of this rank's
views (N=1: config C3 — 1M Gaussians, 1920x1080, softplus(κ=20), global
depth order chunk_size=1 — the configuration the BASELINE metric is quoted
on), gradients accumulated into one flat buffer, plus one NCCL all-reduce
of that buffer when N > 1 (weak scaling: views_per_rank views per GPU).

value : Mpix/s with the scene and seeds resident in HBM (device path,
        CUDA events on the launching stream, max over ranks).
e2e   : the same metric through the public drop-in API
        (render_with_gradients on float64 numpy arrays): host->device copy of
        the scene and seed and device->host copy of image + gradients inside
        the timed region.
roofline: for the kernel with the largest share of the step, measured live
        (per-phase CUDA events, include/nxs.h nxs_view_timings).
cpu_baseline: the stock reference (nexsplat from baseline/_ref, its own
        _forward_sweep/_backward_sweep) on runs of consecutive pixels of the
        same view, all host cores, rank 0 only (forward-only for models the
        reference has no backward for, and labelled so).
--impl reference: times that CPU implementation as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd+bwd megapixels/sec at 1M Gaussians 1080p; fraction of FP32/HBM roofline"
# algorithmic flops per event (FMA = 2)
F_TEST = 24
F_FWD = {"linear": 37, "exponential": 38, "blended": 40, "vicini": 40, "softplus": 43,
         "quadratic": 39, "power_law": 43}
F_BWD = {"softplus": 146, "power_law": 146}
F_BWD_DEFAULT = 140


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--gaussians", type=int, default=1_000_000)
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--model", default="softplus")
    p.add_argument("--param", type=float, default=None)
    p.add_argument("--views-per-rank", type=int, default=1)
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--chunk", default="1",
                   help="ordering: 1 = global depth order (default), none = exact per-pixel order, "
                        "C > 1 = chunked order")
    p.add_argument("--pool", type=int, default=8,
                   help="nxs_view workspaces per rank; the rank's views cycle through them")
    p.add_argument("--deterministic", action="store_true",
                   help="bit-reproducible gradients (NXS_FLAG_DETERMINISTIC)")
    p.add_argument("--adam", action="store_true",
                   help="apply a bounded Adam step to the scene after every step (a moving "
                        "scene, as in training: exercises the per-tile capacity refresh)")
    p.add_argument("--first-phase", type=int, default=0,
                   help="ranks binned in the first depth phase (0 = automatic)")
    return p.parse_args()


def model_of(a):
    from paper_2603_02887_b200 import TransmittanceModel
    defaults = {"softplus": 20.0, "blended": 0.5, "vicini": 0.5, "quadratic": 0.5,
                "power_law": 2.0}
    p = a.param if a.param is not None else defaults.get(a.model, 0.0)
    return TransmittanceModel(a.model, p)


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the reference's own implementation of the
# path, timed on a bounded sample (rank 0)
# ---------------------------------------------------------------------------
# The stock reference package (pip-installed from /root/reference into
# baseline/_ref, which travels to the GPU box) is imported and its own sweep
# functions — nexsplat.render._forward_sweep / _backward_sweep, the body of
# render_with_gradients (reference render.py:147-347, 445-464) with the
# chunk_size=1 order of _depth_chunks (render.py:350-358) — run on contiguous
# runs of pixels of the C3 view, one run per worker process, all host cores.
# A run of pixels is the unit the reference itself vectorises over (its
# render() splits the image into row bands per thread, render.py:394-400).
# The reference has no softplus/blended backward (render.py:229-231): for
# those models the sample is forward-only and says so.  Without
# baseline/_ref the oracle port (oracle/splat_oracle.py, brute force over all
# Gaussians per pixel, slower than the reference) is timed and labelled.

REF_DIR = ROOT / "baseline" / "_ref"
_CPU = {}


def _ref_modules():
    """(render module, Camera, TransmittanceModel) of the stock reference, or None."""
    if not (REF_DIR / "nexsplat").is_dir():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import importlib
    try:
        R = importlib.import_module("nexsplat.render")
        prim = importlib.import_module("nexsplat.primitives")
        tm = importlib.import_module("nexsplat.transmittance")
    except Exception:
        return None
    return R, prim.Camera, tm.TransmittanceModel


def _ref_setup(a, model):
    """Scene, camera, order chunks and seeds, built once before the workers fork."""
    from paper_2603_02887_b200.scenes import canonical_scene
    mods = _ref_modules()
    arrs = canonical_scene(a.gaussians, seed=5)
    seed = np.random.default_rng(1000).uniform(0.2, 1.0, (a.height * a.width, 3))
    if mods is not None:
        R, Camera, TM = mods
        sc = R.SceneArrays(arrs.centers, arrs.scales, arrs.quats, arrs.opacities, arrs.sh)
        cam = Camera.from_look_at([0.0, 0.0, 0.0], [0.0, 0.0, 3.5], [0.0, 1.0, 0.0], 55.0,
                                  a.width, a.height)
        m = TM(model.variant, float(model.param))
        chunk = 1 if a.chunk_size is None else a.chunk_size
        chunks = R._depth_chunks(sc, cam, None if a.chunk_size is None else chunk)
        bwd = m.variant in ("linear", "quadratic", "exponential")
        _CPU.update(kind="reference", R=R, sc=sc, cam=cam, model=m, chunks=chunks, bwd=bwd,
                    dirs=cam.pixel_directions().reshape(-1, 3), seed=seed)
    else:
        from oracle import splat_oracle as O
        from paper_2603_02887_b200.scenes import canonical_camera
        _CPU.update(kind="port", sc=O.Scene.of(arrs), cam=canonical_camera(a.width, a.height),
                    model=model, seed=seed, bwd=True, chunk_size=a.chunk_size)


def _cpu_task(args):
    """One run of `npx` consecutive pixels from flat index `start`: forward
    (+ backward where the reference has one).  Returns (pixels, seconds)."""
    start, npx = args
    px = np.arange(start, start + npx)
    t0 = time.perf_counter()
    if _CPU["kind"] == "reference":
        R, cam = _CPU["R"], _CPU["cam"]
        fwd = R._forward_sweep(_CPU["sc"], _CPU["dirs"][px], cam.position, _CPU["model"],
                               np.zeros(3), 128, 1.0 / 255.0, 1e-4, _CPU["chunks"])
        if _CPU["bwd"]:
            R._backward_sweep(_CPU["sc"], _CPU["dirs"][px], cam.position, _CPU["model"],
                              np.zeros(3), 128, 1.0 / 255.0, 1e-4, _CPU["chunks"], fwd,
                              _CPU["seed"][px])
    else:
        from oracle import splat_oracle as O
        fwd = O.forward(_CPU["sc"], _CPU["cam"], _CPU["model"], np.zeros(3),
                        chunk_size=_CPU["chunk_size"], pixels=px, prune=False, keep_state=True,
                        batch=npx)
        O.backward(_CPU["sc"], _CPU["cam"], _CPU["model"], np.zeros(3), fwd, _CPU["seed"][px])
    return npx, time.perf_counter() - t0


class CpuRunner:
    """A pool of worker processes over all host cores (forked after setup)."""

    def __init__(self, a, model):
        import multiprocessing as mp
        _ref_setup(a, model)
        cores = os.cpu_count() or 1
        workers = cores
        try:  # each worker ends up with its own copy of the scene and chunk list
            import psutil
            workers = max(1, min(workers, int(psutil.virtual_memory().available / 1.5e9)))
        except Exception:
            pass
        self.workers = workers
        self.npix = a.width * a.height
        self.pool = mp.get_context("fork").Pool(workers)
        self.rng = np.random.default_rng(7)

    def step(self, npx):
        """Every worker renders one run of npx pixels; (pixels, wall seconds)."""
        starts = self.rng.integers(0, self.npix - npx, self.workers)
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_task, [(int(s0), npx) for s0 in starts], chunksize=1)
        return sum(r[0] for r in res), time.perf_counter() - t0

    def describe(self, npx, n_steps):
        try:
            cpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
            name = [ln.split(":", 1)[1].strip() for ln in cpu.splitlines()
                    if "Model name" in ln][0]
        except Exception:
            name = "unknown"
        if _CPU["kind"] == "reference":
            what = ("stock reference nexsplat (baseline/_ref) _forward_sweep"
                    + (" + _backward_sweep" if _CPU["bwd"] else
                       " only: the reference has no backward for this model "
                       "(render.py:229-231), so its line is FORWARD-ONLY Mpix/s"))
        else:
            what = ("oracle port (oracle/splat_oracle.py) fwd+bwd, brute force over all "
                    "Gaussians per pixel: slower than the reference (no early exit), "
                    "baseline/_ref missing")
        return (f"{what}; {n_steps} step(s) x {self.workers} processes x {npx} consecutive "
                f"pixels at random positions of the view; {name}")

    def close(self):
        self.pool.close()
        self.pool.join()


def _ref_npx(steps):
    """Pixels per worker task: ~7 s tasks for short runs, smaller for long ones
    (the reference arm must finish within a few minutes)."""
    return int(max(256, min(1024, 1024 * 25 // max(1, steps))))


def cpu_baseline(a, model):
    r = CpuRunner(a, model)
    try:
        npx = _ref_npx(1)
        px, wall = r.step(npx)
        return {"value": px / wall / 1e6, "unit": "Mpix/s", "cores": r.workers,
                "kind": _CPU["kind"], "sample": r.describe(npx, 1) + f"; wall {wall:.1f}s"}
    finally:
        r.close()


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML
    thread polling every ~2 ms (a C3 step is 0.5 ms, so a 30-step region
    lasts ~16 ms — shorter than nvidia-smi's 100 ms period); nvidia-smi
    -lms 100 as the fallback when NVML is unavailable."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        import threading
        self.p = None
        self.samples = []
        self.stop_ev = threading.Event()
        self.th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = gpu
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis and vis.split(",")[gpu].strip().isdigit():
                idx = int(vis.split(",")[gpu])
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop_ev.is_set():
                    try:
                        self.samples.append(
                            (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                             pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
            return
        except Exception:
            self.th = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def mark_start(self):
        """Drop the samples taken before the timed region (NVML thread)."""
        self.samples = []

    def stop(self):
        if self.th is not None:
            self.stop_ev.set()
            self.th.join(timeout=1.0)
            if not self.samples:
                return None
            reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items()
                              if r & bit})
            return {"sm_mhz": statistics.median(c for c, _ in self.samples),
                    "sm_max_mhz": self.mx, "reasons": reasons, "samples": len(self.samples),
                    "source": "nvml"}
        if self.p is None:
            return None
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    model = model_of(a)
    a.chunk_size = None if str(a.chunk).lower() in ("none", "0", "exact") else int(a.chunk)

    if a.impl == "reference":
        return reference_arm(a, rank, model)

    import torch
    import torch.distributed as dist

    from paper_2603_02887_b200 import (DeviceScene, _native, render_with_gradients)
    from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, device_view_renderer
    from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W, H, vpr = a.width, a.height, a.views_per_rank
    n_views = vpr * world
    arrs = canonical_scene(a.gaussians, seed=5)
    dev = DeviceScene.from_arrays(arrs)
    if n_views == 1:
        cams = [canonical_camera(W, H)]
    else:
        cams = [canonical_camera(W, H, v, n_views) for v in range(n_views)]
    # adjoint seeds: view v's own for up to 8 views, else cycled over 8
    # (256 distinct 4K seed images would hold 25 GB)
    seed_pool = [torch.as_tensor(canonical_seed(W, H, v), dtype=torch.float32, device="cuda")
                 for v in range(min(n_views, 8))]

    def seeds(v):
        return seed_pool[v % len(seed_pool)]

    bg = np.zeros(3)
    grads = GradBuffer(len(arrs), arrs.sh.shape[2], device="cuda")
    rv = device_view_renderer(dev, model, bg, cams, seeds, first_phase_ranks=a.first_phase,
                              chunk_size=a.chunk_size, deterministic=a.deterministic,
                              pool=a.pool)
    step = DataParallelStep(n_views, rank, world, grads, rv)
    my_views = step.views()
    if a.adam:  # every step also moves the scene (lr of the reference optimizer's order)
        from paper_2603_02887_b200.optim import AdamState, bounded_adam_step
        params = {k: getattr(dev, k) for k in DeviceScene.FIELDS}
        adam = AdamState.for_params(params)
        lrs = {"centers": 1.6e-4, "scales": 5e-3, "quats": 1e-3, "opacities": 5e-2, "sh": 2.5e-3}
        plain_step = step

        def step():
            g = plain_step()
            bounded_adam_step(params, g.fields, adam, lrs)
            return g

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, device events, barrier + sync both sides
    clocks = Clocks(local)
    time.sleep(0.25)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark_start()
    launches0 = sum(w.stats()["n_launches"] for w in rv.workspaces)
    redo0 = sum(w.stats()["n_redo"] for w in rv.workspaces)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    # hand-written kernels the library launched in the timed steps (counted
    # per enqueue; a captured phase-0 graph counts its kernels each call)
    n_launches = sum(w.stats()["n_launches"] for w in rv.workspaces) - launches0
    n_redo = sum(w.stats()["n_redo"] for w in rv.workspaces) - redo0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ck = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / a.steps
    mpix = W * H * n_views / (ms_step / 1e3) / 1e6

    # ---- per-phase device timings (same steps, events inside the library)
    wss = rv.workspaces
    for w in wss:  # phase events only here (they cost the pipeline a few us)
        w.set_timing(True)
    phase_tot = {}
    step()
    for _ in range(max(3, min(a.steps, 10))):
        step()
        for w in wss:  # each workspace's last call: one view's phases
            for k, x in w.timings().items():
                phase_tot[k] = phase_tot.get(k, 0.0) + x
    nprof = max(3, min(a.steps, 10))
    phase = {k: x / nprof / max(1, len(wss)) for k, x in phase_tot.items()}
    n_depth_phases = phase.pop("n_depth_phases", None)

    # ---- event counts (instrumented run, not timed) for the blend roofline
    from paper_2603_02887_b200 import backward_device, forward_device
    cview = _native.View()
    forward_device(cview, dev, cams[my_views[0]], model, bg, chunk_size=a.chunk_size,
                   count_events=True, first_phase_ranks=a.first_phase)
    backward_device(cview, dev, seeds(my_views[0]))
    st = cview.stats()
    cview.close()

    roof = roofline(a, model, phase, st)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e = e2e_arm(a, arrs, cams, model, my_views, world, render_with_gradients)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a, model)

    if rank == 0:
        out = {
            "metric": METRIC,
            "value": round(mpix, 3),
            "unit": "Mpix/s",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": config_of(a, model, vpr, world),
            "phase_ms": {k: round(v, 4) for k, v in phase.items()},
            "depth_phases": n_depth_phases,
            "events": {k: st[k] for k in ("n_pairs", "n_tests_fwd", "n_composited",
                                           "n_tests_bwd", "n_entries_bwd")},
            "roofline": roof,
            "clocks": ck,
            "gpu_launches": n_launches,
            "redone_passes": n_redo,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def config_of(a, model, vpr, world):
    """The workload description, identical in both arms (same_config)."""
    W, H = a.width, a.height
    n_views = vpr * world
    return {
        "workload": (("C3: " if (a.gaussians, W, H) == (1_000_000, 1920, 1080) else
                      "C5-like: " if a.gaussians >= 5_000_000 else "custom: ")
                     + f"{a.gaussians} Gaussians (canonical synthetic scene, seed 5), "
                     f"{W}x{H}, {model.describe()}, "
                     + ("chunk_size=1 (global depth order), " if a.chunk_size == 1 else
                        "chunk_size=None (exact per-pixel order), " if a.chunk_size is None
                        else f"chunk_size={a.chunk_size} (chunked order), ")
                     + f"fwd+bwd, {vpr} view(s) per GPU"
                     + (", + bounded Adam step on the scene per step" if a.adam else "")
                     + (", deterministic gradients" if a.deterministic else "")),
        "gaussians": a.gaussians, "width": W, "height": H,
        "views_per_gpu": vpr, "total_views": n_views,
        "parallelism": f"dp{world} over views",
        "l2": "inputs larger than L2 (records 128 MB + pairs + 192 MB moments per view)",
    }


def roofline(a, model, phase, st):
    """Dominant kernel vs its bound.  Blend kernels: FP32 pipe (algorithmic
    flops); sort/projection/chain: HBM bytes."""
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    fp32_peak = sms * 128 * 2 * sm_mhz * 1e6 / 1e12  # TFLOP/s
    var = model.variant
    blend_ms = phase.get("blend_fwd", 0.0) + phase.get("blend_bwd", 0.0)
    flops = (st["n_tests_fwd"] * F_TEST + st["n_composited"] * F_FWD.get(var, 40)
             + st["n_tests_bwd"] * F_TEST + st["n_composited"] * F_BWD.get(var, F_BWD_DEFAULT))
    blend = {"bound": "tensor" if False else "fp32", "achieved": flops / (blend_ms / 1e3) / 1e12
             if blend_ms > 0 else 0.0, "peak": round(fp32_peak, 2), "unit": "TFLOP/s"}
    P, npairs = a.gaussians, st["n_pairs"]
    # pair sort: 2 LSD passes over (u32 tile key, u32 rank) pairs, read + write
    sort_bytes = npairs * 8 * 2 * 2
    proj_bytes = P * (92 + 8 + 128 + 16 + 8)  # params + order in; record + rect + count out
    shares = {"blend (fwd+bwd)": blend_ms, "binning": phase.get("binning", 0.0),
              "depth_sort": phase.get("depth_sort", 0.0), "project": phase.get("project", 0.0)}
    dom = max(shares, key=shares.get)
    total = sum(x for k, x in phase.items() if k not in ("forward_total", "fwd_bwd_gap"))
    if dom == "blend (fwd+bwd)":
        r = dict(blend, kernel=dom)
    elif dom == "binning":
        ach = sort_bytes / (phase["binning"] / 1e3) / 1e9
        r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "kernel": dom}
    elif dom == "project":
        ach = proj_bytes / (phase["project"] / 1e3) / 1e9
        r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "kernel": dom}
    else:
        b = P * (8 + 4) * 2 * 8 + P * 12
        ach = b / (phase["depth_sort"] / 1e3) / 1e9
        r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "kernel": dom}
    r["achieved"] = round(r["achieved"], 3)
    r["frac"] = round(r["achieved"] / r["peak"], 4) if r["peak"] else None
    r["traffic"] = None
    # DRAM bytes and FP32-pipe utilisation of the blend kernels from the
    # committed ncu capture of this workload (profiles/r02_blend_traffic.json)
    try:
        cap = json.loads((ROOT / "profiles" / "r02_blend_traffic.json").read_text())
        k = cap["per_step"]
        if dom == "blend (fwd+bwd)" and model.variant == "softplus" and a.chunk_size == 1 \
                and a.gaussians == 1_000_000 and (a.width, a.height) == (1920, 1080):
            r["traffic"] = sum(v["dram_read_bytes"] + v["dram_write_bytes"] for v in k.values())
            r["traffic_unit"] = "bytes per step (fwd + bwd launches)"
            r["ncu_fma_pipe_pct"] = {n: v["fma_pipe_pct"] for n, v in k.items()}
            r["ncu_issue_active_pct"] = {n: v["issue_active_pct"] for n, v in k.items()}
            r["ncu_source"] = "profiles/r02_blend_traffic.json"
    except Exception:
        pass
    r["share_of_step"] = round(shares[dom] / total, 3) if total else None
    r["blend_fp32"] = {"achieved_tflops": round(blend["achieved"], 3),
                       "frac_of_derived_peak": round(blend["achieved"] / fp32_peak, 4),
                       "flops": flops, "ms": round(blend_ms, 4)}
    r["achieved_source"] = ("kernel durations from CUDA events the library records on the "
                            "launching stream around each phase (nxs_view_timings), averaged over "
                            "further timed steps right after the headline region (the headline "
                            "region itself runs without those events); flops from an "
                            "instrumented run's event counts (NXS_FLAG_COUNT_EVENTS)")
    r["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs (measured copy)" if r["unit"] == "GB/s"
                        else f"derived: {sms} SMs x 128 FMA x 2 x {sm_mhz:.0f} MHz "
                             "(MEASURED_PEAKS.json sm_max_mhz)")
    return r


def e2e_arm(a, arrs, cams, model, my_views, world, render_with_gradients):
    """Public drop-in API on host float64 arrays: every step uploads the
    scene + seed and downloads rgb/overdraw/residual + gradients."""
    import torch
    from paper_2603_02887_b200.scenes import canonical_seed
    seeds = {v: canonical_seed(a.width, a.height, v) for v in my_views}

    def one():
        for v in my_views:
            res, g = render_with_gradients(arrs, cams[v], model, np.zeros(3), seeds[v],
                                           chunk_size=a.chunk_size)
        return res, g

    if world > 1:
        return e2e_dp(a, arrs, cams, model, my_views, world)
    # warm-up calls (first-call setup, the pinned result pool, the view's
    # sizing history), as many as the device arm's, at least 3
    for _ in range(max(3, a.warmup)):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.e2e_steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / a.e2e_steps
    from paper_2603_02887_b200.render import _LAST_IO
    npx = a.width * a.height
    # bytes the API moved per view (fp32 scene + seed up; float64 image,
    # residual, int64 overdraw and gradients down)
    h2d = len(my_views) * _LAST_IO["h2d"]
    d2h = len(my_views) * _LAST_IO["d2h"]
    return {"value": round(npx * len(my_views) * world / dt / 1e6, 3), "unit": "Mpix/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 3),
            "api": f"render_with_gradients(numpy float64 SceneArrays, chunk_size={a.chunk_size})"}


def e2e_dp(a, arrs, cams, model, my_views, world):
    """N > 1 end to end through the data-parallel API: every step uploads the
    scene (float64 host arrays -> fp32) and this rank's seeds from the host,
    renders its views into the gradient buffer, all-reduces it across the
    ranks (sparse, NCCL) and downloads the summed gradients to pinned host
    memory.  Wall clock per step, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2603_02887_b200 import DeviceScene
    from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, device_view_renderer
    from paper_2603_02887_b200.render import _h2d_f32
    from paper_2603_02887_b200.scenes import canonical_seed
    host_seeds = {v: canonical_seed(a.width, a.height, v) for v in my_views[:8]}
    dev = DeviceScene.from_arrays(arrs)
    seed_dev = {}
    grads = GradBuffer(len(arrs), arrs.sh.shape[2], device="cuda")
    out = torch.empty(grads.flat.numel(), dtype=torch.float32, pin_memory=True)
    rv = device_view_renderer(dev, model, np.zeros(3), cams, lambda v: seed_dev[v % 8],
                              chunk_size=a.chunk_size, pool=a.pool)
    step = DataParallelStep(len(cams), int(os.environ.get("RANK", "0")), world, grads, rv)

    def one():
        for k in DeviceScene.FIELDS:  # upload the scene
            x = getattr(arrs, k)
            setattr(dev, k, _h2d_f32(np.asarray(x).reshape(tuple(getattr(dev, k).shape)),
                                     dev.centers.device, "e2e_" + k))
        for v, sd in host_seeds.items():
            seed_dev[v % 8] = _h2d_f32(sd, dev.centers.device, f"e2e_seed{v % 8}")
        g = step()
        out.copy_(g.flat, non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(max(3, a.warmup)):
        one()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(a.e2e_steps):
        one()
    dt = (time.perf_counter() - t0) / a.e2e_steps
    t = torch.tensor([dt], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    npx = a.width * a.height
    h2d = sum(int(np.prod(np.shape(getattr(arrs, k)))) * 4 for k in DeviceScene.FIELDS) \
        + len(host_seeds) * npx * 3 * 4
    d2h = grads.flat.numel() * 4
    return {"value": round(npx * len(my_views) * world / dt / 1e6, 3), "unit": "Mpix/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 3),
            "api": "DataParallelStep (device_view_renderer + sparse NCCL all-reduce) with the "
                   "scene and seeds uploaded from host float64 arrays and the summed gradients "
                   "downloaded, every step"}


def reference_arm(a, rank, model):
    """The reference's own CPU implementation of the path (the stock package
    from baseline/_ref, see the CPU-baseline section), rank 0 only, all host
    cores; each step every worker renders one run of pixels."""
    if rank != 0:
        return
    r = CpuRunner(a, model)
    npx = _ref_npx(a.steps + a.warmup)
    vals = []
    try:
        for i in range(a.warmup + a.steps):
            px, wall = r.step(npx)
            if i >= a.warmup:
                vals.append(px / wall / 1e6)
        sample = r.describe(npx, a.steps)
    finally:
        r.close()
    v = statistics.median(vals)
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "Mpix/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": a.steps,
        "warmup": a.warmup,
        "higher_is_better": True,
        "dtype": "f64",
        "data": "synthetic",
        "config": config_of(a, model, a.views_per_rank, int(os.environ.get("WORLD_SIZE", "1"))),
        "cpu_baseline": {"value": v, "unit": "Mpix/s", "cores": r.workers, "kind": _CPU["kind"],
                         "sample": sample},
        "e2e": {"value": v, "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
