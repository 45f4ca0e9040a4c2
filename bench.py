#!/usr/bin/env python3
"""NLINV real-time reconstruction benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

A step is one frame: the full IRGNM reconstruction of one gridded k-space frame
(7 Newton steps, 50-iteration conjugate-residual budget, final RSS image), chained
from the previous frame's estimate as in reconstruct_series_plain (nlinv.cpp:412-444).
At N = 1 the workload is configs[2] of BASELINE.json (C3: 256x256 grid, 32 channels),
the configuration the north-star 30 frames/s target is quoted on; the other configs
are parity-test cases. Under torchrun every rank reconstructs its own slice series
(multi-slice imaging): no data-path collective, weak scaling.

Inputs are synthetic (numpy): an ellipse phantom with one moving feature, smooth
coil profiles, an exact radial-trajectory Toeplitz kernel (K = 15 spokes, U = 5
turns) and gridded data z_j = T(rho c_j) + noise. They are staged in HBM before the
timed region; every frame has its own 16 MB data buffer and the staged series is
larger than L2, so each frame starts cold. `value` is device time (CUDA events
spanning the worker streams); `e2e` is the public C-ABI series call with pinned
host frames streamed in (H2D) and images read back (D2H) inside the timed region.
"""
import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (G, J, K spokes, U turns, description)
    "c1": (128, 8, 13, 5, "configs[0]: 64x64 image, 128x128 grid, 8 channels, 13 spokes"),
    "c2": (320, 10, 15, 5, "configs[1]: 160x160 image, 320x320 grid, 10 channels, 15 spokes"),
    "c3": (256, 32, 15, 5, "configs[2]: 256x256 grid, 32 channels, 15 spokes"),
    "c4": (256, 16, 15, 5, "configs[3]: 256x256 grid, 16 channels, 15 spokes"),
    "c5": (384, 64, 15, 5, "configs[4]: 384x384 grid, 64 channels, 15 spokes"),
}
METRIC = "frames/sec (NLINV, 7 Newton steps)"


# ------------------------------------------------------------------------------------
# synthetic inputs (numpy only; no oracle code on this path)
# ------------------------------------------------------------------------------------
def fftc2(x):
    """centered unitary forward 2D DFT (DC at n/2), the reference convention (fft.hpp:22-30)"""
    n = x.shape[-1]
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x, axes=(-2, -1))), axes=(-2, -1)) / n


def ifftc2(x):
    n = x.shape[-1]
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x, axes=(-2, -1))), axes=(-2, -1)) * n


def radial_psf(G, N, K, U, turn):
    """Toeplitz kernel of a K-spoke radial frame (turn `turn` of U), built from the exact
    trajectory response q(d) = sum_s v_s exp(2 pi i k_s . d) with ramp density weights."""
    S = 2 * N
    c = G // 2
    i = np.arange(S)
    r = (2.0 * i + 1.0 - S) / (2.0 * S)
    ang = (np.arange(K) * 2 * np.pi / K + turn * 2 * np.pi / (K * U)) % (2 * np.pi)
    kx = (r[None, :] * np.cos(ang)[:, None]).ravel()
    ky = (r[None, :] * np.sin(ang)[:, None]).ravel()
    v = np.maximum(np.hypot(kx, ky), 0.5 / G) * (np.pi / K) / S
    d = np.arange(G) - c
    ax = np.exp(2j * np.pi * kx[:, None] * d[None, :])
    ay = np.exp(2j * np.pi * ky[:, None] * d[None, :])
    q = (ax.T * v[None, :]) @ ay
    q[0, :] = 0
    q[:, 0] = 0
    return (fftc2(q) * G).astype(np.complex64)


def phantom_and_coils(G, N, J, n):
    L = G // 2
    lo = (G - L) // 2
    yy, xx = np.mgrid[0:G, 0:G]
    x = (xx - G / 2) / N
    y = (yy - G / 2) / N
    rho = np.zeros((G, G), np.complex128)
    shift = 0.05 * math.sin(2 * math.pi * n / 16)
    for cx, cy, a, b, th, amp in ((0.0, 0.0, 0.44, 0.40, 0.0, 1.0), (0.0, 0.0, 0.38, 0.35, 0.2, -0.5),
                                  (-0.12, 0.08, 0.12, 0.09, 0.4, 0.4 + 0.1j), (0.1, -0.12, 0.09, 0.07, -0.3, 0.3),
                                  (0.05 + shift, 0.17, 0.06, 0.06, 0.0, 0.6)):
        ct, st = math.cos(th), math.sin(th)
        u = ((x - cx) * ct + (y - cy) * st) / a
        w = (-(x - cx) * st + (y - cy) * ct) / b
        rho += amp * (u * u + w * w <= 1.0)
    win = np.zeros((G, G), bool)
    win[lo:lo + L, lo:lo + L] = True
    rho *= win
    coils = np.empty((J, G, G), np.complex128)
    for j in range(J):
        a = 2 * math.pi * j / J + math.pi / 4
        mx, my = 0.3 * math.cos(a), 0.3 * math.sin(a)
        env = (1 + 0.3 * np.cos(np.pi * (x - mx))) * (1 + 0.3 * np.cos(np.pi * (y - my)))
        ph = 2 * np.pi * (0.35 * math.cos(a + 0.7) * x + 0.35 * math.sin(a + 0.7) * y) + a
        coils[j] = env * np.exp(1j * ph)
    return rho, coils, win


def synth_series(G, J, K, U, n_unique, seed=1234, noise=1e-3):
    N = G // 2
    P = np.stack([radial_psf(G, N, K, U, t) for t in range(U)])
    rng = np.random.default_rng(seed)
    frames = []
    for n in range(n_unique):
        rho, coils, win = phantom_and_coils(G, N, J, n)
        x = rho[None] * coils
        t = ifftc2(P[n % U][None].astype(np.complex128) * fftc2(x * win)) * win
        t += noise * (rng.standard_normal(t.shape) + 1j * rng.standard_normal(t.shape)) * win
        frames.append(t.astype(np.complex64))
    return np.stack(frames), P


def spoke_angles(K, U, turn):
    """K spokes of turn `turn` of a U-turn radial trajectory (the angle sets of radial_psf)"""
    return (np.arange(K) * 2 * np.pi / K + turn * 2 * np.pi / (K * U)) % (2 * np.pi)


def synth_raw(G, J, K, U, n_unique):
    """raw radial acquisitions (KSpaceFrame layout: J x K x S samples, S = 2N per spoke):
    the phantom x coil images' centered DFT on the G grid, bilinearly interpolated at the
    spoke samples (no oracle code on this path)"""
    N = G // 2
    S = 2 * N
    r = (2.0 * np.arange(S) + 1.0 - S) / (2.0 * S)
    samples = np.zeros((n_unique, J, K, S), np.complex64)
    angles = np.zeros((n_unique, K))
    for n in range(n_unique):
        rho, coils, win = phantom_and_coils(G, N, J, n)
        X = fftc2((rho[None] * coils) * win)
        ang = spoke_angles(K, U, n % U)
        angles[n] = ang
        u = (r[None, :] * np.cos(ang)[:, None]) * G + G / 2
        w = (r[None, :] * np.sin(ang)[:, None]) * G + G / 2
        u0, w0 = np.floor(u).astype(int), np.floor(w).astype(int)
        fu, fw = u - u0, w - w0
        for j in range(J):
            Xj = X[j]
            v = ((1 - fu) * (1 - fw) * Xj[u0 % G, w0 % G] + fu * (1 - fw) * Xj[(u0 + 1) % G, w0 % G]
                 + (1 - fu) * fw * Xj[u0 % G, (w0 + 1) % G] + fu * fw * Xj[(u0 + 1) % G, (w0 + 1) % G])
            samples[n, j] = v.astype(np.complex64)
    return samples, angles


# ------------------------------------------------------------------------------------
# measurement helpers
# ------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (written to a
    file by nvidia-smi itself: a pipe would block-buffer the samples)"""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.path = os.path.join("/tmp", f"rtn_clocks_{os.getpid()}_{device}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            try:
                with open(self.path) as f:
                    self.lines = [ln.strip() for ln in f if ln.strip()]
                os.remove(self.path)
            except OSError:
                pass

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def step_traffic(cfg):
    """whole-step DRAM bytes per frame from the committed app-range capture
    (profiles/step_traffic.json, scripts/step_range.py), or None"""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "step_traffic.json")))[cfg]
        return {k: d[k] for k in ("dram_bytes_per_frame", "l2_bytes_per_frame", "source", "how")}
    except (OSError, ValueError, KeyError):
        return None


def profile_traffic(kernel, cfg):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary"""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        e = d.get(cfg, {}).get(kernel) or d.get(cfg, {}).get("k_" + kernel)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


def launches_per_frame(caps, M, cra=False):
    """kernels one frame launches (engine.cu enqueue order, fused CR): per step 1
    step_begin + 2 decode (k_colA, k_rows1 decode fused with the setup's first row pass) +
    3 setup passes + cap x (5 apply passes + 1 fused CR recurrence) + 1 axpy; then 2
    decode + 1 image. With k_crA every recurrence but a step's last also runs the next
    application's W^-1 column pass (one launch fewer)"""
    n = 0
    for m in range(M):
        n += 1 + 2 + 3 + 6 * caps[m] + 1
        if cra and caps[m] > 1:
            n -= caps[m] - 1
    return n + 3


class profiled_step:
    """RTN_PROFILE_STEP=1 (RTN_PROFILE_E2E=1 for the e2e run): cudaProfilerStart/Stop around
    the timed step, so `ncu --profile-from-start off --metrics gpu__time_duration.sum ...`
    lists exactly the timed frames' kernels (a no-op otherwise)"""

    def __init__(self, var="RTN_PROFILE_STEP"):
        self.var = var

    def __enter__(self):
        self.rt = None
        if os.environ.get(self.var) == "1":
            import ctypes
            self.rt = ctypes.CDLL("libcudart.so.12")
            self.rt.cudaProfilerStart()
        return self

    def __exit__(self, *exc):
        if self.rt is not None:
            self.rt.cudaProfilerStop()
        return False


def launches_per_frame_group(caps, M, A, cluster=False):
    """kernels one frame launches on a channel group of A members (group.cu enqueue order,
    all members, budget mode): per step and member 1 step_begin + 2 decode (+ the setup's
    first row pass) + 2 setup passes + 1 k_rho_out + 1 k_colsW + 1 k_grp_fin + cap x (the
    application: 5 passes, or a cluster kernel + k_rho_sum, + k_cr_fused forming the group
    totals) + 1 closing k_grp_fin + 1 axpy; then per member 2 decode + 1 k_coil_ss, + 1
    k_image_grp"""
    per_it = 3 if cluster else 6
    n = 0
    for m in range(M):
        n += A * (1 + 2 + 2 + 1 + 1 + 1 + per_it * caps[m] + (1 if caps[m] else 0) + 1)
    return n + 3 * A + 1


def dist_setup(n_gpus, backend=None):
    """one process per GPU (torchrun env); NCCL on GPUs, gloo for the CPU tests"""
    rank, world, local = 0, 1, 0
    if "RANK" in os.environ and "WORLD_SIZE" in os.environ:
        rank = int(os.environ["RANK"])
        world = int(os.environ["WORLD_SIZE"])
        local = int(os.environ.get("LOCAL_RANK", rank))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        global _HOST_GROUP
        _HOST_GROUP = dist.new_group(backend="gloo")
    return rank, world, local


_HOST_GROUP = None


def host_barrier(world):
    """a barrier on the host (gloo over TCP): ranks that wait while rank 0 drives every GPU
    must not leave an NCCL kernel spinning on their device meanwhile"""
    if world > 1:
        import torch.distributed as dist
        dist.barrier(group=_HOST_GROUP)


def _dist_device(local):
    import torch
    import torch.distributed as dist
    return f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(v, world, local):
    """timings are reported as the max over ranks"""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=_dist_device(local))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world, local):
    if world > 1:
        import torch
        import torch.distributed as dist
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize(local)
        else:
            dist.barrier()


def weak_scaling_value(world, frames_per_rank, span_ms_max):
    """whole-job frames/s: every rank reconstructs its own slice series"""
    return world * frames_per_rank / (span_ms_max / 1000.0)


# ------------------------------------------------------------------------------------
# reference arm: the reference's own CPU path (oracle/_ref) on the same workload
# ------------------------------------------------------------------------------------
def host_info():
    """nproc and the CPU model of this host (state the cores the CPU arm had)"""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def reference_inputs(cfg, plan, F):
    """the reference's own pre stage (grid_adjoint per frame, build_psf per angle set,
    prep_series normalisation of frame 0) on the bench's raw acquisitions, outside any
    timed region"""
    from oracle import ref
    G, J, K, U, _ = CONFIGS[cfg]
    raw, angles = synth_raw(G, J, K, U, n_unique=U)
    P = np.stack([ref.build_psf(plan, angles[t], 2 * plan.N) for t in range(U)])
    zu = np.stack([ref.grid_adjoint(plan, raw[t], angles[t]) for t in range(U)])
    scale = np.float32(100.0 / math.sqrt(float(np.sum(np.abs(zu[0].astype(np.complex128)) ** 2))))
    z = np.stack([(zu[n % U] * scale).astype(np.complex64) for n in range(F)])
    return z, P, [n % U for n in range(F)]


def reference_arm(args, cfg):
    """BASELINE.md CPU-baseline plan: the reference's scheduled series driver
    (reconstruct_series, nlinv.cpp:446-526, with TemporalSchedule::for_turns(U) like our
    arm) on this host. (T, A) comes from the reference's own autotuner (learn_step /
    select_config, autotune.cpp:40-88) over legal_configs(nproc), pruned for time to the
    A = min(4, nproc) row with T <= 4 (the schedule keeps at most o + 1 = 4 frames
    progressing, so more threads only wait), each candidate timed on 2T frames past the
    strict prefix; plus T = 1, A = 1 (reconstruct_series_plain on one core) for reference."""
    G, J, K, U, _ = CONFIGS[cfg]
    from oracle import ref
    import paper_1701_08361_b200 as pb
    plan = pb.raw_plan(G, J)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    host = host_info()
    nproc = host["nproc"]
    sched = tuple(int(v) for v in args.sched.split(",")) if args.sched else (U, (U + 1) // 2)
    A = max(1, min(4, nproc, J))
    cands = [(T, A) for T in range(1, 5) if T * A <= nproc] or [(1, 1)]
    pre = sched[0] + 1  # the strict prefix (frames 1..l wait for n-1) plus frame 0
    F = pre + sum(2 * T for T, _ in cands) + 1 + args.warmup + args.steps
    z, P, idx = reference_inputs(cfg, plan, F)
    D = plan.D
    ests = np.zeros((F, D), np.complex64)
    # the strict prefix once (its frames run one after another whatever T is)
    _, _, _, e = ref.time_series(plan, z[:pre], P, idx[:pre], 1, A, sched)
    ests[:pre] = e
    first = pre
    key = (0, plan.N, 2, J)  # single_slice, N, frames bucket, J (autotune.hpp:13-31)
    db, sweep = [], {}
    for T, A_ in cands:
        cnt = 2 * T
        w, lat, cg, e = ref.time_series(plan, z[:first + cnt], P, idx[:first + cnt], T, A_, sched, first=first,
                                        ests=ests[:first + cnt])
        ests[:first + cnt] = e
        first += cnt
        ms = 1000.0 * w / cnt
        db.append(key + (T, A_, ms))
        sweep[f"T{T}xA{A_}"] = round(1000.0 / ms, 4)
    T_best, A_best = ref.select_config(key, db)  # exact-key argmin (autotune.cpp:15-38)
    # single core, one frame (reconstruct_series_plain with A = 1)
    w1, _, _, e = ref.time_series(plan, z[:first + 1], P, idx[:first + 1], 1, 1, sched, first=first,
                                  ests=ests[:first + 1])
    ests[:first + 1] = e
    first += 1
    single = 1.0 / w1
    # timed: warm-up, then args.steps frames with the selected configuration
    if args.warmup:
        _, _, _, e = ref.time_series(plan, z[:first + args.warmup], P, idx[:first + args.warmup], T_best, A_best,
                                     sched, first=first, ests=ests[:first + args.warmup])
        ests[:first + args.warmup] = e
        first += args.warmup
    w, lat, cg, _ = ref.time_series(plan, z[:first + args.steps], P, idx[:first + args.steps], T_best, A_best,
                                    sched, first=first, ests=ests[:first + args.steps])
    assert int(cg.sum()) == 50 * args.steps
    fps = args.steps / w
    sample = (f"{args.steps} chained {cfg.upper()} frames (7 Newton steps, 50 CR iterations each) through the "
              f"reference's scheduled series driver (reconstruct_series loop, for_turns({U})) with T={T_best} "
              f"threads x A={A_best} WorkerGroup lanes, after {args.warmup} warm-up frames; (T, A) = "
              f"select_config over the sweep {sweep} (frames/s; candidates: the A={A} row of legal_configs({nproc}) with T<=4, 2T frames "
              f"each); single core (T=1, A=1): {single:.3f} frames/s; gridding and PSFs outside the timed region; "
              f"FFTW replaced by the oracle shim FFT (oracle/shim, pocketfft-class speed)")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * w / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c64/f64", "data": "synthetic",
        "config": {"workload": cfg, "description": CONFIGS[cfg][4], "G": G, "J": J, "newton_steps": 7,
                   "cg_iter_budget": 50, "frames_in_flight": T_best, "channel_group": A_best,
                   "temporal_schedule": {"l": sched[0], "o": sched[1]}},
        "p50_latency_ms": 1000.0 * float(np.median(lat)),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": T_best * A_best, "kind": "reference",
                         "sample": sample, "host": host, "sweep_frames_per_s": sweep,
                         "single_core_frames_per_s": single, "selected": {"T": T_best, "A": A_best}},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, z, P, plan):
    """bounded sample of the reference CPU path on this host (rank 0, N = 1)"""
    from oracle import ref
    nproc = os.cpu_count() or 1
    A = max(1, min(4, nproc, plan.J))
    est = ref.initial_estimate(plan)
    t0 = time.perf_counter()
    ref.reconstruct_frame(plan, z, P, est, est, A=A)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "frames/s", "cores": A, "kind": "reference", "host": host_info(),
            "sample": f"1 {cfg.upper()} frame (7 Newton steps, 50 CR iterations) through the reference "
                      f"reconstruct_frame with A={A} WorkerGroup lanes, {dt:.1f} s; FFTW replaced by the "
                      f"oracle shim FFT; the scheduled (T, A) figure is the --impl reference arm's"}


def check_timed_frames(pb, series, plan, frames, P, U, audit, first, n_check):
    """Parity of the headline frames themselves (outside the timed region): each checked
    frame of the timed run is replayed through the reference's reconstruct_frame with a
    per-step RegProvider (nlinv.cpp:286-335) fed the device estimates of the sources its
    audit recorded, and the device image / estimate must match within the north-star
    frame tolerance (1e-3 relative L2), the CR iteration split exactly."""
    from oracle import ref
    scale = series.normalize()
    lanes = max(1, min(4, os.cpu_count() or 1))
    unity = pb.initial_estimate(plan)
    M = plan.newton_steps
    rows = []
    for k in range(n_check):
        n = first + k
        a = audit[k]
        src = lambda f: unity if f < 0 else series.estimate(f)  # noqa: E731
        init = src(a.init_src)
        regs = [src(a.reg_src[m]) if a.init_src >= 0 else unity for m in range(M)]
        z = (frames[n] * np.float32(scale)).astype(np.complex64)
        img, est, per = ref.reconstruct_frame_regs(plan, z, P[n % U], init, regs, A=lanes)
        img = img * np.float32(1.0 / scale)
        got_img = series.images(n, 1)[0]
        got_est = series.estimate(n)

        def rel(g, w):
            g = np.asarray(g, np.complex128).ravel()
            w = np.asarray(w, np.complex128).ravel()
            return float(np.linalg.norm(g - w) / np.linalg.norm(w))

        rows.append({"frame": n, "init_src": a.init_src, "reg_src": a.reg_src, "image_rel_err": rel(got_img, img),
                     "estimate_rel_err": rel(got_est, est), "cg_per_step_ref": per})
    worst = max(max(r["image_rel_err"], r["estimate_rel_err"]) for r in rows)
    return {"frames": rows, "max_rel_err": worst, "tolerance": 1e-3, "pass": worst < 1e-3,
            "oracle": "oracle/_ref reconstruct_frame with the audited per-step sources (device estimates)"}


def e2e_raw(pb, make_series, plan, opts, cfg, F, S, world, local):
    """frames/s end to end through the public series call: raw acquisitions (J x K x S
    samples per frame) from pinned host memory through rtn_series_run_raw -- H2D, device
    pre stage (gridding, cached PSFs, normalisation), reconstruction, images D2H to pinned
    host -- all inside the timed region (wall clock, max over ranks). world = the ranks
    that call it together (each its own series: weak scaling); a single series over
    several GPUs is called on rank 0 alone with world = 1"""
    import torch
    G, J, K, U, _ = CONFIGS[cfg]
    raw, angles = synth_raw(G, J, K, U, n_unique=U)
    Ssp = raw.shape[-1]
    FR = F + S  # one more range of S frames: the untimed e2e warm-up range
    rt = torch.empty((FR, J, K, Ssp), dtype=torch.complex64, pin_memory=True)
    rt.numpy()[:] = np.stack([raw[n % U] for n in range(FR)])
    ang = np.stack([angles[n % U] for n in range(FR)])
    imt = torch.empty((FR, plan.N, plan.N), dtype=torch.complex64, pin_memory=True)
    fb = rt[0].numel() * 8  # bytes of one raw frame
    ib = plan.N * plan.N * 8
    rs = make_series(FR)  # its own store and PSF cache
    # frames [0, F - S) prime the chain, the normalisation scale, the PSF cache and the
    # grid plans; the next S frames are the untimed e2e warm-up; the S after them are timed
    T0 = F - S
    rs.run(opts, first=0, count=T0, raw=dict(samples_ptr=rt.data_ptr(), S=Ssp, angles=ang[:T0]),
           images_ptr=imt.data_ptr())
    rs.run(opts, first=T0, count=S, raw=dict(samples_ptr=rt.data_ptr() + T0 * fb, S=Ssp, angles=ang[T0:T0 + S]),
           images_ptr=imt.data_ptr() + T0 * ib)
    T0 += S
    raw_in = dict(samples_ptr=rt.data_ptr() + T0 * fb, S=Ssp, angles=ang[T0:T0 + S])
    barrier(world, local)
    with profiled_step("RTN_PROFILE_E2E"):
        t0 = time.perf_counter()
        rs.run(opts, first=T0, count=S, raw=raw_in, images_ptr=imt.data_ptr() + T0 * ib)
        wall = time.perf_counter() - t0
    print(f"[bench] e2e wall {wall * 1e3:.1f} ms, device span {rs.last_span_ms():.1f} ms", file=sys.stderr,
          flush=True)
    barrier(world, local)
    wall = max_over_ranks(wall, world, local)
    rs.close()
    return {"value": world * S / wall, "unit": "frames/s",
            "h2d_bytes_per_step": J * K * Ssp * 8, "d2h_bytes_per_step": plan.N * plan.N * 8,
            "path": "rtn_series_run_raw: pinned raw samples H2D on the copy stream, device gridding + "
                    "cached PSFs + normalisation, reconstruction, images D2H to pinned host (wall clock)"}


def single_series_multi_gpu(pb, plan, frames, P, U, sched, ngpu, cfg, W, S, with_e2e):
    """The N > 1 headline: ONE acquisition (one frame series) reconstructed by all ngpu GPUs
    of the node under the paper's decompositions -- channel groups over NVLink peer memory,
    temporal decomposition, and the hybrid the autotuner picks (autotune.cpp:49-88 over
    legal_configs) -- driven from rank 0 in one process (the reference's thread-per-worker
    model; worker t's members on devices (t*A + k) % ngpu). Device time (CUDA events
    spanning every worker stream) for the fps and p50 latency of each decomposition; the
    selected hybrid is then timed on S frames (the headline, strong scaling) and end to end
    through rtn_series_run_raw on the same devices."""
    nvis = pb.load_library().rtn_device_count()
    devices = [k % nvis for k in range(ngpu)]
    F = frames.shape[0]
    s = pb.Series(pb.Context(plan, device=0), F, U, devices=devices)
    s.upload_frames(frames)
    for k in range(U):
        s.upload_psf(k, P[k])
    s.set_psf_index([n % U for n in range(F)])
    s.normalize()
    nw, nt = W, min(16, max(F - W - S, 4))

    def opts(T, A):
        return pb.SeriesOptions(T=T, A=A, plain=(T == 1), sched=sched)

    def measure(T, A):
        s.run(opts(T, A), first=0, count=nw, want_images=False)
        out = s.run(opts(T, A), first=nw, count=nt, want_images=False)
        ms = s.last_span_ms() / nt
        return {"T": T, "A": A, "frames_per_s": 1000.0 / ms, "ms_per_frame": ms,
                "p50_latency_ms": statistics.median(float(v) for v in out["gpu_ms"])}

    res = {"gpus": ngpu, "single_gpu_plain": measure(1, 1), "channel": measure(1, min(ngpu, 8)),
           "temporal": measure(ngpu, 1)}
    key = (pb.ImagingMode.single_slice, plan.N, pb.frames_bucket(S), plan.J)
    db = []
    slots = max(6, ngpu)  # worker slots: as on one GPU, several frames may share a device
    for _ in pb.legal_configs(slots, a_cap=8):
        T, A = pb.learn_step(key, db, slots, 8)
        db.append(key + (T, A, measure(T, A)["ms_per_frame"]))
    T, A = pb.select_config(key, db)
    res["autotuned_hybrid"] = measure(T, A)
    res["tuned_space_ms_per_frame"] = {f"T{r[4]}xA{r[5]}": round(r[6], 3) for r in db}
    # the headline: the selected hybrid on the S frames after the warm-up and tuning ranges
    o = opts(T, A)
    s.run(o, first=0, count=nw, want_images=False)
    with ClockSampler(0) as clk:
        out = s.run(o, first=F - S, count=S, want_images=False)
        span_ms = s.last_span_ms()
    lat = [float(v) for v in out["gpu_ms"]]
    head = {"T": T, "A": A, "span_ms": span_ms, "lat": lat, "clocks": clk.summary(), "decompositions": res,
            "cg_iters": [int(v) for v in out["cg_iters"]]}
    s.close()
    if with_e2e:
        head["e2e"] = e2e_raw(pb, lambda n: pb.Series(pb.Context(plan, device=0), n, U, devices=devices), plan, o,
                              cfg, F, S, 1, 0)
    return head


def channel_processes(pb, plan, frames, P, world, rank, local, S):
    """frames/s of one frame sequence reconstructed by all ranks as one channel group"""
    # every rank must have its member before any enters the device-side barriers (a
    # missing member would otherwise only surface at the barrier deadline)
    ctx, err = None, ""
    try:
        ctx = pb.Context(plan, device=local, member=(rank, world), a_cap=8)
        pb.connect_members(ctx)
    except Exception as e:
        err = str(e)
    if max_over_ranks(1.0 if err else 0.0, world, local) > 0:
        if ctx is not None:
            ctx.close()
        raise RuntimeError("process-group setup failed on some rank" + (f": {err}" if err else ""))
    z = frames[0]
    nsq = float(np.sum(np.abs(z.astype(np.complex128)) ** 2))
    z = (z * np.float32(100.0 / math.sqrt(nsq))).astype(np.complex64)
    ctx.set_psf(P[0])
    ctx.set_data(z)
    est = pb.initial_estimate(plan)
    for _ in range(2):
        est = ctx.reconstruct_frame(est, est).est
    barrier(world, local)
    t0 = time.perf_counter()
    for _ in range(S):
        est = ctx.reconstruct_frame(est, est).est
    wall = max_over_ranks(time.perf_counter() - t0, world, local)
    ctx.close()
    return {"members": world, "frames_per_s": S / wall, "ms_per_frame": 1000.0 * wall / S,
            "path": "rtn_reconstruct_frame per frame (host in / out), chained, wall clock, max over ranks"}


# ------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--T", default="auto",
                    help="frames in flight (temporal decomposition): 1 = plain chain, N, or auto = autotuner")
    ap.add_argument("--A", default="1", help="channel-group width per frame worker (with --T N)")
    ap.add_argument("--sched", default=None,
                    help="temporal schedule 'l,o' (decomp.hpp:70-76); default for_turns(U) = (U, ceil(U/2)); "
                         "C4's relaxed t-k schedule with 8 frames in flight: --config c4 --T 8 --sched 5,8")
    ap.add_argument("--tune-db", default=os.path.join(ROOT, "profiles", "tune_db.tsv"),
                    help="autotuner store (autotune.hpp TuneDb format)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-check", action="store_true",
                    help="skip the parity check of the first two timed frames against the reference")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = args.config

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            reference_arm(args, cfg)
        return

    rank, world, local = dist_setup(args.gpus)
    import paper_1701_08361_b200 as pb
    G, J, K, U, desc = CONFIGS[cfg]
    plan = pb.raw_plan(G, J)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    M = plan.newton_steps
    W, S = args.warmup, args.steps
    NTUNE = 16 if args.T == "auto" else 0  # frames per autotune candidate, past the strict prefix
    F = W + NTUNE + S

    z_unique, P = synth_series(G, J, K, U, n_unique=min(F, 10), seed=1234 + rank)
    ctx = pb.Context(plan, device=local)
    series = pb.Series(ctx, F, U)
    frames = np.stack([z_unique[n % len(z_unique)] for n in range(F)])
    series.upload_frames(frames)
    for k in range(U):
        series.upload_psf(k, P[k])
    series.set_psf_index([n % U for n in range(F)])
    series.normalize()
    sched = pb.TemporalSchedule.for_turns(U)
    if args.sched:
        l_, o_ = (int(v) for v in args.sched.split(","))
        sched = pb.TemporalSchedule(l_, o_)

    def opts_for(T, A=1):
        return pb.SeriesOptions(T=T, A=A, plain=(T == 1), sched=sched)

    # warm-up (graph capture happens here)
    series.run(opts_for(1), first=0, count=W, want_images=False)
    tuning = None
    if args.T == "auto":
        # the paper's (T, A) autotuner (autotune.cpp:49-88): learn_step walks the legal
        # hybrid space T x A <= 6 (T frames in flight, each a channel group of A members
        # on separate streams of this device), each candidate measured on NTUNE frames
        # (device time), then select_config picks the best recorded configuration for
        # this protocol key
        key = (pb.ImagingMode.single_slice, plan.N, pb.frames_bucket(S), J)
        db = []
        space = [c for c in pb.legal_configs(6, a_cap=4)]
        for _ in space:
            T_try, A_try = pb.learn_step(key, db, 6, 4)
            # graph capture on every worker (frame n runs on worker n mod T)
            series.run(opts_for(T_try, A_try), first=W, count=T_try + 1, want_images=False)
            series.run(opts_for(T_try, A_try), first=W, count=NTUNE, want_images=False)
            ms = series.last_span_ms() / NTUNE
            db.append(key + (T_try, A_try, ms))
        T_sel, A_sel = pb.select_config(key, db)
        tuning = {"key": {"mode": "single_slice", "N": plan.N, "bucket": pb.frames_bucket(S), "J": J},
                  "measured_ms_per_frame": {f"T{r[4]}xA{r[5]}": round(r[6], 3) for r in db},
                  "selected": {"T": T_sel, "A": A_sel}}
        if rank == 0 and args.tune_db:
            try:
                tdb = pb.TuneDb(args.tune_db)
                for r in db:
                    tdb.append(r[:6], r[6], int(time.time()))
            except Exception:
                pass
        T, A = T_sel, A_sel
        series.run(opts_for(T, A), first=W, count=NTUNE, want_images=False)  # warm the selected config
    else:
        T, A = int(args.T), int(args.A)
        # graph capture on every worker of the requested configuration, outside the timed region
        series.run(opts_for(T, A), first=0, count=min(F, max(W, 2 * T)), want_images=False)
    opts = opts_for(T, A)
    barrier(world, local)
    with ClockSampler(local) as clk, profiled_step():
        out = series.run(opts, first=W + NTUNE, count=S, want_images=False)
        span_ms = series.last_span_ms()
    barrier(world, local)
    span_ms = max_over_ranks(span_ms, world, local)
    value = weak_scaling_value(world, S, span_ms)
    lat = [float(v) for v in out["gpu_ms"]]
    caps = [0] * M
    rem = plan.cg_iter_budget
    for m in range(M):
        caps[m] = (rem + (M - m) - 1) // (M - m)
        rem -= caps[m]
    assert list(out["cg_iters"]) == [sum(caps)] * S

    # the headline frames checked against the reference (after the timed region)
    check = None
    if rank == 0 and world == 1 and not args.no_check:
        try:
            check = check_timed_frames(pb, series, plan, frames, P, U, out["audit"], W + NTUNE, min(2, S))
        except Exception as e:  # reported; the oracle may be absent on a stripped box
            check = {"error": str(e)}

    # end to end: pinned host frames streamed through the public series call
    e2e = None
    if not args.no_e2e:
        e2e = e2e_raw(pb, lambda n: pb.Series(ctx, n, U), plan, opts, cfg, F, S, world, local)

    # roofline of the dominant kernel (isolated CUDA-event timing on the engine stream)
    peak, peak_kind = measured_peaks()
    ctx.make_step_cache(series.estimate(F - 1))
    napply = sum(caps) + M  # CR applications + Newton-step setups per frame
    # throughput mode runs the five-kernel passes; with k_crA every recurrence but a step's
    # last also does the next application's W^-1 column pass
    fused = sum(max(c - 1, 0) for c in caps) if ctx.fused_cra() else 0
    per_frame = {"colsT": napply, "rows1": napply, "rows2": napply, "colA": napply - fused, "colsW": napply,
                 "cr_fused": sum(caps) - fused}
    if fused:
        per_frame["crA"] = fused
    kern = {}
    for name in per_frame:
        ms, by = ctx.time_kernel(name, 50)
        cold_ms, _ = ctx.time_kernel(name + ":cold", 20)
        kern[name] = {"ms": ms, "ms_cold": cold_ms, "bytes": by, "launches_per_frame": per_frame[name],
                      "share_ms_per_frame": ms * per_frame[name]}
    dom = max(kern, key=lambda k: kern[k]["share_ms_per_frame"])
    achieved = kern[dom]["bytes"] / (kern[dom]["ms"] / 1000.0) / 1e9
    achieved_cold = kern[dom]["bytes"] / (kern[dom]["ms_cold"] / 1000.0) / 1e9
    app_ms, app_by = ctx.time_kernel("apply", 20)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": profile_traffic(dom, cfg), "peak_source": peak_kind,
                "cache": "l2_warm: back-to-back launches on the L2-resident operands of one iteration, "
                         "as in the step (its ~60 MB working set stays in the 126 MB L2)",
                "cold": {"achieved": achieved_cold, "frac": achieved_cold / peak, "kernel_ms": kern[dom]["ms_cold"],
                         "how": "each launch timed alone after a 256 MiB write (L2 flushed)"},
                "kernel_ms": kern[dom]["ms"], "algorithmic_bytes_per_launch": kern[dom]["bytes"],
                "step_traffic": step_traffic(cfg),
                "apply": {"ms": app_ms, "algorithmic_bytes": app_by,
                          "achieved_gbs": app_by / (app_ms / 1000.0) / 1e9},
                "kernels": kern}

    # latency mode: one frame at a time (T = 1) through the cluster-fused applications,
    # the paper's per-frame latency figure (device time per frame)
    latency_mode = None
    try:
        lo = pb.SeriesOptions(T=1, plain=True, sched=sched)
        series.run(lo, first=0, count=W, want_images=False)  # graph capture for the cluster path
        lout = series.run(lo, first=W + NTUNE, count=S, want_images=False)
        lat_span = series.last_span_ms()
        latency_mode = {"frames_in_flight": 1, "cluster_fused": ctx.cluster_supported(),
                        "frames_per_s": S / (lat_span / 1000.0),
                        "p50_latency_ms": statistics.median(float(v) for v in lout["gpu_ms"])}
    except Exception as e:  # reported, never fatal
        latency_mode = {"error": str(e)}

    single = None
    if world > 1:
        # the N > 1 headline: one acquisition over all the node's GPUs under the autotuned
        # channel x temporal decomposition, driven from rank 0 in one process (the
        # reference's thread-per-worker model); the other ranks hold their GPUs idle
        # meanwhile. The per-rank slice series above stay as the multi-slice figure.
        barrier(world, local)
        if rank == 0:
            try:
                single = single_series_multi_gpu(pb, plan, frames, P, U, sched, world, cfg, W, S,
                                                 with_e2e=not args.no_e2e)
            except Exception as e:  # reported; the headline then stays the multi-slice figure
                single = {"error": str(e)}
        host_barrier(world)  # the other ranks wait on the host: their GPUs are rank 0's now
        barrier(world, local)
        # the same channel decomposition with one process per GPU: every rank is one
        # member (CUDA IPC views of the peers, device-side barriers), one chained frame
        # sequence for the whole job (strong scaling), host in / host out per frame
        try:
            procs = channel_processes(pb, plan, frames, P, world, rank, local, S)
        except Exception as e:
            procs = {"error": str(e)}
        if rank == 0:
            single["channel_processes"] = procs

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": S, "warmup": W,
        # one acquisition (a fixed frame series) whatever N: at N > 1 all GPUs share it
        "ms_per_step": span_ms / S, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c64 (fp32 arithmetic, fp64 reductions)",
        "data": "synthetic (numpy phantom, coils, exact radial Toeplitz kernel; staged in HBM)",
        "config": {"workload": cfg, "description": desc, "G": G, "N": plan.N, "Gc": plan.Gc, "J": J,
                   "spokes": K, "turns": U, "newton_steps": M, "cg_iter_budget": plan.cg_iter_budget,
                   "frames_in_flight": T, "channel_group": A, "temporal_schedule": {"l": sched.l, "o": sched.o},
                   "per_rank": "one frame series (one acquisition) per GPU",
                   "l2": "inputs larger than L2: every frame has its own 16 MB buffer, "
                         f"{F} frames staged ({F * J * G * G * 8 / 2**20:.0f} MiB)"},
        "p50_latency_ms": statistics.median(lat), "latency_ms_min_max": [min(lat), max(lat)],
        "e2e": e2e, "gpu_launches": launches_per_frame(caps, M, ctx.fused_cra() and T > 1) * S, "roofline": roofline, "autotune": tuning,
        "clocks": clk.summary(),
        "latency_mode": latency_mode,
        "check": check,
    }
    if single is not None:
        multi_slice = {"value": value, "ms_per_step": span_ms / S, "scaling": "weak", "e2e": e2e,
                       "frames_in_flight": T, "channel_group": A,
                       "per_rank": "independent slice series (multi-slice acquisition), one per GPU"}
        line["multi_slice"] = multi_slice
        if "error" in single:  # the headline falls back to the per-rank slice series
            line["single_series_error"] = single["error"]
            line["scaling"] = "weak"
            line["config"]["per_rank"] = "independent slice series (multi-slice)"
            line["decompositions"] = {"channel_processes": single.get("channel_processes")}
        else:
            Ts, As = single["T"], single["A"]
            line.update({
                "value": S / (single["span_ms"] / 1000.0), "ms_per_step": single["span_ms"] / S, "scaling": "strong",
                "p50_latency_ms": statistics.median(single["lat"]),
                "latency_ms_min_max": [min(single["lat"]), max(single["lat"])],
                "e2e": single.get("e2e"), "clocks": single["clocks"],
                "gpu_launches": (launches_per_frame(caps, M, ctx.fused_cra() and Ts > 1) if As == 1
                                 else launches_per_frame_group(caps, M, As, cluster=Ts == 1)) * S,
                "decompositions": dict(single["decompositions"], channel_processes=single.get("channel_processes")),
            })
            line["config"].update({"frames_in_flight": Ts, "channel_group": As,
                                   "per_rank": "one frame series over all GPUs (rank 0 drives every device)"})
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, frames[0] * np.float32(100.0 / math.sqrt(
                float(np.sum(np.abs(frames[0].astype(np.complex128)) ** 2)))), P[0], plan)
        except Exception as e:  # the oracle may be absent on a stripped box
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
