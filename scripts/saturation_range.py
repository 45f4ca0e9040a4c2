"""One saturated window for ncu range profiling: K independent C3 plain series (the
slices of scripts/slices_probe.py) run concurrently between cudaProfilerStart/Stop, so
`ncu --replay-mode app-range --profile-from-start off` reports whole-GPU throughput
metrics while kernels of different frames overlap (per-kernel ncu serialises them)."""
import ctypes
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402

nsl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
F = int(sys.argv[2]) if len(sys.argv) > 2 else 6
G, J, K, U, _ = bench.CONFIGS["c3"]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
z, P = bench.synth_series(G, J, K, U, n_unique=4)
series = []
for k in range(nsl):
    ctx = pb.Context(plan)
    s = pb.Series(ctx, F, U)
    s.upload_frames(np.stack([z[n % 4] for n in range(F)]))
    for u in range(U):
        s.upload_psf(u, P[u])
    s.set_psf_index([n % U for n in range(F)])
    s.normalize()
    s.run(pb.SeriesOptions(plain=True), want_images=False)
    series.append((ctx, s))
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else ctypes.CDLL("libcudart.so")
th = [threading.Thread(target=lambda s=s: s.run(pb.SeriesOptions(plain=True), want_images=False)) for _, s in series]
rt.cudaProfilerStart()
for t in th:
    t.start()
for t in th:
    t.join()
rt.cudaProfilerStop()
print(f"{nsl} slices x {F} frames done", flush=True)
