"""Launch each hot-path kernel class a few times at a C3 linearisation point (eager
launches on the engine stream) — the target for `ncu --set full`. The launches sit
between cudaProfilerStart/Stop, so `ncu --profile-from-start off` skips the frame
reconstruction that builds the linearisation point."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
names = sys.argv[2:] or ["colA", "rows1", "colsT", "rows2", "colsW", "cr_fused"]
G, J, K, U, _ = bench.CONFIGS[cfg]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
z, P = bench.synth_series(G, J, K, U, n_unique=1)
with pb.Context(plan) as ctx:
    ctx.set_psf(P[0])
    ctx.set_data(z[0])
    fr = ctx.reconstruct_frame(pb.initial_estimate(plan))
    ctx.make_step_cache(fr.est)
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaProfilerStart()
    for n in names:
        ms, by = ctx.time_kernel(n, int(os.environ.get("REPS", "50")))
        print(f"{n}: {ms * 1000:.1f} us, {by / 1e6:.2f} MB algorithmic, {by / ms / 1e6:.0f} GB/s", flush=True)
    rt.cudaProfilerStop()
