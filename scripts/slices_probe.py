"""K independent plain series (multi-slice, no temporal chain) run concurrently from K
host threads on one GPU: aggregate frames/s. Separates GPU saturation from the
temporal decomposition's closing-step chain."""
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402

G, J, K, U, _ = bench.CONFIGS["c3"]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
F = 16
z, P = bench.synth_series(G, J, K, U, n_unique=4)
# RTN_SLICE_CLUSTER: -1 auto (clusters at T = 1), 0 five-kernel passes, 1 clusters
cl = int(os.environ.get("RTN_SLICE_CLUSTER", "-1"))
for nsl in [int(a) for a in (sys.argv[1:] or ["1", "2", "3", "4"])]:
    series = []
    for k in range(nsl):
        ctx = pb.Context(plan)
        s = pb.Series(ctx, F, U)
        s.upload_frames(np.stack([z[n % 4] for n in range(F)]))
        for u in range(U):
            s.upload_psf(u, P[u])
        s.set_psf_index([n % U for n in range(F)])
        s.normalize()
        s.run(pb.SeriesOptions(plain=True, cluster=cl), want_images=False)
        series.append((ctx, s))
    def go(s):
        s.run(pb.SeriesOptions(plain=True, cluster=cl), want_images=False)
    th = [threading.Thread(target=go, args=(s,)) for _, s in series]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.perf_counter() - t0
    for ctx, s in series:
        ctx.close()
    print(f"{nsl} slices: {nsl * F / dt:.0f} frames/s aggregate ({dt * 1000 / (nsl * F):.3f} ms/frame)", flush=True)
