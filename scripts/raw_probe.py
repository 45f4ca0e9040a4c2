"""Raw-acquisition series vs resident series: wall clock and device span (C3)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402
import torch  # noqa: E402

G, J, K, U, _ = bench.CONFIGS["c3"]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
S = 20
raw, angles = bench.synth_raw(G, J, K, U, U)
rt = torch.empty((S, J, K, raw.shape[-1]), dtype=torch.complex64, pin_memory=True)
rt.numpy()[:] = np.stack([raw[n % U] for n in range(S)])
ang = np.stack([angles[n % U] for n in range(S)])
imt = torch.empty((S, plan.N, plan.N), dtype=torch.complex64, pin_memory=True)
ctx = pb.Context(plan)
s = pb.Series(ctx, S, U)
sched = pb.TemporalSchedule.for_turns(U)
for T in (1, 3):
    o = pb.SeriesOptions(T=T, plain=(T == 1), sched=sched)
    raw_in = dict(samples_ptr=rt.data_ptr(), S=raw.shape[-1], angles=ang)
    s.run(o, raw=raw_in, images_ptr=imt.data_ptr())
    for _ in range(2):
        t0 = time.perf_counter()
        s.run(o, raw=raw_in, images_ptr=imt.data_ptr())
        wall = time.perf_counter() - t0
        print(f"raw T={T}: wall {wall*1e3:.1f} ms ({S/wall:.0f} fps), device span {s.last_span_ms():.1f} ms", flush=True)
    s.run(o, want_images=False)
    t0 = time.perf_counter()
    s.run(o, want_images=False)
    wall = time.perf_counter() - t0
    print(f"resident T={T}: wall {wall*1e3:.1f} ms, device span {s.last_span_ms():.1f} ms", flush=True)
