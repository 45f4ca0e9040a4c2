"""The bench's e2e pattern in isolation: prime frames [0, T0) from raw samples, then
time frames [T0, T0 + S) (wall clock and device span)."""
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
T0, S = 13, 20
NR = 3  # consecutive new frame ranges
F = T0 + NR * S
raw, angles = bench.synth_raw(G, J, K, U, U)
Ssp = raw.shape[-1]
rt = torch.empty((F, J, K, Ssp), dtype=torch.complex64, pin_memory=True)
rt.numpy()[:] = np.stack([raw[n % U] for n in range(F)])
ang = np.stack([angles[n % U] for n in range(F)])
imt = torch.empty((F, plan.N, plan.N), dtype=torch.complex64, pin_memory=True)
fb = rt[0].numel() * 8
ctx = pb.Context(plan)
for T in (1, 3):
    rs = pb.Series(ctx, F, U)
    o = pb.SeriesOptions(T=T, plain=(T == 1), sched=pb.TemporalSchedule.for_turns(U))
    rs.run(o, first=0, count=T0, raw=dict(samples_ptr=rt.data_ptr(), S=Ssp, angles=ang[:T0]), images_ptr=imt.data_ptr())
    for rep in range(NR + 1):
        f0 = T0 + min(rep, NR - 1) * S
        t0 = time.perf_counter()
        rs.run(o, first=f0, count=S, raw=dict(samples_ptr=rt.data_ptr() + f0 * fb, S=Ssp, angles=ang[f0:f0 + S]),
               images_ptr=imt.data_ptr() + f0 * plan.N * plan.N * 8)
        wall = time.perf_counter() - t0
        print(f"T={T} range {min(rep, NR - 1)}: wall {wall*1e3:.1f} ms ({S/wall:.0f} fps), span {rs.last_span_ms():.1f} ms", flush=True)
    del rs
