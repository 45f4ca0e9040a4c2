"""Probe (T, A) decompositions of the C3 series on the visible GPUs (device time per
frame and p50 frame latency). A members share a GPU when fewer GPUs are visible."""
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
pairs = [tuple(int(v) for v in p.split("x")) for p in (sys.argv[2:] or ["1x1", "1x2", "1x4", "2x2", "3x1", "3x2"])]
G, J, K, U, _ = bench.CONFIGS[cfg]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
F = 24
z, P = bench.synth_series(G, J, K, U, n_unique=8)
ctx = pb.Context(plan)
ndev = pb.load_library().rtn_device_count()
s = pb.Series(ctx, F, U, devices=list(range(ndev)))
s.upload_frames(np.stack([z[n % len(z)] for n in range(F)]))
for k in range(U):
    s.upload_psf(k, P[k])
s.set_psf_index([n % U for n in range(F)])
s.normalize()
sched = pb.TemporalSchedule.for_turns(U)
if os.environ.get("RTN_SCHED"):  # "l,o" override of the reference default for_turns(U)
    sched = pb.TemporalSchedule(*[int(v) for v in os.environ["RTN_SCHED"].split(",")])
for T, A in pairs:
    o = pb.SeriesOptions(T=T, A=A, plain=(T == 1), sched=sched)
    if os.environ.get("RTN_SERIES_CLUSTER"):  # 1 / 0: force the cluster-fused applications on / off
        o.cluster = int(os.environ["RTN_SERIES_CLUSTER"])
    s.run(o, first=0, count=8, want_images=False)
    out = s.run(o, first=8, count=16, want_images=False)
    ms = s.last_span_ms() / 16
    print(f"T={T} A={A}: {ms:.3f} ms/frame ({1000/ms:.0f} fps), p50 latency {statistics.median(out['gpu_ms']):.3f} ms",
          flush=True)
