"""The bench's timed step as one ncu range: a C3-style series at the bench's (T, schedule)
runs S frames between cudaProfilerStart/Stop, so
  ncu --replay-mode app-range --profile-from-start off --metrics dram__bytes_read.sum,...
reports the whole-GPU DRAM traffic of S frames with the kernels of the frames in flight
overlapping as in the bench (per-kernel ncu serialises them and flushes caches).
usage: python scripts/step_range.py [cfg] [T] [S]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S = int(sys.argv[3]) if len(sys.argv) > 3 else 8
G, J, K, U, _ = bench.CONFIGS[cfg]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
W = 8
F = W + S
z, P = bench.synth_series(G, J, K, U, n_unique=min(F, 10))
ctx = pb.Context(plan)
s = pb.Series(ctx, F, U)
s.upload_frames(np.stack([z[n % len(z)] for n in range(F)]))
for u in range(U):
    s.upload_psf(u, P[u])
s.set_psf_index([n % U for n in range(F)])
s.normalize()
o = pb.SeriesOptions(T=T, plain=(T == 1), sched=pb.TemporalSchedule.for_turns(U))
s.run(o, first=0, count=W, want_images=False)  # graph capture on every worker
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaProfilerStart()
s.run(o, first=W, count=S, want_images=False)
rt.cudaProfilerStop()
print(f"{cfg} T={T}: {S} frames, {s.last_span_ms() / S:.3f} ms/frame", flush=True)
