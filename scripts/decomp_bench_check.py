"""The bench's N > 1 headline path (one series over ngpu devices, autotuned hybrid,
timed frames and e2e) on the visible GPUs; with one GPU every 'device' is GPU 0."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
ngpu = int(sys.argv[2]) if len(sys.argv) > 2 else 2
G, J, K, U, _ = bench.CONFIGS[cfg]
plan = pb.raw_plan(G, J)
plan.newton_steps, plan.cg_iter_budget = 7, 50
z, P = bench.synth_series(G, J, K, U, n_unique=6)
W, S = 5, 10
frames = np.stack([z[n % 6] for n in range(W + 16 + S)])
head = bench.single_series_multi_gpu(pb, plan, frames, P, U, pb.TemporalSchedule.for_turns(U), ngpu, cfg, W, S, True)
head.pop("lat")
print(json.dumps(head, indent=1))
