import sys, json
sys.path.insert(0, "/root/repo")
import bench, numpy as np
import paper_1701_08361_b200 as pb
G, J, K, U, _ = bench.CONFIGS["c4"]
plan = pb.raw_plan(G, J); plan.newton_steps, plan.cg_iter_budget = 7, 50
z, P = bench.synth_series(G, J, K, U, n_unique=6)
frames = np.stack([z[n % 6] for n in range(30)])
print(json.dumps(bench.decompositions(pb, plan, frames, P, U, pb.TemporalSchedule.for_turns(U), 2)))
