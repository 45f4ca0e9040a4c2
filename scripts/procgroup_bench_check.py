import os, sys, socket
sys.path.insert(0, "/root/repo")
import torch.multiprocessing as mp

def w(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK="0")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench, numpy as np, paper_1701_08361_b200 as pb
    G, J, K, U, _ = bench.CONFIGS["c4"]
    plan = pb.raw_plan(G, J); plan.newton_steps, plan.cg_iter_budget = 7, 50
    z, P = bench.synth_series(G, J, K, U, n_unique=1)
    r = bench.channel_processes(pb, plan, z, P, world, rank, 0, 4)
    q.put((rank, r))

if __name__ == "__main__":
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ps = [ctx.Process(target=w, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in ps]
    print([q.get(timeout=600) for _ in ps])
    [p.join() for p in ps]
