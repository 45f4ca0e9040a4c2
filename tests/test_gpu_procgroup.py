"""Channel decomposition with one process per GPU (procgroup.hpp): two processes,
each one member, connected by CUDA IPC handles exchanged over torch.distributed
(gloo). With one visible GPU both processes share it (time-sliced contexts); the
member-order arithmetic makes the result bit-identical to the in-process group of the
same width, and it matches the reference's WorkerGroup within the frame tolerance."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import phantom_frame_inputs, rel_err

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _member(rank, world, port, plan_args, z, P, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        import paper_1701_08361_b200 as pb
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n = pb.load_library().rtn_device_count()
        plan = pb.make_plan(*plan_args[:2])
        plan.newton_steps, plan.cg_iter_budget = plan_args[2], plan_args[3]
        ctx = pb.Context(plan, device=rank % n, member=(rank, world))
        pb.connect_members(ctx)
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(pb.initial_estimate(plan))
        fr2 = ctx.reconstruct_frame(pb.initial_estimate(plan))  # graph replay
        q.put((rank, fr.image, fr.est, fr.cg_per_step, bool(np.array_equal(fr.image, fr2.image))))
        ctx.close()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e), None, None))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("budget", [6, 0])  # 0: tolerance mode (the exact two-pass recurrence)
def test_two_process_channel_group_matches_in_process_group_and_reference(gpu, ref, budget):
    plan = gpu.make_plan(16, 3)
    plan.newton_steps, plan.cg_iter_budget = 3, budget
    inp = phantom_frame_inputs(ref, plan, K=7, U=1)
    z, P = inp["z"][0], inp["P"][0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_member, args=(r, 2, port, (16, 3, 3, budget), z, P, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in res:
        assert not isinstance(r[1], str), r
    (_, img0, est0, cg0, replay0), (_, img1, est1, cg1, replay1) = res
    assert replay0 and replay1
    assert np.array_equal(img0, img1) and np.array_equal(est0, est1) and cg0 == cg1
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan, devices=[0, 0]) as grp:
        grp.set_psf(P)
        grp.set_data(z)
        want = grp.reconstruct_frame(init)
    assert np.array_equal(img0, want.image) and np.array_equal(est0, want.est)
    rimg, rest, rper, _ = ref.reconstruct_frame(plan, z, P, init, A=2)
    assert cg0 == rper
    assert rel_err(img0, rimg) < 1e-3 and rel_err(est0, rest) < 1e-3


def _member_absent(rank, world, port, plan_args, z, P, q):
    # rank 1 connects but never reconstructs: rank 0 must fail at the barrier deadline
    # (the reference's WorkerGroup deadline -> DecompFault), not hang
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import time
        import torch.distributed as dist
        import paper_1701_08361_b200 as pb
        dist.init_process_group("gloo", rank=rank, world_size=world)
        plan = pb.make_plan(*plan_args[:2])
        plan.newton_steps, plan.cg_iter_budget = plan_args[2], plan_args[3]
        ctx = pb.Context(plan, device=0, member=(rank, world))
        pb.connect_members(ctx)
        ctx.set_psf(P)
        ctx.set_data(z)
        if rank == 0:
            t0 = time.time()
            try:
                ctx.reconstruct_frame(pb.initial_estimate(plan))
                q.put((rank, "no error", time.time() - t0))
            except pb.DecompFault:
                q.put((rank, "DecompFault", time.time() - t0))
        else:
            time.sleep(25)
            q.put((rank, "idle", 0.0))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


@pytest.mark.timeout(300)
def test_missing_member_fails_at_the_barrier_deadline(gpu, ref):
    plan = gpu.make_plan(16, 2)
    plan.newton_steps, plan.cg_iter_budget = 2, 4
    inp = phantom_frame_inputs(ref, plan, K=7, U=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_member_absent, args=(r, 2, port, (16, 2, 2, 4), inp["z"][0], inp["P"][0], q))
             for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = sorted([q.get(timeout=200) for _ in procs], key=lambda r: r[0])
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert res[0][1] == "DecompFault", res
    assert res[0][2] < 60
