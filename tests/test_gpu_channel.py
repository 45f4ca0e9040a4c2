"""Channel decomposition: a context over A device-group members,
member k owning partition_channels(J, A)[k], with the channel sum read from peer
memory inside k_colsW and the CR scalars summed in member order (group.hpp).

Parity is against the reference's own channel decomposition (WorkerGroup with A
lanes, decomp.cpp:103-134; its results are bit-identical for every A) at the
north-star tolerances. With one visible GPU the members share device 0 (separate
streams, event barriers, the same kernels and peer-pointer reads); with more GPUs
they are spread over the devices.
"""
import numpy as np
import pytest

from helpers import phantom_frame_inputs, radial_psf, random_estimate, rel_err

pytestmark = pytest.mark.gpu

OP_TOL = 1e-5
FRAME_TOL = 1e-3


def _devices(gpu, A):
    n = gpu.load_library().rtn_device_count()
    return [k % n for k in range(A)]


@pytest.mark.parametrize("G,J,A", [(32, 3, 2), (32, 3, 3), (128, 8, 2), (128, 8, 4), (128, 8, 8),
                                   (128, 10, 3), (256, 32, 8)])
def test_group_apply_normal_matches_reference(gpu, ref, G, J, A):
    plan = gpu.raw_plan(G, J)
    P = radial_psf(ref, plan, 7, G + J + A)
    x = random_estimate(plan, 7 * G + J)
    with gpu.Context(plan, devices=_devices(gpu, A)) as ctx, gpu.Context(plan) as one:
        assert ctx.group_blocks == gpu.partition_channels(J, A, 8)
        ctx.set_psf(P)
        one.set_psf(P)
        ctx.make_step_cache(x)
        one.make_step_cache(x)
        for t in range(2):
            dx = random_estimate(plan, 100 * G + 10 * J + t)
            got = ctx.apply_normal(dx)
            want = ref.apply_normal(plan, x, dx, P, A=min(A, 4))
            assert rel_err(got, want) < OP_TOL, t
            # against the single-device path: only the FP64 channel-sum grouping differs
            assert rel_err(got, one.apply_normal(dx)) < 1e-6, t


@pytest.mark.parametrize("A", [2, 4])
@pytest.mark.parametrize("budget", [50, 0])
def test_group_reconstruct_frame_c1(gpu, ref, A, budget):
    plan = gpu.raw_plan(128, 8)
    plan.newton_steps = 7
    plan.cg_iter_budget = budget
    inp = phantom_frame_inputs(ref, plan, K=13, U=5)
    z, P = inp["z"][0], inp["P"][0]
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan, devices=_devices(gpu, A)) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
        fr2 = ctx.reconstruct_frame(init)  # graph replay: identical
    img, est, per, _ = ref.reconstruct_frame(plan, z, P, init, A=A)
    if budget:
        assert fr.cg_per_step == per == [8, 7, 7, 7, 7, 7, 7]
    else:
        # tolerance mode: the two-pass recurrence with the exact |ap|^2 (nlinv.cpp:204-230)
        # stops at the reference's iteration in every step
        assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL
    assert np.array_equal(fr.image, fr2.image)


def test_group_result_independent_of_member_placement(gpu, ref):
    # the same A on different device lists gives bit-identical frames (fixed member
    # order of every cross-member sum)
    plan = gpu.raw_plan(64, 6)
    plan.newton_steps, plan.cg_iter_budget = 4, 16
    inp = phantom_frame_inputs(ref, plan, K=9, U=3)
    init = gpu.initial_estimate(plan)
    outs = []
    n = gpu.load_library().rtn_device_count()
    for devs in ([0, 0, 0], [k % n for k in (0, 1, 2)]):
        with gpu.Context(plan, devices=devs) as ctx:
            ctx.set_psf(inp["P"][0])
            ctx.set_data(inp["z"][0])
            outs.append(ctx.reconstruct_frame(init))
    assert np.array_equal(outs[0].image, outs[1].image)
    assert np.array_equal(outs[0].est, outs[1].est)


@pytest.mark.parametrize("A", [2, 4])
def test_group_device_flag_barriers_match_event_barriers(gpu, ref, A, monkeypatch):
    # the all-member barrier as device-side epoch flags (k_pg_barrier, the default when
    # every member has its own GPU) forced onto members that share this GPU: the frames
    # (graph capture, replay, op-level calls) are bit-identical to the stream-edge
    # barriers and within the frame tolerance of the reference
    plan = gpu.raw_plan(128, 8)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    inp = phantom_frame_inputs(ref, plan, K=13, U=5)
    init = gpu.initial_estimate(plan)
    x = random_estimate(plan, 5)
    outs = {}
    for mode in ("events", "flags"):
        monkeypatch.setenv("RTN_GROUP_BARRIER", mode)
        with gpu.Context(plan, devices=_devices(gpu, A)) as ctx:
            ctx.set_psf(inp["P"][0])
            ctx.set_data(inp["z"][0])
            f1 = ctx.reconstruct_frame(init)
            f2 = ctx.reconstruct_frame(f1.est, f1.est)  # replay of the captured frame graph
            ctx.make_step_cache(x)
            op = ctx.apply_normal(random_estimate(plan, 6))
            outs[mode] = (f1, f2, op)
    for k in range(2):
        assert np.array_equal(outs["flags"][k].image, outs["events"][k].image), k
        assert np.array_equal(outs["flags"][k].est, outs["events"][k].est), k
        assert outs["flags"][k].cg_per_step == outs["events"][k].cg_per_step
    assert np.array_equal(outs["flags"][2], outs["events"][2])
    img, _, per, _ = ref.reconstruct_frame(plan, inp["z"][0], inp["P"][0], init, A=min(A, 4))
    assert outs["flags"][0].cg_per_step == per
    assert rel_err(outs["flags"][0].image, img) < FRAME_TOL


def test_group_fft_accounting(gpu, ref):
    # test_nlinv.cpp:370-389 counts logical transforms, whatever the decomposition
    plan = gpu.make_plan(16, 3)
    plan.newton_steps, plan.cg_iter_budget = 4, 12
    inp = phantom_frame_inputs(ref, plan, K=11, U=1, normalize=False)
    with gpu.Context(plan, devices=_devices(gpu, 3)) as ctx:
        ctx.set_psf(inp["P"][0])
        ctx.set_data(inp["z"][0])
        gpu.fft_reset_counts()
        fr = ctx.reconstruct_frame(gpu.initial_estimate(plan))
    assert fr.cg_per_step == [3, 3, 3, 3]
    c = gpu.fft_counts()
    assert c["normal_op"] == 4 * 3 * 12
    assert c["setup"] == 4 * 3 * 4 + 3


def test_group_rejects_bad_shapes(gpu):
    plan = gpu.raw_plan(32, 2)
    with pytest.raises(gpu.UsageError):
        gpu.Context(plan, devices=[0, 0, 0])  # more members than channels
    with gpu.Context(plan, devices=[0, 0]) as ctx:
        with pytest.raises(gpu.UsageError):
            ctx.cg_solve(np.zeros(ctx.D, np.complex64), 1.0, 0.0, 3)


def _series_inputs(ref, plan, F, K, U, noise=1e-4, seed=11):
    samples, angles = ref.phantom_series(plan.J, F, K, U, plan.N, noise, seed)
    z = np.stack([ref.grid_adjoint(plan, samples[n], angles[n]) for n in range(F)])
    P = np.stack([ref.build_psf(plan, angles[n], 2 * plan.N) for n in range(min(U, F))])
    return samples, angles, z, P, [n % U for n in range(F)]


def _series(gpu, plan, z, P, idx, opts):
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, z.shape[0], P.shape[0], devices=_devices(gpu, 8))
    s.upload_frames(z)
    for k in range(P.shape[0]):
        s.upload_psf(k, P[k])
    s.set_psf_index(idx)
    out = s.run(opts)
    out["series"], out["ctx"] = s, ctx
    return out


def test_channel_decomposed_plain_series_matches_reference(gpu, ref):
    plan = gpu.make_plan(24, 4)
    plan.newton_steps, plan.cg_iter_budget = 7, 30
    samples, angles, z, P, idx = _series_inputs(ref, plan, F=5, K=11, U=5)
    want = ref.reconstruct_series(plan, samples, angles, plain=True, A=2)
    got = _series(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True, A=2))
    for n in range(5):
        assert rel_err(got["images"][n], want["images"][n]) < FRAME_TOL, n
        assert got["audit"][n].workers == 2
    assert list(got["cg_iters"]) == list(want["cg_iters"])


@pytest.mark.parametrize("A", [2, 4])
def test_group_cluster_applications_match_reference(gpu, ref, A):
    # latency mode on a channel group: each member runs one thread-block cluster per own
    # channel, then k_rho_sum forms out.rho over every member's channel terms (peer reads,
    # in the single-device channel order) after an all-member barrier
    plan = gpu.raw_plan(128, 8)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    with gpu.Context(plan) as probe:
        if not probe.cluster_supported():
            pytest.skip("no cluster-fused application for this grid")
    samples, angles, z, P, idx = _series_inputs(ref, plan, F=3, K=13, U=3)
    want = ref.reconstruct_series(plan, samples, angles, plain=True, A=min(A, 4))
    got = {}
    for cl in (1, 0):
        out = _series(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True, A=A, cluster=cl))
        got[cl] = out
        for n in range(3):
            assert rel_err(out["images"][n], want["images"][n]) < FRAME_TOL, (cl, n)
            assert out["audit"][n].workers == A
        assert list(out["cg_iters"]) == list(want["cg_iters"])
    # the two application paths differ only in FP32 rounding of the fused passes
    for n in range(3):
        assert rel_err(got[1]["images"][n], got[0]["images"][n]) < 1e-5, n


def test_group_cluster_applications_at_g256(gpu, ref):
    # the C3/C4 instantiation (16 x 16, one 8-CTA cluster per channel) on a channel group:
    # frames against the reference's WorkerGroup and against the group's five-kernel passes
    plan = gpu.raw_plan(256, 8)
    plan.newton_steps, plan.cg_iter_budget = 4, 16
    with gpu.Context(plan) as probe:
        if not probe.cluster_supported():
            pytest.skip("no cluster-fused application for this grid")
    samples, angles, z, P, idx = _series_inputs(ref, plan, F=2, K=15, U=2)
    want = ref.reconstruct_series(plan, samples, angles, plain=True, A=2)
    got = {}
    for cl in (1, 0):
        out = _series(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True, A=2, cluster=cl))
        got[cl] = out
        for n in range(2):
            assert rel_err(out["images"][n], want["images"][n]) < FRAME_TOL, (cl, n)
        assert list(out["cg_iters"]) == list(want["cg_iters"])
    for n in range(2):
        assert rel_err(got[1]["images"][n], got[0]["images"][n]) < 1e-5, n


def test_group_workers_with_pre_stage_lanes(gpu, ref, monkeypatch):
    # raw acquisitions on T = 2 channel-group workers (A = 2): worker 1's frames go through
    # its own pre-stage lane (forced on one GPU) and its group splits them to its members;
    # with a sequential schedule the frames equal the store path's bit for bit
    plan = gpu.make_plan(24, 4)
    plan.newton_steps, plan.cg_iter_budget = 4, 12
    F, U = 5, 3
    samples, angles = ref.phantom_series(plan.J, F, 11, U, plan.N, 1e-3, 41)
    outs = {}
    for lanes in ("0", "1"):
        monkeypatch.setenv("RTN_PRE_LANES", lanes)
        ctx = gpu.Context(plan)
        s = gpu.Series(ctx, F, U, devices=_devices(gpu, 4))
        outs[lanes] = s.run(gpu.SeriesOptions(T=2, A=2, sched=gpu.TemporalSchedule(F, 1)),
                            raw=dict(samples=samples, angles=angles))
    assert list(outs["0"]["cg_iters"]) == list(outs["1"]["cg_iters"])
    for n in range(F):
        assert np.array_equal(outs["0"]["images"][n], outs["1"]["images"][n]), n


@pytest.mark.parametrize("T,A", [(2, 2), (4, 2), (2, 3)])
def test_hybrid_temporal_channel_series_replays_exactly(gpu, ref, T, A):
    # hybrid T x A split: T frame workers, each a channel group of A members; every
    # frame replayed through the reference with the sources its audit recorded
    plan = gpu.make_plan(16, 3)
    plan.newton_steps, plan.cg_iter_budget = 3, 6
    F = 8
    _, _, z, P, idx = _series_inputs(ref, plan, F=F, K=5, U=3)
    sched = gpu.TemporalSchedule(2, 2)
    out = _series(gpu, plan, z, P, idx, gpu.SeriesOptions(T=T, A=A, sched=sched))
    M = plan.newton_steps
    scale = out["series"].normalize()
    zs = (z * np.float32(scale)).astype(np.complex64)
    unity = gpu.initial_estimate(plan)
    ests = {}
    for n in range(F):
        a = out["audit"][n]
        assert a.reg_final_src == (n - 1 if n > 0 else -1)
        init = unity if a.init_src < 0 else ests[a.init_src]
        regs = [unity if a.init_src < 0 else ests[a.reg_src[m]] for m in range(M)]
        img, est, _ = ref.reconstruct_frame_regs(plan, zs[n], P[idx[n]], init, regs)
        ests[n] = est
        assert rel_err(out["images"][n], img * np.float32(1.0 / scale)) < FRAME_TOL, n
        assert rel_err(out["series"].estimate(n), est) < FRAME_TOL, n


def test_all_reduce_sum_is_the_ordered_fp64_sum(gpu):
    # test_decomp.cpp:82-106 on the device entry point: repeatable bit for bit, FP64
    # accumulation in index order (here checked exactly, not just to 1e-6), zeros stay
    # zero, no terms is a usage error
    from helpers import random_image
    terms = np.stack([random_image(12, 100 + j) for j in range(5)])
    s1 = gpu.all_reduce_sum(terms)
    s2 = gpu.all_reduce_sum(terms)
    assert np.array_equal(s1.view(np.uint32), s2.view(np.uint32))
    acc = np.zeros(terms.shape[1:], np.complex128)
    for t in terms:
        acc += t.astype(np.complex128)
    assert np.array_equal(s1, acc.astype(np.complex64))
    assert not np.any(gpu.all_reduce_sum(np.zeros((3, 8, 8), np.complex64)))
    with pytest.raises(gpu.UsageError):
        gpu.all_reduce_sum(np.zeros((0, 8, 8), np.complex64))
