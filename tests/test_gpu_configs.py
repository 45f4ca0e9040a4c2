"""Frame-level parity at the BASELINE.json configurations the bench measures, through the
exact path the bench times (VERDICT r01 "Next round" item 1).

Every test feeds the bench's own synthetic inputs (bench.synth_series: ellipse phantom,
smooth coils, exact radial Toeplitz kernels, K = 15 spokes, U = 5 turns) into a device
`Series` with the bench's schedule, then replays every frame through the compiled
reference (oracle/_ref) with the sources the frame's audit recorded
(ref.reconstruct_frame_regs = reconstruct_frame with a per-step RegProvider,
nlinv.cpp:286-335 and 446-526). Images and estimates must agree within the north-star
frame tolerance (1e-3 relative L2) and the CR iteration counts exactly; the schedule
must satisfy the ordering contract of test_decomp.cpp:345-387.

Reference frames are expensive on the CPU (C3 ~5 s, C5 ~27 s per frame with 4 lanes),
so the series are short: just long enough to leave the strict prefix (l = 5) and run
frames out of order.
"""
import os
import sys

import numpy as np
import pytest

from helpers import rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402  (the bench's own input builders)

pytestmark = pytest.mark.gpu

FRAME_TOL = 1e-3
LANES = max(1, min(4, os.cpu_count() or 1))  # reference WorkerGroup lanes: bit-identical for any A


def _plan(gpu, G, J, M=7, budget=50):
    plan = gpu.raw_plan(G, J)
    plan.newton_steps, plan.cg_iter_budget = M, budget
    return plan


def _bench_series(gpu, plan, F, opts, U=5, K=15):
    """the bench's staging (bench.py main): frames, U PSFs indexed n mod U, device
    normalisation, then one run of all F frames"""
    z_unique, P = bench.synth_series(plan.G, plan.J, K, U, n_unique=min(F, 10), seed=1234)
    z = np.stack([z_unique[n % len(z_unique)] for n in range(F)])
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, F, U)
    s.upload_frames(z)
    for k in range(U):
        s.upload_psf(k, P[k])
    idx = [n % U for n in range(F)]
    s.set_psf_index(idx)
    scale = s.normalize()
    out = s.run(opts)
    return ctx, s, z, P, idx, scale, out


def _check_contract(audit, F, M, sched):
    for n in range(F):
        a = audit[n]
        assert a.frame == n
        if n == 0:
            assert a.init_src == -1
            continue
        assert 0 <= a.init_src < n
        for m in range(M):
            assert 0 <= a.reg_src[m] < n
            if n > sched.l and m < M - 1:
                assert a.reg_src[m] >= n - sched.o
        assert a.reg_final_src == n - 1
        assert a.reg_final_seq > audit[n - 1].finish_seq
        if n <= sched.l:
            assert a.start_seq > audit[n - 1].finish_seq


def _replay(gpu, ref, plan, s, z, P, idx, scale, out, frames):
    """every listed frame through the reference with its audited sources; sources are
    the reference's own replayed estimates, so errors cannot hide by compounding"""
    M = plan.newton_steps
    zs = (z * np.float32(scale)).astype(np.complex64)
    unity = gpu.initial_estimate(plan)
    ests, worst = {}, 0.0
    for n in frames:
        a = out["audit"][n]
        init = unity if a.init_src < 0 else ests[a.init_src]
        regs = [unity if a.init_src < 0 else ests[a.reg_src[m]] for m in range(M)]
        img, est, per = ref.reconstruct_frame_regs(plan, zs[n], P[idx[n]], init, regs, A=LANES)
        ests[n] = est
        img = img * np.float32(1.0 / scale)
        e_img = rel_err(out["images"][n], img)
        e_est = rel_err(s.estimate(n), est)
        worst = max(worst, e_img, e_est)
        assert e_img < FRAME_TOL, (n, e_img)
        assert e_est < FRAME_TOL, (n, e_est)
        assert int(out["cg_iters"][n]) == sum(per), n
    return worst


def test_c3_bench_path_T3_replays_through_the_reference(gpu, ref):
    """C3 (configs[2]: G=256, J=32, 7 steps, 50 CR) exactly as bench.py times it: T = 3
    frames in flight (the autotuner's pick), TemporalSchedule.for_turns(5), five-kernel
    passes (clusters are off with several frames in flight), frame graphs with PDL; two
    k_rows2 channel groups (H = 2)"""
    plan = _plan(gpu, 256, 32)
    F = 9
    sched = gpu.TemporalSchedule.for_turns(5)
    opts = gpu.SeriesOptions(T=3, sched=sched)
    ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, F, opts)
    _check_contract(out["audit"], F, plan.newton_steps, sched)
    assert any(out["audit"][n].thread != 0 for n in range(F))
    _replay(gpu, ref, plan, s, z, P, idx, scale, out, range(F))


def test_c3_latency_mode_matches_the_reference(gpu, ref):
    """C3 latency mode (T = 1, one thread-block cluster per channel): the bench's
    latency_mode figure"""
    plan = _plan(gpu, 256, 32)
    F = 3
    opts = gpu.SeriesOptions(T=1, plain=True, sched=gpu.TemporalSchedule.for_turns(5), cluster=1)
    ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, F, opts)
    assert ctx.cluster_supported()
    _replay(gpu, ref, plan, s, z, P, idx, scale, out, range(F))


def test_c4_T8_t_minus_k_schedule_replays_through_the_reference(gpu, ref):
    """C4 (configs[3]: G=256, J=16) with 8 frames in flight and the relaxed t-k
    schedule o = 8 (decomp.hpp:70-76)"""
    plan = _plan(gpu, 256, 16)
    F = 16
    sched = gpu.TemporalSchedule(5, 8)
    opts = gpu.SeriesOptions(T=8, sched=sched)
    ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, F, opts)
    _check_contract(out["audit"], F, plan.newton_steps, sched)
    assert len({out["audit"][n].thread for n in range(F)}) == 8
    _replay(gpu, ref, plan, s, z, P, idx, scale, out, range(F))


def test_c2_bench_path_T3_replays_through_the_reference(gpu, ref):
    """C2 (configs[1]: G=320, J=10; the 20 x 16 k_rows2 instantiation)"""
    plan = _plan(gpu, 320, 10)
    F = 8
    sched = gpu.TemporalSchedule.for_turns(5)
    ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, F, gpu.SeriesOptions(T=3, sched=sched))
    _check_contract(out["audit"], F, plan.newton_steps, sched)
    _replay(gpu, ref, plan, s, z, P, idx, scale, out, range(F))


def test_c5_frames_match_the_reference(gpu, ref):
    """C5 (configs[4]: G=384, J=64, the 24 x 16 line factorisation), the bench's T = 2
    path: two chained frames on two workers, full 7 steps and 50-iteration budget"""
    plan = _plan(gpu, 384, 64)
    F = 2
    opts = gpu.SeriesOptions(T=2, sched=gpu.TemporalSchedule.for_turns(5))
    ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, F, opts)
    assert out["audit"][1].thread == 1
    _replay(gpu, ref, plan, s, z, P, idx, scale, out, range(F))


def test_c1_long_chain_does_not_drift(gpu, ref):
    """CR numerics over a long chain: k_cr_fused forms |Ap|^2
    from the expansion b^2|ap|^2 + 2b Re<ap,ar> + |ar|^2 instead of the norm of the
    float-rounded update (nlinv.cpp:204-232). 60 chained C1 frames (configs[0]:
    G=128, J=8) against the reference's own chain, frame by frame."""
    plan = _plan(gpu, 128, 8)
    F = 60
    ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, F, gpu.SeriesOptions(plain=True))
    zs = (z * np.float32(scale)).astype(np.complex64)
    est = gpu.initial_estimate(plan)
    worst = 0.0
    for n in range(F):
        img, est, per, _ = ref.reconstruct_frame(plan, zs[n], P[idx[n]], est, est, A=LANES)
        img = img * np.float32(1.0 / scale)
        e = max(rel_err(out["images"][n], img), rel_err(s.estimate(n), est))
        worst = max(worst, e)
        assert e < FRAME_TOL, (n, e)
    print(f"C1 60-frame chain: worst frame error {worst:.2e}")


def test_c1_large_cr_budget_matches_the_reference(gpu, ref):
    """one C1 frame with a 200-iteration CR budget (late-solve cancellation in the fused
    recurrence's |Ap|^2 expansion would show here first)"""
    plan = _plan(gpu, 128, 8, M=7, budget=200)
    z_unique, P = bench.synth_series(plan.G, plan.J, 13, 5, n_unique=1, seed=77)
    nsq = float(np.sum(np.abs(z_unique[0].astype(np.complex128)) ** 2))
    z = (z_unique[0] * np.float32(100.0 / np.sqrt(nsq))).astype(np.complex64)
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P[0])
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
    img, est, per, _ = ref.reconstruct_frame(plan, z, P[0], init, A=LANES)
    assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL


@pytest.mark.parametrize("cfg", ["c3", "c1"])
def test_deferred_cr_reductions_match_grid_reductions(gpu, monkeypatch, cfg):
    # the budget-mode CR solve with deferred reductions (k_colsW and every recurrence but a
    # step's last leave per-block partials; the next recurrence forms the totals and takes
    # the previous iteration's decisions) against the grid reductions with last-block tails
    # (RTN_DEFER_RED=0): same iteration counts, frames equal to FP64 summation order
    G, J, K, U, _ = bench.CONFIGS[cfg]
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("RTN_DEFER_RED", mode)
        plan = _plan(gpu, G, J)
        # a plain chain on the five-kernel passes (deterministic sources; the cluster path
        # keeps its own reductions)
        ctx, s, z, P, idx, scale, out = _bench_series(gpu, plan, 6, gpu.SeriesOptions(plain=True, cluster=0))
        outs[mode] = (out, [s.estimate(n) for n in range(6)])
        s.close()
        ctx.close()
    a, b = outs["1"], outs["0"]
    assert list(a[0]["cg_iters"]) == list(b[0]["cg_iters"])
    for n in range(6):
        assert rel_err(a[0]["images"][n], b[0]["images"][n]) < 1e-5, n
        assert rel_err(a[1][n], b[1][n]) < 1e-5, n
