"""Parity of the sm_100a operator path against the compiled reference (oracle/_ref).

Tolerances are the north-star ones (BASELINE.json): a single operator application
within relative L2 1e-5; whole frames within 1e-3. Every call goes through the C
ABI (include/rtnlinv_b200.h) with host buffers.
"""
import numpy as np
import pytest

from helpers import phantom_frame_inputs, radial_psf, random_estimate, random_image, rel_err

pytestmark = pytest.mark.gpu

OP_TOL = 1e-5     # single operator application (north star)
FRAME_TOL = 1e-3  # full frame after all Newton steps (north star)


@pytest.mark.parametrize("n", [4, 8, 9, 16, 17, 48, 72, 128, 256, 320, 384])
def test_fft_matches_reference_fft(gpu, ref, n):
    # test_fft.cpp:9-29 sizes plus the configuration grids
    x = random_image(n, 100 + n)
    for sign, ours in ((-1, gpu.fft_forward), (+1, gpu.fft_inverse)):
        want = ref.fft(x, sign)
        got = ours(x)
        assert rel_err(got, want) < OP_TOL, (n, sign)


def test_fft_dc_convention_and_unitarity(gpu):
    # test_fft.cpp:62-76: constant image -> spike n at n/2 (even n)
    n = 10
    x = np.ones((n, n), np.complex64)
    X = gpu.fft_forward(x)
    assert abs(X[n // 2, n // 2] - n) < 1e-4
    X[n // 2, n // 2] = 0
    assert np.abs(X).sum() < 1e-3
    y = random_image(256, 7)
    Y = gpu.fft_forward(y)
    assert abs(np.vdot(Y, Y).real / np.vdot(y, y).real - 1) < 1e-6


def test_fft_counters_follow_context(gpu):
    gpu.fft_reset_counts()
    x = random_image(16, 3)
    gpu.fft_forward(x)
    with gpu.CtxScope(gpu.FftCtx.normal_op):
        gpu.fft_forward(x)
        gpu.fft_inverse(x)
        with gpu.CtxScope(gpu.FftCtx.setup):
            gpu.fft_forward(x)
        gpu.fft_forward(x)
    c = gpu.fft_counts()
    assert (c["other"], c["normal_op"], c["setup"]) == (1, 3, 1)
    gpu.fft_reset_counts()
    assert sum(gpu.fft_counts().values()) == 0


@pytest.mark.parametrize("G", [24, 48, 128, 256])
def test_weight_pair_matches_reference(gpu, ref, G):
    plan = gpu.raw_plan(G, 1)
    winv = gpu.make_weights_inv(plan.Gc, G)
    assert np.array_equal(winv, ref.make_weights_inv(plan.Gc, G))
    with gpu.Context(plan) as ctx:
        a = random_image(plan.Gc, 900 + G)
        u = random_image(G, 950 + G)
        assert rel_err(ctx.apply_W_inv(a), ref.apply_W_inv(a, winv, G)) < OP_TOL
        assert rel_err(ctx.apply_W_invH(u), ref.apply_W_invH(u, winv, plan.Gc)) < OP_TOL
        # DC spike decodes to the constant 1/G (test_nlinv.cpp:158-165)
        spike = np.zeros((plan.Gc, plan.Gc), np.complex64)
        spike[plan.Gc // 2, plan.Gc // 2] = 1
        img = ctx.apply_W_inv(spike)
        assert np.max(np.abs(img - 1.0 / G)) < 1e-7


@pytest.mark.parametrize("G,K", [(16, 5), (48, 7), (128, 13), (256, 15)])
def test_toeplitz_matches_reference(gpu, ref, G, K):
    plan = gpu.raw_plan(G, 1)
    P = radial_psf(ref, plan, K, G + K)
    x = random_image(G, 11 + G)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        assert rel_err(ctx.toeplitz_apply(x), ref.toeplitz_apply(x, P)) < OP_TOL


@pytest.mark.parametrize("G,J", [(16, 1), (16, 3), (32, 3), (48, 2), (72, 2), (128, 8), (256, 4), (320, 3),
                                 (384, 2), (512, 1)])
def test_apply_normal_matches_reference(gpu, ref, G, J):
    plan = gpu.raw_plan(G, J)
    P = radial_psf(ref, plan, 5, G + J)
    x = random_estimate(plan, 10 * G + J)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        rho, coils = ctx.make_step_cache(x)
        rrho, rcoils = ref.make_step_cache(plan, x, P)
        assert rel_err(rho, rrho) == 0.0
        assert rel_err(coils, rcoils) < OP_TOL
        for t in range(3):
            dx = random_estimate(plan, 1000 * G + 100 * J + 4 * t)
            got = ctx.apply_normal(dx)
            want = ref.apply_normal(plan, x, dx, P)
            assert rel_err(got, want) < OP_TOL, t
            # output lives on the window (test_nlinv.cpp:205-220)
            grho = got[:G * G].reshape(G, G)
            L, lo = G // 2, G // 4
            mask = np.ones((G, G), bool)
            mask[lo:lo + L, lo:lo + L] = False
            assert np.all(grho[mask] == 0)


def test_apply_normal_self_adjoint_and_psd(gpu, ref):
    # test_nlinv.cpp:178-203 on the device operator
    for G, J in ((16, 1), (32, 3)):
        plan = gpu.raw_plan(G, J)
        P = radial_psf(ref, plan, 5, G + J)
        with gpu.Context(plan) as ctx:
            ctx.set_psf(P)
            ctx.make_step_cache(random_estimate(plan, 10 * G + J))
            for t in range(5):
                dx = random_estimate(plan, 7 * t + 1).astype(np.complex128)
                dy = random_estimate(plan, 7 * t + 2).astype(np.complex128)
                adx = ctx.apply_normal(dx).astype(np.complex128)
                ady = ctx.apply_normal(dy).astype(np.complex128)
                lhs, rhs = np.vdot(adx, dy), np.vdot(dx, ady)
                assert abs(lhs - rhs) <= 1e-4 * max(abs(lhs), 1e-30)
                assert np.vdot(adx, dx).real >= -1e-4 * np.vdot(dx, dx).real


@pytest.mark.parametrize("tol,max_iter", [(0.0, 1), (0.0, 7), (0.0, 20), (1e-3, 200)])
def test_cg_solve_matches_reference(gpu, ref, tol, max_iter):
    plan = gpu.raw_plan(32, 3)
    P = radial_psf(ref, plan, 5, 31)
    x = random_estimate(plan, 600)
    rhs = random_estimate(plan, 602)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.make_step_cache(x)
        got, it, res = ctx.cg_solve(rhs, 0.5, tol, max_iter)
    want, wit, wres = ref.cg_solve(plan, x, rhs, P, 0.5, tol, max_iter)
    assert it == wit
    assert rel_err(got, want) < 1e-4
    # residuals agree to 1e-4 until they reach float round-off of the first one
    np.testing.assert_allclose(res, wres, rtol=1e-4, atol=1e-6 * wres[0])
    # residual norms never increase (test_nlinv.cpp:279-286)
    assert np.all(res[1:] <= res[:-1] * (1 + 1e-5))


def test_cg_solve_bookkeeping(gpu, ref):
    plan = gpu.raw_plan(16, 2)
    P = radial_psf(ref, plan, 5, 31)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.make_step_cache(random_estimate(plan, 600))
        zero = np.zeros(plan.D, np.complex64)
        gpu.fft_reset_counts()
        x, it, res = ctx.cg_solve(zero, 0.5, 1e-3, 50)
        assert it == 0 and len(res) == 0 and not np.any(x)
        assert sum(gpu.fft_counts().values()) == 0
        rhs = random_estimate(plan, 602)
        for cap in (1, 3, 7):
            gpu.fft_reset_counts()
            _, it, _ = ctx.cg_solve(rhs, 0.5, 0.0, cap)
            assert it == cap
            assert sum(gpu.fft_counts().values()) == 4 * plan.J * cap
        # overwhelming damping: x = rhs / alpha (test_nlinv.cpp:296-305)
        x, _, _ = ctx.cg_solve(rhs, 1e8, 1e-8, 50)
        assert rel_err(x, rhs / np.float32(1e8)) <= 1e-4
        bad = rhs.copy()
        bad[8 * 16 + 8] = np.nan
        with pytest.raises(gpu.SolverError):
            ctx.cg_solve(bad, 0.5, 1e-3, 50)


@pytest.mark.parametrize("cg_tol,cap", [(0.0, 8), (1e-3, 200)])
def test_newton_step_matches_reference(gpu, ref, cg_tol, cap):
    plan = gpu.make_plan(16, 2)
    inp = phantom_frame_inputs(ref, plan, K=7, U=1)
    z, P = inp["z"][0], inp["P"][0]
    x0 = gpu.initial_estimate(plan)
    reg = random_estimate(plan, 70) * np.float32(0.01)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        got, it, r0 = ctx.newton_step(x0, reg, 0.7, cg_tol, cap)
    want, wit, wr0 = ref.newton_step(plan, x0, reg, 0.7, z, P, cg_tol, cap)
    assert it == wit
    assert abs(r0 - wr0) <= 1e-5 * wr0
    assert rel_err(got, want) < 1e-4


@pytest.mark.parametrize("group", [False, True])
def test_newton_step_with_data_outside_the_window(gpu, ref, group):
    # gridded data that is not window-masked (grid_adjoint masks, the API does not
    # require it): the out-of-window rhs.rho term sum_j conj(c_j) z_j is live
    plan = gpu.make_plan(16, 3)
    plan.newton_steps, plan.cg_iter_budget = 3, 9
    inp = phantom_frame_inputs(ref, plan, K=7, U=1)
    z = inp["z"][0] + 0.05 * random_image(plan.G, 5, (plan.J, plan.G, plan.G))
    P = inp["P"][0]
    init = gpu.initial_estimate(plan)
    kw = {"devices": [0, 0]} if group else {}
    with gpu.Context(plan, **kw) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
    img, est, per, _ = ref.reconstruct_frame(plan, z, P, init)
    assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL


def test_fixed_point_needs_no_iterations(gpu, ref):
    # test_nlinv.cpp:314-349: data manufactured from x itself leaves x unchanged
    plan = gpu.make_plan(16, 2)
    plan.newton_steps, plan.cg_iter_budget = 2, 6
    inp = phantom_frame_inputs(ref, plan, K=7, U=1, normalize=False, seed=7)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(inp["P"][0])
        ctx.set_data(inp["z"][0])
        x = ctx.reconstruct_frame(gpu.initial_estimate(plan)).est
        rho, coils = ctx.make_step_cache(x)
        zx = np.stack([ctx.toeplitz_apply(rho * coils[j]) for j in range(plan.J)])
        ctx.set_data(zx)
        moved, it, r0 = ctx.newton_step(x, x, 0.7, 1e-3, 50)
    # the reference itself gets exactly 0 here; the device FFT round trip leaves
    # float rounding in z - T(rho c), so only the size of the move is pinned
    assert r0 <= 1e-5 * np.linalg.norm(zx)
    assert rel_err(moved, x) < 1e-5


@pytest.mark.parametrize("budget", [50, 0])
def test_reconstruct_frame_c1(gpu, ref, budget):
    # configs[0] (C1): 64x64 image, G = 128, 8 channels, 13 spokes, 7 Newton steps
    plan = gpu.raw_plan(128, 8)
    plan.newton_steps = 7
    plan.cg_iter_budget = budget
    inp = phantom_frame_inputs(ref, plan, K=13, U=5)
    z, P = inp["z"][0], inp["P"][0]
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
    img, est, per, _ = ref.reconstruct_frame(plan, z, P, init)
    if budget:
        assert fr.cg_per_step == per == [8, 7, 7, 7, 7, 7, 7]
    else:
        assert sum(fr.cg_per_step) == pytest.approx(sum(per), abs=3)
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL


def test_frame_fft_accounting(gpu, ref):
    # test_nlinv.cpp:370-389: 4 transforms / channel / CG iteration, 4 / channel /
    # step in setup, plus the final decode
    plan = gpu.make_plan(16, 3)
    plan.newton_steps, plan.cg_iter_budget = 4, 12
    inp = phantom_frame_inputs(ref, plan, K=11, U=1, normalize=False)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(inp["P"][0])
        ctx.set_data(inp["z"][0])
        gpu.fft_reset_counts()
        fr = ctx.reconstruct_frame(gpu.initial_estimate(plan))
    assert fr.cg_per_step == [3, 3, 3, 3]
    c = gpu.fft_counts()
    assert c["normal_op"] == 4 * 3 * 12
    assert c["setup"] == 4 * 3 * 4 + 3
    assert c["other"] == 0


def test_budget_spread(gpu, ref):
    plan = gpu.make_plan(16, 2)
    plan.newton_steps, plan.cg_iter_budget = 6, 50
    inp = phantom_frame_inputs(ref, plan, K=11, U=1, normalize=False)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(inp["P"][0])
        ctx.set_data(inp["z"][0])
        fr = ctx.reconstruct_frame(gpu.initial_estimate(plan))
    assert fr.cg_per_step == [9, 9, 8, 8, 8, 8]
    assert fr.cg_iters == 50


def test_shape_and_size_validation(gpu):
    with pytest.raises(gpu.UsageError):
        gpu.Context(gpu.ReconPlan(N=8, G=34, Gc=8, J=1))  # 34 = 2 x 17 not covered
    with pytest.raises(gpu.UsageError):
        gpu.Context(gpu.ReconPlan(N=8, G=16, Gc=32, J=1))
    with pytest.raises(gpu.UsageError):
        gpu.make_weights_inv(8, 4)


@pytest.mark.parametrize("J", [4, 32])
def test_cluster_fused_application_matches_reference(gpu, ref, J, monkeypatch):
    # the one-cluster-per-channel application (kernels_cluster.cuh, G = 256, Gc = G/4)
    # against the reference and against the five-kernel path
    plan = gpu.raw_plan(256, J)
    P = radial_psf(ref, plan, 9, J)
    x = random_estimate(plan, 91 + J)
    outs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RTN_CLUSTER", flag)
        with gpu.Context(plan) as ctx:
            ctx.set_psf(P)
            ctx.make_step_cache(x)
            outs[flag] = [ctx.apply_normal(random_estimate(plan, 500 + t)) for t in range(2)]
    for t in range(2):
        want = ref.apply_normal(plan, x, random_estimate(plan, 500 + t), P)
        assert rel_err(outs["1"][t], want) < OP_TOL, t
        assert rel_err(outs["1"][t], outs["0"][t]) < 1e-6, t


def test_cluster_fused_frame_matches_reference(gpu, ref, monkeypatch):
    # a C4-shaped frame (G = 256, 16 channels) through the cluster path in the budget graphs
    monkeypatch.setenv("RTN_CLUSTER", "1")
    plan = gpu.raw_plan(256, 16)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    inp = phantom_frame_inputs(ref, plan, K=15, U=5)
    z, P = inp["z"][0], inp["P"][0]
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
    img, est, per, _ = ref.reconstruct_frame(plan, z, P, init, A=4)
    assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL


@pytest.mark.parametrize("A,budget", [(1, 12), (1, 0), (2, 12)])
def test_reconstruct_frame_with_a_reg_provider_matches_reference(gpu, ref, A, budget):
    # RegProvider (nlinv.hpp:102): a different regularisation target per Newton step,
    # step 2 keeping step 1's (None); budget mode and tolerance mode (cg_tol 1e-3)
    plan = gpu.make_plan(16, 3)
    plan.newton_steps, plan.cg_iter_budget = 4, budget
    inp = phantom_frame_inputs(ref, plan, K=7, U=1)
    z, P = inp["z"][0], inp["P"][0]
    init = gpu.initial_estimate(plan)
    targets = [random_estimate(plan, 90 + m) * np.float32(0.01) for m in range(plan.newton_steps)]
    provided = [targets[0], targets[1], None, targets[3]]
    regs = [targets[0], targets[1], targets[1], targets[3]]
    devices = [0] * A if A > 1 else None
    with gpu.Context(plan, devices=devices) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init, regs=lambda m: provided[m])
    img, est, per = ref.reconstruct_frame_regs(plan, z, P, init, regs)
    assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL


def test_cg_capacity_growth_keeps_cached_frame_graphs_valid(gpu, ref):
    """a cg_solve with max_iter above the plan's CR capacity reallocates the
    device CR scalars; the frame graphs captured earlier hold the old pointers and must
    be rebuilt, so a frame after the solve equals the frame before it bit for bit"""
    plan = gpu.make_plan(16, 2)
    plan.newton_steps, plan.cg_iter_budget = 3, 9
    inp = phantom_frame_inputs(ref, plan, K=7, U=1)
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(inp["P"][0])
        ctx.set_data(inp["z"][0])
        before = ctx.reconstruct_frame(init)
        ctx.make_step_cache(before.est)
        rhs = random_estimate(plan, 9)
        _, iters, _ = ctx.cg_solve(rhs, 0.5, 0.0, 400)  # capacity grows past max(200, 9)
        assert iters == 400
        after = ctx.reconstruct_frame(init)
    assert np.array_equal(before.image, after.image)
    assert np.array_equal(before.est, after.est)
