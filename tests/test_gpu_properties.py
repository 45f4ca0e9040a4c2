"""Property tests of the reference's suite that compare a reconstruction with another
reconstruction rather than with a stored answer (test_nlinv.cpp:351-368, 460-506,
545-560; test_preproc.cpp:228-251), run on the device path. Each input comes from the
compiled reference's own pre stage, as in the other parity tests."""
import numpy as np
import pytest

from helpers import random_estimate, random_image, rel_err

pytestmark = pytest.mark.gpu


def _series(gpu, plan, z, P, idx, opts):
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, z.shape[0], P.shape[0])
    s.upload_frames(z)
    for k in range(P.shape[0]):
        s.upload_psf(k, P[k])
    s.set_psf_index(idx)
    scale = s.normalize()
    out = s.run(opts)
    out["scale"] = scale
    ctx.close()
    return out


def _gridded(ref, plan, samples, angles, F, U):
    z = np.stack([ref.grid_adjoint(plan, samples[n], angles[n]) for n in range(F)])
    P = np.stack([ref.build_psf(plan, angles[n], 2 * plan.N) for n in range(min(U, F))])
    return z, P, [n % U for n in range(F)]


def test_an_overwhelming_regularizer_pins_the_update_to_its_target(gpu, ref):
    # test_nlinv.cpp:351-368: alpha = 1e8 makes the Newton update land on reg
    plan = gpu.make_plan(16, 2)
    samples, angles = ref.phantom_series(2, 2, 7, 1, 16, 0.0, 7)
    z = ref.grid_adjoint(plan, samples[0], angles[0])
    P = ref.build_psf(plan, angles[0], 2 * plan.N)
    target = random_estimate(plan, 70)
    G = plan.G
    rho = target[: G * G].reshape(G, G)
    lo, L = (G - G // 2) // 2, G // 2
    win = np.zeros_like(rho)
    win[lo:lo + L, lo:lo + L] = rho[lo:lo + L, lo:lo + L]
    target[: G * G] = win.ravel()
    target = (target * np.float32(0.1)).astype(np.complex64)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        x, _, _ = ctx.newton_step(gpu.initial_estimate(plan), target, 1e8, 1e-8, 60)
    assert rel_err(x, target) <= 1e-2


def test_data_scale_does_not_leak_into_the_output(gpu, ref):
    # test_nlinv.cpp:460-484: scaling the samples by 3.7 divides the series scale by
    # 3.7 and multiplies every output image by 3.7
    N = 16
    plan = gpu.make_plan(N, 3)
    plan.newton_steps, plan.cg_iter_budget = 4, 12
    samples, angles = ref.phantom_series(3, 5, 3, 3, N, 0.0, 3)
    z, P, idx = _gridded(ref, plan, samples, angles, 5, 3)
    opts = gpu.SeriesOptions(plain=True, sched=gpu.TemporalSchedule.for_turns(3))
    base = _series(gpu, plan, z, P, idx, opts)
    big = _series(gpu, plan, (z * np.float32(3.7)).astype(np.complex64), P, idx, opts)
    assert big["scale"] == pytest.approx(base["scale"] / 3.7, rel=1e-5)
    for n in range(5):
        assert rel_err(big["images"][n] * np.float32(1.0 / 3.7), base["images"][n]) <= 1e-2, n


def test_a_unitary_channel_rotation_leaves_the_reconstruction_unchanged(gpu, ref):
    # test_nlinv.cpp:486-506: a full-rank compression (J virtual = J physical channels)
    # is a unitary rotation of the channels; the device applies it on the raw samples
    N, J, F = 16, 3, 4
    plan = gpu.make_plan(N, J)
    plan.newton_steps, plan.cg_iter_budget = 3, 9
    samples, angles = ref.phantom_series(J, F, 5, 2, N, 1e-4, 13)
    m, _ = ref.calibrate_compression(samples, angles, J)
    opts = gpu.SeriesOptions(plain=True, sched=gpu.TemporalSchedule.for_turns(2))
    outs = []
    for cmat in (None, m):
        ctx = gpu.Context(plan)
        s = gpu.Series(ctx, F, 2)
        outs.append(s.run(opts, raw=dict(samples=samples, angles=angles, cmat=cmat)))
        ctx.close()
    for n in range(F):
        assert ref.nrmse_scaled(outs[1]["images"][n], outs[0]["images"][n], 1.0) <= 1e-3, n


def test_coil_grid_cropping_hardly_changes_the_image(gpu, ref):
    # test_nlinv.cpp:545-560: Gc = G/4 against no cropping at all (Gc = G)
    N = 24
    plan = gpu.make_plan(N, 4)
    samples, angles = ref.phantom_series(4, 1, 39, 1, N, 0.0, 17)
    z, P, idx = _gridded(ref, plan, samples, angles, 1, 1)
    opts = gpu.SeriesOptions(plain=True)
    cropped = _series(gpu, plan, z, P, idx, opts)
    full = gpu.make_plan(N, 4)
    full.Gc = full.G
    uncropped = _series(gpu, full, z, P, idx, opts)
    assert ref.nrmse_scaled(cropped["images"][0], uncropped["images"][0]) <= 0.02


def test_full_cartesian_sampling_gives_a_constant_kernel_and_identity_operator(gpu, ref):
    # test_preproc.cpp:228-251 on the device PSF builder and Toeplitz operator
    plan = gpu.raw_plan(16, 1)
    G = plan.G
    c = G // 2
    pq = np.array([(p, q) for p in range(G) for q in range(G)], np.float64)
    coords = (pq - c) / G
    weights = np.full(G * G, 1.0 / (G * G))
    x = random_image(G, 3)
    masked = np.zeros_like(x)
    lo, L = (G - G // 2) // 2, G // 2
    masked[lo:lo + L, lo:lo + L] = x[lo:lo + L, lo:lo + L]
    with gpu.Context(plan) as ctx:
        P = ctx.build_psf_coords(coords, weights)
        assert np.max(np.abs(P.real - 1.0)) < 1e-4
        assert np.max(np.abs(P.imag)) < 1e-4
        ctx.set_psf(P)
        assert rel_err(ctx.toeplitz_apply(x), masked) < 1e-5
    assert rel_err(P, ref.build_psf_coords(plan, coords, weights)) < 1e-5
