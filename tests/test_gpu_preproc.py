"""The pre stage on the device against the compiled
reference: adjoint gridding (grid_adjoint, preproc.cpp:167-199), the trajectory's
Toeplitz kernel (build_psf / build_psf_coords, preproc.cpp:223-290) and coil
compression (apply_compression, preproc.cpp:446-471).

The gather reproduces spread_sample's float accumulation exactly, so the gridded
k-space is compared bit for bit; after the inverse FFT (FP64 in the reference,
FP32 here) the single-operator tolerance applies.
"""
import numpy as np
import pytest

from helpers import rel_err

pytestmark = pytest.mark.gpu

OP_TOL = 1e-5


@pytest.mark.parametrize("N,J,K,delay", [(16, 3, 7, 0.0), (64, 8, 13, 0.0), (64, 8, 13, 0.37), (128, 4, 15, -0.2)])
def test_grid_spread_is_bit_identical(gpu, ref, N, J, K, delay):
    plan = gpu.raw_plan(2 * N, J)
    samples, angles = ref.phantom_series(J, 2, K, 5, N, 1e-3, 31 + N)
    with gpu.Context(plan) as ctx:
        got = ctx.grid_spread(samples[1], angles[1], delay)
    want = ref.grid_spread(plan, samples[1], angles[1], delay)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("N,J,K", [(16, 3, 7), (64, 8, 13), (128, 32, 15), (160, 4, 15)])
def test_grid_adjoint_matches_reference(gpu, ref, N, J, K):
    plan = gpu.raw_plan(2 * N, J)
    samples, angles = ref.phantom_series(J, 1, K, 5, N, 1e-3, 5 + K)
    with gpu.Context(plan) as ctx:
        got = ctx.grid_adjoint(samples[0], angles[0])
    want = ref.grid_adjoint(plan, samples[0], angles[0])
    assert rel_err(got, want) < OP_TOL
    # masked to the field-of-view window (preproc.cpp:195)
    G, L = plan.G, plan.G // 2
    lo = (G - L) // 2
    outside = np.ones((G, G), bool)
    outside[lo:lo + L, lo:lo + L] = False
    assert np.all(got[:, outside] == 0)


@pytest.mark.parametrize("N,K", [(16, 5), (64, 13), (128, 15), (160, 15), (192, 15)])
def test_build_psf_matches_reference(gpu, ref, N, K):
    plan = gpu.raw_plan(2 * N, 1)
    rng = np.random.default_rng(N + K)
    angles = rng.uniform(0, 2 * np.pi, K)
    with gpu.Context(plan) as ctx:
        got = ctx.build_psf(angles, 2 * N)
    want = ref.build_psf(plan, angles, 2 * N)
    assert rel_err(got, want) < OP_TOL


def test_build_psf_coords_matches_reference(gpu, ref):
    plan = gpu.make_plan(32, 1)
    rng = np.random.default_rng(3)
    coords = rng.uniform(-0.5, 0.5, (300, 2))
    weights = rng.uniform(0.1, 1.0, 300)
    with gpu.Context(plan) as ctx:
        got = ctx.build_psf_coords(coords, weights)
        with pytest.raises(gpu.DataError):
            ctx.build_psf_coords(np.array([[0.5, 0.0]]), np.array([1.0]))
        with pytest.raises(gpu.DataError):
            ctx.grid_adjoint(np.ones((1, 1, 4), np.complex64), np.zeros(1), delay=3.0)
    want = ref.build_psf_coords(plan, coords, weights)
    assert rel_err(got, want) < OP_TOL


def test_gridded_frame_reconstructs_like_the_reference(gpu, ref):
    # the whole chain on the device: raw samples -> z, angles -> P -> frame
    plan = gpu.make_plan(32, 4)
    plan.newton_steps, plan.cg_iter_budget = 7, 30
    samples, angles = ref.phantom_series(4, 1, 11, 5, 32, 1e-3, 77)
    zr = ref.grid_adjoint(plan, samples[0], angles[0])
    Pr = ref.build_psf(plan, angles[0], 64)
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan) as ctx:
        z = ctx.grid_adjoint(samples[0], angles[0])
        P = ctx.build_psf(angles[0], 64)
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
    img, _, per, _ = ref.reconstruct_frame(plan, zr, Pr, init)
    assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < 1e-3


def test_apply_compression_is_bit_identical(gpu, ref):
    plan = gpu.make_plan(32, 10)
    samples, angles = ref.phantom_series(16, 3, 11, 5, 32, 1e-3, 19)
    m, energy = ref.calibrate_compression(samples, angles, 10)
    want, _ = ref.compress_series(samples, angles, 10, 3)
    with gpu.Context(plan) as ctx:
        for n in range(3):
            got = ctx.apply_compression(m, samples[n])
            assert np.array_equal(got.view(np.uint32), want[n].view(np.uint32)), n
        with pytest.raises(gpu.DataError):
            ctx.apply_compression(m, samples[0][:5])


def test_psf_angle_key_is_the_reference_hash(gpu):
    # PsfCache::angle_key (preproc.cpp:301-313): FNV-1a over S, G, llround(angle * 1e9)
    angles = np.array([0.1, 1.3, 2.9])
    h = 1469598103934665603
    for v in [64, 128] + [int(np.round(a * 1e9)) for a in angles]:
        for b in range(8):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 1099511628211) % (1 << 64)
    assert gpu.psf_angle_key(angles, 64, 128) == h
