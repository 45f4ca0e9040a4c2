"""Shared input builders for the parity tests (inputs come from the reference itself)."""
import numpy as np


def rel_err(got, want):
    """oracles::rel_err (tests/oracles.hpp:98-106), in double"""
    got = np.asarray(got, np.complex128).ravel()
    want = np.asarray(want, np.complex128).ravel()
    num = np.sum(np.abs(got - want) ** 2)
    den = np.sum(np.abs(want) ** 2)
    return float(np.sqrt(num / den) if den > 0 else np.sqrt(num))


def random_image(n, seed, shape=None):
    rng = np.random.default_rng(seed)
    shape = (n, n) if shape is None else shape
    return (rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)).astype(np.complex64)


def random_estimate(plan, seed):
    rho = random_image(plan.G, seed)
    chat = random_image(plan.Gc, seed + 1, (plan.J, plan.Gc, plan.Gc))
    return np.concatenate([rho.ravel(), chat.ravel()])


def radial_psf(ref, plan, K, seed):
    """test_nlinv.cpp:40-46: K random spoke angles, S = G samples per spoke"""
    rng = np.random.default_rng(seed)
    angles = rng.uniform(0.0, 2 * np.pi, K)
    return ref.build_psf(plan, angles, plan.G)


def phantom_frame_inputs(ref, plan, K, U=5, F=1, noise=0.0, seed=1234, normalize=True):
    """gridded data and PSF per frame from the reference's own pre stage (prep_series,
    nlinv.cpp:366-402), normalised so frame 0 has norm 100."""
    samples, angles = ref.phantom_series(plan.J, F, K, U, plan.N, noise, seed)
    z = np.stack([ref.grid_adjoint(plan, samples[n], angles[n]) for n in range(F)])
    P = np.stack([ref.build_psf(plan, angles[n], 2 * plan.N) for n in range(F)])
    scale = 1.0
    if normalize:
        nsq = float(np.sum(np.abs(z[0].astype(np.complex128)) ** 2))
        if nsq > 0:
            scale = 100.0 / np.sqrt(nsq)
            z = (z * np.float32(scale)).astype(np.complex64)
    return dict(samples=samples, angles=angles, z=z, P=P, scale=scale)
