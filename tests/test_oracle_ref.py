"""Pinning the oracle (CPU, no GPU): the compiled reference passes the reference's
own known-answer tests, and the independent numpy restatement (oracle/nlinv_np.py)
agrees with the compiled reference."""
import os
import subprocess

import numpy as np
import pytest

from helpers import random_estimate, random_image, rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = ["test_fft", "test_autotune", "test_planner", "test_seqsim", "test_preproc", "test_decomp", "test_nlinv"]


@pytest.mark.parametrize("name", REF_TESTS)
def test_reference_kats_pass_on_the_oracle_build(ref, name):
    exe = os.path.join(ROOT, "oracle", "_ref", name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd=os.path.join(ROOT, "oracle", "_ref"))
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout


@pytest.fixture(scope="module")
def np_oracle():
    from oracle import nlinv_np
    return nlinv_np


def test_restated_fft_matches_reference(ref, np_oracle):
    for n in (4, 9, 16, 17, 48, 128):
        x = random_image(n, 7 + n)
        assert rel_err(np_oracle.forward(x), ref.fft(x, -1)) < 1e-6
        assert rel_err(np_oracle.inverse(x), ref.fft(x, +1)) < 1e-6


def test_restated_weights_and_pairs_match_reference(ref, np_oracle):
    for Gc, G in ((6, 24), (12, 48), (16, 16), (64, 256)):
        w = np_oracle.make_weights_inv(Gc, G)
        assert np.array_equal(w, ref.make_weights_inv(Gc, G).real)
    winv = np_oracle.make_weights_inv(8, 32)
    a = random_image(8, 1)
    u = random_image(32, 2)
    assert rel_err(np_oracle.apply_W_inv(a, winv, 32), ref.apply_W_inv(a, winv.astype(np.complex64), 32)) < 1e-6
    assert rel_err(np_oracle.apply_W_invH(u, winv, 8), ref.apply_W_invH(u, winv.astype(np.complex64), 8)) < 1e-6


@pytest.mark.parametrize("G,J", [(16, 1), (32, 3), (48, 2)])
def test_restated_apply_normal_and_cr_match_reference(ref, np_oracle, G, J):
    import paper_1701_08361_b200 as pb
    plan = pb.raw_plan(G, J)
    rng = np.random.default_rng(G + J)
    P = ref.build_psf(plan, rng.uniform(0, 2 * np.pi, 5), G)
    x = random_estimate(plan, 10 * G + J)
    dx = random_estimate(plan, 11 * G + J)
    lay = np_oracle.Layout(G, plan.Gc, J)
    sc = np_oracle.StepCache(x, lay, P, np_oracle.make_weights_inv(plan.Gc, G))
    assert rel_err(np_oracle.apply_normal(dx, sc), ref.apply_normal(plan, x, dx, P)) < 1e-6
    for tol, cap in ((0.0, 7), (1e-3, 200)):
        got, it, res = np_oracle.cg_solve(dx, sc, 0.5, tol, cap)
        want, wit, wres = ref.cg_solve(plan, x, dx, P, 0.5, tol, cap)
        assert it == wit
        assert rel_err(got, want) < 1e-5


def test_restated_frame_matches_reference(ref, np_oracle):
    plan = ref.make_plan(16, 2)
    plan.newton_steps, plan.cg_iter_budget = 4, 12
    samples, angles = ref.phantom_series(2, 1, 11, 1, 16, 0.0, 7)
    z = ref.grid_adjoint(plan, samples[0], angles[0])
    P = ref.build_psf(plan, angles[0], 32)
    init = ref.initial_estimate(plan)
    img, est, per, _ = ref.reconstruct_frame(plan, z, P, init)
    lay = np_oracle.Layout(plan.G, plan.Gc, plan.J)
    nimg, nest, nper = np_oracle.reconstruct_frame(z, P, lay, plan.N, init, lambda m: init, M=4, budget=12)
    assert nper == per == [3, 3, 3, 3]
    assert rel_err(nimg, img) < 1e-4 and rel_err(nest, est) < 1e-4


def test_restated_scheduling_and_autotune_match_reference(ref, np_oracle):
    for J in range(1, 20):
        for A in range(1, 5):
            if A <= J:
                assert np_oracle.partition_channels(J, A) == ref.partition_channels(J, A)
    for total in range(1, 10):
        assert np_oracle.legal_configs(total) == ref.legal_configs(total)
    rng = np.random.default_rng(3)
    for _ in range(200):
        db = [(int(rng.integers(0, 3)), int(rng.choice([64, 160])), int(rng.integers(0, 6)), int(rng.choice([4, 10])),
               int(rng.integers(1, 4)), int(rng.integers(1, 4)), float(rng.choice([10.0, 20.0])))
              for _ in range(int(rng.integers(0, 8)))]
        key = (int(rng.integers(0, 3)), int(rng.choice([64, 160])), int(rng.integers(0, 6)), int(rng.choice([4, 10])))
        assert np_oracle.select_config(key, db) == ref.select_config(key, db)
        assert np_oracle.learn_step(key, db) == ref.learn_step(key, db)
