"""Golden fixtures (tests/golden/nlinv_small.npz, generated from the compiled
reference by oracle/make_golden.py): the oracle and the numpy restatement must
reproduce them on CPU; the CUDA path must match them within the north-star
tolerances on GPU."""
import os

import numpy as np
import pytest

from helpers import rel_err

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nlinv_small.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_oracle_reproduces_goldens(ref, gold):
    for n in (9, 16, 48):
        assert np.array_equal(ref.fft(gold[f"fft{n}_x"], -1), gold[f"fft{n}_fwd"])
    import paper_1701_08361_b200 as pb
    plan = pb.raw_plan(32, 3)
    assert np.array_equal(ref.apply_normal(plan, gold["op_x"], gold["op_dx"], gold["op_P"]), gold["op_apply_normal"])
    for row in gold["hchoose"]:
        mask, n, m, M, l, o, want = (int(v) for v in row)
        comp = [(mask >> i) & 1 for i in range(6)]
        assert ref.h_choose(n, m, M, l, o, comp) == want


def test_restatement_reproduces_goldens(gold):
    from oracle import nlinv_np as o
    for n in (9, 16, 48):
        assert rel_err(o.forward(gold[f"fft{n}_x"]), gold[f"fft{n}_fwd"]) < 1e-6
    lay = o.Layout(32, 8, 3)
    sc = o.StepCache(gold["op_x"], lay, gold["op_P"], o.make_weights_inv(8, 32))
    assert rel_err(o.apply_normal(gold["op_dx"], sc), gold["op_apply_normal"]) < 1e-6
    x, it, _ = o.cg_solve(gold["op_rhs"], sc, 0.5, 0.0, 7)
    assert it == int(gold["op_cg_iters"]) and rel_err(x, gold["op_cg_x"]) < 1e-5
    for row in gold["hchoose"]:
        mask, n, m, M, l, oo, want = (int(v) for v in row)
        comp = [(mask >> i) & 1 for i in range(6)]
        src, blocked = o.h_choose_nonblocking(n, m, M, l, oo, comp)
        assert blocked is None and src == want
    assert [tuple(r) for r in gold["legal8"]] == o.legal_configs(8)


def test_host_scheduling_reproduces_goldens(gold):
    import paper_1701_08361_b200 as pb
    for row in gold["hchoose"]:
        mask, n, m, M, l, o, want = (int(v) for v in row)
        led = pb.CompletionLedger(6)
        for i in range(6):
            if (mask >> i) & 1:
                led.mark_complete(i)
        assert pb.h_choose(n, m, M, pb.TemporalSchedule(l, o), led) == want
    assert [tuple(r) for r in gold["legal8"]] == pb.legal_configs(8)


@pytest.mark.gpu
def test_cuda_path_reproduces_goldens(gpu, gold):
    pb = gpu
    for n in (9, 16, 48):
        assert rel_err(pb.fft_forward(gold[f"fft{n}_x"]), gold[f"fft{n}_fwd"]) < 1e-5
        assert rel_err(pb.fft_inverse(gold[f"fft{n}_x"]), gold[f"fft{n}_inv"]) < 1e-5
    plan = pb.raw_plan(32, 3)
    with pb.Context(plan) as ctx:
        ctx.set_psf(gold["op_P"])
        ctx.make_step_cache(gold["op_x"])
        assert rel_err(ctx.apply_normal(gold["op_dx"]), gold["op_apply_normal"]) < 1e-5
        x, it, res = ctx.cg_solve(gold["op_rhs"], 0.5, 0.0, 7)
        assert it == int(gold["op_cg_iters"]) and rel_err(x, gold["op_cg_x"]) < 1e-4
        x, it, res = ctx.cg_solve(gold["op_rhs"], 0.5, 1e-3, 200)
        assert it == int(gold["op_cgtol_iters"]) and rel_err(x, gold["op_cgtol_x"]) < 1e-4
    fp = pb.make_plan(16, 2)
    fp.newton_steps, fp.cg_iter_budget = 4, 12
    with pb.Context(fp) as ctx:
        ctx.set_psf(gold["fr_P"])
        ctx.set_data(gold["fr_z"])
        fr = ctx.reconstruct_frame(gold["fr_init"])
        assert fr.cg_per_step == list(gold["fr_per"])
        assert rel_err(fr.image, gold["fr_image"]) < 1e-3 and rel_err(fr.est, gold["fr_est"]) < 1e-3
        nx, nit, r0 = ctx.newton_step(gold["fr_init"], gold["fr_init"], 1.0, 0.0, 3)
        assert nit == int(gold["ns_iters"]) and abs(r0 - float(gold["ns_r0"])) <= 1e-5 * float(gold["ns_r0"])
        assert rel_err(nx, gold["ns_x"]) < 1e-4
