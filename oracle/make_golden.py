"""ORACLE TEST INFRASTRUCTURE — generates tests/golden/*.npz from the compiled reference.

    python oracle/make_golden.py      (needs oracle/_ref, i.e. /root/reference at build time)

The reference ships no numeric golden vectors for the NLINV path, so
these fixtures are outputs of the reference itself (oracle/_ref, built from
/root/reference/proj/src) on small seeded inputs; tests/test_golden.py checks the
numpy restatement, the compiled reference and the CUDA path against them.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
import paper_1701_08361_b200 as pb  # noqa: E402


def rimg(shape, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)).astype(np.complex64)


def main():
    out = {}
    # centered FFT (fft.cpp:37-77), even and odd sides
    for n in (9, 16, 48):
        x = rimg((n, n), 100 + n)
        out[f"fft{n}_x"] = x
        out[f"fft{n}_fwd"] = ref.fft(x, -1)
        out[f"fft{n}_inv"] = ref.fft(x, +1)
    # operator pieces at G = 32, J = 3 (raw plan, random radial PSF)
    plan = pb.raw_plan(32, 3)
    rng = np.random.default_rng(35)
    P = ref.build_psf(plan, rng.uniform(0, 2 * np.pi, 5), plan.G)
    x = np.concatenate([rimg((32, 32), 320).ravel(), rimg((3, 8, 8), 321).ravel()])
    dx = np.concatenate([rimg((32, 32), 330).ravel(), rimg((3, 8, 8), 331).ravel()])
    rhs = np.concatenate([rimg((32, 32), 340).ravel(), rimg((3, 8, 8), 341).ravel()])
    out.update(op_P=P, op_x=x, op_dx=dx, op_rhs=rhs, op_winv=ref.make_weights_inv(8, 32))
    out["op_apply_normal"] = ref.apply_normal(plan, x, dx, P)
    cx, it, res = ref.cg_solve(plan, x, rhs, P, 0.5, 0.0, 7)
    out.update(op_cg_x=cx, op_cg_iters=np.int32(it), op_cg_res=res)
    cx, it, res = ref.cg_solve(plan, x, rhs, P, 0.5, 1e-3, 200)
    out.update(op_cgtol_x=cx, op_cgtol_iters=np.int32(it), op_cgtol_res=res)
    # a phantom frame at make_plan(16, 2): G = 48, M = 4, budget 12
    fp = ref.make_plan(16, 2)
    fp.newton_steps, fp.cg_iter_budget = 4, 12
    samples, angles = ref.phantom_series(2, 1, 11, 1, 16, 0.0, 7)
    z = ref.grid_adjoint(fp, samples[0], angles[0])
    Pf = ref.build_psf(fp, angles[0], 32)
    init = ref.initial_estimate(fp)
    img, est, per, _ = ref.reconstruct_frame(fp, z, Pf, init)
    out.update(fr_z=z, fr_P=Pf, fr_init=init, fr_image=img, fr_est=est, fr_per=np.asarray(per, np.int32))
    nx, nit, r0 = ref.newton_step(fp, init, init, 1.0, z, Pf, 0.0, 3)
    out.update(ns_x=nx, ns_iters=np.int32(nit), ns_r0=np.float64(r0))
    # scheduling: h_choose on every completion state of 6 frames (non-blocking cases)
    rows = []
    M = 4
    for mask in range(1 << 6):
        comp = [(mask >> i) & 1 for i in range(6)]
        for n in range(1, 6):
            for l, o in ((1, 1), (1, 2), (2, 3), (3, 2)):
                for m in (0, M - 1):
                    pinned = n <= l or m == M - 1
                    lo = max(n - o, 0)
                    need = (n - 1) if pinned else (None if any(comp[w] for w in range(lo, n)) else lo)
                    if need is not None and not comp[need]:
                        continue
                    rows.append([mask, n, m, M, l, o, ref.h_choose(n, m, M, l, o, comp)])
    out["hchoose"] = np.asarray(rows, np.int32)
    out["legal8"] = np.asarray(ref.legal_configs(8), np.int32)
    path = os.path.join(ROOT, "tests", "golden", "nlinv_small.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
