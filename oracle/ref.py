"""ORACLE TEST INFRASTRUCTURE — not product code.

ctypes binding of oracle/_ref/librtnlinv_ref.so: the UNMODIFIED reference
(/root/reference/proj/src, compiled in place by oracle/Makefile) behind the flat
wrapper oracle/ref_capi.cpp. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "librtnlinv_ref.so")
REFERENCE_SRC = "/root/reference/proj"


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Plan(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int), ("G", ctypes.c_int), ("Gc", ctypes.c_int), ("J", ctypes.c_int),
        ("newton_steps", ctypes.c_int), ("alpha0", ctypes.c_float), ("alpha_q", ctypes.c_float),
        ("alpha_min", ctypes.c_float), ("cg_tol", ctypes.c_float), ("cg_max_iter", ctypes.c_int),
        ("cg_iter_budget", ctypes.c_int), ("prev_damping", ctypes.c_float), ("gamma", ctypes.c_double),
    ]


class _Opts(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int), ("A", ctypes.c_int), ("sched_l", ctypes.c_int), ("sched_o", ctypes.c_int),
                ("chain", ctypes.c_int), ("normalize", ctypes.c_int), ("delay_samples", ctypes.c_double)]


def build(quiet=True):
    """Compile the reference in place (needs /root/reference; the GPU box uses the prebuilt .so)."""
    if not os.path.isdir(REFERENCE_SRC):
        return os.path.exists(LIB_PATH)
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = ctypes.c_char_p
    return _lib


def _fp(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _dp(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _chk(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _c64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex64))


def plan_c(plan) -> _Plan:
    return _Plan(plan.N, plan.G, plan.Gc, plan.J, plan.newton_steps, plan.alpha0, plan.alpha_q, plan.alpha_min,
                 plan.cg_tol, plan.cg_max_iter, plan.cg_iter_budget, plan.prev_damping, plan.gamma)


def make_plan(N, J):
    from paper_1701_08361_b200 import ReconPlan
    p = _Plan()
    _chk(lib().ref_make_plan(N, J, ctypes.byref(p)))
    return ReconPlan(N=p.N, gamma=p.gamma, G=p.G, Gc=p.Gc, J=p.J, newton_steps=p.newton_steps, alpha0=p.alpha0,
                     alpha_q=p.alpha_q, alpha_min=p.alpha_min, cg_tol=p.cg_tol, cg_max_iter=p.cg_max_iter,
                     cg_iter_budget=p.cg_iter_budget, prev_damping=p.prev_damping)


# ---- synthetic acquisition / pre stage -------------------------------------------------
def phantom_series(J, F, K, U, N, noise=0.0, seed=7):
    """frames of default_phantom(J, seed): samples (F, J, K, 2N) complex64, angles (F, K)"""
    S = 2 * N
    samples = np.zeros((F, J, K, S), np.complex64)
    angles = np.zeros((F, K), np.float64)
    _chk(lib().ref_phantom_series(J, F, K, U, N, ctypes.c_double(noise), ctypes.c_uint64(seed), _fp(samples),
                                  _dp(angles)))
    return samples, angles


def grid_adjoint(plan, samples, angles):
    samples = _c64(samples)
    angles = np.ascontiguousarray(angles, np.float64)
    J, K, S = samples.shape
    z = np.zeros((J, plan.G, plan.G), np.complex64)
    _chk(lib().ref_grid_adjoint(ctypes.byref(plan_c(plan)), _fp(samples), _dp(angles), J, K, S, _fp(z)))
    return z


def build_psf(plan, angles, S):
    angles = np.ascontiguousarray(angles, np.float64)
    P = np.zeros((plan.G, plan.G), np.complex64)
    _chk(lib().ref_build_psf(ctypes.byref(plan_c(plan)), _dp(angles), len(angles), S, _fp(P)))
    return P


def grid_spread(plan, samples, angles, delay=0.0):
    """the density-compensated KB spread of grid_adjoint before its inverse FFT"""
    samples = _c64(samples)
    angles = np.ascontiguousarray(angles, np.float64)
    J, K, S = samples.shape
    g = np.zeros((J, plan.G, plan.G), np.complex64)
    _chk(lib().ref_grid_spread(ctypes.byref(plan_c(plan)), _fp(samples), _dp(angles), J, K, S,
                               ctypes.c_double(delay), _fp(g)))
    return g


def build_psf_coords(plan, coords, weights):
    coords = np.ascontiguousarray(coords, np.float64)
    weights = np.ascontiguousarray(weights, np.float64)
    P = np.zeros((plan.G, plan.G), np.complex64)
    _chk(lib().ref_build_psf_coords(ctypes.byref(plan_c(plan)), _dp(coords), _dp(weights), len(weights), _fp(P)))
    return P


def calibrate_compression(samples, angles, Jv):
    samples = _c64(samples)
    angles = np.ascontiguousarray(angles, np.float64)
    F, Jp, K, S = samples.shape
    m = np.zeros((Jv, Jp), np.complex64)
    energy = ctypes.c_double(0)
    _chk(lib().ref_calibrate_compression(_fp(samples), _dp(angles), F, Jp, K, S, Jv, _fp(m), ctypes.byref(energy)))
    return m, energy.value


def compress_series(samples, angles, Jv, ncal):
    samples = _c64(samples)
    angles = np.ascontiguousarray(angles, np.float64)
    F, Jp, K, S = samples.shape
    out = np.zeros((F, Jv, K, S), np.complex64)
    energy = ctypes.c_double(0)
    _chk(lib().ref_compress_series(_fp(samples), _dp(angles), F, Jp, K, S, Jv, ncal, _fp(out),
                                   ctypes.byref(energy)))
    return out, energy.value


def bandlimited_truth_rss(J, seed, n, N):
    out = np.zeros((N, N), np.complex64)
    _chk(lib().ref_bandlimited_truth_rss(J, ctypes.c_uint64(seed), n, N, _fp(out)))
    return out


def nrmse_scaled(got, want, interior=0.45):
    got, want = _c64(got), _c64(want)
    v = ctypes.c_double(0)
    _chk(lib().ref_nrmse_scaled(_fp(got), _fp(want), got.shape[0], ctypes.c_double(interior), ctypes.byref(v)))
    return v.value


# ---- primitives ------------------------------------------------------------------------------
def fft(x, sign):
    a = _c64(x).copy()
    _chk(lib().ref_fft(_fp(a), a.shape[0], sign))
    return a


def fft_counts():
    out = (ctypes.c_uint64 * 4)()
    lib().ref_fft_counts(out)
    return list(out)


def fft_reset_counts():
    lib().ref_fft_reset_counts()


def make_weights_inv(Gc, G):
    out = np.zeros((Gc, Gc), np.complex64)
    _chk(lib().ref_make_weights_inv(Gc, G, _fp(out)))
    return out


def apply_W_inv(chat, winv, G):
    chat, winv = _c64(chat), _c64(winv)
    out = np.zeros((G, G), np.complex64)
    _chk(lib().ref_apply_W_inv(_fp(chat), _fp(winv), chat.shape[0], G, _fp(out)))
    return out


def apply_W_invH(u, winv, Gc):
    u, winv = _c64(u), _c64(winv)
    out = np.zeros((Gc, Gc), np.complex64)
    _chk(lib().ref_apply_W_invH(_fp(u), _fp(winv), u.shape[0], Gc, _fp(out)))
    return out


def toeplitz_apply(x, P):
    a = _c64(x).copy()
    _chk(lib().ref_toeplitz_apply(_fp(a), _fp(_c64(P)), a.shape[0]))
    return a


def make_step_cache(plan, x, P):
    rho = np.zeros((plan.G, plan.G), np.complex64)
    coils = np.zeros((plan.J, plan.G, plan.G), np.complex64)
    _chk(lib().ref_make_step_cache(ctypes.byref(plan_c(plan)), _fp(_c64(x)), _fp(_c64(P)), _fp(rho), _fp(coils)))
    return rho, coils


def apply_normal(plan, x, dx, P, A=1):
    out = np.zeros_like(_c64(dx))
    _chk(lib().ref_apply_normal(ctypes.byref(plan_c(plan)), _fp(_c64(x)), _fp(_c64(dx)), _fp(_c64(P)), A, _fp(out)))
    return out


def cg_solve(plan, x, rhs, P, alpha, tol, max_iter):
    out = np.zeros_like(_c64(rhs))
    iters = ctypes.c_int(0)
    res = np.zeros(max(max_iter, 1), np.float64)
    _chk(lib().ref_cg_solve(ctypes.byref(plan_c(plan)), _fp(_c64(x)), _fp(_c64(rhs)), _fp(_c64(P)),
                            ctypes.c_float(alpha), ctypes.c_float(tol), max_iter, _fp(out), ctypes.byref(iters),
                            _dp(res)))
    return out, iters.value, res[:iters.value].copy()


def newton_step(plan, x, reg, alpha, z, P, cg_tol, cg_max_iter):
    xx = _c64(x).copy()
    iters = ctypes.c_int(0)
    r0 = ctypes.c_double(0)
    _chk(lib().ref_newton_step(ctypes.byref(plan_c(plan)), _fp(xx), _fp(_c64(reg)), ctypes.c_float(alpha),
                               _fp(_c64(z)), _fp(_c64(P)), ctypes.c_float(cg_tol), cg_max_iter, ctypes.byref(iters),
                               ctypes.byref(r0)))
    return xx, iters.value, r0.value


def initial_estimate(plan):
    out = np.zeros(plan.G * plan.G + plan.J * plan.Gc * plan.Gc, np.complex64)
    _chk(lib().ref_initial_estimate(ctypes.byref(plan_c(plan)), _fp(out)))
    return out


def reconstruct_frame(plan, z, P, init, reg=None, A=1):
    img = np.zeros((plan.N, plan.N), np.complex64)
    est = np.zeros_like(_c64(init))
    per = np.zeros(max(plan.newton_steps, 1), np.int32)
    secs = ctypes.c_double(0)
    _chk(lib().ref_reconstruct_frame(ctypes.byref(plan_c(plan)), _fp(_c64(z)), _fp(_c64(P)), _fp(_c64(init)),
                                     _fp(None if reg is None else _c64(reg)), A, _fp(img), _fp(est), _ip(per),
                                     ctypes.byref(secs)))
    return img, est, per[:plan.newton_steps].tolist(), secs.value


def reconstruct_frame_regs(plan, z, P, init, regs, A=1):
    """frame with a per-step regularisation target regs[m] (audit replay); A WorkerGroup
    lanes (bit-identical results for every A, test_decomp.cpp:309-326)"""
    regs = _c64(np.stack([_c64(r) for r in regs]))
    img = np.zeros((plan.N, plan.N), np.complex64)
    est = np.zeros_like(_c64(init))
    per = np.zeros(max(plan.newton_steps, 1), np.int32)
    _chk(lib().ref_reconstruct_frame_regs(ctypes.byref(plan_c(plan)), _fp(_c64(z)), _fp(_c64(P)), _fp(_c64(init)),
                                          _fp(regs), A, _fp(img), _fp(est), _ip(per)))
    return img, est, per[:plan.newton_steps].tolist()


def reconstruct_series(plan, samples, angles, T=1, A=1, sched=(1, 1), chain=True, normalize=True, plain=False):
    samples = _c64(samples)
    angles = np.ascontiguousarray(angles, np.float64)
    F, J, K, S = samples.shape
    M = plan.newton_steps
    images = np.zeros((F, plan.N, plan.N), np.complex64)
    audit = np.zeros((F, 5 + M), np.int32)
    seqs = np.zeros((F, 3), np.uint64)
    cg = np.zeros(F, np.int32)
    secs = np.zeros(F, np.float64)
    scale = ctypes.c_double(0)
    o = _Opts(T, A, sched[0], sched[1], int(chain), int(normalize), 0.0)
    _chk(lib().ref_reconstruct_series(ctypes.byref(plan_c(plan)), ctypes.byref(o), _fp(samples), _dp(angles), F, K,
                                      S, int(plain), _fp(images), _ip(audit),
                                      seqs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _ip(cg), _dp(secs),
                                      ctypes.byref(scale)))
    return dict(images=images, audit=audit, seqs=seqs, cg_iters=cg, seconds=secs, data_scale=scale.value)


def psf_cache_save(plan, angle_sets, S, path):
    a = np.ascontiguousarray(angle_sets, np.float64)
    _chk(lib().ref_psf_cache_save(ctypes.byref(plan_c(plan)), _dp(a), a.shape[0], a.shape[1], S, str(path).encode()))


def psf_cache_get(plan, path, angles, S):
    """(P, hits, size) after loading the sidecar and asking for one angle set"""
    a = np.ascontiguousarray(angles, np.float64)
    P = np.zeros((plan.G, plan.G), np.complex64)
    hits, size = ctypes.c_int(0), ctypes.c_int(0)
    _chk(lib().ref_psf_cache_get(ctypes.byref(plan_c(plan)), str(path).encode(), _dp(a), len(a), S, _fp(P),
                                 ctypes.byref(hits), ctypes.byref(size)))
    return P, hits.value, size.value


# ---- planner / postprocessing -------------------------------------------------------------------
def select_grid(N, table, gamma_min=1.4, gamma_max=2.0):
    sizes = np.array(sorted(table), np.int32)
    us = np.array([table[k] for k in sorted(table)], np.float64)
    G = ctypes.c_int(0)
    gamma = ctypes.c_double(0)
    _chk(lib().ref_select_grid(N, _ip(sizes), _dp(us), len(sizes), ctypes.c_double(gamma_min),
                               ctypes.c_double(gamma_max), ctypes.byref(G), ctypes.byref(gamma)))
    return G.value, gamma.value


def table_roundtrip(path, table):
    sizes = np.array(sorted(table), np.int32)
    us = np.array([table[k] for k in sorted(table)], np.float64)
    so = np.zeros(len(sizes) + 1, np.int32)
    uo = np.zeros(len(sizes) + 1, np.float64)
    n = ctypes.c_int(0)
    _chk(lib().ref_table_roundtrip(str(path).encode(), _ip(sizes), _dp(us), len(sizes), _ip(so), _dp(uo),
                                   ctypes.byref(n)))
    return {int(so[i]): float(uo[i]) for i in range(n.value)}


def magnitude_image(img):
    img = _c64(img)
    out = np.zeros(img.shape, np.float32)
    _chk(lib().ref_magnitude_image(_fp(img), img.shape[0], _fp(out)))
    return out


def phase_difference_image(even, odd):
    even, odd = _c64(even), _c64(odd)
    out = np.zeros(even.shape, np.float32)
    _chk(lib().ref_phase_difference_image(_fp(even), _fp(odd), even.shape[0], _fp(out)))
    return out


def median_filter(mags):
    mags = np.ascontiguousarray(mags, np.float32)
    out = np.zeros_like(mags)
    _chk(lib().ref_median_filter(_fp(mags), mags.shape[0], mags.shape[1], _fp(out)))
    return out


# ---- decomposition / autotune --------------------------------------------------------------
def partition_channels(J, A):
    out = np.zeros(2 * max(A, 1), np.int32)
    _chk(lib().ref_partition_channels(J, A, _ip(out)))
    return [(int(out[2 * a]), int(out[2 * a + 1])) for a in range(A)]


def h_choose(n, m, M, l, o, completed, late=None, delay_ms=30):
    comp = np.ascontiguousarray(np.asarray(completed, np.int32))
    lt = None if late is None else np.ascontiguousarray(np.asarray(list(late) + [-1], np.int32))
    out = ctypes.c_int(0)
    _chk(lib().ref_h_choose(n, m, M, l, o, _ip(comp), len(comp), _ip(lt), delay_ms, ctypes.byref(out)))
    return out.value


def legal_configs(total):
    buf = np.zeros(2 * 128, np.int32)
    n = lib().ref_legal_configs(total, _ip(buf), 128)
    if n < 0:
        raise RefError(-n, lib().ref_last_error().decode())
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n)]


def frames_bucket(frames):
    out = ctypes.c_int(0)
    _chk(lib().ref_frames_bucket(frames, ctypes.byref(out)))
    return out.value


def _records(db):
    rows = np.zeros((max(len(db), 1), 6), np.int32)
    ms = np.zeros(max(len(db), 1), np.float64)
    for i, r in enumerate(db):
        rows[i] = [r[0], r[1], r[2], r[3], r[4], r[5]]
        ms[i] = r[6]
    return rows, ms


def select_config(key, db):
    rows, ms = _records(db)
    k = np.asarray(key, np.int32)
    out = np.zeros(2, np.int32)
    _chk(lib().ref_select_config(_ip(k), _ip(rows), _dp(ms), len(db), _ip(out)))
    return int(out[0]), int(out[1])


def learn_step(key, db, total=8):
    rows, ms = _records(db)
    k = np.asarray(key, np.int32)
    out = np.zeros(2, np.int32)
    _chk(lib().ref_learn_step(_ip(k), _ip(rows), _dp(ms), len(db), total, _ip(out)))
    return int(out[0]), int(out[1])


def time_series(plan, z, P, psf_idx, T, A, sched, first=0, ests=None):
    """the reference's scheduled series driver on pre-gridded, normalised frames (bench
    reference arm). Frames [0, first) are taken as complete with estimates ests[:first]
    (a continuing series); frames [first, F) run with T threads x A lanes. Returns wall
    seconds, per-frame latency seconds, CR iterations and the (updated) estimates."""
    z = _c64(z)
    P = _c64(P)
    if P.ndim == 2:
        P = P[None]
    F = z.shape[0]
    D = plan.G * plan.G + plan.J * plan.Gc * plan.Gc
    ests = np.zeros((F, D), np.complex64) if ests is None else np.ascontiguousarray(ests, np.complex64)
    idx = np.ascontiguousarray(np.asarray(psf_idx, np.int32))
    wall = ctypes.c_double(0)
    lat = np.zeros(F, np.float64)
    cg = np.zeros(F, np.int32)
    _chk(lib().ref_time_series(ctypes.byref(plan_c(plan)), _fp(z), _fp(P), P.shape[0], _ip(idx), F, int(first),
                               int(T), int(A), int(sched[0]), int(sched[1]), _fp(ests), ctypes.byref(wall), _dp(lat),
                               _ip(cg)))
    return wall.value, lat[first:], cg[first:], ests


def rti_write(path, header, records, pixels):
    """the reference's RtiWriter: header = 9 ints (DatasetHeader), records [(frame, slice,
    kind)], pixels (n, N, N) float32"""
    h = np.ascontiguousarray(header, np.int32)
    rec = np.asarray(records, np.int32).reshape(-1, 3)
    px = np.ascontiguousarray(pixels, np.float32)
    fr, sl, kd = (np.ascontiguousarray(rec[:, k]) for k in range(3))
    _chk(lib().ref_rti_write(str(path).encode(), _ip(h), len(rec), _ip(fr), _ip(sl), _ip(kd),
                             px.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))


def rti_read(path, max_records=4096):
    """the reference's RtiReader: (header 9 ints, records [(frame, slice, kind)], pixels)"""
    h = np.zeros(9, np.int32)
    n = ctypes.c_int(0)
    probe = np.zeros(3, np.int32)
    _chk(lib().ref_rti_read(str(path).encode(), _ip(h), 0, ctypes.byref(n), _ip(probe), None))
    N = int(h[1])
    cnt = min(n.value, max_records)
    rec = np.zeros((max(cnt, 1), 3), np.int32)
    px = np.zeros((max(cnt, 1), N, N), np.float32)
    _chk(lib().ref_rti_read(str(path).encode(), _ip(h), cnt, ctypes.byref(n), _ip(rec),
                            px.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
    return h.tolist(), [tuple(int(v) for v in r) for r in rec[:cnt]], px[:cnt]
