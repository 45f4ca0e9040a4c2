"""ORACLE TEST INFRASTRUCTURE — not product code.

A numpy restatement of the reference's NLINV hot path (/root/reference/proj),
independent of the compiled reference, used as a second checker. Storage is
complex64 like rtnlinv::CImage; transforms run in float64 and round to float32 at
the same points as the reference (fft.cpp:62-74); dots and norms accumulate in
float64 (types.hpp:47-59). Every function cites the reference lines it follows.
Only tests/ may import this module. It is pinned against oracle/_ref by
tests/test_oracle_ref.py.
"""
from __future__ import annotations

import numpy as np

c64 = np.complex64


def dc(n):  # types.hpp:43
    return n // 2


# ---- fft.cpp:37-77: centered unitary transform, DC at n/2, 1/n scale -------------------
def fft_centered(x, sign):
    n = x.shape[0]
    c = n // 2
    a = np.roll(np.roll(x.astype(np.complex128), -c, axis=0), -c, axis=1)  # load roll
    if sign < 0:
        y = np.fft.fft2(a)
    else:
        y = np.fft.ifft2(a) * (n * n)
    y = np.roll(np.roll(y, c, axis=0), c, axis=1) / n  # store roll + scale
    return y.astype(c64)


def forward(x):
    return fft_centered(x, -1)


def inverse(x):
    return fft_centered(x, +1)


# ---- planner.cpp:187-207 ------------------------------------------------------------------
def crop_k(x, Gc):
    off = dc(x.shape[0]) - dc(Gc)
    return x[off:off + Gc, off:off + Gc].copy()


def pad_k(x, G):
    off = dc(G) - dc(x.shape[0])
    out = np.zeros((G, G), c64)
    out[off:off + x.shape[0], off:off + x.shape[0]] = x
    return out


# ---- preproc.cpp:152-165, 292-299 -------------------------------------------------------------
def window_mask(G):
    L = G // 2
    lo = (G - L) // 2
    m = np.zeros((G, G), bool)
    m[lo:lo + L, lo:lo + L] = True
    return m


def mask_window(x):
    y = x.copy()
    y[~window_mask(x.shape[0])] = 0
    return y


def toeplitz_apply(x, P):
    t = forward(mask_window(x))
    t = (t * P).astype(c64)
    return mask_window(inverse(t))


# ---- nlinv.cpp:101-133 -------------------------------------------------------------------------
def make_weights_inv(Gc, G):
    c = dc(Gc)
    r = np.arange(Gc)
    ky = (r[:, None] - c) / G
    kx = (r[None, :] - c) / G
    w = (1.0 + 880.0 * (kx * kx + ky * ky)) ** 16
    return (1.0 / w).astype(np.float32)  # real part only


def apply_W_inv(chat, winv, G):
    t = (chat * winv).astype(c64)
    return inverse(pad_k(t, G))


def apply_W_invH(u, winv, Gc):
    t = crop_k(forward(u), Gc)
    return (t * winv).astype(c64)


# ---- Estimate helpers (nlinv.cpp:60-99), flat layout rho | chat_0 | ... -------------------------
class Layout:
    def __init__(self, G, Gc, J):
        self.G, self.Gc, self.J = G, Gc, J
        self.D = G * G + J * Gc * Gc

    def split(self, e):
        G, Gc, J = self.G, self.Gc, self.J
        return e[:G * G].reshape(G, G), e[G * G:].reshape(J, Gc, Gc)

    def join(self, rho, chat):
        return np.concatenate([rho.ravel(), chat.ravel()]).astype(c64)


def est_axpy(y, a, x):  # y += float(a) * x  (nlinv.cpp:77-81)
    af = np.float32(a)
    return (y + (af * x).astype(c64)).astype(c64)


def est_scale(e, a):
    return (e * np.float32(a)).astype(c64)


def est_dot(a, b):
    return complex(np.sum(np.conj(a.astype(np.complex128)) * b.astype(np.complex128)))


def est_nrm2sq(e):
    e = e.astype(np.complex128)
    return float(np.sum(e.real * e.real + e.imag * e.imag))


def initial_estimate(lay):
    rho = np.zeros((lay.G, lay.G), c64)
    rho[window_mask(lay.G)] = 1
    return lay.join(rho, np.zeros((lay.J, lay.Gc, lay.Gc), c64))


# ---- StepCache, apply_normal (nlinv.cpp:135-177) --------------------------------------------------
class StepCache:
    def __init__(self, x, lay, P, winv):
        rho, chat = lay.split(x)
        self.lay, self.P, self.winv = lay, P, winv
        self.rho = mask_window(rho)
        self.coils = [apply_W_inv(chat[j], winv, lay.G) for j in range(lay.J)]


def apply_normal(dx, sc):
    lay = sc.lay
    drho, dchat = lay.split(dx)
    acc = np.zeros((lay.G, lay.G), np.complex128)  # all_reduce_sum in channel order (decomp.cpp:26-39)
    out_chat = np.zeros((lay.J, lay.Gc, lay.Gc), c64)
    for j in range(lay.J):
        cj = sc.coils[j]
        t = apply_W_inv(dchat[j], sc.winv, lay.G)
        t = ((cj * drho).astype(c64) + (sc.rho * t).astype(c64)).astype(c64)
        t = toeplitz_apply(t, sc.P)
        rc = (np.conj(cj) * t).astype(c64)
        rt = (np.conj(sc.rho) * t).astype(c64)
        acc += rc.astype(np.complex128)
        out_chat[j] = apply_W_invH(rt, sc.winv, lay.Gc)
    return lay.join(acc.astype(c64), out_chat)


# ---- cg_solve: conjugate residual (nlinv.cpp:179-234) ---------------------------------------------
class SolverError(RuntimeError):
    pass


def cg_solve(rhs, sc, alpha, tol, max_iter):
    alpha = np.float32(alpha)
    tol = np.float32(tol)
    x = np.zeros_like(rhs)
    rhs_norm = np.sqrt(est_nrm2sq(rhs))
    if not np.isfinite(rhs_norm):
        raise SolverError("cg_solve: right-hand side is not finite")
    if max_iter < 1 or rhs_norm == 0.0:
        return x, 0, []

    def apply(p):
        return est_axpy(apply_normal(p, sc), float(alpha), p)

    r = rhs.copy()
    p = r.copy()
    ar = apply(r)
    ap = ar.copy()
    r_ar = est_dot(r, ar).real
    target = float(tol) * rhs_norm
    res, iters = [], 0
    for it in range(1, max_iter + 1):
        denom = est_nrm2sq(ap)
        if not np.isfinite(denom) or not np.isfinite(r_ar):
            raise SolverError("cg_solve: iteration diverged")
        if denom <= 0.0 and tol > 0:
            break
        if denom > 0.0:
            a = r_ar / denom
            x = est_axpy(x, a, p)
            r = est_axpy(r, -a, ap)
        rn = np.sqrt(est_nrm2sq(r))
        if not np.isfinite(rn):
            raise SolverError("cg_solve: residual is not finite")
        res.append(rn)
        iters = it
        if tol > 0 and (rn == 0.0 or rn <= target):
            break
        if it == max_iter:
            break
        ar_next = apply(r)
        r_ar_next = est_dot(r, ar_next).real
        b = r_ar_next / r_ar if r_ar != 0.0 else 0.0
        p = est_axpy(est_scale(p, b), 1.0, r)
        ap = est_axpy(est_scale(ap, b), 1.0, ar_next)
        r_ar = r_ar_next
    return x, iters, res


# ---- newton_step, reconstruct_frame (nlinv.cpp:236-335) ------------------------------------------
def newton_step(x, reg, alpha, z, P, lay, winv, cg_tol, cg_max_iter, damping=1.0):
    sc = StepCache(x, lay, P, winv)
    acc = np.zeros((lay.G, lay.G), np.complex128)
    rhs_chat = np.zeros((lay.J, lay.Gc, lay.Gc), c64)
    rsq = 0.0
    for j in range(lay.J):
        cj = sc.coils[j]
        e = toeplitz_apply((sc.rho * cj).astype(c64), P)
        e = (z[j] - e).astype(c64)
        rsq += est_nrm2sq(e)
        acc += (np.conj(cj) * e).astype(c64).astype(np.complex128)
        rhs_chat[j] = apply_W_invH((np.conj(sc.rho) * e).astype(c64), winv, lay.Gc)
    rhs = lay.join(acc.astype(c64), rhs_chat)
    rhs = est_axpy(rhs, -float(np.float32(alpha)), x)
    rhs = est_axpy(rhs, float(np.float32(alpha)) * float(np.float32(damping)), reg)
    dx, iters, _ = cg_solve(rhs, sc, alpha, cg_tol, cg_max_iter)
    return est_axpy(x, 1.0, dx), iters, float(np.sqrt(rsq))


def reconstruct_frame(z, P, lay, N, init, reg_fn, M=7, alpha0=1.0, q=0.5, alpha_min=1e-6, cg_tol=1e-3,
                      cg_max_iter=200, budget=0):
    winv = make_weights_inv(lay.Gc, lay.G)
    x = init.copy()
    alpha = np.float32(alpha0)
    remaining = budget
    per = []
    for m in range(M):
        cap, tol = cg_max_iter, np.float32(cg_tol)
        if budget > 0:
            cap = (remaining + (M - m) - 1) // (M - m)
            tol = np.float32(0)
        x, it, _ = newton_step(x, reg_fn(m), alpha, z, P, lay, winv, tol, cap)
        per.append(it)
        if budget > 0:
            remaining -= it
        alpha = max(np.float32(alpha * np.float32(q)), np.float32(alpha_min))
    rho, chat = lay.split(x)
    acc = np.zeros((lay.G, lay.G), np.float64)
    for j in range(lay.J):
        cj = apply_W_inv(chat[j], winv, lay.G).astype(np.complex128)
        acc += cj.real * cj.real + cj.imag * cj.imag
    comb = (rho * np.sqrt(acc).astype(np.float32)).astype(c64)
    o = dc(lay.G) - dc(N)
    return comb[o:o + N, o:o + N].copy(), x, per


# ---- decomposition / scheduling (decomp.cpp:10-24, 193-209) ----------------------------------------
def partition_channels(J, A, cap=4):
    if A < 1 or A > cap or A > J:
        raise ValueError("partition_channels: worker count out of range")
    base, rem = divmod(J, A)
    out, b = [], 0
    for a in range(A):
        s = base + (1 if a < rem else 0)
        out.append((b, b + s))
        b += s
    return out


def h_choose_nonblocking(n, m, M, l, o, completed):
    """h(n, m) given the completed set; returns (source, blocked_on or None)"""
    if n < 1:
        raise ValueError("h_choose: defined for n >= 1 only")
    if n <= l or m == M - 1:
        return n - 1, (None if completed[n - 1] else n - 1)
    lo = max(n - o, 0)
    for w in range(n - 1, lo - 1, -1):
        if completed[w]:
            return w, None
    return lo, lo


# ---- autotune.cpp:40-88 -----------------------------------------------------------------------------
def legal_configs(total=8, a_cap=4):
    return [(T, A) for A in range(1, min(a_cap, total) + 1) for T in range(1, total // A + 1)]


def select_config(key, db):
    same = [r for r in db if r[0] == key[0]]
    if not same:
        return (1, 1)
    dist = lambda k: (abs(k[1] - key[1]), abs(k[2] - key[2]), abs(k[3] - key[3]), tuple(k))  # noqa: E731
    chosen = min((tuple(r[:4]) for r in same), key=dist)
    best = None
    for r in db:
        if tuple(r[:4]) != chosen:
            continue
        if best is None or r[6] < best[6] or (r[6] == best[6] and (r[5], r[4]) < (best[5], best[4])):
            best = r
    return best[4], best[5]


def learn_step(key, db, total=8, a_cap=4):
    seen = {(r[4], r[5]) for r in db if tuple(r[:4]) == tuple(key)}
    for c in legal_configs(total, a_cap):
        if c not in seen:
            return c
    return select_config(key, db)
