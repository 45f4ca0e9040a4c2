"""B200-native NLINV (arXiv 1701.08361) hot path — Python host mirror.

The product is the sm_100a library ``librtnlinv_b200.so`` (built in-tree by
``build.py``) behind the C ABI ``include/rtnlinv_b200.h``. This module binds that
ABI with ctypes and mirrors the reference's C++ operator / frame API
(proj/include/rtnlinv/nlinv.hpp, fft.hpp) with the same names, argument meaning
and error types, so the parity tests read like the reference's own tests.

There is no CPU fallback: importing works anywhere, but every compute call goes
through the CUDA library and raises ``RuntimeError`` when it is missing or no
GPU is visible.
"""
from __future__ import annotations

import ctypes
import weakref
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RTN_LIB", os.path.join(_HERE, "librtnlinv_b200.so"))

__all__ = [
    "ReconPlan", "Context", "UsageError", "DataError", "SolverError", "DecompFault",
    "make_plan", "raw_plan", "make_weights_inv", "fft_forward", "fft_inverse",
    "fft_counts", "fft_reset_counts", "FftCtx", "est_dim", "est_split", "est_join",
    "initial_estimate", "load_library", "library_loaded",
]


# ---- error taxonomy (types.hpp:12-25) --------------------------------------------
class UsageError(RuntimeError):
    pass


class DataError(RuntimeError):
    pass


class SolverError(RuntimeError):
    pass


class DecompFault(RuntimeError):
    pass


_ERRORS = {2: UsageError, 3: DataError, 4: SolverError}

# rtn_reg_provider: const float* (*)(int m, void* user)
_REG_PROVIDER = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


class _Plan(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int), ("G", ctypes.c_int), ("Gc", ctypes.c_int), ("J", ctypes.c_int),
        ("newton_steps", ctypes.c_int), ("alpha0", ctypes.c_float), ("alpha_q", ctypes.c_float),
        ("alpha_min", ctypes.c_float), ("cg_tol", ctypes.c_float), ("cg_max_iter", ctypes.c_int),
        ("cg_iter_budget", ctypes.c_int), ("prev_damping", ctypes.c_float), ("gamma", ctypes.c_double),
    ]


class _SeriesOpts(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int), ("A", ctypes.c_int), ("sched_l", ctypes.c_int), ("sched_o", ctypes.c_int),
                ("chain", ctypes.c_int), ("normalize", ctypes.c_int), ("plain", ctypes.c_int),
                ("cluster", ctypes.c_int)]


@dataclass
class ReconPlan:
    """rtnlinv::ReconPlan (planner.hpp:21-35) with the reference defaults."""
    N: int = 0
    gamma: float = 1.5
    G: int = 0
    Gc: int = 0
    J: int = 1
    newton_steps: int = 6
    alpha0: float = 1.0
    alpha_q: float = 0.5
    alpha_min: float = 1e-6
    cg_tol: float = 1e-3
    cg_max_iter: int = 200
    cg_iter_budget: int = 0
    prev_damping: float = 1.0

    def to_c(self) -> _Plan:
        return _Plan(self.N, self.G, self.Gc, self.J, self.newton_steps, self.alpha0, self.alpha_q,
                     self.alpha_min, self.cg_tol, self.cg_max_iter, self.cg_iter_budget,
                     self.prev_damping, self.gamma)

    @property
    def D(self) -> int:
        return est_dim(self)


def raw_plan(G: int, J: int) -> ReconPlan:
    """The tests' raw plan: N = G/2, Gc = G/4 (test_nlinv.cpp:22-29)."""
    return ReconPlan(N=G // 2, G=G, Gc=G // 4, J=J)


def _even_ceil(x: float) -> int:
    import math
    v = int(math.ceil(x - 1e-9))
    return v + 1 if v % 2 else v


def make_plan(N: int, J: int) -> ReconPlan:
    """make_plan without a lookup table: G = even_ceil(3N), Gc = floor(G/4) (planner.cpp:126-140)."""
    G = _even_ceil(2.0 * 1.5 * N)
    return ReconPlan(N=N, J=J, G=G, gamma=G / (2.0 * N), Gc=G // 4)


# ---- library loading ------------------------------------------------------------
_lib = None


def load_library(path: str = LIB_PATH):
    """Load the sm_100a library (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA library not built: {path} (run python -m paper_1701_08361_b200.build)")
    lib = ctypes.CDLL(path)
    f = ctypes.POINTER(ctypes.c_float)
    d = ctypes.POINTER(ctypes.c_double)
    i = ctypes.POINTER(ctypes.c_int)
    vp = ctypes.c_void_p
    sig = {
        "rtn_abi_version": ([], ctypes.c_int),
        "rtn_last_error": ([], ctypes.c_char_p),
        "rtn_grid_supported": ([ctypes.c_int], ctypes.c_int),
        "rtn_device_count": ([], ctypes.c_int),
        "rtn_ctx_create": ([ctypes.POINTER(_Plan), ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "rtn_ctx_destroy": ([vp], None),
        "rtn_ctx_create_group": ([ctypes.POINTER(_Plan), i, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
                                 ctypes.c_int),
        "rtn_ctx_group_blocks": ([vp, i], ctypes.c_int),
        "rtn_ctx_create_proc_member": ([ctypes.POINTER(_Plan), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(vp)], ctypes.c_int),
        "rtn_ctx_proc_handles": ([vp, vp, i], ctypes.c_int),
        "rtn_ctx_proc_attach": ([vp, vp, ctypes.c_int], ctypes.c_int),
        "rtn_grid_adjoint": ([vp, f, ctypes.c_int, d, ctypes.c_int, ctypes.c_int, ctypes.c_double, f], ctypes.c_int),
        "rtn_grid_spread": ([vp, f, ctypes.c_int, d, ctypes.c_int, ctypes.c_int, ctypes.c_double, f], ctypes.c_int),
        "rtn_build_psf": ([vp, d, ctypes.c_int, ctypes.c_int, f], ctypes.c_int),
        "rtn_build_psf_coords": ([vp, d, d, ctypes.c_int, f], ctypes.c_int),
        "rtn_apply_compression": ([vp, f, ctypes.c_int, ctypes.c_int, f, ctypes.c_int, f], ctypes.c_int),
        "rtn_psf_angle_key": ([d, ctypes.c_int, ctypes.c_int, ctypes.c_int], ctypes.c_uint64),
        "rtn_benchmark_fft": ([i, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, d], ctypes.c_int),
        "rtn_select_grid": ([ctypes.c_int, i, d, ctypes.c_int, ctypes.c_double, ctypes.c_double, i, d], ctypes.c_int),
        "rtn_fft_table_save": ([ctypes.c_char_p, i, d, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p], ctypes.c_int),
        "rtn_fft_table_load": ([ctypes.c_char_p, i, d, ctypes.c_int, i, ctypes.c_char_p, ctypes.c_char_p,
                                ctypes.c_int], ctypes.c_int),
        "rtn_post_magnitude": ([f, ctypes.c_longlong, f], ctypes.c_int),
        "rtn_post_phase_difference": ([f, f, ctypes.c_longlong, f], ctypes.c_int),
        "rtn_post_median3": ([f, ctypes.c_int, ctypes.c_longlong, f], ctypes.c_int),
        "rtn_series_post": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, f], ctypes.c_int),
        "rtn_fft2": ([f, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "rtn_fft_set_ctx": ([ctypes.c_int], None),
        "rtn_fft_get_ctx": ([], ctypes.c_int),
        "rtn_fft_counts": ([ctypes.POINTER(ctypes.c_uint64)], None),
        "rtn_fft_reset_counts": ([], None),
        "rtn_make_weights_inv": ([ctypes.c_int, ctypes.c_int, f], ctypes.c_int),
        "rtn_set_psf": ([vp, f], ctypes.c_int),
        "rtn_set_data": ([vp, f], ctypes.c_int),
        "rtn_apply_W_inv": ([vp, f, f], ctypes.c_int),
        "rtn_apply_W_invH": ([vp, f, f], ctypes.c_int),
        "rtn_toeplitz_apply": ([vp, f], ctypes.c_int),
        "rtn_make_step_cache": ([vp, f, f, f], ctypes.c_int),
        "rtn_apply_normal": ([vp, f, f], ctypes.c_int),
        "rtn_cg_solve": ([vp, f, ctypes.c_float, ctypes.c_float, ctypes.c_int, f, i, d], ctypes.c_int),
        "rtn_newton_step": ([vp, f, f, ctypes.c_float, ctypes.c_float, ctypes.c_int, i, d], ctypes.c_int),
        "rtn_reconstruct_frame": ([vp, f, f, f, f, i, d], ctypes.c_int),
        "rtn_all_reduce_sum": ([f, ctypes.c_int, ctypes.c_int, f], ctypes.c_int),
        "rtn_reconstruct_frame_provider": ([vp, f, _REG_PROVIDER, vp, f, f, i, d], ctypes.c_int),
        "rtn_series_create": ([vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "rtn_series_destroy": ([vp], None),
        "rtn_series_create_multi": ([vp, ctypes.c_int, ctypes.c_int, i, ctypes.c_int, ctypes.POINTER(vp)],
                                    ctypes.c_int),
        "rtn_series_upload_frames": ([vp, ctypes.c_int, ctypes.c_int, vp], ctypes.c_int),
        "rtn_series_upload_psf": ([vp, ctypes.c_int, f], ctypes.c_int),
        "rtn_series_set_psf_index": ([vp, i], ctypes.c_int),
        "rtn_series_normalize": ([vp, d], ctypes.c_int),
        "rtn_series_run": ([vp, ctypes.POINTER(_SeriesOpts), ctypes.c_int, ctypes.c_int, vp, vp, i,
                            ctypes.POINTER(ctypes.c_uint64), i, f], ctypes.c_int),
        "rtn_series_images": ([vp, ctypes.c_int, ctypes.c_int, f], ctypes.c_int),
        "rtn_series_run_raw": ([vp, ctypes.POINTER(_SeriesOpts), ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int,
                                ctypes.c_int, ctypes.c_double, vp, ctypes.c_int, vp, i,
                                ctypes.POINTER(ctypes.c_uint64), i, f], ctypes.c_int),
        "rtn_series_psf_cache_size": ([vp], ctypes.c_int),
        "rtn_series_psf_cache_save": ([vp, ctypes.c_char_p], ctypes.c_int),
        "rtn_series_psf_cache_load": ([vp, ctypes.c_char_p], ctypes.c_int),
        "rtn_series_estimate": ([vp, ctypes.c_int, f], ctypes.c_int),
        "rtn_series_last_span_ms": ([vp], ctypes.c_float),
        "rtn_partition_channels": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, i], ctypes.c_int),
        "rtn_ledger_create": ([ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "rtn_ledger_destroy": ([vp], None),
        "rtn_ledger_mark_step": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "rtn_ledger_mark_complete": ([vp, ctypes.c_int], ctypes.c_int),
        "rtn_ledger_completed": ([vp, ctypes.c_int], ctypes.c_int),
        "rtn_ledger_last_step": ([vp, ctypes.c_int, i], ctypes.c_int),
        "rtn_ledger_wait_complete": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "rtn_ledger_poison": ([vp], None),
        "rtn_ledger_poisoned": ([vp], ctypes.c_int),
        "rtn_ledger_next_seq": ([vp], ctypes.c_uint64),
        "rtn_h_choose": ([ctypes.c_int] * 5 + [vp, i], ctypes.c_int),
        "rtn_legal_configs": ([ctypes.c_int, ctypes.c_int, i, ctypes.c_int], ctypes.c_int),
        "rtn_frames_bucket": ([ctypes.c_int, i], ctypes.c_int),
        "rtn_select_config": ([i, i, d, ctypes.c_int, i], ctypes.c_int),
        "rtn_learn_step": ([i, i, d, ctypes.c_int, ctypes.c_int, ctypes.c_int, i], ctypes.c_int),
        "rtn_tunedb_append": ([ctypes.c_char_p, i, ctypes.c_double, ctypes.c_int64], ctypes.c_int),
        "rtn_tunedb_load": ([ctypes.c_char_p, i, d, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, i, i],
                            ctypes.c_int),
        "rtn_time_kernel": ([vp, ctypes.c_char_p, ctypes.c_int, d, d], ctypes.c_int),
        "rtn_cluster_supported": ([vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "rtn_fused_cra": ([vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "rtn_last_error_kind": ([], ctypes.c_int),
        "rtn_series_set_slices": ([vp, ctypes.c_int], ctypes.c_int),
        "rtn_series_slice_scale": ([vp, ctypes.c_int, d], ctypes.c_int),
        "rtn_set_weights": ([vp, f], ctypes.c_int),
        "rtn_set_step_cache": ([vp, f, f], ctypes.c_int),
        "rtn_rti_open": ([ctypes.c_char_p, i, ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "rtn_rti_write": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, f], ctypes.c_int),
        "rtn_rti_count": ([vp], ctypes.c_int),
        "rtn_rti_close": ([vp], ctypes.c_int),
        "rtn_series_write_rti": ([vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def library_loaded() -> bool:
    return _lib is not None


def _check(status: int):
    if status == 0:
        return
    msg = _lib.rtn_last_error().decode(errors="replace")
    if status == 4 and _lib.rtn_last_error_kind() == 6:
        raise DecompFault(msg)
    raise _ERRORS.get(status, RuntimeError)(msg)


def _fp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _c64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex64))
    if shape is not None and a.size != int(np.prod(shape)):
        raise UsageError(f"expected {int(np.prod(shape))} complex entries, got {a.size}")
    return a


# ---- Estimate layout (nlinv.hpp:21-24) -------------------------------------------
def est_dim(plan: ReconPlan) -> int:
    return plan.G * plan.G + plan.J * plan.Gc * plan.Gc


def est_split(e: np.ndarray, plan: ReconPlan):
    """flat estimate -> (rho G x G, chat J x Gc x Gc) views"""
    G, Gc, J = plan.G, plan.Gc, plan.J
    return e[:G * G].reshape(G, G), e[G * G:].reshape(J, Gc, Gc)


def est_join(rho: np.ndarray, chat: np.ndarray) -> np.ndarray:
    return np.concatenate([np.asarray(rho, np.complex64).ravel(), np.asarray(chat, np.complex64).ravel()])


def initial_estimate(plan: ReconPlan) -> np.ndarray:
    """rho = 1 on the field-of-view window, coils 0 (nlinv.cpp:60-70)"""
    G = plan.G
    L = G // 2
    lo = (G - L) // 2
    rho = np.zeros((G, G), np.complex64)
    rho[lo:lo + L, lo:lo + L] = 1.0
    return est_join(rho, np.zeros((plan.J, plan.Gc, plan.Gc), np.complex64))


# ---- fft.hpp -----------------------------------------------------------------------
class FftCtx:
    other, normal_op, setup, bench = 0, 1, 2, 3


def _fft(x: np.ndarray, sign: int) -> np.ndarray:
    lib = load_library()
    a = _c64(x).copy()
    n = a.shape[0]
    _check(lib.rtn_fft2(_fp(a), n, sign))
    return a


def fft_forward(x: np.ndarray) -> np.ndarray:
    """centered unitary forward 2D transform (fft::forward)"""
    return _fft(x, -1)


def fft_inverse(x: np.ndarray) -> np.ndarray:
    return _fft(x, +1)


def fft_counts():
    lib = load_library()
    out = (ctypes.c_uint64 * 4)()
    lib.rtn_fft_counts(out)
    return {"other": out[0], "normal_op": out[1], "setup": out[2], "bench": out[3]}


def fft_reset_counts():
    load_library().rtn_fft_reset_counts()


class CtxScope:
    """fft::CtxScope"""

    def __init__(self, ctx: int):
        self.ctx = ctx

    def __enter__(self):
        lib = load_library()
        self.prev = lib.rtn_fft_get_ctx()
        lib.rtn_fft_set_ctx(self.ctx)

    def __exit__(self, *exc):
        load_library().rtn_fft_set_ctx(self.prev)


def make_weights_inv(Gc: int, G: int) -> np.ndarray:
    lib = load_library()
    out = np.zeros((max(Gc, 1), max(Gc, 1)), np.complex64)
    _check(lib.rtn_make_weights_inv(Gc, G, _fp(out)))
    return out


# ---- device context -------------------------------------------------------------------
@dataclass
class FrameResult:
    image: np.ndarray
    est: np.ndarray
    cg_per_step: list = field(default_factory=list)
    cg_iters: int = 0
    seconds: float = 0.0


class Context:
    """One plan on one GPU: owns the device buffers and the CUDA stream.

    devices=[d0, d1, ...] builds a channel-decomposed context instead (the
    reference's WorkerGroup passed to apply_normal / reconstruct_frame,
    decomp.hpp:25-66): member k owns partition_channels(J, len(devices), a_cap)[k]
    on device devices[k]; a device may repeat (members then share that GPU)."""

    def __init__(self, plan: ReconPlan, device: int = 0, devices: Optional[Sequence[int]] = None,
                 a_cap: int = 8, member: Optional[Sequence[int]] = None):
        """member=(rank, members): this process's member of a one-process-per-GPU channel
        group (connect the members with connect_members)"""
        self.lib = load_library()
        self.plan = plan
        self._h = ctypes.c_void_p()
        self.devices = None if devices is None else [int(d) for d in devices]
        self.member = None if member is None else (int(member[0]), int(member[1]))
        c = plan.to_c()
        if self.member is not None:
            _check(self.lib.rtn_ctx_create_proc_member(ctypes.byref(c), device, self.member[0], self.member[1], a_cap,
                                                       ctypes.byref(self._h)))
        elif self.devices is None:
            _check(self.lib.rtn_ctx_create(ctypes.byref(c), device, ctypes.byref(self._h)))
        else:
            arr = (ctypes.c_int * len(self.devices))(*self.devices)
            _check(self.lib.rtn_ctx_create_group(ctypes.byref(c), arr, len(self.devices), a_cap,
                                                 ctypes.byref(self._h)))

    def ipc_handles(self) -> bytes:
        """this member's CUDA IPC handles (process-group members)"""
        n = ctypes.c_int(0)
        _check(self.lib.rtn_ctx_proc_handles(self._h, None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(self.lib.rtn_ctx_proc_handles(self._h, buf, ctypes.byref(n)))
        return buf.raw

    def attach(self, handles: Sequence[bytes]):
        """every member's ipc_handles() in rank order"""
        blob = b"".join(handles)
        _check(self.lib.rtn_ctx_proc_attach(self._h, blob, len(blob)))

    @property
    def group_blocks(self):
        """channel blocks [(j0, j1), ...] of a channel-decomposed context"""
        if self.devices is None:
            return [(0, self.plan.J)]
        out = (ctypes.c_int * (2 * len(self.devices)))()
        _check(self.lib.rtn_ctx_group_blocks(self._h, out))
        return [(out[2 * k], out[2 * k + 1]) for k in range(len(self.devices))]

    def close(self):
        # a series borrows the context's engine: close every live one first
        for ser in list(getattr(self, "_series", ())):
            ser.close()
        if self._h:
            self.lib.rtn_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def D(self) -> int:
        return est_dim(self.plan)

    def set_psf(self, P):
        P = _c64(P, (self.plan.G, self.plan.G))
        _check(self.lib.rtn_set_psf(self._h, _fp(P)))

    def set_data(self, z):
        z = _c64(z, (self.plan.J, self.plan.G, self.plan.G))
        _check(self.lib.rtn_set_data(self._h, _fp(z)))

    def apply_W_inv(self, chat):
        chat = _c64(chat, (self.plan.Gc, self.plan.Gc))
        out = np.zeros((self.plan.G, self.plan.G), np.complex64)
        _check(self.lib.rtn_apply_W_inv(self._h, _fp(chat), _fp(out)))
        return out

    def apply_W_invH(self, u):
        u = _c64(u, (self.plan.G, self.plan.G))
        out = np.zeros((self.plan.Gc, self.plan.Gc), np.complex64)
        _check(self.lib.rtn_apply_W_invH(self._h, _fp(u), _fp(out)))
        return out

    def toeplitz_apply(self, x):
        x = _c64(x, (self.plan.G, self.plan.G)).copy()
        _check(self.lib.rtn_toeplitz_apply(self._h, _fp(x)))
        return x.reshape(self.plan.G, self.plan.G)

    def make_step_cache(self, x):
        x = _c64(x, (self.D,))
        if self.devices is not None:
            _check(self.lib.rtn_make_step_cache(self._h, _fp(x), None, None))
            return None, None
        G, J = self.plan.G, self.plan.J
        rho = np.zeros((G, G), np.complex64)
        coils = np.zeros((J, G, G), np.complex64)
        _check(self.lib.rtn_make_step_cache(self._h, _fp(x), _fp(rho), _fp(coils)))
        return rho, coils

    def apply_normal(self, dx):
        dx = _c64(dx, (self.D,))
        out = np.zeros(self.D, np.complex64)
        _check(self.lib.rtn_apply_normal(self._h, _fp(dx), _fp(out)))
        return out

    def cg_solve(self, rhs, alpha: float, tol: float, max_iter: int):
        rhs = _c64(rhs, (self.D,))
        x = np.zeros(self.D, np.complex64)
        iters = ctypes.c_int(0)
        res = np.zeros(max(max_iter, 1), np.float64)
        _check(self.lib.rtn_cg_solve(self._h, _fp(rhs), alpha, tol, max_iter, _fp(x), ctypes.byref(iters),
                                     res.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return x, iters.value, res[:iters.value].copy()

    def newton_step(self, x, reg, alpha: float, cg_tol: float, cg_max_iter: int):
        """returns (x_new, cg_iters, residual0); x is not modified"""
        x = _c64(x, (self.D,)).copy()
        reg = _c64(reg, (self.D,))
        iters = ctypes.c_int(0)
        r0 = ctypes.c_double(0)
        _check(self.lib.rtn_newton_step(self._h, _fp(x), _fp(reg), alpha, cg_tol, cg_max_iter,
                                        ctypes.byref(iters), ctypes.byref(r0)))
        return x, iters.value, r0.value

    def reconstruct_frame(self, init, reg=None, regs=None) -> FrameResult:
        """nlinv.hpp:112. reg: one fixed target (None: init). regs: the RegProvider, a
        callable m -> estimate (or None to keep the previous target) or a per-step list"""
        if regs is not None:
            return self._reconstruct_frame_provider(init, regs)
        init = _c64(init, (self.D,))
        regc = None if reg is None else _c64(reg, (self.D,))
        N = self.plan.N
        img = np.zeros((N, N), np.complex64)
        est = np.zeros(self.D, np.complex64)
        per = (ctypes.c_int * max(self.plan.newton_steps, 1))()
        secs = ctypes.c_double(0)
        _check(self.lib.rtn_reconstruct_frame(self._h, _fp(init), _fp(regc), _fp(img), _fp(est), per,
                                              ctypes.byref(secs)))
        cg = [per[m] for m in range(self.plan.newton_steps)]
        return FrameResult(img, est, cg, sum(cg), secs.value)

    def _reconstruct_frame_provider(self, init, regs) -> FrameResult:
        init = _c64(init, (self.D,))
        fetch = regs if callable(regs) else (lambda m: regs[m])
        keep = []

        def provider(m, _user):
            r = fetch(m)
            if r is None:
                return None
            arr = _c64(r, (self.D,))
            keep.append(arr)  # alive until the call returns
            return arr.ctypes.data

        cb = _REG_PROVIDER(provider)
        N = self.plan.N
        img = np.zeros((N, N), np.complex64)
        est = np.zeros(self.D, np.complex64)
        per = (ctypes.c_int * max(self.plan.newton_steps, 1))()
        secs = ctypes.c_double(0)
        _check(self.lib.rtn_reconstruct_frame_provider(self._h, _fp(init), cb, None, _fp(img), _fp(est), per,
                                                       ctypes.byref(secs)))
        cg = [per[m] for m in range(self.plan.newton_steps)]
        return FrameResult(img, est, cg, sum(cg), secs.value)

    # ---- pre stage (preproc.hpp:81-133), on the device ---------------------------------
    def _frame(self, samples, angles):
        samples = np.ascontiguousarray(samples, np.complex64)
        if samples.ndim != 3:
            raise UsageError("samples must be J x K x S")
        angles = np.ascontiguousarray(angles, np.float64)
        if angles.shape != (samples.shape[1],):
            raise UsageError("one angle per spoke")
        return samples, angles

    def grid_adjoint(self, samples, angles, delay: float = 0.0):
        """grid_adjoint(frame, plan, delay): J x G x G gridded, window-masked data"""
        samples, angles = self._frame(samples, angles)
        J, K, S = samples.shape
        z = np.zeros((J, self.plan.G, self.plan.G), np.complex64)
        _check(self.lib.rtn_grid_adjoint(self._h, _fp(samples), J, angles.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         K, S, delay, _fp(z)))
        return z

    def grid_spread(self, samples, angles, delay: float = 0.0):
        """the density-compensated KB spread of grid_adjoint, before its inverse FFT"""
        samples, angles = self._frame(samples, angles)
        J, K, S = samples.shape
        g = np.zeros((J, self.plan.G, self.plan.G), np.complex64)
        _check(self.lib.rtn_grid_spread(self._h, _fp(samples), J, angles.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        K, S, delay, _fp(g)))
        return g

    def build_psf(self, angles, S: int):
        angles = np.ascontiguousarray(angles, np.float64)
        P = np.zeros((self.plan.G, self.plan.G), np.complex64)
        _check(self.lib.rtn_build_psf(self._h, angles.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(angles),
                                      S, _fp(P)))
        return P

    def build_psf_coords(self, coords, weights):
        coords = np.ascontiguousarray(coords, np.float64).reshape(-1, 2)
        weights = np.ascontiguousarray(weights, np.float64)
        if len(weights) != len(coords):
            raise UsageError("build_psf_coords: coordinate/weight count mismatch")
        P = np.zeros((self.plan.G, self.plan.G), np.complex64)
        dp = ctypes.POINTER(ctypes.c_double)
        _check(self.lib.rtn_build_psf_coords(self._h, coords.ctypes.data_as(dp), weights.ctypes.data_as(dp),
                                             len(weights), _fp(P)))
        return P

    def apply_compression(self, m, samples):
        """samples (Jp, ...) -> (Jv, ...) with the Jv x Jp matrix m"""
        m = np.ascontiguousarray(m, np.complex64)
        samples = np.ascontiguousarray(samples, np.complex64)
        Jv, Jp = m.shape
        if samples.shape[0] != Jp:
            raise DataError("apply_compression: channel count does not match matrix")
        n = samples[0].size
        out = np.zeros((Jv,) + samples.shape[1:], np.complex64)
        _check(self.lib.rtn_apply_compression(self._h, _fp(m), Jv, Jp, _fp(samples), n, _fp(out)))
        return out

    def cluster_supported(self) -> bool:
        """whether this plan's grid has the cluster-fused application (latency mode)"""
        v = ctypes.c_int(0)
        _check(self.lib.rtn_cluster_supported(self._h, ctypes.byref(v)))
        return bool(v.value)

    def fused_cra(self) -> bool:
        """whether the budget-mode CR solve fuses the recurrence with the next
        application's W^-1 column pass (k_crA) on the five-kernel path"""
        v = ctypes.c_int(0)
        _check(self.lib.rtn_fused_cra(self._h, ctypes.byref(v)))
        return bool(v.value)

    def time_kernel(self, which: str, reps: int = 20):
        """(average ms per launch, algorithmic bytes per launch) of one kernel class"""
        ms = ctypes.c_double(0)
        by = ctypes.c_double(0)
        _check(self.lib.rtn_time_kernel(self._h, which.encode(), reps, ctypes.byref(ms), ctypes.byref(by)))
        return ms.value, by.value


# ---- decomposition / scheduling (decomp.hpp) ------------------------------------------------
@dataclass
class TemporalSchedule:
    """decomp.hpp:70-76"""
    l: int = 1
    o: int = 1

    @staticmethod
    def for_turns(U: int) -> "TemporalSchedule":
        return TemporalSchedule(U, (U + 1) // 2)


@dataclass
class SeriesOptions:
    """nlinv.hpp:136-145 (T = frames in flight on the device)"""
    sched: TemporalSchedule = field(default_factory=TemporalSchedule)
    T: int = 1
    A: int = 1
    chain: bool = True
    normalize: bool = True
    plain: bool = False
    cluster: int = -1  # cluster-fused applications: 1 on, 0 off, -1 auto (on when T == 1)

    def to_c(self) -> _SeriesOpts:
        return _SeriesOpts(self.T, self.A, self.sched.l, self.sched.o, int(self.chain), int(self.normalize),
                           int(self.plain), int(self.cluster))


@dataclass
class FrameAudit:
    frame: int
    thread: int
    workers: int
    init_src: int
    reg_final_src: int
    reg_src: list
    start_seq: int = 0
    reg_final_seq: int = 0
    finish_seq: int = 0


def format_audit(a: FrameAudit) -> str:
    return (f"frame {a.frame}: init<-{a.init_src}, reg_final<-{a.reg_final_src}, "
            f"thread {a.thread}, workers {a.workers}")


class Series:
    """Device-resident frame series (reconstruct_series / _plain, nlinv.cpp:412-526)."""

    def __init__(self, ctx: Context, frames: int, n_psf: int, devices: Optional[Sequence[int]] = None):
        """devices: spread the frame workers over these GPUs (temporal decomposition
        across devices in one process); default: the context's device only"""
        self.ctx = ctx
        self.lib = ctx.lib
        self.F = frames
        self._h = ctypes.c_void_p()
        if not hasattr(ctx, "_series"):
            ctx._series = weakref.WeakSet()
        ctx._series.add(self)
        if devices:
            dv = (ctypes.c_int * len(devices))(*devices)
            _check(self.lib.rtn_series_create_multi(ctx._h, frames, n_psf, dv, len(devices), ctypes.byref(self._h)))
        else:
            _check(self.lib.rtn_series_create(ctx._h, frames, n_psf, ctypes.byref(self._h)))

    def close(self):
        if self._h:
            self.lib.rtn_series_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload_frames(self, z, first: int = 0):
        p = self.ctx.plan
        z = _c64(z)
        count = z.size // (p.J * p.G * p.G)
        _check(self.lib.rtn_series_upload_frames(self._h, first, count, z.ctypes.data))

    def upload_psf(self, k: int, P):
        P = _c64(P, (self.ctx.plan.G, self.ctx.plan.G))
        _check(self.lib.rtn_series_upload_psf(self._h, k, _fp(P)))

    def set_psf_index(self, idx):
        a = np.ascontiguousarray(np.asarray(idx, np.int32))
        _check(self.lib.rtn_series_set_psf_index(self._h, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))

    def set_slices(self, slices: int):
        """interleaved slice chains: store index g = frame * slices + slice (pipeline.cpp:315-334)"""
        _check(self.lib.rtn_series_set_slices(self._h, slices))
        self.slices = slices

    def slice_scale(self, sl: int) -> float:
        v = ctypes.c_double(0)
        _check(self.lib.rtn_series_slice_scale(self._h, sl, ctypes.byref(v)))
        return v.value

    def normalize(self) -> float:
        v = ctypes.c_double(0)
        _check(self.lib.rtn_series_normalize(self._h, ctypes.byref(v)))
        return v.value

    def run(self, opts: SeriesOptions, first: int = 0, count: Optional[int] = None, z_host=None,
            want_images: bool = True, z_host_ptr: Optional[int] = None, images_ptr: Optional[int] = None,
            raw: Optional[dict] = None):
        """raw = dict(samples=(count, Jp, K, S) complex64 or samples_ptr=int, angles=(count, K),
        delay=0.0, cmat=(J, Jp) or None): raw acquisitions through the device pre stage"""
        p = self.ctx.plan
        count = self.F - first if count is None else count
        M = p.newton_steps
        images = np.zeros((count, p.N, p.N), np.complex64) if (want_images and images_ptr is None) else None
        audit = np.zeros((count, 5 + M), np.int32)
        seqs = np.zeros((count, 3), np.uint64)
        cg = np.zeros(count, np.int32)
        ms = np.zeros(count, np.float32)
        zp = None
        if z_host_ptr is not None:
            zp = z_host_ptr
        elif z_host is not None:
            z_host = _c64(z_host)
            zp = z_host.ctypes.data
        ip = images_ptr if images_ptr is not None else (None if images is None else images.ctypes.data)
        o = opts.to_c()
        outs = (audit.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), seqs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                cg.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _fp(ms))
        if raw is not None:
            ang = np.ascontiguousarray(raw["angles"], np.float64)
            K = ang.shape[-1]
            cm = raw.get("cmat")
            keep = [ang]
            if "samples_ptr" in raw:
                sp, S, Jp = raw["samples_ptr"], raw["S"], raw.get("Jp", p.J)
            else:
                smp = _c64(raw["samples"])
                keep.append(smp)
                sp, Jp, S = smp.ctypes.data, smp.shape[1], smp.shape[-1]
                if smp.shape[0] != count or smp.shape[2] != K:
                    raise UsageError("raw samples must be (count, Jp, K, S) with K = angles per frame")
            cmp = None
            if cm is not None:
                cm = np.ascontiguousarray(cm, np.complex64)
                keep.append(cm)
                cmp = cm.ctypes.data
            elif Jp != p.J:
                raise UsageError("raw samples have Jp != J channels and no compression matrix")
            _check(self.lib.rtn_series_run_raw(self._h, ctypes.byref(o), first, count, sp, ang.ctypes.data, K, S,
                                               float(raw.get("delay", 0.0)), cmp, Jp, ip, *outs))
        else:
            _check(self.lib.rtn_series_run(self._h, ctypes.byref(o), first, count, zp, ip, *outs))
        audits = [FrameAudit(int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), [int(v) for v in r[5:]],
                             int(q[0]), int(q[1]), int(q[2])) for r, q in zip(audit, seqs)]
        return dict(images=images, audit=audits, cg_iters=cg, gpu_ms=ms)

    def post(self, first: int = 0, count: Optional[int] = None, mode: str = "magnitude"):
        """device postprocessing of the stored images: magnitude, median3 (magnitude +
        MedianFilter3) or phase_difference (frame pairs)"""
        p = self.ctx.plan
        count = self.F - first if count is None else count
        m = {"magnitude": 0, "median3": 1, "phase_difference": 2}[mode]
        n = count // 2 if m == 2 else count
        out = np.zeros((n, p.N, p.N), np.float32)
        _check(self.lib.rtn_series_post(self._h, first, count, m, _fp(out)))
        return out

    def write_rti(self, sink: "RtiSink", first: int = 0, count: Optional[int] = None, mode: str = "magnitude",
                  slice_id: int = 0):
        """device postprocessing of the stored images into an .rti sink (the pipeline's
        pst + snk stages, pipeline.cpp:60-137)"""
        count = self.F - first if count is None else count
        m = {"magnitude": 0, "median3": 1, "phase_difference": 2}[mode]
        _check(self.lib.rtn_series_write_rti(self._h, sink._h, first, count, m, slice_id))

    def save_psf_cache(self, path):
        _check(self.lib.rtn_series_psf_cache_save(self._h, str(path).encode()))

    def load_psf_cache(self, path):
        _check(self.lib.rtn_series_psf_cache_load(self._h, str(path).encode()))

    def psf_cache_size(self) -> int:
        return int(self.lib.rtn_series_psf_cache_size(self._h))

    def last_span_ms(self) -> float:
        """device time of the last run (CUDA events across all worker streams)"""
        return float(self.lib.rtn_series_last_span_ms(self._h))

    def images(self, first: int = 0, count: Optional[int] = None):
        p = self.ctx.plan
        count = self.F - first if count is None else count
        out = np.zeros((count, p.N, p.N), np.complex64)
        _check(self.lib.rtn_series_images(self._h, first, count, _fp(out)))
        return out

    def estimate(self, n: int):
        out = np.zeros(self.ctx.D, np.complex64)
        _check(self.lib.rtn_series_estimate(self._h, n, _fp(out)))
        return out


class RtiSink:
    """.rti image sink in the reference's RtiWriter format (ingest.hpp:105-126). header:
    DatasetHeader fields {version, N, J_physical, K, U, frames, slices, mode, samples}
    (mode 0 single_slice, 1 multi_slice, 2 flow)."""

    KINDS = {"magnitude": 0, "phase_difference": 1}

    def __init__(self, path, header, strict_order: bool = True):
        self.lib = load_library()
        self._h = ctypes.c_void_p()
        h = np.ascontiguousarray(header, np.int32)
        if h.size != 9:
            raise UsageError("rti header needs 9 fields")
        _check(self.lib.rtn_rti_open(str(path).encode(), h.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                     int(strict_order), ctypes.byref(self._h)))
        self.N = int(h[1])

    def write(self, frame: int, slice_id: int, kind: str, pixels):
        px = np.ascontiguousarray(pixels, np.float32)
        if px.size != self.N * self.N:
            raise UsageError("rti image does not match the header's N")
        _check(self.lib.rtn_rti_write(self._h, frame, slice_id, self.KINDS[kind], _fp(px)))

    @property
    def count(self) -> int:
        return int(self.lib.rtn_rti_count(self._h))

    def close(self):
        if self._h:
            h, self._h = self._h, ctypes.c_void_p()
            _check(self.lib.rtn_rti_close(h))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def reconstruct_series(ctx: Context, z, P, opts: SeriesOptions, psf_index=None):
    """gridded frames z (F, J, G, G) + PSF set P (U, G, G) -> images (F, N, N) and audit"""
    z = _c64(z)
    P = _c64(P)
    if P.ndim == 2:
        P = P[None]
    F = z.shape[0]
    s = Series(ctx, F, P.shape[0])
    try:
        s.upload_frames(z)
        for k in range(P.shape[0]):
            s.upload_psf(k, P[k])
        if psf_index is not None:
            s.set_psf_index(psf_index)
        out = s.run(opts)
        return out
    finally:
        s.close()


# ---- planner.hpp:12-64 over the device transforms --------------------------------------------
@dataclass
class FftLookupTable:
    """planner.hpp:12-18: size -> device time (us) of one 2D transform"""
    entries_us: dict = field(default_factory=dict)
    machine_key: str = ""
    library_key: str = "rtnlinv_b200-line-fft-sm100a"

    def _arrays(self):
        sizes = np.array(sorted(self.entries_us), np.int32)
        us = np.array([self.entries_us[k] for k in sorted(self.entries_us)], np.float64)
        return sizes, us


def benchmark_fft(sizes, trials: int = 5, batch: int = 1, device: int = 0) -> FftLookupTable:
    lib = load_library()
    sz = np.ascontiguousarray(list(sizes), np.int32)
    us = np.zeros(len(sz), np.float64)
    _check(lib.rtn_benchmark_fft(sz.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), len(sz), trials, batch, device,
                                 us.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return FftLookupTable({int(a): float(b) for a, b in zip(sz, us)})


def select_grid(N: int, table: FftLookupTable, gamma_min: float = 1.4, gamma_max: float = 2.0):
    """planner.cpp:112-131: (G, gamma) of the fastest even grid in [2 gamma_min N, 2 gamma_max N]"""
    lib = load_library()
    sizes, us = table._arrays()
    G, gamma = ctypes.c_int(0), ctypes.c_double(0)
    _check(lib.rtn_select_grid(N, sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                               us.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(sizes), gamma_min, gamma_max,
                               ctypes.byref(G), ctypes.byref(gamma)))
    return G.value, gamma.value


def save_table(table: FftLookupTable, path: str):
    lib = load_library()
    sizes, us = table._arrays()
    _check(lib.rtn_fft_table_save(str(path).encode(), sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                  us.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(sizes),
                                  table.machine_key.encode(), table.library_key.encode()))


def load_table(path: str) -> FftLookupTable:
    lib = load_library()
    cap = 8192
    sizes = np.zeros(cap, np.int32)
    us = np.zeros(cap, np.float64)
    n = ctypes.c_int(0)
    mk, lk = ctypes.create_string_buffer(512), ctypes.create_string_buffer(512)
    _check(lib.rtn_fft_table_load(str(path).encode(), sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                  us.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap, ctypes.byref(n), mk, lk,
                                  512))
    k = min(n.value, cap)
    return FftLookupTable({int(sizes[i]): float(us[i]) for i in range(k)}, mk.value.decode(), lk.value.decode())


def plan_from_table(N: int, J: int, table: FftLookupTable, gamma_min: float = 1.4, gamma_max: float = 2.0):
    """make_plan(N, J, &table) (planner.cpp:133-149)"""
    G, gamma = select_grid(N, table, gamma_min, gamma_max)
    p = raw_plan(G, J)
    p.N, p.gamma = N, gamma
    return p


# ---- pipeline.cpp:60-137 postprocessing on the device ------------------------------------------
def magnitude_image(img) -> np.ndarray:
    lib = load_library()
    img = _c64(img)
    out = np.zeros(img.shape, np.float32)
    _check(lib.rtn_post_magnitude(_fp(img), img.size, _fp(out)))
    return out


def phase_difference_image(even, odd) -> np.ndarray:
    lib = load_library()
    even, odd = _c64(even), _c64(odd)
    if even.shape != odd.shape:
        raise UsageError("phase_difference_image: size mismatch")
    out = np.zeros(even.shape, np.float32)
    _check(lib.rtn_post_phase_difference(_fp(even), _fp(odd), even.size, _fp(out)))
    return out


def median3_sequence(mags) -> np.ndarray:
    """MedianFilter3 over one slice's magnitude frames (F, N, N)"""
    lib = load_library()
    mags = np.ascontiguousarray(mags, np.float32)
    out = np.zeros_like(mags)
    _check(lib.rtn_post_median3(_fp(mags), mags.shape[0], mags[0].size, _fp(out)))
    return out


def grid_supported(G: int) -> bool:
    """the fused line engine covers grid side G (else transforms fall back to the direct DFT kernel)"""
    return bool(load_library().rtn_grid_supported(G))


def connect_members(ctx: "Context", group=None):
    """exchange the members' IPC handles over torch.distributed (any backend; the
    handles are small host objects) and attach them"""
    import torch.distributed as dist
    mine = ctx.ipc_handles()
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    ctx.attach(allh)


def psf_angle_key(angles, S: int, G: int) -> int:
    """PsfCache::angle_key (preproc.cpp:301-313)"""
    a = np.ascontiguousarray(angles, np.float64)
    return int(load_library().rtn_psf_angle_key(a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(a), S, G))


def all_reduce_sum(terms):
    """decomp.hpp:25-30: sum of the terms (n x G x G complex64) in order in FP64, on the device"""
    terms = np.ascontiguousarray(terms, np.complex64)
    if terms.ndim != 3 or terms.shape[1] != terms.shape[2]:
        raise UsageError("all_reduce_sum: terms must be n x G x G")
    out = np.zeros(terms.shape[1:], np.complex64)
    _check(load_library().rtn_all_reduce_sum(_fp(terms), terms.shape[0], terms.shape[1], _fp(out)))
    return out


def partition_channels(J: int, A: int, cap: int = 4):
    lib = load_library()
    out = (ctypes.c_int * (2 * max(A, 1)))()
    _check(lib.rtn_partition_channels(J, A, cap, out))
    return [(out[2 * a], out[2 * a + 1]) for a in range(A)]


class CompletionLedger:
    """decomp.hpp:81-109"""

    def __init__(self, frames: int):
        self.lib = load_library()
        self._h = ctypes.c_void_p()
        _check(self.lib.rtn_ledger_create(frames, ctypes.byref(self._h)))

    def __del__(self):
        try:
            self.lib.rtn_ledger_destroy(self._h)
        except Exception:
            pass

    def mark_step(self, n, m):
        _check(self.lib.rtn_ledger_mark_step(self._h, n, m))

    def mark_complete(self, n):
        _check(self.lib.rtn_ledger_mark_complete(self._h, n))

    def completed(self, n) -> bool:
        return bool(self.lib.rtn_ledger_completed(self._h, n))

    def last_step(self, n) -> int:
        v = ctypes.c_int(0)
        _check(self.lib.rtn_ledger_last_step(self._h, n, ctypes.byref(v)))
        return v.value

    def wait_complete(self, n, deadline_ms=600000):
        st = self.lib.rtn_ledger_wait_complete(self._h, n, deadline_ms)
        if st == 4:
            raise DecompFault(self.lib.rtn_last_error().decode())
        _check(st)

    def poison(self):
        self.lib.rtn_ledger_poison(self._h)

    def poisoned(self) -> bool:
        return bool(self.lib.rtn_ledger_poisoned(self._h))

    def next_seq(self) -> int:
        return int(self.lib.rtn_ledger_next_seq(self._h))


def h_choose(n: int, m: int, M: int, sched: TemporalSchedule, ledger: CompletionLedger) -> int:
    lib = load_library()
    v = ctypes.c_int(0)
    st = lib.rtn_h_choose(n, m, M, sched.l, sched.o, ledger._h, ctypes.byref(v))
    if st == 4:
        raise DecompFault(lib.rtn_last_error().decode())
    _check(st)
    return v.value


# ---- autotune (autotune.hpp) --------------------------------------------------------------------
class ImagingMode:
    single_slice, multi_slice, flow = 0, 1, 2


def frames_bucket(frames: int) -> int:
    lib = load_library()
    v = ctypes.c_int(0)
    _check(lib.rtn_frames_bucket(frames, ctypes.byref(v)))
    return v.value


def legal_configs(total_workers: int = 8, a_cap: int = 4):
    lib = load_library()
    buf = (ctypes.c_int * 512)()
    n = lib.rtn_legal_configs(total_workers, a_cap, buf, 256)
    if n < 0:
        _check(-n)
    return [(buf[2 * k], buf[2 * k + 1]) for k in range(n)]


def _db_arrays(db):
    rows = np.zeros((max(len(db), 1), 6), np.int32)
    ms = np.zeros(max(len(db), 1), np.float64)
    for k, r in enumerate(db):
        rows[k] = r[:6]
        ms[k] = r[6]
    return rows, ms


def select_config(key, db):
    """key = (mode, N, bucket, J); db rows = (mode, N, bucket, J, T, A, runtime_ms)"""
    lib = load_library()
    rows, ms = _db_arrays(db)
    k = np.asarray(key, np.int32)
    out = np.zeros(2, np.int32)
    ip = ctypes.POINTER(ctypes.c_int)
    _check(lib.rtn_select_config(k.ctypes.data_as(ip), rows.ctypes.data_as(ip),
                                 ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(db), out.ctypes.data_as(ip)))
    return int(out[0]), int(out[1])


def learn_step(key, db, total_workers: int = 8, a_cap: int = 4):
    lib = load_library()
    rows, ms = _db_arrays(db)
    k = np.asarray(key, np.int32)
    out = np.zeros(2, np.int32)
    ip = ctypes.POINTER(ctypes.c_int)
    _check(lib.rtn_learn_step(k.ctypes.data_as(ip), rows.ctypes.data_as(ip),
                              ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(db), total_workers, a_cap,
                              out.ctypes.data_as(ip)))
    return int(out[0]), int(out[1])


class TuneDb:
    """append-only TSV store (autotune.hpp:57-75)"""

    def __init__(self, path: str):
        self.path = path
        self.skipped = 0

    def append(self, row, runtime_ms: float, timestamp: int):
        lib = load_library()
        r = np.asarray(row[:6], np.int32)
        _check(lib.rtn_tunedb_append(self.path.encode(), r.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                     runtime_ms, timestamp))

    def load(self):
        lib = load_library()
        cap = 4096
        rows = np.zeros((cap, 6), np.int32)
        ms = np.zeros(cap, np.float64)
        ts = np.zeros(cap, np.int64)
        n = ctypes.c_int(0)
        sk = ctypes.c_int(0)
        ip = ctypes.POINTER(ctypes.c_int)
        _check(lib.rtn_tunedb_load(self.path.encode(), rows.ctypes.data_as(ip),
                                   ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   ts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap, ctypes.byref(n),
                                   ctypes.byref(sk)))
        self.skipped = sk.value
        return [tuple(int(v) for v in rows[k]) + (float(ms[k]), int(ts[k])) for k in range(n.value)]
