"""Thin Python binding of the C ABI in include/pint.h (ctypes; argument marshalling only).

Every step of the WR iteration runs in the CUDA kernels of libpint.so.  There is no CPU
fallback: if the library is missing or fails to load, `lib()` raises.  Host arrays are numpy
complex128 (mem = PINT_HOST); device arrays are torch CUDA complex128 tensors (PINT_DEVICE).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PINT_LIB", os.path.join(HERE, "libpint.so"))

PINT_OK, PINT_ERR_ARG, PINT_ERR_ALLOC, PINT_ERR_CUDA, PINT_ERR_COMM, PINT_ERR_STATE, \
    PINT_ERR_NOT_CONVERGED, PINT_ERR_DIVERGED, PINT_ERR_UNSUPPORTED = range(9)
PINT_OP_FD1D_DIRICHLET, PINT_OP_FD2D_DIRICHLET, PINT_OP_FEM1D_DIRICHLET, PINT_OP_FEM2D_DIRICHLET = 1, 2, 3, 4
PINT_HOST, PINT_DEVICE = 0, 1
PINT_FLAG_U0_ZERO = 1
PINT_FLAG_FULL_FFT = 2
PINT_FLAG_STREAM = 4
PINT_FLAG_DST_PER_ITER = 8
PINT_NL_ALLEN_CAHN = 1
PINT_FLAG_REAL_DATA = 16
PINT_FLAG_MODAL = 32
PINT_FLAG_FULL_UPDATE_NORM = 64

EXPORTED = [
    "pint_plan_create", "pint_set_problem_separable", "pint_set_initial_guess", "pint_wr_iterate",
    "pint_wr_solve", "pint_get_levels", "pint_get_solution", "pint_get_modal_levels",
    "pint_modal_to_physical", "pint_partition", "pint_get_partition", "pint_set_timing", "pint_get_timing",
    "pint_get_info", "pint_plan_destroy", "pint_status_string", "pint_last_error",
    "pint_kappa_log_rule", "pint_get_path", "pint_set_nonlinearity", "pint_newton_solve", "pint_set_problem",
    "pint_residual", "pint_wr_run",
]


class pint_operator(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("mx", ctypes.c_int64), ("my", ctypes.c_int64)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p)


class pint_options(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("flags", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("allreduce_max", ALLREDUCE_FN), ("allreduce_ctx", ctypes.c_void_p)]


_LIB = None


def lib(path: str = LIB_PATH):
    """Load libpint.so (raises if absent: the product path has no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built; run `python -m paper_2007_13125_b200.build`")
    L = ctypes.CDLL(path)
    P, I64, I32, D, VP = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
    sig = {
        "pint_plan_create": [I64, I64, I32, D, D, ctypes.POINTER(pint_operator), ctypes.POINTER(pint_options),
                             ctypes.POINTER(P)],
        "pint_set_problem_separable": [P, VP, I32, VP, VP, VP, I32],
        "pint_set_initial_guess": [P, VP, I32],
        "pint_wr_iterate": [P, ctypes.POINTER(D)],
        "pint_wr_solve": [P, D, I32, ctypes.POINTER(I32), ctypes.POINTER(D)],
        "pint_get_levels": [P, I64, I64, VP, I32],
        "pint_get_solution": [P, VP, I32],
        "pint_get_modal_levels": [P, I64, I64, VP, I32],
        "pint_modal_to_physical": [P, I64, VP, VP, I32],
        "pint_partition": [I64, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "pint_get_partition": [P, ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "pint_set_timing": [P, I32],
        "pint_get_timing": [P, ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "pint_get_info": [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "pint_plan_destroy": [P],
        "pint_status_string": [I32],
        "pint_last_error": [],
        "pint_kappa_log_rule": [I64],
        "pint_get_path": [P, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32)],
        "pint_set_nonlinearity": [P, I32, D],
        "pint_set_problem": [P, VP, VP, VP, VP, I32],
        "pint_newton_solve": [P, I32, D, D, I32, ctypes.POINTER(I32), ctypes.POINTER(D), ctypes.POINTER(I32)],
        "pint_residual": [P, ctypes.POINTER(D), ctypes.POINTER(D)],
        "pint_wr_run": [P, I32, ctypes.POINTER(D)],
    }
    for name, args in sig.items():
        if not hasattr(L, name) and "PINT_LIB" in os.environ:
            continue          # older variant library (A/B timing via PINT_LIB): extension symbols may be absent
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.pint_status_string.restype = ctypes.c_char_p
    L.pint_last_error.restype = ctypes.c_char_p
    L.pint_kappa_log_rule.restype = ctypes.c_double
    _LIB = L
    return L


class PintError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(f"{lib().pint_status_string(status).decode()}: {message}")


def _check(status: int):
    if status != PINT_OK:
        raise PintError(status, lib().pint_last_error().decode())


def _ptr(x):
    """(pointer, mem) for a numpy host array or a torch CUDA tensor; None -> (None, HOST)."""
    if x is None:
        return None, PINT_HOST
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data, PINT_HOST
    if hasattr(x, "data_ptr") and getattr(x, "is_cuda", False):
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return x.data_ptr(), PINT_DEVICE
    if hasattr(x, "data_ptr"):
        return _ptr(x.numpy())
    raise TypeError(f"unsupported array type {type(x)}")


def partition(mx: int, rank: int, nranks: int) -> tuple[int, int]:
    """Host-only x-mode slab of `rank` (pint_partition)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().pint_partition(mx, rank, nranks, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def kappa_log_rule(N: int) -> float:
    return lib().pint_kappa_log_rule(N)


class Plan:
    """One WR/ParaDiag plan (pint_plan) on one device; see include/pint.h."""

    def __init__(self, mx: int, my: int, N: int, k: int, kappa: float, tau: float, alpha: float = 1.0,
                 device: int = 0, stream: int | None = None, u0_zero: bool = False,
                 rank: int = 0, nranks: int = 1, allreduce_max=None, full_fft: bool = False,
                 stream_path: bool = False, dst_per_iter: bool = False, real_data: bool = False,
                 modal: bool = False, fem: bool = False, full_update_norm: bool = False):
        """fem=True: P1 finite elements (1D mesh: PINT_OP_FEM1D_DIRICHLET; 2D uniform triangulation:
        PINT_OP_FEM2D_DIRICHLET; nodal coefficient vectors)."""
        L = lib()
        self.mx, self.my, self.N, self.k = int(mx), int(my), int(N), int(k)
        self.M = self.mx * self.my
        if fem:
            kind = PINT_OP_FEM1D_DIRICHLET if my == 1 else PINT_OP_FEM2D_DIRICHLET
        else:
            kind = PINT_OP_FD1D_DIRICHLET if my == 1 else PINT_OP_FD2D_DIRICHLET
        op = pint_operator(kind, mx, my)
        self._cb = ALLREDUCE_FN(0)
        if allreduce_max is not None:
            def _cb(p, ctx):
                try:
                    p[0] = float(allreduce_max(float(p[0])))
                    return 0
                except Exception:   # noqa: BLE001 - reported through PINT_ERR_COMM
                    return 1
            self._cb = ALLREDUCE_FN(_cb)
        flags = (PINT_FLAG_U0_ZERO if u0_zero else 0) | (PINT_FLAG_FULL_FFT if full_fft else 0) | \
            (PINT_FLAG_STREAM if stream_path else 0) | (PINT_FLAG_DST_PER_ITER if dst_per_iter else 0) | \
            (PINT_FLAG_REAL_DATA if real_data else 0) | (PINT_FLAG_MODAL if modal else 0) | \
            (PINT_FLAG_FULL_UPDATE_NORM if full_update_norm else 0)
        opt = pint_options(alpha, device, stream or 0, flags, rank, nranks,
                           self._cb, None)
        h = ctypes.c_void_p()
        _check(L.pint_plan_create(self.M, N, k, kappa, tau, ctypes.byref(op), ctypes.byref(opt), ctypes.byref(h)))
        self._h = h

    # -- problem ---------------------------------------------------------------------------
    def set_problem(self, v, g=None, phi=None, dphi=None):
        """v [M] complex; g [R][M] complex; phi [R][N+1] float64 (host); dphi [R][k-2] float64 (host)."""
        R = 0 if g is None else int(g.shape[0])
        vp, mem = _ptr(v)
        gp, gmem = _ptr(g) if R else (None, mem)
        if R and gmem != mem:
            raise ValueError("v and g must live in the same memory space")
        phi_a = np.ascontiguousarray(phi, dtype=np.float64) if R else None
        dphi_a = np.ascontiguousarray(dphi, dtype=np.float64) if (R and dphi is not None and dphi.size) else None
        _check(lib().pint_set_problem_separable(
            self._h, vp, R, gp, None if phi_a is None else phi_a.ctypes.data,
            None if dphi_a is None else dphi_a.ctypes.data, mem))

    def set_problem_dense(self, v, f, f0=None, fderiv=None):
        """v [M]; f [N][M] = f(t_1..t_N); f0 [M] = f(0); fderiv [k-2][M] (pint_set_problem)."""
        vp, mem = _ptr(v)
        fp, fm = _ptr(f)
        f0p, m0 = _ptr(f0) if f0 is not None else (None, mem)
        fdp, md = _ptr(fderiv) if fderiv is not None else (None, mem)
        if len({mem, fm, m0, md}) != 1:
            raise ValueError("all arrays must live in the same memory space")
        _check(lib().pint_set_problem(self._h, vp, fp, f0p, fdp, mem))

    @classmethod
    def from_problem(cls, prob, device_arrays: bool = False, **kw) -> "Plan":
        kw.setdefault("fem", getattr(prob, "space", "fd") == "fem")
        p = cls(prob.mx, prob.my, prob.N, prob.k, prob.kappa, prob.tau, prob.alpha,
                u0_zero=(prob.u0 == "zero"), **kw)
        v, g = prob.v, (prob.g if prob.R else None)
        if device_arrays:
            import torch
            v = torch.from_numpy(np.ascontiguousarray(v)).cuda()
            g = None if g is None else torch.from_numpy(np.ascontiguousarray(g)).cuda()
        p.set_problem(np.ascontiguousarray(v) if not device_arrays else v,
                      (np.ascontiguousarray(g) if (g is not None and not device_arrays) else g),
                      prob.phi if prob.R else None, prob.dphi if prob.R else None)
        return p

    def set_initial_guess(self, U0=None):
        p, mem = _ptr(U0)
        _check(lib().pint_set_initial_guess(self._h, p, mem))

    # -- iteration -----------------------------------------------------------------------------
    def iterate(self) -> float:
        u = ctypes.c_double()
        _check(lib().pint_wr_iterate(self._h, ctypes.byref(u)))
        return u.value

    def run(self, iters: int) -> float:
        """Exactly `iters` iterations, one synchronisation (pint_wr_run); returns the last update."""
        u = ctypes.c_double()
        _check(lib().pint_wr_run(self._h, iters, ctypes.byref(u)))
        return u.value

    def solve(self, tol: float = 1e-12, max_iters: int = 50, raise_on_fail: bool = True):
        it, u = ctypes.c_int32(), ctypes.c_double()
        st = lib().pint_wr_solve(self._h, tol, max_iters, ctypes.byref(it), ctypes.byref(u))
        if st != PINT_OK and raise_on_fail:
            _check(st)
        return it.value, u.value, st

    # -- output ------------------------------------------------------------------------------
    def get_levels(self, n0: int, count: int, out=None):
        if out is None:
            out = np.empty((count, self.M), np.complex128)
        p, mem = _ptr(out)
        _check(lib().pint_get_levels(self._h, n0, count, p, mem))
        return out

    def get_solution(self, out=None):
        return self.get_levels(0, self.N, out)

    def get_modal_levels(self, n0: int, count: int, out=None):
        qb, qe = self.partition()
        if out is None:
            out = np.empty((count, self.my, qe - qb), np.complex128)
        p, mem = _ptr(out)
        _check(lib().pint_get_modal_levels(self._h, n0, count, p, mem))
        return out

    def modal_to_physical(self, Uq_full, out=None):
        count = int(Uq_full.shape[0])
        if out is None:
            out = np.empty((count, self.M), np.complex128)
        pin, mem = _ptr(Uq_full)
        pout, mem2 = _ptr(out)
        if mem != mem2:
            raise ValueError("input and output must live in the same memory space")
        _check(lib().pint_modal_to_physical(self._h, count, pin, pout, mem))
        return out

    def partition(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().pint_get_partition(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    # -- instrumentation -------------------------------------------------------------------
    def set_timing(self, enable: bool = True):
        _check(lib().pint_set_timing(self._h, 1 if enable else 0))

    def get_timing(self):
        t, s, tn, sn = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().pint_get_timing(self._h, ctypes.byref(t), ctypes.byref(s), ctypes.byref(tn), ctypes.byref(sn)))
        return {"tpass_ms": t.value, "spass_ms": s.value, "tpass_launches": tn.value, "spass_launches": sn.value}

    def residual(self) -> tuple[float, float]:
        """(max |residual of the BDF-k scheme at U_m|, max |F_static|) — pint_residual: heat and CQ,
        FD, fully modal and P1-FEM plans (not: CQ on the modal path, semilinear plans,
        PINT_FLAG_DST_PER_ITER, dense forcing; include/pint.h)."""
        r, f = ctypes.c_double(), ctypes.c_double()
        _check(lib().pint_residual(self._h, ctypes.byref(r), ctypes.byref(f)))
        return r.value, f.value

    def info(self):
        m, l, b = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().pint_get_info(self._h, ctypes.byref(m), ctypes.byref(l), ctypes.byref(b)))
        return {"m": m.value, "kernel_launches": l.value, "device_bytes": b.value}

    # -- semilinear extension (Newton-WR) ------------------------------------------------------
    def set_nonlinearity(self, eps: float, kind: int = PINT_NL_ALLEN_CAHN):
        _check(lib().pint_set_nonlinearity(self._h, kind, eps))

    def newton_solve(self, max_outer: int, inner_tol: float = 1e-12, max_inner: int = 60,
                     outer_tol: float = 0.0, raise_on_fail: bool = True):
        """Returns (inner_counts, outer_updates, status)."""
        cnt = (ctypes.c_int32 * max(max_outer, 1))()
        upd = (ctypes.c_double * max(max_outer, 1))()
        done = ctypes.c_int32()
        st = lib().pint_newton_solve(self._h, max_outer, outer_tol, inner_tol, max_inner, cnt, upd, ctypes.byref(done))
        if st != PINT_OK and raise_on_fail:
            _check(st)
        return list(cnt[:done.value]), list(upd[:done.value]), st

    def path(self):
        """{"fused": bool, "chunks": int, "nk": int} (pint_get_path)."""
        f, c, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().pint_get_path(self._h, ctypes.byref(f), ctypes.byref(c), ctypes.byref(n)))
        return {"fused": bool(f.value), "chunks": c.value, "nk": n.value}

    def close(self):
        if getattr(self, "_h", None):
            lib().pint_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
