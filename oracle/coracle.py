"""ctypes binding of oracle/liboracle.so -- the C restatement of the
reference path (TEST INFRASTRUCTURE / CPU BASELINE ONLY; see oracle.c)."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import port

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")


class LevelDesc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("omega2", C.c_double), ("vcoef", C.c_double)] + \
               [(n, C.c_void_p) for n in ("wx", "wy", "av", "vh", "sumw", "dr", "vprof",
                                          "volprof")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError("oracle/liboracle.so not built (make -C oracle)")
        L = C.CDLL(LIB)
        L.or_hier_create.restype = C.c_void_p
        L.or_hier_create.argtypes = [C.c_int, C.POINTER(LevelDesc), C.c_int, C.c_int]
        L.or_hier_create_lean.restype = C.c_void_p
        L.or_hier_create_lean.argtypes = [C.c_int, C.POINTER(LevelDesc), C.c_int, C.c_int,
                                          C.c_int]
        L.or_hier_destroy.argtypes = [C.c_void_p]
        L.or_threads.restype = C.c_int
        P = C.c_void_p
        L.or_mg_solve.argtypes = [P, P, P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_double, C.c_int, P, P, P, P]
        L.or_pcg_solve.argtypes = [P, P, P, C.c_double, C.c_int, C.c_double, C.c_int, P, P,
                                   P, P]
        I, D = C.c_int, C.c_double
        L.or_apply.argtypes = [P, I, P, P, P]
        L.or_half_sweep.argtypes = [P, I, P, P, I, D, I, I, D]
        L.or_sweep.argtypes = [P, I, P, P, I, D]
        L.or_ssor.argtypes = [P, I, P, P, D]
        L.or_restrict.argtypes = [P, I, P, P, D]
        L.or_prolong.argtypes = [P, I, P, P]
        _lib = L
    return _lib


def threads() -> int:
    return lib().or_threads()


class Hierarchy:
    """C oracle hierarchy built from oracle.port factor functions."""

    def __init__(self, nx, ny, nlev, factor_fn, omega2, lambda2, periodic=(True, True),
                 lean=False):
        self._keep = []
        descs = (LevelDesc * nlev)()
        self.nx, self.ny = nx, ny
        self.nz = None
        for c in range(nlev):
            fac = factor_fn(nx, ny)
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                    (fac.wx, fac.wy, fac.av, fac.vh, fac.sumw, fac.dr, fac.vprof, fac.volprof)]
            self._keep.append(arrs)
            descs[c] = LevelDesc(nx, ny, fac.nz, omega2, omega2 * lambda2,
                                 *[a.ctypes.data for a in arrs])
            self.nz = fac.nz
            nx //= 2
            ny //= 2
        # lean: no N-sized coefficient caches (recomputed per column, same values)
        self.h = lib().or_hier_create_lean(nlev, descs, int(periodic[0]), int(periodic[1]),
                                           int(bool(lean)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_hier_destroy(self.h)
            self.h = None

    def mg_solve(self, f, eps=1e-5, maxiter=100, nu_pre=1, nu_post=1, coarse_sweeps=1,
                 rho=1.0, max_cycles=0, want_u=True):
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.empty_like(f) if want_u else None
        hist = np.zeros(maxiter + 1)
        it, conv, wall = C.c_int(), C.c_int(), C.c_double()
        lib().or_mg_solve(self.h, f.ctypes.data, None if u is None else u.ctypes.data, eps,
                          maxiter, nu_pre, nu_post, coarse_sweeps, rho, max_cycles,
                          hist.ctypes.data, C.byref(it), C.byref(conv), C.byref(wall))
        n = it.value
        return u, port.Report(n, list(hist[:n + 1]), bool(conv.value), wall.value)

    def pcg_solve(self, f, eps=1e-5, maxiter=500, rho=1.0, max_iters=0, want_u=True):
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.empty_like(f) if want_u else None
        hist = np.zeros(maxiter + 1)
        it, conv, wall = C.c_int(), C.c_int(), C.c_double()
        rc = lib().or_pcg_solve(self.h, f.ctypes.data, None if u is None else u.ctypes.data,
                                eps, maxiter, rho, max_iters, hist.ctypes.data, C.byref(it),
                                C.byref(conv), C.byref(wall))
        if rc == -3:
            raise port.BreakdownError("CG breakdown")
        n = it.value
        return u, port.Report(n, list(hist[:n + 1]), bool(conv.value), wall.value)


    # ---- per-operation entry points (owned (nx, ny, nz) arrays) ---------------

    def _dims(self, c):
        return (self.nx >> c, self.ny >> c, self.nz)

    def apply(self, u, c=0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(self._dims(c))
        lib().or_apply(self.h, c, u.ctypes.data, None, out.ctypes.data)
        return out

    def residual(self, f, u, c=0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.empty(self._dims(c))
        lib().or_apply(self.h, c, u.ctypes.data, f.ctypes.data, out.ctypes.data)
        return out

    def half_sweep(self, u, f, color, rho=1.0, zero_start=False, neighbors_zero=False,
                   post_scale=1.0, c=0):
        """In place on ``u`` (owned array)."""
        f = np.ascontiguousarray(f, dtype=np.float64)
        assert u.flags.c_contiguous and u.dtype == np.float64
        lib().or_half_sweep(self.h, c, u.ctypes.data, f.ctypes.data, color, rho,
                            int(zero_start), int(neighbors_zero), post_scale)

    def sweep(self, u, f, nsweeps=1, rho=1.0, c=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        assert u.flags.c_contiguous and u.dtype == np.float64
        lib().or_sweep(self.h, c, u.ctypes.data, f.ctypes.data, nsweeps, rho)

    def ssor(self, r, rho=1.0, c=0):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(self._dims(c))
        lib().or_ssor(self.h, c, r.ctypes.data, z.ctypes.data, rho)
        return z

    def restrict(self, fine, weight=0.25, c=0):
        fine = np.ascontiguousarray(fine, dtype=np.float64)
        out = np.empty(self._dims(c + 1))
        lib().or_restrict(self.h, c, fine.ctypes.data, out.ctypes.data, weight)
        return out

    def prolong(self, coarse, c=0):
        coarse = np.ascontiguousarray(coarse, dtype=np.float64)
        out = np.empty(self._dims(c))
        lib().or_prolong(self.h, c, coarse.ctypes.data, out.ctypes.data)
        return out


def config_hierarchy(cfg: "port.Config", nlev=None, lean=False):
    return Hierarchy(cfg.nx, cfg.ny, cfg.levels if nlev is None else nlev, cfg.factor_fn(),
                     cfg.omega2, cfg.lambda2, lean=lean)
