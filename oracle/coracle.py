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
        L.or_hier_destroy.argtypes = [C.c_void_p]
        L.or_threads.restype = C.c_int
        P = C.c_void_p
        L.or_mg_solve.argtypes = [P, P, P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_double, C.c_int, P, P, P, P]
        L.or_pcg_solve.argtypes = [P, P, P, C.c_double, C.c_int, C.c_double, C.c_int, P, P,
                                   P, P]
        _lib = L
    return _lib


def threads() -> int:
    return lib().or_threads()


class Hierarchy:
    """C oracle hierarchy built from oracle.port factor functions."""

    def __init__(self, nx, ny, nlev, factor_fn, omega2, lambda2, periodic=(True, True)):
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
        self.h = lib().or_hier_create(nlev, descs, int(periodic[0]), int(periodic[1]))

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


def config_hierarchy(cfg: "port.Config", nlev=None):
    return Hierarchy(cfg.nx, cfg.ny, cfg.levels if nlev is None else nlev, cfg.factor_fn(),
                     cfg.omega2, cfg.lambda2)
