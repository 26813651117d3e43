"""Tensor-product geometric multigrid on the device (reference ``multigrid.py``).

Same level policies, V-cycle (Alg. 1, ``multigrid.py:271-294``) and
stopping rule (``multigrid.py:297-330``).  B200-specific execution:

* the residual is fused with the children-sum restriction
  (``pmg_residual_restrict``): the fine residual is never written to HBM;
* prolongation adds straight into the iterate (``u += P e``), same
  arithmetic as the reference's two steps;
* the convergence check computes ||f - A u||^2 without storing r;
* with all parts on this device the whole V-cycle plus the norm is
  captured once into a CUDA graph (hierarchy-owned scratch) and replayed
  per cycle, so coarse levels are not launch-bound; one 8-byte
  device-to-host read per cycle feeds the stopping test.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from ._lib import MGDesc, PartDesc, call, destroy, load
from .geometry import PanelGrid
from .krylov import SolveReport
from .params import ModelParameters, is_power_of_two
from .partition import (Decomposition, DistField, LevelLayout, _dist, _stream, collect,
                        distribute, dist_norm, halo_exchange, reduce_parts, scalar_buffer)
from .smoother import BLACK, RED, LineSmoother
from .stencil import PanelOperator
from .tracing import nvtx_range, tracing_enabled

POLICIES = ("standard", "shallow", "very_shallow", "explicit")


@dataclass(frozen=True)
class MGConfig:
    """Cycle shape, level policy and stopping rule (multigrid.py:54-89).

    B200 extras (keyword, default on): ``fused`` residual+restriction,
    ``graph`` CUDA-graph replay of the V-cycle, ``lagged_norm``: the
    native driver sums each cycle's ||f - A u|| inside the next cycle's
    first red half-sweep (the black residual is exactly zero after the
    last black line solve with rho = 1), so the convergence check costs no
    separate pass; same iterates bit for bit, the history omits the black
    cells' rounding-level residual; ``red_restrict``:
    the pre-smoothed residual is restricted from its red cells only (the
    black residual after the exact black line solves is zero), 14 instead
    of 18 bytes per cell -- fast smoother mode only (the exact mode stays
    bit-identical to the reference); ``overlap``: multi-part solves relax
    the part boundaries first and exchange their halos while the interior
    relaxes on levels of at least ``OVERLAP_NX`` columns per
    part -- same values bit for bit.
    """

    nu_pre: int = 1
    nu_post: int = 1
    policy: str = "standard"
    explicit_levels: int | None = None
    coarse_sweeps: int | None = None
    eps: float = 1e-5
    maxiter: int = 100
    l_split: int | None = None
    rho: float = 1.0
    deterministic: bool = False
    fused: bool = True
    graph: bool = True
    lagged_norm: bool = True
    red_restrict: bool = True
    overlap: bool = True

    def __post_init__(self):
        if self.nu_pre < 0 or self.nu_post < 0 or self.nu_pre + self.nu_post < 1:
            raise ValueError("need at least one smoothing step per level")
        if self.policy not in POLICIES:
            raise ValueError(f"policy must be one of {POLICIES}")
        if self.policy == "explicit" and (self.explicit_levels is None
                                          or self.explicit_levels < 1):
            raise ValueError("explicit policy needs explicit_levels >= 1")
        if not 0.0 < self.eps < 1.0:
            raise ValueError("eps must lie in (0, 1)")
        if self.maxiter < 1:
            raise ValueError("maxiter must be positive")
        if not 0.0 < self.rho < 2.0:
            raise ValueError("overrelaxation weight must lie in (0, 2)")
        if self.coarse_sweeps is not None and self.coarse_sweeps < 1:
            raise ValueError("coarse_sweeps must be positive")

    def resolved_coarse_sweeps(self) -> int:
        if self.coarse_sweeps is not None:
            return self.coarse_sweeps
        return 5 if self.policy == "very_shallow" else 1


@dataclass
class Level:
    grid: PanelGrid
    layout: LevelLayout
    op: PanelOperator
    smoother: LineSmoother
    fold_layout: LevelLayout | None = None

    @property
    def nx(self) -> int:
        return self.grid.nx


@dataclass
class _Scratch:
    u: DistField
    f: DistField
    r: DistField


class LevelHierarchy:
    """Ladder of levels, finest first (multigrid.py:116-155)."""

    def __init__(self, levels, decomp: Decomposition, params: ModelParameters):
        self.levels = levels
        self.decomp = decomp
        self.params = params
        self._persist = None
        self._graphs = {}
        self._native = {}

    def __len__(self) -> int:
        return len(self.levels)

    @property
    def fine(self) -> Level:
        return self.levels[0]

    def level_sizes(self):
        return [lev.nx for lev in self.levels]

    def first_fold_level(self):
        """Level number (finest = len(self)) below which workers fold
        (multigrid.py:135-140)."""
        for c, lev in enumerate(self.levels):
            if lev.fold_layout is not None:
                return len(self.levels) - c - 1
        return None

    def make_scratch(self):
        nz = self.params.nz if self.params.nz == self.fine.grid.nz else self.fine.grid.nz
        return [_Scratch(DistField.zeros(lev.layout, nz), DistField.zeros(lev.layout, nz),
                         DistField.zeros(lev.layout, nz)) for lev in self.levels]

    def reset_counters(self) -> None:
        for lev in self.levels:
            lev.layout.halo_count = 0
        self.decomp.collect_calls = 0
        self.decomp.distribute_calls = 0

    def persistent_scratch(self):
        if self._persist is None:
            self._persist = self.make_scratch()
        return self._persist

    def native_parts(self, cfg: "MGConfig") -> "NativePartsHierarchy":
        """The multi-part device-resident driver (pmg_phier) of this
        hierarchy for ``cfg`` (cached); under torch.distributed with NCCL it
        runs over the library's own communicator."""
        from .partition import native_comm
        key = ("parts", cfg.nu_pre, cfg.nu_post, cfg.resolved_coarse_sweeps(), cfg.rho,
               bool(cfg.red_restrict), bool(cfg.overlap), bool(cfg.lagged_norm))
        h = self._native.get(key)
        if h is None:
            h = NativePartsHierarchy(self, cfg, native_comm() if _dist() is not None else None)
            self._native[key] = h
        return h

    def native(self, cfg: "MGConfig") -> "NativeHierarchy":
        """The device-resident driver (pmg_hier) of this single-part
        hierarchy for ``cfg``'s cycle shape (cached)."""
        key = (cfg.nu_pre, cfg.nu_post, cfg.resolved_coarse_sweeps(), cfg.rho,
               bool(cfg.lagged_norm), bool(cfg.red_restrict))
        h = self._native.get(key)
        if h is None:
            h = NativeHierarchy(self, cfg)
            self._native[key] = h
        return h


class NativeHierarchy:
    """Owner of a ``pmg_hier``: the C++ V-cycle / mg_solve driver over this
    hierarchy's level handles (include/pmg.h, drivers section)."""

    def __init__(self, hier: LevelHierarchy, cfg: "MGConfig"):
        lay = hier.fine.layout
        if len(lay.local_workers) != 1 or lay.px != 1 or lay.py != 1:
            raise ValueError("the native driver runs single-part hierarchies")
        w = lay.local_workers[0]
        self._levels = [lev.op.handles[w] for lev in hier.levels]   # keep alive
        arr = (C.c_void_p * len(self._levels))(*[h.h.value for h in self._levels])
        per = int(bool(lay.periodic))
        d = MGDesc(cfg.nu_pre, cfg.nu_post, cfg.resolved_coarse_sweeps(), float(cfg.rho), per,
                   per, int(bool(cfg.lagged_norm)), int(bool(cfg.red_restrict)))
        h = C.c_void_p()
        call("pmg_hier_create", arr, len(self._levels), C.byref(d), C.byref(h))
        self.h = h
        self._lib = load()

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            destroy("pmg_hier_destroy", h)
            self.h = None

    def graph_launches(self, f_ptr: int, u_ptr: int, first: bool) -> int:
        return int(self._lib.pmg_hier_graph_launches(self.h, f_ptr, u_ptr, int(first)))

    def replayed_launches(self) -> int:
        """Cumulative kernels issued by this driver's graph replays."""
        return int(self._lib.pmg_hier_replayed_launches(self.h))


#: narrowest part (columns) that relaxes boundary-first in a multi-part solve
OVERLAP_NX = 1024


class NativePartsHierarchy:
    """Owner of a ``pmg_phier``: the C++ multi-part V-cycle / mg_solve driver
    over every part this process holds (all of them in-process, or one per
    rank with the library's NCCL communicator), halo exchanges and
    reductions issued inside the captured cycle graph (include/pmg.h,
    multi-part drivers)."""

    def __init__(self, hier: LevelHierarchy | None, cfg: "MGConfig", comm=None, ops=None):
        # ``ops``: operators of the levels, finest first (default: the
        # hierarchy's); a one-level list serves the CG driver
        ops = [lev.op for lev in hier.levels] if ops is None else ops
        lay = ops[0].layout
        ws = list(lay.local_workers)
        self._levels = [[op.handles[w] for op in ops] for w in ws]   # keep alive
        flat = [h.h.value for hs in self._levels for h in hs]
        arr = (C.c_void_p * len(flat))(*flat)
        parts = (PartDesc * len(ws))()
        for n, w in enumerate(ws):
            parts[n].worker = w
            for face, (di, dj) in enumerate(((-1, 0), (1, 0), (0, -1), (0, 1))):
                nb = lay.neighbor(w, di, dj)
                parts[n].nbr[face] = -1 if nb is None else nb
            for corner, (di, dj) in enumerate(((-1, -1), (1, -1), (-1, 1), (1, 1))):
                nb = lay.neighbor(w, di, dj)
                parts[n].diag[corner] = -1 if nb is None else nb
        per = int(bool(lay.periodic))
        d = MGDesc(cfg.nu_pre, cfg.nu_post, cfg.resolved_coarse_sweeps(), float(cfg.rho), per,
                   per, int(bool(cfg.lagged_norm)), int(bool(cfg.red_restrict)))
        h = C.c_void_p()
        call("pmg_phier_create", arr, len(ops), len(ws), parts, C.byref(d),
             comm, OVERLAP_NX if cfg.overlap else 0, C.byref(h))
        self.h = h
        self.workers = ws
        self._lib = load()

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            destroy("pmg_phier_destroy", h)
            self.h = None

    def replayed_launches(self) -> int:
        return int(self._lib.pmg_phier_replayed_launches(self.h))

    def exchanges(self) -> int:
        return int(self._lib.pmg_phier_exchanges(self.h))

    def ptrs(self, df: DistField):
        return (C.c_void_p * len(self.workers))(*[df.parts[w].data.data_ptr()
                                                  for w in self.workers])


def _level_count(nx: int, pside: int, cfg: MGConfig) -> int:
    lmax = int(math.log2(nx)) + 1
    if cfg.policy == "standard":
        return lmax
    if cfg.policy == "shallow":
        return int(math.log2(nx // pside)) + 1
    if cfg.policy == "very_shallow":
        return min(4, lmax)
    if cfg.explicit_levels > lmax:
        raise ValueError(f"{cfg.explicit_levels} levels would coarsen an nx={nx} grid "
                         f"below one column (at most {lmax})")
    return cfg.explicit_levels


def build_hierarchy(grid: PanelGrid, params: ModelParameters, cfg: MGConfig,
                    decomp: Decomposition | None = None) -> LevelHierarchy:
    """Grids, layouts, operators and smoothers of every level (multigrid.py:173-206)."""
    if not (is_power_of_two(grid.nx) and is_power_of_two(grid.ny)):
        raise ValueError("multigrid needs a power-of-two horizontal size")
    if decomp is None:
        decomp = Decomposition(grid.nx, 1, ny=grid.ny, periodic=grid.periodic)
    decomp.bind_periodic(grid.periodic)
    side = min(decomp.px, decomp.py)
    nlev = _level_count(min(grid.nx, grid.ny), side, cfg)
    if cfg.l_split is not None and not 1 <= cfg.l_split <= nlev:
        raise ValueError(f"l_split must lie in [1, {nlev}]")
    levels = []
    g = grid
    apx, apy = decomp.px, decomp.py
    for c in range(nlev):
        # active workers: as many per direction as the level has columns,
        # fewer below l_split (reference multigrid.py:188-199)
        wx, wy = apx, apy
        paper_level = nlev - c
        if cfg.l_split is not None and paper_level <= cfg.l_split:
            folds = cfg.l_split - paper_level + 1
            wx, wy = max(1, decomp.px >> folds), max(1, decomp.py >> folds)
        apx, apy = min(apx, wx, g.nx), min(apy, wy, g.ny)
        layout = decomp.layout(g.nx, active=(apx, apy))
        op = PanelOperator(g, params, layout)
        levels.append(Level(g, layout, op, LineSmoother(op)))
        if c + 1 < nlev:
            g = g.coarsen()
    for c in range(nlev - 1):
        fine, coarse = levels[c], levels[c + 1]
        fl, cl = fine.layout, coarse.layout
        if (cl.px, cl.py) != (fl.px, fl.py):
            if fl.px not in (cl.px, 2 * cl.px) or fl.py not in (cl.py, 2 * cl.py):
                raise ValueError("worker folding must at most halve the active grid per level")
            fine.fold_layout = decomp.layout(fine.nx, active=(cl.px, cl.py))
    return LevelHierarchy(levels, decomp, params)


def restrict(df: DistField, fine: Level, coarse: Level) -> DistField:
    """Cell-average restriction (mean of the 4 children, multigrid.py:226-230)."""
    out = DistField.zeros(coarse.layout, df.nz)
    _restrict_into(df, fine, coarse, out, 0.25)
    return out


def _restrict_into(df: DistField, fine: Level, coarse: Level, out: DistField,
                   weight: float) -> DistField:
    """coarse f = weight x children sum; a folding level first collects the
    fine parts onto the coarse level's workers (multigrid.py:216-223)."""
    if fine.fold_layout is not None:
        df = collect(df, fine.fold_layout)
    st = _stream()
    for w, ff in df.parts.items():
        call("pmg_restrict", ff.geom.h, out.parts[w].geom.h, ff.ptr, out.parts[w].ptr,
             float(weight), st)
    return out


def prolong(df: DistField, coarse: Level, fine: Level, out: DistField | None = None) -> DistField:
    """Bilinear cell-centre interpolation (multigrid.py:249-268); the
    coarse halo (incl. corners) must be current.  Across a fold the result
    is staged on the folded workers and distributed."""
    st = _stream()
    if fine.fold_layout is not None:
        staged = DistField.zeros(fine.fold_layout, df.nz)
        for w, cf in df.parts.items():
            call("pmg_prolong", staged.parts[w].geom.h, cf.geom.h, cf.ptr,
                 staged.parts[w].ptr, 0, st)
        return distribute(staged, fine.layout, out=out)
    if out is None:
        out = DistField.zeros(fine.layout, df.nz)
    for w, cf in df.parts.items():
        call("pmg_prolong", out.parts[w].geom.h, cf.geom.h, cf.ptr, out.parts[w].ptr, 0, st)
    return out


def _prolong_add(cu: DistField, coarse: Level, fine: Level, u: DistField,
                 black_only: bool = False, exchange: bool = False) -> None:
    """u += P e (into black cells only if ``black_only``); ``exchange``
    also refreshes u's halo."""
    st = _stream()
    for w, cf in cu.parts.items():
        call("pmg_prolong_colors", fine.op.handles[w].h, coarse.op.handles[w].h, cf.ptr,
             u.parts[w].ptr, 1, 2 if black_only else 3, st)
    if exchange:
        halo_exchange(u)


def _residual_restrict(lev: Level, coarse: Level, f: DistField, u: DistField,
                       cf: DistField, red_only: bool = False) -> None:
    """cf = R (f - A u) (pmg_residual_restrict); ``red_only``: right after
    an exact black half-sweep with rho = 1 the black residual is zero and
    only the red children are summed (pmg_residual_restrict_red), where
    the level allows it."""
    st = _stream()
    lib = load()
    for w, uf in u.parts.items():
        h = lev.op.handles[w].h
        name = ("pmg_residual_restrict_red"
                if red_only and lib.pmg_residual_restrict_red_ok(h) else "pmg_residual_restrict")
        call(name, h, coarse.op.handles[w].h, f.parts[w].ptr, uf.ptr, cf.parts[w].ptr, st)


def self_coupled(hier: LevelHierarchy) -> bool:
    """A periodic level one column wide (nx = 1 or ny = 1 of a rectangular
    periodic grid coarsened far enough) makes every cell its own neighbour
    through the wrap.  The identities the fused cycle rests on -- the black
    half-sweep never reads black values, the black residual after an exact
    black line solve is zero -- do not hold there."""
    return any(lev.grid.periodic and (lev.grid.nx == 1 or lev.grid.ny == 1)
               for lev in hier.levels)


def plain_if_self_coupled(hier: LevelHierarchy, cfg: MGConfig) -> MGConfig:
    """The cycle configuration the drivers run: ``cfg``, or -- on a
    hierarchy with a self-coupled level -- the reference's plain op sequence
    (zero fills, full prolongation, full residual and restriction, the
    separate convergence norm), which needs none of those identities."""
    if (cfg.fused or cfg.lagged_norm or cfg.red_restrict) and self_coupled(hier):
        return replace(cfg, fused=False, lagged_norm=False, red_restrict=False)
    return cfg


def v_cycle(hier: LevelHierarchy, cfg: MGConfig, scratch, c: int = 0,
            first: bool = False) -> None:
    """One V-cycle on ``scratch[c].u`` (halo-consistent on entry), Alg. 1.

    With ``cfg.fused`` and rho = 1 two pieces of provably dead work are
    skipped (bit-identical result): the zero fill of the coarse iterate (its
    first red half-sweep runs with neighbours_zero, rhs = f exactly as
    f + drw*0, and the black half-sweep never reads old black values) and the
    prolongation into red cells (the post-smoothing red half-sweep overwrites
    them without reading them).
    """
    if c == 0:
        cfg = plain_if_self_coupled(hier, cfg)
    with nvtx_range(f"level {c}"):
        _v_cycle_level(hier, cfg, scratch, c, first)


def _v_cycle_level(hier: LevelHierarchy, cfg: MGConfig, scratch, c: int, first: bool) -> None:
    lev = hier.levels[c]
    s = scratch[c]
    lean = cfg.fused and cfg.rho == 1.0
    if c + 1 < len(hier.levels):
        # ``first``: the finest iterate is zero on entry but was not filled
        _pre_smooth(lev, s, cfg.nu_pre, cfg.rho, lean and (c > 0 or first))
        coarse = hier.levels[c + 1]
        fold = lev.fold_layout is not None
        if cfg.fused and not fold:
            _residual_restrict(lev, coarse, s.f, s.u, scratch[c + 1].f,
                               cfg.red_restrict and lean and cfg.nu_pre >= 1)
        else:
            lev.op.residual(s.f, s.u, out=s.r)
            _restrict_into(s.r, lev, coarse, scratch[c + 1].f, 1.0)
        if not (lean and (cfg.nu_pre >= 1 or c + 2 == len(hier.levels))):
            scratch[c + 1].u.fill(0.0)
        v_cycle(hier, cfg, scratch, c + 1)
        post = cfg.nu_post
        if fold:
            corr = prolong(scratch[c + 1].u, coarse, lev, out=s.r)
            _add_owned(s.u, corr)
            halo_exchange(s.u)
        elif cfg.fused:
            _prolong_add(scratch[c + 1].u, coarse, lev, s.u, black_only=lean and post >= 1,
                         exchange=True)
        else:
            corr = prolong(scratch[c + 1].u, coarse, lev, out=s.r)
            _add_owned(s.u, corr)
            halo_exchange(s.u)
        lev.smoother.sweep(s.u, s.f, post, cfg.rho)
    else:
        _pre_smooth(lev, s, cfg.resolved_coarse_sweeps(), cfg.rho, lean and c > 0)


def _pre_smooth(lev: Level, s: _Scratch, nsweeps: int, rho: float, from_zero: bool) -> None:
    """``nsweeps`` red-black sweeps; ``from_zero``: the iterate is zero on
    entry but was not filled, so the first red half-sweep ignores u."""
    for n in range(nsweeps):
        lev.smoother.half_sweep_exchange(s.u, s.f, RED, rho, neighbors_zero=(from_zero and n == 0))
        lev.smoother.half_sweep_exchange(s.u, s.f, BLACK, rho)


def _add_owned(u: DistField, e: DistField) -> None:
    """u += e on owned cells (multigrid.py:287-290); halos are refreshed by
    the exchange that follows, so the full-array add is equivalent."""
    for w, uf in u.parts.items():
        call("pmg_axpy", uf.geom.ndoubles, 1.0, e.parts[w].ptr, uf.ptr, _stream())


def _echo(hier: LevelHierarchy, cfg: MGConfig) -> dict:
    return {"solver": "mg", "policy": cfg.policy, "levels": len(hier.levels),
            "nu_pre": cfg.nu_pre, "nu_post": cfg.nu_post, "rho": cfg.rho,
            "coarse_sweeps": cfg.resolved_coarse_sweeps(), "eps": cfg.eps,
            "maxiter": cfg.maxiter, "deterministic": cfg.deterministic,
            "workers": hier.decomp.workers}


class _CycleGraph:
    """CUDA graph of one V-cycle + fine residual norm over ``scratch``
    (whose level-0 entries may be the caller's f and iterate)."""

    def __init__(self, hier: LevelHierarchy, cfg: MGConfig, scratch, first: bool):
        self.res = scalar_buffer(len(scratch[0].u.parts))
        s0 = scratch[0]
        fine = hier.fine
        # warm-up outside capture (allocations, kernel attributes); it runs
        # on the solve's own buffers before the iteration starts, and the
        # first cycle never reads the iterate's initial contents
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            v_cycle(hier, cfg, scratch, first=first)
            fine.op.residual_norm2_dev(s0.f, s0.u, None, self.res)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        from .partition import lib
        l0 = lib().pmg_launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            v_cycle(hier, cfg, scratch, first=first)
            fine.op.residual_norm2_dev(s0.f, s0.u, None, self.res)
        self.launches = lib().pmg_launch_count() - l0   # library kernels per replay

    def replay(self, clock: list | None = None) -> torch.Tensor:
        """One cycle; ``clock`` (tracing): append its device milliseconds."""
        if clock is None:
            self.graph.replay()
            return self.res
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        self.graph.replay()
        b.record()
        b.synchronize()
        clock.append(a.elapsed_time(b))
        return self.res


#: single-part graph solves run the C++ driver (pmg_mg_solve); False keeps
#: the Python V-cycle (same kernels, same order: bit-identical results)
USE_NATIVE = True
#: multi-part solves (in-process parts, or one part per rank over NCCL) run
#: the C++ multi-part driver (pmg_phier_mg_solve); False keeps the Python
#: V-cycle (same kernels, same order: bit-identical results)
USE_NATIVE_PARTS = True


def _mg_solve_native(f: DistField, hier: LevelHierarchy, cfg: MGConfig, out):
    """mg_solve through pmg_mg_solve: the V-cycle sequence of ``v_cycle``
    (fused path) captured once per buffer pair into a CUDA graph by the
    library, one 8-byte host read per cycle."""
    nh = hier.native(cfg)
    if out is None:
        u = hier.persistent_scratch()[0].u
    else:
        u = out
    (w, uf), = u.parts.items()
    fp = f.parts[w]
    hist = np.zeros(cfg.maxiter + 1)
    iters, conv = C.c_int(), C.c_int()
    torch.cuda.current_stream().synchronize()
    t0 = time.perf_counter()
    call("pmg_mg_solve", nh.h, fp.ptr, uf.ptr, float(cfg.eps), int(cfg.maxiter),
         hist.ctypes.data_as(C.c_void_p), C.byref(iters), C.byref(conv), _stream())
    wall = time.perf_counter() - t0
    history = hist[:iters.value + 1].tolist()
    if out is None:
        u = u.copy()
    return u, SolveReport(iters.value, history, bool(conv.value), wall, _echo(hier, cfg),
                          cycle_times_ms=_cycle_times(nh._lib.pmg_hier_cycle_times, nh.h))


def _cycle_times(fn, h) -> list:
    """Per-cycle device times of a driver's last solve (empty when untraced)."""
    n = int(fn(h, None, 0))
    if n <= 0:
        return []
    buf = np.zeros(n)
    fn(h, buf.ctypes.data_as(C.c_void_p), n)
    return buf.tolist()


def _parts_native_ok(hier: LevelHierarchy, cfg: MGConfig) -> bool:
    """The multi-part native driver takes hierarchies without folding whose
    parts all live here (in-process) or one per rank over NCCL."""
    from .partition import native_comm_ok
    if not (cfg.graph and cfg.fused and USE_NATIVE and len(hier) > 0):
        return False
    if any(lev.fold_layout is not None for lev in hier.levels):
        return False
    if _dist() is not None:
        return native_comm_ok()
    return True


def _mg_solve_parts(f: DistField, hier: LevelHierarchy, cfg: MGConfig, out):
    """mg_solve through pmg_phier_mg_solve: every part's V-cycle, the halo
    exchanges (boundary-first where the level allows) and the reductions in
    one captured graph per cycle, one 8-byte host read per cycle."""
    nh = hier.native_parts(cfg)
    u = out if out is not None else hier.persistent_scratch()[0].u
    hist = np.zeros(cfg.maxiter + 1)
    iters, conv = C.c_int(), C.c_int()
    torch.cuda.current_stream().synchronize()
    t0 = time.perf_counter()
    call("pmg_phier_mg_solve", nh.h, nh.ptrs(f), nh.ptrs(u), float(cfg.eps), int(cfg.maxiter),
         hist.ctypes.data_as(C.c_void_p), C.byref(iters), C.byref(conv), _stream())
    wall = time.perf_counter() - t0
    history = hist[:iters.value + 1].tolist()
    if out is None:
        u = u.copy()
    return u, SolveReport(iters.value, history, bool(conv.value), wall, _echo(hier, cfg),
                          cycle_times_ms=_cycle_times(nh._lib.pmg_phier_cycle_times, nh.h))


def _ptrs(df: DistField):
    return tuple(p.data.data_ptr() for p in df.parts.values())


def graph_key(cfg: MGConfig, f: DistField, u: DistField) -> tuple:
    """Cache key of the Python driver's captured cycle graphs (+ first):
    cycle shape, buffers, and the process-wide kernel selection (smoother
    mode) the graph's kernels were chosen under."""
    return (cfg.nu_pre, cfg.nu_post, cfg.rho, cfg.resolved_coarse_sweeps(), cfg.fused,
            cfg.red_restrict, _ptrs(f), _ptrs(u), int(load().pmg_get_smoother_mode()))


def mg_solve(f: DistField, hier: LevelHierarchy, cfg: MGConfig, out: DistField | None = None):
    """Repeat V-cycles from u = 0 until ||r|| / ||r0|| < eps (multigrid.py:297-330).

    Non-convergence within ``maxiter`` is reported, not raised.

    B200 execution: ``f`` is read in place (never copied) and, if ``out`` is
    given, the iterate lives in ``out`` -- the V-cycle graphs are captured
    over those buffers and cached per buffer identity, so repeated solves
    copy nothing.  Without ``out`` a fresh field is returned.  With rho = 1
    the first cycle starts from zero without a fill (its first red
    half-sweep ignores u, exactly as f + drw*0 = f).
    """
    cfg = plain_if_self_coupled(hier, cfg)
    use_graph = cfg.graph and _dist() is None
    single = hier.fine.layout.px == 1 and hier.fine.layout.py == 1 and _dist() is None
    if (use_graph and cfg.fused and USE_NATIVE and single):
        return _mg_solve_native(f, hier, cfg, out)
    if not single and USE_NATIVE_PARTS and _parts_native_ok(hier, cfg):
        return _mg_solve_parts(f, hier, cfg, out)
    coarse = hier.persistent_scratch() if use_graph else hier.make_scratch()
    # iterate: the caller's ``out``; else the hierarchy's level-0 scratch
    # (graph reuse across calls), copied out at the end
    u = out if out is not None else coarse[0].u
    scratch = [_Scratch(u, f, coarse[0].r)] + coarse[1:]
    r0 = dist_norm(f, cfg.deterministic)
    history = [r0]
    echo = _echo(hier, cfg)
    if r0 == 0.0:
        u.fill(0.0)
        return (u if out is not None else u.copy()), SolveReport(0, history, True, 0.0, echo)
    lean_first = (cfg.fused and cfg.rho == 1.0 and cfg.nu_pre >= 1 and len(hier.levels) > 1)
    graphs = {}
    if use_graph:
        base = graph_key(cfg, f, u)
        for first in ((True, False) if lean_first else (False,)):
            key = base + (first,)
            g = hier._graphs.get(key)
            if g is None:
                if len(hier._graphs) > 16:          # bound the cache
                    hier._graphs.clear()
                g = _CycleGraph(hier, cfg, scratch, first)
                hier._graphs[key] = g
            graphs[first] = g
    if not lean_first:
        u.fill(0.0)
    res = scalar_buffer(len(u.parts))
    converged = False
    clock = [] if tracing_enabled() else None
    torch.cuda.current_stream().synchronize()
    t0 = time.perf_counter()
    for it in range(cfg.maxiter):
        first = lean_first and it == 0
        with nvtx_range(f"cycle {it + 1}"):
            if use_graph:
                rr = graphs[first].replay(clock)
            else:
                v_cycle(hier, cfg, scratch, first=first)
                hier.fine.op.residual_norm2_dev(f, u, None, res)
                rr = res
        rnorm = math.sqrt(reduce_parts(rr))
        history.append(rnorm)
        if rnorm / r0 < cfg.eps:
            converged = True
            break
    wall = time.perf_counter() - t0
    if out is None:
        u = u.copy()
    return u, SolveReport(len(history) - 1, history, converged, wall, echo,
                          cycle_times_ms=clock or [])
