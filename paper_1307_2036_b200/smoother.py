"""Block red-black vertical-line relaxation on the device (reference
``smoother.py``).

One half-sweep updates every column of one colour with a Thomas solve of
its vertical tridiagonal block (``smoother.py:122-170``), ``pmg_half_sweep``
on the device.  The default (fast) column solver is k-segmented: the
linear forward / backward recurrences are solved per segment of levels by
separate warps and joined by short scans (~1e-15 relative from the
sequential recurrence); on the large levels of nz = 128 it runs in the
TMA-fed band kernel (rows streamed once through shared memory), below in
the register kernel, and for variable coefficients in their
per-column-coefficient variants.  ``exact_smoother()`` selects the
sequential recurrence in the reference's operation order (bit-identical to
the reference).  DESIGN.md section 3.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass

from ._lib import call, load
from .partition import DistField, _stream, halo_exchange
from .stencil import PanelOperator

RED, BLACK = 0, 1
ORDERINGS = ("redblack", "symmetric", "jacobi")


def set_exact_smoother(exact: bool) -> None:
    """Select the column solver of every half-sweep in this process:
    exact=False (default) -- k-segmented solve (reassociated elimination,
    ~1e-15 relative from the sequential recurrence), the fast path;
    exact=True -- the sequential Thomas recurrence of smoother.py:151-161,
    bit-identical to the reference.  Variable-coefficient levels always
    run the exact solver."""
    call("pmg_set_smoother_mode", 1 if exact else 0)


def exact_smoother_enabled() -> bool:
    return bool(load().pmg_get_smoother_mode())


@contextmanager
def exact_smoother(exact: bool = True):
    prev = exact_smoother_enabled()
    set_exact_smoother(exact)
    try:
        yield
    finally:
        set_exact_smoother(prev)


@dataclass(frozen=True)
class SmootherConfig:
    """Overrelaxation weight, sweep count and ordering (smoother.py:39-53)."""

    rho: float = 1.0
    sweeps: int = 1
    ordering: str = "redblack"

    def __post_init__(self):
        if not 0.0 < self.rho < 2.0:
            raise ValueError("overrelaxation weight must lie in (0, 2)")
        if self.sweeps < 0:
            raise ValueError("sweep count must be non-negative")
        if self.ordering not in ORDERINGS:
            raise ValueError(f"ordering must be one of {ORDERINGS}")


class LineSmoother:
    """Red-black (or Jacobi) line relaxation bound to one level operator."""

    def __init__(self, op: PanelOperator):
        self.op = op
        self._tmp = None

    def half_sweep(self, u: DistField, f: DistField, color: int, rho: float = 1.0,
                   zero_start: bool = False, neighbors_zero: bool = False,
                   post_scale: float = 1.0) -> None:
        """Update all columns of one colour; no halo exchange."""
        st = _stream()
        for w, uf in u.parts.items():
            call("pmg_half_sweep", self.op.handles[w].h, uf.ptr, f.parts[w].ptr, int(color),
                 float(rho), int(bool(zero_start)), int(bool(neighbors_zero)),
                 float(post_scale), st)

    def half_sweep_exchange(self, u: DistField, f: DistField, color: int, rho: float = 1.0,
                            zero_start: bool = False, neighbors_zero: bool = False,
                            post_scale: float = 1.0) -> None:
        """half_sweep followed by halo_exchange (one exchange)."""
        self.half_sweep(u, f, color, rho, zero_start, neighbors_zero, post_scale)
        halo_exchange(u)

    def sweep(self, u: DistField, f: DistField, nsweeps: int = 1, rho: float = 1.0) -> None:
        """Red-black sweeps with a halo exchange after each half (smoother.py:184-191)."""
        for _ in range(nsweeps):
            self.half_sweep_exchange(u, f, RED, rho)
            self.half_sweep_exchange(u, f, BLACK, rho)

    def symmetric_sweep(self, u: DistField, f: DistField, nsweeps: int = 1,
                        rho: float = 1.0) -> None:
        """Forward (red, black) then backward (black, red) (smoother.py:193-208)."""
        for _ in range(nsweeps):
            self.half_sweep(u, f, RED, rho)
            halo_exchange(u)
            self.half_sweep(u, f, BLACK, rho)
            if rho != 1.0:
                self.half_sweep(u, f, BLACK, rho)
            halo_exchange(u)
            self.half_sweep(u, f, RED, rho)
            halo_exchange(u)

    def jacobi_sweep(self, u: DistField, f: DistField, nsweeps: int = 1,
                     rho: float = 1.0) -> None:
        """Block-Jacobi: every column from the pre-sweep state, one exchange
        per sweep (smoother.py:210-222).  Black is relaxed in a copy so it
        still sees the old red columns; the split layout then copies the
        black colour array back in one memcpy."""
        for _ in range(nsweeps):
            tmp = u.copy()
            self.half_sweep(u, f, RED, rho)
            self.half_sweep(tmp, f, BLACK, rho)
            for w, uf in u.parts.items():
                cs = uf.geom.cstride
                uf.data[cs:].copy_(tmp.parts[w].data[cs:])
            halo_exchange(u)

    def ssor_apply(self, r: DistField, rho: float = 1.0, out: DistField | None = None) -> DistField:
        """z = M^{-1} r, symmetric red-black block SSOR from zero
        (smoother.py:224-244): red (zero start, no neighbours), black (zero
        start, x (2 - rho)), red; three exchanges."""
        # the reference zero-fills z first (smoother.py:235-238); that fill is
        # dead work here: the first red half-sweep ignores z (neighbours zero,
        # zero start), the black one reads only the fresh red values
        z = DistField.zeros(self.op.layout, self.op.nz) if out is None else out
        if out is not None and getattr(self.op, "self_coupled", False):
            z.fill(0.0)      # not dead there: the black half-sweep reads copies of black
        self.half_sweep_exchange(z, r, RED, rho, zero_start=True, neighbors_zero=True)
        self.half_sweep_exchange(z, r, BLACK, rho, zero_start=True, post_scale=2.0 - rho)
        self.half_sweep_exchange(z, r, RED, rho)
        return z


def smooth(u: DistField, f: DistField, smoother: LineSmoother, cfg: SmootherConfig) -> DistField:
    """Run ``cfg.sweeps`` sweeps of the configured ordering in place (smoother.py:247-256)."""
    if cfg.ordering == "redblack":
        smoother.sweep(u, f, cfg.sweeps, cfg.rho)
    elif cfg.ordering == "symmetric":
        smoother.symmetric_sweep(u, f, cfg.sweeps, cfg.rho)
    else:
        smoother.jacobi_sweep(u, f, cfg.sweeps, cfg.rho)
    return u


def apply_ssor_preconditioner(r: DistField, smoother: LineSmoother,
                              cfg: SmootherConfig) -> DistField:
    return smoother.ssor_apply(r, cfg.rho)
