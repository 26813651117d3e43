"""Model parameters (reference ``params.py``).

The parameter container the solver API needs, plus the physics-derived
coefficients the experiment harness (``experiment.py``) uses: the
reference's formulas for omega^2 / lambda^2 from (nx, nz, dt), the
fixed-Courant refinement schedule and the anisotropy ratio
(``params.py:41-203``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class ModelParameters:
    """omega^2, lambda^2 and the grid they belong to (params.py:75-107)."""

    nx: int
    nz: int
    dx: float
    dt: float
    omega2: float
    lambda2: float
    courant: float
    f_omega2: float = 1.0
    f_lambda2: float = 1.0

    def __post_init__(self):
        if not is_power_of_two(self.nx):
            raise ValueError("nx must be a power of two (horizontal coarsening halves it)")
        if self.nz < 1:
            raise ValueError("nz must be at least 1")
        if self.dx <= 0.0 or self.dt <= 0.0:
            raise ValueError("dx and dt must be strictly positive")
        if self.omega2 < 0.0 or self.lambda2 < 0.0:
            raise ValueError("omega2 and lambda2 must be non-negative")

    @property
    def dof(self) -> int:
        return self.nx * self.nx * self.nz


def toy_parameters(nx: int, nz: int, omega2: float, lambda2: float) -> ModelParameters:
    """Hand-set coefficients (the reference's ``tests/conftest.py:24-27``
    pattern and the way the BASELINE configs set omega^2, lambda^2)."""
    return ModelParameters(nx=nx, nz=nz, dx=1.0 / nx, dt=1.0, omega2=omega2,
                           lambda2=lambda2, courant=1.0)


@dataclass(frozen=True)
class PhysicalConstants:
    """Constants of the model problem (params.py:41-70): fastest wave speed
    c [m/s], earth radius R [m], buoyancy frequency N [1/s], shell depth H
    (dimensionless, in units of R) and the off-centering weight alpha."""

    wave_speed: float = 550.0
    earth_radius: float = 6.371e6
    buoyancy_freq: float = 0.018
    shell_depth: float = 0.01
    off_centering: float = 0.5

    def __post_init__(self):
        for name in ("wave_speed", "earth_radius", "buoyancy_freq", "shell_depth"):
            if not getattr(self, name) > 0.0:
                raise ValueError(f"{name} must be strictly positive")
        if not 0.0 < self.off_centering <= 1.0:
            raise ValueError("off_centering must lie in (0, 1]")


DEFAULT_CONSTANTS = PhysicalConstants()


def derive_parameters(nx: int, nz: int, dt: float,
                      constants: PhysicalConstants = DEFAULT_CONSTANTS,
                      f_omega2: float = 1.0, f_lambda2: float = 1.0) -> ModelParameters:
    """omega^2 = (alpha c dt / R)^2 f_omega2, lambda^2 = f_lambda2 /
    (1 + (alpha dt N)^2), dx = 2 pi R / (4 nx), Courant = c dt / dx
    (params.py:110-149)."""
    if not (isinstance(nx, int) and nx >= 4 and is_power_of_two(nx)):
        raise ValueError(f"nx must be a power of two >= 4, got {nx}")
    if nz < 2:
        raise ValueError(f"nz must be at least 2, got {nz}")
    if dt <= 0.0:
        raise ValueError(f"dt must be positive, got {dt}")
    if f_omega2 <= 0.0 or f_lambda2 <= 0.0:
        raise ValueError("robustness multipliers must be positive")
    k = constants
    dx = 2.0 * math.pi * k.earth_radius / (4.0 * nx)
    omega2 = (k.off_centering * k.wave_speed * dt / k.earth_radius) ** 2 * f_omega2
    lambda2 = f_lambda2 / (1.0 + (k.off_centering * dt * k.buoyancy_freq) ** 2)
    return ModelParameters(nx=nx, nz=nz, dx=dx, dt=dt, omega2=omega2, lambda2=lambda2,
                           courant=k.wave_speed * dt / dx, f_omega2=f_omega2,
                           f_lambda2=f_lambda2)


def weak_scaling_schedule(base: ModelParameters, doublings: int,
                          constants: PhysicalConstants = DEFAULT_CONSTANTS):
    """nx doubled and dt halved ``doublings`` times: the Courant number is
    held exactly (params.py:152-174)."""
    if doublings < 0:
        raise ValueError("doublings must be non-negative")
    return [derive_parameters(base.nx * 2 ** i, base.nz, base.dt / 2 ** i, constants,
                              base.f_omega2, base.f_lambda2) for i in range(doublings + 1)]


def anisotropy(params: ModelParameters, grid, k: int,
               constants: PhysicalConstants = DEFAULT_CONSTANTS) -> float:
    """beta_k = lambda^2 (dx / dz_k)^2 with dz_k the physical thickness of
    vertical cell k (params.py:177-187)."""
    if not 0 <= k < grid.nz:
        raise ValueError(f"vertical cell index {k} out of range [0, {grid.nz})")
    dz = (grid.levels[k + 1] - grid.levels[k]) * constants.earth_radius
    return params.lambda2 * (params.dx / dz) ** 2


def horizontal_coupling(params: ModelParameters, level: int,
                        constants: PhysicalConstants = DEFAULT_CONSTANTS) -> float:
    """(alpha Courant)^2 / 4^level: the fine-grid horizontal coupling after
    ``level`` coarsenings (params.py:190-203)."""
    if level < 0:
        raise ValueError("coarsening depth must be non-negative")
    return (constants.off_centering * params.courant) ** 2 * 4.0 ** (-level)
