"""Model parameters (reference ``params.py:75-107``).

Only the parameter container the solver API needs is mirrored; the
physics-derived schedules of the reference (``derive_parameters`` and
friends, Table 1) are outside the hot path.  ``derive_parameters`` is
provided with the reference's formula so reference call sites work.
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


def derive_parameters(nx: int, nz: int, dt: float, wave_speed: float = 550.0,
                      earth_radius: float = 6.371e6, buoyancy_freq: float = 0.018,
                      off_centering: float = 0.5, f_omega2: float = 1.0,
                      f_lambda2: float = 1.0) -> ModelParameters:
    """omega^2 = (alpha c dt / R)^2 f_omega2, lambda^2 = f_lambda2 /
    (1 + (alpha dt N)^2), dx = 2 pi R / (4 nx) (params.py:110-149)."""
    if not (isinstance(nx, int) and nx >= 4 and is_power_of_two(nx)):
        raise ValueError(f"nx must be a power of two >= 4, got {nx}")
    if nz < 2:
        raise ValueError(f"nz must be at least 2, got {nz}")
    if dt <= 0.0:
        raise ValueError(f"dt must be positive, got {dt}")
    dx = 2.0 * math.pi * earth_radius / (4.0 * nx)
    omega2 = (off_centering * wave_speed * dt / earth_radius) ** 2 * f_omega2
    lambda2 = f_lambda2 / (1.0 + (off_centering * dt * buoyancy_freq) ** 2)
    return ModelParameters(nx=nx, nz=nz, dx=dx, dt=dt, omega2=omega2, lambda2=lambda2,
                           courant=wave_speed * dt / dx, f_omega2=f_omega2,
                           f_lambda2=f_lambda2)
