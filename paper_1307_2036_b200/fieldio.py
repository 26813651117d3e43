"""``ANMG`` binary field container (reference ``field.py:12-15, 81-108``).

Magic ``ANMG``, four little-endian uint32 (rows, cols, nz, flags), then the
float64 payload in the reference layout (vertical index fastest); flag bit
0 = the stored array includes the one-cell halo ring.  Used to exchange
right-hand sides and solutions with the CPU reference.
"""

from __future__ import annotations

import numpy as np

MAGIC = b"ANMG"
FLAG_HAS_HALO = 1


def dump_array(path, arr: np.ndarray, has_halo: bool = False) -> None:
    """Write a (rows, cols, nz) array (owned block, or with halo ring)."""
    arr = np.ascontiguousarray(arr, dtype="<f8")
    if arr.ndim != 3:
        raise ValueError("field array must be 3-d (rows, cols, nz)")
    header = np.array([arr.shape[0], arr.shape[1], arr.shape[2],
                       FLAG_HAS_HALO if has_halo else 0], dtype="<u4")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(header.tobytes())
        fh.write(arr.tobytes())


def load_array(path) -> np.ndarray:
    """Read a dump; returns the OWNED (rows, cols, nz) block (halo stripped)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != MAGIC:
            raise ValueError(f"not a field dump (bad magic {magic!r})")
        rows, cols, nz, flags = (int(x) for x in np.frombuffer(fh.read(16), dtype="<u4"))
        payload = np.frombuffer(fh.read(rows * cols * nz * 8), dtype="<f8")
    if payload.size != rows * cols * nz:
        raise ValueError("truncated field dump")
    arr = payload.reshape(rows, cols, nz).astype(np.float64)
    if flags & FLAG_HAS_HALO:
        arr = arr[1:-1, 1:-1, :].copy()
    return arr


def dump_field(path, df) -> None:
    """Gather a DistField and write its owned values (no halo)."""
    from .partition import gather_owned
    dump_array(path, gather_owned(df), has_halo=False)


def load_field(path, layout):
    """Read a dump and scatter it over ``layout``."""
    from .partition import scatter_owned
    return scatter_owned(load_array(path), layout)


class Field:
    """Host field in the reference layout (field.py:28-108): an
    (m + 2, m + 2, nz) float64 array with a one-cell halo ring, vertical
    index fastest.  The exchange format between host codes and the device
    solvers (``scatter_owned(field.owned, layout)``)."""

    def __init__(self, data: np.ndarray):
        data = np.asarray(data)
        if data.ndim != 3 or data.shape[0] != data.shape[1] or data.shape[0] < 3:
            raise ValueError("field data must be (m + 2, m + 2, nz) with m >= 1")
        self.data = np.ascontiguousarray(data, dtype=np.float64)

    @classmethod
    def zeros(cls, m: int, nz: int) -> "Field":
        return cls(np.zeros((m + 2, m + 2, nz)))

    @classmethod
    def from_owned(cls, owned: np.ndarray) -> "Field":
        owned = np.asarray(owned, dtype=np.float64)
        if owned.ndim != 3 or owned.shape[0] != owned.shape[1]:
            raise ValueError("owned block must be (m, m, nz)")
        f = cls.zeros(owned.shape[0], owned.shape[2])
        f.owned[...] = owned
        return f

    @property
    def owned(self) -> np.ndarray:
        return self.data[1:-1, 1:-1, :]

    @property
    def m(self) -> int:
        return self.data.shape[0] - 2

    @property
    def nz(self) -> int:
        return self.data.shape[2]

    def copy(self) -> "Field":
        return Field(self.data.copy())

    def fill(self, value: float) -> None:
        self.data.fill(value)

    def flat_index(self, i: int, j: int, k: int) -> int:
        """Offset of array index (i, j, k) (halo ring included: owned cells
        are 1..m) in the flattened data."""
        return self.nz * ((self.m + 2) * i + j) + k

    def dump(self, path, include_halo: bool = True) -> None:
        if include_halo:
            dump_array(path, self.data, has_halo=True)
        else:
            dump_array(path, self.owned, has_halo=False)

    @classmethod
    def load(cls, path) -> "Field":
        """Read a dump; a dump with its halo ring restores the ring too."""
        with open(path, "rb") as fh:
            fh.read(4)
            rows, cols, nz, flags = (int(x) for x in np.frombuffer(fh.read(16), dtype="<u4"))
        if rows != cols:
            raise ValueError("field dump must be square in the horizontal")
        if flags & FLAG_HAS_HALO:
            arr = load_array(path)            # validates, strips the ring
            with open(path, "rb") as fh:
                fh.seek(20)
                full = np.frombuffer(fh.read(rows * cols * nz * 8), dtype="<f8")
            return cls(full.reshape(rows, cols, nz).astype(np.float64))
        return cls.from_owned(load_array(path))
