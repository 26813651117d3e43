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
