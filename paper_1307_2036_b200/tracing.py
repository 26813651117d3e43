"""Tracing mode.

The reference's only instrumentation is wall time around the iteration
loop (``multigrid.py:321,329``, ``krylov.py:125,159``) plus communication
counters (``LevelLayout.halo_count``, ``Decomposition.collect_calls``) --
both kept here too.  With tracing on:

* the library's drivers push NVTX ranges (solve, cycle / CG iteration,
  level, halo exchange; the level ranges mark the capture of a cycle graph,
  the cycle ranges every replay) and time every cycle on the device with a
  CUDA event pair read after the per-cycle host sync they already do;
* the Python drivers push the same ranges (``torch.cuda.nvtx``) and time
  their graph replays the same way;
* ``SolveReport.cycle_times_ms`` holds the device time of each V-cycle.

Off by default; a profiler (Nsight Systems) shows the ranges, nothing here
depends on one being attached.
"""

from __future__ import annotations

from contextlib import contextmanager

from ._lib import call, load

__all__ = ["set_tracing", "tracing_enabled", "tracing", "nvtx_range"]


def set_tracing(on: bool) -> None:
    call("pmg_set_tracing", 1 if on else 0)


def tracing_enabled() -> bool:
    return bool(load().pmg_get_tracing())


@contextmanager
def tracing(on: bool = True):
    prev = tracing_enabled()
    set_tracing(on)
    try:
        yield
    finally:
        set_tracing(prev)


@contextmanager
def nvtx_range(name: str):
    """An NVTX range around the block while tracing is on (no-op otherwise)."""
    if not tracing_enabled():
        yield
        return
    import torch
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()
