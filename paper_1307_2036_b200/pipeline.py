"""Pipelined end-to-end solves: host right-hand sides in, host solutions out.

``SolvePipeline.run`` is the public entry point for a stream of solves on
one hierarchy (e.g. one pressure solve per time step).  For step i it
uploads step i+1's right-hand side and downloads step i-1's solution on
side streams while step i's V-cycles run, double-buffering the device
fields, so PCIe traffic in both directions overlaps the solve.  Each step
is exactly ``scatter_block -> mg_solve -> owned_to`` (same results).
Within a step the block moves in SLABS of columns (i is the slowest index
of the reference layout, so a slab is a contiguous piece of the host
block): the layout kernel converts slab c while slab c + 1 is still on the
bus, in both directions, so a lone step pays the conversion of one slab
only on top of the two transfers.
Single part per process (one GPU per rank).
"""

from __future__ import annotations

import ctypes as C

import torch

from ._lib import call
from .multigrid import MGConfig, mg_solve
from .partition import DistField, _stream


#: slabs per block transfer (fewer when a slab would fall below 64 MB)
SLABS = 8


class SolvePipeline:
    def __init__(self, hier, cfg: MGConfig, nz: int, slabs: int = SLABS,
                 min_slab_bytes: int = 64 << 20):
        lay = hier.fine.layout
        if len(lay.local_workers) != 1:
            raise ValueError("SolvePipeline needs exactly one local part")
        self.hier, self.cfg, self.lay = hier, cfg, lay
        (self.w,) = lay.local_workers
        self.geom = lay.geometry(self.w, nz)
        n = self.geom.mx * self.geom.my * nz
        self.n = n
        self.fdev = [DistField.zeros(lay, nz) for _ in range(2)]
        self.udev = [DistField.zeros(lay, nz) for _ in range(2)]
        self.stage_in = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        self.stage_out = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        self.s_h2d = torch.cuda.Stream()
        self.s_d2h = torch.cuda.Stream()
        # slabs of whole 32-column tiles, >= 64 MB each (PCIe efficiency)
        mx = self.geom.mx
        per_col = self.geom.my * nz
        nslab = max(1, min(slabs, (mx + 31) // 32, (n * 8) // max(1, min_slab_bytes)))
        step = ((mx + nslab - 1) // nslab + 31) // 32 * 32
        self.slabs = [(i0, min(mx, i0 + step)) for i0 in range(0, mx, step)]
        self.per_col = per_col

    def _upload(self, i: int, f_host: torch.Tensor, consumed: list) -> list:
        """Enqueue the slab-wise H2D copy of step i's block; one event per slab."""
        b = i % 2
        src, dst = f_host.reshape(-1), self.stage_in[b]
        evs = []
        with torch.cuda.stream(self.s_h2d):
            if consumed[b] is not None:
                self.s_h2d.wait_event(consumed[b])
            for i0, i1 in self.slabs:
                a, e = i0 * self.per_col, i1 * self.per_col
                dst[a:e].copy_(src[a:e], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_h2d)
                evs.append(ev)
        return evs

    def run(self, f_hosts, u_hosts):
        """Solve A u_i = f_i for every pinned host block f_hosts[i]
        ((mx, my, nz) reference layout), writing u_hosts[i]; returns the
        SolveReports.  Host buffers should be pinned for the overlap."""
        comp = torch.cuda.current_stream()
        nsteps = len(f_hosts)
        consumed = [None, None]       # stage_in[b] free again (after from_ref)
        drained = [None, None]        # stage_out[b] free again (after D2H)
        up = [None] * nsteps
        reports = []
        if nsteps:
            up[0] = self._upload(0, f_hosts[0], consumed)
        for i in range(nsteps):
            b = i % 2
            fd, ud = self.fdev[b], self.udev[b]
            for (i0, i1), arrived in zip(self.slabs, up[i]):
                comp.wait_event(arrived)
                call("pmg_from_ref_layout_slab", self.geom.h,
                     C.c_void_p(self.stage_in[b].data_ptr()), fd.parts[self.w].ptr, i0, i1,
                     _stream())
            ev = torch.cuda.Event()
            ev.record(comp)
            consumed[b] = ev
            if i + 1 < nsteps:                      # next upload overlaps this solve
                up[i + 1] = self._upload(i + 1, f_hosts[i + 1], consumed)
            _, rep = mg_solve(fd, self.hier, self.cfg, out=ud)
            reports.append(rep)
            if drained[b] is not None:
                comp.wait_event(drained[b])
            dst, src = u_hosts[i].reshape(-1), self.stage_out[b]
            for i0, i1 in self.slabs:
                call("pmg_to_ref_layout_slab", self.geom.h, ud.parts[self.w].ptr,
                     C.c_void_p(src.data_ptr()), i0, i1, _stream())
                done = torch.cuda.Event()
                done.record(comp)
                with torch.cuda.stream(self.s_d2h):
                    self.s_d2h.wait_event(done)
                    a, e = i0 * self.per_col, i1 * self.per_col
                    dst[a:e].copy_(src[a:e], non_blocking=True)
            dev = torch.cuda.Event()
            dev.record(self.s_d2h)
            drained[b] = dev
        self.s_d2h.synchronize()
        comp.synchronize()
        return reports
