"""Pipelined end-to-end solves: host right-hand sides in, host solutions out.

``SolvePipeline.run`` is the public entry point for a stream of solves on
one hierarchy (e.g. one pressure solve per time step).  For step i it
uploads step i+1's right-hand side and downloads step i-1's solution on
side streams while step i's V-cycles run, double-buffering the device
fields, so PCIe traffic in both directions overlaps the solve.  Each step
is exactly ``scatter_block -> mg_solve -> owned_to`` (same results).
Single part per process (one GPU per rank).
"""

from __future__ import annotations

import ctypes as C

import torch

from ._lib import call
from .multigrid import MGConfig, mg_solve
from .partition import DistField, _stream


class SolvePipeline:
    def __init__(self, hier, cfg: MGConfig, nz: int):
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

    def _upload(self, i: int, f_host: torch.Tensor, consumed: list) -> torch.cuda.Event:
        b = i % 2
        with torch.cuda.stream(self.s_h2d):
            if consumed[b] is not None:
                self.s_h2d.wait_event(consumed[b])
            self.stage_in[b].copy_(f_host.reshape(-1), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.s_h2d)
        return ev

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
            comp.wait_event(up[i])
            fd, ud = self.fdev[b], self.udev[b]
            call("pmg_from_ref_layout", self.geom.h, C.c_void_p(self.stage_in[b].data_ptr()),
                 fd.parts[self.w].ptr, _stream())
            ev = torch.cuda.Event()
            ev.record(comp)
            consumed[b] = ev
            if i + 1 < nsteps:                      # next upload overlaps this solve
                up[i + 1] = self._upload(i + 1, f_hosts[i + 1], consumed)
            _, rep = mg_solve(fd, self.hier, self.cfg, out=ud)
            reports.append(rep)
            if drained[b] is not None:
                comp.wait_event(drained[b])
            call("pmg_to_ref_layout", self.geom.h, ud.parts[self.w].ptr,
                 C.c_void_p(self.stage_out[b].data_ptr()), _stream())
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(done)
                u_hosts[i].reshape(-1).copy_(self.stage_out[b], non_blocking=True)
                dev = torch.cuda.Event()
                dev.record(self.s_d2h)
                drained[b] = dev
        self.s_d2h.synchronize()
        comp.synchronize()
        return reports
