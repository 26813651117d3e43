"""Horizontal domain decomposition, device fields, halo exchange, reductions.

Mirrors the reference communication layer (``partition.py``) with real
devices behind it:

* a worker ("part") owns an ``mx x my`` block of whole vertical columns
  (``PAPER.md:527``); its field lives in HBM in the red/black split,
  horizontal-fastest layout of ``include/pmg.h``;
* with ``torch.distributed`` initialised and ``world_size > 1`` every rank
  owns exactly one part and halos / reductions go over NCCL (or gloo);
  otherwise all parts live on the current device in one process, which
  is how the reference's simulated workers (``partition.py:1-19``) and
  its partition-invariance tests are reproduced on one GPU;
* one part that is its own neighbour in both directions refreshes its
  halo ring with a single kernel (``pmg_halo_self``).

The decomposition is a px x py grid of parts (the reference's 4^p square
tilings are the special case px = py = 2^p).  Coarse levels keep every
worker active (no folding): build hierarchies with at least one column
per part on the coarsest level.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from ._lib import LevelDesc, call

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _lib.load()
    return _LIB


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dist():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist
    return None


_COMM = None


def native_comm_ok() -> bool:
    """The library's own NCCL communicator can serve this process group:
    torch.distributed over NCCL (device buffers), one GPU per rank, and
    libnccl.so.2 loadable by the library."""
    d = _dist()
    return (d is not None and d.get_backend() == "nccl" and torch.cuda.is_available()
            and bool(lib().pmg_comm_available()))


def native_comm():
    """The process-wide pmg_comm over the torch.distributed world (created
    once: rank 0's NCCL unique id is broadcast through torch.distributed,
    then ncclCommInitRank on every rank's current device)."""
    global _COMM
    if _COMM is None:
        d = _dist()
        if d is None:
            raise ValueError("native_comm needs an initialised torch.distributed world")
        uid = (C.c_ubyte * 128)()
        if d.get_rank() == 0:
            call("pmg_comm_unique_id", uid)
        box = [bytes(uid)]
        d.broadcast_object_list(box, src=0)
        uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        comm = C.c_void_p()
        call("pmg_comm_create", uid, d.get_world_size(), d.get_rank(), C.byref(comm))
        _COMM = comm
    return _COMM


def _split_workers(workers: int):
    """px x py for a worker count: 4^p -> square (reference), 2 -> 2x1,
    8 -> 4x2 (BASELINE configs[3])."""
    if workers < 1 or workers & (workers - 1):
        raise ValueError(f"worker count must be a power of two (got {workers})")
    a = workers.bit_length() - 1
    px = 1 << ((a + 1) // 2)
    return px, workers // px


class Decomposition:
    """Static px x py tiling of the finest level (reference
    ``Decomposition``, partition.py:45-68)."""

    def __init__(self, nx: int, workers: int = 1, ny: int | None = None, px: int | None = None,
                 py: int | None = None, periodic: bool | None = None):
        ny = nx if ny is None else ny
        if px is None or py is None:
            px, py = _split_workers(workers)
        if px * py != workers:
            raise ValueError(f"{px} x {py} process grid does not hold {workers} workers")
        if nx % px or ny % py:
            raise ValueError(f"grid {nx} x {ny} not divisible by the {px} x {py} worker grid")
        self.nx, self.ny = nx, ny
        self.workers = workers
        self.px, self.py = px, py
        self.pside = px if px == py else None
        self.periodic = periodic
        self.collect_calls = 0
        self.distribute_calls = 0
        self._layouts = {}

    def layout(self, nx_level: int, pside: int | None = None, active=None) -> "LevelLayout":
        """Layout of a level with ``nx_level`` columns (and the decomposition's
        aspect ratio).  By default as many workers stay active per direction
        as the level has columns (reference partition.py:60-68); ``pside``
        (square, reference API) or ``active`` = (apx, apy) choose fewer: the
        coarse-level folding of the standard policy."""
        ny_level = nx_level * self.ny // self.nx
        if active is None:
            if pside is not None:
                active = (pside, pside)
            else:
                active = (min(self.px, nx_level), min(self.py, ny_level))
        apx, apy = active
        key = (nx_level, ny_level, apx, apy)
        if key not in self._layouts:
            self._layouts[key] = LevelLayout(self, nx_level, ny_level, apx, apy)
        return self._layouts[key]

    def bind_periodic(self, periodic: bool) -> None:
        if self.periodic is None:
            self.periodic = bool(periodic)
        elif self.periodic != bool(periodic):
            raise ValueError("decomposition already bound to the other boundary type")


def decompose(nx: int, workers: int) -> Decomposition:
    """The reference's validating constructor (partition.py:71-73): a square
    tiling of 4^p workers.  ``Decomposition`` itself also takes the 2 x 1 and
    4 x 2 grids of BASELINE configs[3]."""
    side = math.isqrt(workers) if workers >= 1 else 0
    if side * side != workers or side & (side - 1):
        raise ValueError(f"worker count must be 4^p (got {workers})")
    if nx % side:
        raise ValueError(f"nx={nx} not divisible by sqrt(workers)={side}")
    return Decomposition(nx, workers)


class LevelLayout:
    """Owned rectangles of one grid level (reference ``LevelLayout``,
    partition.py:76-118).  Worker ids index the full px x py grid
    (id = wi * py + wj); on a folded level only an apx x apy sub-grid is
    active, every (px / apx) x (py / apy) group represented by its
    lowest-indexed worker."""

    def __init__(self, decomp: Decomposition, nx: int, ny: int, apx: int | None = None,
                 apy: int | None = None):
        apx = decomp.px if apx is None else apx
        apy = decomp.py if apy is None else apy
        for a, p in ((apx, decomp.px), (apy, decomp.py)):
            if a < 1 or a & (a - 1) or p % a:
                raise ValueError("active side must be a power of two dividing the worker grid")
        if nx % apx or ny % apy:
            raise ValueError(f"level {nx} x {ny} not divisible by the {apx} x {apy} active "
                             "worker grid")
        self.decomp = decomp
        self.nx, self.ny = nx, ny
        self.px, self.py = apx, apy
        self.gx, self.gy = decomp.px // apx, decomp.py // apy
        self.mx, self.my = nx // apx, ny // apy
        self.pside = apx if apx == apy else None
        self.mloc = self.mx
        self.group = self.gx
        self.workers = [self.worker_at(ai, aj) for ai in range(apx) for aj in range(apy)]
        self.halo_count = 0
        self._geom = {}
        d = _dist()
        if d is not None:
            if d.get_world_size() != decomp.workers:
                raise ValueError("one worker per rank: world size must equal the worker count")
            # one part per rank; on a folded level (fewer active workers)
            # the ranks outside the active sub-grid hold no part
            r = d.get_rank()
            self.local_workers = [r] if r in self.workers else []
        else:
            self.local_workers = list(self.workers)

    @property
    def periodic(self) -> bool:
        return bool(self.decomp.periodic)

    def coords(self, worker: int):
        wi, wj = divmod(worker, self.decomp.py)
        if wi % self.gx or wj % self.gy:
            raise ValueError(f"worker {worker} not active on this layout")
        return wi // self.gx, wj // self.gy

    def worker_at(self, ai: int, aj: int) -> int:
        return (ai * self.gx) * self.decomp.py + aj * self.gy

    def origin(self, worker: int):
        ai, aj = self.coords(worker)
        return ai * self.mx, aj * self.my

    def neighbor(self, worker: int, di: int, dj: int):
        ai, aj = self.coords(worker)
        ni, nj = ai + di, aj + dj
        if self.periodic:
            return self.worker_at(ni % self.px, nj % self.py)
        if 0 <= ni < self.px and 0 <= nj < self.py:
            return self.worker_at(ni, nj)
        return None

    def geometry(self, worker: int, nz: int) -> "LevelHandle":
        """Layout-only level handle of one part (unit factors)."""
        key = (worker, nz)
        h = self._geom.get(key)
        if h is None:
            i0, j0 = self.origin(worker)
            h = LevelHandle.unit(self.mx, self.my, nz, i0, j0)
            self._geom[key] = h
        return h


class LevelHandle:
    """Owner of one ``pmg_level`` (coefficients + layout of one part)."""

    def __init__(self, mx, my, nz, i0, j0, omega2, vcoef, dr, vprof, volprof,
                 wx, wy, av, vh, sumw):
        self._keep = [np.ascontiguousarray(a, dtype=np.float64)
                      for a in (dr, vprof, volprof, wx, wy, av, vh, sumw)]
        ptr = [a.ctypes.data_as(C.c_void_p) for a in self._keep]
        desc = LevelDesc(mx, my, nz, i0, j0, float(omega2), float(vcoef), *ptr)
        h = C.c_void_p()
        call("pmg_level_create", C.byref(desc), C.byref(h))
        self.h = h
        self.mx, self.my, self.nz = mx, my, nz
        self.i0, self.j0 = i0, j0
        self.ndoubles = int(lib().pmg_level_field_doubles(h))
        pitch, plane, cstr = C.c_int(), C.c_longlong(), C.c_longlong()
        par, uni = C.c_int(), C.c_int()
        call("pmg_level_layout", h, C.byref(pitch), C.byref(plane), C.byref(cstr),
             C.byref(par), C.byref(uni))
        self.pitch, self.plane, self.cstride = pitch.value, plane.value, cstr.value
        self.parity, self.uniform = par.value, bool(uni.value)
        self._keep = None

    @classmethod
    def unit(cls, mx, my, nz, i0, j0):
        one = np.ones(1)
        return cls(mx, my, nz, i0, j0, 0.0, 0.0, np.ones(nz), np.ones(nz + 1), np.ones(nz),
                   np.broadcast_to(one, (my, mx + 1)), np.broadcast_to(one, (my + 1, mx)),
                   np.broadcast_to(one, (my, mx)), np.broadcast_to(one, (my, mx)),
                   np.broadcast_to(one, (my, mx)))

    def tables(self):
        nz = self.nz
        d, b, v = np.empty(nz), np.empty(nz + 1), np.empty(nz)
        call("pmg_level_tables", self.h, d.ctypes.data_as(C.c_void_p),
             b.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p))
        return d, b, v

    def __del__(self):
        try:
            if self.h:
                from ._lib import destroy
                destroy("pmg_level_destroy", self.h)
                self.h = None
        except Exception:
            pass


class DevField:
    """One part of a field in HBM (flat float64 tensor, split layout)."""

    __slots__ = ("geom", "data")

    def __init__(self, geom: LevelHandle, data: torch.Tensor | None = None):
        self.geom = geom
        if data is None:
            data = torch.zeros(geom.ndoubles, dtype=torch.float64, device="cuda")
        self.data = data

    @property
    def ptr(self):
        return C.c_void_p(self.data.data_ptr())

    @property
    def m(self):
        return self.geom.mx

    @property
    def nz(self):
        return self.geom.nz

    def copy(self) -> "DevField":
        return DevField(self.geom, self.data.clone())

    def fill(self, value: float) -> None:
        self.data.fill_(value)

    def owned_array(self) -> np.ndarray:
        """(mx, my, nz) host copy of the owned cells (reference layout)."""
        g = self.geom
        buf = torch.empty(g.mx * g.my * g.nz, dtype=torch.float64, device=self.data.device)
        call("pmg_to_ref_layout", g.h, self.ptr, C.c_void_p(buf.data_ptr()), _stream())
        return buf.cpu().numpy().reshape(g.mx, g.my, g.nz)

    def owned_to(self, host: torch.Tensor, staging: torch.Tensor | None = None) -> None:
        """Copy the owned cells into a preallocated (pinned) host tensor of
        mx*my*nz doubles, reference layout; synchronous."""
        g = self.geom
        n = g.mx * g.my * g.nz
        buf = staging if staging is not None else torch.empty(n, dtype=torch.float64,
                                                              device=self.data.device)
        call("pmg_to_ref_layout", g.h, self.ptr, C.c_void_p(buf.data_ptr()), _stream())
        host.view(-1).copy_(buf[:n], non_blocking=host.is_pinned())
        torch.cuda.current_stream().synchronize()

    def load_owned(self, arr, staging: torch.Tensor | None = None) -> None:
        """Write an (mx, my, nz) block (numpy or torch, host or device)."""
        g = self.geom
        if isinstance(arr, np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
        else:
            t = arr.contiguous()
        if t.numel() != g.mx * g.my * g.nz:
            raise ValueError("block does not match the part size")
        if t.device.type != "cuda":
            dev = staging if staging is not None else torch.empty(
                t.numel(), dtype=torch.float64, device=self.data.device)
            dev[:t.numel()].copy_(t.reshape(-1), non_blocking=t.is_pinned())
            t = dev
        call("pmg_from_ref_layout", g.h, C.c_void_p(t.data_ptr()), self.ptr, _stream())


class DistField:
    """A field split over the parts of one layout (reference ``DistField``,
    partition.py:121-155).  ``parts`` holds the parts hosted here."""

    __slots__ = ("layout", "parts", "_nz")

    def __init__(self, layout: LevelLayout, parts: dict, nz: int | None = None):
        self.layout = layout
        self.parts = parts
        self._nz = nz

    @classmethod
    def zeros(cls, layout: LevelLayout, nz: int) -> "DistField":
        return cls(layout, {w: DevField(layout.geometry(w, nz)) for w in layout.local_workers},
                   nz)

    @property
    def nz(self) -> int:
        # a rank that is inactive on a folded level holds no part
        if self._nz is None:
            self._nz = next(iter(self.parts.values())).nz
        return self._nz

    def copy(self) -> "DistField":
        return DistField(self.layout, {w: f.copy() for w, f in self.parts.items()}, self._nz)

    def copy_from(self, other: "DistField") -> None:
        for w, f in self.parts.items():
            f.data.copy_(other.parts[w].data)

    def fill(self, value: float) -> None:
        for f in self.parts.values():
            f.fill(value)

    def add_scaled(self, alpha: float, other: "DistField") -> None:
        """self += alpha * other over the full arrays, halo included
        (partition.py:145-148)."""
        for w, f in self.parts.items():
            call("pmg_axpy", f.geom.ndoubles, float(alpha), other.parts[w].ptr, f.ptr,
                 _stream())

    def scale_plus(self, beta: float, other: "DistField") -> None:
        """self = other + beta * self over the full arrays (partition.py:150-155)."""
        for w, f in self.parts.items():
            call("pmg_xpby", f.geom.ndoubles, other.parts[w].ptr, float(beta), f.ptr,
                 _stream())


# ---------------------------------------------------------------------------
# halo exchange (partition.py:158-191)
# ---------------------------------------------------------------------------
_OPP = {0: 1, 1: 0, 2: 3, 3: 2}
_DIR = {0: (-1, 0), 1: (1, 0), 2: (0, -1), 3: (0, 1)}


class _FaceBuffers:
    cache = {}

    @classmethod
    def get(cls, geom: LevelHandle, tag: str, face: int, owner: int = -1) -> torch.Tensor:
        key = (geom.mx, geom.my, geom.nz, tag, face, owner)
        t = cls.cache.get(key)
        if t is None:
            n = int(lib().pmg_face_doubles(geom.h, face))
            t = torch.empty(n, dtype=torch.float64, device="cuda")
            cls.cache[key] = t
        return t


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def halo_exchange(df: DistField) -> None:
    """Refresh every halo cell: x strips first, then y strips over the
    extended range (corners), periodic wrap or mirror at physical
    boundaries.  Counted once per call on the layout."""
    lay = df.layout
    st = _stream()
    if not df.parts:          # a rank outside a folded level's active grid
        lay.halo_count += 1
        return
    if lay.px == 1 and lay.py == 1:
        f = df.parts[lay.workers[0]]
        call("pmg_halo_self", f.geom.h, f.ptr, int(lay.periodic), int(lay.periodic), st)
        lay.halo_count += 1
        return
    d = _dist()
    for faces in ((0, 1), (2, 3)):
        if d is None:
            _phase_local(df, faces, st)
        else:
            _phase_dist(df, faces, st, d)
    lay.halo_count += 1


def _phase_local(df: DistField, faces, st) -> None:
    lay = df.layout
    for w, f in df.parts.items():
        for face in faces:
            nb = lay.neighbor(w, *_DIR[face])
            if nb is None:
                call("pmg_unpack_face", f.geom.h, f.ptr, face, None, 1, st)
                continue
            src = df.parts[nb]
            buf = _FaceBuffers.get(f.geom, "local", face)
            call("pmg_pack_face", src.geom.h, src.ptr, _OPP[face], _ptr(buf), st)
            call("pmg_unpack_face", f.geom.h, f.ptr, face, _ptr(buf), 0, st)


def exchange_plan(lay: LevelLayout, w: int, faces):
    """Message plan of one part for one phase: [(send_face, peer_send,
    recv_face, peer_recv)], ordered [send f0, recv h1, send f1, recv h0]
    so that two faces exchanged with the same peer (2 ranks along a
    periodic axis) pair up correctly under NCCL's in-order matching; gloo
    matches them by tag (= the sender's face index)."""
    a, b = faces
    return [(sf, lay.neighbor(w, *_DIR[sf]), rf, lay.neighbor(w, *_DIR[rf]))
            for sf, rf in ((a, b), (b, a))]


def exchange_messages(dist, w: int, plan, sendbufs: dict, recvbufs: dict) -> dict:
    """Post the plan's sends/receives (device-agnostic: NCCL with CUDA
    tensors, gloo with CPU tensors) and wait.  Returns recv_face ->
    "buf" (recvbufs[face] holds the neighbour strip), "mirror"
    (physical boundary) or "self" (own neighbour: copied locally)."""
    ops, how = [], {}
    for sf, ps, rf, pr in plan:
        if ps == w and pr == w:
            recvbufs[rf].copy_(sendbufs[sf])
            how[rf] = "self"
            continue
        if ps is not None:
            ops.append(dist.P2POp(dist.isend, sendbufs[sf], ps, tag=sf))
        if pr is not None:
            ops.append(dist.P2POp(dist.irecv, recvbufs[rf], pr, tag=sf))
            how[rf] = "buf"
        else:
            how[rf] = "mirror"
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return how


def _phase_dist(df: DistField, faces, st, dist) -> None:
    """One rank = one part: pack own faces, exchange, unpack halos."""
    lay = df.layout
    (w, f), = df.parts.items()
    plan = exchange_plan(lay, w, faces)
    sendbufs, recvbufs = {}, {}
    for sf, ps, rf, pr in plan:
        sendbufs[sf] = _FaceBuffers.get(f.geom, "send", sf, w)
        recvbufs[rf] = _FaceBuffers.get(f.geom, "recv", rf, w)
        if ps is not None:
            call("pmg_pack_face", f.geom.h, f.ptr, sf, _ptr(sendbufs[sf]), st)
    if dist.get_backend() == "nccl" or not f.data.is_cuda:
        how = exchange_messages(dist, w, plan, sendbufs, recvbufs)
    else:
        # host-staged exchange for CPU backends (gloo): device faces -> host,
        # send/recv, host -> device (the NCCL path moves device buffers)
        torch.cuda.current_stream().synchronize()
        hs = {k: v.cpu() for k, v in sendbufs.items()}
        hr = {k: torch.empty(v.shape, dtype=v.dtype) for k, v in recvbufs.items()}
        how = exchange_messages(dist, w, plan, hs, hr)
        for k, v in hr.items():
            if how.get(k) in ("buf", "self"):
                recvbufs[k].copy_(v)
    for face, kind in how.items():
        if kind == "mirror":
            call("pmg_unpack_face", f.geom.h, f.ptr, face, None, 1, st)
        else:
            call("pmg_unpack_face", f.geom.h, f.ptr, face, _ptr(recvbufs[face]), 0, st)


# ---------------------------------------------------------------------------
# global <-> parts (partition.py:243-264)
# ---------------------------------------------------------------------------
def collect(df: DistField, to_layout: LevelLayout) -> DistField:
    """Fold each group of parts onto its lowest-indexed worker (reference
    partition.py:194-218): the owned blocks are copied into one part of
    ``to_layout`` (same nx, fewer active workers); halos are left zero."""
    lay = df.layout
    fx, fy = lay.px // to_layout.px, lay.py // to_layout.py
    if (to_layout.nx != lay.nx or to_layout.ny != lay.ny or fx * to_layout.px != lay.px
            or fy * to_layout.py != lay.py or fx * fy < 2):
        raise ValueError("collect target must fold the active grid at the same level size")
    out = DistField.zeros(to_layout, df.nz)
    st = _stream()
    d = _dist()
    if d is not None:
        _collect_dist(df, out, fx, fy, st, d)
        lay.decomp.collect_calls += 1
        return out
    for pw, big in out.parts.items():
        ai, aj = to_layout.coords(pw)
        for di in range(fx):
            for dj in range(fy):
                ch = df.parts[lay.worker_at(fx * ai + di, fy * aj + dj)]
                call("pmg_copy_block", ch.geom.h, ch.ptr, big.geom.h, big.ptr, 0, 0,
                     di * lay.mx, dj * lay.my, lay.mx, lay.my, st)
    lay.decomp.collect_calls += 1
    return out


def fold_root(lay: LevelLayout, to_layout: LevelLayout, w: int) -> int:
    """The worker of ``to_layout`` (folded) whose part holds worker ``w``'s
    block of ``lay`` (partition.py:194-218: the group's lowest index)."""
    fx, fy = lay.px // to_layout.px, lay.py // to_layout.py
    ai, aj = lay.coords(w)
    return to_layout.worker_at(ai // fx, aj // fy)


def _p2p(dist, sends, recvs) -> None:
    """Post point-to-point transfers [(tensor, peer)] and wait: device
    tensors under NCCL; under a CPU backend (gloo) device tensors are
    staged through host memory."""
    if not sends and not recvs:
        return
    staged = dist.get_backend() != "nccl"
    if staged:
        torch.cuda.current_stream().synchronize()
        hs = [(t.cpu(), p) for t, p in sends]
        hr = [(torch.empty(t.shape, dtype=t.dtype), p) for t, p in recvs]
    else:
        hs, hr = sends, recvs
    ops = [dist.P2POp(dist.isend, t, p) for t, p in hs]
    ops += [dist.P2POp(dist.irecv, t, p) for t, p in hr]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if staged:
        for (t, _), (h, _) in zip(recvs, hr):
            t.copy_(h)


def _collect_dist(df: DistField, out: DistField, fx: int, fy: int, st, dist) -> None:
    """collect across ranks: a part whose group root is another rank sends
    its whole part buffer there; the root places every block of its group
    (received ones through a temporary part of the sender's geometry)."""
    lay, to = df.layout, out.layout
    sends, recvs, place = [], [], []
    for w, f in df.parts.items():
        root = fold_root(lay, to, w)
        if root != w:
            sends.append((f.data, root))
    for pw, big in out.parts.items():
        ai, aj = to.coords(pw)
        for di in range(fx):
            for dj in range(fy):
                cw = lay.worker_at(fx * ai + di, fy * aj + dj)
                if cw in df.parts:
                    src = df.parts[cw]
                else:
                    src = DevField(lay.geometry(cw, df.nz))
                    recvs.append((src.data, cw))
                place.append((src, big, di, dj))
    _p2p(dist, sends, recvs)
    for src, big, di, dj in place:
        call("pmg_copy_block", src.geom.h, src.ptr, big.geom.h, big.ptr, 0, 0,
             di * lay.mx, dj * lay.my, lay.mx, lay.my, st)


def distribute(df: DistField, to_layout: LevelLayout, out: DistField | None = None) -> DistField:
    """Inverse of ``collect`` (reference partition.py:221-240): every part
    of ``to_layout`` receives its owned block plus the surrounding one-cell
    ring from the folded part."""
    lay = df.layout
    fx, fy = to_layout.px // lay.px, to_layout.py // lay.py
    if (to_layout.nx != lay.nx or to_layout.ny != lay.ny or fx * lay.px != to_layout.px
            or fy * lay.py != to_layout.py or fx * fy < 2):
        raise ValueError("distribute target must unfold the active grid at the same level size")
    if out is None:
        out = DistField.zeros(to_layout, df.nz)
    st = _stream()
    m, n = to_layout.mx, to_layout.my
    d = _dist()
    if d is not None:
        # across ranks: the root cuts every child's block + ring into a
        # part of the child's geometry and sends the whole part buffer
        sends, recvs = [], []
        for pw, big in df.parts.items():
            pi, pj = lay.coords(pw)
            for di in range(fx):
                for dj in range(fy):
                    cw = to_layout.worker_at(fx * pi + di, fy * pj + dj)
                    ch = (out.parts[cw] if cw in out.parts
                          else DevField(to_layout.geometry(cw, df.nz)))
                    call("pmg_copy_block", big.geom.h, big.ptr, ch.geom.h, ch.ptr,
                         di * m - 1, dj * n - 1, -1, -1, m + 2, n + 2, st)
                    if cw not in out.parts:
                        sends.append((ch.data, cw))
        for cw, ch in out.parts.items():
            root = fold_root(to_layout, lay, cw)
            if root != cw:
                recvs.append((ch.data, root))
        _p2p(d, sends, recvs)
        lay.decomp.distribute_calls += 1
        return out
    for cw, ch in out.parts.items():
        ai, aj = to_layout.coords(cw)
        big = df.parts[lay.worker_at(ai // fx, aj // fy)]
        call("pmg_copy_block", big.geom.h, big.ptr, ch.geom.h, ch.ptr, (ai % fx) * m - 1,
             (aj % fy) * n - 1, -1, -1, m + 2, n + 2, st)
    lay.decomp.distribute_calls += 1
    return out


def scatter_owned(arr, layout: LevelLayout) -> DistField:
    """Split a global (nx, ny, nz) array (numpy, or torch on host/device)
    over the layout's local parts; halos start at zero."""
    if arr.shape[0] != layout.nx or arr.shape[1] != layout.ny:
        raise ValueError("array does not match the layout size")
    nz = int(arr.shape[2])
    df = DistField.zeros(layout, nz)
    for w, f in df.parts.items():
        i0, j0 = layout.origin(w)
        if layout.px == 1 and layout.py == 1:
            f.load_owned(arr)
        else:
            f.load_owned(arr[i0:i0 + layout.mx, j0:j0 + layout.my, :])
    return df


def scatter_block(block, layout: LevelLayout, out: DistField | None = None,
                  staging: torch.Tensor | None = None) -> DistField:
    """Field whose (single) local part is ``block`` (mx, my, nz): the
    multi-rank entry point, each rank passing only its own columns."""
    if len(layout.local_workers) != 1:
        raise ValueError("scatter_block needs exactly one local part")
    nz = int(block.shape[2])
    df = out if out is not None else DistField.zeros(layout, nz)
    (w, f), = df.parts.items()
    f.load_owned(block, staging)
    return df


def gather_owned(df: DistField) -> np.ndarray:
    """Assemble the global (nx, ny, nz) host array of owned values (on every
    rank when distributed)."""
    lay = df.layout
    out = np.empty((lay.nx, lay.ny, df.nz))
    d = _dist()
    if d is None:
        for w, f in df.parts.items():
            i0, j0 = lay.origin(w)
            out[i0:i0 + lay.mx, j0:j0 + lay.my, :] = f.owned_array()
        return out
    (w, f), = df.parts.items()
    mine = torch.from_numpy(f.owned_array())
    dev = "cuda" if d.get_backend() == "nccl" else "cpu"
    mine = mine.to(dev)
    allp = [torch.empty_like(mine) for _ in range(d.get_world_size())]
    d.all_gather(allp, mine)
    for wk, blk in enumerate(allp):
        i0, j0 = lay.origin(wk)
        out[i0:i0 + lay.mx, j0:j0 + lay.my, :] = blk.cpu().numpy()
    return out


# ---------------------------------------------------------------------------
# reductions (partition.py:267-286)
# ---------------------------------------------------------------------------
class _Scratch:
    t = None
    res = None

    @classmethod
    def get(cls):
        if cls.t is None:
            cls.t = torch.empty(int(lib().pmg_partials_size()), dtype=torch.float64, device="cuda")
            cls.res = torch.zeros(64, dtype=torch.float64, device="cuda")
        return cls.t, cls.res


def scalar_buffer(n: int) -> torch.Tensor:
    """Per-part reduction results.  Single process: pinned, device-mapped
    host memory (UVA) -- the finalize kernel stores the scalar straight into
    host memory, so reading it needs a stream sync but no copy-engine
    transfer (a tiny D2H copy would queue behind bulk downloads of a
    pipelined solve).  Distributed: device memory for the NCCL all-reduce."""
    if _dist() is None:
        return torch.zeros(n, dtype=torch.float64, pin_memory=True)
    return torch.zeros(n, dtype=torch.float64, device="cuda")


def _ordered_sum(xs) -> float:
    """Left-to-right sum from 0.0, the reference's worker loop
    (partition.py:278-280; Python >= 3.12's ``sum`` of floats is
    compensated, a different rounding)."""
    total = 0.0
    for x in xs:
        total += x
    return total


def reduce_parts(vals: torch.Tensor) -> float:
    """Sum per-part scalars in part order, then over ranks."""
    if not vals.is_cuda and _dist() is None:   # host-mapped results
        torch.cuda.current_stream().synchronize()
        return _ordered_sum(vals.tolist())
    tot = vals.sum() if vals.numel() > 1 else vals[0]
    d = _dist()
    if d is not None:
        # gather the per-rank sums and add them in rank (= worker) order on
        # every rank: the same left-to-right order as the in-process sum over
        # parts, independent of the backend's all-reduce algorithm
        t = tot.reshape(1).clone()
        if d.get_backend() != "nccl":
            t = t.cpu()
        allp = [torch.empty_like(t) for _ in range(d.get_world_size())]
        d.all_gather(allp, t)
        return _ordered_sum(torch.cat(allp).cpu().tolist())   # one device -> host copy
    return float(tot.item())


def dist_dot(a: DistField, b: DistField, deterministic: bool = False) -> float:
    """Owned-cell inner product over all parts (fixed per-part reduction
    order; part results summed in worker order, then across ranks)."""
    scratch, res = _Scratch.get()
    st = _stream()
    ws = list(a.parts.keys())
    out = scalar_buffer(len(ws))
    for n, w in enumerate(ws):
        fa, fb = a.parts[w], b.parts[w]
        call("pmg_dot", fa.geom.h, fa.ptr, fb.ptr, _ptr(scratch),
             C.c_void_p(out.data_ptr() + 8 * n), st)
    return reduce_parts(out)


def dist_norm(a: DistField, deterministic: bool = False) -> float:
    return math.sqrt(dist_dot(a, a, deterministic))
