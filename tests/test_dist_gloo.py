"""Multi-rank host logic on CPU (gloo): the halo message plan, face matching
(incl. two faces to the same peer along a periodic axis of 2 ranks and
self-neighbours), mirror boundaries and the cross-rank reductions -- the
exact code path NCCL runs on a multi-GPU box, with CPU tensors standing in
for the packed device face strips."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, px, py, periodic, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1307_2036_b200.partition import (Decomposition, exchange_messages,
                                                    exchange_plan, reduce_parts)
        nx, ny = 8 * px, 4 * py
        dec = Decomposition(nx, world, ny=ny, px=px, py=py, periodic=periodic)
        lay = dec.layout(nx)
        assert lay.local_workers == [rank]
        out = {}
        for faces in ((0, 1), (2, 3)):
            plan = exchange_plan(lay, rank, faces)
            send = {f: torch.full((5,), 100.0 * rank + f) for f in faces}
            recv = {f: torch.full((5,), -1.0) for f in faces}
            how = exchange_messages(dist, rank, plan, send, recv)
            for f in faces:
                out[f] = (how[f], float(recv[f][0]))
        tot = reduce_parts(torch.tensor([rank + 1.0]))
        q.put((rank, out, tot))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as err:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(err), None))


def _run(px, py, periodic):
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, px, py, periodic, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, tot = q.get(timeout=120)
        res[rank] = (out, tot)
    for p in procs:
        p.join(timeout=60)
    for rank, (out, tot) in res.items():
        assert isinstance(out, dict), out
    return res


DIRS = {0: (-1, 0), 1: (1, 0), 2: (0, -1), 3: (0, 1)}
OPP = {0: 1, 1: 0, 2: 3, 3: 2}


def _expect(rank, face, px, py, periodic):
    """Halo strip on side `face` must hold the neighbour's opposite face."""
    ai, aj = divmod(rank, py)
    di, dj = DIRS[face]
    ni, nj = ai + di, aj + dj
    if periodic:
        ni, nj = ni % px, nj % py
    elif not (0 <= ni < px and 0 <= nj < py):
        return "mirror", None
    nb = ni * py + nj
    kind = "self" if nb == rank else "buf"
    return kind, 100.0 * nb + OPP[face]


@pytest.mark.parametrize("px,py,periodic", [(2, 1, True), (2, 1, False), (2, 2, True),
                                            (2, 2, False)])
def test_halo_plan_and_reductions(px, py, periodic):
    res = _run(px, py, periodic)
    world = px * py
    for rank, (out, tot) in res.items():
        assert tot == pytest.approx(world * (world + 1) / 2)
        for face in range(4):
            kind, val = _expect(rank, face, px, py, periodic)
            got_kind, got_val = out[face]
            assert got_kind == kind, (rank, face, out)
            if val is not None:
                assert got_val == val, (rank, face, out)


def test_worker_split():
    from paper_1307_2036_b200.partition import Decomposition
    assert (Decomposition(64, 2).px, Decomposition(64, 2).py) == (2, 1)
    assert (Decomposition(64, 8).px, Decomposition(64, 8).py) == (4, 2)
    assert (Decomposition(64, 16).px, Decomposition(64, 16).py) == (4, 4)
    with pytest.raises(ValueError):
        Decomposition(64, 3)
    with pytest.raises(ValueError):
        Decomposition(6, 16)


@pytest.mark.parametrize("px,py,apx,apy", [(2, 2, 1, 1), (4, 2, 2, 1), (4, 4, 2, 2)])
def test_fold_roots(px, py, apx, apy):
    """Cross-rank folding plan (partition.collect / distribute under a
    process group): every worker of the unfolded layout maps to the
    lowest-indexed worker of its (px/apx) x (py/apy) group, which is active
    on the folded layout and maps to itself."""
    from paper_1307_2036_b200.partition import Decomposition, fold_root
    dec = Decomposition(64, px * py, px=px, py=py, periodic=True)
    lay, fol = dec.layout(64), dec.layout(64, active=(apx, apy))
    gx, gy = px // apx, py // apy
    roots = {}
    for w in lay.workers:
        wi, wj = divmod(w, py)
        want = (wi // gx * gx) * py + (wj // gy * gy)
        r = fold_root(lay, fol, w)
        assert r == want and r in fol.workers
        roots.setdefault(r, []).append(w)
    assert sorted(roots) == sorted(fol.workers)
    assert all(len(v) == gx * gy for v in roots.values())
    assert all(fold_root(lay, fol, r) == r for r in fol.workers)
