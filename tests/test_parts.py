"""Host logic of the native multi-part driver (pmg_parts.cu), on CPU:

* ``pmg_exchange_plan8`` -- the ordered NCCL message plan each rank posts
  inside the one ncclGroupStart/End of a (single-phase) halo exchange: four
  face strips and four corner columns -- is consistent across ranks for
  every process grid the configs use (1x1, 2x1, 1x2, 2x2, 4x2, 4x4;
  periodic and mirror): for every ordered pair of ranks, the strips A sends
  to B, in order, are exactly the strips B expects from A, in order, side
  for opposite side (NCCL matches point-to-point messages between two ranks
  in posting order);
* ``pmg_exchange_plan`` -- one phase of the two-phase plan the Python
  multi-rank path posts -- has the same property and equals
  partition.exchange_plan;
* both plans executed by world-size-2 and -4 gloo process groups with a
  single tag (so messages match in posting order, as under NCCL) deliver
  every halo strip from the right neighbour side.
"""

import ctypes as C
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GRIDS = [(1, 1), (2, 1), (1, 2), (2, 2), (4, 2), (4, 4)]
OPP = {0: 1, 1: 0, 2: 3, 3: 2, 4: 7, 5: 6, 6: 5, 7: 4}
DIRS = ((-1, 0), (1, 0), (0, -1), (0, 1))
DIRS8 = DIRS + ((-1, -1), (1, -1), (-1, 1), (1, 1))     # W E S N SW SE NW NE


def _lib():
    from paper_1307_2036_b200 import _lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("libpmg.so not built")
    return L


def neighbours(px, py, periodic):
    from paper_1307_2036_b200.partition import Decomposition
    dec = Decomposition(8 * px, px * py, ny=8 * py, px=px, py=py, periodic=periodic)
    lay = dec.layout(8 * px)
    out = {}
    for w in lay.workers:
        nb = [lay.neighbor(w, *d) for d in DIRS]
        out[w] = [-1 if n is None else n for n in nb]
    return lay, out


def neighbours8(px, py, periodic):
    lay, _ = neighbours(px, py, periodic)
    out = {}
    for w in lay.workers:
        nb = [lay.neighbor(w, *d) for d in DIRS8]
        out[w] = [-1 if n is None else n for n in nb]
    return lay, out


def c_plan8(L, nbr8):
    ops = (C.c_int * 48)()
    n = C.c_int()
    L.call("pmg_exchange_plan8", (C.c_int * 8)(*nbr8), ops, C.byref(n))
    return [tuple(ops[3 * i:3 * i + 3]) for i in range(n.value)]


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("px,py", GRIDS)
def test_plan8_pairs_up_in_order(px, py, periodic):
    L = _lib()
    _, nbrs = neighbours8(px, py, periodic)
    plans = {w: c_plan8(L, nbrs[w]) for w in nbrs}
    for a in nbrs:
        for b in nbrs:
            sends = [d for kind, d, peer in plans[a] if kind == 0 and peer == b]
            recvs = [d for kind, d, peer in plans[b] if kind == 1 and peer == a]
            # the k-th strip A sends to B lands in B's k-th receive from A, in
            # the halo side opposite to the strip's side
            assert [OPP[d] for d in sends] == recvs, (a, b, sends, recvs)
    for w, pl in plans.items():
        # every side with a neighbour sends once and receives once
        want = sorted(d for d in range(8) if nbrs[w][d] >= 0)
        assert sorted(d for kind, d, _ in pl if kind == 1) == want
        assert sorted(d for kind, d, _ in pl if kind == 0) == want
        # a diagonal neighbour exists exactly where both faces have one
        for c, (a, b) in enumerate(((0, 2), (1, 2), (0, 3), (1, 3))):
            assert (nbrs[w][4 + c] >= 0) == (nbrs[w][a] >= 0 and nbrs[w][b] >= 0)


def c_plan(L, nbr, phase):
    ops = (C.c_int * 12)()
    n = C.c_int()
    L.call("pmg_exchange_plan", (C.c_int * 4)(*nbr), phase, ops, C.byref(n))
    return [tuple(ops[3 * i:3 * i + 3]) for i in range(n.value)]


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("px,py", GRIDS)
def test_plan_pairs_up_in_order(px, py, periodic):
    L = _lib()
    lay, nbrs = neighbours(px, py, periodic)
    from paper_1307_2036_b200.partition import exchange_plan
    for phase in (0, 1):
        plans = {w: c_plan(L, nbrs[w], phase) for w in nbrs}
        for a in nbrs:
            for b in nbrs:
                sends = [face for kind, face, peer in plans[a] if kind == 0 and peer == b]
                recvs = [face for kind, face, peer in plans[b] if kind == 1 and peer == a]
                # the k-th strip A sends to B lands in B's k-th receive from A,
                # in the halo face opposite to the strip's face
                assert [OPP[f] for f in sends] == recvs, (phase, a, b, sends, recvs)
        # every non-boundary halo face receives exactly once per phase
        for w, pl in plans.items():
            got = sorted(face for kind, face, _ in pl if kind == 1)
            want = sorted(f for f in (2 * phase, 2 * phase + 1) if nbrs[w][f] >= 0)
            assert got == want
            # the Python driver posts the same plan
            py_plan = []
            for sf, ps, rf, pr in exchange_plan(lay, w, (2 * phase, 2 * phase + 1)):
                if ps is not None:
                    py_plan.append((0, sf, ps))
                if pr is not None:
                    py_plan.append((1, rf, pr))
            assert py_plan == pl


def test_plan_rejects_bad_arguments():
    L = _lib()
    ops = (C.c_int * 12)()
    n = C.c_int()
    lib = L.load()
    assert lib.pmg_exchange_plan((C.c_int * 4)(0, 0, 0, 0), 2, ops, C.byref(n)) == L.PMG_ERR_VALUE
    assert lib.pmg_exchange_plan(None, 0, ops, C.byref(n)) == L.PMG_ERR_VALUE
    assert lib.pmg_exchange_plan8(None, ops, C.byref(n)) == L.PMG_ERR_VALUE


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
        dist.barrier()      # connect every pair before the point-to-point phase
        from paper_1307_2036_b200 import _lib as L
        _, nbrs = neighbours8(px, py, periodic)
        got = {}
        # the native driver's single-phase plan, then the Python path's two phases
        for phase in (8, 0, 1):
            plan = c_plan8(L, nbrs[rank]) if phase == 8 else c_plan(L, nbrs[rank][:4], phase)
            # strip content identifies (sender, face)
            bufs = {}
            ops = []
            selfq = []      # NCCL delivers messages to self in posting order
            for kind, face, peer in plan:
                if kind == 0:
                    t = torch.full((3,), 10.0 * rank + face)
                    if peer == rank:
                        selfq.append(t)
                    else:
                        ops.append(dist.P2POp(dist.isend, t, peer, tag=0))
                else:
                    t = torch.full((3,), -1.0)
                    bufs[face] = t
                    if peer == rank:
                        t.copy_(selfq.pop(0))
                    else:
                        ops.append(dist.P2POp(dist.irecv, t, peer, tag=0))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            for face, t in bufs.items():
                got[(phase == 8, face)] = float(t[0])
        q.put((rank, got, nbrs[rank]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as err:  # pragma: no cover
        q.put((rank, repr(err), None))


@pytest.mark.parametrize("px,py,periodic", [(2, 1, True), (2, 1, False), (2, 2, True),
                                            (1, 2, True)])
def test_plan_over_gloo_in_order(px, py, periodic):
    _lib()
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
        rank, got, nbr = q.get(timeout=180)
        assert nbr is not None, got
        res[rank] = (got, nbr)
    for p in procs:
        p.join(timeout=60)
    for rank, (got, nbr) in res.items():
        for (single, face), v in got.items():
            # halo side `face` holds the neighbour's strip from the opposite side
            assert v == 10.0 * nbr[face] + OPP[face], (rank, single, face, v)
        assert sorted(f for s1, f in got if not s1) == sorted(f for f in range(4) if nbr[f] >= 0)
        assert sorted(f for s1, f in got if s1) == sorted(f for f in range(8) if nbr[f] >= 0)
