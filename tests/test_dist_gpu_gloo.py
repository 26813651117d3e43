"""The multi-rank solve path on the device: 2 or 4 ranks (processes) on one
GPU with the gloo backend and host-staged halo strips.  No kernel waits on
another rank (the exchange is host-side), so this is a functional check of
the rank code path -- one part per rank, P2P face exchange, cross-rank
reductions -- against the same decomposition run in-process, bit for bit.
(The NCCL path differs only in moving device buffers.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(pmg, policy):
    if policy == "explicit":
        return pmg.MGConfig(policy="explicit", explicit_levels=3, eps=1e-8)
    if policy == "standard":      # down to one global column: folds at nx = 1
        return pmg.MGConfig(policy="standard", eps=1e-8)
    return pmg.MGConfig(policy="standard", l_split=3, eps=1e-8)   # folds from l_split on


def _worker(rank, world, port, px, q, policy="explicit"):
    trace = os.environ.get("PMG_TEST_TRACE")
    if trace:                       # debugging aid: dump stacks if stuck
        import faulthandler
        faulthandler.dump_traceback_later(90, exit=True,
                                          file=open(f"{trace}.{rank}", "w"))
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1307_2036_b200 as pmg
        nx, nz = 32, 16
        py = world // px
        grid = pmg.periodic_box(nx, nz, 0.01)
        params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
        dec = pmg.Decomposition(nx, world, px=px, py=py, periodic=True)
        cfg = _cfg(pmg, policy)
        hier = pmg.build_hierarchy(grid, params, cfg, dec)
        lay = hier.fine.layout
        i0, j0 = lay.origin(rank)
        fg = np.random.default_rng(3).uniform(-1, 1, (nx, nx, nz))
        f = pmg.partition.scatter_block(fg[i0:i0 + lay.mx, j0:j0 + lay.my], lay)
        u, rep = pmg.mg_solve(f, hier, cfg)
        ug = pmg.gather_owned(u)
        op = hier.fine.op
        uc, rc = pmg.pcg_solve(f, op, pmg.SSORPreconditioner(pmg.LineSmoother(op)), eps=1e-8,
                               maxiter=200)
        ucg = pmg.gather_owned(uc)          # collective: every rank calls it
        q.put((rank, rep.residual_history, ug if rank == 0 else None, rc.residual_history,
               ucg if rank == 0 else None, dec.collect_calls, dec.distribute_calls))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as err:  # surfaced by the parent
        import traceback
        q.put((rank, repr(err) + traceback.format_exc(), None, None, None, 0, 0))


@pytest.mark.parametrize("world,px,policy", [(2, 2, "explicit"), (4, 2, "explicit"),
                                             (4, 2, "standard"), (4, 2, "lsplit")])
def test_rank_path_matches_in_process(world, px, policy):
    """Rank path == in-process decomposition, bit for bit, also with
    coarse-level folding across ranks (standard policy down to one global
    column, and l_split): collect / distribute move whole part buffers
    between a group's ranks and its root."""
    import torch.multiprocessing as mp
    import paper_1307_2036_b200 as pmg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, px, q, policy))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        assert isinstance(r[1], list), r[1]
    # the same decomposition in one process
    nx, nz = 32, 16
    grid = pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    dec = pmg.Decomposition(nx, world, px=px, py=world // px, periodic=True)
    cfg = _cfg(pmg, policy)
    hier = pmg.build_hierarchy(grid, params, cfg, dec)
    fg = np.random.default_rng(3).uniform(-1, 1, (nx, nx, nz))
    f = pmg.scatter_owned(fg, hier.fine.layout)
    u, rep = pmg.mg_solve(f, hier, cfg)
    op = hier.fine.op
    uc, rc = pmg.pcg_solve(f, op, pmg.SSORPreconditioner(pmg.LineSmoother(op)), eps=1e-8,
                           maxiter=200)
    for r in res.values():
        assert r[1] == rep.residual_history
        assert r[3] == rc.residual_history
    assert np.array_equal(res[0][2], pmg.gather_owned(u))
    assert np.array_equal(res[0][4], pmg.gather_owned(uc))
    if policy != "explicit":      # one fold per V-cycle, on every rank
        cycles = len(rep.residual_history) - 1
        for r in res.values():
            assert (r[5], r[6]) == (cycles, cycles)
