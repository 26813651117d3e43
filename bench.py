"""Benchmark: BASELINE metric "MG solve time & DOF/s to 1e-5 residual;
achieved HBM GB/s vs peak, 1-8 GPU".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one complete MG solve (u = 0 -> ||r||/||r0|| < 1e-5, V(1,1),
7 levels) of a 1024 x 1024 x 128 fp64 subdomain per GPU: at N = 1 exactly
BASELINE configs[1]; at N > 1 the configs[3] weak-scaling decomposition
(px x py parts, periodic global grid) with configs[1]'s per-GPU size, so
the per-N values are comparable.  Inputs are synthetic: f ~ U[-1, 1] from
default_rng(0) in global (i, j, k) order, generated per rank.

value   = global DOF x K / (max over ranks of the device time of K solves)
e2e     = same metric through the public API with host buffers: pinned
          host f -> scatter_block (H2D + layout kernel) -> mg_solve ->
          owned_to (layout kernel + D2H of u), every step
roofline= the dominant kernel (fine-level line-smoother half-sweep):
          12 algorithmic bytes per fine cell / CUDA-event time
cpu_baseline = oracle/oracle.c (C restatement of the reference, OpenMP)
          running the full configs[1] solve on the host cores, rank 0, N = 1.

--impl reference: the reference algorithm's CPU implementation (the same
C restatement; the Python reference cannot travel) on this host's cores,
same config and metric; each step one V-cycle + convergence residual,
solve time = mean step time x the cycle count of a full reference solve.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NX_PER_GPU, NZ, LEVELS = 1024, 128, 7
PX = {1: 1, 2: 2, 4: 2, 8: 4}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh).get(kernel)
    return None


class ClockSampler:
    """NVML SM clock / throttle-reason sampling during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(n):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    # PMG_DIST_BACKEND=gloo PMG_DIST_DEVICE=0: every rank on one device with
    # host-staged halos -- a functional check of the multi-rank path on a
    # one-GPU box (no kernel waits on another rank); timings meaningless
    dev = int(os.environ.get("PMG_DIST_DEVICE", local))
    backend = os.environ.get("PMG_DIST_BACKEND", "nccl")
    if torch.cuda.is_available():
        torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    return world, rank, dev


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline_sample():
    """Full configs[1] MG solve with the C restatement on this host's cores."""
    from oracle import coracle, port
    cfg = port.CONFIGS[1]
    f = port.rhs(cfg.nx, cfg.ny, cfg.nz, 0)
    h = coracle.config_hierarchy(cfg)
    _, rep = h.mg_solve(f, want_u=False)
    dof = cfg.nx * cfg.ny * cfg.nz
    return {"value": dof / rep.wall_time, "unit": "DOF/s", "cores": coracle.threads(),
            "kind": "port",
            "sample": (f"full configs[1] MG solve ({rep.iterations} V-cycles to 1e-5, "
                       f"{rep.wall_time:.2f} s) by oracle/oracle.c (C restatement of the "
                       "reference, OpenMP, reference op order)"),
            "iterations": rep.iterations, "solve_s": rep.wall_time}


def run_reference(args):
    """--impl reference: rank 0 times the CPU implementation; others exit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import coracle, port
    cfg = port.CONFIGS[1]
    f = port.rhs(cfg.nx, cfg.ny, cfg.nz, 0)
    h = coracle.config_hierarchy(cfg)
    _, full = h.mg_solve(f, want_u=False)          # establishes the cycle count
    cycles = full.iterations
    for _ in range(args.warmup):
        h.mg_solve(f, want_u=False, max_cycles=1)
    times = []
    for _ in range(args.steps):
        _, rep = h.mg_solve(f, want_u=False, max_cycles=1)
        times.append(rep.wall_time)
    t_cycle = sum(times) / len(times)
    dof = cfg.nx * cfg.ny * cfg.nz
    value = dof / (t_cycle * cycles)
    out = {
        "metric": "MG solve DOF/s to 1e-5 residual (configs[1] per GPU)", "value": value,
        "unit": "DOF/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_cycle * cycles,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: f ~ U[-1,1], default_rng(0)",
        "config": {"workload": "configs[1] MG solve 1024x1024x128 fp64, 7 levels, V(1,1), "
                               "eps 1e-5", "levels": LEVELS},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": coracle.threads(),
                         "kind": "port",
                         "sample": (f"oracle/oracle.c, each step one V-cycle + residual at "
                                    f"full configs[1] size; solve = {cycles} cycles "
                                    f"(full reference solve {full.wall_time:.2f} s)")},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def time_kernel(fn, reps, torch):
    """Mean device time of one call of ``fn``: ``reps`` calls captured into a
    CUDA graph (no host launch gaps between them) and replayed between two
    CUDA events on the replaying stream."""
    fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=32)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world, rank, local = dist_setup(args.gpus)
    import paper_1307_2036_b200 as pmg
    from paper_1307_2036_b200 import _lib, configs
    from paper_1307_2036_b200.partition import scatter_block

    px = PX[world]
    py = world // px
    nxg, nyg = NX_PER_GPU * px, NX_PER_GPU * py
    prob = configs.Problem(nxg, nyg, NZ, 1e-3, 1.0, LEVELS)
    grid, params = prob.grid(), prob.params()
    cfg = prob.mg_config()
    dec = pmg.Decomposition(nxg, world, ny=nyg, px=px, py=py)
    hier = pmg.build_hierarchy(grid, params, cfg, dec)
    lay = hier.fine.layout
    (w,) = lay.local_workers
    i0, j0 = lay.origin(w)
    mx, my = lay.mx, lay.my
    block = configs.rhs_block(nxg, nyg, NZ, i0, j0, mx, my, 0)
    f = scatter_block(block, lay)
    dof_local = mx * my * NZ
    dof = nxg * nyg * NZ
    lib = _lib.load()

    # ---- device-resident solves --------------------------------------------
    reps = []
    u = pmg.DistField.zeros(lay, NZ)        # iterate buffer reused by every solve
    for _ in range(max(1, args.warmup)):    # (graphs are captured for (f, u) here)
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
        reps.append(rep)
    torch.cuda.synchronize()
    barrier(world)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.pmg_launch_count()
    from paper_1307_2036_b200 import multigrid as mgm
    native = lay.px == 1 and lay.py == 1 and mgm.USE_NATIVE
    r0_graph = hier.native(cfg).replayed_launches() if native else 0
    sampler = ClockSampler(local)
    iters = []
    with sampler:
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            u, rep = pmg.mg_solve(f, hier, cfg, out=u)
            iters.append(rep.iterations)
        e1.record(st)
        torch.cuda.synchronize()
    barrier(world)
    t_local = e0.elapsed_time(e1) * 1e-3
    t = max_over_ranks(t_local, world)
    launches_lib = lib.pmg_launch_count() - l0
    # kernels replayed from the captured V-cycle graphs (first cycle + the rest)
    gpu_launches = launches_lib
    if native:
        # single part: the C++ driver counts the kernels of its graph replays
        gpu_launches += hier.native(cfg).replayed_launches() - r0_graph
    else:
        gkey = mgm.graph_key(cfg, f, u)
        g_first = hier._graphs.get(gkey + (True,))
        g_rest = hier._graphs.get(gkey + (False,))
        for n_it in iters:
            if g_first is not None:
                gpu_launches += g_first.launches + (n_it - 1) * g_rest.launches
            elif g_rest is not None:
                gpu_launches += n_it * g_rest.launches
    value = dof * args.steps / t

    # ---- dominant kernel: fine-level half-sweep (12 B per fine cell) ---------
    fine = hier.fine
    scratch = hier.persistent_scratch()
    s0 = scratch[0]
    n_fine = dof_local
    flip = [0]

    def hs():
        fine.smoother.half_sweep(s0.u, s0.f, flip[0] & 1, 1.0)
        flip[0] += 1

    t_hs = time_kernel(hs, 20, torch)
    kern = {}
    coarse = hier.levels[1]
    from paper_1307_2036_b200 import multigrid as mgmod
    import ctypes as C
    # the fine-level kernels of the solve: fused-residual red sweep, red-only
    # residual restriction, black-only prolongation (DESIGN.md sections 3-4)
    part = s0.u.parts[w]
    hh = fine.op.handles[w].h
    scr = torch.empty(int(lib.pmg_partials_size()), dtype=torch.float64, device="cuda")
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    t_res = time_kernel(lambda: lib.pmg_half_sweep_res(
        hh, part.ptr, s0.r.parts[w].ptr, s0.f.parts[w].ptr, C.c_void_p(scr.data_ptr()),
        C.c_void_p(res.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)),
        10, torch)
    t_rr = time_kernel(lambda: mgmod._residual_restrict(fine, coarse, s0.f, s0.u,
                                                        scratch[1].f, True), 10, torch)
    t_pa = time_kernel(lambda: mgmod._prolong_add(scratch[1].u, coarse, fine, s0.u,
                                                  black_only=True), 10, torch)
    for name, tt, b in (("half_sweep", t_hs, 12), ("half_sweep_res", t_res, 16),
                        ("residual_restrict_red", t_rr, 14), ("prolong_black", t_pa, 10)):
        kern[name] = {"ms": tt * 1e3, "alg_bytes_per_cell": b,
                      "GB_s": b * n_fine / tt / 1e9}
    peak, peak_src = measured_peak()
    ach = 12 * n_fine / t_hs / 1e9
    traffic = ncu_traffic("k_half_sweep_band")
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": traffic,
                "kernel": "k_half_sweep_band (fine level, TMA-fed line relaxation)",
                "alg_bytes_per_launch": 12 * n_fine, "launch_ms": t_hs * 1e3,
                "peak_source": peak_src}

    # ---- end to end through the public API with host buffers -----------------
    # pinned host f in, pinned host u out, every step; SolvePipeline overlaps
    # step i+1's upload and step i-1's download with step i's solve
    from paper_1307_2036_b200.pipeline import SolvePipeline
    ne = max(2, args.e2e_steps)
    f_host = torch.from_numpy(block).pin_memory()
    # two pinned result buffers, reused every other step (a D2H into a buffer
    # is stream-ordered after the previous one out of it)
    u_bufs = [torch.empty(dof_local, dtype=torch.float64).pin_memory() for _ in range(2)]
    u_hosts = [u_bufs[i % 2] for i in range(ne)]
    pipe = SolvePipeline(hier, cfg, NZ)
    pipe.run([f_host] * 2, u_hosts[:2])                 # warm-up (graph capture)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps_e = pipe.run([f_host] * ne, u_hosts)
    torch.cuda.synchronize()
    te = max_over_ranks(time.perf_counter() - t0, world)
    ok = all(r.iterations == iters[-1] for r in reps_e)
    e2e = {"value": dof * ne / te, "unit": "DOF/s", "h2d_bytes_per_step": 8 * dof_local,
           "d2h_bytes_per_step": 8 * dof_local + 8 * (reps_e[-1].iterations + 1),
           "ms_per_step": te / ne * 1e3, "steps": ne, "same_iterations": ok,
           "path": "SolvePipeline.run: pinned host f -> H2D + layout kernel -> mg_solve -> "
                   "layout kernel + D2H -> pinned host u, every step; transfers of "
                   "neighbouring steps overlap the solve (double buffered)"}

    if rank != 0:
        return
    out = {
        "metric": "MG solve DOF/s to 1e-5 residual (configs[1] per GPU)",
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: f ~ U[-1,1] from default_rng(0), global (i,j,k) order",
        "config": {"workload": "configs[1] MG solve 1024x1024x128 fp64 per GPU, 7 levels, "
                               "V(1,1), rho 1, coarse_sweeps 1, eps 1e-5",
                   "global_grid": [nxg, nyg, NZ], "levels": LEVELS,
                   "parallelism": f"{px}x{py} horizontal domain decomposition",
                   "iterations": iters[-1], "l2": "inputs larger than L2 (1.09 GB/field)"},
        "solve_ms": t / args.steps * 1e3,
        "v_cycle_ms": t / sum(iters) * 1e3,
        "residual_history": reps[-1].residual_history if reps else None,
        "roofline": roofline, "kernels": kern, "e2e": e2e,
        "gpu_launches": int(gpu_launches),
        "clocks": sampler.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample()
        except Exception as err:  # the oracle library may be missing
            out["cpu_baseline"] = {"value": None, "unit": "DOF/s", "cores": 0, "kind": "port",
                                   "sample": f"unavailable: {err}"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
