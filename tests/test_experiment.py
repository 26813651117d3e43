"""Experiment harness (reference bench.py / tests/test_bench_cli.py) against
golden rows generated from the reference itself
(tests/golden/make_harness_golden.py)."""

import csv
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "harness.json")
SKIP = ("wall_time_s", "time_per_iter_s")


@pytest.fixture(scope="module")
def gold():
    return json.load(open(GOLD))


def strip(row):
    return {k: str(v) for k, v in row.items() if k not in SKIP}


def read_rows(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(fh))


# ---------------------------------------------------------------- host only


def test_param_space_table_equals_reference(gold, tmp_path):
    from paper_1307_2036_b200 import run_table
    from paper_1307_2036_b200.experiment import PARAM_SPACE_COLUMNS
    out = tmp_path / "p.csv"
    rows = run_table("param_space", str(out), nx=256, nx_max=16384, nz=128, dt=600.0)
    assert [list(r) for r in rows] == [PARAM_SPACE_COLUMNS] * len(rows)
    assert [strip(r) for r in rows] == gold["param_space"]
    assert [r["nx"] for r in read_rows(out)] == [r["nx"] for r in gold["param_space"]]


def test_spec_validation_and_memory_cap():
    from paper_1307_2036_b200 import ExperimentSpec, MemoryCapError, SpecError, run_experiment
    from paper_1307_2036_b200.experiment import estimate_memory_bytes, run_table
    for bad in (dict(solver="gmres"), dict(policy="explicit"), dict(rhs="file"),
                dict(eps=1.5), dict(rho=2.0), dict(nu_pre=0, nu_post=0), dict(maxiter=0)):
        with pytest.raises(SpecError):
            ExperimentSpec(**bad).validate()
    with pytest.raises(SpecError):                 # not 4^p workers (reference rule)
        run_experiment(ExperimentSpec(nx=16, nz=4, workers=8))
    with pytest.raises(SpecError):                 # nx not a power of two
        run_experiment(ExperimentSpec(nx=100, nz=4))
    spec = ExperimentSpec(nx=256, nz=128, memory_cap_bytes=10 ** 6)
    assert estimate_memory_bytes(spec) > 10 ** 6
    with pytest.raises(MemoryCapError):
        run_experiment(spec)
    with pytest.raises(MemoryCapError):            # checked before any solve
        run_table("weak_scaling", None, nx=16, nx_max=1024, nz=128, dt=600.0,
                  memory_cap_bytes=10 ** 6)
    with pytest.raises(SpecError):
        run_table("nosuch")


def test_csv_header_guard(tmp_path):
    from paper_1307_2036_b200 import SpecError
    from paper_1307_2036_b200.experiment import EXPERIMENT_COLUMNS, append_rows
    out = tmp_path / "o.csv"
    row = {c: "1" for c in EXPERIMENT_COLUMNS}
    append_rows(str(out), [row], EXPERIMENT_COLUMNS)
    append_rows(str(out), [row], EXPERIMENT_COLUMNS)
    assert len(read_rows(out)) == 2 and open(out).read().count("nx,nz,dof") == 1
    bad = tmp_path / "bad.csv"
    bad.write_text("alpha,beta\n1,2\n")
    with pytest.raises(SpecError):
        append_rows(str(bad), [row], EXPERIMENT_COLUMNS)


def test_decompose_rule():
    from paper_1307_2036_b200 import Decomposition, decompose
    assert decompose(16, 4).px == 2 and decompose(16, 16).px == 4
    for w in (2, 8, 3):
        with pytest.raises(ValueError):
            decompose(16, w)
    assert (Decomposition(16, 8).px, Decomposition(16, 8).py) == (4, 2)   # configs[3] grids


# ---------------------------------------------------------------- device


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mg16", "cg16", "mg32_shallow_w4", "mg16_seed7_det",
                                  "mg32_manufactured", "mg16_flat"])
def test_run_experiment_rows_equal_reference(gold, tmp_path, name):
    from paper_1307_2036_b200 import ExperimentSpec, run_experiment
    from paper_1307_2036_b200.experiment import EXPERIMENT_COLUMNS
    g = gold["runs"][name]
    out = tmp_path / "rows.csv"
    report, row = run_experiment(ExperimentSpec(**g["spec"], output=str(out)))
    assert list(row) == EXPERIMENT_COLUMNS
    mine, ref = strip(row), g["row"]
    # the residual is printed to 7 significant digits: equal unless the
    # last digit sits on a rounding boundary
    assert float(mine.pop("final_rel_residual")) == pytest.approx(
        float(ref.pop("final_rel_residual")), rel=1e-5)
    assert mine == ref
    assert read_rows(out)[0]["iterations"] == ref["iterations"]


@pytest.mark.gpu
def test_tables_equal_reference(gold, tmp_path):
    from paper_1307_2036_b200 import run_table
    for which, kw in (("weak_scaling", dict(nx=8, nx_max=16)), ("levels", dict(nx=8)),
                      ("robustness", dict(nx=8))):
        rows = run_table(which, str(tmp_path / f"{which}.csv"), nz=4, dt=600.0, **kw)
        assert len(rows) == len(gold[which])
        for mine, ref in zip(rows, gold[which]):
            mine, ref = strip(mine), dict(ref)
            assert float(mine.pop("final_rel_residual")) == pytest.approx(
                float(ref.pop("final_rel_residual")), rel=1e-5)
            assert mine == ref, which


@pytest.mark.gpu
def test_manufactured_solution_is_discrete_exact():
    """tests/test_bench_cli.py:23-47 on the device (standard policy: down to
    one column; with 4 parts the coarse levels fold onto one worker)."""
    import paper_1307_2036_b200 as pmg
    params = pmg.derive_parameters(64, 16, 2400.0)
    grid = pmg.panel_grid(64, 16)
    f, uex = pmg.manufactured_rhs(grid, params)
    for workers in (1, 4):
        cfg = pmg.MGConfig(eps=1e-10, maxiter=50, deterministic=workers > 1)
        hier = pmg.build_hierarchy(grid, params, cfg, pmg.Decomposition(64, workers))
        u, rep = pmg.mg_solve(pmg.scatter_owned(f.owned, hier.fine.layout), hier, cfg)
        assert rep.converged
        err = np.linalg.norm(pmg.gather_owned(u) - uex.owned)
        assert err / np.linalg.norm(uex.owned) <= 1e-8


@pytest.mark.gpu
def test_rhs_file_round_trip(tmp_path):
    import paper_1307_2036_b200 as pmg
    f = pmg.Field.from_owned(np.random.default_rng(0).uniform(-1, 1, (16, 16, 4)))
    path = tmp_path / "rhs.anmg"
    f.dump(path)
    rep, row = pmg.run_experiment(pmg.ExperimentSpec(nx=16, nz=4, rhs="file",
                                                     rhs_file=str(path)))
    assert rep.converged and row["seed"] == ""
    with pytest.raises(pmg.SpecError):
        pmg.run_experiment(pmg.ExperimentSpec(nx=32, nz=4, rhs="file", rhs_file=str(path)))
