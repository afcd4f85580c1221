"""Edge cases of the grid and the step range, GPU vs the CPU oracle on the
same plan: tiny domains (Nx = 2, 3, 5, ... where every cell is an edge or a
boundary cell and the tile depth exceeds the domain), a single time step,
records on the first and last cell, sources on the boundary cells, a run
shorter than one fused launch and one not a multiple of k.

Two-level cases with quantum groups of more than 32 cells must be
bit-identical in the exact variant (the oracle equals the reference bit for
bit there, tests/test_oracle_golden.py) and within 1e-9 in the fast one;
N >= 3, RK4 and tiny groups within 1e-9 in both.
"""

import math
import sys

import numpy as np
import pytest
from conftest import ROOT

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb

sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _rel(a, b):
    scale = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / scale if scale else np.max(np.abs(a))


def _build(nx, levels, steps, stepper="splitting", hard_right=False, whole=True):
    mb.clear_material_library()
    if levels == 2:
        qm = mb.two_level_description(1e24, 2 * math.pi * 2e14, 6.24e-11, 1e11, 1e12, -1.0)
        rho0 = mb.QmOperator([0.9, 0.1], [0.1 + 0.05j])
    else:
        rng = np.random.default_rng(7 + levels)
        from cases import random_medium

        qm = random_medium(mb, rng, levels)
        d = np.zeros(levels)
        d[0] = 1.0
        rho0 = mb.QmOperator(d)
    mb.add_material(mb.Material("Vacuum"))
    mb.add_material(mb.Material("Act", rel_permittivity=1.5, losses=300.0, qm=qm))
    length = 4e-6
    dev = mb.Device("edge", bc_left=mb.BoundaryReflectivity(0.3), bc_right=mb.BoundaryReflectivity(0.8))
    if nx >= 5:
        dev.add_region(mb.Region("v", "Vacuum", 0.0, length / 4))
        dev.add_region(mb.Region("a", "Act", length / 4, length))
    else:
        dev.add_region(mb.Region("a", "Act", 0.0, length))
    dx = length / (nx - 1)
    c_max = mb.C0 if nx >= 5 else mb.C0 / math.sqrt(1.5)  # fastest medium present
    dt0 = 0.5 * dx / c_max
    sce = mb.Scenario("s", nx, steps * dt0 * (1 - 1e-12), rho0, ic_e_field=mb.RandomField(1e6, seed=3),
                      ic_h_field=mb.RandomField(1e3, seed=4))
    sce.add_source(mb.SechPulse("l", 0.0, "soft", 1e9, 2e14, 3.0, 1e15))
    sce.add_source(mb.GaussianPulse("r", length, "hard" if hard_right else "soft", 5e8, 1.8e14, 2e-15, 1e-15))
    for name, pos in (("first", 0.0), ("last", length)):
        sce.add_record(mb.Record(f"e_{name}", quantity="e", position=pos))
        sce.add_record(mb.Record(f"h_{name}", quantity="h", position=pos))
        sce.add_record(mb.Record(f"d1n_{name}", quantity="d", i=1, j=levels, position=pos))
        sce.add_record(mb.Record(f"dnn_{name}", quantity="d", i=levels, j=levels, position=pos))
    if whole:
        sce.add_record(mb.Record("e", quantity="e"))
        sce.add_record(mb.Record("d12", quantity="d", i=1, j=2))
    return dev, sce, stepper


CASES = [
    # (nx, levels, steps, stepper, tile_steps)
    (2, 2, 1, "splitting", None), (2, 2, 37, "splitting", None), (3, 2, 200, "splitting", None),
    (5, 2, 130, "splitting", 64), (33, 2, 300, "splitting", 7), (257, 2, 1000, "splitting", None),
    (2049, 2, 129, "splitting", None), (2, 3, 20, "splitting", None), (3, 3, 50, "splitting", 16),
    (5, 6, 30, "splitting", 4), (130, 3, 97, "splitting", None), (129, 6, 41, "splitting", None),
    (3, 2, 40, "rk4", None), (7, 4, 25, "rk4", 3), (97, 3, 60, "rk4", None),
]


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("nx,levels,steps,stepper,k", CASES)
def test_tiny_domains_and_short_runs_match_the_oracle(nx, levels, steps, stepper, k, exact):
    dev, sce, stepper = _build(nx, levels, steps, stepper, hard_right=(nx % 2 == 1))
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, tile_steps=k, exact=exact)
    assert solver.grid.num_t - 1 == steps and solver.grid.num_x == nx
    ref, bad = orc.run_oracle(solver.plan)
    if bad:
        # RK4 at this Courant step is unstable (|omega dt| ~ 5): the GPU must
        # fail at the same scan step as the reference does
        with pytest.raises(mb.SolverError, match=f"at step {bad}$"):
            solver.run()
        return
    got = solver.run()
    # groups of <= 32 cells follow the reference's ScalarKernel (numpy) in the oracle
    big = all(hi - lo > 32 for lo, hi, _ in solver.plan.groups)
    bitwise = exact and levels == 2 and stepper == "splitting" and big
    for r, want in zip(got, ref):
        assert r.data.shape == want.shape, r.name
        if bitwise:
            assert np.array_equal(r.data.view(np.float64), want.view(np.float64)), (r.name, _rel(r.data, want))
        else:
            assert _rel(r.data, want) <= TOL, (r.name, _rel(r.data, want))


@pytest.mark.parametrize("levels", [2, 3])
def test_advance_in_uneven_pieces_equals_one_run(levels):
    """mbg_advance called with step counts that straddle fused launches and
    persistent chunks (1, k-1, k+1, a prime, the rest) gives the same bits as
    one call."""
    import ctypes as C

    dev, sce, stepper = _build(3000, levels, 700)
    whole = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    dev, sce, stepper = _build(3000, levels, 700)
    sol = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    h = sol.open_handle()
    sol.upload_initial_state(h)
    k = C.c_int32(0)
    h.call("mbg_tile_steps", C.byref(k))
    h.call("mbg_sample", 0)
    n = 1
    for cnt in (1, k.value - 1, k.value + 1, 101, 700):
        cnt = min(cnt, 701 - n)
        if cnt <= 0:
            break
        h.call("mbg_advance", n, cnt)
        n += cnt
    assert n == 701
    got = sol.download_results(h)
    h.close()
    for a, b in zip(whole, got):
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name
