"""Pin the CPU oracle to the reference: oracle records vs the golden records
the reference solver itself produced (tests/golden/make_golden.py).

Two-level (Bloch), RK4-free classical and FDTD paths are bit-exact; the
N >= 3 splitting loop of the reference is compiled with fastmath
(_kernels.py:55), so those cases are pinned at 1e-11 relative; groups of
<= 32 cells use the reference's numpy ScalarKernel (_kernels.py:404-425),
pinned at 1e-11.  The longest cases run only with MBG_SLOW=1.
"""

import os

import numpy as np
import pytest
from cases import CASES, SLOW
from conftest import build_case, load_golden, rel_err

import oracle as orc
import paper_2005_05412_b200 as gpu
from paper_2005_05412_b200.reference import mblight as mb

BITWISE = {"cfg1_full", "cfg2_r16", "cfg2_full", "cfg2_stress_full", "sit_hard_whole", "multi_material", "bragg_stack",
           "vacuum_sources", "rand2_split", "kernel2_split", "rand2_rk4", "kernel2_rk4"}
LONG = {"cfg3_r16", "cfg3_r16_stress", "cfg4_r14", "cfg2_full", "cfg2_stress_full", "ladder6"}
NAMES = sorted(n for n in CASES if n not in LONG or os.environ.get("MBG_SLOW"))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_golden(name):
    meta, recs = load_golden(name)
    dev, sce, stepper = build_case(name)
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    assert [plan.grid.num_x, plan.grid.dx, plan.grid.num_t, plan.grid.dt] == meta["grid"]
    got, bad = orc.run_oracle(plan)
    assert bad == 0
    for g, (rname, ref, _) in zip(got, recs):
        assert g.shape == ref.shape, rname
        if name in BITWISE:
            assert np.array_equal(g, ref), f"{rname}: {rel_err(g, ref):.3e}"
        else:
            assert rel_err(g, ref) <= 1e-11, f"{rname}: {rel_err(g, ref):.3e}"


def test_long_cases_are_listed():
    assert LONG <= set(CASES) and SLOW <= set(CASES)


def test_oracle_is_thread_count_independent():
    dev, sce, stepper = build_case("rand3_split")
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    a, _ = orc.run_oracle(plan, threads=1)
    b, _ = orc.run_oracle(plan, threads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_oracle_reports_the_first_failing_scan():
    """solver_fdtd.py:386-388: the non-finite scan runs every 1024 steps and on
    the last step (blow-up recipe of pkg/tests/test_solver.py:409-429)."""
    desc = mb.QmDescription(1e28, mb.QmOperator([0.0, 1e-19]), mb.QmOperator([0.0, 0.0], [1e-27]),
                            mb.LindbladRelaxation([[0.0, 1e21], [1e21, 0.0]], [0.0]))
    mb.add_material(mb.Material("stiff", qm=desc))
    dev = mb.Device("blow")
    dev.add_region(mb.Region("a", "stiff", 0.0, 10e-6))
    sce = mb.Scenario("s", 64, 2e-13, mb.QmOperator([1.0, 0.0]))
    sce.add_source(mb.SechPulse("s", 5e-6, "hard", 1e10, 2e14, 10.0, 2e14))
    plan = gpu.GpuFdtdSolver(dev, sce, stepper="rk4").plan
    _, bad = orc.run_oracle(plan)
    assert bad > 0 and (bad % 1024 == 0 or bad == plan.grid.num_t - 1)
