"""Host-side setup (plan.py / setup_model.py / qm.py) against the reference's
known answers: grid sizing (pkg/tests/test_solver.py:63-75), coefficients
(:119-141), relaxation propagator closed form (pkg/tests/test_quantum.py:349-359),
splitmix64 (core.py:377-388), and the region table vs per-cell maps."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest
from conftest import build_case

import paper_2005_05412_b200 as mb
from paper_2005_05412_b200 import plan as P


def _vacuum(length=150e-6):
    mb.add_material(mb.Material("Vacuum"))
    dev = mb.Device("v")
    dev.add_region(mb.Region("v", "Vacuum", 0.0, length))
    return dev


def test_sit_grid_numbers():
    dev = _vacuum()
    sce = mb.Scenario("s", 32768, 200e-15, mb.QmOperator([1.0, 0.0]))
    g = mb.init_fdtd_simulation(dev, sce)
    dx = 150e-6 / 32767
    dt0 = 0.5 * dx / mb.C0
    nt = math.ceil(200e-15 / dt0) + 1
    assert g.dx == dx and g.num_t == nt and g.dt == 200e-15 / (nt - 1)
    assert abs(dx - 4.5778e-9) < 1e-13 and abs(g.dt - 7.6348e-18) < 1e-21


def test_single_point_grid():
    mb.add_material(mb.Material("AR"))
    dev = mb.Device("p")
    dev.add_region(mb.Region("p", "AR", 0.0, 0.0))
    g = mb.init_fdtd_simulation(dev, mb.Scenario("s", 1, 80e-15, mb.QmOperator([1.0]), num_timesteps=10000))
    assert g.num_t == 10000 and g.dt == 80e-15 / 9999


def test_coefficients():
    cf = mb.get_fdtd_constants(mb.Material("Vacuum"), 1e-17, 1e-9)
    assert cf.a_prime == 1.0
    assert cf.b_prime == pytest.approx(1e-17 / mb.EPS0)
    assert cf.c_prime == pytest.approx(1e-17 / (1e-9 * mb.MU0))
    m = mb.Material("AR", rel_permittivity=12.96, overlap_factor=0.9, losses=1100.0)
    cf = mb.get_fdtd_constants(m, 1e-16, 1e-8)
    loss = 1e-16 * m.conductivity / (2 * m.permittivity)
    assert cf.a_prime == pytest.approx((1 - loss) / (1 + loss)) and cf.gamma == 0.9


def test_relaxation_half_step_closed_form():
    relax = mb.LindbladRelaxation([[0.0, 1e10], [0.0, 0.0]], [0.0])
    desc = mb.QmDescription(1e24, mb.QmOperator([0.0, 0.0]), mb.QmOperator([0.0, 0.0]), relax)
    ws = mb.precompute_relaxation_propagator(desc, 2e-12)
    e = math.exp(-0.01)
    assert np.allclose(ws.pop_half, [[1.0, 1.0 - e], [0.0, e]], rtol=1e-12)
    assert ws.coh_half[0, 1] == pytest.approx(math.exp(-0.005), rel=1e-12)


def test_relaxation_half_step_is_stochastic():
    from cases import random_medium

    rng = np.random.default_rng(8)
    for _ in range(50):
        dim = int(rng.integers(2, 7))
        desc = random_medium(mb, rng, dim, rate_scale=10 ** rng.uniform(8, 12))
        ws = mb.precompute_relaxation_propagator(desc, 10 ** rng.uniform(-18, -12))
        assert np.all(ws.pop_half >= 0.0)
        assert np.allclose(ws.pop_half.sum(axis=0), 1.0, atol=1e-12)


def _splitmix_loop(seed, count):
    mask = (1 << 64) - 1
    state = seed & mask
    out = []
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        out.append((z ^ (z >> 31)) / 2.0**64)
    return np.array(out)


@pytest.mark.parametrize("seed", [0, 7, 0xB10C, 2**64 - 1, 123456789123])
def test_vectorised_splitmix64_equals_the_sequential_stream(seed):
    assert np.array_equal(mb.splitmix64_uniform(seed, 5000), _splitmix_loop(seed, 5000))


def test_cfg2_initial_inversion():
    u = mb.splitmix64_uniform(0xB10C, 1)[0]
    assert abs(u - 0.923420) < 1e-6


@pytest.mark.parametrize("case", ["cfg3_r16", "multi_material", "vacuum_sources", "tiny_group"])
def test_region_table_reproduces_per_cell_maps(case):
    dev, sce, stepper = build_case(case)
    plan = mb.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    nx, dx = plan.grid.num_x, plan.grid.dx
    ends = np.array([r.x_end for r in dev.regions])
    cell_region = np.minimum(np.searchsorted(ends, np.arange(nx) * dx, side="right"), len(ends) - 1)
    h_region = np.minimum(np.searchsorted(ends, (np.arange(1, nx) - 0.5) * dx, side="right"), len(ends) - 1)
    cells = plan.regions.per_cell(nx)
    assert np.array_equal(cells["cell_region"], cell_region)
    coeffs = [mb.get_fdtd_constants(m, plan.grid.dt, dx) for m in plan.materials]
    assert np.array_equal(cells["coef_a"], np.array([coeffs[r].a_prime for r in cell_region]))
    assert np.array_equal(cells["coef_ch"][1:nx], np.array([coeffs[r].c_prime for r in h_region]))
    assert cells["coef_ch"][0] == 0.0 and cells["coef_ch"][nx] == 0.0


@pytest.mark.parametrize("replicas", [1, 2, 3, 8])
def test_weak_scaling_device_builds_for_every_gpu_count(replicas):
    """bench.py --gpus G: G copies of the cfg2 device side by side (G = 8 once
    failed: replica starts unit * j did not equal the previous end in fp64)."""
    mb.clear_material_library()
    from paper_2005_05412_b200 import configs

    nx = 4096 * replicas
    dev, sce = configs.cfg2(mb, nx=nx, steps=10, replicas=replicas, cells=(16, nx // 2))
    plan = mb.GpuFdtdSolver(dev, sce).plan
    assert len(dev.regions) == 3 * replicas and len(plan.groups) == replicas
    # the reference's per-cell group runs (solver_fdtd.py:276-285)
    ends = np.array([r.x_end for r in dev.regions])
    cell_region = np.minimum(np.searchsorted(ends, np.arange(nx) * plan.grid.dx, side="right"), len(ends) - 1)
    runs = []
    start = 0
    for m in range(1, nx + 1):
        if m == nx or cell_region[m] != cell_region[m - 1]:
            if cell_region[start] % 3 == 1:
                runs.append((start, m))
            start = m
    assert [(a, b) for a, b, _ in plan.groups] == runs


@pytest.mark.parametrize("n,stepper", [(2, "splitting"), (2, "rk4"), (3, "splitting"), (6, "splitting")])
def test_density_packing_round_trip(n, stepper):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    rho = a @ a.conj().T
    rho /= np.trace(rho).real
    w = P.pack_density(rho, stepper)
    assert w.size == P.state_words(n, stepper)
    back = P.unpack_density(w[:, None], n, stepper)[0]
    assert np.allclose(back, rho, atol=1e-15)


def test_validation_before_any_work_and_registry():
    dev, sce, _ = build_case("sit_hard_whole")
    sce.rho_init = mb.QmOperator([1.0, 0.0, 0.0])
    with pytest.raises(mb.ValidationError):
        mb.create_solver("gpu-fdtd-reg-cayley", dev, sce)
    with pytest.raises(mb.NotFoundError):
        mb.create_solver("no-such-solver", dev, sce)
    assert {"gpu-fdtd-reg-cayley", "gpu-fdtd-rk4"} <= set(mb.available_solvers())


def test_bad_stepper_rejected():
    dev, sce, _ = build_case("sit_hard_whole")
    with pytest.raises(ValueError):
        mb.GpuFdtdSolver(dev, sce, stepper="euler")


def test_solver_keeps_reference_attributes():
    dev, sce, _ = build_case("sit_hard_whole")
    s = mb.create_solver("gpu-fdtd-rk4", dev, sce, threads=2, seed=5)
    assert s.stepper == "rk4" and s.threads == 2 and s.seed == 5 and s.invariant_report is None
    assert isinstance(s.grid, mb.GridLayout)


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")
def test_plan_from_reference_objects_equals_plan_from_mirror():
    """Drop-in: the GPU solver accepts the reference's own Device/Scenario."""
    import os

    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    import mblight

    from cases import CASES

    for case in ("cfg2_r16", "multi_material", "rand5_split"):
        build, stepper = CASES[case]
        mblight.clear_material_library()
        mb.clear_material_library()
        a = mb.GpuFdtdSolver(*build(mblight), stepper=stepper).plan
        b = mb.GpuFdtdSolver(*build(mb), stepper=stepper).plan
        assert a.grid == b.grid
        assert np.array_equal(a.e_init, b.e_init) and np.array_equal(a.h_init, b.h_init)
        assert np.array_equal(a.src_values, b.src_values)
        for name in ("e_start", "h_start", "coef_a", "coef_bg", "coef_bdx", "coef_ch", "qm_index"):
            assert np.array_equal(getattr(a.regions, name), getattr(b.regions, name)), name
        for qa, qb in zip(a.qm, b.qm):
            for f in ("pop_half", "coh_half", "b_const", "b_field"):
                if getattr(qa, f) is not None:
                    assert np.array_equal(getattr(qa, f), getattr(qb, f)), f
            assert qa.bloch == qb.bloch
    mblight.clear_material_library()


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")
def test_registration_into_the_reference_registry():
    import os

    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    import mblight

    from cases import CASES

    mb.register_with_reference(mblight)
    assert {"gpu-fdtd-reg-cayley", "gpu-fdtd-rk4"} <= set(mblight.available_solvers())
    build, _ = CASES["sit_hard_whole"]
    mblight.clear_material_library()
    dev, sce = build(mblight)
    s = mblight.create_solver("gpu-fdtd-reg-cayley", dev, sce, seed=3)
    assert isinstance(s, mb.GpuFdtdSolver) and s.seed == 3
    assert s._result_cls is mblight.Result
    mblight.clear_material_library()
