"""Host-side setup (plan.py) against the reference: its known answers for grid
sizing (pkg/tests/test_solver.py:63-75), coefficients (:119-141) and the
relaxation propagator closed form (pkg/tests/test_quantum.py:349-359), and the
plan against the reference's own ``FdtdSolver.__init__`` for the same objects."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest
from conftest import build_case

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb
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


def test_cfg2_initial_inversion():
    from importlib import import_module

    u = import_module("mblight.core")._splitmix64_stream(0xB10C, 1)[0]
    assert abs(u - 0.923420) < 1e-6


@pytest.mark.parametrize("case", ["cfg3_r16", "multi_material", "vacuum_sources", "tiny_group"])
def test_region_table_reproduces_per_cell_maps(case):
    dev, sce, stepper = build_case(case)
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
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
    plan = gpu.GpuFdtdSolver(dev, sce).plan
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
        gpu.GpuFdtdSolver(dev, sce, stepper="euler")


def test_solver_keeps_reference_attributes():
    dev, sce, _ = build_case("sit_hard_whole")
    s = mb.create_solver("gpu-fdtd-rk4", dev, sce, threads=2, seed=5)
    assert s.stepper == "rk4" and s.threads == 2 and s.seed == 5 and s.invariant_report is None
    assert isinstance(s.grid, mb.GridLayout)


@pytest.mark.parametrize("case", ["cfg2_r16", "multi_material", "rand5_split", "sit_hard_whole",
                                  "vacuum_sources", "tiny_group", "song_point"])
def test_plan_equals_the_reference_constructor(case):
    """Everything the kernels consume equals what the reference's own
    ``FdtdSolver.__init__`` (solver_fdtd.py:207-326) builds for the same
    objects: per-cell coefficients, initial fields, boundary constants, source
    cells, record schedules and the stepper constants of every quantum group."""
    dev, sce, stepper = build_case(case)
    ref = mb.FdtdSolver(dev, sce, stepper=stepper)
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    g = plan.grid
    assert g == ref.grid
    assert np.array_equal(plan.e_init, ref.e) and np.array_equal(plan.h_init, ref.h)
    if g.num_x > 1:
        cells = plan.regions.per_cell(g.num_x)
        for name in ("coef_a", "coef_bg", "coef_bdx", "coef_ch"):
            assert np.array_equal(cells[name], getattr(ref, name)), name
        assert plan.boundary == ref._bc
    assert [(c, k) for c, k in zip(plan.src_cells, plan.src_hard)] == \
        [(cell, 1 if src.kind == "hard" else 0) for src, cell in ref._sources]
    for k, (src, _) in enumerate(ref._sources):
        n = np.arange(1, g.num_t, max(1, g.num_t // 97))
        assert np.array_equal(plan.src_values[n, k], [src.value(i * g.dt) for i in n])
    for p, rp in zip(plan.plans, ref._plans):
        assert (p.every, p.rows, p.cell, p.cols) == (rp.every, rp.rows, rp.cell, rp.cols)
        assert repr(p.x0) == repr(rp.x0)  # -0.0 != 0.0 in the archive's json
    assert [(a, b) for a, b, _ in plan.groups] == [(gr.start, gr.stop) for gr in ref.groups]
    for (_, _, q), gr in zip(plan.groups, ref.groups):
        qc, k = plan.qm[q], gr.kernel
        if type(k).__name__ == "ScalarKernel":  # groups of <= 32 cells step through numpy
            continue
        assert qc.pol_factor == k._pol_factor and np.array_equal(qc.pol_v, k._pol_v)
        if qc.bloch is not None:
            assert (qc.bloch["kz"], qc.bloch["cz"], qc.bloch["fxy"]) == (k._kz, k._cz, k._fxy)
            assert (qc.bloch["ax_c"], qc.bloch["ax_s"]) == k._ax and (qc.bloch["az_c"], qc.bloch["az_s"]) == k._az
        elif qc.pop_half is not None:
            assert np.array_equal(qc.pop_half, k.pop_half) and np.array_equal(qc.b_const, k._b_const)
            assert np.array_equal(qc.coh_half, k.coh_half) and np.array_equal(qc.b_field, k._b_field)
        elif qc.h0 is not None and hasattr(k, "_h0"):
            assert np.array_equal(qc.h0, k._h0) and np.array_equal(qc.pop_matrix, k._pop)


def test_whole_domain_record_origin_is_positive_zero():
    """x0 of a whole-domain e/inv record is +0.0 as in the reference
    (solver_fdtd.py:150), so meta.json of the archive matches byte for byte."""
    import json

    dev, sce, stepper = build_case("sit_hard_whole")
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    whole = [p for p in plan.plans if p.cell is None and p.record.quantity != "h"]
    assert whole and all(json.dumps(p.x0) == "0.0" for p in whole)


def test_registration_into_the_reference_registry():
    from cases import CASES

    gpu.register_with_reference(mb)
    assert {"gpu-fdtd-reg-cayley", "gpu-fdtd-rk4"} <= set(mb.available_solvers())
    build, _ = CASES["sit_hard_whole"]
    dev, sce = build(mb)
    s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce, seed=3)
    assert isinstance(s, gpu.GpuFdtdSolver) and s.seed == 3


def test_source_sample_cache_is_per_sweep():
    """Without a caller-owned cache every plan samples its sources with
    Source.value again, as the reference does on every run; subclasses are
    never shared."""
    from paper_2005_05412_b200 import plan as P

    calls = []

    class Counting(mb.SechPulse):
        def value(self, t):
            calls.append(t)
            return super().value(t)

    src = Counting("c", 0.0, "soft", 1.0, 2e14, 5.0, 1e15)
    assert P._cached_samples(src, 1e-17, 50, {}) is None
    assert P._cached_samples(mb.SechPulse("s", 0.0, "soft", 1.0, 2e14, 5.0, 1e15), 1e-17, 50, None) is None
    cache = {}
    s2 = mb.SechPulse("s", 0.0, "soft", 1.0, 2e14, 5.0, 1e15)
    a = P._cached_samples(s2, 1e-17, 50, cache)
    b = P._cached_samples(mb.SechPulse("s", 0.0, "soft", 1.0, 2e14, 5.0, 1e15), 1e-17, 50, cache)
    assert a is b and len(cache) == 1
    assert np.array_equal(a[1:], [s2.value(n * 1e-17) for n in range(1, 50)])


def test_sources_sampled_in_segments_equal_one_pass():
    """The run samples its sources segment by segment (plan.sample_sources);
    any split gives the table a single pass of Source.value gives."""
    dev, sce, stepper = build_case("vacuum_sources")
    full = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan.src_values.copy()
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    assert plan.sampled_to == 1
    n = plan.grid.num_t
    for hi in (2, 7, 7, n // 3, n // 2 + 1, n + 5):
        lo, got_hi = plan.sample_sources(hi)
        assert got_hi == min(hi, n) and plan.sampled_to == got_hi
    assert np.array_equal(plan.src_buffer, full)


@pytest.mark.parametrize("seed", range(6))
def test_region_starts_equal_searchsorted_maps(seed):
    """The region table is derived from the region ends alone; it equals the
    first-cell-of-each-region of the reference's per-cell maps
    (searchsorted(ends, m dx, 'right') and (m - 1/2) dx for H nodes,
    solver_fdtd.py:245-266), also for ends that fall exactly on a cell or
    node position and for empty regions."""
    from paper_2005_05412_b200 import plan as P

    rng = np.random.default_rng(seed)
    nx = int(rng.integers(2, 3000))
    dx = float(rng.uniform(1e-11, 1e-8))
    n_reg = int(rng.integers(1, 9))
    cuts = []
    for _ in range(n_reg - 1):
        m = int(rng.integers(0, nx + 2))
        kind = rng.integers(0, 3)
        cuts.append(m * dx if kind == 0 else (m - 0.5) * dx if kind == 1 else float(rng.uniform(0, nx * dx)))
    ends = sorted(cuts) + [(nx - 1) * dx]
    cell_region = np.minimum(np.searchsorted(ends, np.arange(nx) * dx, side="right"), n_reg - 1)
    h_region = np.minimum(np.searchsorted(ends, (np.arange(1, nx) - 0.5) * dx, side="right"), n_reg - 1)
    want_e = np.searchsorted(cell_region, np.arange(n_reg), side="left")
    want_h = np.searchsorted(h_region, np.arange(n_reg), side="left") + 1
    got_e = [0] + [P._first_at_or_after(ends[r - 1], dx, 0, nx) for r in range(1, n_reg)]
    got_h = [1] + [P._first_at_or_after(ends[r - 1], dx, 1, nx, 0.5) for r in range(1, n_reg)]
    assert list(want_e) == got_e and list(want_h) == got_h
