"""GPU parity: the fused sm_100a solver against the reference's own records.

Golden fixtures were produced by running the reference ``FdtdSolver`` (see
tests/golden/make_golden.py).  Tolerance (max-norm relative per record,
BASELINE.json north star): 1e-9; dark records must be exactly zero.  The
two-level (Bloch) and field-only paths in ``exact`` mode (no FMA
contraction) must be bit-identical to the reference.
"""

import numpy as np
import pytest
from cases import CASES
from conftest import build_case, load_golden, rel_err

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb

pytestmark = pytest.mark.gpu

TOL = 1e-9
# cases whose arithmetic the exact variant reproduces bit for bit: the Bloch
# splitting kernel and the pure FDTD path (tiny_group excluded: the reference
# steps groups of <= 32 cells with numpy's ScalarKernel, _kernels.py:404-425)
BITWISE = {"cfg1_full", "cfg2_r16", "cfg2_full", "cfg2_stress_full", "sit_hard_whole", "multi_material", "bragg_stack",
           "vacuum_sources", "rand2_split", "kernel2_split"}
ALL = sorted(CASES)


def _run(name, **kw):
    dev, sce, stepper = build_case(name)
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, **kw)
    return solver, solver.run()


def _compare(name, results, bitwise):
    meta, recs = load_golden(name)
    assert [r.name for r in results] == [n for n, _, _ in recs]
    worst = 0.0
    for r, (rname, ref, axes) in zip(results, recs):
        assert r.data.shape == ref.shape, rname
        assert r.data.dtype == ref.dtype, rname
        assert r.dt_sample == axes["dt_sample"] and r.x0 == axes["x0"] and r.dx == axes["dx"], rname
        if bitwise:
            assert np.array_equal(r.data.view(np.float64), ref.view(np.float64)), (
                f"{rname}: not bit-identical (rel err {rel_err(r.data, ref):.3e})")
        else:
            err = rel_err(r.data, ref)
            worst = max(worst, err)
            assert err <= TOL, f"{name}/{rname}: rel err {err:.3e} > {TOL:g}"
    return worst


@pytest.mark.parametrize("name", ALL)
def test_fast_variant_matches_reference(name):
    solver, res = _run(name)
    meta, _ = load_golden(name)
    assert [solver.grid.num_x, solver.grid.dx, solver.grid.num_t, solver.grid.dt] == meta["grid"]
    _compare(name, res, bitwise=False)


@pytest.mark.parametrize("name", ALL)
def test_exact_variant_matches_reference(name):
    _, res = _run(name, exact=True)
    _compare(name, res, bitwise=name in BITWISE)


@pytest.mark.parametrize("k", [1, 2, 7, 16, 33, 64])
@pytest.mark.parametrize("name", ["sit_hard_whole", "multi_material", "vacuum_sources"])
def test_tile_depth_is_bitwise_invisible(name, k):
    """Temporal tiling recomputes halo cells redundantly; every cell runs the
    same instruction sequence, so results must not depend on k."""
    _, ref = _run(name, tile_steps=1)
    mb.clear_material_library()
    _, got = _run(name, tile_steps=k)
    for a, b in zip(ref, got):
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


@pytest.mark.parametrize("k", [None, 1, 5, 64, 112])
@pytest.mark.parametrize("name", ["sit_hard_whole", "multi_material", "vacuum_sources", "bragg_stack", "cfg2_r16"])
def test_persistent_wavefront_matches_per_launch(name, k):
    """The persistent kernel (one launch, chunk-major work items waiting on
    their neighbours of the previous chunk) against one launch per k steps."""
    _, ref = _run(name, tile_steps=k, persistent=False)
    mb.clear_material_library()
    solver, got = _run(name, tile_steps=k, persistent=True)
    assert solver.launches < solver.grid.num_t // 2
    for a, b in zip(ref, got):
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


@pytest.mark.parametrize("name,k", [("rand3_split", 5), ("rand6_split", 3), ("rand4_rk4", 6), ("cfg4_r14", 7)])
def test_tile_depth_dense_kernels(name, k):
    _, ref = _run(name, tile_steps=1)
    mb.clear_material_library()
    _, got = _run(name, tile_steps=k)
    for a, b in zip(ref, got):
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


def test_gpu_matches_oracle_on_fresh_seeds():
    """Random media not in the golden set: GPU vs the CPU oracle at 1e-9."""
    import oracle as orc
    from cases import random_case

    for dim, seed in ((3, 901), (5, 902), (6, 903), (8, 904)):
        mb.clear_material_library()
        build, stepper = random_case(dim, seed, nx=700, end=30e-15)
        dev, sce = build(mb)
        solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
        got = solver.run()
        recs, bad = orc.run_oracle(solver.plan)
        assert bad == 0
        for r, ref in zip(got, recs):
            assert rel_err(r.data, ref) <= TOL, (dim, r.name, rel_err(r.data, ref))


@pytest.mark.parametrize("stepper", ["splitting", "rk4"])
@pytest.mark.parametrize("dim", [3, 4, 5, 6, 7, 8])
def test_real_media_fast_paths_match_the_oracle(dim, stepper):
    """Real H0 and dipole: the symmetric-triangle inversion (splitting) and
    the real-H commutator (RK4) of the fast variant against the CPU oracle."""
    import oracle as orc
    from cases import random_case

    mb.clear_material_library()
    build, _ = random_case(dim, 950 + dim, nx=600, end=25e-15, stepper=stepper, real=True)
    dev, sce = build(mb)
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    got = solver.run()
    recs, bad = orc.run_oracle(solver.plan)
    assert bad == 0
    for r, ref in zip(got, recs):
        assert rel_err(r.data, ref) <= TOL, (dim, stepper, r.name, rel_err(r.data, ref))
