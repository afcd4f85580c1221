"""Host side of the batched single-point mode (no GPU): the precomputed field
sequence equals the reference's per-step source application, and the batch
API validates its inputs before any work."""

import math

import numpy as np
import pytest

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb
from paper_2005_05412_b200 import points as P
from paper_2005_05412_b200.plan import build_plan


def _loop(plan):
    """solver_fdtd.py:366-385 at one grid point: sources in order on the previous E."""
    nt = plan.grid.num_t
    e = np.empty(nt)
    e[0] = cur = plan.e_init[0]
    for n in range(1, nt):
        for k in range(len(plan.src_hard)):
            cur = plan.src_values[n, k] if plan.src_hard[k] else cur + plan.src_values[n, k]
        e[n] = cur
    return e


def _point(kinds, ic=0.0):
    mb.clear_material_library()
    qm = mb.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e11, 1e12, -1.0)
    act = mb.ensure_material(mb.Material("P", qm=qm))
    dev = mb.Device("p")
    dev.add_region(mb.Region("point", act.id, 0.0, 0.0))
    sce = mb.Scenario("s", 1, 100e-15, mb.QmOperator([1.0, 0.0]), num_timesteps=3000,
                      ic_e_field=mb.CurveField(np.array([ic])))
    for k, kind in enumerate(kinds):
        sce.add_source(mb.SechPulse(f"s{k}", 0.0, kind, 1e9 * (k + 1), 2e14 * (1 + 0.1 * k), 5.0, 2e14))
    sce.add_record(mb.Record("e", quantity="e", position=0.0))
    return dev, sce


@pytest.mark.parametrize("kinds", [[], ["soft"], ["hard"], ["soft", "soft"], ["hard", "soft"],
                                   ["soft", "hard"], ["soft", "hard", "soft", "soft"], ["hard", "hard"]])
def test_field_sequence_equals_the_reference_loop(kinds):
    dev, sce = _point(kinds, ic=123.0)
    plan = build_plan(dev, sce)
    assert np.array_equal(P._field_sequence(plan), _loop(plan))


def test_batch_rejects_extended_grids_before_any_work():
    mb.clear_material_library()
    qm = mb.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e11, 1e12, -1.0)
    act = mb.ensure_material(mb.Material("P", qm=qm))
    dev = mb.Device("line")
    dev.add_region(mb.Region("a", act.id, 0.0, 1e-6))
    sce = mb.Scenario("s", 64, 10e-15, mb.QmOperator([1.0, 0.0]))
    with pytest.raises(ValueError):
        P.run_points([(dev, sce)])
    assert P.run_points([]) == []


def test_vector_samples_within_two_ulp_of_source_value():
    """run_points(fast_sources=True) samples the reference's pulse types with
    one numpy evaluation; every sample is within 2 ulp (of the pulse
    amplitude's scale) of Source.value."""
    import numpy as np

    from paper_2005_05412_b200.points import vector_samples
    from paper_2005_05412_b200.reference import mblight as mb

    srcs = [mb.SechPulse("s", 0.0, "soft", 3.5e9, 3.8e14, 17.2, 3.5e14, -1.5),
            mb.SechPulse("h", 0.0, "hard", 1.0, 2e14, 10.0, 2e14),
            mb.GaussianPulse("g", 0.0, "soft", 1e9, 1.9e14, 0.75e-15, 0.25e-15),
            mb.GaussianPulse("g2", 0.0, "soft", 2e9, 2.1e14, 600e-15, 200e-15, 0.3)]
    for src in srcs:
        dt, n = 7.6e-18, 20000
        got = vector_samples(src, dt, n)
        want = np.array([src.value(i * dt) for i in range(n)])
        scale = abs(src.amplitude)
        assert np.max(np.abs(got - want)) <= 2 * np.spacing(scale), src.name
    assert vector_samples(mb.ConstantField(0.0), 1e-18, 10) is None
