"""Batched single-grid-point runs (paper_2005_05412_b200.points.run_points,
C ABI mbg_batch_points): every system of a batch gives what the solver gives
for it alone, and the reference's own records where the golden set has them."""

import math

import numpy as np
import pytest
from conftest import load_golden, rel_err

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb
from paper_2005_05412_b200.points import run_points

pytestmark = pytest.mark.gpu


def _song(scale=1.0, density=6e24, tag=""):
    """song2005's driven V-type three-level point (tests/cases.py song_point)
    with the pulse amplitude scaled and the density changed."""
    hb, e0 = mb.HBAR, mb.E0
    h0 = mb.QmOperator([0.0, 2.3717e15 * hb, 2.4165e15 * hb])
    mu = mb.QmOperator([0.0, 0.0, 0.0], [-e0 * 9.2374e-11, -e0 * 9.2374e-11 * math.sqrt(2.0), 0.0])
    rates = [[0.0, 1e10, 1e10], [1e10, 0.0, 1e10], [1e10, 1e10, 0.0]]
    qm = mb.QmDescription(density, h0, mu, mb.LindbladRelaxation(rates, [0.0, 0.0, 0.0]))
    act = mb.ensure_material(mb.Material("Song3" + tag, qm=qm))
    dev = mb.Device("Song")
    dev.add_region(mb.Region("point", act.id, 0.0, 0.0))
    sce = mb.Scenario("s", 1, 80e-15, mb.QmOperator([1.0, 0.0, 0.0]), num_timesteps=10000)
    for i in (1, 2, 3):
        sce.add_record(mb.Record(f"d{i}{i}", quantity="d", i=i, j=i, position=0.0))
    sce.add_record(mb.Record("d12", quantity="d", i=1, j=2, position=0.0))
    sce.add_record(mb.Record("e", quantity="e", position=0.0))
    sce.add_source(mb.SechPulse("sech", position=0.0, kind="hard", amplitude=3.5471e9 * scale,
                                carrier_freq=3.8118e14, envelope_shift=17.248, envelope_rate=1.76 / 5e-15,
                                carrier_phase=-math.pi / 2.0))
    return dev, sce


def _two_level(scale=1.0, t2=1e12, tag=""):
    """tests/cases.py point2 with the soft pulse scaled and T2 changed."""
    qm = mb.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e11, t2, -1.0)
    act = mb.ensure_material(mb.Material("P2" + tag, qm=qm))
    dev = mb.Device("p2")
    dev.add_region(mb.Region("point", act.id, 0.0, 0.0))
    sce = mb.Scenario("s", 1, 100e-15, mb.QmOperator([1.0, 0.0]), num_timesteps=5000)
    sce.add_record(mb.Record("inv", quantity="inv", position=0.0))
    sce.add_record(mb.Record("d12", quantity="d", i=1, j=2, position=0.0))
    sce.add_record(mb.Record("e", quantity="e", position=0.0))
    sce.add_source(mb.SechPulse("s", 0.0, "soft", 4e9 * scale, 2e14, 5.0, 2e14))
    return dev, sce


def _alone(build, stepper, exact, **kw):
    mb.clear_material_library()
    dev, sce = build(**kw)
    return gpu.GpuFdtdSolver(dev, sce, stepper=stepper, exact=exact).run()


@pytest.mark.parametrize("stepper", ["splitting", "rk4"])
@pytest.mark.parametrize("exact", [False, True])
def test_three_level_batch_equals_single_runs(stepper, exact):
    """Same cell function, same constants: bit for bit the single-point solver."""
    variants = [dict(scale=s, density=d, tag=t) for s, d, t in
                ((1.0, 6e24, ""), (0.5, 6e24, ""), (2.0, 6e24, ""), (1.0, 3e24, "b"), (1.3, 3e24, "b"))]
    mb.clear_material_library()
    batch = run_points([_song(**v) for v in variants], stepper=stepper, exact=exact)
    for v, got in zip(variants, batch):
        ref = _alone(_song, stepper, exact, **v)
        for a, b in zip(ref, got):
            assert a.name == b.name and a.data.shape == b.data.shape and a.dt_sample == b.dt_sample
            assert np.array_equal(a.data, b.data), (v, a.name, rel_err(b.data, a.data))


@pytest.mark.parametrize("stepper", ["splitting", "rk4"])
@pytest.mark.parametrize("exact", [False, True])
def test_two_level_batch_matches_single_runs(exact, stepper):
    """Bloch systems (the reference's rotation order in the batch kernel;
    the single solver's fast variant steps a relaxed frame, so 1e-9) and
    two-level RK4 (the same cell function: bit for bit)."""
    variants = [dict(scale=s, t2=t, tag=g) for s, t, g in ((1.0, 1e12, ""), (0.3, 1e12, ""), (3.0, 5e11, "b"))]
    mb.clear_material_library()
    batch = run_points([_two_level(**v) for v in variants], stepper=stepper, exact=exact)
    for v, got in zip(variants, batch):
        ref = _alone(_two_level, stepper, exact, **v)
        for a, b in zip(ref, got):
            assert a.data.shape == b.data.shape
            if stepper == "rk4":
                assert np.array_equal(a.data, b.data), (v, a.name, rel_err(b.data, a.data))
            else:
                assert rel_err(b.data, a.data) <= 1e-9, (v, a.name, rel_err(b.data, a.data))


@pytest.mark.parametrize("case,build,stepper", [("song_point", _song, "splitting"), ("song_point_rk4", _song, "rk4"),
                                                ("point2", _two_level, "splitting")])
def test_batch_member_matches_the_reference_golden(case, build, stepper):
    mb.clear_material_library()
    batch = run_points([build(), build(scale=0.7)], stepper=stepper)
    _, recs = load_golden(case)
    for r, (name, ref, _) in zip(batch[0], recs):
        assert r.name == name
        assert rel_err(r.data, ref) <= 1e-9, (case, name, rel_err(r.data, ref))


def test_batch_refuses_mixed_problems():
    mb.clear_material_library()
    a = _song()
    dev, sce = _song(tag="c")
    sce.num_timesteps = 5000
    with pytest.raises(ValueError):
        run_points([a, (dev, sce)])
    with pytest.raises(ValueError):
        run_points([a, _two_level()])


@pytest.mark.parametrize("stepper", ["splitting", "rk4"])
def test_sweep_over_many_media_in_one_call(stepper):
    """A dephasing-rate sweep over 4096 distinct two-level media (constant
    sets in device memory, no per-launch cap) with one shared pulse: every
    sampled member equals its single-point run (splitting: the batch kernel
    keeps the reference's rotation order, the solver's fast frame path is
    tolerance-level; RK4: the same cell function, bit for bit)."""
    from paper_2005_05412_b200.points import LAST_RUN

    mb.clear_material_library()
    t2s = np.linspace(2e11, 5e12, 4096)
    problems = [_two_level(t2=float(t), tag=f"m{i}") for i, t in enumerate(t2s)]
    batch = run_points(problems, stepper=stepper)
    assert len(batch) == 4096 and LAST_RUN["systems"] == 4096
    for i in (0, 1, 2047, 4095):
        ref = _alone(_two_level, stepper, False, t2=float(t2s[i]), tag=f"m{i}")
        for a, b in zip(ref, batch[i]):
            assert a.data.shape == b.data.shape
            if stepper == "rk4":
                assert np.array_equal(a.data, b.data), (i, a.name, rel_err(b.data, a.data))
            else:
                assert rel_err(b.data, a.data) <= 1e-9, (i, a.name, rel_err(b.data, a.data))
    # distinct media give distinct populations
    inv = np.array([batch[i][0].data[-1, 0] for i in (0, 4095)])
    assert inv[0] != inv[1]


def test_fast_sources_match_reference_sampling():
    """run_points(fast_sources=True): the pulse sweep with numpy-sampled
    sources agrees with the Source.value-sampled batch to tolerance."""
    mb.clear_material_library()
    variants = [dict(scale=s) for s in (0.3, 1.0, 2.7)]
    a = run_points([_song(**v) for v in variants])
    mb.clear_material_library()
    b = run_points([_song(**v) for v in variants], fast_sources=True)
    for ra, rb in zip(a, b):
        for x, y in zip(ra, rb):
            assert rel_err(y.data, x.data) <= 1e-11, (x.name, rel_err(y.data, x.data))
