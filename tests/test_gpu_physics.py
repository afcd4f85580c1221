"""Physics of the reference's own built-in setups, run by the GPU solver at
their published scale (the criteria of the reference's acceptance suite,
pkg/tests/test_acceptance.py, evaluated here on the GPU solver's results):

* self-induced transparency (ziolkowski1995, test_acceptance.py:203-229): a
  2-pi sech pulse leaves the two-level medium behind it in the ground state,
  a pi pulse inverts it;
* vacuum propagation (test_acceptance.py:232-259): the pulse peak travels at
  c0 within 3 dx with < 2 % amplitude loss;
* laser build-up and gain clamping (tzenov2016, the paper's five-level QCL
  frequency comb, test_acceptance.py:432-469): the field energy grows by at
  least 20 dB from the noise seed and then clamps (< 1 dB variation of its
  10 ps average over the last 50 ps).

These are whole-run properties at full size (the golden records pin the
numbers on the same setups at tolerance); the reference needs 20 s (SIT) and
15 min (laser) on 8 CPU workers for them.
"""

import dataclasses
import math
import time

import numpy as np
import pytest

import paper_2005_05412_b200 as gpu  # noqa: F401  (registers the GPU solver names)
from paper_2005_05412_b200.reference import mblight as mb

pytestmark = pytest.mark.gpu


def _run(dev, sce, **kw):
    t0 = time.perf_counter()
    res = {r.name: r for r in mb.create_solver("gpu-fdtd-reg-cayley", dev, sce, **kw).run()}
    return res, time.perf_counter() - t0


def _inversion_behind_the_peak(res, margin=10e-6):
    """Inversion at the last record row between 10 um into the medium and
    10 um behind the field maximum."""
    e, inv = res["e"], res["inv12"]
    last = e.data[-1]
    x = e.positions
    peak = x[int(np.argmax(np.abs(last)))]
    sel = (x > margin) & (x < peak - margin)
    assert sel.sum() > 100, "pulse did not get far enough into the medium"
    return inv.data[-1][sel], peak


def test_self_induced_transparency_and_pi_pulse_inversion():
    mb.clear_material_library()
    dev, sce = mb.builtin_setup("ziolkowski1995")
    res, t_full = _run(dev, sce)
    behind, peak = _inversion_behind_the_peak(res)
    assert np.max(np.abs(behind + 1.0)) < 0.05, (np.max(np.abs(behind + 1.0)), peak)

    # the same setup with the pulse amplitude halved: a pi pulse
    mb.clear_material_library()
    dev, sce = mb.builtin_setup("ziolkowski1995")
    src = sce.sources[0]
    sce.sources[0] = dataclasses.replace(src, amplitude=src.amplitude / 2.0)
    res, t_half = _run(dev, sce)
    behind, _ = _inversion_behind_the_peak(res)
    assert np.max(np.abs(behind - 1.0)) < 0.1, np.max(np.abs(behind - 1.0))
    assert t_full < 60.0 and t_half < 60.0


def test_vacuum_pulse_travels_at_c0():
    mb.clear_material_library()
    vac = mb.ensure_material(mb.Material("Vacuum"))
    dev = mb.Device("vac")
    dev.add_region(mb.Region("v", vac.id, 0.0, 200e-6))
    nx = 8192
    sce = mb.Scenario("s", nx, 610e-15, mb.QmOperator([1.0, 0.0]))
    sce.add_source(mb.SechPulse("sech", 0.0, "hard", 1.0, 2e14, 10.0, 2e14))
    sce.add_record(mb.Record("e", quantity="e", interval=150e-15))
    res, _ = _run(dev, sce)
    e = res["e"]
    last = e.data[-1]
    dx = 200e-6 / (nx - 1)
    travelled = mb.C0 * (e.times[-1] - 10.0 / 2e14)  # envelope centred at shift / rate
    x_peak = e.positions[int(np.argmax(np.abs(last)))]
    assert travelled >= 150e-6
    assert abs(x_peak - travelled) <= 3 * dx, (x_peak, travelled, dx)
    assert np.max(np.abs(last)) >= 0.98


def test_laser_gain_build_up_and_clamping():
    mb.clear_material_library()
    dev, sce = mb.builtin_setup("tzenov2016")
    res, elapsed = _run(dev, sce)
    e, h = res["e"], res["h"]
    eps = mb.EPS0 * 12.96
    energy = 0.5 * eps * np.sum(e.data ** 2, axis=1) + 0.5 * mb.MU0 * np.sum(h.data ** 2, axis=1)
    growth = 10.0 * math.log10(float(np.max(energy)) / float(energy[0]))
    dts = e.dt_sample
    w = max(1, round(10e-12 / dts))
    avg = np.convolve(energy, np.ones(w) / w, mode="valid")
    tail = avg[-(round(50e-12 / dts) - w + 1):]
    clamp = 10.0 * math.log10(float(np.max(tail)) / float(np.min(tail)))
    assert growth >= 20.0, growth
    assert clamp < 1.0, clamp
    assert elapsed < 900.0
