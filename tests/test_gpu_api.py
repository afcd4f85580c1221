"""The GPU solver honours the reference solver's run() contract and physics
checks (pkg/tests/test_solver.py, test_acceptance.py analogues)."""

import math

import numpy as np
import pytest
from conftest import build_case

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb

pytestmark = pytest.mark.gpu


def _sit_small(gridpoints=1024, end=20e-15):
    qm = mb.two_level_description(1e24, 2 * math.pi * 2e14, 6.24e-11, 1e10, 1e10, -1.0)
    mb.add_material(mb.Material("Vacuum"))
    mb.add_material(mb.Material("Active", qm=qm))
    dev = mb.Device("small")
    dev.add_region(mb.Region("l", "Vacuum", 0.0, 7.5e-6))
    dev.add_region(mb.Region("a", "Active", 7.5e-6, 142.5e-6))
    dev.add_region(mb.Region("r", "Vacuum", 142.5e-6, 150e-6))
    return dev, mb.Scenario("s", gridpoints, end, mb.QmOperator([1.0, 0.0]))


def test_run_is_not_reentrant():
    dev, sce = _sit_small(128, 1e-15)
    s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce)
    s.run()
    with pytest.raises(mb.SolverError):
        s.run()


def test_record_shapes_axes_and_order():
    dev, sce = _sit_small()
    sce.add_record(mb.Record("e", quantity="e", interval=2.5e-15))
    sce.add_record(mb.Record("inv12", quantity="inv", interval=2.5e-15))
    sce.add_record(mb.Record("probe", quantity="e", position=75e-6))
    sce.add_record(mb.Record("d12", quantity="d", i=1, j=2, position=75e-6))
    s = gpu.GpuFdtdSolver(dev, sce)
    res = {r.name: r for r in s.run()}
    every = round(2.5e-15 / s.grid.dt)
    rows = (s.grid.num_t - 1) // every + 1
    assert res["e"].data.shape == (rows, 1024) and res["inv12"].data.shape == (rows, 1024)
    assert res["e"].dt_sample == every * s.grid.dt
    assert res["probe"].cols == 1 and res["probe"].rows == s.grid.num_t
    assert res["d12"].is_complex
    assert [r.name for r in s.results] == ["e", "inv12", "probe", "d12"]


def test_inversion_outside_quantum_region_is_zero():
    dev, sce = _sit_small()
    sce.add_record(mb.Record("inv12", quantity="inv", interval=2.5e-15))
    inv = gpu.GpuFdtdSolver(dev, sce).run()[0]
    x = inv.positions
    vac = (x < 7.5e-6) | (x > 142.5e-6)
    assert np.count_nonzero(inv.data[-1][vac]) == 0
    assert np.allclose(inv.data[-1][~vac], -1.0, atol=1e-12)


def test_zero_state_stays_zero():
    qm = mb.two_level_description(1e24, 2 * math.pi * 2e14, 6.24e-11, 1e10, 1e10, -1.0)
    mb.add_material(mb.Material("Active", qm=qm))
    dev = mb.Device("quiet")
    dev.add_region(mb.Region("a", "Active", 0.0, 1e-6))
    sce = mb.Scenario("s", 64, 2e-15, mb.QmOperator([1.0, 0.0]))
    sce.add_record(mb.Record("e", quantity="e"))
    sce.add_record(mb.Record("h", quantity="h"))
    for r in gpu.GpuFdtdSolver(dev, sce).run():
        assert np.count_nonzero(r.data) == 0


def test_nonfinite_field_aborts_with_the_scan_step():
    desc = mb.QmDescription(1e28, mb.QmOperator([0.0, 1e-19]), mb.QmOperator([0.0, 0.0], [1e-27]),
                            mb.LindbladRelaxation([[0.0, 1e21], [1e21, 0.0]], [0.0]))
    mb.add_material(mb.Material("stiff", qm=desc))
    dev = mb.Device("blow")
    dev.add_region(mb.Region("a", "stiff", 0.0, 10e-6))
    sce = mb.Scenario("s", 64, 2e-13, mb.QmOperator([1.0, 0.0]))
    sce.add_source(mb.SechPulse("s", 5e-6, "hard", 1e10, 2e14, 10.0, 2e14))
    import oracle as orc

    solver = gpu.GpuFdtdSolver(dev, sce, stepper="rk4")
    _, bad = orc.run_oracle(solver.plan)
    with pytest.raises(mb.SolverError, match=f"at step {bad}$"):
        solver.run()


def test_pulse_travels_at_light_speed():
    mb.add_material(mb.Material("Vacuum"))
    dev = mb.Device("v", bc_left=mb.BoundaryReflectivity(1.0), bc_right=mb.BoundaryReflectivity(0.0))
    dev.add_region(mb.Region("v", "Vacuum", 0.0, 40e-6))
    sce = mb.Scenario("s", 2048, 100e-15, mb.QmOperator([1.0, 0.0]))
    sce.add_source(mb.SechPulse("sech", 0.0, "hard", 1.0, 2e14, 10.0, 2e14))
    sce.add_record(mb.Record("e", quantity="e", interval=100e-15))
    e = gpu.GpuFdtdSolver(dev, sce).run()[0]
    x_peak = e.positions[int(np.argmax(np.abs(e.data[-1])))]
    assert abs(x_peak - mb.C0 * (e.times[-1] - 50e-15)) <= 3 * (40e-6 / 2047)
    assert np.max(np.abs(e.data[-1])) >= 0.98


def _reflection_energy_ratio(r):
    mb.clear_material_library()
    mb.add_material(mb.Material("Vacuum"))
    dev = mb.Device("bc", bc_left=mb.BoundaryReflectivity(0.0), bc_right=mb.BoundaryReflectivity(r))
    dev.add_region(mb.Region("v", "Vacuum", 0.0, 60e-6))
    sce = mb.Scenario("s", 4096, 240e-15, mb.QmOperator([1.0, 0.0]))
    sce.add_source(mb.SechPulse("sech", 20e-6, "soft", 1.0, 2e14, 10.0, 2e14))
    sce.add_record(mb.Record("e", quantity="e", interval=5e-15))
    sce.add_record(mb.Record("h", quantity="h", interval=5e-15))
    res = {x.name: x for x in gpu.GpuFdtdSolver(dev, sce).run()}
    dx = 60e-6 / 4095
    energy = 0.5 * mb.EPS0 * np.sum(res["e"].data ** 2, axis=1) * dx
    energy += 0.5 * mb.MU0 * np.sum(res["h"].data ** 2, axis=1) * dx
    t = res["e"].times
    return energy[np.argmin(np.abs(t - 230e-15))] / energy[np.argmin(np.abs(t - 160e-15))]


def test_boundary_energy_contract():
    """pkg/tests/test_solver.py:286-296 on the GPU solver."""
    assert _reflection_energy_ratio(1.0) == pytest.approx(1.0, abs=0.02)
    assert _reflection_energy_ratio(0.0) < 0.01
    for r in (0.25, 0.64):
        assert _reflection_energy_ratio(r) == pytest.approx(r, rel=0.10)


def test_sit_physics_full_run():
    """Self-induced transparency (pkg/tests/test_acceptance.py:203-229): the
    medium is left inverted-back (|w+1| < 0.05) behind a 2 pi pulse."""
    dev, sce, _ = build_case("cfg1_full")
    res = {r.name: r for r in gpu.GpuFdtdSolver(dev, sce).run()}
    inv = res["inv@2000"].data[:, 0]
    assert np.max(np.abs(inv[-1] + 1.0)) < 0.05
    assert np.min(inv) > -1.0 - 1e-9 and np.max(inv) <= 1.0 + 1e-9


def test_invariant_monitor():
    dev, sce, stepper = build_case("rand4_split")
    s = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, monitor_invariants=True)
    s.run()
    rep = s.invariant_report
    assert rep["max_trace_dev"] < 1e-9 and rep["max_herm_dev"] < 1e-12 and rep["min_eigenvalue"] > -1e-9


def test_results_are_independent_arrays():
    dev, sce = _sit_small(256, 5e-15)
    sce.add_record(mb.Record("e", quantity="e"))
    s = gpu.GpuFdtdSolver(dev, sce)
    r = s.run()[0]
    r.data[:] = 1.0  # caller owns the buffers
    assert s.results[0].data is r.data


@pytest.mark.parametrize("case", ["rand3_split", "rand6_split", "rand8_split", "rand4_rk4", "multi_material"])
def test_device_invariant_monitor_matches_numpy(case):
    """mbg_invariants (device reduction + Jacobi eigenvalues) vs numpy eigvalsh
    of the downloaded state (the reference's invariant_stats, _kernels.py:394-401)."""
    from paper_2005_05412_b200 import native
    from paper_2005_05412_b200.plan import unpack_density

    dev, sce, stepper = build_case(case)
    s = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    h = s.open_handle()
    s.upload_initial_state(h)
    h.call("mbg_sample", 0)
    h.call("mbg_advance", 1, min(200, s.grid.num_t - 1))
    out = np.zeros(3)
    h.call("mbg_invariants", native.ptr(out))
    words = np.zeros((s.plan.state_words, s.grid.num_x))
    h.call("mbg_download_state", native.ptr(words))
    h.close()
    cells = np.concatenate([np.arange(lo, hi) for lo, hi, _ in s.plan.groups])
    rho = unpack_density(words[:, cells], s.plan.levels, s.plan.stepper)
    if s.plan.levels == 2 and stepper == "splitting":
        want_eig = 0.5 * (1.0 - np.max(np.sqrt(np.sum(words[:, cells] ** 2, axis=0))))
        want_tr = 0.0
    else:
        want_eig = np.min(np.linalg.eigvalsh(rho))
        want_tr = np.max(np.abs(np.trace(rho, axis1=1, axis2=2).real - 1.0))
    assert out[0] == pytest.approx(want_tr, abs=1e-15)
    assert out[1] == 0.0
    assert out[2] == pytest.approx(want_eig, abs=1e-13)


def test_sit_run_invariants_like_the_acceptance_suite():
    """pkg/tests/test_acceptance.py:74-116: trace < 1e-9, Hermiticity < 1e-12,
    eigenvalues > -1e-9 over the full transparency run (monitor at record cadence)."""
    dev, sce, _ = build_case("sit_hard_whole")
    s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce, monitor_invariants=True)
    s.run()
    rep = s.invariant_report
    assert rep["max_trace_dev"] < 1e-9 and rep["max_herm_dev"] < 1e-12 and rep["min_eigenvalue"] > -1e-9


def test_single_step_matches_hand_computed_update():
    """pkg/tests/test_solver.py:150-199 on the GPU: one step over random E/H
    and a random density matrix, against a hand-written update."""
    rng = np.random.default_rng(21)
    nx = 16
    qm = mb.two_level_description(1e24, 2 * math.pi * 2e14, 6.24e-11, 1e10, 1e10, -1.0)
    mb.add_material(mb.Material("Active", qm=qm))
    dev = mb.Device("tiny")
    dev.add_region(mb.Region("a", "Active", 0.0, 1e-6))
    e0 = rng.standard_normal(nx) * 1e9
    h0 = rng.standard_normal(nx) * 1e3
    a = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    rho0 = a @ a.conj().T
    rho0 /= np.trace(rho0).real
    sce = mb.Scenario("one", nx, 0.5 * (1e-6 / (nx - 1)) / mb.C0, mb.QmOperator.from_matrix(rho0),
                      ic_e_field=mb.CurveField(e0), ic_h_field=mb.CurveField(h0))
    sce.add_record(mb.Record("e", quantity="e"))
    sce.add_record(mb.Record("h", quantity="h"))
    for exact in (True, False):
        s = gpu.GpuFdtdSolver(dev, sce, exact=exact)
        assert s.grid.num_t == 2
        res = {r.name: r for r in s.run()}
        cf = mb.get_fdtd_constants(dev.material_at(0.0), s.grid.dt, s.grid.dx)
        hf = np.zeros(nx + 1)
        hf[:nx] = h0
        hn = hf.copy()
        hn[1:nx] = hf[1:nx] + cf.c_prime * (e0[1:] - e0[:-1])
        import oracle as orc
        ref, _ = orc.run_oracle(s.plan)
        got_e, got_h = res["e"].data[1], res["h"].data[1]
        assert np.allclose(got_h[1:], hn[1:nx], rtol=1e-13, atol=0)
        assert got_e[0] == 0.0 and got_e[-1] == 0.0  # R = 1 mirrors
        # interior E against the oracle's stencil (bit-exact in the exact variant)
        if exact:
            assert np.array_equal(got_e, ref[0][1])
        else:
            assert np.allclose(got_e, ref[0][1], rtol=1e-12, atol=1e-6)


def test_phase_velocity_error_below_one_percent():
    """pkg/tests/test_solver.py:234-278: standing-mode phase velocity and the
    discrete dispersion relation."""
    nx, wl = 2048, 1.5e-6
    dx = wl / 20.0
    length = dx * (nx - 1)
    k = 2 * math.pi / wl
    mb.add_material(mb.Material("Vacuum"))
    dev = mb.Device("v", bc_left=mb.BoundaryReflectivity(1.0), bc_right=mb.BoundaryReflectivity(1.0))
    dev.add_region(mb.Region("v", "Vacuum", 0.0, length))
    x_e = np.arange(nx) * dx
    x_h = (np.arange(nx) - 0.5) * dx
    dt = 0.5 * dx / mb.C0
    z0 = math.sqrt(mb.MU0 / mb.EPS0)
    sce = mb.Scenario("cw", nx, 240e-15, mb.QmOperator([1.0, 0.0]),
                      ic_e_field=mb.CurveField(np.sin(k * x_e)),
                      ic_h_field=mb.CurveField(-np.sin(k * (x_h + 0.5 * mb.C0 * dt)) / z0))
    sce.add_record(mb.Record("probe", quantity="e", position=length / 2))
    r = gpu.GpuFdtdSolver(dev, sce).run()[0]
    trace, times = r.data[:, 0], r.times
    good = times < (length / 2) / mb.C0
    trace, times = trace[good], times[good]
    cross = []
    for i in range(1, trace.size):
        if trace[i - 1] < 0.0 <= trace[i] or trace[i - 1] >= 0.0 > trace[i]:
            f = trace[i - 1] / (trace[i - 1] - trace[i])
            cross.append(times[i - 1] + f * (times[i] - times[i - 1]))
    cross = np.array(cross)
    assert cross.size > 40
    period = 2.0 * np.mean(np.diff(cross))
    assert abs((2 * math.pi / period) / k - mb.C0) / mb.C0 <= 0.01
    omega_num = (2.0 / dt) * math.asin(0.5 * math.sin(k * dx / 2.0))
    assert abs(2 * math.pi / period - omega_num) / omega_num < 2e-3


# ---------------------------------------------------------------- C ABI details

def _cfg2_small(nx=1 << 14, steps=600, stress=True):
    from paper_2005_05412_b200 import configs

    mb.clear_material_library()
    return configs.cfg2(mb, nx=nx, steps=steps, stress=stress, cells=(16, nx // 2, nx - 17))


def test_event_marks_time_the_advance():
    import ctypes as C

    dev, sce = _cfg2_small(stress=False)
    s = gpu.GpuFdtdSolver(dev, sce)
    h = s.open_handle()
    s.upload_initial_state(h)
    h.call("mbg_mark", 0)
    h.call("mbg_sample", 0)
    h.call("mbg_mark", 1)
    h.call("mbg_advance", 1, s.grid.num_t - 1)
    h.call("mbg_mark", 2)
    part, total = C.c_float(0), C.c_float(0)
    h.call("mbg_mark_elapsed", 1, 2, C.byref(part))
    h.call("mbg_mark_elapsed", 0, 2, C.byref(total))
    assert 0.0 < part.value <= total.value
    with pytest.raises(gpu.NativeError):
        h.call("mbg_mark_elapsed", 0, 7, C.byref(part))  # slot never recorded
    h.close()


def test_zero_field_upload_is_a_memset():
    """mbg_upload_fields(NULL, NULL) == uploading explicit zero arrays; a half
    NULL pair is an argument error."""
    from paper_2005_05412_b200 import native

    dev, sce = _cfg2_small(stress=False)
    a = gpu.GpuFdtdSolver(dev, sce)
    assert a.plan.fields_zero
    ra = a.run()
    b = gpu.GpuFdtdSolver(dev, sce)
    h = b.open_handle()
    e, hf = np.zeros(b.grid.num_x), np.zeros(b.grid.num_x + 1)
    h.call("mbg_upload_fields", native.ptr(e), native.ptr(hf))
    h.call("mbg_upload_density", native.ptr(native.f64(b.plan.rho_init_packed())))
    with pytest.raises(gpu.NativeError):
        h.call("mbg_upload_fields", native.ptr(e), None)
    b._ran = True
    b._run_on(h)
    rb = b.download_results(h)
    h.close()
    for x, y in zip(ra, rb):
        assert np.array_equal(x.data, y.data), x.name


@pytest.mark.parametrize("exact", [False, True])
def test_state_round_trip_through_the_relaxed_frame(exact):
    """The fast two-level path keeps (X, Y, Z) = pre-relaxation vectors on the
    device; uploads map in, downloads map out: a round trip returns the state
    to rounding (bitwise in the exact variant, which keeps the reference's form)."""
    from paper_2005_05412_b200 import native

    dev, sce = _cfg2_small()
    s = gpu.GpuFdtdSolver(dev, sce, exact=exact)
    h = s.open_handle()
    s.upload_initial_state(h)
    nx, w = s.grid.num_x, s.plan.state_words
    rng = np.random.default_rng(3)
    planes = np.zeros((w, nx))
    cells = np.concatenate([np.arange(lo, hi) for lo, hi, _ in s.plan.groups])
    v = rng.normal(size=(3, cells.size))
    v *= 0.9 / np.linalg.norm(v, axis=0)
    planes[:, cells] = v
    h.call("mbg_upload_state", native.ptr(native.f64(planes)))
    back = np.zeros_like(planes)
    h.call("mbg_download_state", native.ptr(back))
    h.close()
    if exact:
        assert np.array_equal(back, planes)
    else:
        assert np.max(np.abs(back - planes)) <= 1e-15


@pytest.mark.parametrize("case", ["sit_hard_whole", "multi_material", "rand3_split", "four_media_rk4", "cfg2_r16"])
@pytest.mark.parametrize("segment", [1, 37, 1000])
def test_streamed_records_equal_resident_records(case, segment):
    """Records streamed through a device window of rows (copied to the host
    after every segment of `segment` steps) equal the HBM-resident records bit
    for bit, for point and whole-domain, real and complex records."""
    dev, sce, stepper = build_case(case)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    mb.clear_material_library()
    dev, sce, stepper = build_case(case)
    got = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, record_segment=segment).run()
    for a, b in zip(ref, got):
        assert a.name == b.name and a.data.shape == b.data.shape
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), (case, segment, a.name)


def test_records_stream_automatically_past_the_device_budget(monkeypatch):
    from paper_2005_05412_b200 import solver as S

    dev, sce, stepper = build_case("sit_hard_whole")
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    monkeypatch.setattr(S, "RECORD_HBM_BYTES", 1 << 10)
    monkeypatch.setattr(S, "RECORD_SEGMENT_BYTES", 1 << 16)
    mb.clear_material_library()
    dev, sce, stepper = build_case("sit_hard_whole")
    sol = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    assert sol._segment_steps() >= 1024
    got = sol.run()
    assert sol._streamed
    for a, b in zip(ref, got):
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


def test_advance_refuses_rows_outside_the_device_window():
    from paper_2005_05412_b200 import native

    dev, sce, stepper = build_case("sit_hard_whole")
    sol = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    h = sol.open_handle()
    try:
        sol.upload_initial_state(h)
        every = sol.plan.plans[0].every
        h.call("mbg_set_record_rows", 0, 2)  # rows 0 and 1 resident
        h.call("mbg_sample", 0)
        h.call("mbg_advance", 1, every)  # writes row 1: fine
        with pytest.raises(native.NativeError):
            h.call("mbg_advance", every + 1, every)  # would write row 2
        with pytest.raises(native.NativeError):
            h.call("mbg_download_record", 0, native.ptr(np.zeros(10)), None)
    finally:
        h.close()


def test_streamed_records_with_the_invariant_monitor():
    """Segments end on monitor steps: same records and the same invariant
    report as the resident run."""
    dev, sce, stepper = build_case("rand3_split")
    a = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, monitor_invariants=True)
    ra = a.run()
    mb.clear_material_library()
    dev, sce, stepper = build_case("rand3_split")
    b = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, monitor_invariants=True, record_segment=37)
    rb = b.run()
    assert b._streamed
    for x, y in zip(ra, rb):
        assert np.array_equal(x.data, y.data), x.name
    assert a.invariant_report == b.invariant_report


def test_two_level_equivalence_bloch_vs_three_level_kernel():
    """The reference's 2-level equivalence check (test_acceptance.py:163-190:
    Bloch form vs the generic N-level step) across the GPU's two kernel
    families: a two-level medium run by the Bloch kernel and the same medium
    embedded in three levels (an isolated, empty third level) run by the
    N-level kernel, 10^4 steps, E and the two-level block within 1e-9."""
    qm2 = mb.two_level_description(1e24, 2 * math.pi * 2e14, 6.24e-11, 1e11, 1e12, -1.0)
    h0 = np.zeros(3)
    h0[:2] = np.real(np.diag(qm2.hamiltonian.matrix()))
    mu_off = np.zeros(3, dtype=complex)
    mu_off[0] = qm2.dipole_op.matrix()[0, 1]  # pair (0, 1) first in storage order
    rates = np.zeros((3, 3))
    rates[:2, :2] = qm2.dissipator.rates
    deph = np.zeros(3)
    deph[0] = 1e12 - 0.5 * 1e11
    qm3 = mb.QmDescription(1e24, mb.QmOperator(h0), mb.QmOperator(np.zeros(3), mu_off),
                           mb.LindbladRelaxation(rates, deph))

    def build(qm, rho0, tag):
        mb.clear_material_library()
        mb.add_material(mb.Material("Vacuum"))
        mb.add_material(mb.Material("Act" + tag, qm=qm))
        dev = mb.Device("eq")
        dev.add_region(mb.Region("l", "Vacuum", 0.0, 7.5e-6))
        dev.add_region(mb.Region("a", "Act" + tag, 7.5e-6, 142.5e-6))
        dev.add_region(mb.Region("r", "Vacuum", 142.5e-6, 150e-6))
        dt0 = 0.5 * (150e-6 / 1023) / mb.C0
        sce = mb.Scenario("s", 1024, 10000 * dt0 * (1 - 1e-12), mb.QmOperator(rho0))
        sce.add_source(mb.SechPulse("s", 0.0, "hard", 4.2186e9, 2e14, 10.0, 2e14))
        sce.add_record(mb.Record("e", quantity="e", interval=50 * dt0))
        for i, j in ((1, 1), (2, 2), (1, 2)):
            sce.add_record(mb.Record(f"d{i}{j}", quantity="d", i=i, j=j, interval=50 * dt0))
        return gpu.GpuFdtdSolver(dev, sce)

    two = build(qm2, [1.0, 0.0], "2")
    three = build(qm3, [1.0, 0.0, 0.0], "3")
    assert two.grid.num_t - 1 == 10000 and three.plan.levels == 3
    ra, rb = two.run(), three.run()
    for a, b in zip(ra, rb):
        scale = np.max(np.abs(a.data))
        assert np.max(np.abs(a.data - b.data)) <= 1e-9 * scale, (a.name, np.max(np.abs(a.data - b.data)) / scale)


@pytest.mark.parametrize("case", ["sit_hard_whole", "multi_material", "cfg2_r16"])
def test_fused_two_level_monitor_equals_stepwise_numpy(case):
    """The two-level step kernels fold the monitor themselves (mbg_set_monitor):
    the report equals numpy's eigenvalues (1 - |v|)/2 of the state downloaded
    at every monitored step of a stepwise run (_kernels.py:541-546)."""
    from paper_2005_05412_b200 import native

    dev, sce, stepper = build_case(case)
    fused = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, monitor_invariants=True)
    fused.run()
    mb.clear_material_library()
    dev, sce, stepper = build_case(case)
    s = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    every = min(p.every for p in s.plan.plans)
    cells = np.concatenate([np.arange(lo, hi) for lo, hi, _ in s.plan.groups])
    h = s.open_handle()
    mins = []
    try:
        s.upload_initial_state(h)
        h.call("mbg_sample", 0)
        words = np.zeros((3, s.grid.num_x))
        n = 0
        while True:
            h.call("mbg_download_state", native.ptr(words))
            v = words[:, cells]
            mins.append(0.5 * (1.0 - np.max(np.sqrt(np.sum(v * v, axis=0)))))
            if n + every > s.grid.num_t - 1:
                break
            h.call("mbg_advance", n + 1, every)
            n += every
    finally:
        h.close()
    rep = fused.invariant_report
    assert rep["max_trace_dev"] == 0.0 and rep["max_herm_dev"] == 0.0
    assert rep["min_eigenvalue"] == pytest.approx(min(mins), abs=1e-15)


@pytest.mark.parametrize("records", [False, True])
@pytest.mark.parametrize("persistent", [None, True, False])
def test_monitor_report_equals_the_reference_solver(records, persistent):
    """The invariant report of a two-level run with and without records
    (record-less: the reference's default cadence of 256 steps,
    solver_fdtd.py:302-304) equals the reference solver's own report for the
    same objects, whichever launch path runs the steps."""
    dev, sce = _sit_small(2048, 40e-15)
    sce.add_source(mb.SechPulse("sech", 0.0, "hard", 4.2186e9, 2e14, 10.0, 2e14))
    if records:
        sce.add_record(mb.Record("inv", quantity="inv", interval=1.3e-15))
    ref = mb.FdtdSolver(dev, sce, monitor_invariants=True, threads=4)
    ref.run()
    s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce, monitor_invariants=True, persistent=persistent,
                         tile_steps=16)
    s.run()
    want, got = ref.invariant_report, s.invariant_report
    assert got["max_trace_dev"] == want["max_trace_dev"] and got["max_herm_dev"] == want["max_herm_dev"]
    assert got["min_eigenvalue"] == pytest.approx(want["min_eigenvalue"], abs=1e-12)


def test_monitor_without_quantum_media_keeps_the_initial_report():
    mb.add_material(mb.Material("Vacuum"))
    dev = mb.Device("v")
    dev.add_region(mb.Region("v", "Vacuum", 0.0, 20e-6))
    sce = mb.Scenario("s", 512, 10e-15, mb.QmOperator([1.0, 0.0]))
    sce.add_source(mb.SechPulse("sech", 0.0, "soft", 1e9, 2e14, 5.0, 1e15))
    ref = mb.FdtdSolver(dev, sce, monitor_invariants=True, threads=1)
    ref.run()
    s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce, monitor_invariants=True)
    s.run()
    assert s.invariant_report == ref.invariant_report == {"max_trace_dev": 0.0, "max_herm_dev": 0.0,
                                                          "min_eigenvalue": math.inf}


@pytest.mark.gpu
def test_fp64_operand_probes_order_as_the_register_file_model_says():
    """bench.py's roofline denominators: DFMAs with a uniform operand reach the
    pipe's peak, three distinct register operands cost three register-file
    cycles per instruction (about 2/3 of it), a shared multiplier lies between."""
    import ctypes as C

    from paper_2005_05412_b200 import native

    lib = native.load()
    rate = {}
    for mode in (1, 2, 3):
        v = C.c_double(0)
        assert lib.mbg_fp64_peak_operands(0, mode, C.byref(v)) == 0
        rate[mode] = v.value
    peak = C.c_double(0)
    assert lib.mbg_fp64_peak(0, C.byref(peak)) == 0
    assert 20.0 < rate[3] < rate[2] < rate[1] < 45.0
    assert abs(peak.value - rate[1]) < 0.05 * rate[1]
    assert 0.6 < rate[3] / rate[1] < 0.75
    assert lib.mbg_fp64_peak_operands(0, 7, C.byref(peak)) != 0  # unknown pattern
