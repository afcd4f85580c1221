"""Named parity cases, buildable through either setup API.

Each case is ``name -> (builder(api) -> (device, scenario), stepper)``.  The
golden generator (``tests/golden/make_golden.py``) runs them through the
reference ``mblight`` in this container; the tests rebuild the identical
setups through ``paper_2005_05412_b200`` on any box and compare.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2005_05412_b200 import configs


def _diagonal_basis(n):
    rows = np.zeros((n - 1, n))
    for k in range(1, n):
        s = 1.0 / np.sqrt(k * (k + 1))
        rows[k - 1, :k] = s
        rows[k - 1, k] = -k * s
    return rows


def random_medium(api, rng, dim, rate_scale=1e11, freq_scale=1e14, dipole_scale=1e-29, density=1e24, real=False):
    """Random valid N-level description; same draw sequence as the reference's
    test helper ``random_description`` (pkg/tests/conftest.py:49-73).  ``real``:
    the same draws with the imaginary parts of H and the dipole dropped."""
    n_off = dim * (dim - 1) // 2
    energies = np.sort(rng.uniform(0.0, 1.0, dim)) * api.HBAR * freq_scale
    off_h = (rng.standard_normal(n_off) + 1j * rng.standard_normal(n_off)) * api.HBAR * freq_scale * 0.05
    off_mu = (rng.standard_normal(n_off) + 1j * rng.standard_normal(n_off)) * dipole_scale
    if real:
        off_h, off_mu = off_h.real.astype(complex), off_mu.real.astype(complex)
    rates = rng.uniform(0.0, 1.0, (dim, dim)) * rate_scale
    np.fill_diagonal(rates, 0.0)
    basis = _diagonal_basis(dim)
    coeffs = rng.uniform(0.0, 1.0, dim - 1) * rate_scale
    pairs = [(i, j) for j in range(1, dim) for i in range(j)]
    deph = np.array([0.5 * np.sum(coeffs * (basis[:, i] - basis[:, j]) ** 2) for i, j in pairs])
    return api.QmDescription(
        density, api.QmOperator(energies, off_h), api.QmOperator(np.zeros(dim), off_mu),
        api.LindbladRelaxation(rates, deph))


def random_case(dim, seed, nx=512, end=20e-15, whole=False, stepper="splitting", real=False):
    def build(api):
        rng = np.random.default_rng(seed)
        desc = random_medium(api, rng, dim, real=real)
        act = api.ensure_material(api.Material(f"Rand{dim}_{seed}" + ("r" if real else ""), qm=desc))
        vac = api.ensure_material(api.Material("Vacuum"))
        dev = api.Device(f"rand{dim}")
        dev.add_region(api.Region("v", vac.id, 0.0, 5e-6))
        dev.add_region(api.Region("a", act.id, 5e-6, 20e-6))
        rho0 = np.zeros(dim)
        rho0[0] = 1.0
        sce = api.Scenario("s", nx, end, api.QmOperator(rho0))
        sce.add_source(api.SechPulse("sech", 0.0, "hard", 1e9, 2e14, 5.0, 1e15))
        iv = 0.0 if whole else 1e-15
        sce.add_record(api.Record("e", quantity="e", interval=iv))
        sce.add_record(api.Record("d1n", quantity="d", i=1, j=dim, interval=iv))
        sce.add_record(api.Record("d22", quantity="d", i=2, j=2, interval=iv, position=12e-6))
        sce.add_record(api.Record("dn1", quantity="d", i=dim, j=1, interval=iv, position=10e-6))
        sce.add_record(api.Record("h", quantity="h", interval=iv, position=9e-6))
        return dev, sce
    return build, stepper


def sit_hard_whole(api):
    """Ziolkowski-like SIT with a hard source; whole-domain e/inv/h records."""
    qm = api.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1.0e10, 1.0e10, -1.0)
    vac = api.ensure_material(api.Material("Vacuum"))
    act = api.ensure_material(api.Material("AR_Z", qm=qm))
    dev = api.Device("Z")
    dev.add_region(api.Region("l", vac.id, 0.0, 7.5e-6))
    dev.add_region(api.Region("a", act.id, 7.5e-6, 142.5e-6))
    dev.add_region(api.Region("r", vac.id, 142.5e-6, 150e-6))
    sce = api.Scenario("s", 1024, 150e-15, api.QmOperator([1.0, 0.0]),
                       ic_h_field=api.RandomField(1e-3, seed=5))
    sce.add_source(api.SechPulse("sech", position=0.0, kind="hard", amplitude=4.2186e9,
                                 carrier_freq=2e14, envelope_shift=10.0, envelope_rate=2e14))
    sce.add_record(api.Record("e", quantity="e", interval=5e-15))
    sce.add_record(api.Record("inv", quantity="inv", interval=5e-15))
    sce.add_record(api.Record("h", quantity="h", interval=5e-15))
    sce.add_record(api.Record("d12", quantity="d", i=1, j=2, position=30e-6))
    sce.add_record(api.Record("d21", quantity="d", i=2, j=1, position=30e-6))
    sce.add_record(api.Record("h0", quantity="h", position=0.0))
    return dev, sce


def multi_material(api):
    """Two distinct two-level media, a lossy dielectric, partial mirrors, an
    off-edge soft source, loss and overlap factors in play."""
    qa = api.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e11, 2e12, -1.0)
    qb = api.two_level_description(5e23, 2.0 * math.pi * 1.8e14, 8e-11, 1e10, 1e12, 0.5)
    vac = api.ensure_material(api.Material("Vacuum"))
    a = api.ensure_material(api.Material("MA", qm=qa))
    gl = api.ensure_material(api.Material("Glass", rel_permittivity=2.25, losses=500.0))
    b = api.ensure_material(api.Material("MB", rel_permittivity=1.5, overlap_factor=0.5, losses=1e3, qm=qb))
    dev = api.Device("multi", bc_left=api.BoundaryReflectivity(0.25), bc_right=api.BoundaryReflectivity(0.64))
    for name, mat, x0, x1 in (("v", vac, 0.0, 4e-6), ("a", a, 4e-6, 20e-6), ("g", gl, 20e-6, 26e-6),
                              ("b", b, 26e-6, 40e-6), ("v2", vac, 40e-6, 44e-6)):
        dev.add_region(api.Region(name, mat.id, x0, x1))
    sce = api.Scenario("s", 3000, 200e-15, api.QmOperator([0.9, 0.1], [0.2 - 0.1j]),
                       ic_e_field=api.RandomField(1e5, seed=3))
    sce.add_source(api.SechPulse("s1", 2e-6, "soft", 3e9, 2e14, 8.0, 1e14))
    sce.add_source(api.GaussianPulse("s2", 2e-6, "soft", 1e9, 1.8e14, 60e-15, 20e-15))
    sce.add_record(api.Record("e", quantity="e", interval=20e-15))
    sce.add_record(api.Record("inv", quantity="inv", interval=20e-15))
    for x in (1e-6, 10e-6, 23e-6, 30e-6, 43.9e-6):
        sce.add_record(api.Record(f"e@{x}", quantity="e", position=x))
        sce.add_record(api.Record(f"d12@{x}", quantity="d", i=1, j=2, position=x, interval=1e-15))
    return dev, sce


def vacuum_sources(api):
    """No quantum material: reflectivity mix, hard + soft sources, CurveField ICs."""
    vac = api.ensure_material(api.Material("Vacuum"))
    die = api.ensure_material(api.Material("Die", rel_permittivity=4.0, rel_permeability=1.2, losses=100.0))
    dev = api.Device("vac", bc_left=api.BoundaryReflectivity(0.3), bc_right=api.BoundaryReflectivity(0.7))
    dev.add_region(api.Region("v", vac.id, 0.0, 20e-6))
    dev.add_region(api.Region("d", die.id, 20e-6, 40e-6))
    nx = 1500
    x = np.arange(nx) / (nx - 1)
    sce = api.Scenario("s", nx, 300e-15, api.QmOperator([1.0, 0.0]),
                       ic_e_field=api.CurveField(np.sin(7 * np.pi * x) * 1e3),
                       ic_h_field=api.CurveField(np.cos(5 * np.pi * x)))
    sce.add_source(api.SechPulse("hard", 10e-6, "hard", 1.0, 2e14, 10.0, 2e14))
    sce.add_source(api.GaussianPulse("soft", 10e-6, "soft", 2.0, 1e14, 100e-15, 30e-15))
    sce.add_record(api.Record("e", quantity="e", interval=20e-15))
    sce.add_record(api.Record("h", quantity="h", interval=20e-15))
    sce.add_record(api.Record("edge", quantity="e", position=40e-6))
    return dev, sce


def tiny_group(api):
    """A 20-cell two-level group: the reference steps it with ScalarKernel."""
    qm = api.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e10, 1e11, -1.0)
    vac = api.ensure_material(api.Material("Vacuum"))
    act = api.ensure_material(api.Material("Tiny", qm=qm))
    dev = api.Device("tiny")
    dev.add_region(api.Region("v", vac.id, 0.0, 10e-6))
    dev.add_region(api.Region("a", act.id, 10e-6, 10.4e-6))
    dev.add_region(api.Region("v2", vac.id, 10.4e-6, 20e-6))
    sce = api.Scenario("s", 1024, 100e-15, api.QmOperator([1.0, 0.0]))
    sce.add_source(api.SechPulse("s", 0.0, "hard", 4e9, 2e14, 5.0, 2e14))
    sce.add_record(api.Record("e", quantity="e", interval=2e-15))
    sce.add_record(api.Record("inv", quantity="inv", position=10.2e-6))
    return dev, sce


CASES = {
    # BASELINE configs (full or reduced grids)
    "cfg1_full": (lambda api: configs.cfg1(api), "splitting"),
    "cfg2_r16": (lambda api: configs.cfg2(api, nx=1 << 16, steps=20000, stress=True), "splitting"),
    "cfg2_full": (lambda api: configs.cfg2(api), "splitting"),
    "cfg2_stress_full": (lambda api: configs.cfg2(api, stress=True), "splitting"),
    # the headline grid with density records inside the medium as well (its
    # first cell, the middle of the device, the last medium cell): the BASELINE
    # record cells all lie in the 7.5 um vacuum lead
    "cfg2_medium_full": (lambda api: configs.cfg2(api, cells=(16, 4096, 8192, 209716, 1 << 21, 3984587),
                                                  quantities=("e", "d11", "d22", "inv", "d12")), "splitting"),
    "cfg3_r16": (lambda api: configs.cfg3(api, nx=1 << 16, steps=50000, cells=(4096, 12288, 20000)), "splitting"),
    "cfg3_r16_stress": (lambda api: configs.cfg3(api, nx=1 << 16, steps=50000, stress=True), "splitting"),
    "cfg4_r14": (lambda api: configs.cfg4(api, nx=1 << 14, steps=100000), "splitting"),
    # feature coverage
    "sit_hard_whole": (sit_hard_whole, "splitting"),
    "multi_material": (multi_material, "splitting"),
    "vacuum_sources": (vacuum_sources, "splitting"),
    "tiny_group": (tiny_group, "splitting"),
}
for _n in (3, 4, 5, 6, 7, 8):
    CASES[f"rand{_n}_split"] = random_case(_n, 30 + _n)
for _n in (2, 3, 4):
    CASES[f"rand{_n}_rk4"] = random_case(_n, 60 + _n, stepper="rk4")
CASES["rand2_split"] = random_case(2, 32)

def song_point(api):
    """Driven V-type three-level system at a single grid point (the reference's
    song2005 parameters, setups.py:108-146): the Nx = 1 master-equation mode."""
    hb, e0 = api.HBAR, api.E0
    h0 = api.QmOperator([0.0, 2.3717e15 * hb, 2.4165e15 * hb])
    mu = api.QmOperator([0.0, 0.0, 0.0], [-e0 * 9.2374e-11, -e0 * 9.2374e-11 * math.sqrt(2.0), 0.0])
    rates = [[0.0, 1e10, 1e10], [1e10, 0.0, 1e10], [1e10, 1e10, 0.0]]
    qm = api.QmDescription(6e24, h0, mu, api.LindbladRelaxation(rates, [0.0, 0.0, 0.0]))
    act = api.ensure_material(api.Material("Song3", qm=qm))
    dev = api.Device("Song")
    dev.add_region(api.Region("point", act.id, 0.0, 0.0))
    sce = api.Scenario("s", 1, 80e-15, api.QmOperator([1.0, 0.0, 0.0]), num_timesteps=10000)
    for i in (1, 2, 3):
        sce.add_record(api.Record(f"d{i}{i}", quantity="d", i=i, j=i, position=0.0))
    sce.add_record(api.Record("d12", quantity="d", i=1, j=2, position=0.0))
    sce.add_record(api.Record("e", quantity="e", position=0.0))
    sce.add_source(api.SechPulse("sech", position=0.0, kind="hard", amplitude=3.5471e9, carrier_freq=3.8118e14,
                                 envelope_shift=17.248, envelope_rate=1.76 / 5e-15, carrier_phase=-math.pi / 2.0))
    return dev, sce


def point2(api):
    """Two-level medium at a single grid point driven by a soft source."""
    qm = api.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e11, 1e12, -1.0)
    act = api.ensure_material(api.Material("P2", qm=qm))
    dev = api.Device("p2")
    dev.add_region(api.Region("point", act.id, 0.0, 0.0))
    sce = api.Scenario("s", 1, 100e-15, api.QmOperator([1.0, 0.0]), num_timesteps=5000)
    sce.add_record(api.Record("inv", quantity="inv", position=0.0))
    sce.add_record(api.Record("d12", quantity="d", i=1, j=2, position=0.0))
    sce.add_record(api.Record("e", quantity="e", position=0.0))
    sce.add_source(api.SechPulse("s", 0.0, "soft", 4e9, 2e14, 5.0, 2e14))
    return dev, sce


def bragg_stack(api):
    """A 100-layer periodic stack (the reference's material library exists for
    such structures, core.py:1-9) around a two-level slab: 103 regions."""
    qm = api.two_level_description(1e24, 2.0 * math.pi * 2e14, 6.24e-11, 1e10, 1e11, -1.0)
    lo = api.ensure_material(api.Material("LowN", rel_permittivity=1.0))
    hi = api.ensure_material(api.Material("HighN", rel_permittivity=2.25, losses=50.0))
    act = api.ensure_material(api.Material("BraggActive", qm=qm))
    dev = api.Device("bragg", bc_left=api.BoundaryReflectivity(0.0), bc_right=api.BoundaryReflectivity(0.5))
    x = 0.0
    dev.add_region(api.Region("lead", lo.id, 0.0, 5e-6))
    x = 5e-6
    for k in range(100):
        w = 0.25e-6 if k % 2 == 0 else 0.1667e-6
        dev.add_region(api.Region(f"l{k}", (hi if k % 2 == 0 else lo).id, x, x + w))
        x = x + w
    dev.add_region(api.Region("slab", act.id, x, x + 10e-6))
    x = x + 10e-6
    dev.add_region(api.Region("tail", lo.id, x, x + 5e-6))
    sce = api.Scenario("s", 4000, 250e-15, api.QmOperator([1.0, 0.0]))
    sce.add_source(api.SechPulse("s", 1e-6, "soft", 4e9, 2e14, 8.0, 1e14))
    sce.add_record(api.Record("e", quantity="e", interval=25e-15))
    sce.add_record(api.Record("inv", quantity="inv", interval=25e-15))
    sce.add_record(api.Record("probe", quantity="e", position=3e-6))
    return dev, sce


def kernel_case(dim, seed, stepper="splitting", nx=64):
    """One time step over nx cells with random E: isolates the per-cell
    stepper (the scenario-level twin of pkg/tests/test_solver.py:437-480)."""
    def build(api):
        rng = np.random.default_rng(seed)
        desc = random_medium(api, rng, dim)
        a = rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))
        rho = a @ a.conj().T
        rho = rho / np.trace(rho).real
        e_vals = rng.uniform(-5e9, 5e9, nx)
        act = api.ensure_material(api.Material(f"K{dim}_{seed}", qm=desc))
        dev = api.Device("k")
        dev.add_region(api.Region("a", act.id, 0.0, 1e-6))
        end = 0.5 * (1e-6 / (nx - 1)) / api.C0  # exactly one step
        sce = api.Scenario("k", nx, end, api.QmOperator.from_matrix(rho), ic_e_field=api.CurveField(e_vals))
        for i in range(1, dim + 1):
            for j in range(i, dim + 1):
                sce.add_record(api.Record(f"d{i}{j}", quantity="d", i=i, j=j))
        sce.add_record(api.Record(f"d{dim}1", quantity="d", i=dim, j=1))
        sce.add_record(api.Record("e", quantity="e"))
        return dev, sce
    return build, stepper


def qcl5(api):
    """The reference's built-in tzenov2016 QCL comb setup (setups.py:212-277:
    five levels with tunnelling couplings, one laser dipole, a dense
    scattering matrix, split dephasing, losses 1100/m, overlap factor 0.9,
    mirrors R = 0.8, random initial field) at its default 4096 cells, run
    for 20 of its 200 ps.  make_golden.py checks this builder against
    builtin_setup("tzenov2016") record for record."""
    e0 = api.E0
    h_off = np.zeros(10, dtype=complex)
    h_off[1] = 1.2329e-3 * e0
    h_off[2] = -1.3447e-3 * e0
    mu_off = np.zeros(10, dtype=complex)
    mu_off[5] = -e0 * 4e-9
    rates = np.array([[0.0, 0.4947e12, 0.0974e12, 0.8116e12, 1.0410e12],
                      [0.8245e12, 0.0, 0.1358e12, 0.6621e12, 1.1240e12],
                      [0.0229e12, 0.0469e12, 0.0, 0.0794e12, 0.0357e12],
                      [0.0047e12, 0.0029e12, 0.1252e12, 0.0, 0.2810e12],
                      [0.0049e12, 0.0049e12, 0.1101e12, 0.4949e12, 0.0]])
    deph = np.full(10, 1.0 / 1.0e-12)
    deph[0] = 0.0
    deph[1] = deph[2] = 1.0 / 0.6e-12
    qm = api.QmDescription(5.6e21, api.QmOperator(np.array([0.10103, 0.09677, 0.09720, 0.08129, 0.07633]) * e0,
                                                  h_off),
                           api.QmOperator(np.zeros(5), mu_off), api.LindbladRelaxation(rates, deph))
    act = api.ensure_material(api.Material("AR_Tzenov", rel_permittivity=12.96, overlap_factor=0.9, losses=1100.0,
                                           qm=qm))
    dev = api.Device("tzenov2016", bc_left=api.BoundaryReflectivity(0.8), bc_right=api.BoundaryReflectivity(0.8))
    dev.add_region(api.Region("Active region", act.id, 0.0, 0.5e-3))
    sce = api.Scenario("basic", 4096, 20e-12, api.QmOperator([0.0, 0.0, 1.0, 0.0, 0.0]),
                       ic_e_field=api.RandomField(amplitude=3e4, seed=None))
    sce.add_record(api.Record("e0", quantity="e", position=0.0))
    sce.add_record(api.Record("e", quantity="e", interval=1e-12))
    sce.add_record(api.Record("h", quantity="h", interval=1e-12))
    return dev, sce


def ladder6(api):
    """The reference's built-in marskar2011 six-level anharmonic ladder
    (setups.py:149-209) at its default 8192 cells, run for 1.2 of its 2000 ps
    (the hard Gaussian pulse peaks at 600 fs); two probes added after the
    setup's own records."""
    levels = 6
    w0 = 2.0 * math.pi * 1e13
    energies = np.zeros(levels)
    for n in range(1, levels):
        energies[n] = energies[n - 1] + api.HBAR * w0 * (1.0 - 0.1 * (n - 3))
    n_off = levels * (levels - 1) // 2
    dipoles = np.zeros(n_off, dtype=complex)
    rates = np.zeros((levels, levels))
    k = 0
    for j in range(1, levels):
        for i in range(j):
            if j == i + 1:
                dipoles[k] = -api.E0 * 1e-10 * math.sqrt(i + 1.0)
                rates[i, j] = 1e10
            k += 1
    qm = api.QmDescription(1e24, api.QmOperator(energies), api.QmOperator(np.zeros(levels), dipoles),
                           api.LindbladRelaxation(rates, np.zeros(n_off)))
    vac = api.ensure_material(api.Material("Vacuum"))
    act = api.ensure_material(api.Material("AR_Marskar_6lvl", qm=qm))
    dev = api.Device("Marskar_6lvl")
    dev.add_region(api.Region("Vacuum left", vac.id, 0.0, 7.5e-6))
    dev.add_region(api.Region("Active region", act.id, 7.5e-6, 142.5e-6))
    dev.add_region(api.Region("Vacuum right", vac.id, 142.5e-6, 150e-6))
    rho = np.zeros(levels)
    rho[0] = 1.0
    sce = api.Scenario("Basic", 8192, 1.2e-12, api.QmOperator(rho))
    sce.add_record(api.Record("e", quantity="e", interval=1e-12))
    sce.add_record(api.Record("d11", quantity="d", i=1, j=1, interval=1e-12, position=75e-6))
    sce.add_source(api.GaussianPulse("gaussian", position=0.0, kind="hard", amplitude=1e9, carrier_freq=1e13,
                                     peak_time=600e-15, width=200e-15))
    sce.add_record(api.Record("e@20um", quantity="e", interval=10e-15, position=20e-6))
    sce.add_record(api.Record("d12@20um", quantity="d", i=1, j=2, interval=10e-15, position=20e-6))
    return dev, sce


def four_media(api):
    """Four distinct three-level media (random draws) separated by dielectric
    spacers, partial mirrors, soft source: every constant-set slot of the
    N-level kernels in use."""
    rng = np.random.default_rng(44)
    vac = api.ensure_material(api.Material("Vacuum"))
    spacer = api.ensure_material(api.Material("Spacer", rel_permittivity=2.0, losses=200.0))
    dev = api.Device("four", bc_left=api.BoundaryReflectivity(0.5), bc_right=api.BoundaryReflectivity(0.9))
    dev.add_region(api.Region("lead", vac.id, 0.0, 3e-6))
    x = 3e-6
    for m in range(4):
        desc = random_medium(api, rng, 3, rate_scale=10 ** (10 + m / 2), density=(m + 1) * 3e23)
        mat = api.ensure_material(api.Material(f"Med3_{m}", rel_permittivity=1.0 + 0.5 * m, overlap_factor=1.0 - 0.1 * m,
                                               qm=desc))
        dev.add_region(api.Region(f"m{m}", mat.id, x, x + 4e-6))
        dev.add_region(api.Region(f"s{m}", spacer.id, x + 4e-6, x + 5e-6))
        x += 5e-6
    sce = api.Scenario("s", 2400, 60e-15, api.QmOperator([0.8, 0.15, 0.05]), ic_e_field=api.RandomField(1e4, seed=9))
    sce.add_source(api.SechPulse("sech", 1e-6, "soft", 2e9, 1.5e14, 6.0, 2e14))
    sce.add_record(api.Record("e", quantity="e", interval=5e-15))
    for m in range(4):
        xm = 3e-6 + 5e-6 * m + 2e-6
        sce.add_record(api.Record(f"d13@{m}", quantity="d", i=1, j=3, position=xm, interval=0.5e-15))
        sce.add_record(api.Record(f"d22@{m}", quantity="d", i=2, j=2, position=xm, interval=0.5e-15))
    return dev, sce


# cfg3's real three-level medium under RK4 (the real-operator derivative path)
CASES["cfg3_rk4_r12"] = (lambda api: configs.cfg3(api, nx=1 << 12, steps=4000, cells=(300, 1100, 2500)), "rk4")
CASES["four_media"] = (four_media, "splitting")
CASES["four_media_rk4"] = (four_media, "rk4")

# the reference's built-in setups that the cases above do not already cover
# (ziolkowski1995 ~ cfg1, song2005 = song_point): name -> (builtin args, case)
BUILTIN_TWINS = {"qcl5": (("tzenov2016", None, 20e-12), 3), "ladder6": (("marskar2011-6lvl", None, 1.2e-12), 2)}

CASES["qcl5"] = (qcl5, "splitting")
CASES["ladder6"] = (ladder6, "splitting")
CASES["bragg_stack"] = (bragg_stack, "splitting")
CASES["song_point"] = (song_point, "splitting")
CASES["song_point_rk4"] = (song_point, "rk4")
CASES["point2"] = (point2, "splitting")
for _n in range(2, 9):
    CASES[f"kernel{_n}_split"] = kernel_case(_n, 100 + _n)
for _n in (2, 3, 4, 5):
    CASES[f"kernel{_n}_rk4"] = kernel_case(_n, 200 + _n, stepper="rk4")

# cases whose reference run takes minutes; generated once, marked slow
SLOW = {"cfg2_full", "cfg2_stress_full", "cfg2_medium_full", "cfg3_r16", "cfg3_r16_stress", "cfg4_r14"}
