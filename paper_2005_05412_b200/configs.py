"""The five BASELINE.json workloads, built through the public setup API.

Every builder takes an ``api`` namespace -- this package, or the reference
``mblight`` module itself -- and returns ``(device, scenario)``.  The same
function therefore produces the scenario the GPU solver runs, the one the CPU
oracle runs, and (in this container only) the one the reference solver runs
to generate golden records.  The interpretations of items BASELINE.json leaves
open follow SURVEY.md section 8(d) (record cells, source parameters, the
splitmix64-drawn initial inversion of cfg 2, the seeded six-level medium).

``nx``/``steps`` overrides produce the reduced-grid parity variants; the
simulated window is always ``steps`` time steps (end time = steps * dt0 *
(1 - 1e-12), so ``ceil`` lands on exactly ``steps``).
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

RECORD_EVERY = 100


def _api_constants(api):
    return api.HBAR, api.E0


def _end_time(api, dev, nx, steps):
    c_max = max(m.light_speed for m in dev.materials())
    dx = dev.length / (nx - 1)
    dt0 = 0.5 * dx / c_max
    return steps * dt0 * (1.0 - 1e-12)


def _add_records(api, dev, sce, cells, quantities):
    grid = api.init_fdtd_simulation(dev, sce)
    interval = RECORD_EVERY * grid.dt
    for c in cells:
        for q in quantities:
            if q == "e":
                rec = api.Record(f"e@{c}", quantity="e", interval=interval, position=c * grid.dx)
            elif q == "h":
                rec = api.Record(f"h@{c}", quantity="h", interval=interval, position=c * grid.dx)
            elif q == "inv":
                rec = api.Record(f"inv@{c}", quantity="inv", interval=interval, position=c * grid.dx)
            else:  # "dIJ"
                i, j = int(q[1]), int(q[2])
                rec = api.Record(f"d{i}{j}@{c}", quantity="d", i=i, j=j, interval=interval,
                                 position=c * grid.dx)
            sce.add_record(rec)
    return grid


def sit_medium(api, gamma1=0.0, gamma2=0.0):
    """Two-level SIT medium of cfg 1/2."""
    _, e0 = _api_constants(api)
    return api.two_level_description(1e24, 2.0 * math.pi * 2e14, 1.0276e-29 / e0, gamma1, gamma2, -1.0)


def sit_source(api):
    hbar, _ = _api_constants(api)
    beta = 2e14
    amp = 2.0 * hbar * beta / 1.0276e-29  # pulse area 2 pi
    return api.SechPulse("sech", position=0.0, kind="soft", amplitude=amp, carrier_freq=2e14,
                         envelope_shift=20.0, envelope_rate=beta)


def cfg1(api, nx=32768, steps=None, cells=(2000, 4000, 6000), tag=""):
    """Two-level SIT, 150 um, vacuum | medium | vacuum, R = 1, soft sech source."""
    vac = api.ensure_material(api.Material("Vacuum"))
    act = api.ensure_material(api.Material("SIT_2lvl" + tag, qm=sit_medium(api)))
    dev = api.Device("cfg1")
    dev.add_region(api.Region("vacuum left", vac.id, 0.0, 7.5e-6))
    dev.add_region(api.Region("medium", act.id, 7.5e-6, 142.5e-6))
    dev.add_region(api.Region("vacuum right", vac.id, 142.5e-6, 150e-6))
    end = 200e-15 if steps is None else _end_time(api, dev, nx, steps)
    sce = api.Scenario("cfg1", nx, end, api.QmOperator([1.0, 0.0]))
    sce.add_source(sit_source(api))
    _add_records(api, dev, sce, cells, ("e", "d11", "d22", "inv"))
    return dev, sce


def cfg2_rho0(api):
    u = float(_splitmix(api)(0xB10C, 1)[0])
    return api.QmOperator([(1.0 - u) / 2.0, (1.0 + u) / 2.0])


def _splitmix(api):
    # the reference keeps it private as core._splitmix64_stream
    fn = getattr(api, "splitmix64_uniform", None)
    if fn is None:
        from importlib import import_module
        fn = import_module(api.__name__ + ".core")._splitmix64_stream
    return fn


def cfg2(api, nx=1 << 22, steps=20000, cells=None, stress=False, tag="", replicas=1,
         quantities=("e", "d11", "d22", "inv")):
    """cfg 1 lengthened to 2^22 cells with T1 = 1 ns, T2 = 1 ps, drawn inversion.

    ``replicas`` G > 1 builds the weak-scaling variant: G copies of the 150 um
    device side by side (each vacuum | medium | vacuum) on nx = 2^22 * G
    cells, so dx and dt stay (almost exactly) fixed and every slab of the
    G-way partition holds the same mix of medium and vacuum cells as cfg 2."""
    vac = api.ensure_material(api.Material("Vacuum"))
    act = api.ensure_material(api.Material("SIT_2lvl_relax" + tag, qm=sit_medium(api, 1e9, 1e12)))
    dev = api.Device("cfg2")
    unit = 150e-6
    x0 = 0.0
    for j in range(replicas):
        # each copy starts exactly where the previous one ended (the device
        # refuses gaps/overlaps, and unit * j need not equal that end in fp64)
        sfx = f" {j}" if replicas > 1 else ""
        x1, x2, x3 = x0 + 7.5e-6, x0 + unit - 7.5e-6, x0 + unit
        dev.add_region(api.Region("vacuum left" + sfx, vac.id, x0, x1))
        dev.add_region(api.Region("medium" + sfx, act.id, x1, x2))
        dev.add_region(api.Region("vacuum right" + sfx, vac.id, x2, x3))
        x0 = x3
    ic_e = api.RandomField(1e7, seed=7) if stress else None
    sce = api.Scenario("cfg2", nx, _end_time(api, dev, nx, steps), cfg2_rho0(api), ic_e_field=ic_e)
    sce.add_source(sit_source(api))
    if cells is None:
        cells = (16, nx // 2, nx - 17) if stress else (16, 4096, 8192)
    _add_records(api, dev, sce, cells, quantities)
    return dev, sce


def lambda_medium(api):
    hbar, _ = _api_constants(api)
    h0 = api.QmOperator(2.0 * math.pi * hbar * np.array([0.0, 0.2e14, 2.1e14]))
    mu = api.QmOperator([0.0, 0.0, 0.0], [0.0, 1e-29, 5e-30])
    rates = np.zeros((3, 3))
    rates[0, 2] = 1e11
    rates[1, 2] = 1e10
    rates[0, 1] = rates[1, 0] = 1e9
    relax = api.LindbladRelaxation(rates, [1e12, 1e12, 1e12])
    return api.QmDescription(5e23, h0, mu, relax)


def cfg3(api, nx=1 << 23, steps=50000, cells=None, stress=False, tag=""):
    """Three-level Lambda medium in 4 alternating sections, two-colour Gaussian source."""
    act = api.ensure_material(api.Material("Lambda3" + tag, rel_permittivity=1.0, qm=lambda_medium(api)))
    pas = api.ensure_material(api.Material("Passive12.96", rel_permittivity=12.96))
    length = 150e-6
    dev = api.Device("cfg3")
    q = length / 4
    for k, mat in enumerate((act, pas, act, pas)):
        dev.add_region(api.Region(f"s{k}", mat.id, k * q, (k + 1) * q if k < 3 else length))
    ic_e = api.RandomField(1e7, seed=11) if stress else None
    sce = api.Scenario("cfg3", nx, _end_time(api, dev, nx, steps), api.QmOperator([1.0, 0.0, 0.0]),
                       ic_e_field=ic_e)
    for f in (1.9e14, 2.1e14):
        sce.add_source(api.GaussianPulse(f"g{f:.1e}", position=0.0, kind="soft", amplitude=1e9,
                                         carrier_freq=f, peak_time=0.75e-15, width=0.25e-15))
    if cells is None:
        off = nx // 2048  # 4096 at the full 2^23 grid
        cells = (off, nx // 2 + off, 3 * (nx // 4) + off) if stress else (4096, 12288, 20000)
    _add_records(api, dev, sce, cells, ("e", "d11", "d22", "d33"))
    return dev, sce


def qcl6_medium(api, seed=4, real=False):
    """Seeded six-level QCL-like medium (draw order of SURVEY 8(d) cfg 4).
    ``real``: drop the imaginary parts of the drawn couplings (same draws; a
    real-Hamiltonian twin of the medium for timing the real-operator path)."""
    hbar, _ = _api_constants(api)
    rng = np.random.default_rng(seed)
    unit = 2.0 * math.pi * hbar
    spacing = rng.uniform(1e12, 4e12, 5) * unit
    energies = np.concatenate([[0.0], np.cumsum(spacing)])
    off_h = (rng.standard_normal(15) + 1j * rng.standard_normal(15)) * unit * 1e11
    if real:
        off_h = off_h.real.astype(complex)
    mu_nn = rng.uniform(1e-28, 5e-28, 5)
    rates = 10.0 ** rng.uniform(10, 12, (6, 6))
    np.fill_diagonal(rates, 0.0)
    pairs = [(i, j) for j in range(1, 6) for i in range(j)]  # storage order
    off_mu = np.zeros(15, dtype=complex)
    for k, (i, j) in enumerate(pairs):
        if j == i + 1:
            off_mu[k] = mu_nn[i]
    return api.QmDescription(
        5e21, api.QmOperator(energies, off_h), api.QmOperator(np.zeros(6), off_mu),
        api.LindbladRelaxation(rates, np.full(15, 1e12)))


def cfg4(api, nx=1 << 24, steps=100000, cells=None, length=2e-3, tag="", real=False):
    """Six-level QCL-like cavity, eps_r 12.96, R = 0.3, noise-seeded field."""
    act = api.ensure_material(api.Material("QCL6" + tag + ("r" if real else ""), rel_permittivity=12.96,
                                           qm=qcl6_medium(api, real=real)))
    dev = api.Device("cfg4", bc_left=api.BoundaryReflectivity(0.3), bc_right=api.BoundaryReflectivity(0.3))
    dev.add_region(api.Region("cavity", act.id, 0.0, length))
    rho0 = np.zeros(6)
    rho0[2] = 1.0
    sce = api.Scenario("cfg4", nx, _end_time(api, dev, nx, steps), api.QmOperator(rho0),
                       ic_e_field=api.RandomField(1e4, seed=7))
    if cells is None:
        cells = (1, nx // 2, nx - 2)
    _add_records(api, dev, sce, cells, ("e", "d33"))
    return dev, sce


def cfg5(api, gpus=1, steps=20000, tag=""):
    """Weak-scaling slab of cfg 4's medium: 2^22 cells and 0.5 mm per GPU."""
    return cfg4(api, nx=(1 << 22) * gpus, steps=steps, length=0.5e-3 * gpus, tag=tag)


CONFIGS = SimpleNamespace(cfg1=cfg1, cfg2=cfg2, cfg3=cfg3, cfg4=cfg4, cfg5=cfg5)
