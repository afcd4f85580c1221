"""Stepper accuracy properties the reference's own tests pin
(pkg/tests/test_quantum.py:391-430), here for the GPU kernels at a single
grid point under a constant field (no sources: E keeps its initial value):

* with no unitary part (H0 = 0, dipole 0) the splitting step equals the exact
  propagator of the Lindblad dissipator;
* with a random three-level medium the splitting error against the exact
  propagator falls with order 2 (and RK4's with order 4) as dt halves.

The exact solution is expm of the Liouvillian built from the plan's own
operators (scipy), independent of the stepper code.
"""

import math

import numpy as np
import pytest
from scipy.linalg import expm

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb

pytestmark = pytest.mark.gpu


def _desc(rng, dim, unitary=True):
    from cases import random_medium

    d = random_medium(mb, rng, dim, rate_scale=1e12, freq_scale=1e14, dipole_scale=1e-29)
    if unitary:
        return d
    return mb.QmDescription(d.density_3d, mb.QmOperator(np.zeros(dim)), mb.QmOperator(np.zeros(dim)),
                            d.dissipator)


def _rho0(rng, dim):
    a = rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))
    r = a @ a.conj().T
    return r / np.trace(r).real


def _exact(desc, rho0, e_field, t):
    n = rho0.shape[0]
    h = desc.hamiltonian.matrix() - e_field * desc.dipole_op.matrix()
    eye = np.eye(n)
    lv = -1j / mb.HBAR * (np.kron(h, eye) - np.kron(eye, h.T))
    pop = np.asarray(desc.dissipator.pop_matrix, dtype=float)
    deph = np.asarray(desc.dissipator.dephasing_matrix, dtype=float)
    for i in range(n):
        for j in range(n):
            if i == j:
                for k in range(n):
                    lv[i * n + i, k * n + k] += pop[i, k]
            else:
                lv[i * n + j, i * n + j] -= deph[i, j]
    return (expm(lv * t) @ rho0.reshape(-1)).reshape(n, n)


def _gpu(desc, rho0, e_field, horizon, steps, stepper, tag):
    mb.clear_material_library()
    n = rho0.shape[0]
    act = mb.ensure_material(mb.Material("Conv" + tag, qm=desc))
    dev = mb.Device("pt")
    dev.add_region(mb.Region("p", act.id, 0.0, 0.0))
    sce = mb.Scenario("s", 1, horizon, mb.QmOperator.from_matrix(rho0), num_timesteps=steps + 1,
                      ic_e_field=mb.CurveField(np.array([e_field])))
    pairs = [(i, j) for i in range(n) for j in range(i, n)]
    for i, j in pairs:
        sce.add_record(mb.Record(f"d{i}{j}", quantity="d", i=i + 1, j=j + 1, position=0.0, interval=horizon))
    res = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    out = np.zeros((n, n), complex)
    for (i, j), r in zip(pairs, res):
        out[i, j] = r.data[-1, 0]
        out[j, i] = np.conj(out[i, j])
    return out


@pytest.mark.parametrize("dim", [2, 3, 4])
def test_dissipation_only_splitting_is_exact(dim):
    rng = np.random.default_rng(9 + dim)
    desc = _desc(rng, dim, unitary=False)
    rho0 = _rho0(rng, dim)
    horizon, steps = 2e-12, 20
    got = _gpu(desc, rho0, 0.0, horizon, steps, "splitting", f"d{dim}")  # dim 2: the Bloch kernel
    assert np.allclose(got, _exact(desc, rho0, 0.0, horizon), atol=1e-13)


@pytest.mark.parametrize("stepper,order", [("splitting", 2.0), ("rk4", 4.0)])
def test_convergence_order(stepper, order):
    rng = np.random.default_rng(42)
    desc = _desc(rng, 3)
    rho0 = _rho0(rng, 3)
    e_field, horizon = 1e8, 50e-15
    exact = _exact(desc, rho0, e_field, horizon)
    errors = [np.linalg.norm(_gpu(desc, rho0, e_field, horizon, s, stepper, f"{stepper}{s}") - exact)
              for s in (64, 128, 256)]
    for k in range(2):
        assert abs(math.log2(errors[k] / errors[k + 1]) - order) <= 0.15, (stepper, errors)
