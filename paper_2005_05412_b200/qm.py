"""N-level quantum description and the host-side precompute of the stepper.

This is the part of the reference's quantum layer (``mblight/quantum.py``)
that the time-stepping core consumes: Hermitian operators in packed form,
the Lindblad relaxation model, and the one-time relaxation propagator
(``precompute_relaxation_propagator``, ``quantum.py:408-422``) that the GPU
kernels receive as constants.  The per-cell stepping itself lives in the
CUDA kernels (``csrc/``); nothing here runs inside the time loop.

Arithmetic that feeds kernel constants (rate matrices, the Taylor/squaring
exponential, the decay factors) is evaluated in the same order as the
reference so the constants are bit-identical to the ones ``mblight``
hands its numba kernels.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from .constants import E0, HBAR

__all__ = [
    "triangle_pairs",
    "QmOperator",
    "LindbladRelaxation",
    "QmDescription",
    "PropagatorWorkspace",
    "two_level_description",
    "matrix_exponential",
    "precompute_relaxation_propagator",
]


def triangle_pairs(dim: int) -> list[tuple[int, int]]:
    """Upper-triangle (i<j) pairs in operator storage order: column by column.

    ``quantum.py:48-55``: dim=3 gives (0,1), (0,2), (1,2).
    """
    out = []
    for col in range(1, dim):
        out.extend((row, col) for row in range(col))
    return out


class QmOperator:
    """Hermitian operator: real main diagonal + complex upper triangle.

    Same storage contract as ``QmOperator`` (``quantum.py:58-131``).
    """

    def __init__(self, main_diag, off_diag=None):
        diag = np.atleast_1d(np.asarray(main_diag, dtype=float))
        if diag.ndim != 1 or diag.size == 0:
            raise ValueError("main_diag must be a non-empty 1-d real vector")
        self.main_diag = diag
        n_upper = diag.size * (diag.size - 1) // 2
        if off_diag is None:
            self.off_diag = np.zeros(n_upper, dtype=complex)
        else:
            upper = np.atleast_1d(np.asarray(off_diag, dtype=complex))
            if upper.shape != (n_upper,):
                raise ValueError(
                    f"off_diag has length {upper.size}, expected {n_upper} "
                    f"for a {diag.size}x{diag.size} operator"
                )
            self.off_diag = upper

    @property
    def dim(self) -> int:
        return int(self.main_diag.size)

    def matrix(self) -> np.ndarray:
        full = np.diag(self.main_diag.astype(complex))
        for idx, (r, c) in enumerate(triangle_pairs(self.dim)):
            full[r, c] = self.off_diag[idx]
            full[c, r] = np.conj(self.off_diag[idx])
        return full

    @classmethod
    def from_matrix(cls, m) -> "QmOperator":
        m = np.asarray(m)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("expected a square matrix")
        n = m.shape[0]
        upper = np.array([m[r, c] for r, c in triangle_pairs(n)], dtype=complex)
        return cls(np.real(np.diag(m)), upper if n > 1 else None)

    def density_problems(self) -> list[str]:
        """Violations of the density-matrix invariants (``quantum.py:106-121``)."""
        issues = []
        tr = float(np.sum(self.main_diag))
        if abs(tr - 1.0) > 1e-12:
            issues.append(f"density matrix trace is {tr!r}, expected 1")
        d = self.main_diag
        if np.any(d < -1e-12) or np.any(d > 1 + 1e-12):
            issues.append("density matrix populations must lie in [0, 1]")
        if np.min(np.linalg.eigvalsh(self.matrix())) < -1e-10:
            issues.append("density matrix is not positive semidefinite")
        return issues

    def __eq__(self, other):
        if not isinstance(other, QmOperator):
            return NotImplemented
        return np.array_equal(self.main_diag, other.main_diag) and np.array_equal(
            self.off_diag, other.off_diag
        )

    def __repr__(self):
        return f"QmOperator(dim={self.dim})"


def _traceless_diagonal_basis(n: int) -> np.ndarray:
    """Generalized Gell-Mann diagonal set, one row per operator."""
    rows = np.zeros((n - 1, n))
    for k in range(1, n):
        s = 1.0 / np.sqrt(k * (k + 1))
        rows[k - 1, :k] = s
        rows[k - 1, k] = -k * s
    return rows


class LindbladRelaxation:
    """Scattering-rate matrix + pure dephasing (``quantum.py:134-226``).

    ``rates[i][j]`` is the rate into level i from level j.  Derived members
    used by the stepper: ``pop_matrix`` (rates minus the inverse lifetimes
    on the diagonal) and ``dephasing_matrix`` (total decay per coherence).
    """

    def __init__(self, rates, pure_dephasing):
        r = np.asarray(rates, dtype=float)
        if r.ndim != 2 or r.shape[0] != r.shape[1]:
            raise ValueError("rates must be a square matrix")
        n = r.shape[0]
        offdiag = ~np.eye(n, dtype=bool)
        if np.any(r[offdiag] < 0):
            raise ValueError("scattering rates must be non-negative")
        gp = np.atleast_1d(np.asarray(pure_dephasing, dtype=float))
        if gp.shape != (n * (n - 1) // 2,):
            raise ValueError(
                f"pure_dephasing has length {gp.size}, expected {n * (n - 1) // 2}"
            )
        if np.any(gp < 0):
            raise ValueError("pure dephasing rates must be non-negative")
        self.dim = n
        self.rates = np.where(offdiag, r, 0.0)
        self.pure_dephasing = gp
        self.tau_inv = self.rates.sum(axis=0)
        self.pop_matrix = self.rates - np.diag(self.tau_inv)
        deph = 0.5 * (self.tau_inv[:, None] + self.tau_inv[None, :])
        for idx, (a, b) in enumerate(triangle_pairs(n)):
            deph[a, b] += gp[idx]
            deph[b, a] += gp[idx]
        np.fill_diagonal(deph, 0.0)
        self.dephasing_matrix = deph
        self.coeff_matrix, self.psd_ok = self._lindblad_coefficients()
        if not self.psd_ok:
            warnings.warn(
                "pure dephasing rates are not representable by a positive "
                "semidefinite coefficient matrix; the Lindblad form of the "
                "dissipator is not guaranteed",
                stacklevel=2,
            )

    def _lindblad_coefficients(self):
        # diagnostic only (never feeds the stepper): least-squares fit of the
        # pure dephasing onto the traceless diagonal operators
        n = self.dim
        if n == 1:
            return np.zeros((0, 0)), True
        basis = _traceless_diagonal_basis(n)
        pairs = triangle_pairs(n)
        design = np.array([0.5 * (basis[:, a] - basis[:, b]) ** 2 for a, b in pairs])
        coeff = np.linalg.lstsq(design, self.pure_dephasing, rcond=None)[0]
        scale = np.linalg.norm(self.pure_dephasing)
        resid = np.linalg.norm(design @ coeff - self.pure_dephasing)
        fits = resid <= 1e-6 * scale if scale > 0 else True
        floor = -1e-9 * max(float(np.max(coeff, initial=0.0)), 1.0)
        return np.diag(coeff), bool(fits and np.min(coeff) >= floor)

    def apply(self, rho: np.ndarray) -> np.ndarray:
        rho = np.asarray(rho)
        if rho.shape != (self.dim, self.dim):
            raise ValueError(
                f"density matrix has shape {rho.shape}, expected ({self.dim}, {self.dim})"
            )
        out = -self.dephasing_matrix * rho
        np.fill_diagonal(out, self.pop_matrix @ np.diagonal(rho))
        return out

    def __eq__(self, other):
        if not isinstance(other, LindbladRelaxation):
            return NotImplemented
        return np.array_equal(self.rates, other.rates) and np.array_equal(
            self.pure_dephasing, other.pure_dephasing
        )


@dataclass
class QmDescription:
    """Carrier density + H0 + dipole operator + relaxation (``quantum.py:243-270``)."""

    density_3d: float
    hamiltonian: QmOperator
    dipole_op: QmOperator
    dissipator: LindbladRelaxation

    def __post_init__(self):
        dims = {self.hamiltonian.dim, self.dipole_op.dim, self.dissipator.dim}
        if len(dims) != 1:
            raise ValueError(f"operator dimensions differ: {sorted(dims)}")
        if not self.density_3d > 0:
            raise ValueError("density_3d must be positive")

    @property
    def dim(self) -> int:
        return self.hamiltonian.dim


def two_level_description(
    density_3d, transition_freq, dipole_length, rate_scattering, rate_dephasing,
    equilibrium_inversion,
) -> QmDescription:
    """Classic two-level medium (``quantum.py:273-308``)."""
    g1, g2, w0 = rate_scattering, rate_dephasing, equilibrium_inversion
    if g2 < g1 / 2:
        raise ValueError(
            "dephasing rate must be at least half the scattering rate "
            "(implied pure dephasing would be negative)"
        )
    if abs(w0) > 1:
        raise ValueError("equilibrium inversion must lie in [-1, 1]")
    half_e = 0.5 * HBAR * transition_freq
    h0 = QmOperator([-half_e, half_e])
    mu = QmOperator([0.0, 0.0], [-E0 * dipole_length])
    rates = 0.5 * g1 * np.array([[0.0, 1.0 - w0], [1.0 + w0, 0.0]])
    return QmDescription(density_3d, h0, mu, LindbladRelaxation(rates, [g2 - 0.5 * g1]))


_TAYLOR_TERMS = 18
_NORM_TARGET = 0.5


def matrix_exponential(a: np.ndarray) -> np.ndarray:
    """exp(a): scale by 2^-s to 1-norm <= 0.5, Horner Taylor-18, square s times.

    Same algorithm and evaluation order as ``quantum.py:319-340`` so the
    relaxation constants match the reference bit for bit.
    """
    a = np.asarray(a)
    n = a.shape[0]
    ident = np.eye(n, dtype=a.dtype if np.iscomplexobj(a) else float)
    nrm = np.linalg.norm(a, 1)
    if nrm == 0.0:
        return ident.copy()
    s = max(0, int(np.ceil(np.log2(nrm / _NORM_TARGET))))
    x = a / (2.0**s)
    acc = ident + x / _TAYLOR_TERMS
    for k in range(_TAYLOR_TERMS - 1, 0, -1):
        acc = ident + (x / k) @ acc
    for _ in range(s):
        acc = acc @ acc
    return acc


@dataclass
class PropagatorWorkspace:
    """Relaxation action over dt/2: ``pop_half`` (stochastic) and ``coh_half``."""

    dim: int
    dt: float
    pop_half: np.ndarray
    coh_half: np.ndarray


def precompute_relaxation_propagator(desc: QmDescription, dt: float) -> PropagatorWorkspace:
    """Field-free relaxation half step (``quantum.py:408-422``)."""
    if not dt > 0:
        raise ValueError("dt must be positive")
    rel = desc.dissipator
    pop = matrix_exponential(rel.pop_matrix * (0.5 * dt))
    if np.min(pop) < -1e-12:
        raise ValueError("population propagator has significant negative entries")
    pop = np.maximum(pop, 0.0)
    coh = np.exp(-rel.dephasing_matrix * (0.5 * dt))
    np.fill_diagonal(coh, 0.0)
    return PropagatorWorkspace(desc.dim, dt, pop, coh)
