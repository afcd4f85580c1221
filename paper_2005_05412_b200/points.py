"""Batched single-grid-point runs.

At one grid point the reference solver does not update the field
(``_phase2`` returns for ``num_x == 1``, solver_fdtd.py:347-349): E^n is the
initial value plus the sources applied in scenario order (hard = overwrite,
soft = add, solver_fdtd.py:366-385), so it is known before the run.  A batch
of such master-equation problems -- a sweep over pulse areas, detunings,
relaxation rates -- then runs as one launch with one GPU thread per system
(``mbg_batch_points``), each system stepped by the same cell functions as the
solver.  ``run_points(problems)`` returns, per problem, the list of
``Result`` objects ``GpuFdtdSolver(device, scenario).run()`` returns.

All problems share the stepper, the number of levels, the time grid and the
record layout; their quantum materials are free (up to MBG_MAX_BATCH_QM
distinct ones: the constant sets live in device memory, one per medium).
Equal sources are sampled once per call (a caller-owned sample cache, see
plan._cached_samples).
"""

from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

from . import native
from .reference import core, mblight

SolverError = mblight.SolverError
from .plan import QUANTITY_CODES, build_plan, unpack_density
from .solver import GpuFdtdSolver

MBG_Q_E, MBG_Q_H, MBG_Q_D, MBG_Q_INV = (QUANTITY_CODES[k] for k in ("e", "h", "d", "inv"))
# wall time of the last batch's native call (host setup -- one plan per system,
# the sources sampled with the reference's own Source.value -- excluded)
LAST_RUN: dict = {}


def _field_sequence(plan) -> np.ndarray:
    """E^n, n = 0..num_t-1, at the single grid point (solver_fdtd.py:362-389):
    every step applies the sources in scenario order to the previous E.  The
    last hard source of the list resets E each step, so E^n = its value plus
    the soft sources after it; without hard sources E accumulates -- the
    same sequential additions as the reference, as one running sum."""
    nt = plan.grid.num_t
    vals, hard = plan.src_values, np.asarray(plan.src_hard, dtype=bool)
    e = np.empty(nt)
    e[0] = plan.e_init[0]
    if nt == 1:
        return e
    if hard.any():
        last = int(np.flatnonzero(hard)[-1])
        cur = vals[1:, last].copy()
        for k in range(last + 1, len(hard)):
            cur = cur + vals[1:, k]
        e[1:] = cur
        return e
    if len(hard) == 0:
        e[1:] = e[0]
        return e
    seq = np.concatenate([[e[0]], vals[1:, :].reshape(-1)])  # step-major, sources in order
    run = np.add.accumulate(seq)
    e[1:] = run[len(hard)::len(hard)]
    return e


def _sample_columns(plan):
    """The shared (cached) sample column of each source of a plan, or None."""
    from .plan import _cached_samples

    g = plan.grid
    return [_cached_samples(s, g.dt, g.num_t, plan.sample_cache) for s in plan.sources]


def cache_ok(plan) -> bool:
    """Every source of the plan has a shared cached sample column (so equal
    columns are the same object and the field sequence can be shared)."""
    return plan.sample_cache is not None and all(c is not None for c in _sample_columns(plan))


def _check_finite(e: np.ndarray, num_t: int) -> None:
    """The reference's scan (every 1024 steps and the last, solver_fdtd.py:386-388)."""
    steps = np.arange(1, num_t)
    scan = steps[(steps % 1024 == 0) | (steps == num_t - 1)]
    bad = scan[~np.isfinite(e[scan])]
    if bad.size:
        raise SolverError(f"non-finite electric field at step {int(bad[0])}")


def vector_samples(src, dt: float, num_t: int):
    """Source.value(n dt), n = 0..num_t-1, as one numpy evaluation, for the
    reference's two frozen pulse types (None for any other source): the
    expressions of SechPulse.value / GaussianPulse.value (core.py:296-300,
    320-324; the sech in the overflow-safe exp form of core.py:251-254) in the
    same operation order, with numpy's exp/cos in place of libm's -- so each
    sample is within an ulp or two of the reference's (tests/test_points_host.py),
    not bit-identical.  Opt-in: ``run_points(..., fast_sources=True)``."""
    if type(src) not in (core.SechPulse, core.GaussianPulse):
        return None
    t = np.arange(num_t) * dt
    phase = np.cos(2.0 * math.pi * src.carrier_freq * t - src.carrier_phase)
    if type(src) is core.SechPulse:
        e = np.exp(-np.abs(src.envelope_rate * t - src.envelope_shift))
        return src.amplitude * (2.0 * e / (1.0 + e * e)) * phase
    arg = (t - src.peak_time) / src.width
    return src.amplitude * np.exp(-arg * arg) * phase


def run_points(problems, stepper: str = "splitting", *, exact: bool = False, gpu: int = 0, seed=None,
               fast_sources: bool = False):
    """Run many single-grid-point (device, scenario) problems in one launch.

    ``fast_sources``: sample the reference's pulse types with one numpy
    evaluation per source (:func:`vector_samples`, within an ulp or two of
    Source.value) instead of one Python call per step -- for sweeps over the
    pulses themselves, where the per-call sampling dominates the host time."""
    problems = list(problems)
    if not problems:
        return []
    t_host = time.perf_counter()
    cache: dict = {}  # equal pulses of the sweep sampled once
    qm_cache: dict = {}  # one constant set per quantum description
    plans = [build_plan(dev, sce, stepper, seed, cache, qm_cache) for dev, sce in problems]
    if fast_sources:
        for p in plans:
            cols = [vector_samples(src, p.grid.dt, p.grid.num_t) for src in p.sources]
            if cols and all(c is not None for c in cols):
                buf = p.src_buffer
                for k, c in enumerate(cols):
                    buf[1:, k] = c[1:]  # row 0 unused (solver_fdtd.py:379-385 samples n >= 1)
                p.sampled_to = p.grid.num_t
    p0 = plans[0]
    if any(p.grid.num_x != 1 for p in plans):
        raise ValueError("run_points takes single-grid-point scenarios (num_gridpoints == 1)")
    if p0.levels < 2:
        raise ValueError("run_points needs a quantum medium at the grid point")
    layout = [(r.quantity, r.i, r.j, r.every) for r in p0.plans]
    for p in plans[1:]:
        if (p.levels, p.grid.num_t) != (p0.levels, p0.grid.num_t) or p.grid.dt != p0.grid.dt:
            raise ValueError("run_points: every problem needs the same levels and time grid")
        if [(r.quantity, r.i, r.j, r.every) for r in p.plans] != layout:
            raise ValueError("run_points: every problem needs the same record layout")
    # distinct quantum materials (by id) -> constant sets of the batch
    media, index, medium = [], {}, []
    for p in plans:
        mid = p.materials[0].id
        if mid not in index:
            index[mid] = len(media)
            media.append(p.qm[0])
        medium.append(index[mid])
    if len(media) > native.MAX_BATCH_QM:
        raise ValueError(f"run_points supports at most {native.MAX_BATCH_QM} distinct quantum materials")

    B, nt = len(plans), p0.grid.num_t
    # E^n per system, built system-major (contiguous rows) and transposed once;
    # systems with the same initial field and the same (shared, cached) source
    # samples have the same sequence, computed once
    seq_b = np.empty((B, nt))
    memo: dict = {}
    for b, p in enumerate(plans):
        key = None
        if not fast_sources and cache_ok(p):
            key = (float(p.e_init[0]), tuple(id(c) for c in _sample_columns(p)), tuple(p.src_hard.tolist()))
        row = memo.get(key) if key is not None else None
        if row is None:
            row = _field_sequence(p)
            _check_finite(row, nt)
            if key is not None:
                memo[key] = row
        seq_b[b] = row
    e_seq = np.ascontiguousarray(seq_b.T)
    words = p0.state_words
    state = np.empty((words, B))
    for b, p in enumerate(plans):
        state[:, b] = p.rho_init_packed()

    # a num_x = 1 handle carrying the media; the first problem's solver builds it
    solver = GpuFdtdSolver(*problems[0], stepper=stepper, exact=exact, gpu=gpu, seed=seed)
    h = solver.open_handle()
    try:
        for q, qc in enumerate(media):
            solver._upload_qm(h, q, qc)
        dens = [r for r, pl in enumerate(p0.plans) if pl.quantity in (MBG_Q_D, MBG_Q_INV)]
        outs = {r: (np.zeros((B, p0.plans[r].rows)),
                    np.zeros((B, p0.plans[r].rows)) if p0.plans[r].is_complex else None) for r in dens}
        q = native.i32([p0.plans[r].quantity for r in dens] or [0])
        ii = native.i32([p0.plans[r].i for r in dens] or [0])
        jj = native.i32([p0.plans[r].j for r in dens] or [0])
        ev = native.i64([p0.plans[r].every for r in dens] or [1])
        re_ptrs = (native._dp * max(1, len(dens)))(*[native.ptr(outs[r][0]) for r in dens])
        im_ptrs = (native._dp * max(1, len(dens)))(*[native.ptr(outs[r][1]) if outs[r][1] is not None
                                                     else native._dp() for r in dens])
        med = native.i32(medium)
        es = np.ascontiguousarray(e_seq)
        t0 = time.perf_counter()
        LAST_RUN["host_setup_s"] = t0 - t_host  # plans, media, field sequences, handle
        h.call("mbg_batch_points", B, native.ptr(med, native._i32p), native.ptr(es), native.ptr(state),
               len(dens), native.ptr(q, native._i32p), native.ptr(ii, native._i32p), native.ptr(jj, native._i32p),
               native.ptr(ev, native._i64p), C.cast(re_ptrs, C.POINTER(native._dp)),
               C.cast(im_ptrs, C.POINTER(native._dp)))
        LAST_RUN["batch_s"] = time.perf_counter() - t0  # the C call: copies in, kernel, copies out
        LAST_RUN["systems"], LAST_RUN["steps"] = B, nt - 1
    finally:
        h.close()

    t1 = time.perf_counter()
    results = []
    for b, p in enumerate(plans):
        res = []
        for r, pl in enumerate(p.plans):
            rows = pl.rows
            if pl.quantity == MBG_Q_E:
                data = seq_b[b, ::pl.every][:rows, None].copy()
            elif pl.quantity == MBG_Q_H:
                data = np.full((rows, 1), p.h_init[0])
            else:
                re, im = outs[r]
                col = re[b] + 1j * im[b] if im is not None else re[b].copy()
                col[0] = _initial_entry(p, pl)  # row 0: the initial state (solver_fdtd.py:449)
                data = col[:, None]
            res.append(pl.to_result(p.grid, data))
        results.append(res)
    LAST_RUN["host_results_s"] = time.perf_counter() - t1
    return results


def _initial_entry(plan, rec):
    """Row 0 of a density record, read from the packed initial state the way
    the sample kernel reads a cell (bloch_entry / packed Hermitian words)."""
    w = plan.rho_init_packed()
    n, i, j = plan.levels, rec.i, rec.j
    if n == 2 and plan.stepper == "splitting":
        x, y, z = w
        if rec.quantity == MBG_Q_INV:
            return -z
        if i == j:
            return 0.5 * (1.0 + z) if i == 0 else 0.5 * (1.0 - z)
        return complex(0.5 * x, 0.5 * -y if i == 0 else 0.5 * y)
    if rec.quantity == MBG_Q_INV:
        return w[1] - w[0]
    rho = unpack_density(w[:, None], n, plan.stepper)[0]
    return rho[i, j] if i != j else rho[i, i].real
