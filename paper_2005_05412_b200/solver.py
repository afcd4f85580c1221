"""GPU drop-in for the reference solver (``FdtdSolver``, solver_fdtd.py:198-498).

``GpuFdtdSolver`` keeps the reference's constructor signature, attributes and
``run()`` contract (one ``Result`` per record in record order, blocking,
``SolverError`` on a second call or on a non-finite field, validation before
any work) and replaces the hot loop with the fused sm_100a kernels of
``libmbgpu.so``.  Setup comes from :mod:`.plan`, which calls the reference's own setup
functions and kernel constructors (``FdtdSolver.__init__``), so every
coefficient the kernels see is the one the reference's numba loops see.

Registered names: ``gpu-fdtd-reg-cayley`` (splitting stepper) and
``gpu-fdtd-rk4``.  :func:`register_with_reference` adds the same names to the
reference's own registry so ``mblight.create_solver("gpu-fdtd-reg-cayley", ...)``
and the mblight CLI resolve to this solver.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time

import numpy as np

from . import native
from .plan import build_plan, resolve_threads
from .reference import core, mblight

SolverError = mblight.SolverError

SOLVER_NAMES = ("gpu-fdtd-reg-cayley", "gpu-fdtd-rk4")
# records larger than this stream through a device window of rows ...
RECORD_HBM_BYTES = 4 << 30
# ... sized so one segment's rows take about this much device memory
RECORD_SEGMENT_BYTES = 512 << 20
# first run segment when the sources are sampled during the run (see _run_on),
# and the factor by which the segments grow
FIRST_FEED = 1024
FEED_GROWTH = 4


class GpuFdtdSolver:
    """One simulation run on a B200; same protocol as the reference's ``FdtdSolver``.

    Extra keyword arguments (all optional):
      ``tile_steps`` -- time steps fused per kernel launch (k; default per N),
      ``exact``      -- disable FMA contraction (bit-exact two-level path);
                        None (default): the MBG_EXACT environment variable
                        ("1": exact), so CLI runs can ask for it too,
      ``gpu``        -- CUDA device ordinal,
      ``persistent`` -- two-level / classical runs: True = one persistent
                        wavefront launch per advance, False = one launch per
                        k steps, None (default) = the wavefront when a fused
                        chunk has at least one tile per SM,
      ``record_segment`` -- stream the records: keep only the rows of this
                        many time steps in HBM and copy completed rows into
                        the host result arrays after every segment (None:
                        automatic -- streamed when the records would take
                        more than RECORD_HBM_BYTES of device memory; 0: never).
    """

    def __init__(self, device, scenario, stepper="splitting", threads=None, seed=None,
                 monitor_invariants=False, *, tile_steps=None, exact=None, gpu=0, persistent=None,
                 record_segment=None):
        self.plan = build_plan(device, scenario, stepper, seed)
        self.device = device
        self.scenario = scenario
        self.stepper = stepper
        self.grid = self.plan.grid
        self.seed = self.plan.seed
        self.threads = resolve_threads(threads, self.grid.num_x)
        self.monitor_invariants = monitor_invariants
        self.invariant_report = None
        self.tile_steps = tile_steps
        if exact is None:
            exact = os.environ.get("MBG_EXACT", "0") == "1"
        self.exact = bool(exact)
        self.gpu = int(gpu)
        self.persistent = None if persistent is None else bool(persistent)
        self.record_segment = record_segment
        self._streamed = False
        self._fed = 0
        self.results = None
        self.launches = 0
        self.kernel_ms = None
        self._ran = False
        if len(self.plan.plans) > native.MAX_RECORDS:
            raise ValueError(f"the GPU solver supports at most {native.MAX_RECORDS} records")
        if len(self.plan.src_cells) > native.MAX_SOURCES:
            raise ValueError(f"the GPU solver supports at most {native.MAX_SOURCES} sources")
        if len(self.plan.qm) > native.MAX_QM:
            raise ValueError(f"the GPU solver supports at most {native.MAX_QM} distinct quantum materials")
        if len(self.plan.regions.e_start) > native.MAX_REGIONS:
            raise ValueError(f"the GPU solver supports at most {native.MAX_REGIONS} device regions")

    # -- device setup ------------------------------------------------------

    def _grid_struct(self, win=None, own=None):
        g = self.grid
        s = native.MbgGrid()
        s.num_x, s.num_t, s.dt, s.dx = g.num_x, g.num_t, g.dt, g.dx
        s.levels = self.plan.levels
        s.stepper = native.MBG_STEPPER[self.stepper]
        s.tile_steps = int(self.tile_steps or 0)
        s.exact = 1 if self.exact else 0
        s.device = self.gpu
        s.flags = {None: 0, True: native.MBG_FLAG_PERSISTENT, False: native.MBG_FLAG_PER_LAUNCH}[self.persistent]
        s.win_lo, s.win_hi = win if win is not None else (0, g.num_x)
        s.own_lo, s.own_hi = own if own is not None else (s.win_lo, s.win_hi)
        return s

    def open_handle(self, win=None, own=None, records=True, stream_sources=False) -> native.Handle:
        """Create the device solver and upload everything but the initial state
        (``records=False``: a handle that never samples, e.g. the edge-strip
        solvers of a slab; ``stream_sources``: the source samples not taken
        yet are uploaded by the run as it samples them, see _run_on)."""
        plan = self.plan
        h = native.Handle(self._grid_struct(win, own))
        rt = plan.regions
        keep = [native.i64(rt.e_start), native.i64(rt.h_start), native.f64(rt.coef_a), native.f64(rt.coef_bg),
                native.f64(rt.coef_bdx), native.f64(rt.coef_ch), native.i32(rt.qm_index)]
        h.call("mbg_set_regions", len(rt.e_start), native.ptr(keep[0], native._i64p),
               native.ptr(keep[1], native._i64p), *[native.ptr(a) for a in keep[2:6]],
               native.ptr(keep[6], native._i32p))
        for q, qc in enumerate(plan.qm):
            self._upload_qm(h, q, qc)
        if plan.boundary is not None:
            (wl, cl, zl), (wr, cr, zr) = plan.boundary
            h.call("mbg_set_boundary", wl, cl, zl, wr, cr, zr)
        cells, hard = native.i64(plan.src_cells), native.i32(plan.src_hard)
        if stream_sources and len(cells) and plan.sampled_to < self.grid.num_t:
            h.call("mbg_set_sources", len(cells), native.ptr(cells, native._i64p), native.ptr(hard, native._i32p),
                   None)
            if plan.sampled_to > 1:  # rows sampled before the run
                buf = plan.src_buffer
                h.call("mbg_set_source_rows", 1, plan.sampled_to, native.ptr(buf[1:plan.sampled_to]))
            self._fed = plan.sampled_to
        else:
            vals = native.f64(plan.src_values)
            h.call("mbg_set_sources", len(cells), native.ptr(cells, native._i64p), native.ptr(hard, native._i32p),
                   native.ptr(vals))
            self._fed = self.grid.num_t
        ps = plan.plans if records else []
        q = native.i32([p.quantity for p in ps])
        cell = native.i64([-1 if p.cell is None else p.cell for p in ps])
        ii, jj = native.i32([p.i for p in ps]), native.i32([p.j for p in ps])
        every = native.i64([p.every for p in ps])
        h.call("mbg_set_records", len(ps), native.ptr(q, native._i32p), native.ptr(cell, native._i64p),
               native.ptr(ii, native._i32p), native.ptr(jj, native._i32p), native.ptr(every, native._i64p))
        return h

    def _upload_qm(self, h, q, qc):
        # the numpy temporaries below stay referenced until each call returns
        if qc.bloch is not None:
            b = qc.bloch
            c = native.f64([b[k] for k in ("kz", "cz", "fxy", "ax_c", "ax_s", "ay_c", "ay_s", "az_c", "az_s",
                                           "a0_c", "a0_s", "mu_x", "mu_y", "mu_z")] + [qc.pol_factor])
            h.call("mbg_set_qm_bloch", q, native.ptr(c))
            return
        args = self._pol_args(qc)
        if qc.h0 is not None:
            mats = [native.f64(np.ascontiguousarray(qc.h0, complex).view(np.float64)),
                    native.f64(np.ascontiguousarray(qc.mu, complex).view(np.float64)),
                    native.f64(qc.pop_matrix), native.f64(qc.deph_matrix)]
            h.call("mbg_set_qm_rk4", q, *[native.ptr(m) for m in mats], *args[0])
        else:
            mats = [native.f64(qc.pop_half), native.f64(qc.coh_half),
                    native.f64(np.ascontiguousarray(qc.b_const, complex).view(np.float64)),
                    native.f64(np.ascontiguousarray(qc.b_field, complex).view(np.float64))]
            h.call("mbg_set_qm_dense", q, *[native.ptr(m) for m in mats], *args[0])

    @staticmethod
    def _pol_args(qc):
        pi = native.i32(qc.pol_i if len(qc.pol_i) else [0])
        pj = native.i32(qc.pol_j if len(qc.pol_j) else [0])
        pv = native.f64(np.asarray(qc.pol_v, dtype=complex).view(np.float64) if len(qc.pol_v) else [0.0, 0.0])
        di = native.i32(qc.pol_di if len(qc.pol_di) else [0])
        dv = native.f64(qc.pol_dv if len(qc.pol_dv) else [0.0])
        keep = (pi, pj, pv, di, dv)
        return ((len(qc.pol_i), native.ptr(pi, native._i32p), native.ptr(pj, native._i32p), native.ptr(pv),
                 len(qc.pol_di), native.ptr(di, native._i32p), native.ptr(dv), qc.pol_factor), keep)

    def upload_initial_state(self, h, win=None):
        lo, hi = win if win is not None else (0, self.grid.num_x)
        if self.plan.fields_zero:  # zero ICs: a device memset, no host copy
            h.call("mbg_upload_fields", None, None)
        else:
            e = native.f64(self.plan.e_init[lo:hi])
            hf = native.f64(self.plan.h_init[lo:hi + 1])
            h.call("mbg_upload_fields", native.ptr(e), native.ptr(hf))
        if self.plan.levels:
            w = native.f64(self.plan.rho_init_packed())
            h.call("mbg_upload_density", native.ptr(w))

    def download_results(self, h):
        """Every record into the reference's own host buffer (``_RecordPlan.buffer``)
        and out as its ``Result`` (``_RecordPlan.to_result``)."""
        out = []
        for r, p in enumerate(self.plan.plans):
            if not self._streamed:  # streamed: the rows are already in the buffer
                self._download_rows(h, r, p, 0, p.rows, whole=True)
            out.append(p.to_result(self.grid))
        return out

    @staticmethod
    def _download_rows(h, r, p, lo, hi, whole=False):
        """Rows [lo, hi) of record r into its host buffer: straight into the
        buffer for real records, through re/im halves for complex ones."""
        buf = p.buffer
        if not p.is_complex:
            dst = buf[lo:hi]
            if whole:
                h.call("mbg_download_record", r, native.ptr(dst), None)
            else:
                h.call("mbg_download_record_rows", r, lo, hi, native.ptr(dst), None)
            return
        re = np.empty((hi - lo, p.cols))
        im = np.empty((hi - lo, p.cols))
        if whole:
            h.call("mbg_download_record", r, native.ptr(re), native.ptr(im))
        else:
            h.call("mbg_download_record_rows", r, lo, hi, native.ptr(re), native.ptr(im))
        buf[lo:hi].real = re
        buf[lo:hi].imag = im

    # -- streamed records ---------------------------------------------------------

    def _segment_steps(self) -> int:
        """Steps per streamed record segment (0: records stay whole in HBM)."""
        seg = self._segment_unaligned()
        monitor = self._monitor_cadence()
        if seg and monitor is not None:  # segments end on invariant-monitor steps
            seg = max(1, seg // monitor) * monitor
        return seg

    def _segment_unaligned(self) -> int:
        if self.record_segment is not None:
            return max(0, int(self.record_segment))
        plans = self.plan.plans
        total = sum(p.rows * p.cols * (16 if p.is_complex else 8) for p in plans)
        if total <= RECORD_HBM_BYTES:
            return 0
        # rows of S steps for every record within RECORD_SEGMENT_BYTES
        per_step = sum(p.cols * (16 if p.is_complex else 8) / p.every for p in plans)
        return max(1024, int(RECORD_SEGMENT_BYTES / per_step) // 1024 * 1024)

    def _open_streams(self, h, segment):
        """Device windows of floor(S/every) + 1 rows; the host side is the
        reference's own full buffer (it keeps every row in host memory,
        solver_fdtd.py:136-172)."""
        self._streamed = True
        self._row0 = []
        for r, p in enumerate(self.plan.plans):
            cap = min(p.rows, segment // p.every + 1)
            if cap < p.rows:
                h.call("mbg_set_record_rows", r, cap)
            self._row0.append(0)

    def _drain_streams(self, h, last_step):
        """Copy every row completed up to ``last_step`` to the host and move
        each record's device window past it."""
        for r, p in enumerate(self.plan.plans):
            done = min(p.rows, last_step // p.every + 1)
            lo = self._row0[r]
            if done <= lo:
                continue
            self._download_rows(h, r, p, lo, done)
            h.call("mbg_set_record_row0", r, done)
            self._row0[r] = done

    # -- run ------------------------------------------------------------------

    def run(self):
        """Execute the run; returns one Result per record (``solver_fdtd.py:444-455``)."""
        if self._ran:
            raise SolverError("run() may only be called once per solver instance")
        self._ran = True
        h = self.open_handle(stream_sources=True)
        try:
            self.upload_initial_state(h)
            self._run_on(h)
            self.results = self.download_results(h)
        finally:
            h.close()
        return self.results

    def _run_on(self, h, poll_every: int = 1 << 14):
        """Sample row 0, then advance steps 1..num_t-1 in chunks, polling the
        device-side non-finite flag every ``poll_every`` steps and at the end
        (the device keeps the first failing scan step, so that is the one
        reported).  The invariant monitor's statistics are folded on the device
        without a host synchronisation (inside the two-level step kernels, or
        by a reduction at each monitored step) and read once at the end."""
        num_t = self.grid.num_t
        segment = self._segment_steps()
        if segment:
            self._open_streams(h, segment)
        h.call("mbg_sample", 0)
        every = self._monitor_cadence()
        if every is not None:
            h.call("mbg_invariants_accumulate")  # the initial state
        # two-level splitting: the step kernels fold the monitor at its steps
        # themselves; otherwise the run stops at each monitored step for it
        fused = every is not None and self.plan.levels == 2 and self.stepper == "splitting"
        if fused:
            h.call("mbg_set_monitor", every)
        split = None if fused else every
        chunk = poll_every if split is None else max(1, split)
        if segment:
            chunk = min(chunk, segment)  # with the monitor: a multiple of its cadence (see _segment_steps)
        # sources not sampled yet: sampled (Source.value, as the reference's
        # loop calls it per step) by a host thread while the device steps the
        # rows already there; each advance takes the rows sampled by then
        # (see _SourceSampler / _next_count).  With the monitor split the run
        # cuts at monitored steps: rows are then sampled segment by segment.
        feed = self._fed < num_t
        sampler = _SourceSampler(self.plan) if feed and split is None else None
        last = 0
        n = 1
        since = 0
        h.call("mbg_event_begin")
        try:
            while n < num_t:
                if sampler is not None:
                    cnt = self._next_count(h, sampler, n, min(chunk, num_t - n), last)
                    last = cnt
                else:
                    cnt = min(chunk, num_t - n)
                    self.plan.sample_sources(n + cnt)
                self._feed_sources(h, n + cnt)
                h.call("mbg_advance", n, cnt)
                n += cnt
                since += cnt
                if split is not None and (n - 1) % split == 0:
                    h.call("mbg_invariants_accumulate")
                if segment:
                    self._drain_streams(h, n - 1)
                if since >= poll_every or n >= num_t or segment:
                    since = 0
                    bad = C.c_int64(-1)
                    h.call("mbg_poll_nonfinite", C.byref(bad))
                    if bad.value >= 0:
                        raise SolverError(f"non-finite electric field at step {bad.value}")
        finally:
            if sampler is not None:
                sampler.stop()
        ms = C.c_float(0)
        h.call("mbg_event_end", C.byref(ms))
        self.kernel_ms = float(ms.value)
        if every is not None:
            self._read_invariants(h)
        elif self.monitor_invariants:
            # no quantum cells: the reference's report keeps its initial
            # values (solver_fdtd.py:428-434)
            self.invariant_report = {"max_trace_dev": 0.0, "max_herm_dev": 0.0, "min_eigenvalue": math.inf}
        launches = C.c_int64(0)
        h.call("mbg_launch_count", C.byref(launches))
        self.launches = int(launches.value)

    def _feed_sources(self, h, hi):
        """Queue the sampled source rows [fed, hi) for the device
        (stream-ordered before the next launch)."""
        hi = min(hi, self.plan.sampled_to)
        if hi <= self._fed:
            return
        lo = self._fed
        h.call("mbg_set_source_rows", lo, hi, native.ptr(self.plan.src_buffer[lo:hi]))
        self._fed = hi

    @staticmethod
    def _next_count(h, sampler, n, most, last):
        """Steps of the next advance from step n (at most ``most``): once the
        sampler is at least twice the last advance (and FIRST_FEED) ahead, or
        has every row up to n + most, or the device has run dry with
        FIRST_FEED rows ready -- so the device queue stays fed while the rows
        are sampled, and advances grow as fast as the sampling allows."""
        want = max(FIRST_FEED, FEED_GROWTH * last)
        idle = C.c_int32(0)
        while True:
            ready = sampler.ready()
            if ready - n >= min(want, most):
                return min(ready - n, most)
            if ready - n >= min(FIRST_FEED, most):
                h.call("mbg_stream_idle", C.byref(idle))
                if idle.value:
                    return min(ready - n, most)
            sampler.wait(n + min(want, most))

    # -- invariant monitor (solver_fdtd.py:306-308, 425-440) ---------------------

    def _monitor_cadence(self):
        if not self.monitor_invariants or not self.plan.levels:
            return None
        return min((p.every for p in self.plan.plans), default=256)

    def _read_invariants(self, h):
        """The device-side running statistics of every monitored step."""
        out = np.zeros(3)
        h.call("mbg_invariants_read", native.ptr(out))
        self.invariant_report = {"max_trace_dev": float(out[0]), "max_herm_dev": float(out[1]),
                                 "min_eigenvalue": float(out[2])}


class _SourceSampler:
    """Samples the plan's sources (Source.value, plan.sample_sources) on a
    host thread, block by block, ahead of the run; the run's thread releases
    the GIL inside every native call, so the sampling proceeds while it
    enqueues launches or waits for the device.  Errors of Source.value are
    re-raised in the run's thread."""

    BLOCK = 256

    def __init__(self, plan):
        import threading

        self.plan = plan
        plan.src_buffer  # allocated here, before the thread writes into it
        self.cv = threading.Condition()
        self.error = None
        self.stopped = False
        self.thread = threading.Thread(target=self._work, name="mbg-source-sampler", daemon=True)
        self.thread.start()

    def _work(self):
        try:
            end = self.plan.grid.num_t
            while not self.stopped and self.plan.sampled_to < end:
                self.plan.sample_sources(self.plan.sampled_to + self.BLOCK)
                with self.cv:
                    self.cv.notify_all()
                time.sleep(0)  # hand the GIL to the run's thread between blocks
        except BaseException as exc:  # noqa: BLE001  (re-raised in the run's thread)
            self.error = exc
            with self.cv:
                self.cv.notify_all()

    def ready(self) -> int:
        if self.error is not None:
            raise self.error
        return self.plan.sampled_to

    def wait(self, rows: int):
        with self.cv:
            self.cv.wait_for(lambda: self.error is not None or self.plan.sampled_to >= min(rows, self.plan.grid.num_t),
                             timeout=2e-4)
        if self.error is not None:
            raise self.error

    def stop(self):
        self.stopped = True
        self.thread.join()


def _rk4_factory(device, scenario, **kw):
    return GpuFdtdSolver(device, scenario, stepper="rk4", **kw)


def register(registry_fn=None):
    """Add the GPU solver names to the reference's solver registry
    (``core.register_solver``, core.py:617)."""
    registry_fn = core.register_solver if registry_fn is None else registry_fn
    registry_fn("gpu-fdtd-reg-cayley", GpuFdtdSolver)
    registry_fn("gpu-fdtd-rk4", _rk4_factory)


def register_with_reference(mblight_module=None):
    """Register the GPU solver names in the reference's own registry
    (``mblight.core.register_solver``, core.py:617); importing this package
    already did so for the ``mblight`` it binds to."""
    if mblight_module is None:
        mblight_module = mblight
    from importlib import import_module  # noqa: PLC0415

    register(import_module(mblight_module.__name__ + ".core").register_solver)
    return mblight_module


register()
