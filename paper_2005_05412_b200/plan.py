"""Host-side setup of one run: everything the fused GPU kernels consume.

The constructor of the reference solver (``FdtdSolver.__init__``,
``mblight/solver_fdtd.py:207-326``) minus the time loop and the state arrays.
Everything that is a function or class of the reference is called, not
restated: validation (``scenario_validate``), grid sizing
(``init_fdtd_simulation``, ``solver_fdtd.py:80-102``), per-material
coefficients (``get_fdtd_constants``, ``solver_fdtd.py:122-133``), record
schedules (``_RecordPlan``, ``solver_fdtd.py:136-172``), the worker count
(``_resolve_threads``) and the stepper constants, read from the reference's
own kernel objects built for one cell (``BlochSplittingKernel`` /
``VectorSplittingKernel`` / ``VectorRk4Kernel``, ``_kernels.py:340-560``).
What remains here is the layout the GPU needs instead of the reference's
per-cell arrays.

Where the reference stores per-cell coefficient arrays (32 B/cell read
every step), the plan keeps a *region table*: region r covers E cells
[e_start[r], e_start[r+1]) and H nodes [h_start[r], h_start[r+1]); the
kernels look coefficients up by region, so no coefficient bytes cross HBM.
The tables are derived from the very same ``searchsorted`` maps the
reference builds (``solver_fdtd.py:242-272``), so the per-cell values are
identical.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .reference import core, kernels, mblight, solver_fdtd

COURANT_NUMBER = solver_fdtd.COURANT_NUMBER
NONFINITE_CHECK_EVERY = solver_fdtd._NONFINITE_CHECK_EVERY
QUANTITY_CODES = {"e": 0, "h": 1, "d": 2, "inv": 3}
STEPPERS = ("splitting", "rk4")

GridLayout = solver_fdtd.GridLayout
CellCoefficients = solver_fdtd.CellCoefficients
init_fdtd_simulation = solver_fdtd.init_fdtd_simulation
get_fdtd_constants = solver_fdtd.get_fdtd_constants
resolve_threads = solver_fdtd._resolve_threads


class RecordPlan:
    """Sampling schedule of one record: the reference's ``_RecordPlan``
    (``solver_fdtd.py:136-172``: every, rows, cell, cols, x0, the host
    buffer and ``to_result``) plus the kernels' quantity code and 0-based
    density indices."""

    def __init__(self, record, grid):
        self.ref = solver_fdtd._RecordPlan(record, grid, grid.num_t)
        self.record = record
        self.every, self.rows, self.cell = self.ref.every, self.ref.rows, self.ref.cell
        self.cols, self.x0 = self.ref.cols, self.ref.x0
        self.quantity = QUANTITY_CODES[record.quantity]
        self.i = record.i - 1 if record.quantity == "d" else 0
        self.j = record.j - 1 if record.quantity == "d" else 0
        self.is_complex = bool(record.is_complex)

    @property
    def buffer(self) -> np.ndarray:
        """The reference's host buffer of this record (rows x cols, float or complex)."""
        return self.ref.buffer

    def to_result(self, grid, data=None):
        """The reference's ``Result`` (``_RecordPlan.to_result``) over ``data``
        (default: the plan's own buffer)."""
        if data is not None:
            self.ref.buffer = data
        return self.ref.to_result(grid)


def state_words(levels: int, stepper: str = "splitting") -> int:
    """fp64 planes per quantum cell: Bloch (x, y, z) for two-level splitting,
    Hermitian-packed N^2 otherwise (N real diagonal planes, then re/im planes of
    the upper triangle in row-major i<j order)."""
    if levels == 0:
        return 0
    if levels == 2 and stepper == "splitting":
        return 3
    return levels * levels


def upper_pairs_rowmajor(n: int) -> list[tuple[int, int]]:
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def pack_density(rho: np.ndarray, stepper: str = "splitting") -> np.ndarray:
    """Density matrix -> per-cell state vector in the kernels' plane order."""
    rho = np.asarray(rho, dtype=complex)
    n = rho.shape[0]
    if n == 2 and stepper == "splitting":
        # Bloch vector (_kernels.py:496-500)
        return np.array([2.0 * rho[0, 1].real, -2.0 * rho[0, 1].imag, (rho[0, 0] - rho[1, 1]).real])
    out = [rho[i, i].real for i in range(n)]
    for i, j in upper_pairs_rowmajor(n):
        out.extend((rho[i, j].real, rho[i, j].imag))
    return np.array(out, dtype=float)


def unpack_density(words: np.ndarray, n: int, stepper: str = "splitting") -> np.ndarray:
    """Inverse of :func:`pack_density` on a (words, cells) array -> (cells, n, n).

    The two-level Bloch form maps back with the accessor formulas of
    ``_kernels.py:530-536``.
    """
    words = np.asarray(words, dtype=float)
    cells = words.shape[1]
    rho = np.zeros((cells, n, n), dtype=complex)
    if n == 2 and stepper == "splitting":
        x, y, z = words
        rho[:, 0, 0] = 0.5 * (1.0 + z)
        rho[:, 1, 1] = 0.5 * (1.0 - z)
        rho[:, 0, 1] = 0.5 * (x - 1j * y)
        rho[:, 1, 0] = 0.5 * (x + 1j * y)
        return rho
    for i in range(n):
        rho[:, i, i] = words[i]
    for p, (i, j) in enumerate(upper_pairs_rowmajor(n)):
        v = words[n + 2 * p] + 1j * words[n + 2 * p + 1]
        rho[:, i, j] = v
        rho[:, j, i] = np.conj(v)
    return rho


@dataclass
class QmConstants:
    """Stepper constants of one quantum material (host precompute, uploaded once)."""

    levels: int
    pol_factor: float
    # dipole entries driving the polarisation (_kernels.py:360-374)
    pol_i: np.ndarray
    pol_j: np.ndarray
    pol_v: np.ndarray
    pol_di: np.ndarray
    pol_dv: np.ndarray
    # Bloch form, N == 2 splitting (_kernels.py:472-494)
    bloch: dict | None = None
    # dense splitting, N >= 3 (_kernels.py:433-439)
    pop_half: np.ndarray | None = None
    coh_half: np.ndarray | None = None
    b_const: np.ndarray | None = None
    b_field: np.ndarray | None = None
    # RK4 (_kernels.py:554-557)
    h0: np.ndarray | None = None
    mu: np.ndarray | None = None
    pop_matrix: np.ndarray | None = None
    deph_matrix: np.ndarray | None = None


def qm_constants(desc, dt: float, stepper: str) -> QmConstants:
    """The stepper constants of one medium, read from the reference's own
    kernel object for it (built for one cell; nothing is stepped): the
    polarisation entries (``_kernels.py:360-374``), the Bloch constants
    (``BlochSplittingKernel.__init__``, ``_kernels.py:467-494``), the
    relaxation half step and the affine Cayley operands
    (``VectorSplittingKernel.__init__``, ``_kernels.py:431-439``) or the RK4
    operators (``VectorRk4Kernel.__init__``, ``_kernels.py:554-557``)."""
    n = desc.dim
    if stepper == "rk4":
        k = kernels.VectorRk4Kernel(desc, dt, 1)
    elif n == 2:
        k = kernels.BlochSplittingKernel(desc, dt, 1)
    else:
        k = kernels.VectorSplittingKernel(desc, dt, 1)
    qc = QmConstants(
        levels=n,
        pol_factor=k._pol_factor,
        pol_i=k._pol_i.astype(np.int32),
        pol_j=k._pol_j.astype(np.int32),
        pol_v=k._pol_v,
        pol_di=k._pol_di.astype(np.int32),
        pol_dv=k._pol_dv,
    )
    if stepper == "rk4":
        qc.h0 = np.asarray(k._h0, dtype=complex)
        qc.mu = np.asarray(k._mu, dtype=complex)
        qc.pop_matrix = np.asarray(k._pop, dtype=float)
        qc.deph_matrix = np.asarray(k._deph, dtype=float)
    elif n == 2:
        # the argument list _bloch_step_range receives (_kernels.py:505-528)
        qc.bloch = dict(
            kz=k._kz, cz=k._cz, fxy=k._fxy,
            ax_c=k._ax[0], ax_s=k._ax[1], ay_c=k._ay[0], ay_s=k._ay[1],
            az_c=k._az[0], az_s=k._az[1], a0_c=k._a0[0], a0_s=k._a0[1],
            mu_x=k._mu01.real, mu_y=-k._mu01.imag, mu_z=k._mu_zdiff,
        )
    else:
        qc.pop_half = k.pop_half
        qc.coh_half = k.coh_half
        qc.b_const = k._b_const
        qc.b_field = k._b_field
    return qc


@dataclass
class RegionTable:
    e_start: np.ndarray  # int64[R]: first E cell of region r
    h_start: np.ndarray  # int64[R]: first H node (1..Nx-1) of region r
    coef_a: np.ndarray
    coef_bg: np.ndarray
    coef_bdx: np.ndarray
    coef_ch: np.ndarray
    qm_index: np.ndarray  # int32[R]; -1 = classical material

    def per_cell(self, num_x: int) -> dict:
        """Expand to the reference's per-cell arrays (tests / oracle)."""
        e_reg = np.searchsorted(self.e_start, np.arange(num_x), side="right") - 1
        out = dict(
            coef_a=self.coef_a[e_reg], coef_bg=self.coef_bg[e_reg],
            coef_bdx=self.coef_bdx[e_reg], cell_region=e_reg,
        )
        ch = np.zeros(num_x + 1)
        if num_x > 1:
            m = np.arange(1, num_x)
            h_reg = np.searchsorted(self.h_start, m, side="right") - 1
            ch[1:num_x] = self.coef_ch[h_reg]
        out["coef_ch"] = ch
        return out


@dataclass
class SolverPlan:
    grid: GridLayout
    seed: int
    stepper: str
    levels: int  # N of the quantum materials, 0 if none
    regions: RegionTable
    qm: list
    groups: list  # (start, stop, qm_index)
    rho_init: np.ndarray  # complex N x N (or None)
    src_cells: np.ndarray
    src_hard: np.ndarray
    plans: list
    boundary: tuple  # ((w, c dt/dx, Z) left, (...) right) or None
    materials: list = field(default_factory=list)
    # the initial fields are identically zero (the scenario's default
    # ConstantField(0)): the upload is a device memset instead of a copy
    fields_zero: bool = False
    sources: list = field(default_factory=list)
    # initial fields: built by the scenario's own IC objects; a ConstantField
    # (which cannot fail) is built only when first read
    ic_fields: tuple = (None, None)
    _e_init: np.ndarray | None = None
    _h_init: np.ndarray | None = None
    # source samples [num_t, n_src] (row n = Source.value(n dt)), filled on
    # demand: the GPU run samples them segment by segment while the device
    # steps the previous segment (the reference calls Source.value inside its
    # time loop, solver_fdtd.py:379-385); sampled_to = rows [0, sampled_to) done
    _src_values: np.ndarray | None = None
    sampled_to: int = 1
    sample_cache: dict | None = None

    @property
    def state_words(self) -> int:
        return state_words(self.levels, self.stepper)

    def rho_init_packed(self) -> np.ndarray:
        if self.levels == 0:
            return np.zeros(0)
        return pack_density(self.rho_init, self.stepper)

    @property
    def e_init(self) -> np.ndarray:
        if self._e_init is None:
            self._e_init = np.ascontiguousarray(self.ic_fields[0].build(self.grid.num_x, self.seed), dtype=float)
        return self._e_init

    @property
    def h_init(self) -> np.ndarray:
        """num_x + 1 entries, the last one 0 (solver_fdtd.py:238-239)."""
        if self._h_init is None:
            nx = self.grid.num_x
            h = np.zeros(nx + 1)
            h[0:nx] = self.ic_fields[1].build(nx, self.seed + 1)
            self._h_init = h
        return self._h_init

    @property
    def src_buffer(self) -> np.ndarray:
        """The [num_t, n_src] sample table (rows past ``sampled_to`` not filled yet)."""
        if self._src_values is None:
            self._src_values = np.zeros((self.grid.num_t, len(self.sources)))
        return self._src_values

    def sample_sources(self, hi: int) -> tuple[int, int]:
        """Fill sample rows up to ``hi`` (exclusive) with each source's own
        ``value(n dt)``; returns the rows [lo, hi) filled by this call."""
        buf = self.src_buffer
        lo = self.sampled_to
        hi = min(int(hi), self.grid.num_t)
        if hi <= lo:
            return lo, lo
        dt = self.grid.dt
        for k, s in enumerate(self.sources):
            full = _cached_samples(s, dt, self.grid.num_t, self.sample_cache)
            if full is not None:
                buf[lo:hi, k] = full[lo:hi]
                continue
            col = buf[:, k]
            for n in range(lo, hi):
                col[n] = s.value(n * dt)
        self.sampled_to = hi
        return lo, hi

    @property
    def src_values(self) -> np.ndarray:
        """Every source sample (solver_fdtd.py:378-385), rows 1..num_t-1 (row 0 unused)."""
        self.sample_sources(self.grid.num_t)
        return self.src_buffer


def _cached_samples(src, dt: float, num_t: int, cache: dict | None):
    """Shared samples of equal sources across the plans of one sweep
    (``cache`` owned by the caller, e.g. one ``run_points`` call), for the two
    frozen pulse types the reference defines; None when not cacheable."""
    if cache is None or type(src) not in (core.SechPulse, core.GaussianPulse):
        return None
    key = (type(src), src, dt, num_t)  # frozen dataclasses: hashable by value
    col = cache.get(key)
    if col is None:
        col = np.zeros(num_t)
        for n in range(1, num_t):
            col[n] = src.value(n * dt)
        col.flags.writeable = False
        cache[key] = col
    return col


def _first_at_or_after(end: float, dx: float, lo: int, hi: int, offset: float = 0.0) -> int:
    """Smallest m in [lo, hi] with fl((m - offset) * dx) >= end (hi if none):
    the count of grid positions (np.arange(..) - offset) * dx below ``end``,
    which is what ``searchsorted(region_ends, x, side='right')`` compares
    (solver_fdtd.py:245-266).  The positions are monotone in m, so a guess
    from the division is corrected by exact comparisons of the same products."""
    def x(m):
        return (float(m) - offset) * dx

    if not end > x(lo):
        return lo
    m = min(max(int(math.ceil(end / dx + offset)), lo), hi)
    while m > lo and x(m - 1) >= end:
        m -= 1
    while m < hi and x(m) < end:
        m += 1
    return m


def build_plan(device, scenario, stepper: str = "splitting", seed=None, sample_cache: dict | None = None,
               qm_cache: dict | None = None) -> SolverPlan:
    """Validate and precompute a run (``FdtdSolver.__init__`` minus state
    arrays, same checks in the same order).  ``sample_cache``: see
    :func:`_cached_samples`; ``qm_cache``: a caller-owned dict that shares
    the stepper constants of one quantum description across the plans of a
    sweep (``run_points``).

    Nothing here is O(Nx) for the default zero initial fields: the region
    table comes from the region ends by exact comparisons of the reference's
    own grid positions (no per-cell map), and the source samples are taken
    when the run needs them."""
    problems = core.scenario_validate(device, scenario)
    if problems:
        raise mblight.ValidationError(problems)
    if stepper not in STEPPERS:
        raise ValueError(f"unknown stepper {stepper!r}")
    grid = init_fdtd_simulation(device, scenario)
    seed = core.DEFAULT_SEED if seed is None else int(seed)
    nx, dt, dx = grid.num_x, grid.dt, grid.dx

    # initial fields (solver_fdtd.py:235-239): the IC objects' own build(),
    # called here -- so a failing IC raises before any work -- except for the
    # constant IC, whose array is only made when it is read
    ic_e, ic_h = scenario.ic_e_field, scenario.ic_h_field
    consts = [type(ic) is core.ConstantField for ic in (ic_e, ic_h)]
    e_init = None if consts[0] else np.ascontiguousarray(ic_e.build(nx, seed), dtype=float)
    h_init = None
    if not consts[1]:
        h_init = np.zeros(nx + 1)
        h_init[0:nx] = ic_h.build(nx, seed + 1)
    fields_zero = ((ic_e.value == 0.0) if consts[0] else not e_init.any()) and \
                  ((ic_h.value == 0.0) if consts[1] else not h_init.any())

    mats = [core.get_material(r.material_id) for r in device.regions]
    n_reg = len(device.regions)
    ends = [float(r.x_end) for r in device.regions]
    if nx > 1:
        coeffs = [get_fdtd_constants(m, dt, dx) for m in mats]
        # cell m is in region min(#{ends <= m dx}, n_reg - 1), H node m in
        # min(#{ends <= (m - 1/2) dx}, n_reg - 1) (searchsorted side='right',
        # solver_fdtd.py:245-266): region r >= 1 starts at the first position
        # not below ends[r - 1]
        e_start = [0] + [_first_at_or_after(ends[r - 1], dx, 0, nx) for r in range(1, n_reg)]
        h_start = [1] + [_first_at_or_after(ends[r - 1], dx, 1, nx, 0.5) for r in range(1, n_reg)]
        h_start = [min(v, nx) for v in h_start]
    else:
        coeffs = [CellCoefficients(1.0, 0.0, 0.0, m.overlap_factor, 0.0, m.qm) for m in mats]
        e_start = [0] + [nx] * (n_reg - 1)
        h_start = [1] + [1] * (n_reg - 1)

    def region_of_cell(m):
        r = 0
        for q in range(1, n_reg):
            if e_start[q] <= m:
                r = q
        return r

    # quantum materials (one constant set per distinct qm material)
    qm_ids: list[str] = []
    qm_list: list[QmConstants] = []
    qm_index = np.full(n_reg, -1, dtype=np.int32)
    for r, m in enumerate(mats):
        if m.qm is None:
            continue
        if m.id not in qm_ids:
            qm_ids.append(m.id)
            # qm_cache (caller-owned, one sweep): the stepper constants of the
            # same quantum description at the same dt are built once
            # (the entry keeps the description alive, so its id is not reused)
            key = (id(m.qm), dt, stepper) if qm_cache is not None else None
            hit = qm_cache.get(key) if key is not None else None
            qc = hit[1] if hit is not None and hit[0] is m.qm else None
            if qc is None:
                qc = qm_constants(m.qm, dt, stepper)
                if key is not None:
                    qm_cache[key] = (m.qm, qc)
            qm_list.append(qc)
        qm_index[r] = qm_ids.index(m.id)
    levels = qm_list[0].levels if qm_list else 0

    regions = RegionTable(
        e_start=np.array(e_start, dtype=np.int64),
        h_start=np.array(h_start, dtype=np.int64),
        coef_a=np.array([c.a_prime for c in coeffs]),
        coef_bg=np.array([c.b_prime * c.gamma for c in coeffs]),
        coef_bdx=np.array([c.b_prime * c.inv_dx for c in coeffs]),
        coef_ch=np.array([c.c_prime for c in coeffs]),
        qm_index=qm_index,
    )

    # maximal runs of cells in one region (solver_fdtd.py:276-285): the
    # non-empty regions, in order
    groups = []
    bounds = e_start + [nx]
    for r in range(n_reg):
        start, stop = bounds[r], bounds[r + 1]
        if stop > start and qm_index[r] >= 0:
            groups.append((start, stop, int(qm_index[r])))

    srcs = list(scenario.sources)
    cells = [0 if nx == 1 else int(math.floor(s.position / dx + 0.5)) for s in srcs]

    plans = [RecordPlan(rec, grid) for rec in scenario.records]
    names = [p.record.name for p in plans]
    if len(set(names)) != len(names):
        raise ValueError("record names must be unique")

    boundary = None
    if nx > 1:
        left, right = mats[region_of_cell(0)], mats[region_of_cell(nx - 1)]
        boundary = (
            (1.0 - math.sqrt(device.bc_left.reflectivity), left.light_speed * dt / dx,
             math.sqrt(left.permeability / left.permittivity)),
            (1.0 - math.sqrt(device.bc_right.reflectivity), right.light_speed * dt / dx,
             math.sqrt(right.permeability / right.permittivity)),
        )

    rho0 = np.asarray(scenario.rho_init.matrix(), dtype=complex) if levels else None
    return SolverPlan(
        grid=grid, seed=seed, stepper=stepper, levels=levels,
        regions=regions, qm=qm_list, groups=groups, rho_init=rho0,
        src_cells=np.array(cells, dtype=np.int64),
        src_hard=np.array([1 if s.kind == "hard" else 0 for s in srcs], dtype=np.int32),
        plans=plans, boundary=boundary, materials=mats, fields_zero=bool(fields_zero),
        sources=srcs, ic_fields=(ic_e, ic_h), _e_init=e_init, _h_init=h_init, sample_cache=sample_cache,
    )
