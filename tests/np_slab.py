"""CPU twin of one native slab (TEST DOUBLE for the gloo multi-process tests).

Implements the interface ``slabs.run_slab_rank`` drives (sample / advance /
pack_into / unpack_from / poll / records / close) on numpy arrays, so the
multi-rank host logic -- partitioning, ghost windows, neighbour exchange,
record assembly, the non-finite reduction -- is exercised on CPU with
torch.distributed/gloo.  Each step restates solver_fdtd.py:53-66 and
solver_fdtd.py:362-426 on the window with elementwise IEEE numpy arithmetic
in the reference's evaluation order; the density step is _kernels.py:200-232
in numpy for two-level splitting, and for N-level splitting / RK4 the
oracle's own per-cell step (oracle/mb_oracle.c orc_density_step) on the
window's quantum runs -- so every rank is bit-exact against the oracle.
"""

import numpy as np

from paper_2005_05412_b200.plan import NONFINITE_CHECK_EVERY


class NumpySlab:
    def __init__(self, solver, slab):
        plan = solver.plan
        self.plan, self.slab = plan, slab
        self.dense = plan.levels > 2 or (plan.levels == 2 and plan.stepper == "rk4")
        g = plan.grid
        self.nx, self.num_t = g.num_x, g.num_t
        lo, hi = slab.win_lo, slab.win_hi
        self.lo, self.hi, self.n = lo, hi, hi - lo
        self.e = plan.e_init[lo:hi].copy()
        self.h = plan.h_init[lo:hi + 1].copy()
        cells = plan.regions.per_cell(self.nx)
        self.a = cells["coef_a"][lo:hi]
        self.bg = cells["coef_bg"][lo:hi]
        self.bdx = cells["coef_bdx"][lo:hi]
        self.ch = cells["coef_ch"][lo:hi]
        qm_of_cell = plan.regions.qm_index[cells["cell_region"][lo:hi]]
        self.qm = qm_of_cell >= 0
        self.qi = np.where(self.qm, qm_of_cell, 0)
        self.x = np.zeros(self.n)
        self.y = np.zeros(self.n)
        self.z = np.zeros(self.n)
        if self.dense:
            import oracle as orc

            n = plan.levels
            self.orc = orc.OracleRun(plan, threads=1, step_limit=1)  # the plan's constants (nothing is run)
            self.rho = np.zeros((self.n, n, n), complex)
            self.rho[self.qm] = plan.rho_init
            # contiguous runs of quantum cells of one material
            self.runs = []
            l = 0
            while l < self.n:
                if not self.qm[l]:
                    l += 1
                    continue
                r = l
                while r < self.n and self.qm[r] and self.qi[r] == self.qi[l]:
                    r += 1
                self.runs.append((l, r, int(self.qi[l])))
                l = r
        elif plan.levels:
            w = plan.rho_init_packed()
            self.x[self.qm], self.y[self.qm], self.z[self.qm] = w
            keys = ("kz", "cz", "fxy", "ax_c", "ax_s", "ay_c", "ay_s", "az_c", "az_s", "a0_c", "a0_s",
                    "mu_x", "mu_y", "mu_z")
            self.bc = {k: np.array([q.bloch[k] for q in plan.qm])[self.qi] for k in keys}
            self.pf = np.array([q.pol_factor for q in plan.qm])[self.qi]
        self.words = 2 + 2 * plan.levels ** 2 if self.dense else 5
        self.bad = -1
        self.rec = []
        for p in plan.plans:
            cols = 1 if p.cell is not None else slab.own_hi - slab.own_lo
            self.rec.append([np.zeros((p.rows, cols)), np.zeros((p.rows, cols)) if p.is_complex else None])

    # -- helpers ---------------------------------------------------------------
    def _bloch(self, e):
        c = self.bc
        x0, y0, z0 = self.x, self.y, self.z
        x1, y1, z1 = c["fxy"] * x0, c["fxy"] * y0, c["kz"] * z0 + c["cz"]
        ax, ay = c["ax_c"] + c["ax_s"] * e, c["ay_c"] + c["ay_s"] * e
        az, a0 = c["az_c"] + c["az_s"] * e, c["a0_c"] + c["a0_s"] * e
        q = ax * ax + ay * ay + az * az
        u = a0 * a0
        num = 1.0 + u - q
        t1 = 1.0 + q - u
        inv = 1.0 / (t1 * t1 + 4.0 * u)
        k1 = (num * num - 4.0 * q) * inv
        g = 4.0 * num * inv
        dotb = 8.0 * inv * (ax * x1 + ay * y1 + az * z1)
        x2 = k1 * x1 + g * (ay * z1 - az * y1) + dotb * ax
        y2 = k1 * y1 + g * (az * x1 - ax * z1) + dotb * ay
        z2 = k1 * z1 + g * (ax * y1 - ay * x1) + dotb * az
        x3, y3, z3 = c["fxy"] * x2, c["fxy"] * y2, c["kz"] * z2 + c["cz"]
        p = self.pf * (c["mu_x"] * (x3 - x0) + c["mu_y"] * (y3 - y0) + c["mu_z"] * (z3 - z0))
        m = self.qm
        self.x = np.where(m, x3, x0)
        self.y = np.where(m, y3, y0)
        self.z = np.where(m, z3, z0)
        return np.where(m, p, 0.0)

    def _dense_step(self, e):
        p = np.zeros(self.n)
        for l0, l1, q in self.runs:
            st = np.ascontiguousarray(self.rho[l0:l1]).view(np.float64).reshape(-1)
            nxt = np.zeros_like(st)
            pp = np.zeros(l1 - l0)
            self.orc.density_step(q, st, nxt, np.ascontiguousarray(e[l0:l1]), pp)
            self.rho[l0:l1] = nxt.view(np.complex128).reshape(l1 - l0, *self.rho.shape[1:])
            p[l0:l1] = pp
        return p

    def _owned(self):
        return slice(self.slab.own_lo - self.lo, self.slab.own_hi - self.lo)

    # -- slab interface ----------------------------------------------------------
    def sample(self, n):
        own = self._owned()
        for (re, im), p in zip(self.rec, self.plan.plans):
            if n % p.every:
                continue
            row = n // p.every
            if p.record.quantity == "e":
                v = self.e
            elif p.record.quantity == "h":
                v = self.h[:self.n]
            elif self.dense:
                i, j = p.i, p.j
                if p.record.quantity == "inv":  # _kernels.py:391-392
                    v = np.where(self.qm, self.rho[:, 1, 1].real - self.rho[:, 0, 0].real, 0.0)
                elif i == j:
                    v = np.where(self.qm, self.rho[:, i, i].real, 0.0)
                else:
                    v = np.where(self.qm, self.rho[:, i, j], 0.0)
            elif p.record.quantity == "inv":
                v = np.where(self.qm, -self.z, 0.0)
            else:
                i, j = p.i, p.j
                if i == j:
                    v = np.where(self.qm, 0.5 * (1.0 + self.z) if i == 0 else 0.5 * (1.0 - self.z), 0.0)
                else:
                    vi = 0.5 * -self.y if i == 0 else 0.5 * self.y
                    v = np.where(self.qm, 0.5 * self.x, 0.0) + 1j * np.where(self.qm, vi, 0.0)
            if p.cell is None:
                vals = v[own]
            elif self.slab.own_lo <= p.cell < self.slab.own_hi:
                vals = v[p.cell - self.lo:p.cell - self.lo + 1]
            else:
                continue
            re[row, :] = np.real(vals)
            if im is not None:
                im[row, :] = np.imag(vals)

    def advance(self, first, count):
        plan = self.plan
        nx = self.nx
        c = np.arange(self.lo, self.hi)
        for n in range(first, first + count):
            e_old = self.e.copy()
            h_old = self.h.copy()
            hn = self.h.copy()
            upd = (c >= 1) & (c <= nx - 1)
            upd[0] = False  # no left neighbour inside the window
            l = np.nonzero(upd)[0]
            hn[l] = h_old[l] + self.ch[l] * (e_old[l] - e_old[l - 1])
            if self.dense:
                p = self._dense_step(e_old)
            else:
                p = self._bloch(e_old) if plan.levels else np.zeros(self.n)
            if nx > 1:
                en = self.a * e_old - self.bg * p + self.bdx * (hn[1:] - hn[:-1])
            else:
                en = e_old.copy()
            if plan.boundary is not None:
                (wl, cl, zl), (wr, cr, zr) = plan.boundary
                if self.lo == 0:
                    e_at = (1.0 - cl) * e_old[0] + cl * e_old[1]
                    h_at = 0.5 * (h_old[1] + hn[1])
                    en[0] = wl * 0.5 * (e_at + zl * h_at)
                if self.hi == nx:
                    e_at = (1.0 - cr) * e_old[-1] + cr * e_old[-2]
                    h_at = 0.5 * (h_old[self.n - 1] + hn[self.n - 1])
                    en[-1] = wr * 0.5 * (e_at - zr * h_at)
            for s, cell in enumerate(plan.src_cells):
                if self.lo <= cell < self.hi:
                    v = plan.src_values[n, s]
                    en[cell - self.lo] = v if plan.src_hard[s] else en[cell - self.lo] + v
            self.e, self.h = en, hn
            if (n % NONFINITE_CHECK_EVERY == 0 or n == self.num_t - 1) and self.bad < 0:
                if not np.all(np.isfinite(self.e[self._owned()])):
                    self.bad = n
            self.sample(n)

    def _pack(self, cell0, count):
        l0 = cell0 - self.lo
        sl = slice(l0, l0 + count)
        if self.dense:
            return np.concatenate([self.e[sl], self.h[sl], np.ascontiguousarray(self.rho[sl]).view(np.float64).reshape(-1)])
        return np.concatenate([self.e[sl], self.h[sl], self.x[sl], self.y[sl], self.z[sl]])

    def pack_into(self, cell0, count, tensor):
        tensor.numpy()[:] = self._pack(cell0, count)

    def unpack_from(self, cell0, count, tensor):
        buf = tensor.numpy()
        l0 = cell0 - self.lo
        sl = slice(l0, l0 + count)
        if self.dense:
            self.e[sl] = buf[:count]
            self.h[sl] = buf[count:2 * count]
            rest = buf[2 * count:self.words * count]
            self.rho[sl] = rest.view(np.complex128).reshape(count, *self.rho.shape[1:])
            return
        for k, arr in enumerate((self.e, self.h, self.x, self.y, self.z)):
            arr[sl] = buf[k * count:(k + 1) * count]

    def poll(self):
        return self.bad

    def records(self):
        return [re if im is None else re + 1j * im for re, im in self.rec]

    def close(self):
        pass
