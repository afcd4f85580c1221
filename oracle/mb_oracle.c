/*
 * mb_oracle.c -- CPU ORACLE for the Maxwell-Bloch time-stepping core.
 *
 * TEST INFRASTRUCTURE ONLY.  This file restates, in plain C, the algorithm
 * of the reference solver's hot loop (/root/reference/pkg/src/mblight):
 *
 *   orc_update_h       solver_fdtd.py:53-56    (_update_h_range)
 *   orc_update_e       solver_fdtd.py:59-66    (_update_e_range)
 *   orc_bloch_step     _kernels.py:163-232     (_bloch_step_range)
 *   orc_split_step     _kernels.py:55-160      (_split_step_range)
 *   orc_rk4_step       _kernels.py:235-332     (_rk4_step_range)
 *   after_phase1/2     solver_fdtd.py:354-389  (swap, boundary, sources,
 *                                               non-finite scan)
 *   sample             solver_fdtd.py:391-426  (_sample)
 *   orc_run            solver_fdtd.py:444-498  (run / _run_serial)
 *
 * It is the checker for the CUDA path (tests/, __graft_entry__.smoke and
 * the cpu_baseline leg of bench.py) and never part of the product path.
 *
 * Pinning: the oracle is checked against golden records produced by the
 * reference itself (tests/golden/make_golden.py imports /root/reference and
 * runs FdtdSolver).  Built with -ffp-contract=off and no fast-math, the
 * FDTD updates, the Bloch (N=2) step and the RK4 step execute the same IEEE
 * operation sequence as the reference's numba loops (which are compiled
 * without fastmath), so those paths are bit-exact.  The reference compiles
 * the N>=3 splitting loop with fastmath=True (_kernels.py:55), which licenses
 * LLVM to contract/reassociate, so that path is pinned within tolerance.
 * Groups of <= 32 cells use the reference's numpy ScalarKernel
 * (_kernels.py:404-425); the oracle steps them with the same compiled-loop
 * restatement (tolerance-level difference, documented in DESIGN.md).
 *
 * Complex numbers are explicit (re, im) pairs so the evaluation order is
 * exactly the one written here; OpenMP parallelises the per-cell loops only,
 * so results are bitwise independent of the thread count (the reference's
 * contract).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAXN 8
#define ORC_MAXP 28
#define ORC_NONFINITE_EVERY 1024

typedef struct {
    int64_t num_x, num_t;
    double dt;
    int32_t stepper; /* 0 = splitting, 1 = rk4 */
    int32_t threads;
    int32_t levels;  /* N of the quantum materials (0 = none) */
    double *e, *h, *p_rate; /* e[Nx], h[Nx+1], p_rate[Nx] (in/out) */
    const double *coef_a, *coef_bg, *coef_bdx, *coef_ch; /* per cell, ch has Nx+1 */
    int32_t has_boundary;
    double wl, cl, zl, wr, cr, zr;
    int32_t n_src;
    const int64_t *src_cell;
    const int32_t *src_hard;
    const double *src_values; /* [num_t][n_src] */
    int32_t n_groups;
    const int64_t *g_start, *g_stop;
    const int32_t *g_qm;
    double **g_state, **g_next; /* Bloch: 3 planes of M; dense: M*N*N complex (re,im) AoS */
    int32_t n_qm;
    const double *qm_bloch;        /* [n_qm][14] kz cz fxy ax_c ax_s ay_c ay_s az_c az_s a0_c a0_s mu_x mu_y mu_z */
    const double *qm_pop_half;     /* [n_qm][N*N] */
    const double *qm_coh_half;     /* [n_qm][N*N] */
    const double *qm_b_const;      /* [n_qm][N*N][2] */
    const double *qm_b_field;      /* [n_qm][N*N][2] */
    const double *qm_h0, *qm_mu;   /* [n_qm][N*N][2] (rk4) */
    const double *qm_pop_matrix;   /* [n_qm][N*N] (rk4) */
    const double *qm_deph;         /* [n_qm][N*N] (rk4) */
    const int32_t *qm_npol;        /* [n_qm] */
    const int32_t *qm_pol_i, *qm_pol_j; /* [n_qm][ORC_MAXP] */
    const double *qm_pol_v;        /* [n_qm][ORC_MAXP][2] */
    const int32_t *qm_ndpol;       /* [n_qm] */
    const int32_t *qm_pol_di;      /* [n_qm][ORC_MAXN] */
    const double *qm_pol_dv;       /* [n_qm][ORC_MAXN] */
    const double *qm_pol_factor;   /* [n_qm] */
    int32_t n_rec;
    const int32_t *rec_q, *rec_i, *rec_j; /* q: 0 e, 1 h, 2 d, 3 inv; i, j 0-based */
    const int64_t *rec_cell;        /* -1 = whole domain */
    const int64_t *rec_every;
    double **rec_re, **rec_im;      /* [rows][cols]; im NULL for real records */
    int64_t step_limit;             /* run steps 1..min(num_t-1, step_limit) (bench sample) */
} orc_problem;

/* ------------------------------------------------------------------ FDTD */

static void orc_update_h(double *h, const double *e, const double *ch, int64_t m0, int64_t m1)
{
    /* solver_fdtd.py:53-56 */
#pragma omp parallel for schedule(static)
    for (int64_t m = m0; m < m1; ++m)
        h[m] += ch[m] * (e[m] - e[m - 1]);
}

static void orc_update_e(double *e, const double *h, const double *p, const double *a,
                         const double *bg, const double *bdx, int64_t lo, int64_t hi)
{
    /* solver_fdtd.py:59-66: a e - bg p + bdx (h[m+1] - h[m]), left to right */
#pragma omp parallel for schedule(static)
    for (int64_t m = lo; m < hi; ++m)
        e[m] = a[m] * e[m] - bg[m] * p[m] + bdx[m] * (h[m + 1] - h[m]);
}

/* --------------------------------------------------------- N = 2 (Bloch) */

static void orc_bloch_step(const double *s, double *sn, int64_t M, const double *e_vals,
                           const double *c, double pol_factor, double *p_out)
{
    /* _kernels.py:200-232 */
    const double kz = c[0], cz = c[1], fxy = c[2];
    const double ax_c = c[3], ax_s = c[4], ay_c = c[5], ay_s = c[6];
    const double az_c = c[7], az_s = c[8], a0_c = c[9], a0_s = c[10];
    const double mu_x = c[11], mu_y = c[12], mu_z = c[13];
    const double *X = s, *Y = s + M, *Z = s + 2 * M;
    double *Xn = sn, *Yn = sn + M, *Zn = sn + 2 * M;
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        const double e = e_vals[m];
        const double x0 = X[m], y0 = Y[m], z0 = Z[m];
        const double x1 = fxy * x0, y1 = fxy * y0, z1 = kz * z0 + cz;
        const double ax = ax_c + ax_s * e, ay = ay_c + ay_s * e;
        const double az = az_c + az_s * e, a0 = a0_c + a0_s * e;
        const double q = ax * ax + ay * ay + az * az;
        const double u = a0 * a0;
        const double num = 1.0 + u - q;
        const double t1 = 1.0 + q - u;
        const double inv = 1.0 / (t1 * t1 + 4.0 * u);
        const double k1 = (num * num - 4.0 * q) * inv;
        const double g = 4.0 * num * inv;
        const double dotb = 8.0 * inv * (ax * x1 + ay * y1 + az * z1);
        const double x2 = k1 * x1 + g * (ay * z1 - az * y1) + dotb * ax;
        const double y2 = k1 * y1 + g * (az * x1 - ax * z1) + dotb * ay;
        const double z2 = k1 * z1 + g * (ax * y1 - ay * x1) + dotb * az;
        const double x3 = fxy * x2, y3 = fxy * y2, z3 = kz * z2 + cz;
        Xn[m] = x3;
        Yn[m] = y3;
        Zn[m] = z3;
        p_out[m] = pol_factor * (mu_x * (x3 - x0) + mu_y * (y3 - y0) + mu_z * (z3 - z0));
    }
}

/* ---------------------------------------------------- complex helpers */

typedef struct { double re, im; } cplx;
static inline cplx cmul(cplx a, cplx b) { cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; return r; }
static inline cplx cadd(cplx a, cplx b) { cplx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cplx csub(cplx a, cplx b) { cplx r = {a.re - b.re, a.im - b.im}; return r; }
static inline cplx cconj(cplx a) { cplx r = {a.re, -a.im}; return r; }
/* real * complex as numba promotes it: (d + 0i)(b) */
static inline cplx rmul(double d, cplx b) { cplx r = {d * b.re - 0.0 * b.im, d * b.im + 0.0 * b.re}; return r; }

/* --------------------------------------------- N >= 3 Strang splitting */

static void orc_split_step(const cplx *rho, cplx *rho_next, int64_t M, int n, const double *e_vals,
                           const double *pop_half, const double *coh_half, const cplx *b_const,
                           const cplx *b_field, int npol, const int32_t *pi, const int32_t *pj,
                           const cplx *pv, int ndpol, const int32_t *pdi, const double *pdv,
                           double pol_factor, double *p_out)
{
    /* _kernels.py:87-160; row-major [i*n + j] */
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        cplx b[ORC_MAXN * ORC_MAXN], u[ORC_MAXN * ORC_MAXN], t[ORC_MAXN * ORC_MAXN];
        cplx r1[ORC_MAXN * ORC_MAXN], pops[ORC_MAXN];
        const cplx *rm = rho + m * n * n;
        cplx *out = rho_next + m * n * n;
        /* relaxation half step */
        for (int i = 0; i < n; ++i) {
            cplx acc = rmul(pop_half[i * n], rm[0]);
            for (int j = 1; j < n; ++j) acc = cadd(acc, rmul(pop_half[i * n + j], rm[j * n + j]));
            pops[i] = acc;
        }
        for (int i = 0; i < n; ++i) {
            for (int j = 0; j < n; ++j) r1[i * n + j] = rmul(coh_half[i * n + j], rm[i * n + j]);
            r1[i * n + i] = pops[i];
        }
        /* Cayley unitary U = B^-1 B^H by unpivoted elimination */
        const double e = e_vals[m];
        for (int i = 0; i < n * n; ++i) b[i] = cadd(b_const[i], rmul(e, b_field[i]));
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) u[i * n + j] = cconj(b[j * n + i]);
        for (int k = 0; k < n; ++k) {
            const cplx p = b[k * n + k];
            const double den = p.re * p.re + p.im * p.im;
            const cplx inv_piv = {p.re / den, -p.im / den};
            for (int i = k + 1; i < n; ++i) {
                const cplx f = cmul(b[i * n + k], inv_piv);
                for (int j = k + 1; j < n; ++j) b[i * n + j] = csub(b[i * n + j], cmul(f, b[k * n + j]));
                for (int j = 0; j < n; ++j) u[i * n + j] = csub(u[i * n + j], cmul(f, u[k * n + j]));
            }
        }
        for (int k = n - 1; k >= 0; --k) {
            const cplx p = b[k * n + k];
            const double den = p.re * p.re + p.im * p.im;
            const cplx inv_piv = {p.re / den, -p.im / den};
            for (int j = 0; j < n; ++j) {
                cplx acc = u[k * n + j];
                for (int i = k + 1; i < n; ++i) acc = csub(acc, cmul(b[k * n + i], u[i * n + j]));
                u[k * n + j] = cmul(acc, inv_piv);
            }
        }
        /* rho <- U r1 U^H, Hermitian result written directly */
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                cplx acc = cmul(u[i * n], r1[j]);
                for (int k = 1; k < n; ++k) acc = cadd(acc, cmul(u[i * n + k], r1[k * n + j]));
                t[i * n + j] = acc;
            }
        for (int i = 0; i < n; ++i)
            for (int j = i; j < n; ++j) {
                cplx acc = cmul(t[i * n], cconj(u[j * n]));
                for (int k = 1; k < n; ++k) acc = cadd(acc, cmul(t[i * n + k], cconj(u[j * n + k])));
                out[i * n + j] = acc;
                if (j > i) out[j * n + i] = cconj(acc);
            }
        /* second relaxation half step in place */
        for (int i = 0; i < n; ++i) {
            cplx acc = rmul(pop_half[i * n], out[0]);
            for (int j = 1; j < n; ++j) acc = cadd(acc, rmul(pop_half[i * n + j], out[j * n + j]));
            pops[i] = acc;
        }
        for (int i = 0; i < n; ++i) {
            for (int j = 0; j < n; ++j) out[i * n + j] = rmul(coh_half[i * n + j], out[i * n + j]);
            out[i * n + i] = pops[i];
        }
        /* polarization rate from the nonzero dipole entries */
        double acc_p = 0.0;
        for (int k = 0; k < npol; ++k) {
            const int i = pi[k], j = pj[k];
            const cplx d = csub(out[j * n + i], rm[j * n + i]);
            acc_p += 2.0 * cmul(pv[k], d).re;
        }
        for (int k = 0; k < ndpol; ++k) {
            const int i = pdi[k];
            acc_p += pdv[k] * csub(out[i * n + i], rm[i * n + i]).re;
        }
        p_out[m] = pol_factor * acc_p;
    }
}

/* ------------------------------------------------------------------ RK4 */

static void orc_rk4_step(const cplx *rho, cplx *rho_next, int64_t M, int n, const double *e_vals,
                         double dt, const cplx *h0, const cplx *mu, const double *pop_matrix,
                         const double *deph, int npol, const int32_t *pi, const int32_t *pj,
                         const cplx *pv, int ndpol, const int32_t *pdi, const double *pdv,
                         double pol_factor, double *p_out)
{
    /* _kernels.py:256-332 */
    const double hbar = 1.054571817e-34;
    const cplx minus_i_hbar = {-0.0 / hbar, -1.0 / hbar}; /* -1j / HBAR */
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        cplx h[ORC_MAXN * ORC_MAXN], stage[ORC_MAXN * ORC_MAXN];
        cplx kk[4][ORC_MAXN * ORC_MAXN];
        const cplx *rm = rho + m * n * n;
        const double e = e_vals[m];
        for (int i = 0; i < n * n; ++i) h[i] = csub(h0[i], rmul(e, mu[i]));
        for (int s = 0; s < 4; ++s) {
            const cplx *src;
            cplx *dst = kk[s];
            if (s == 0) {
                src = rm;
            } else {
                const double f = (s == 3) ? dt : 0.5 * dt;
                for (int i = 0; i < n * n; ++i) stage[i] = cadd(rm[i], rmul(f, kk[s - 1][i]));
                src = stage;
            }
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    cplx acc = csub(cmul(h[i * n], src[j]), cmul(src[i * n], h[j]));
                    for (int k = 1; k < n; ++k)
                        acc = cadd(acc, csub(cmul(h[i * n + k], src[k * n + j]), cmul(src[i * n + k], h[k * n + j])));
                    dst[i * n + j] = cmul(minus_i_hbar, acc);
                }
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    if (i != j) dst[i * n + j] = csub(dst[i * n + j], rmul(deph[i * n + j], src[i * n + j]));
            for (int i = 0; i < n; ++i) {
                cplx acc = rmul(pop_matrix[i * n], src[0]);
                for (int j = 1; j < n; ++j) acc = cadd(acc, rmul(pop_matrix[i * n + j], src[j * n + j]));
                dst[i * n + i] = cadd(dst[i * n + i], acc);
            }
        }
        cplx *out = rho_next + m * n * n;
        const double sixth = dt / 6.0;
        for (int i = 0; i < n * n; ++i) {
            const cplx sum = cadd(cadd(cadd(kk[0][i], rmul(2.0, kk[1][i])), rmul(2.0, kk[2][i])), kk[3][i]);
            out[i] = cadd(rm[i], rmul(sixth, sum));
        }
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                const cplx sym = rmul(0.5, cadd(out[i * n + j], cconj(out[j * n + i])));
                out[i * n + j] = sym;
                out[j * n + i] = cconj(sym);
            }
        double acc_p = 0.0;
        for (int k = 0; k < npol; ++k) {
            const int i = pi[k], j = pj[k];
            acc_p += 2.0 * cmul(pv[k], csub(out[j * n + i], rm[j * n + i])).re;
        }
        for (int k = 0; k < ndpol; ++k) {
            const int i = pdi[k];
            acc_p += pdv[k] * csub(out[i * n + i], rm[i * n + i]).re;
        }
        p_out[m] = pol_factor * acc_p;
    }
}

/* ------------------------------------------------------------- driver */

static int is_bloch(const orc_problem *P) { return P->levels == 2 && P->stepper == 0; }

static void advance_group(const orc_problem *P, int g)
{
    const int64_t lo = P->g_start[g], M = P->g_stop[g] - lo;
    const int q = P->g_qm[g], n = P->levels;
    const double *ev = P->e + lo;
    double *pout = P->p_rate + lo;
    if (is_bloch(P)) {
        orc_bloch_step(P->g_state[g], P->g_next[g], M, ev, P->qm_bloch + 14 * q, P->qm_pol_factor[q], pout);
        return;
    }
    const int nn = n * n;
    const cplx *pv = (const cplx *)(P->qm_pol_v + 2 * ORC_MAXP * q);
    if (P->stepper == 0) {
        orc_split_step((const cplx *)P->g_state[g], (cplx *)P->g_next[g], M, n, ev,
                       P->qm_pop_half + nn * q, P->qm_coh_half + nn * q,
                       (const cplx *)(P->qm_b_const + 2 * nn * q), (const cplx *)(P->qm_b_field + 2 * nn * q),
                       P->qm_npol[q], P->qm_pol_i + ORC_MAXP * q, P->qm_pol_j + ORC_MAXP * q, pv,
                       P->qm_ndpol[q], P->qm_pol_di + ORC_MAXN * q, P->qm_pol_dv + ORC_MAXN * q,
                       P->qm_pol_factor[q], pout);
    } else {
        orc_rk4_step((const cplx *)P->g_state[g], (cplx *)P->g_next[g], M, n, ev, P->dt,
                     (const cplx *)(P->qm_h0 + 2 * nn * q), (const cplx *)(P->qm_mu + 2 * nn * q),
                     P->qm_pop_matrix + nn * q, P->qm_deph + nn * q,
                     P->qm_npol[q], P->qm_pol_i + ORC_MAXP * q, P->qm_pol_j + ORC_MAXP * q, pv,
                     P->qm_ndpol[q], P->qm_pol_di + ORC_MAXN * q, P->qm_pol_dv + ORC_MAXN * q,
                     P->qm_pol_factor[q], pout);
    }
}

/* density entry (i, j) of group g at local cell c (_kernels.py:388-392, 530-539) */
static cplx density_entry(const orc_problem *P, int g, int64_t c, int i, int j)
{
    const int64_t M = P->g_stop[g] - P->g_start[g];
    const double *s = P->g_state[g];
    if (is_bloch(P)) {
        const double x = s[c], y = s[M + c], z = s[2 * M + c];
        cplx r;
        if (i == j) {
            r.re = (i == 0) ? 0.5 * (1.0 + z) : 0.5 * (1.0 - z);
            r.im = 0.0;
        } else if (i == 0) {
            r.re = 0.5 * x; r.im = 0.5 * -y; /* 0.5 * (x - 1j*y) */
        } else {
            r.re = 0.5 * x; r.im = 0.5 * y;
        }
        return r;
    }
    const int n = P->levels;
    const cplx *rho = (const cplx *)s + c * n * n;
    return rho[i * n + j];
}

static double inversion(const orc_problem *P, int g, int64_t c)
{
    if (is_bloch(P)) {
        const int64_t M = P->g_stop[g] - P->g_start[g];
        return -P->g_state[g][2 * M + c];
    }
    const int n = P->levels;
    const cplx *rho = (const cplx *)P->g_state[g] + c * n * n;
    return rho[n + 1].re - rho[0].re;
}

static void sample(const orc_problem *P, int64_t n)
{
    /* solver_fdtd.py:391-426 */
    const int64_t nx = P->num_x;
    for (int r = 0; r < P->n_rec; ++r) {
        if (n % P->rec_every[r]) continue;
        const int64_t row = n / P->rec_every[r];
        const int64_t cell = P->rec_cell[r];
        const int64_t cols = cell < 0 ? nx : 1;
        double *re = P->rec_re[r] + row * cols;
        double *im = P->rec_im[r] ? P->rec_im[r] + row * cols : NULL;
        const int q = P->rec_q[r];
        if (q == 0 || q == 1) {
            const double *src = q == 0 ? P->e : P->h;
            if (cell < 0) memcpy(re, src, sizeof(double) * nx);
            else re[0] = src[cell];
            continue;
        }
        for (int g = 0; g < P->n_groups; ++g) {
            const int64_t lo = P->g_start[g], hi = P->g_stop[g];
            int64_t c0 = lo, c1 = hi;
            if (cell >= 0) {
                if (cell < lo || cell >= hi) continue;
                c0 = cell; c1 = cell + 1;
            }
            for (int64_t c = c0; c < c1; ++c) {
                const int64_t col = cell < 0 ? c : 0;
                if (q == 2) {
                    const cplx v = density_entry(P, g, c - lo, P->rec_i[r], P->rec_j[r]);
                    re[col] = v.re;
                    if (im) im[col] = v.im;
                } else {
                    re[col] = inversion(P, g, c - lo);
                }
            }
        }
    }
}

/* Runs steps 1 .. min(num_t-1, step_limit).  Returns 0, or the first step whose
 * non-finite scan failed (solver_fdtd.py:386-388) as a positive number. */
int64_t orc_run(orc_problem *P)
{
#ifdef _OPENMP
    if (P->threads > 0) omp_set_num_threads(P->threads);
#endif
    const int64_t nx = P->num_x;
    int64_t last = P->num_t - 1;
    if (P->step_limit > 0 && P->step_limit < last) last = P->step_limit;
    double h1_prev = 0.0, hm_prev = 0.0;
    if (nx > 1) { h1_prev = P->h[1]; hm_prev = P->h[nx - 1]; }
    sample(P, 0);
    for (int64_t n = 1; n <= last; ++n) {
        /* phase 1: H^{n-1/2} from E^{n-1}; density step with E^{n-1} */
        if (nx > 1) orc_update_h(P->h, P->e, P->coef_ch, 1, nx);
        for (int g = 0; g < P->n_groups; ++g) advance_group(P, g);
        /* after phase 1: swap, remember the edge values of E^{n-1} */
        for (int g = 0; g < P->n_groups; ++g) {
            double *t = P->g_state[g]; P->g_state[g] = P->g_next[g]; P->g_next[g] = t;
        }
        double e0_old = 0, e1_old = 0, em_old = 0, em1_old = 0;
        if (nx > 1) { e0_old = P->e[0]; e1_old = P->e[1]; em_old = P->e[nx - 1]; em1_old = P->e[nx - 2]; }
        /* phase 2: E^n */
        if (nx > 1) orc_update_e(P->e, P->h, P->p_rate, P->coef_a, P->coef_bg, P->coef_bdx, 0, nx);
        /* after phase 2: boundary, then sources, then checks and records */
        if (nx > 1 && P->has_boundary) {
            double e_at = (1.0 - P->cl) * e0_old + P->cl * e1_old;
            double h_at = 0.5 * (h1_prev + P->h[1]);
            P->e[0] = P->wl * 0.5 * (e_at + P->zl * h_at);
            e_at = (1.0 - P->cr) * em_old + P->cr * em1_old;
            h_at = 0.5 * (hm_prev + P->h[nx - 1]);
            P->e[nx - 1] = P->wr * 0.5 * (e_at - P->zr * h_at);
            h1_prev = P->h[1];
            hm_prev = P->h[nx - 1];
        }
        for (int s = 0; s < P->n_src; ++s) {
            const double v = P->src_values[n * P->n_src + s];
            const int64_t c = P->src_cell[s];
            if (P->src_hard[s]) P->e[c] = v;
            else P->e[c] += v;
        }
        if (n % ORC_NONFINITE_EVERY == 0 || n == P->num_t - 1) {
            for (int64_t m = 0; m < nx; ++m)
                if (!isfinite(P->e[m])) return n;
        }
        sample(P, n);
    }
    return 0;
}

/* One density step of M consecutive cells of quantum material q with the
 * constants of P (TEST DOUBLE support: the CPU slab twin of the gloo
 * multi-process tests steps its window's quantum runs with this, so an
 * N-level slab rank runs the very arithmetic of orc_run).  state/next in the
 * group layout of P->stepper (Bloch planes of M, or dense AoS complex). */
void orc_density_step(const orc_problem *P, int32_t q, const double *state, double *next, int64_t M,
                      const double *e_vals, double *p_out)
{
#ifdef _OPENMP
    if (P->threads > 0) omp_set_num_threads(P->threads);
#endif
    if (M <= 0) return;
    if (is_bloch(P)) {
        orc_bloch_step(state, next, M, e_vals, P->qm_bloch + 14 * q, P->qm_pol_factor[q], p_out);
        return;
    }
    const int n = P->levels, nn = n * n;
    const cplx *pv = (const cplx *)(P->qm_pol_v + 2 * ORC_MAXP * q);
    if (P->stepper == 0)
        orc_split_step((const cplx *)state, (cplx *)next, M, n, e_vals, P->qm_pop_half + nn * q,
                       P->qm_coh_half + nn * q, (const cplx *)(P->qm_b_const + 2 * nn * q),
                       (const cplx *)(P->qm_b_field + 2 * nn * q), P->qm_npol[q], P->qm_pol_i + ORC_MAXP * q,
                       P->qm_pol_j + ORC_MAXP * q, pv, P->qm_ndpol[q], P->qm_pol_di + ORC_MAXN * q,
                       P->qm_pol_dv + ORC_MAXN * q, P->qm_pol_factor[q], p_out);
    else
        orc_rk4_step((const cplx *)state, (cplx *)next, M, n, e_vals, P->dt, (const cplx *)(P->qm_h0 + 2 * nn * q),
                     (const cplx *)(P->qm_mu + 2 * nn * q), P->qm_pop_matrix + nn * q, P->qm_deph + nn * q,
                     P->qm_npol[q], P->qm_pol_i + ORC_MAXP * q, P->qm_pol_j + ORC_MAXP * q, pv, P->qm_ndpol[q],
                     P->qm_pol_di + ORC_MAXN * q, P->qm_pol_dv + ORC_MAXN * q, P->qm_pol_factor[q], p_out);
}

int orc_version(void) { return 2; }
