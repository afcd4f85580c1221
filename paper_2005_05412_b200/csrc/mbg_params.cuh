// Launch parameter blocks of the fused step kernels.
//
// Everything a kernel needs is passed by value as a __grid_constant__
// parameter block (constant bank 0): material coefficients, stepper constants,
// boundary, source cells, record plans and the per-step sampling masks of the
// launch.  Constants indexed at compile time become immediate constant-bank
// operands of the FP64 instructions, and no process-global device state
// exists, so any number of solver handles can coexist.
#pragma once
#include <cstdint>
#include <cstdio>

#include "../../include/mbgpu.h"

namespace mbg {

constexpr int kMaxRegions = MBG_MAX_REGIONS;
constexpr int kMaxQm = MBG_MAX_QM;
constexpr int kMaxDenseQm = kMaxQm;  // param block: DenseParams<8, *> with 4 media stays under the 32 KB launch limit
constexpr int kMaxSources = MBG_MAX_SOURCES;
constexpr int kMaxRecords = MBG_MAX_RECORDS;
constexpr int kMaxTileSteps = MBG_MAX_TILE_STEPS;

// region table (replaces the reference's per-cell coefficient arrays,
// solver_fdtd.py:252-268): E cell m belongs to the last region r with
// e_start[r] <= m; H node m (1..Nx-1) to the last r with h_start[r] <= m
struct Regions {
    int n;
    long long e_start[kMaxRegions];
    long long h_start[kMaxRegions];
    double a[kMaxRegions];    // a'
    double bg[kMaxRegions];   // b' * Gamma
    double bdx[kMaxRegions];  // b' / dx
    double ch[kMaxRegions];   // c'
    int qm[kMaxRegions];      // quantum material index, -1 classical
};

struct Launch {
    long long num_x;
    long long win_lo, win_n;  // window: global cells [win_lo, win_lo + win_n)
    long long res_lo, res_hi; // cells valid after this launch
    long long own_lo, own_hi; // cells recorded / scanned here
    long long n0;             // global step index of the first fused step
    int k;                    // fused steps in this launch
    int tile_own;             // result cells per tile
    long long plane;          // stride between state planes (elements)
    const double *e_in, *h_in, *s_in;
    double *e_out, *h_out, *s_out;
    // boundary terms evaluated as solver_fdtd.py:372-377 does:
    // e_at = omc*e_edge + c*e_inner; h_at = 0.5*(h_prev + h_new); e = hw*(e_at +/- z*h_at)
    int has_boundary;
    double l_omc, l_c, l_hw, l_z;
    double r_omc, r_c, r_hw, r_z;
    int n_src;
    long long src_cell[kMaxSources];
    int src_hard[kMaxSources];
    const double *src_values;  // [num_t][n_src]
    int n_rec;
    int rec_q[kMaxRecords], rec_i[kMaxRecords], rec_j[kMaxRecords];
    long long rec_cell[kMaxRecords];  // -1: whole domain
    long long rec_every[kMaxRecords];
    long long rec_cols[kMaxRecords];
    long long rec_col0[kMaxRecords];  // global cell of column 0
    long long rec_row0[kMaxRecords];  // first row resident on the device (streamed records; 0 otherwise)
    double *rec_re[kMaxRecords];
    double *rec_im[kMaxRecords];
    unsigned long long step_mask[kMaxTileSteps];  // bit r: record r samples at fused step s
    unsigned char check[kMaxTileSteps];           // MBG_STEP_* flags of fused step s
    unsigned long long *bad_step;
    // two-level invariant monitor fused into the record steps (null: off):
    // running min-eigenvalue key at inv[2], every inv_every steps
    unsigned long long *inv;
    long long inv_every;
    // extents for the bounds-checked build (MBG_BOUNDS): state words per cell,
    // time steps of the source table, resident elements of each record
    int words;
    long long num_t;
    long long rec_len[kMaxRecords];
    Regions rg;
};

// Bounds-checked build (make EXTRA=-DMBG_BOUNDS=1, tools/bounds_check.sh): every
// global access of the step, sample and halo kernels is checked against the
// extents of its buffer; a violation prints the site and index and traps (the
// launch fails with an error, the run raises).  compute-sanitizer is not
// available on this GPU pool; this is the evidence in its place.
#if defined(MBG_BOUNDS) && MBG_BOUNDS && defined(__CUDACC__)
__device__ __noinline__ inline void mbg_oob(const char *site, long long idx, long long len) {
    printf("MBG_BOUNDS violation: %s index %lld of %lld (block %d thread %d)\n", site, idx, len, (int)blockIdx.x,
           (int)threadIdx.x);
    __trap();
}
#define MBG_CHK(idx, len, site)                                                   \
    do {                                                                          \
        const long long _i = (long long)(idx), _n = (long long)(len);           \
        if (_i < 0 || _i >= _n) mbg_oob(site, _i, _n);                           \
    } while (0)
#else
#define MBG_CHK(idx, len, site) \
    do {                        \
    } while (0)
#endif

// per-step flags (Launch::check, the persistent launch's check bytes)
enum : unsigned char { MBG_STEP_SCAN = 1, MBG_STEP_MONITOR = 2 };

// the reference's non-finite scan (every 1024 steps and the last,
// solver_fdtd.py:386-388) and the invariant monitor's cadence
// (solver_fdtd.py:425-426: every monitored step, records or not)
__host__ __device__ inline unsigned char step_flags(const Launch &L, long long n, long long last_step) {
    unsigned char f = (n % 1024 == 0 || n == last_step) ? MBG_STEP_SCAN : 0;
    if (L.inv && L.inv_every > 0 && n % L.inv_every == 0) f |= MBG_STEP_MONITOR;
    return f;
}

// two-level splitting in Bloch form (_kernels.py:200-232)
struct BlochQm {
    double kz, cz, fxy, ax_c, ax_s, ay_c, ay_s, az_c, az_s, a0_c, a0_s, mu_x, mu_y, mu_z, pol_factor;
};

// real dipole and diagonal H0 (every two_level_description medium): ax_c, ay_c,
// ay_s, az_s, a0_s, mu_y, mu_z vanish, so A = (ax_s E, 0, az_c) with a0 = a0_c
// constant; the field-independent products are hoisted (same IEEE values)
struct BlochReal {
    double u;     // a0_c * a0_c
    double c1;    // 1.0 + u
    double c4u;   // 4.0 * u
    double az2;   // az_c * az_c
    double pfmu;  // pol_factor * mu_x * fxy (fast variant, relaxed-frame state)
    double f2;    // fxy * fxy
    double kz2;   // kz * kz
    double czz;   // kz * cz + cz
    double c1h;   // (1 + u) / 2
};

// Relaxed-frame state of the fast two-level path: the device holds each
// Bloch vector after the Cayley rotation and before the second half
// relaxation, (X, Y, Z) with x = fxy X, y = fxy Y, z = kz Z + cz.  Then one
// step's two half relaxations fold into one (x1 = fxy^2 X, z1 = kz^2 Z + kz cz
// + cz), three operations fewer per cell and step.  Every reader of the state
// (records, sample, invariants, download) maps back with frame_true; uploads
// map in with frame_in.
struct BlochFrame {
    int on;
    double fxy[kMaxQm], kz[kMaxQm], cz[kMaxQm];
};

__host__ __device__ inline void frame_true(const BlochFrame &F, int q, double X, double Y, double Z, double &x,
                                           double &y, double &z) {
    if (F.on && q >= 0) {
        x = F.fxy[q] * X;
        y = F.fxy[q] * Y;
        z = fma(F.kz[q], Z, F.cz[q]);
    } else {
        x = X;
        y = Y;
        z = Z;
    }
}

struct BlochParams {
    Launch L;
    int n_qm;
    int real_dipole;  // all materials satisfy the BlochReal pattern (fast variant: and the frame applies)
    BlochFrame frame; // fast variant with real_dipole: the state is in the relaxed frame
    BlochQm qm[kMaxQm];
    BlochReal rq[kMaxQm];
};

// dipole weights of the polarisation trace (_kernels.py:360-374), stored
// densely: pol_re/pol_im per upper pair (row-major i<j), pol_dv per diagonal;
// entries where mu vanishes are 0 and add exact zeros
template <int N>
struct PolTerms {
    static constexpr int kUpper = N * (N - 1) / 2;
    double pol_re[kUpper], pol_im[kUpper];
    double pol_dv[N];
    double pol_factor;
};

// N-level Strang splitting (_kernels.py:428-439): B = bc + E * bf
template <int N>
struct DenseQm {
    double pop[N * N], coh[N * N];
    double bc_re[N * N], bc_im[N * N], bf_re[N * N], bf_im[N * N];
    PolTerms<N> pol;
};

// N-level RK4 (_kernels.py:549-557): H = h0 - E mu
template <int N>
struct Rk4Qm {
    double h0_re[N * N], h0_im[N * N], mu_re[N * N], mu_im[N * N];
    double popm[N * N], deph[N * N];
    double dt;
    PolTerms<N> pol;
};

template <int N, class Q>
struct DenseParams {
    Launch L;
    int n_qm;
    int real_a;  // every medium has a real Hamiltonian and dipole (fast variant: real inversion)
    Q qm[kMaxDenseQm];
};

// Batched single-point systems (Nx = 1, solver_fdtd.py:89-96, 347-349): the
// field is only source-driven there, so every system's E^n is precomputed on
// the host and one thread per system steps its density matrix and writes its
// density records (rows [B][rows]; E / H records are filled on the host).
struct BatchRecs {
    int n;
    int q[kMaxRecords], i[kMaxRecords], j[kMaxRecords];
    long long every[kMaxRecords], rows[kMaxRecords];
    double *re[kMaxRecords], *im[kMaxRecords];
};

// The media of a batch live in device global memory (one constant set per
// distinct medium, up to MBG_MAX_BATCH_QM): a sweep over detunings or rates
// is not capped by the 32 KB parameter block; each thread reads its own set
// (L1-cached, one set per system).
template <int N, class Q>
struct BatchParams {
    int B;
    long long num_t;
    const double *e_seq;  // [num_t][B]
    double *state;        // [words][B], in and out
    const int *medium;    // [B] constant-set index
    int n_qm, real_a;
    const Q *qm;          // [n_qm], device
    BatchRecs R;
};

struct BlochBatchParams {
    int B;
    long long num_t;
    const double *e_seq;
    double *state;  // Bloch (x, y, z) planes
    const int *medium;
    int n_qm, real_dipole;
    const BlochQm *qm;    // [n_qm], device
    const BlochReal *rq;  // [n_qm], device
    BatchRecs R;
};

// shared helpers (host + device)
// last region r with start[r] <= m (0 if none); starts are non-decreasing,
// empty regions repeat a start and are skipped by taking the last match
__host__ __device__ inline int region_of(const long long *start, int n, long long m) {
    int lo = 0, hi = n - 1;
#pragma unroll 1
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (start[mid] <= m)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// two-level kernel geometry: tile t covers result cells [t_lo, t_hi) and loads
// slots [base, base + width); the tile at the physical left edge starts at 0
__host__ __device__ inline long long tile_base(const Launch &L, long long t_lo) {
    return (t_lo - L.k < 0) ? 0 : t_lo - L.k;
}

// interior tile: all slots regular cells (1 <= c <= Nx-2) inside the window,
// one E region and one H region, no source cell
__host__ __device__ inline bool tile_is_interior(const Launch &L, long long base, int width) {
    const long long hi = base + width - 1;
    if (base < 1 || hi > L.num_x - 2 || base < L.win_lo || hi >= L.win_lo + L.win_n) return false;
    if (region_of(L.rg.e_start, L.rg.n, base) != region_of(L.rg.e_start, L.rg.n, hi)) return false;
    if (region_of(L.rg.h_start, L.rg.n, base) != region_of(L.rg.h_start, L.rg.n, hi)) return false;
    for (int q = 0; q < L.n_src; ++q)
        if (L.src_cell[q] >= base && L.src_cell[q] <= hi) return false;
    return true;
}

// result ranges [lo, hi) of the non-interior tiles, each processed by one warp
constexpr int kMaxEdgeTiles = 128;
struct EdgeTiles {
    int n;
    long long lo[kMaxEdgeTiles];
    long long hi[kMaxEdgeTiles];
};

}  // namespace mbg
