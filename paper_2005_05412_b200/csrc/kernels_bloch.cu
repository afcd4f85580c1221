// Fused time-step kernel for two-level media (and purely classical devices).
//
// One launch advances the Yee fields and the Bloch vectors by k time steps
// (temporal tiling).  Each warp owns a tile of 32*C consecutive cells laid out
// cyclically (slot i*32 + lane), so every global load/store is a coalesced
// 256-byte row.  E, H and the Bloch vector (x, y, z) stay in registers for all
// k steps; the only neighbour traffic of the stencil is one warp shuffle of E
// to the right (H update needs E[m-1]) and one of H to the left (E update
// needs H[m+1]) per cell and step.  The dependency cone shrinks by one cell per
// side per step, so a tile that loads 32*C cells delivers the 32*C - 2k cells
// in its middle ("redundant halo"); tiles touching a physical edge keep their
// edge cells.
//
// Per step the operation sequence is the reference's (solver_fdtd.py:457-463):
//   H^{n-1/2}[m] = H + c' (E[m] - E[m-1])            solver_fdtd.py:53-56
//   Bloch step with E^{n-1}, p = pol_factor d<mu>     _kernels.py:200-232
//   E^n[m] = a' E - b'G p + b'/dx (H[m+1] - H[m])      solver_fdtd.py:59-66
//   edge cells <- (1 - sqrt R) * outgoing char.        solver_fdtd.py:366-378
//   sources (hard overwrite / soft add), in order      solver_fdtd.py:379-385
//   non-finite scan, record sampling                   solver_fdtd.py:386-426
// Built without FMA contraction (exact variant) every value is bit-identical
// to the reference.
#include "mbg_kernels.h"

#ifndef MBG_VARIANT
#error "compile with -DMBG_VARIANT=fast|exact"
#endif

namespace mbg {
namespace MBG_VARIANT {

namespace {

constexpr int C = kBlochCellsPerLane;
constexpr int W = kBlochTile;
constexpr unsigned kFull = 0xffffffffu;

// One fused chunk of k steps: where it reads and writes, its first step and
// per-step record masks / scan flags.  Per-launch kernels point it at the
// launch parameters, the persistent kernel at its chunk's slice.
struct Chunk {
    const double *e_in, *h_in, *s_in;
    double *e_out, *h_out, *s_out;
    long long n0;
    int steps;
    const unsigned long long *mask;
    const unsigned char *check;
};

__device__ __forceinline__ Chunk launch_chunk(const Launch &L) {
    return Chunk{L.e_in, L.h_in, L.s_in, L.e_out, L.h_out, L.s_out, L.n0, L.k, L.step_mask, L.check};
}

// field / state loads bypass L1 (streamed once per chunk; in the persistent
// kernel another CTA of the same launch produced them)
__device__ __forceinline__ double ld(const double *p) { return __ldcg(p); }
__device__ __forceinline__ void ld2(const double *p, double &a, double &b) {
    const double2 v = __ldcg(reinterpret_cast<const double2 *>(p));
    a = v.x;
    b = v.y;
}
__device__ __forceinline__ void st2(double *p, double a, double b) {
    *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}

// order-preserving key of a double (atomicMin over doubles), as the monitor kernel's
__device__ __forceinline__ unsigned long long order_key(double v) {
    const unsigned long long b = __double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// fused invariant monitor of a two-level warp: min over its lanes' keys, one atomic
__device__ __forceinline__ void fold_min_eig(unsigned long long *inv, unsigned long long key) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(kFull, key, o);
        key = other < key ? other : key;
    }
    if ((threadIdx.x & 31) == 0 && key != ~0ull) atomicMin(inv + 2, key);
}

// _kernels.py:200-232, same expression order (each mad(a, b, c) is the
// reference's "c + a*b" term)
__device__ __forceinline__ double bloch_cell(const BlochQm &q, double e, double &x, double &y, double &z) {
    const double x0 = x, y0 = y, z0 = z;
    const double x1 = q.fxy * x0, y1 = q.fxy * y0, z1 = mad(q.kz, z0, q.cz);
    const double ax = mad(q.ax_s, e, q.ax_c), ay = mad(q.ay_s, e, q.ay_c);
    const double az = mad(q.az_s, e, q.az_c), a0 = mad(q.a0_s, e, q.a0_c);
    const double qq = mad(az, az, mad(ay, ay, ax * ax));
    const double u = a0 * a0;
    const double num = 1.0 + u - qq;
    const double t1 = 1.0 + qq - u;
    const double inv = 1.0 / mad(t1, t1, 4.0 * u);
    const double k1 = mad(num, num, -(4.0 * qq)) * inv;
    const double g = 4.0 * num * inv;
    const double dotb = 8.0 * inv * mad(az, z1, mad(ay, y1, ax * x1));
    const double x2 = mad(dotb, ax, mad(g, mad(ay, z1, -(az * y1)), k1 * x1));
    const double y2 = mad(dotb, ay, mad(g, mad(az, x1, -(ax * z1)), k1 * y1));
    const double z2 = mad(dotb, az, mad(g, mad(ax, y1, -(ay * x1)), k1 * z1));
    x = q.fxy * x2;
    y = q.fxy * y2;
    z = mad(q.kz, z2, q.cz);
    return q.pol_factor * mad(q.mu_z, z - z0, mad(q.mu_y, y - y0, q.mu_x * (x - x0)));
}

// Same step for real-dipole / diagonal-H0 media.  Every dropped term is an
// exact zero in the reference's evaluation (0*E, 0*x), so each nonzero value
// equals the general formula's bit for bit; only the sign of an exact zero
// could differ.
__device__ __forceinline__ double bloch_cell_real(const BlochQm &q, const BlochReal &r, double e, double &x,
                                                  double &y, double &z) {
    const double x0 = x, y0 = y, z0 = z;
    const double x1 = q.fxy * x0, y1 = q.fxy * y0, z1 = mad(q.kz, z0, q.cz);
    const double ax = q.ax_s * e, az = q.az_c;
    const double qq = mad(ax, ax, r.az2);
    const double num = r.c1 - qq;
    const double t1 = 1.0 + qq - r.u;
    const double inv = 1.0 / mad(t1, t1, r.c4u);
    const double k1 = mad(num, num, -(4.0 * qq)) * inv;
    const double g = 4.0 * num * inv;
    const double dotb = 8.0 * inv * mad(az, z1, ax * x1);
    const double x2 = mad(dotb, ax, mad(g, -(az * y1), k1 * x1));
    const double y2 = mad(g, mad(az, x1, -(ax * z1)), k1 * y1);
    const double z2 = mad(dotb, az, mad(g, ax * y1, k1 * z1));
    x = q.fxy * x2;
    y = q.fxy * y2;
    z = mad(q.kz, z2, q.cz);
    return q.pol_factor * (q.mu_x * (x - x0));
}

#if !(defined(MBG_EXACT) && MBG_EXACT)
// 2/d for d >= 1/4 (a quarter of the Cayley denominator (1+q-u)^2 + 4u >= 1):
// hardware seed r ~ 1/d refined by one cubically convergent step
// 2r + 2r(e + e^2), e = 1 - d r (seed error 2^-22 -> below double rounding),
// no special cases.  The doubling 2r is exact and done on the integer pipe
// (exponent + 1 of the normal seed, 1/4 <= ... so r <= 4), so the factor 2
// of the rotation costs no FP64 operation.
__device__ __forceinline__ double rcp2_ge1(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    const double e = fma(-d, r, 1.0);
    const double r2 = __hiloint2double(__double2hiint(r) + (1 << 20), __double2loint(r));
    return fma(r2, fma(e, e, e), r2);
}

// Fast variant of bloch_cell_real on the relaxed-frame state (BlochFrame):
// the two half relaxations of consecutive steps are one multiply (one FMA for
// z), the rotation is evaluated in Rodrigues form (below; tolerance-level,
// not bitwise).  Returns X_new - X_old: the factor
// pol_factor * mu_x * fxy is folded into the E update's coefficient (pol_coef).
__device__ __forceinline__ double bloch_cell_real_frame(const BlochQm &q, const BlochReal &r, double e, double &x,
                                                        double &y, double &z) {
    const double x0 = x;
    const double x1 = r.f2 * x, y1 = r.f2 * y, z1 = fma(r.kz2, z, r.czz);
    // The Cayley rotation in Rodrigues form around a = (ax, 0, az):
    //   v2 = v1 + P (a x v1) + Q (a x (a x v1)),  P = 2 nh / D, Q = 2 / D,
    //   nh = (1 + u - |a|^2) / 2,  D = nh^2 + |a|^2  (= ((1 - u + |a|^2)/2)^2 + u = W/4),
    // the same rotation as the reference's k1 v1 + g (a x v1) + (8/W)(a.v1) a:
    // cos = (nh^2 - |a|^2)/D, sin = 2 nh |a|/D.  With ay = 0 the y component
    // of a x (a x v1) is -|a|^2 y1, and the x and z components share one factor:
    //   x2 = x1 - 2az s,  z2 = z1 + 2ax s,  s = (nh y1 + cy) / D,
    //   y2 = ((nh^2 - |a|^2) y1 + 2 nh cy) / D,  cy = az x1 - ax z1.
    // With D = nh^2 + |a|^2 the y row simplifies to y2 = 2 nh s - y1:
    //   2 nh (nh y1 + cy)/D - y1 = ((nh^2 - |a|^2) y1 + 2 nh cy)/D,
    // so with t = 2 s (exact doubling) all three rows are one FMA each:
    //   x2 = x1 - az t,  z2 = z1 + ax t,  y2 = nh t - y1,
    // and 2/D comes out of the reciprocal's refinement (rcp2_ge1).
    // 18 FP64 operations (30 in the g / dot-product grouping), tolerance-level
    // against the reference (not bitwise).
    const double ax = q.ax_s * e, az = q.az_c;
    const double qq = fma(ax, ax, r.az2);
    const double nh = fma(-0.5, qq, r.c1h);
    const double i2D = rcp2_ge1(fma(nh, nh, qq));
    const double cy = fma(az, x1, -(ax * z1));
    const double t = i2D * fma(nh, y1, cy);
    x = fma(-az, t, x1);
    y = fma(nh, t, -y1);
    z = fma(ax, t, z1);
    return x - x0;
}
#define MBG_BLOCH_REAL bloch_cell_real_frame
#define MBG_POL_FOLD 1
#else
#define MBG_BLOCH_REAL bloch_cell_real
#define MBG_POL_FOLD 0
#endif

// coefficient of the polarisation term in the E update (b' G, times the
// real-dipole factor the fast cell function leaves out); interior and edge
// paths form it from the same operands, so their E values agree bitwise
__device__ __forceinline__ double pol_coef(double bg, const BlochReal &r, bool real) {
    return (MBG_POL_FOLD && real) ? bg * r.pfmu : bg;
}

// E^n = a E - b'G p + b'/dx (H[m+1] - H[m]) (solver_fdtd.py:59-66).  The fast
// variant fuses the polarisation term into E when a == 1 (lossless medium;
// 1*E is exact, so only the rounding of the fused term changes); every path
// uses this one function, so interior and edge cells stay bitwise equal.
template <bool A1>
__device__ __forceinline__ double e_update(double a, double bdx, double bgp, double e, double dh, double p) {
    if (MBG_POL_FOLD && A1) return mad(bdx, dh, fma(-bgp, p, e));
    return mad(bdx, dh, mad(a, e, -(bgp * p)));
}

// density entry (i, j) of a Bloch vector (_kernels.py:530-536)
__device__ __forceinline__ void bloch_entry(int i, int j, double x, double y, double z, double &re, double &im) {
    if (i == j) {
        re = (i == 0) ? 0.5 * (1.0 + z) : 0.5 * (1.0 - z);
        im = 0.0;
    } else {
        re = 0.5 * x;
        im = (i == 0) ? 0.5 * -y : 0.5 * y;
    }
}

// General tile (domain/window ends, region interfaces, source cells): cyclic
// layout (slot i*32 + lane), every per-slot property decided once per launch
// and kept as bit masks; UNI tiles (one E and one H region) take scalar
// coefficients and one material, the rare interface tiles look them up per slot.
template <bool UNI>
__device__ __forceinline__ void run_tile(const BlochParams &P, const Chunk &K, long long t_lo, long long t_hi,
                                         long long base, int lane) {
    const Launch &L = P.L;
    const long long nx = L.num_x;
    double E[C], H[C], X[C], Y[C], Z[C];
    int qi[C];  // quantum material of the slot, -1 classical / outside (used when !UNI)
    double ca[C], cbg[C], cbdx[C], cch[C];
    unsigned hmask = 0, emask = 0, qmask = 0, rmask = 0, smask = 0;
    const long long c_first = base < 0 ? 0 : base;
    const int re_u = region_of(L.rg.e_start, L.rg.n, c_first);
    const int rh_u = region_of(L.rg.h_start, L.rg.n, c_first < 1 ? 1 : c_first);
    const int qu = L.rg.qm[re_u];
    const bool right_edge = L.has_boundary && base <= nx - 1 && nx - 1 < base + W;
    const bool left_edge = L.has_boundary && base == 0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const long long c = base + i * 32 + lane;
        const long long l = c - L.win_lo;
        const bool in_e = (l >= 0 && l < L.win_n);
        if (in_e) MBG_CHK(l, L.win_n, "run_tile e_in");
        E[i] = in_e ? ld(K.e_in + l) : 0.0;
        if (l >= 0 && l <= L.win_n) MBG_CHK(l, L.win_n + 1, "run_tile h_in");
        H[i] = (l >= 0 && l <= L.win_n) ? ld(K.h_in + l) : 0.0;
        const int re = UNI ? re_u : region_of(L.rg.e_start, L.rg.n, c);
        const int rh = UNI ? rh_u : region_of(L.rg.h_start, L.rg.n, c);
        if (!UNI) {
            ca[i] = L.rg.a[re];
            cbg[i] = L.rg.bg[re];
            cbdx[i] = L.rg.bdx[re];
            cch[i] = L.rg.ch[rh];
        }
        qi[i] = (in_e && c >= 0 && c < nx) ? L.rg.qm[re] : -1;
        hmask |= (c >= 1 && c <= nx - 1) ? 1u << i : 0u;
        emask |= (nx > 1 && c >= 0 && c < nx) ? 1u << i : 0u;
        qmask |= qi[i] >= 0 ? 1u << i : 0u;
        rmask |= (right_edge && c == nx - 1) ? 1u << i : 0u;
        for (int q = 0; q < L.n_src; ++q) smask |= c == L.src_cell[q] ? 1u << i : 0u;
        if (qi[i] >= 0) {
            MBG_CHK(l, L.plane, "run_tile s_in");
            MBG_CHK(2 * L.plane + l, L.plane * L.words, "run_tile s_in plane");
            X[i] = ld(K.s_in + l);
            Y[i] = ld(K.s_in + L.plane + l);
            Z[i] = ld(K.s_in + 2 * L.plane + l);
        } else {
            X[i] = Y[i] = Z[i] = 0.0;
        }
    }
    const double ua = L.rg.a[re_u], ubg = L.rg.bg[re_u], ubdx = L.rg.bdx[re_u], uch = L.rg.ch[rh_u];
    const int qs = qu < 0 ? 0 : qu;
    const double ubgp = pol_coef(ubg, P.rq[qs], P.real_dipole);

    for (int s = 0; s < K.steps; ++s) {
        const long long n = K.n0 + s;
        // ---- H update: needs E[m-1] (left neighbour) -----------------------
        double t[C];
#pragma unroll
        for (int i = 0; i < C; ++i) t[i] = __shfl_sync(kFull, E[i], (lane + 31) & 31);
        double e_right0 = 0.0, h_right0 = 0.0;  // old E[1], H[1] for the left edge
        if (left_edge) {
            e_right0 = __shfl_sync(kFull, E[0], (lane + 1) & 31);
            h_right0 = __shfl_sync(kFull, H[0], (lane + 1) & 31);
        }
        double Hn[C], El[C];
#pragma unroll
        for (int i = 0; i < C; ++i) {
            El[i] = (lane == 0) ? t[i > 0 ? i - 1 : 0] : t[i];
            Hn[i] = ((hmask >> i) & 1u) ? mad(UNI ? uch : cch[i], E[i] - El[i], H[i]) : H[i];
        }
        // ---- density step with E^{n-1} and polarisation rate -----------------
        double p[C];
#pragma unroll
        for (int i = 0; i < C; ++i) {
            p[i] = 0.0;
            if ((qmask >> i) & 1u) {
                const int qq = UNI ? qs : qi[i];
                p[i] = P.real_dipole ? MBG_BLOCH_REAL(P.qm[qq], P.rq[qq], E[i], X[i], Y[i], Z[i])
                                     : bloch_cell(P.qm[qq], E[i], X[i], Y[i], Z[i]);
            }
        }
        // ---- E update: needs H[m+1] (right neighbour) --------------------------
        double u[C];
#pragma unroll
        for (int i = 0; i < C; ++i) u[i] = __shfl_sync(kFull, Hn[i], (lane + 1) & 31);
#pragma unroll
        for (int i = 0; i < C; ++i) {
            const double hr = (lane == 31) ? u[i < C - 1 ? i + 1 : i] : u[i];
            double en = E[i];
            if ((emask >> i) & 1u)
            {
                const double a = UNI ? ua : ca[i], bdx = UNI ? ubdx : cbdx[i];
                const double bgp =
                    UNI ? ubgp : pol_coef(cbg[i], P.rq[qi[i] < 0 ? 0 : qi[i]], P.real_dipole);
                en = a == 1.0 ? e_update<true>(a, bdx, bgp, E[i], hr - Hn[i], p[i])
                              : e_update<false>(a, bdx, bgp, E[i], hr - Hn[i], p[i]);
            }
            if (left_edge && i == 0 && lane == 0) {
                // solver_fdtd.py:372-374
                const double e_at = mad(L.l_c, e_right0, L.l_omc * E[0]);
                const double h_at = 0.5 * (h_right0 + hr);
                en = L.l_hw * mad(L.l_z, h_at, e_at);
            }
            if ((rmask >> i) & 1u) {
                // solver_fdtd.py:375-377 (E[Nx-2] old is the left neighbour)
                const double e_at = mad(L.r_c, El[i], L.r_omc * E[i]);
                const double h_at = 0.5 * (H[i] + Hn[i]);
                en = L.r_hw * mad(-L.r_z, h_at, e_at);
            }
            if ((smask >> i) & 1u) {
                const long long c = base + i * 32 + lane;
                for (int q = 0; q < L.n_src; ++q) {
                    if (c == L.src_cell[q]) {
                        MBG_CHK(n * L.n_src + q, L.num_t * L.n_src, "run_tile src_values");
                        const double v = L.src_values[n * L.n_src + q];
                        en = L.src_hard[q] ? v : en + v;
                    }
                }
            }
            E[i] = en;
            H[i] = Hn[i];
        }
        // ---- non-finite scan and records (owned result cells only) --------------
        const unsigned long long mask = K.mask[s];
        const unsigned char flags = K.check[s];
        const bool check = (flags & MBG_STEP_SCAN) != 0;
        if (mask || flags) {
#pragma unroll
            for (int i = 0; i < C; ++i) {
                const long long c = base + i * 32 + lane;
                const bool own = c >= t_lo && c < t_hi && c >= L.own_lo && c < L.own_hi;
                if (!own) continue;
                if (check && !isfinite(E[i])) atomicMin(L.bad_step, (unsigned long long)n);
                for (int r = 0; r < L.n_rec; ++r) {
                    if (!((mask >> r) & 1ull)) continue;
                    const long long cell = L.rec_cell[r];
                    if (cell >= 0 && cell != c) continue;
                    const long long col = cell >= 0 ? 0 : c - L.rec_col0[r];
                    const long long idx = (n / L.rec_every[r] - L.rec_row0[r]) * L.rec_cols[r] + col;
                    double vre = 0.0, vim = 0.0;
                    switch (L.rec_q[r]) {
                        case MBG_Q_E: vre = E[i]; break;
                        case MBG_Q_H: vre = H[i]; break;
                        case MBG_Q_D:
                        default:
                            if (qi[i] >= 0) {
                                double x, y, z;
                                frame_true(P.frame, qi[i], X[i], Y[i], Z[i], x, y, z);
                                if (L.rec_q[r] == MBG_Q_D)
                                    bloch_entry(L.rec_i[r], L.rec_j[r], x, y, z, vre, vim);
                                else
                                    vre = -z;
                            }
                    }
                    MBG_CHK(idx, L.rec_len[r], "bloch record");
                    L.rec_re[r][idx] = vre;
                    if (L.rec_im[r]) L.rec_im[r][idx] = vim;
                }
            }
            if (L.inv && (flags & MBG_STEP_MONITOR)) {  // eigenvalues (1 +- |v|)/2 (_kernels.py:541-546)
                unsigned long long key = ~0ull;
#pragma unroll
                for (int i = 0; i < C; ++i) {
                    const long long c = base + i * 32 + lane;
                    if (c < t_lo || c >= t_hi || c < L.own_lo || c >= L.own_hi || qi[i] < 0) continue;
                    double x, y, z;
                    frame_true(P.frame, qi[i], X[i], Y[i], Z[i], x, y, z);
                    const unsigned long long kk = order_key(0.5 * (1.0 - sqrt(x * x + y * y + z * z)));
                    key = kk < key ? kk : key;
                }
                fold_min_eig(L.inv, key);
            }
        }
    }
    // ---- write back the tile's result cells -------------------------------------
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const long long c = base + i * 32 + lane;
        if (c < t_lo || c >= t_hi) continue;
        const long long l = c - L.win_lo;
        MBG_CHK(l, L.win_n, "run_tile e_out");
        MBG_CHK(l, L.plane, "run_tile s_out");
        K.e_out[l] = E[i];
        K.h_out[l] = H[i];
        if (qi[i] >= 0) {
            K.s_out[l] = X[i];
            K.s_out[L.plane + l] = Y[i];
            K.s_out[2 * L.plane + l] = Z[i];
        }
    }
}

// record masks / scan flags of the chunk being stepped, staged by the hook
// (read after the first step's barriers)
__shared__ unsigned long long s_mask[kMaxTileSteps];
__shared__ unsigned char s_check[kMaxTileSteps];

// records a tile with result cells [lo, hi) can write: whole-domain records
// and the point records inside the range.  The staged step masks are cut to
// them, so the tiles without a record cell (all but a handful) skip the
// per-cell record loop on record steps (it cost cfg2 ~4 % of its issue slots)
__device__ __forceinline__ unsigned long long range_records(const Launch &L, long long lo, long long hi) {
    unsigned long long m = 0;
    for (int r = 0; r < L.n_rec; ++r) {
        const long long c = L.rec_cell[r];
        if (c < 0 || (c >= lo && c < hi)) m |= 1ull << r;
    }
    return m;
}

// result range [lo, hi) of the CTA tile and its first loaded cell, re-derived
// where they are used instead of being held in registers across the steps:
// from blockIdx and the parameter bank (per-launch kernel) ...
struct LaunchSpan {
    static constexpr bool kPersistent = false;
    const Launch &L;
    __device__ long long lo() const { return L.res_lo + (long long)blockIdx.x * L.tile_own; }
    __device__ long long hi() const {
        const long long h = lo() + L.tile_own;
        return h < L.res_hi ? h : L.res_hi;
    }
    __device__ long long base() const { return tile_base(L, lo()); }
};

// ... or from the item range the persistent kernel staged in shared memory
struct SharedSpan {
    static constexpr bool kPersistent = true;
    const Launch &L;
    const WaveItem &it;
    __device__ long long lo() const { return it.lo; }
    __device__ long long hi() const { return it.hi; }
    __device__ long long base() const { return tile_base(L, it.lo); }
};

// Interior tiles (the overwhelming majority): every slot is a regular cell of
// the window (1 <= c <= Nx-2), one E region and one H region, no source and no
// boundary cell.  A CTA of kBlochWarpsPerBlock warps owns kBlochCtaTile
// consecutive cells; inside a warp the layout is blocked (lane l holds C
// consecutive cells), so the stencil needs one shuffle of E up and one of H
// down per lane and step, and the two cells at each warp seam go through
// double-buffered shared slots (two barriers per step).  For a single quantum
// material the stepper constants are constant-bank operands.
// hook(): runs once the tile's loads are in flight, before the first step
// (the persistent kernel stages its step masks and claims its next item there)
template <bool QM, bool ONE_QM, bool REAL, bool A1, bool MON, class Span, class Hook>
__device__ __forceinline__ void interior_cta(const BlochParams &P, const Chunk &K, const Span &span, int r_e, int r_h,
                                             const Hook &hook) {
    __shared__ double seam_e[2][kBlochWarpsPerBlock], seam_h[2][kBlochWarpsPerBlock];
    const Launch &L = P.L;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double a = L.rg.a[r_e], bg = L.rg.bg[r_e], bdx = L.rg.bdx[r_e], ch = L.rg.ch[r_h];
    const int qmi = QM ? (ONE_QM ? 0 : L.rg.qm[r_e]) : 0;
    const BlochQm &q = P.qm[qmi];
    const double bgp = pol_coef(bg, P.rq[qmi], REAL);
    const long long lane_off = (long long)warp * W + (long long)lane * C;  // this lane's first cell - base
    double E[C], H[C], X[C], Y[C], Z[C];
    const long long l0 = span.base() + lane_off - L.win_lo;
    MBG_CHK(l0, L.win_n, "interior e_in");
    MBG_CHK(l0 + C - 1, L.win_n, "interior e_in");
    if (QM) MBG_CHK(2 * L.plane + l0 + C - 1, L.plane * L.words, "interior s_in");
    if ((l0 & 1) == 0) {  // 16-byte aligned pairs (the usual case: even tile bases, padded planes)
#pragma unroll
        for (int i = 0; i < C; i += 2) {
            ld2(K.e_in + l0 + i, E[i], E[i + 1]);
            ld2(K.h_in + l0 + i, H[i], H[i + 1]);
            if (QM) {
                ld2(K.s_in + l0 + i, X[i], X[i + 1]);
                ld2(K.s_in + L.plane + l0 + i, Y[i], Y[i + 1]);
                ld2(K.s_in + 2 * L.plane + l0 + i, Z[i], Z[i + 1]);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < C; ++i) {
            E[i] = ld(K.e_in + l0 + i);
            H[i] = ld(K.h_in + l0 + i);
            if (QM) {
                X[i] = ld(K.s_in + l0 + i);
                Y[i] = ld(K.s_in + L.plane + l0 + i);
                Z[i] = ld(K.s_in + 2 * L.plane + l0 + i);
            }
        }
    }
    hook();
    // two steps per loop iteration in the persistent kernel's hot instantiation
    // (one real-dipole medium, no monitor): the loop-carried state needs no
    // register copies at the back edge (16 moves per step otherwise) and the
    // seam slot parity is static -- cfg2 5.70e11 -> 5.82e11; the per-launch
    // path of small domains measured 4 % slower unrolled (cfg1), so it stays rolled
#ifndef MBG_BLOCH_UNROLL
#define MBG_BLOCH_UNROLL 2
#endif
    constexpr int kStepUnroll = (Span::kPersistent && QM && ONE_QM && REAL && !MON) ? MBG_BLOCH_UNROLL : 1;
#pragma unroll kStepUnroll
    for (int s = 0; s < K.steps; ++s) {
        const int b = s & 1;
        // H update (uses E^{n-1}); H is overwritten in place with H^{n-1/2}
        if (lane == 31) seam_e[b][warp] = E[C - 1];
        double el0 = __shfl_up_sync(kFull, E[C - 1], 1);
        __syncthreads();
        if (lane == 0 && warp > 0) el0 = seam_e[b][warp - 1];
#pragma unroll
        for (int i = C - 1; i >= 0; --i) H[i] = mad(ch, E[i] - (i == 0 ? el0 : E[i - 1]), H[i]);
        if (lane == 0) seam_h[b][warp] = H[0];
        double hr_last = __shfl_down_sync(kFull, H[0], 1);
        __syncthreads();
        if (lane == 31 && warp < kBlochWarpsPerBlock - 1) hr_last = seam_h[b][warp + 1];
        // density step + E update, slot by slot
#pragma unroll
        for (int i = 0; i < C; ++i) {
            double p = 0.0;
            if (QM) p = REAL ? MBG_BLOCH_REAL(q, P.rq[qmi], E[i], X[i], Y[i], Z[i])
                             : bloch_cell(q, E[i], X[i], Y[i], Z[i]);
            const double hr = i == C - 1 ? hr_last : H[i + 1];
            // p = 0 in classical cells: a E - bg*0 == a E exactly, so the term is dropped
            E[i] = QM ? e_update<A1>(a, bdx, bgp, E[i], hr - H[i], p)
                      : mad(bdx, hr - H[i], (MBG_POL_FOLD && A1) ? E[i] : a * E[i]);
        }
        const unsigned long long mask = s_mask[s];
        const unsigned char flags = s_check[s];
        const bool check = (flags & MBG_STEP_SCAN) != 0;
        if (mask || flags) {
            const long long n = K.n0 + s;
            const long long first = span.base() + lane_off, t_lo = span.lo(), t_hi = span.hi();
#pragma unroll
            for (int i = 0; i < C; ++i) {
                const long long c = first + i;
                if (c < t_lo || c >= t_hi || c < L.own_lo || c >= L.own_hi) continue;
                if (check && !isfinite(E[i])) atomicMin(L.bad_step, (unsigned long long)n);
                for (int r = 0; r < L.n_rec; ++r) {
                    if (!((mask >> r) & 1ull)) continue;
                    const long long cell = L.rec_cell[r];
                    if (cell >= 0 && cell != c) continue;
                    const long long idx = (n / L.rec_every[r] - L.rec_row0[r]) * L.rec_cols[r] + (cell >= 0 ? 0 : c - L.rec_col0[r]);
                    double vre = 0.0, vim = 0.0;
                    switch (L.rec_q[r]) {
                        case MBG_Q_E: vre = E[i]; break;
                        case MBG_Q_H: vre = H[i]; break;
                        case MBG_Q_D:
                        default:
                            if (QM) {
                                double x, y, z;
                                frame_true(P.frame, qmi, X[i], Y[i], Z[i], x, y, z);
                                if (L.rec_q[r] == MBG_Q_D)
                                    bloch_entry(L.rec_i[r], L.rec_j[r], x, y, z, vre, vim);
                                else
                                    vre = -z;
                            }
                    }
                    MBG_CHK(idx, L.rec_len[r], "bloch record");
                    L.rec_re[r][idx] = vre;
                    if (L.rec_im[r]) L.rec_im[r][idx] = vim;
                }
            }
            if (MON && QM && L.inv && (flags & MBG_STEP_MONITOR)) {  // fused invariant monitor (see run_tile)
                unsigned long long key = ~0ull;
#pragma unroll
                for (int i = 0; i < C; ++i) {
                    const long long c = first + i;
                    if (c < t_lo || c >= t_hi || c < L.own_lo || c >= L.own_hi) continue;
                    double x, y, z;
                    frame_true(P.frame, qmi, X[i], Y[i], Z[i], x, y, z);
                    const unsigned long long kk = order_key(0.5 * (1.0 - sqrt(x * x + y * y + z * z)));
                    key = kk < key ? kk : key;
                }
                fold_min_eig(L.inv, key);
            }
        }
    }
    const long long first = span.base() + lane_off, t_lo = span.lo(), t_hi = span.hi();
    const long long o0 = first - L.win_lo;
    if (first >= t_lo && first + C <= t_hi && (o0 & 1) == 0) {  // the whole lane, 16-byte pairs
        MBG_CHK(o0, L.win_n, "interior e_out");
        MBG_CHK(o0 + C - 1, L.win_n, "interior e_out");
#pragma unroll
        for (int i = 0; i < C; i += 2) {
            st2(K.e_out + o0 + i, E[i], E[i + 1]);
            st2(K.h_out + o0 + i, H[i], H[i + 1]);
            if (QM) {
                st2(K.s_out + o0 + i, X[i], X[i + 1]);
                st2(K.s_out + L.plane + o0 + i, Y[i], Y[i + 1]);
                st2(K.s_out + 2 * L.plane + o0 + i, Z[i], Z[i + 1]);
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const long long c = first + i;
        if (c < t_lo || c >= t_hi) continue;
        MBG_CHK(o0 + i, L.win_n, "interior e_out");
        K.e_out[o0 + i] = E[i];
        K.h_out[o0 + i] = H[i];
        if (QM) {
            K.s_out[o0 + i] = X[i];
            K.s_out[L.plane + o0 + i] = Y[i];
            K.s_out[2 * L.plane + o0 + i] = Z[i];
        }
    }
}

// 16 resident warps per SM (128 registers per thread)
#ifndef MBG_BLOCH_MINB
#define MBG_BLOCH_MINB (16 / MBG_BLOCH_WARPS > 0 ? 16 / MBG_BLOCH_WARPS : 1)
#endif
// interior CTA tile: dispatch on the medium (the density step must be the very
// same formula the edge path uses -- bitwise independence of the tiling -- so
// the real-dipole choice is global)
template <class Span, class Hook>
__device__ __forceinline__ void interior_tile(const BlochParams &P, const Chunk &K, const Span &span, const Hook &hook) {
    const Launch &L = P.L;
    const long long base = span.base();
    const int re = region_of(L.rg.e_start, L.rg.n, base), rh = region_of(L.rg.h_start, L.rg.n, base);
    const int qm = L.rg.qm[re];
    const bool a1 = L.rg.a[re] == 1.0;  // lossless region (the fast variant fuses the p term)
    // MON: the fused invariant monitor; the hot single-medium variants get a
    // monitor-free instantiation so the unmonitored step loop is unchanged
    if (qm < 0)
        a1 ? interior_cta<false, true, false, true, false>(P, K, span, re, rh, hook)
           : interior_cta<false, true, false, false, false>(P, K, span, re, rh, hook);
    else if (P.real_dipole && P.n_qm == 1 && !L.inv)
        a1 ? interior_cta<true, true, true, true, false>(P, K, span, re, rh, hook)
           : interior_cta<true, true, true, false, false>(P, K, span, re, rh, hook);
    else if (P.real_dipole && P.n_qm == 1)
        a1 ? interior_cta<true, true, true, true, true>(P, K, span, re, rh, hook)
           : interior_cta<true, true, true, false, true>(P, K, span, re, rh, hook);
    else if (P.real_dipole)
        interior_cta<true, false, true, false, true>(P, K, span, re, rh, hook);
    else
        P.n_qm == 1 ? interior_cta<true, true, false, false, true>(P, K, span, re, rh, hook)
                    : interior_cta<true, false, false, false, true>(P, K, span, re, rh, hook);
}

// General tile as a CTA: the W = 32*C cells of one edge tile with ONE cell
// per thread (kEdgeCtaWarps warps x 32 lanes, blocked by warp), so a step of
// an edge tile costs one cell's dependency chain instead of C cells' worth of
// one warp (run_tile, ~2.6 us per step: the per-launch critical path of small
// domains).  Every per-cell property (coefficients, quantum material, H/E
// update, boundary and source flags) is a register of its thread; neighbours
// come by shuffle, across warps through double-buffered shared seams (two
// barriers per step).  The cell arithmetic is run_tile's, operation for
// operation (bitwise equal to every other path).
constexpr int kEdgeCtaWarps = W / 32;
static_assert(kEdgeCtaWarps * 32 == W, "one cell per thread");

__device__ __forceinline__ void edge_cta(const BlochParams &P, const Chunk &K, long long t_lo, long long t_hi) {
    __shared__ double seam_e[2][kEdgeCtaWarps], seam_h[2][kEdgeCtaWarps];
    const Launch &L = P.L;
    const long long nx = L.num_x;
    const long long base = tile_base(L, t_lo);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long c = base + tid;
    const long long l = c - L.win_lo;
    const bool in_e = (l >= 0 && l < L.win_n);
    if (in_e) MBG_CHK(l, L.win_n, "edge_cta e_in");
    double E = in_e ? ld(K.e_in + l) : 0.0;
    if (l >= 0 && l <= L.win_n) MBG_CHK(l, L.win_n + 1, "edge_cta h_in");
    double H = (l >= 0 && l <= L.win_n) ? ld(K.h_in + l) : 0.0;
    const int re = region_of(L.rg.e_start, L.rg.n, c);
    const int rh = region_of(L.rg.h_start, L.rg.n, c);
    const int qi = (in_e && c >= 0 && c < nx) ? L.rg.qm[re] : -1;
    const double ca = L.rg.a[re], cbdx = L.rg.bdx[re], cch = L.rg.ch[rh];
    const double bgp = pol_coef(L.rg.bg[re], P.rq[qi < 0 ? 0 : qi], P.real_dipole);
    const bool hf = c >= 1 && c <= nx - 1;
    const bool ef = nx > 1 && c >= 0 && c < nx;
    const bool lf = L.has_boundary && base == 0 && tid == 0;  // cell 0
    const bool rf = L.has_boundary && c == nx - 1;
    bool sf = false;
    for (int q = 0; q < L.n_src; ++q) sf |= c == L.src_cell[q];
    double X = 0.0, Y = 0.0, Z = 0.0;
    if (qi >= 0) {
        MBG_CHK(l, L.plane, "edge_cta s_in");
        MBG_CHK(2 * L.plane + l, L.plane * L.words, "edge_cta s_in plane");
        X = ld(K.s_in + l);
        Y = ld(K.s_in + L.plane + l);
        Z = ld(K.s_in + 2 * L.plane + l);
    }
    const bool own_tile = c >= t_lo && c < t_hi;
    const bool own = own_tile && c >= L.own_lo && c < L.own_hi;
    for (int s = 0; s < K.steps; ++s) {
        const long long n = K.n0 + s;
        const int b = s & 1;
        // ---- H update: needs E[m-1] (left neighbour) -------------------------
        if (lane == 31) seam_e[b][warp] = E;
        double El = __shfl_up_sync(kFull, E, 1);
        const double e_right0 = __shfl_down_sync(kFull, E, 1);  // old E[1], H[1] for cell 0
        const double h_right0 = __shfl_down_sync(kFull, H, 1);
        __syncthreads();
        if (lane == 0 && warp > 0) El = seam_e[b][warp - 1];
        const double Hn = hf ? mad(cch, E - El, H) : H;
        // ---- density step with E^{n-1} and polarisation rate -----------------
        double p = 0.0;
        if (qi >= 0)
            p = P.real_dipole ? MBG_BLOCH_REAL(P.qm[qi], P.rq[qi], E, X, Y, Z) : bloch_cell(P.qm[qi], E, X, Y, Z);
        // ---- E update: needs H[m+1] (right neighbour) ---------------------------
        if (lane == 0) seam_h[b][warp] = Hn;
        double hr = __shfl_down_sync(kFull, Hn, 1);
        __syncthreads();
        if (lane == 31 && warp < kEdgeCtaWarps - 1) hr = seam_h[b][warp + 1];
        double en = E;
        if (ef)
            en = ca == 1.0 ? e_update<true>(ca, cbdx, bgp, E, hr - Hn, p) : e_update<false>(ca, cbdx, bgp, E, hr - Hn, p);
        if (lf) {
            // solver_fdtd.py:372-374
            const double e_at = mad(L.l_c, e_right0, L.l_omc * E);
            const double h_at = 0.5 * (h_right0 + hr);
            en = L.l_hw * mad(L.l_z, h_at, e_at);
        }
        if (rf) {
            // solver_fdtd.py:375-377 (E[Nx-2] old is the left neighbour)
            const double e_at = mad(L.r_c, El, L.r_omc * E);
            const double h_at = 0.5 * (H + Hn);
            en = L.r_hw * mad(-L.r_z, h_at, e_at);
        }
        if (sf) {
            for (int q = 0; q < L.n_src; ++q) {
                if (c == L.src_cell[q]) {
                    MBG_CHK(n * L.n_src + q, L.num_t * L.n_src, "edge_cta src_values");
                    const double v = L.src_values[n * L.n_src + q];
                    en = L.src_hard[q] ? v : en + v;
                }
            }
        }
        E = en;
        H = Hn;
        // ---- non-finite scan and records (owned result cells only) ------------
        const unsigned long long mask = K.mask[s];
        const unsigned char flags = K.check[s];
        const bool check = (flags & MBG_STEP_SCAN) != 0;
        if (mask || flags) {
            if (own) {
                if (check && !isfinite(E)) atomicMin(L.bad_step, (unsigned long long)n);
                for (int r = 0; r < L.n_rec; ++r) {
                    if (!((mask >> r) & 1ull)) continue;
                    const long long cell = L.rec_cell[r];
                    if (cell >= 0 && cell != c) continue;
                    const long long col = cell >= 0 ? 0 : c - L.rec_col0[r];
                    const long long idx = (n / L.rec_every[r] - L.rec_row0[r]) * L.rec_cols[r] + col;
                    double vre = 0.0, vim = 0.0;
                    switch (L.rec_q[r]) {
                        case MBG_Q_E: vre = E; break;
                        case MBG_Q_H: vre = H; break;
                        case MBG_Q_D:
                        default:
                            if (qi >= 0) {
                                double x, y, z;
                                frame_true(P.frame, qi, X, Y, Z, x, y, z);
                                if (L.rec_q[r] == MBG_Q_D)
                                    bloch_entry(L.rec_i[r], L.rec_j[r], x, y, z, vre, vim);
                                else
                                    vre = -z;
                            }
                    }
                    MBG_CHK(idx, L.rec_len[r], "edge_cta record");
                    L.rec_re[r][idx] = vre;
                    if (L.rec_im[r]) L.rec_im[r][idx] = vim;
                }
            }
            if (L.inv && (flags & MBG_STEP_MONITOR)) {  // eigenvalues (1 +- |v|)/2 (_kernels.py:541-546)
                unsigned long long key = ~0ull;
                if (own && qi >= 0) {
                    double x, y, z;
                    frame_true(P.frame, qi, X, Y, Z, x, y, z);
                    key = order_key(0.5 * (1.0 - sqrt(x * x + y * y + z * z)));
                }
                fold_min_eig(L.inv, key);
            }
        }
    }
    // ---- write back the tile's result cells -------------------------------------
    if (own_tile) {
        MBG_CHK(l, L.win_n, "edge_cta e_out");
        MBG_CHK(l, L.plane, "edge_cta s_out");
        K.e_out[l] = E;
        K.h_out[l] = H;
        if (qi >= 0) {
            K.s_out[l] = X;
            K.s_out[L.plane + l] = Y;
            K.s_out[2 * L.plane + l] = Z;
        }
    }
}

// one warp over the result range [t_lo, t_hi) of at most 32*C - 2k cells
__device__ __forceinline__ void edge_range(const BlochParams &P, const Chunk &K, long long t_lo, long long t_hi,
                                           int lane) {
    const Launch &L = P.L;
    const long long base = tile_base(L, t_lo);
    const long long lo = base, hi = base + W - 1 < L.num_x ? base + W - 1 : L.num_x - 1;
    const bool uni = region_of(L.rg.e_start, L.rg.n, lo) == region_of(L.rg.e_start, L.rg.n, hi) &&
                     region_of(L.rg.h_start, L.rg.n, lo < 1 ? 1 : lo) ==
                         region_of(L.rg.h_start, L.rg.n, hi < 1 ? 1 : hi);
    if (uni)
        run_tile<true>(P, K, t_lo, t_hi, base, lane);
    else
        run_tile<false>(P, K, t_lo, t_hi, base, lane);
}

// the persistent kernel's edge items of one range (flag 2): the whole CTA
// steps the range's 32C-cell tile one cell per thread (edge_cta), so an edge
// item takes about as long as an interior one -- edge items sit on the
// wavefront's dependency chain, and stepped by single warps at 8 cells per
// lane they made it ~0.45 ms per chunk (2^20 cells: 60 % of the CTA time
// waiting on them).  A call keeps its registers out of the interior path.
static_assert(kEdgeCtaWarps == kBlochWarpsPerBlock, "edge items use the wave CTA as one tile");
__device__ __noinline__ void edge_cta_call(const BlochParams &P, const Chunk &K, long long t_lo, long long t_hi) {
    edge_cta(P, K, t_lo, t_hi);
}

// the persistent kernel's rare edge items: a call keeps the general path's
// register allocation (and spills) out of the interior path
__device__ __noinline__ void edge_range_call(const BlochParams &P, const Chunk &K, long long t_lo, long long t_hi,
                                             int lane) {
    edge_range(P, K, t_lo, t_hi, lane);
}

// interior tiles: one CTA per tile; the whole CTA leaves if its tile is not
// interior (the host hands those to the edge kernel)
__global__ void __launch_bounds__(kBlochWarpsPerBlock * 32, MBG_BLOCH_MINB)
bloch_interior_kernel(const __grid_constant__ BlochParams P) {
    const Launch &L = P.L;
    const LaunchSpan span{L};
    if (span.lo() >= L.res_hi) return;
    if (!tile_is_interior(L, span.base(), kBlochCtaTile)) return;
    interior_tile(P, launch_chunk(L), span, [&]() {
        if (threadIdx.x < L.k) {
            s_mask[threadIdx.x] = L.step_mask[threadIdx.x] & range_records(L, span.lo(), span.hi());
            s_check[threadIdx.x] = L.check[threadIdx.x];
        }
    });
}

// One step launch of the per-launch path: CTAs [0, tiles) are the CTA tiles
// (interior ones step, the others leave), CTAs [tiles, tiles + T.n) the edge
// ranges (edge_cta) -- one kernel, no second stream and no fork/join events
// per launch (the cross-stream pair cost cfg1 ~20 % of its device time)
static_assert(kEdgeCtaWarps == kBlochWarpsPerBlock, "edge ranges run in the step kernel's CTAs");
__global__ void __launch_bounds__(kBlochWarpsPerBlock * 32, MBG_BLOCH_MINB)
bloch_step_kernel(const __grid_constant__ BlochParams P, const __grid_constant__ EdgeTiles T, int tiles) {
    const Launch &L = P.L;
    if ((int)blockIdx.x >= tiles) {
        const int e = (int)blockIdx.x - tiles;
        edge_cta(P, launch_chunk(L), T.lo[e], T.hi[e]);
        return;
    }
    const LaunchSpan span{L};
    if (span.lo() >= L.res_hi) return;
    if (!tile_is_interior(L, span.base(), kBlochCtaTile)) return;
    interior_tile(P, launch_chunk(L), span, [&]() {
        if (threadIdx.x < L.k) {
            s_mask[threadIdx.x] = L.step_mask[threadIdx.x] & range_records(L, span.lo(), span.hi());
            s_check[threadIdx.x] = L.check[threadIdx.x];
        }
    });
}

// the few remaining cells (domain/window edges, region interfaces, sources):
// one CTA per result range of at most 32*C - 2k cells, one cell per thread
// (edge_cta), so these ranges keep pace with the interior CTAs
__global__ void __launch_bounds__(kEdgeCtaWarps * 32)
bloch_edge_kernel(const __grid_constant__ BlochParams P, const __grid_constant__ EdgeTiles T) {
    if ((int)blockIdx.x >= T.n) return;
    edge_cta(P, launch_chunk(P.L), T.lo[blockIdx.x], T.hi[blockIdx.x]);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// record masks / scan flags of every step of a persistent launch, one thread
// per step (the per-launch path computes them on the host: solver_fdtd.py:386-393)
__global__ void wave_mask_kernel(const __grid_constant__ Launch L, long long n_steps, long long last_step,
                                 unsigned long long *masks, unsigned char *checks) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_steps) return;
    const long long n = L.n0 + i;
    unsigned long long m = 0;
    for (int r = 0; r < L.n_rec; ++r)
        if (n % L.rec_every[r] == 0) m |= 1ull << r;
    masks[i] = m;
    checks[i] = step_flags(L, n, last_step);
}

// item's dependencies: items t-1 .. t+1 of the previous chunk.  One pass
// (three acquire loads in flight) or, with wait, spin until they are done.
__device__ bool deps_done(const BlochWave &V, long long item, bool wait) {
    const long long c = item / V.tiles, t = item - c * V.tiles;
    if (c == 0) return true;
    const unsigned *prev = V.done + (c - 1) * V.tiles;
    const long long a = t > 0 ? t - 1 : t, b = t + 1 < V.tiles ? t + 1 : t;
    MBG_CHK((c - 1) * V.tiles + b, (long long)V.n_chunks * V.tiles, "wave done flags");
    unsigned long long deadline = 0;
    for (;;) {
        const unsigned fa = ld_acquire(prev + a), ft = ld_acquire(prev + t), fb = ld_acquire(prev + b);
        if (fa && ft && fb) return true;
        if (!wait) return false;
        if (ld_acquire(V.stall)) return false;
        const unsigned long long now = global_ns();
        if (deadline == 0) {
            deadline = now + 10000000000ull;
        } else if (now > deadline) {
            atomicExch(V.stall, 1u);
            return false;
        }
        __nanosleep(100);
    }
}

// Persistent wavefront kernel (see BlochWave).  A CTA claims its next item
// when it starts the current one and checks the next item's dependencies
// while its warps finish, so between two items there are only the two
// barriers and the release.  Deadlock-free: an item only waits on items with
// smaller tickets, every claimed ticket belongs to a resident CTA, and a CTA
// releases its current item before it waits for its next one.  A wait longer
// than 10 s (a bug, never the schedule) raises the stall flag and every CTA
// drains without waiting.
__global__ void __launch_bounds__(kBlochWarpsPerBlock * 32, MBG_BLOCH_MINB)
bloch_wave_kernel(const __grid_constant__ BlochParams P, const __grid_constant__ BlochWave V) {
    __shared__ unsigned item_s, next_s;
    // the current item's chunk and range live in shared memory: the tile code
    // reads them where it needs them instead of holding them in registers
    // across the step loop (the per-launch kernels read the same from the
    // parameter bank)
    __shared__ Chunk chunk_s;
    __shared__ WaveItem item_range_s;
    __shared__ unsigned long long item_rec_s;  // range_records of the item
    const Launch &L = P.L;
    const long long items = (long long)V.n_chunks * V.tiles;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long warp_own = W - 2 * L.k;
    // thread 0: publish item `item` (chunk pointers, step range, cell range)
    const auto stage = [&](unsigned item) {
        item_s = item;
        if (item >= items) return;
        const int c = (int)(item / V.tiles);
        const long long t = item - (long long)c * V.tiles;
        const int buf = (V.cur + c) & 1;
        chunk_s = Chunk{V.e[buf],     V.h[buf],  V.s[buf], V.e[buf ^ 1], V.h[buf ^ 1],
                        V.s[buf ^ 1], V.n0 + (long long)c * L.k,
                        c == V.n_chunks - 1 ? V.last_steps : L.k, s_mask, s_check};
        MBG_CHK(t, V.tiles, "wave items");
        item_range_s = V.items[t];
        item_rec_s = range_records(L, V.items[t].lo, V.items[t].hi);
    };
    if (threadIdx.x == 0) {
        const unsigned first = atomicAdd(V.ticket, 1u);
        deps_done(V, first, true);
        stage(first);
    }
    __syncthreads();
    for (;;) {
        const long long item = item_s;
        if (item >= items) return;
        if (V.trace && threadIdx.x == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            V.trace[4 * item] = V.trace[4 * item + 1] = global_ns();
            V.trace[4 * item + 3] = sm | ((unsigned long long)blockIdx.x << 32);
        }
        const Chunk &K = chunk_s;
        // with the tile loads in flight: claim the next item, stage the masks
        // (read after the first step's barriers)
        const auto hook = [&]() {
            if (threadIdx.x == 0) next_s = atomicAdd(V.ticket, 1u);
            const long long k0 = K.n0 - V.n0;
            if (threadIdx.x < K.steps) {
                MBG_CHK(k0 + threadIdx.x, (long long)V.n_chunks * L.k, "wave masks");
                s_mask[threadIdx.x] = V.masks[k0 + threadIdx.x] & item_rec_s;
                s_check[threadIdx.x] = V.checks[k0 + threadIdx.x];
            }
        };
        if (!item_range_s.edge) {
            interior_tile(P, K, SharedSpan{L, item_range_s}, hook);
        } else if (item_range_s.edge == 2) {
            const long long lo = item_range_s.lo, hi = item_range_s.hi;
            hook();
            __syncthreads();
            edge_cta_call(P, K, lo, hi);
        } else {
            const long long lo = item_range_s.lo, hi = item_range_s.hi;
            hook();
            __syncthreads();
            const long long n_sub = (hi - lo + warp_own - 1) / warp_own;
            for (long long u = warp; u < n_sub; u += kBlochWarpsPerBlock) {
                const long long sub = lo + u * warp_own;
                edge_range_call(P, K, sub, sub + warp_own < hi ? sub + warp_own : hi, lane);
            }
        }
        // item and next come back from shared memory (nothing stays live in
        // registers across the tile); thread 0 wrote next_s before the tile's barriers
        const unsigned next = next_s;
        const bool ready = threadIdx.x == 0 && next < items ? deps_done(V, next, false) : true;
        __syncthreads();  // every write of the item precedes the release; item_s may be reused
        if (threadIdx.x == 0) {
            const unsigned done_item = item_s;
            if (V.trace) V.trace[4 * done_item + 2] = global_ns();
            __threadfence();
            MBG_CHK(done_item, items, "wave release");
            st_release(V.done + done_item, 1u);
            if (!ready) deps_done(V, next, true);
            stage(next);
        }
        __syncthreads();
    }
}

// batched single points (see BatchParams): one thread per two-level system,
// the reference's rotation order (bloch_cell_real / bloch_cell, the Bloch
// vector in the reference's own frame)
__global__ void bloch_batch_kernel(const __grid_constant__ BlochBatchParams P) {
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= P.B) return;
    const int m = P.medium[b];
    const BlochQm &q = P.qm[m];
    double x = P.state[b], y = P.state[P.B + b], z = P.state[2 * (long long)P.B + b];
    for (long long n = 1; n < P.num_t; ++n) {
        const double e = P.e_seq[(n - 1) * P.B + b];
        if (P.real_dipole)
            bloch_cell_real(q, P.rq[m], e, x, y, z);
        else
            bloch_cell(q, e, x, y, z);
        for (int r = 0; r < P.R.n; ++r) {
            if (n % P.R.every[r]) continue;
            const long long idx = b * P.R.rows[r] + n / P.R.every[r];
            double vre = 0.0, vim = 0.0;
            if (P.R.q[r] == MBG_Q_D)
                bloch_entry(P.R.i[r], P.R.j[r], x, y, z, vre, vim);
            else
                vre = -z;  // inversion (_kernels.py:538-539)
            P.R.re[r][idx] = vre;
            if (P.R.im[r]) P.R.im[r][idx] = vim;
        }
    }
    P.state[b] = x;
    P.state[P.B + b] = y;
    P.state[2 * (long long)P.B + b] = z;
}

}  // namespace

int bloch_cta_tile() { return kBlochCtaTile; }

// One step launch (bloch_step_kernel): the CTA tiles and, in the same grid,
// the edge ranges the host classifies (overflow beyond kMaxEdgeTiles in
// further edge-only launches on the same stream).
cudaError_t launch_bloch(const BlochParams &P, long long tiles, cudaStream_t st, int *kernels) {
    const Launch &L = P.L;
    *kernels = 0;
    // host-side twin of the device classification: collect the non-interior tiles
    EdgeTiles T;
    T.n = 0;
    bool fused = false;  // the first batch of edge ranges rides with the CTA tiles
    cudaError_t err = cudaSuccess;
    auto flush = [&]() -> cudaError_t {
        if (!fused) {
            bloch_step_kernel<<<(unsigned)(tiles + T.n), kBlochWarpsPerBlock * 32, 0, st>>>(P, T, (int)tiles);
            fused = true;
        } else if (T.n > 0) {
            bloch_edge_kernel<<<T.n, kEdgeCtaWarps * 32, 0, st>>>(P, T);
        } else {
            return cudaSuccess;
        }
        ++*kernels;
        T.n = 0;
        return cudaGetLastError();
    };
    const long long warp_own = W - 2 * L.k;  // result cells one edge range can deliver
    for (long long t = 0; t < tiles; ++t) {
        const long long t_lo = L.res_lo + t * L.tile_own;
        if (tile_is_interior(L, tile_base(L, t_lo), kBlochCtaTile)) continue;
        const long long t_hi = t_lo + L.tile_own < L.res_hi ? t_lo + L.tile_own : L.res_hi;
        for (long long lo = t_lo; lo < t_hi; lo += warp_own) {
            T.lo[T.n] = lo;
            T.hi[T.n] = lo + warp_own < t_hi ? lo + warp_own : t_hi;
            if (++T.n == kMaxEdgeTiles && (err = flush()) != cudaSuccess) return err;
        }
    }
    return flush();
}

cudaError_t launch_wave_masks(const Launch &L, long long n_steps, long long last_step, unsigned long long *masks,
                              unsigned char *checks, cudaStream_t st) {
    const unsigned blocks = (unsigned)((n_steps + 255) / 256);
    wave_mask_kernel<<<blocks, 256, 0, st>>>(L, n_steps, last_step, masks, checks);
    return cudaGetLastError();
}

cudaError_t launch_batch_bloch(const BlochBatchParams &P, cudaStream_t st) {
    const unsigned blocks = (unsigned)((P.B + 127) / 128);
    bloch_batch_kernel<<<blocks, 128, 0, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_bloch_wave(const BlochParams &P, const BlochWave &V, cudaStream_t st) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bloch_wave_kernel, kBlochWarpsPerBlock * 32, 0);
    if (err != cudaSuccess) return err;
    const long long items = (long long)V.n_chunks * V.tiles;
    const long long slots = (long long)sms * (per_sm > 0 ? per_sm : 1);
    const unsigned grid = (unsigned)(items < slots ? items : slots);
    bloch_wave_kernel<<<grid, kBlochWarpsPerBlock * 32, 0, st>>>(P, V);
    return cudaGetLastError();
}

}  // namespace MBG_VARIANT
}  // namespace mbg
