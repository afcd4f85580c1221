// Fused time-step kernels for N-level media, N = 2 (RK4) and 3..8.
//
// One thread per cell, one CTA per tile of dense_tile_width consecutive cells, k
// time steps per launch (temporal tiling with redundant halos, as in the
// two-level kernel).  The per-cell density matrix never leaves the SM while
// the launch runs: it is Hermitian-packed (N real diagonal words, then re/im
// of the upper triangle in row-major order) in registers for N <= 4 and in a
// per-thread shared-memory column for larger N (G always in registers).  E and H live in registers;
// neighbours are exchanged through two small double-buffered shared arrays
// (two barriers per step).
//
// Splitting step (_kernels.py:87-160, quantum.py:444-460), same mathematics,
// restructured for registers:
//   r1 = relax_half(rho)                                    quantum.py:425-428
//   G  = (I + iA)^-1 by in-place Gauss-Jordan, no pivoting   (|leading minors| >= 1)
//   U  = 2G - I  ( = (I + iA)^-1 (I - iA), the Cayley unitary of quantum.py:431-441 )
//   rho' = U r1 U^H row by row (upper triangle), relax_half(rho')
//   p = pol_factor * [sum_{i<j} 2 Re(mu_ij (rho'-rho)_ji) + sum_i mu_ii (rho'-rho)_ii]
// RK4 step (_kernels.py:256-332): classical RK4 of the master equation on the
// packed Hermitian state (the reference symmetrises after each step).
#pragma once
#include "mbg_kernels.h"

#ifndef MBG_VARIANT
#error "compile with -DMBG_VARIANT=fast|exact"
#endif

namespace mbg {
namespace MBG_VARIANT {
namespace dense {

// tile width (threads = cells per CTA); the largest state layouts use 64
template <int N, bool RK4>
constexpr int tile_width() { return dense_tile_width(N, RK4); }

// packed word index of upper pair (i < j), row-major
__host__ __device__ constexpr int pair_index(int n, int i, int j) { return i * n - i * (i + 1) / 2 + (j - i - 1); }
__host__ __device__ constexpr int wre(int n, int i, int j) { return n + 2 * pair_index(n, i, j); }
__host__ __device__ constexpr int wim(int n, int i, int j) { return n + 2 * pair_index(n, i, j) + 1; }

template <int NW>
struct RegVec {
    double v[NW];
    __device__ __forceinline__ double &operator[](int w) { return v[w]; }
};
template <int TW>
struct SmemVec {
    double *p;  // this thread's column; word w at p[w * TW]
    __device__ __forceinline__ double &operator[](int w) { return p[w * TW]; }
};
template <int N>
struct RegMat {
    double re[N * N], im[N * N];
    __device__ __forceinline__ double &r(int i, int j) { return re[i * N + j]; }
    __device__ __forceinline__ double &m(int i, int j) { return im[i * N + j]; }
};
// Hermitian element (i, j) of a packed state
template <int N, class V>
__device__ __forceinline__ void herm(V &s, int i, int j, double &re, double &im) {
    if (i == j) {
        re = s[i];
        im = 0.0;
    } else if (i < j) {
        re = s[wre(N, i, j)];
        im = s[wim(N, i, j)];
    } else {
        re = s[wre(N, j, i)];
        im = -s[wim(N, j, i)];
    }
}

// 1/d for a normal positive d (|pivot|^2 of (I + iA)/2 is >= 1/4): the fast
// variant refines the hardware seed (error 2^-22) once, cubically, no special-case branch
__device__ __forceinline__ double recip_pos(double d) {
#if defined(MBG_EXACT) && MBG_EXACT
    return 1.0 / d;
#else
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    const double e = fma(-d, r, 1.0);  // one cubically convergent step r + r(e + e^2)
    return fma(r, fma(e, e, e), r);
#endif
}

// symmetric complex matrix as two upper triangles (row-major, i <= j)
template <int N>
struct SymMat {
    double re[N * (N + 1) / 2], im[N * (N + 1) / 2];
    static constexpr int at(int i, int j) {
        return i <= j ? i * N - i * (i - 1) / 2 + (j - i) : j * N - j * (j - 1) / 2 + (i - j);
    }
    __device__ __forceinline__ double &r(int i, int j) { return re[at(i, j)]; }
    __device__ __forceinline__ double &m(int i, int j) { return im[at(i, j)]; }
};

#ifndef MBG_OPERAND_STATIONARY
#define MBG_OPERAND_STATIONARY 1
#endif
template <int N, class VA, class VB, class MG, class VR>
__device__ __forceinline__ double congruence(const DenseQm<N> &q, VA &A, VB &B, MG &G, VR &raw);

// ---------------------------------------------------------------------------
// splitting: A holds rho (in/out), B is scratch for r1, G scratch N x N complex
template <int N, bool RA, class VA, class VB, class MG, class VR>
__device__ __forceinline__ double split_cell(const DenseQm<N> &q, double e, VA &A, VB &B, MG &G, VR &raw) {
    // relaxation half step -> B
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double acc = q.pop[i * N] * A[0];
#pragma unroll
        for (int j = 1; j < N; ++j) acc = mad(q.pop[i * N + j], A[j], acc);
        B[i] = acc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
            B[wre(N, i, j)] = A[wre(N, i, j)] * q.coh[i * N + j];
            B[wim(N, i, j)] = A[wim(N, i, j)] * q.coh[i * N + j];
        }
#ifndef MBG_SPLIT_FENCE
#define MBG_SPLIT_FENCE (N >= 7 ? 3 : 1)
#endif
    // compiler fences (bit 0 here, bit 1 per congruence row): the state words
    // are re-read from shared memory where used again instead of being held
    // (spilled) across the inversion.  Measured on cfg4: none 4.77e9, bit 0
    // 4.92e9 (1588 -> 324 spill bytes), bits 0+1 4.54e9 (120 spill bytes),
    // bit 1 alone 4.54e9 -- at six levels the per-row fence costs more
    // schedule freedom than the spills it removes.  At seven and eight levels
    // (G alone is 98 / 128 registers) it is the other way round: the shared
    // memory of the resident CTAs leaves no L1 for local memory, every spill
    // access runs at L2 latency, and the row fence cuts the spills from 8.7 KB
    // to 0.7 KB (N = 7: 1.35e9 -> 2.57e9) and from 48 KB to 4.4 KB (N = 8)
    if constexpr ((MBG_SPLIT_FENCE & 1) != 0) asm volatile("" ::: "memory");
    if constexpr (RA) {
        // Real Hamiltonian and dipole (fast variant): A real symmetric, so
        // U = (I + iA)^-1 (I - iA) = (2P - I) - 2iAP with P = (I + A^2)^-1 real
        // symmetric, and AP symmetric too: both parts of U live as upper
        // triangles (N(N+1) words instead of 2N^2).  (I + A^2)/2 (SPD, ~I/2) is
        // inverted by the symmetric sweep operator (no pivoting), which ends at
        // -((I + A^2)/2)^-1 = -2P.
        SymMat<N> S;
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = i; j < N; ++j) S.m(i, j) = mad(e, q.bf_im[i * N + j], q.bc_im[i * N + j]);  // A/2
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = i; j < N; ++j) {
                double acc = S.m(i, 0) * S.m(0, j);
#pragma unroll
                for (int k = 1; k < N; ++k) acc = mad(S.m(i, k), S.m(k, j), acc);
                S.r(i, j) = mad(2.0, acc, i == j ? 0.5 : 0.0);  // (I + A^2)/2 = I/2 + 2 (A/2)^2
            }
#pragma unroll
        for (int k = 0; k < N; ++k) {  // sweep k: a_ij -= a_ik a_kj / a_kk, a_ik /= a_kk, a_kk = -1/a_kk
            const double d = recip_pos(S.r(k, k));
            double t[N];
#pragma unroll
            for (int i = 0; i < N; ++i) t[i] = i == k ? 0.0 : S.r(i, k) * d;
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = i; j < N; ++j)
                    if (i != k && j != k) S.r(i, j) = mad(-t[i], S.r(k, j), S.r(i, j));
#pragma unroll
            for (int i = 0; i < N; ++i)
                if (i != k) S.r(i, k) = t[i];
            S.r(k, k) = -d;
        }
        // Im U = -2AP = -4 (A/2) P = 2 (A/2) S.r, in place from the last row up:
        // row i reads A/2 at (i, k >= i) -- its own, rewritten after the row
        // -- and at (k < i, i), rows not rewritten yet
#pragma unroll
        for (int i = N - 1; i >= 0; --i) {
            double t[N];
#pragma unroll
            for (int j = i; j < N; ++j) {
                double acc = S.m(i, 0) * S.r(0, j);
#pragma unroll
                for (int k = 1; k < N; ++k) acc = mad(S.m(i, k), S.r(k, j), acc);
                t[j] = 2.0 * acc;
            }
#pragma unroll
            for (int j = i; j < N; ++j) S.m(i, j) = t[j];
        }
        // Re U = 2P - I = -S.r - I
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = i; j < N; ++j) S.r(i, j) = i == j ? -S.r(i, j) - 1.0 : -S.r(i, j);
        return congruence<N>(q, A, B, S, raw);
    } else {
        // G = (B/2)^-1 = 2 (I + iA)^-1: the host halves bc and bf (exact), so the
        // Gauss-Jordan inverse (in place, no pivoting) is already 2(I + iA)^-1
#pragma unroll
        for (int i = 0; i < N * N; ++i) {
            G.r(i / N, i % N) = mad(e, q.bf_re[i], q.bc_re[i]);
            G.m(i / N, i % N) = mad(e, q.bf_im[i], q.bc_im[i]);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const double pr = G.r(k, k), pi = G.m(k, k);
            const double rd = recip_pos(mad(pi, pi, pr * pr));
            const double ir = pr * rd, ii = -pi * rd;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                if (j == k) continue;
                const double xr = G.r(k, j), xi = G.m(k, j);
                G.r(k, j) = mad(xr, ir, -(xi * ii));
                G.m(k, j) = mad(xr, ii, xi * ir);
            }
            G.r(k, k) = ir;
            G.m(k, k) = ii;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                if (i == k) continue;
                const double fr = G.r(i, k), fi = G.m(i, k);
#if MBG_OPERAND_STATIONARY
                // the row factor stays the shared multiplier of consecutive DFMAs (see congruence)
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (j != k) G.r(i, j) = mad(fi, G.m(k, j), G.r(i, j));
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (j != k) G.m(i, j) = mad(-fi, G.r(k, j), G.m(i, j));
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (j != k) G.r(i, j) = mad(-fr, G.r(k, j), G.r(i, j));
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (j != k) G.m(i, j) = mad(-fr, G.m(k, j), G.m(i, j));
#else
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    if (j == k) continue;
                    const double kr = G.r(k, j), ki = G.m(k, j);
                    G.r(i, j) = mad(-fr, kr, mad(fi, ki, G.r(i, j)));
                    G.m(i, j) = mad(-fr, ki, mad(-fi, kr, G.m(i, j)));
                }
#endif
                G.r(i, k) = mad(-fr, ir, fi * ii);
                G.m(i, k) = mad(-fr, ii, -(fi * ir));
            }
        }
        // U = 2(I + iA)^-1 - I = G - I
#pragma unroll
        for (int i = 0; i < N; ++i) G.r(i, i) -= 1.0;
        return congruence<N>(q, A, B, G, raw);
    }
}

// rho' = U r1 U^H, one row at a time; second relaxation half step and the
// polarisation trace fused (_kernels.py:87-160)
template <int N, class VA, class VB, class MG, class VR>
__device__ __forceinline__ double congruence(const DenseQm<N> &q, VA &A, VB &B, MG &G, VR &raw) {
    double acc_p = 0.0;  // raw[i]: row i's diagonal before the second half relaxation
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if constexpr ((MBG_SPLIT_FENCE & 2) != 0) asm volatile("" ::: "memory");  // per row
        double tr[N], ti[N];
#if MBG_OPERAND_STATIONARY
        // Operand-stationary order: consecutive DFMAs share one multiplier
        // register (an element of U's row, then of T's row), so the operand
        // reuse cache serves it and each instruction reads two fresh 64-bit
        // operands instead of three -- the register file feeds the FP64 pipe
        // one 64-bit operand per cycle against one warp DFMA per two cycles
        // (tools/fp64_peaks.py: 24.7 TFLOP/s with three fresh operands, 28.2
        // with a shared multiplier, 36.9 with a uniform operand).
#pragma unroll
        for (int k = 0; k < N; ++k) tr[k] = ti[k] = 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) {
            const double ur = G.r(i, m), ui = G.m(i, m);
            double rr[N], ri[N];  // row m of r1
#pragma unroll
            for (int k = 0; k < N; ++k) {
                if (k == m) {
                    rr[k] = B[m];
                    ri[k] = 0.0;
                } else {
                    herm<N>(B, m, k, rr[k], ri[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < N; ++k) tr[k] = mad(ur, rr[k], tr[k]);
#pragma unroll
            for (int k = 0; k < N; ++k) ti[k] = mad(ui, rr[k], ti[k]);
#pragma unroll
            for (int k = 0; k < N; ++k)
                if (k != m) tr[k] = mad(-ui, ri[k], tr[k]);
#pragma unroll
            for (int k = 0; k < N; ++k)
                if (k != m) ti[k] = mad(ur, ri[k], ti[k]);
        }
        double oar[N], oai[N];
#pragma unroll
        for (int j = i; j < N; ++j) oar[j] = oai[j] = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
#pragma unroll
            for (int j = i; j < N; ++j) oar[j] = mad(tr[k], G.r(j, k), oar[j]);
#pragma unroll
            for (int j = i + 1; j < N; ++j) oai[j] = mad(-tr[k], G.m(j, k), oai[j]);
#pragma unroll
            for (int j = i; j < N; ++j) oar[j] = mad(ti[k], G.m(j, k), oar[j]);
#pragma unroll
            for (int j = i + 1; j < N; ++j) oai[j] = mad(ti[k], G.r(j, k), oai[j]);
        }
#pragma unroll
        for (int j = i; j < N; ++j) {
            const double ar = oar[j], ai = oai[j];
            if (j == i) {
                raw[i] = ar;
            } else {
                const double c = q.coh[i * N + j];
                const double fr = ar * c, fi = ai * c;
                const int p = pair_index(N, i, j);
                acc_p += 2.0 * mad(q.pol.pol_im[p], fi - A[wim(N, i, j)], q.pol.pol_re[p] * (fr - A[wre(N, i, j)]));
                A[wre(N, i, j)] = fr;
                A[wim(N, i, j)] = fi;
            }
        }
#else
#pragma unroll
        for (int k = 0; k < N; ++k) {
            double ar = 0.0, ai = 0.0;
#pragma unroll
            for (int m = 0; m < N; ++m) {
                const double ur = G.r(i, m), ui = G.m(i, m);
                if (m == k) {  // real diagonal of r1
                    const double rr = B[m];
                    ar = mad(ur, rr, ar);
                    ai = mad(ui, rr, ai);
                } else {
                    double rr, ri;
                    herm<N>(B, m, k, rr, ri);
                    ar = mad(ur, rr, mad(-ui, ri, ar));
                    ai = mad(ur, ri, mad(ui, rr, ai));
                }
            }
            tr[k] = ar;
            ti[k] = ai;
        }
#pragma unroll
        for (int j = i; j < N; ++j) {
            double ar = 0.0, ai = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const double ur = G.r(j, k), ui = G.m(j, k);  // conj(U_jk) = ur - i ui
                ar = mad(tr[k], ur, mad(ti[k], ui, ar));
                if (j != i) ai = mad(ti[k], ur, mad(-tr[k], ui, ai));  // diagonal is real
            }
            if (j == i) {
                raw[i] = ar;  // raw diagonal; relaxed below (A keeps the old one until then)
            } else {
                const double c = q.coh[i * N + j];
                const double fr = ar * c, fi = ai * c;
                const int p = pair_index(N, i, j);
                acc_p += 2.0 * mad(q.pol.pol_im[p], fi - A[wim(N, i, j)], q.pol.pol_re[p] * (fr - A[wre(N, i, j)]));
                A[wre(N, i, j)] = fr;
                A[wim(N, i, j)] = fi;
            }
        }
#endif
    }
    double nd[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double acc = q.pop[i * N] * raw[0];
#pragma unroll
        for (int j = 1; j < N; ++j) acc = mad(q.pop[i * N + j], raw[j], acc);
        nd[i] = acc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc_p = mad(q.pol.pol_dv[i], nd[i] - A[i], acc_p);
        A[i] = nd[i];
    }
    return q.pol.pol_factor * acc_p;
}

// One k term of the commutator [H, S]_ij: (a s - t b) accumulated into (cr, ci)
// for complex a = H_ik, s = S_kj, t = S_ik, b = H_kj.  The exact variant keeps
// the reference's grouping (two rounded products per part, their difference
// added: 12 FP64 instructions per term without contraction); the fast variant
// accumulates the same eight products as one FMA chain per part (8
// instructions, each product rounded once into the sum).
__device__ __forceinline__ void comm_term(double ar, double ai, double sr, double si, double tr, double ti, double br,
                                          double bi, double &cr, double &ci) {
#if defined(MBG_EXACT) && MBG_EXACT
    cr += mad(ar, sr, -(ai * si)) - mad(tr, br, -(ti * bi));
    ci += mad(ar, si, ai * sr) - mad(tr, bi, ti * br);
#else
    cr = fma(ti, bi, fma(-tr, br, fma(-ai, si, fma(ar, sr, cr))));
    ci = fma(-ti, br, fma(-tr, bi, fma(ai, sr, fma(ar, si, ci))));
#endif
}
// real H: (a s - t b) with real a, b
__device__ __forceinline__ void comm_term_real(double ar, double sr, double si, double tr, double ti, double br,
                                               double &cr, double &ci) {
#if defined(MBG_EXACT) && MBG_EXACT
    cr += mad(ar, sr, -(tr * br));
    ci += mad(ar, si, -(ti * br));
#else
    cr = fma(-tr, br, fma(ar, sr, cr));
    ci = fma(-ti, br, fma(ar, si, ci));
#endif
}

// ---------------------------------------------------------------------------
// RK4: f(src) = -i/hbar [H, src] + D(src) on packed Hermitian states.
// Only the upper triangle + diagonal of the (Hermitian) derivative is formed.
// RH (fast variant, real H0 and dipole): H real, the commutator in half the
// operations.
template <int N, bool RH, class VS, class VD>
__device__ __forceinline__ void master_rhs(const Rk4Qm<N> &q, const double *hr, const double *hi, VS &src, VD &dst) {
    constexpr double kInvHbar = 1.0 / 1.054571817e-34;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i; j < N; ++j) {
            // [H, S]_ij = sum_k H_ik S_kj - S_ik H_kj
            double cr = 0.0, ci = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                double sr, si, tr, ti;
                herm<N>(src, k, j, sr, si);
                herm<N>(src, i, k, tr, ti);
                const double ar = hr[i * N + k], br = hr[k * N + j];
                if constexpr (RH) {
                    comm_term_real(ar, sr, si, tr, ti, br, cr, ci);
                } else {
                    const double ai = hi[i * N + k], bi = hi[k * N + j];
                    comm_term(ar, ai, sr, si, tr, ti, br, bi, cr, ci);
                }
            }
            // -i/hbar * (cr + i ci) = (ci/hbar, -cr/hbar)
            double dr = ci * kInvHbar, di = -cr * kInvHbar;
            if (i == j) {
                double acc = q.popm[i * N] * src[0];
#pragma unroll
                for (int m = 1; m < N; ++m) acc = mad(q.popm[i * N + m], src[m], acc);
                dst[i] = dr + acc;
            } else {
                const double g = q.deph[i * N + j];
                dst[wre(N, i, j)] = mad(-g, src[wre(N, i, j)], dr);
                dst[wim(N, i, j)] = mad(-g, src[wim(N, i, j)], di);
            }
        }
}

// Same derivative for N >= 4 from H = h0 - E mu held packed (Hermitian: N
// real diagonal words, re/im of the upper pairs; RH: the imaginary words are
// zero and never read), formed once per cell step for the four stages.  The
// stage source A + c K is formed while it is read into registers, so no stage
// buffer is kept in shared memory; dst may be K itself (every source word is
// read before the first write).  The fence keeps the compiler from holding
// shared-memory words in registers across stages (N = 6: 4456 -> 0 spill bytes).
template <int N, bool RH, class VH>
__device__ __forceinline__ void herm_h(VH &hp, int i, int j, double &re, double &im) {
    if constexpr (RH) {
        re = i == j ? hp[i] : (i < j ? hp[wre(N, i, j)] : hp[wre(N, j, i)]);
        im = 0.0;
    } else {
        herm<N>(hp, i, j, re, im);
    }
}

template <int N, bool RH, class VA, class VK, class VD>
__device__ __forceinline__ void master_rhs_packed(const Rk4Qm<N> &q, RegVec<N * N> &hp, VA &a0, VK &k0, double c,
                                                  VD &dst) {
    constexpr double kInvHbar = 1.0 / 1.054571817e-34;
    asm volatile("" ::: "memory");
    RegVec<N * N> src;
#pragma unroll
    for (int w = 0; w < N * N; ++w) src[w] = c == 0.0 ? a0[w] : mad(c, k0[w], a0[w]);  // c is a literal per call
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i; j < N; ++j) {
            // [H, S]_ij = sum_k H_ik S_kj - S_ik H_kj
            double cr = 0.0, ci = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                double sr, si, tr, ti, ar, ai, br, bi;
                herm<N>(src, k, j, sr, si);
                herm<N>(src, i, k, tr, ti);
                herm_h<N, RH>(hp, i, k, ar, ai);
                herm_h<N, RH>(hp, k, j, br, bi);
                if constexpr (RH)
                    comm_term_real(ar, sr, si, tr, ti, br, cr, ci);
                else
                    comm_term(ar, ai, sr, si, tr, ti, br, bi, cr, ci);
            }
            const double dr = ci * kInvHbar, di = -cr * kInvHbar;
            if (i == j) {
                double acc = q.popm[i * N] * src[0];
#pragma unroll
                for (int m = 1; m < N; ++m) acc = mad(q.popm[i * N + m], src[m], acc);
                dst[i] = dr + acc;
            } else {
                const double g = q.deph[i * N + j];
                dst[wre(N, i, j)] = mad(-g, src[wre(N, i, j)], dr);
                dst[wim(N, i, j)] = mad(-g, src[wim(N, i, j)], di);
            }
        }
}

// Classical RK4 on the packed state.  Registers (N <= 3): explicit stage
// state S.  Shared memory (N >= 4): S is never stored -- each derivative reads
// A + c K on the fly (the same mad(c, K, A) values), three buffers instead of four.
template <int N, bool RH, class VA, class VB>
__device__ __forceinline__ double rk4_cell(const Rk4Qm<N> &q, double e, VA &A, VB &S, VB &K, VB &Acc) {
    constexpr int NW = N * N;
    constexpr int NH = N >= 4 ? 1 : N * N;
    double hr[NH], hi[NH];
    if constexpr (N < 4) {
#pragma unroll
        for (int i = 0; i < N * N; ++i) {
            hr[i] = mad(-e, q.mu_re[i], q.h0_re[i]);
            hi[i] = mad(-e, q.mu_im[i], q.h0_im[i]);
        }
    }
    const double dt = q.dt;
    if constexpr (N >= 4) {
        RegVec<NW> hp;  // H = h0 - E mu, packed (_kernels.py:270-272)
#pragma unroll
        for (int i = 0; i < N; ++i) {
            hp[i] = mad(-e, q.mu_re[i * N + i], q.h0_re[i * N + i]);
#pragma unroll
            for (int j = i + 1; j < N; ++j) {
                hp[wre(N, i, j)] = mad(-e, q.mu_re[i * N + j], q.h0_re[i * N + j]);
                hp[wim(N, i, j)] = RH ? 0.0 : mad(-e, q.mu_im[i * N + j], q.h0_im[i * N + j]);
            }
        }
        master_rhs_packed<N, RH>(q, hp, A, K, 0.0, K);  // k1
#pragma unroll
        for (int w = 0; w < NW; ++w) Acc[w] = K[w];
        master_rhs_packed<N, RH>(q, hp, A, K, 0.5 * dt, K);  // k2
#pragma unroll
        for (int w = 0; w < NW; ++w) Acc[w] = mad(2.0, K[w], Acc[w]);
        master_rhs_packed<N, RH>(q, hp, A, K, 0.5 * dt, K);  // k3
#pragma unroll
        for (int w = 0; w < NW; ++w) Acc[w] = mad(2.0, K[w], Acc[w]);
        master_rhs_packed<N, RH>(q, hp, A, K, dt, K);  // k4
        asm volatile("" ::: "memory");
    } else {
        master_rhs<N, RH>(q, hr, hi, A, K);  // k1
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            Acc[w] = K[w];
            S[w] = mad(0.5 * dt, K[w], A[w]);
        }
        master_rhs<N, RH>(q, hr, hi, S, K);  // k2
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            Acc[w] = mad(2.0, K[w], Acc[w]);
            S[w] = mad(0.5 * dt, K[w], A[w]);
        }
        master_rhs<N, RH>(q, hr, hi, S, K);  // k3
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            Acc[w] = mad(2.0, K[w], Acc[w]);
            S[w] = mad(dt, K[w], A[w]);
        }
        master_rhs<N, RH>(q, hr, hi, S, K);  // k4
    }
    const double sixth = dt / 6.0;
    double acc_p = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
            const int p = pair_index(N, i, j);
            const double nr = mad(sixth, Acc[wre(N, i, j)] + K[wre(N, i, j)], A[wre(N, i, j)]);
            const double ni = mad(sixth, Acc[wim(N, i, j)] + K[wim(N, i, j)], A[wim(N, i, j)]);
            acc_p += 2.0 * mad(q.pol.pol_im[p], ni - A[wim(N, i, j)], q.pol.pol_re[p] * (nr - A[wre(N, i, j)]));
            A[wre(N, i, j)] = nr;
            A[wim(N, i, j)] = ni;
        }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double nd = mad(sixth, Acc[i] + K[i], A[i]);
        acc_p = mad(q.pol.pol_dv[i], nd - A[i], acc_p);
        A[i] = nd;
    }
    return q.pol.pol_factor * acc_p;
}

// ---------------------------------------------------------------------------
// the fused step kernel

template <int N, bool RK4>
struct Layout {
    static constexpr int NW = N * N;
    static constexpr bool kRegState = RK4 ? (N <= 3) : (N <= 4);
    // smem words per thread: A/B (or A/K/Acc for RK4) when not in registers; G is always in registers
    static constexpr int kStateWords = kRegState ? 0 : (RK4 ? 3 * NW : 2 * NW);
    // shared-memory splitting: the congruence's raw diagonal in shared memory too
    static constexpr int kRawWords = (RK4 || kRegState) ? 0 : N;
    static constexpr int kFieldWords = 6;  // Es[2], Hs[2], Ho[2]
    static constexpr int TW = tile_width<N, RK4>();
    static constexpr size_t smem_bytes() {
        return sizeof(double) * TW * (kFieldWords + kStateWords + kRawWords);
    }
};

template <int N, bool RK4, bool RA, class Q>
__device__ __forceinline__ double cell_step(const Q &q, double e, double *col, RegVec<N * N> &A) {
    using Lay = Layout<N, RK4>;
    constexpr int NW = N * N, TW = Lay::TW;
    if constexpr (RK4) {
        if constexpr (Lay::kRegState) {
            RegVec<NW> S, K, Acc;
            return rk4_cell<N, RA>(q, e, A, S, K, Acc);
        } else {
            SmemVec<TW> As{col}, K{col + NW * TW}, Acc{col + 2 * NW * TW};
            return rk4_cell<N, RA>(q, e, As, K, K, Acc);  // S unused (stage states formed on the fly)
        }
    } else {
        if constexpr (Lay::kRegState) {
            RegVec<NW> B;
            RegMat<N> G;
            RegVec<N> raw;
            return split_cell<N, RA>(q, e, A, B, G, raw);
        } else {
            SmemVec<TW> As{col}, B{col + NW * TW}, raw{col + 2 * NW * TW};
            RegMat<N> G;
            return split_cell<N, RA>(q, e, As, B, G, raw);
        }
    }
}

// One tile of the fused step.  INTERIOR: every cell regular, one E and one H
// region, no source/boundary (no per-cell predicates, scalar coefficients);
// ONE_QM: the stepper constants are compile-time offsets into the parameter
// block (constant-bank operands of the FP64 instructions).
// Register economy around the density step when the state lives in shared
// memory (N >= 5, at the 255-register limit): the cell's E and new H are
// re-read from the shared exchange slots after the step, the E-update
// coefficients are read after it and the cell / window indices re-derived
// from the tile base where used, so little but the step's own values is live
// across it (cfg4 4.32e9 -> 4.64e9).  Register-state kernels (N <= 4) and
// RK4 keep them in registers, which measured faster there.
template <int N, bool RK4, class Q, bool INTERIOR, bool ONE_QM, bool RA>
__device__ __forceinline__ void dense_tile(const DenseParams<N, Q> &P, double *sm, long long t_lo, long long t_hi,
                                           long long base) {
    using Lay = Layout<N, RK4>;
    constexpr int NW = N * N, W = Lay::TW;
    double *Es = sm, *Hs = sm + 2 * W, *Ho = sm + 4 * W;
    double *col = sm + 6 * W + threadIdx.x;  // per-thread state column
    const Launch &L = P.L;
    const long long nx = L.num_x;
#ifndef MBG_LEAN_MIN_N
#define MBG_LEAN_MIN_N 5
#endif
    // splitting N >= MBG_LEAN_MIN_N (RK4 measured 1.5 % slower lean)
    constexpr bool kLean = !RK4 && (!Lay::kRegState || N >= MBG_LEAN_MIN_N);
    const int j = threadIdx.x;
    const long long c0 = base + j, l0 = c0 - L.win_lo;
    const auto cell = [&]() { return kLean ? base + j : c0; };
    const auto loc = [&]() { return kLean ? base + j - L.win_lo : l0; };
    const bool in_e = INTERIOR || (l0 >= 0 && l0 < L.win_n && c0 < nx);
    if (in_e) MBG_CHK(l0, L.win_n, "dense e_in");
    double E = in_e ? L.e_in[l0] : 0.0;
    if (INTERIOR || (l0 >= 0 && l0 <= L.win_n)) MBG_CHK(l0, L.win_n + 1, "dense h_in");
    double H = (INTERIOR || (l0 >= 0 && l0 <= L.win_n)) ? L.h_in[l0] : 0.0;
    const int re = region_of(L.rg.e_start, L.rg.n, INTERIOR ? base : c0);
    const int rh = region_of(L.rg.h_start, L.rg.n, INTERIOR ? base : c0);
    const int qi = in_e ? L.rg.qm[re] : -1;
    // E-update coefficients: held from here (register state) or read per step (lean)
    const double ca0 = kLean ? 0.0 : L.rg.a[re], cbg0 = kLean ? 0.0 : L.rg.bg[re];
    const double cbdx0 = kLean ? 0.0 : L.rg.bdx[re], cch0 = kLean ? 0.0 : L.rg.ch[rh];
    const Q &q = P.qm[ONE_QM ? 0 : (qi < 0 ? 0 : qi)];
    RegVec<NW> rA;
    if (qi >= 0) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            MBG_CHK(l0, L.plane, "dense s_in");
            MBG_CHK(w * L.plane + l0, L.plane * L.words, "dense s_in plane");
            const double v = L.s_in[w * L.plane + l0];
            if constexpr (Lay::kRegState) rA[w] = v; else col[w * W] = v;
        }
    }
    const bool own0 = c0 >= t_lo && c0 < t_hi && c0 >= L.own_lo && c0 < L.own_hi;
    const auto own = [&]() {
        if constexpr (kLean) {
            const long long c = cell();
            return c >= t_lo && c < t_hi && c >= L.own_lo && c < L.own_hi;
        } else {
            return own0;
        }
    };
    const auto upd_h = [&]() { return INTERIOR || (cell() >= 1 && cell() <= nx - 1); };
    const auto upd_e = [&]() { return INTERIOR || (nx > 1 && cell() >= 0 && cell() < nx); };

    for (int s = 0; s < L.k; ++s) {
        const long long n = L.n0 + s;
        const int b = (s & 1) * W;
        double en, hn;
        if (INTERIOR && qi < 0) {
            // Classical interior tile (one region, so the branch is uniform over
            // the CTA): no density step to hide a second barrier behind, so the
            // old E and H are published together and each thread forms its right
            // neighbour's new H itself -- the neighbour's own expression on the
            // same operands, bit for bit -- one barrier per step instead of two
            // (passive sections cost 15 % of an active three-level cell before:
            // 13 % of cfg3's time)
            Es[b + j] = E;
            Hs[b + j] = H;
            __syncthreads();
            const double ch = kLean ? L.rg.ch[rh] : cch0;
            const double ca = kLean ? L.rg.a[re] : ca0, cbg = kLean ? L.rg.bg[re] : cbg0;
            const double cbdx = kLean ? L.rg.bdx[re] : cbdx0;
            const double el = j > 0 ? Es[b + j - 1] : 0.0;
            hn = mad(ch, E - el, H);
            const double hr = j < W - 1 ? mad(ch, Es[b + j + 1] - E, Hs[b + j + 1]) : 0.0;
            en = mad(cbdx, hr - hn, mad(ca, E, -(cbg * 0.0)));
        } else {
        Es[b + j] = E;
        if (!INTERIOR) Ho[b + j] = H;
        __syncthreads();
        const double el = j > 0 ? Es[b + j - 1] : 0.0;
        const double hn0 = upd_h() ? mad(kLean ? L.rg.ch[rh] : cch0, E - el, H) : H;
        Hs[b + j] = hn0;
        double p = 0.0;
        if (qi >= 0) p = cell_step<N, RK4, RA>(q, E, col, rA);
        __syncthreads();
        // lean: E and H of this cell back from the exchange slots (not live across the step)
        if constexpr (kLean) E = Es[b + j];
        hn = kLean ? Hs[b + j] : hn0;
        const double hr = j < W - 1 ? Hs[b + j + 1] : 0.0;
        const double ca = kLean ? L.rg.a[re] : ca0, cbg = kLean ? L.rg.bg[re] : cbg0;
        const double cbdx = kLean ? L.rg.bdx[re] : cbdx0;
        en = upd_e() ? mad(cbdx, hr - hn, mad(ca, E, -(cbg * p))) : E;
        if (!INTERIOR) {
            const long long c = cell();
            if (L.has_boundary && base == 0 && j == 0) {
                const double e_at = mad(L.l_c, Es[b + 1], L.l_omc * E);
                const double h_at = 0.5 * (Ho[b + 1] + hr);
                en = L.l_hw * mad(L.l_z, h_at, e_at);
            }
            if (L.has_boundary && c == nx - 1) {
                const double e_at = mad(L.r_c, el, L.r_omc * E);
                const double h_at = 0.5 * (Ho[b + j] + hn);
                en = L.r_hw * mad(-L.r_z, h_at, e_at);
            }
            for (int qq = 0; qq < L.n_src; ++qq) {
                if (c == L.src_cell[qq]) {
                    MBG_CHK(n * L.n_src + qq, L.num_t * L.n_src, "dense src_values");
                    const double v = L.src_values[n * L.n_src + qq];
                    en = L.src_hard[qq] ? v : en + v;
                }
            }
        }
        }
        E = en;
        H = hn;
        const unsigned long long mask = L.step_mask[s];
        const bool check = (L.check[s] & MBG_STEP_SCAN) != 0;
        if ((mask || check) && own()) {
            const long long c = cell();
            if (check && !isfinite(E)) atomicMin(L.bad_step, (unsigned long long)n);
            for (int r = 0; r < L.n_rec; ++r) {
                if (!((mask >> r) & 1ull)) continue;
                const long long rc = L.rec_cell[r];
                if (rc >= 0 && rc != c) continue;
                const long long idx = (n / L.rec_every[r] - L.rec_row0[r]) * L.rec_cols[r] + (rc >= 0 ? 0 : c - L.rec_col0[r]);
                double vre = 0.0, vim = 0.0;
                const int qq = L.rec_q[r];
                if (qq == MBG_Q_E) {
                    vre = E;
                } else if (qq == MBG_Q_H) {
                    vre = H;
                } else if (qi >= 0) {
                    if constexpr (Lay::kRegState) {
                        RegVec<NW> &A = rA;
                        if (qq == MBG_Q_D) {
                            // runtime (i, j): walk the compile-time index space
#pragma unroll
                            for (int a = 0; a < N; ++a)
#pragma unroll
                                for (int bb = 0; bb < N; ++bb)
                                    if (a == L.rec_i[r] && bb == L.rec_j[r]) herm<N>(A, a, bb, vre, vim);
                        } else {
                            vre = A[1] - A[0];
                        }
                    } else {
                        SmemVec<W> A{col};
                        if (qq == MBG_Q_D) {
                            const int a = L.rec_i[r], bb = L.rec_j[r];
                            if (a == bb) {
                                vre = A[a];
                            } else if (a < bb) {
                                vre = A[wre(N, a, bb)];
                                vim = A[wim(N, a, bb)];
                            } else {
                                vre = A[wre(N, bb, a)];
                                vim = -A[wim(N, bb, a)];
                            }
                        } else {
                            vre = A[1] - A[0];
                        }
                    }
                }
                MBG_CHK(idx, L.rec_len[r], "dense record");
                L.rec_re[r][idx] = vre;
                if (L.rec_im[r]) L.rec_im[r][idx] = vim;
            }
        }
    }
    const long long c = cell();
    if (c >= t_lo && c < t_hi) {
        const long long l = loc();
        MBG_CHK(l, L.win_n, "dense e_out");
        MBG_CHK(l, L.plane, "dense s_out");
        L.e_out[l] = E;
        L.h_out[l] = H;
        if (qi >= 0) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                if constexpr (Lay::kRegState) L.s_out[w * L.plane + l] = rA[w];
                else L.s_out[w * L.plane + l] = col[w * W];
            }
        }
    }
}

template <int N, bool RK4, class Q, bool RA>
__device__ __forceinline__ void dense_dispatch(const DenseParams<N, Q> &P, double *sm, long long t_lo, long long t_hi,
                                               long long base) {
    using Lay = Layout<N, RK4>;
    if (tile_is_interior(P.L, base, Lay::TW)) {
        if (P.n_qm == 1)
            dense_tile<N, RK4, Q, true, true, RA>(P, sm, t_lo, t_hi, base);
        else
            dense_tile<N, RK4, Q, true, false, RA>(P, sm, t_lo, t_hi, base);
    } else {
        dense_tile<N, RK4, Q, false, false, RA>(P, sm, t_lo, t_hi, base);
    }
}

template <int N, bool RK4, class Q, int MINB>
__global__ void __launch_bounds__(Layout<N, RK4>::TW, MINB) dense_step_kernel(const __grid_constant__ DenseParams<N, Q> P) {
    using Lay = Layout<N, RK4>;
    extern __shared__ double sm[];
    const Launch &L = P.L;
    const long long t_lo = L.res_lo + (long long)blockIdx.x * L.tile_own;
    if (t_lo >= L.res_hi) return;  // uniform per block
    const long long t_hi = t_lo + L.tile_own < L.res_hi ? t_lo + L.tile_own : L.res_hi;
    const long long base = tile_base(L, t_lo);
#if defined(MBG_EXACT) && MBG_EXACT
    constexpr bool kRa = false;  // the exact variant keeps the reference's complex arithmetic
#else
    // real operators (the choice is per run, from the host's exact test):
    // symmetric-triangle U for the splitting step, real H for RK4
    constexpr bool kRa = true;
#endif
    if (kRa && P.real_a)
        dense_dispatch<N, RK4, Q, kRa>(P, sm, t_lo, t_hi, base);
    else
        dense_dispatch<N, RK4, Q, false>(P, sm, t_lo, t_hi, base);
}

// ---------------------------------------------------------------------------
// batched single points: one thread per system, all steps in one launch
template <int N, bool RK4, class Q, bool RA>
__global__ void __launch_bounds__(Layout<N, RK4>::TW, dense_min_blocks(N, RK4))
    dense_batch_kernel(const __grid_constant__ BatchParams<N, Q> P) {
    using Lay = Layout<N, RK4>;
    constexpr int NW = N * N, W = Lay::TW;
    extern __shared__ double sm[];
    double *col = sm + 6 * W + threadIdx.x;  // same column layout as the step kernel
    const long long b = (long long)blockIdx.x * W + threadIdx.x;
    if (b >= P.B) return;  // no barriers below
    const Q &q = P.qm[P.medium[b]];
    RegVec<NW> rA;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const double v = P.state[w * (long long)P.B + b];
        if constexpr (Lay::kRegState) rA[w] = v; else col[w * W] = v;
    }
    for (long long n = 1; n < P.num_t; ++n) {
        cell_step<N, RK4, RA>(q, P.e_seq[(n - 1) * P.B + b], col, rA);
        for (int r = 0; r < P.R.n; ++r) {
            if (n % P.R.every[r]) continue;
            const long long idx = b * P.R.rows[r] + n / P.R.every[r];
            const int a = P.R.i[r], c = P.R.j[r];
            double vre = 0.0, vim = 0.0;
            if (P.R.q[r] == MBG_Q_INV) {  // two-level inversion rho_11 - rho_00 (_kernels.py:391-392)
                if constexpr (Lay::kRegState) vre = rA[1] - rA[0];
                else vre = col[W] - col[0];
            } else if constexpr (Lay::kRegState) {
#pragma unroll
                for (int u = 0; u < N; ++u)
#pragma unroll
                    for (int v = 0; v < N; ++v)
                        if (u == a && v == c) herm<N>(rA, u, v, vre, vim);
            } else {
                SmemVec<W> A{col};
                if (a == c) {
                    vre = A[a];
                } else if (a < c) {
                    vre = A[wre(N, a, c)];
                    vim = A[wim(N, a, c)];
                } else {
                    vre = A[wre(N, c, a)];
                    vim = -A[wim(N, c, a)];
                }
            }
            P.R.re[r][idx] = vre;
            if (P.R.im[r]) P.R.im[r][idx] = vim;
        }
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) P.state[w * (long long)P.B + b] = Lay::kRegState ? rA[w] : col[w * W];
}

}  // namespace dense
}  // namespace MBG_VARIANT
}  // namespace mbg
