// Auxiliary kernels: initial-state broadcast, step-0 sampling, halo packing.
#include "mbg_kernels.h"

namespace mbg {

namespace {

__device__ __forceinline__ int pair_index(int n, int i, int j) { return i * n - i * (i + 1) / 2 + (j - i - 1); }

// DensityKernel.init_state: the same rho0 in every quantum cell
// (_kernels.py:376-377, Bloch form _kernels.py:496-500)
__global__ void broadcast_state_kernel(double *s, long long plane, long long win_n, int words,
                                       const double *w, const Regions rg, long long win_lo) {
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= win_n) return;
    const int r = region_of(rg.e_start, rg.n, win_lo + l);
    const bool qm = rg.qm[r] >= 0;
    for (int k = 0; k < words; ++k) s[k * plane + l] = qm ? w[k] : 0.0;
}

// relaxed-frame state (BlochFrame): map an uploaded true state in (to_frame)
// or the device state out into `out` (true values) for a download
__global__ void frame_kernel(bool to_frame, double *s, long long plane, long long win_n, const Regions rg,
                             long long win_lo, const BlochFrame F, double *out) {
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= win_n) return;
    const int q = rg.qm[region_of(rg.e_start, rg.n, win_lo + l)];
    double *x = s + l, *y = s + plane + l, *z = s + 2 * plane + l;
    if (to_frame) {
        if (q < 0) return;
        *x = *x / F.fxy[q];
        *y = *y / F.fxy[q];
        *z = (*z - F.cz[q]) / F.kz[q];
    } else {
        double a, b, c;
        frame_true(F, q, *x, *y, *z, a, b, c);
        out[l] = a;
        out[win_n + l] = b;
        out[2 * win_n + l] = c;
    }
}

// _sample(step) from the current state (used for row 0, solver_fdtd.py:449)
__global__ void sample_kernel(const Launch L, int levels, int bloch, long long step, const BlochFrame F) {
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L.win_n) return;
    const long long c = L.win_lo + l;
    if (c < L.own_lo || c >= L.own_hi) return;
    const int qm = L.rg.qm[region_of(L.rg.e_start, L.rg.n, c)];
    for (int r = 0; r < L.n_rec; ++r) {
        if (step % L.rec_every[r]) continue;
        const long long cell = L.rec_cell[r];
        if (cell >= 0 && cell != c) continue;
        const long long idx = (step / L.rec_every[r] - L.rec_row0[r]) * L.rec_cols[r] + (cell >= 0 ? 0 : c - L.rec_col0[r]);
        double re = 0.0, im = 0.0;
        const int q = L.rec_q[r];
        if (q == MBG_Q_E) {
            re = L.e_in[l];
        } else if (q == MBG_Q_H) {
            re = L.h_in[l];
        } else if (qm >= 0) {
            const double *s = L.s_in + l;
            const long long P = L.plane;
            if (bloch) {
                double x, y, z;
                frame_true(F, qm, s[0], s[P], s[2 * P], x, y, z);
                if (q == MBG_Q_INV) {
                    re = -z;
                } else {
                    const int i = L.rec_i[r], j = L.rec_j[r];
                    if (i == j) {
                        re = (i == 0) ? 0.5 * (1.0 + z) : 0.5 * (1.0 - z);
                    } else {
                        re = 0.5 * x;
                        im = (i == 0) ? 0.5 * -y : 0.5 * y;
                    }
                }
            } else if (q == MBG_Q_INV) {
                re = s[P] - s[0];
            } else {
                const int i = L.rec_i[r], j = L.rec_j[r], n = levels;
                if (i == j) {
                    re = s[i * P];
                } else if (i < j) {
                    const int w = n + 2 * pair_index(n, i, j);
                    re = s[w * P];
                    im = s[(w + 1) * P];
                } else {
                    const int w = n + 2 * pair_index(n, j, i);
                    re = s[w * P];
                    im = -s[(w + 1) * P];
                }
            }
        }
        L.rec_re[r][idx] = re;
        if (L.rec_im[r]) L.rec_im[r][idx] = im;
    }
}

// ghost exchange: [E | H | state planes] x count cells starting at local l0
__global__ void halo_kernel(bool pack, double *e, double *h, double *s, long long plane, int words, long long l0,
                            long long count, double *buf) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)(2 + words) * count;
    if (t >= total) return;
    const long long w = t / count, c = t % count, l = l0 + c;
    double *p = (w == 0) ? e + l : (w == 1) ? h + l : s + (w - 2) * plane + l;
    if (pack)
        buf[t] = *p;
    else
        *p = buf[t];
}

// 16 independent FMA chains per thread keep the DFMA pipe busy
__global__ void __launch_bounds__(256) fp64_fma_kernel(double *out, int iters, double m, double c) {
    double a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = 1e-3 * (threadIdx.x + k);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fma(a[k], m, c);
    }
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) sum += a[k];
    if (sum == 12345.678) out[0] = sum;  // keep the chains alive
}

// ---- invariant monitor (solver_fdtd.py:428-440, _kernels.py:394-401, 541-546) ----
// order-preserving uint64 key of a double (for atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = __double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// smallest eigenvalue of a complex Hermitian n x n matrix (n <= 8) through the
// real symmetric 2n x 2n embedding [[Re, -Im], [Im, Re]] and cyclic Jacobi
__device__ double min_eigenvalue(const double *re, const double *im, int n) {
    double a[16][16];
    const int m = 2 * n;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            a[i][j] = a[i + n][j + n] = re[i * n + j];
            a[i + n][j] = im[i * n + j];
            a[i][j + n] = -im[i * n + j];
        }
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, scale = 0.0;
        for (int p = 0; p < m; ++p) {
            scale += a[p][p] * a[p][p];
            for (int q = p + 1; q < m; ++q) off += a[p][q] * a[p][q];
        }
        if (off <= 1e-32 * (scale + 1e-300)) break;
        for (int p = 0; p < m; ++p)
            for (int q = p + 1; q < m; ++q) {
                const double apq = a[p][q];
                if (apq == 0.0) continue;
                const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int k = 0; k < m; ++k) {
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - sn * akq;
                    a[k][q] = sn * akp + c * akq;
                }
                for (int k = 0; k < m; ++k) {
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - sn * aqk;
                    a[q][k] = sn * apk + c * aqk;
                }
            }
    }
    double mn = a[0][0];
    for (int p = 1; p < m; ++p) mn = fmin(mn, a[p][p]);
    return mn;
}

__global__ void invariants_kernel(const Launch L, int levels, int bloch, const BlochFrame F,
                                  unsigned long long *out) {
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L.win_n) return;
    const long long c = L.win_lo + l;
    if (c < L.own_lo || c >= L.own_hi) return;
    const int qm = L.rg.qm[region_of(L.rg.e_start, L.rg.n, c)];
    if (qm < 0) return;
    const double *s = L.s_in + l;
    const long long P = L.plane;
    double trace_dev = 0.0, min_eig;
    if (bloch) {
        // eigenvalues (1 +- |v|)/2; trace and Hermiticity exact in this form
        double x, y, z;
        frame_true(F, qm, s[0], s[P], s[2 * P], x, y, z);
        min_eig = 0.5 * (1.0 - sqrt(x * x + y * y + z * z));
    } else {
        const int n = levels;
        double re[64], im[64], tr = 0.0;
        for (int i = 0; i < n; ++i) {
            re[i * n + i] = s[i * P];
            im[i * n + i] = 0.0;
            tr += re[i * n + i];
        }
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                const int w = n + 2 * pair_index(n, i, j);
                re[i * n + j] = re[j * n + i] = s[w * P];
                im[i * n + j] = s[(w + 1) * P];
                im[j * n + i] = -s[(w + 1) * P];
            }
        trace_dev = fabs(tr - 1.0);
        min_eig = min_eigenvalue(re, im, n);
    }
    atomicMax(&out[0], dkey(trace_dev));
    atomicMin(&out[2], dkey(min_eig));
}

unsigned blocks_for(long long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

cudaError_t measure_fp64_peak(double *ms, double *flops) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *out = nullptr;
    cudaError_t err = cudaMalloc(&out, sizeof(double));
    if (err != cudaSuccess) return err;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        fp64_fma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float t = 0.f;
        cudaEventElapsedTime(&t, a, b);
        if (rep > 0 && t < best) best = t;
    }
    err = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *ms = best;
    *flops = 2.0 * 16.0 * iters * (double)blocks * threads;
    return err;
}

cudaError_t launch_frame(bool to_frame, double *s, long long plane, long long win_n, const Regions &rg,
                         long long win_lo, const BlochFrame &F, double *out, cudaStream_t st) {
    if (win_n <= 0) return cudaSuccess;
    frame_kernel<<<blocks_for(win_n, 256), 256, 0, st>>>(to_frame, s, plane, win_n, rg, win_lo, F, out);
    return cudaGetLastError();
}

cudaError_t launch_invariants(const Launch &L, int levels, int bloch, const BlochFrame &F, unsigned long long *out,
                              cudaStream_t st) {
    if (L.win_n <= 0) return cudaSuccess;
    invariants_kernel<<<blocks_for(L.win_n, 128), 128, 0, st>>>(L, levels, bloch, F, out);
    return cudaGetLastError();
}

cudaError_t launch_sample(const Launch &L, int levels, int bloch, long long step, const BlochFrame &F,
                          cudaStream_t st) {
    if (L.win_n <= 0) return cudaSuccess;
    sample_kernel<<<blocks_for(L.win_n, 256), 256, 0, st>>>(L, levels, bloch, step, F);
    return cudaGetLastError();
}

cudaError_t launch_broadcast_state(double *s, long long plane, long long win_n, int words, const double *w,
                                   const Regions &rg, long long win_lo, cudaStream_t st) {
    if (win_n <= 0 || words == 0) return cudaSuccess;
    broadcast_state_kernel<<<blocks_for(win_n, 256), 256, 0, st>>>(s, plane, win_n, words, w, rg, win_lo);
    return cudaGetLastError();
}

cudaError_t launch_halo(bool pack, double *e, double *h, double *s, long long plane, int words, long long l0,
                        long long count, double *buf, cudaStream_t st) {
    const long long total = (long long)(2 + words) * count;
    if (total <= 0) return cudaSuccess;
    halo_kernel<<<blocks_for(total, 256), 256, 0, st>>>(pack, e, h, s, plane, words, l0, count, buf);
    return cudaGetLastError();
}

}  // namespace mbg
