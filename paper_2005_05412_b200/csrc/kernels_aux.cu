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
            MBG_CHK(l, P, "sample s_in");
            MBG_CHK((long long)(L.words - 1) * P + l, P * L.words, "sample s_in plane");
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
        MBG_CHK(idx, L.rec_len[r], "sample record");
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
    MBG_CHK(l, plane, "halo cell");  // the host checks the window range (mbg_pack_halo / mbg_unpack_halo)
    double *p = (w == 0) ? e + l : (w == 1) ? h + l : s + (w - 2) * plane + l;
    if (pack)
        buf[t] = *p;
    else
        *p = buf[t];
}

// Peer-memory ghost exchange (no library collective on the data path).  The
// receiver owns a mailbox per interface: two slots of [E | H | state planes] x
// count doubles and one 64-bit sequence flag per slot.  The sender's push
// kernel stores its edge cells straight into the receiver's slot -- peer
// device memory mapped through CUDA IPC, NVLink stores on a multi-GPU box --
// and the last block to finish publishes the period's sequence number with a
// system-scope release; the receiver's pull kernel acquires the flag and
// copies the slot into its ghost cells.  Neither kernel is ever waited on by
// the sender, so the exchange cannot deadlock; a strip that does not arrive
// within the timeout sets the handle's sticky stall flag (bit 1) instead.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long aux_global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double *halo_word(double *e, double *h, double *s, long long plane, long long l0,
                                             long long count, long long t) {
    const long long w = t / count, l = l0 + t % count;
    MBG_CHK(l, plane, "halo cell");
    return (w == 0) ? e + l : (w == 1) ? h + l : s + (w - 2) * plane + l;
}

__global__ void __launch_bounds__(256) halo_push_kernel(double *e, double *h, double *s, long long plane, int words,
                                                        long long l0, long long count, double *slot,
                                                        unsigned long long *flag, unsigned long long seq,
                                                        unsigned *ticket) {
    const long long total = (long long)(2 + words) * count;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x)
        slot[t] = *halo_word(e, h, s, plane, l0, count, t);
    __threadfence_system();  // this thread's stores before its block's ticket
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned done = atomicAdd(ticket, 1u);
        if (done == gridDim.x - 1) {  // every block's stores are ordered before its ticket
            *ticket = 0;              // re-armed for the next push on this stream
            __threadfence_system();
            st_release_sys(flag, seq);
        }
    }
}

__global__ void __launch_bounds__(256) halo_pull_kernel(double *e, double *h, double *s, long long plane, int words,
                                                        long long l0, long long count, const double *slot,
                                                        const unsigned long long *flag, unsigned long long seq,
                                                        unsigned long long timeout_ns, unsigned *stall) {
    __shared__ int arrived;
    if (threadIdx.x == 0) {
        const unsigned long long t0 = aux_global_ns();
        int ok = 1;
        while (ld_acquire_sys(flag) < seq) {
            if (aux_global_ns() - t0 > timeout_ns) {
                ok = 0;
                atomicOr(stall, 2u);
                break;
            }
            __nanosleep(200);
        }
        arrived = ok;
    }
    __syncthreads();
    if (!arrived) return;  // ghosts stay stale; the host reports the stall at its next synchronisation
    const long long total = (long long)(2 + words) * count;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x)
        *halo_word(e, h, s, plane, l0, count, t) = __ldcg(slot + t);
}

// FP64 roofline probes: 16 independent FMA chains per thread keep the DFMA
// pipe busy; the operand pattern decides the rate.  MODE 1: two registers and
// a uniform addend (a[k] = a[k] * b[k] + c) -- the pipe's peak, the roofline
// denominator (36.9 TFLOP/s measured, 99 % of the nominal 37.2); MODE 0: the
// multiplier and addend are two registers shared by every instruction, served
// by the operand reuse cache (33.6); MODE 2: one multiplier register shared by
// the 16 consecutive DFMAs (a[k] = x * b[k] + a[k], 28.2); MODE 3: three
// DISTINCT register operands per DFMA (a[k] = a[k] * b[k] + d[k]), what
// matrix-times-matrix code issues when every operand is fresh (24.7).  The
// register file delivers one 64-bit operand per cycle to the FP64 pipe, which
// issues a warp DFMA every two cycles: three fresh operands cost three cycles.
template <int MODE>
__global__ void __launch_bounds__(256) fp64_fma_operand_kernel(double *out, int iters, double m, double c) {
    double a[16], b[16], d[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        a[k] = 1e-3 * (threadIdx.x + k);
        b[k] = m - 1e-9 * (threadIdx.x + 3 * k);
        d[k] = c * (1 + k) + 1e-12 * threadIdx.x;
    }
    double x = m - 1e-8 * threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (MODE == 0) a[k] = fma(a[k], x, d[0]);
            if (MODE == 3) a[k] = fma(a[k], b[k], d[k]);
            if (MODE == 2) a[k] = fma(x, b[k], a[k]);
            if (MODE == 1) a[k] = fma(a[k], b[k], c);
        }
        if (MODE == 2) x = -x;  // keeps |a| bounded (alternating sum); one extra DADD-class op per 16
    }
    double sum = x;
#pragma unroll
    for (int k = 0; k < 16; ++k) sum += a[k];
    if (sum == 12345.678) out[0] = sum;
}

// ---- invariant monitor (solver_fdtd.py:428-440, _kernels.py:394-401, 541-546) ----
// order-preserving uint64 key of a double (for atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = __double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// smallest eigenvalue of a complex Hermitian N x N matrix by cyclic complex
// Jacobi: each off-diagonal element's phase is moved into its column/row, then
// a real plane rotation zeroes it (a quarter of the real 2N x 2N embedding's
// work, compile-time indices so the matrix stays in registers)
template <int N>
__device__ double min_eigenvalue_herm(double (&re)[N * N], double (&im)[N * N]) {
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, scale = 0.0;
#pragma unroll
        for (int p = 0; p < N; ++p) {
            scale += re[p * N + p] * re[p * N + p];
#pragma unroll
            for (int q = p + 1; q < N; ++q) off += re[p * N + q] * re[p * N + q] + im[p * N + q] * im[p * N + q];
        }
        if (off <= 1e-32 * (scale + 1e-300)) break;
#pragma unroll
        for (int p = 0; p < N; ++p)
#pragma unroll
            for (int q = p + 1; q < N; ++q) {
                const double ar = re[p * N + q], ai = im[p * N + q];
                const double mag = sqrt(ar * ar + ai * ai);
                if (mag == 0.0) continue;
                const double ur = ar / mag, ui = ai / mag;  // a_pq = mag u
                // column q times conj(u), row q times u: a_pq becomes mag, a_qq unchanged
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    if (k == q) continue;
                    const double xr = re[k * N + q], xi = im[k * N + q];
                    re[k * N + q] = xr * ur + xi * ui;
                    im[k * N + q] = xi * ur - xr * ui;
                    re[q * N + k] = re[k * N + q];
                    im[q * N + k] = -im[k * N + q];
                }
                const double theta = (re[q * N + q] - re[p * N + p]) / (2.0 * mag);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                const double app = re[p * N + p], aqq = re[q * N + q];
                re[p * N + p] = app - t * mag;
                re[q * N + q] = aqq + t * mag;
                re[p * N + q] = im[p * N + q] = re[q * N + p] = im[q * N + p] = 0.0;
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    if (k == p || k == q) continue;
                    const double pr = re[k * N + p], pi = im[k * N + p];
                    const double qr = re[k * N + q], qi = im[k * N + q];
                    re[k * N + p] = c * pr - sn * qr;
                    im[k * N + p] = c * pi - sn * qi;
                    re[k * N + q] = sn * pr + c * qr;
                    im[k * N + q] = sn * pi + c * qi;
                    re[p * N + k] = re[k * N + p];
                    im[p * N + k] = -im[k * N + p];
                    re[q * N + k] = re[k * N + q];
                    im[q * N + k] = -im[k * N + q];
                }
            }
    }
    double mn = re[0];
#pragma unroll
    for (int p = 1; p < N; ++p) mn = fmin(mn, re[p * N + p]);
    return mn;
}

template <int N>
__device__ double packed_min_eigenvalue(const double *s, long long P, double &tr) {
    double re[N * N], im[N * N];
    tr = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        re[i * N + i] = s[i * P];
        im[i * N + i] = 0.0;
        tr += re[i * N + i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
            const int w = N + 2 * pair_index(N, i, j);
            re[i * N + j] = re[j * N + i] = s[w * P];
            im[i * N + j] = s[(w + 1) * P];
            im[j * N + i] = -s[(w + 1) * P];
        }
    return min_eigenvalue_herm<N>(re, im);
}

// per-cell (|trace - 1|, min eigenvalue); false for cells without a density matrix
__device__ __forceinline__ bool cell_invariants(const Launch &L, int levels, int bloch, const BlochFrame &F,
                                                long long l, double &trace_dev, double &min_eig) {
    if (l >= L.win_n) return false;
    const long long c = L.win_lo + l;
    if (c < L.own_lo || c >= L.own_hi) return false;
    const int qm = L.rg.qm[region_of(L.rg.e_start, L.rg.n, c)];
    if (qm < 0) return false;
    const double *s = L.s_in + l;
    const long long P = L.plane;
    trace_dev = 0.0;
    if (bloch) {
        // eigenvalues (1 +- |v|)/2; trace and Hermiticity exact in this form
        double x, y, z;
        frame_true(F, qm, s[0], s[P], s[2 * P], x, y, z);
        min_eig = 0.5 * (1.0 - sqrt(x * x + y * y + z * z));
    } else {
        double tr = 0.0;
        switch (levels) {
            case 2: min_eig = packed_min_eigenvalue<2>(s, P, tr); break;
            case 3: min_eig = packed_min_eigenvalue<3>(s, P, tr); break;
            case 4: min_eig = packed_min_eigenvalue<4>(s, P, tr); break;
            case 5: min_eig = packed_min_eigenvalue<5>(s, P, tr); break;
            case 6: min_eig = packed_min_eigenvalue<6>(s, P, tr); break;
            case 7: min_eig = packed_min_eigenvalue<7>(s, P, tr); break;
            default: min_eig = packed_min_eigenvalue<8>(s, P, tr); break;
        }
        trace_dev = fabs(tr - 1.0);
    }
    return true;
}

// warp and block reductions first: one pair of atomics per block, not per
// cell (4M same-address atomics cost milliseconds per monitor step)
__global__ void __launch_bounds__(128) invariants_kernel(const Launch L, int levels, int bloch, const BlochFrame F,
                                                         unsigned long long *out) {
    __shared__ unsigned long long s_max[4], s_min[4];
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double tdev = 0.0, mev = 0.0;
    unsigned long long kmax = dkey(0.0), kmin = ~0ull;
    if (cell_invariants(L, levels, bloch, F, l, tdev, mev)) {
        kmax = dkey(tdev);
        kmin = dkey(mev);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmax, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmin, o);
        kmax = a > kmax ? a : kmax;
        kmin = b < kmin ? b : kmin;
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_max[w] = kmax;
        s_min[w] = kmin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            kmax = s_max[i] > kmax ? s_max[i] : kmax;
            kmin = s_min[i] < kmin ? s_min[i] : kmin;
        }
        atomicMax(&out[0], kmax);
        if (kmin != ~0ull) atomicMin(&out[2], kmin);
    }
}

unsigned blocks_for(long long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

cudaError_t measure_fp64_peak_operands(int mode, double *ms, double *flops) {
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
        if (mode == 3) fp64_fma_operand_kernel<3><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        else if (mode == 0) fp64_fma_operand_kernel<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        else if (mode == 2) fp64_fma_operand_kernel<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        else fp64_fma_operand_kernel<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
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
        fp64_fma_operand_kernel<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
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

// the same DFMA chains back to back for at least `seconds` (one event pair
// around the whole train): the throughput a kernel that runs for seconds
// sees under the clocks and power of sustained FP64 load
cudaError_t measure_fp64_sustained(double seconds, double *ms, double *flops) {
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
    fp64_fma_operand_kernel<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);  // warm
    cudaEventRecord(a);
    cudaEventSynchronize(a);
    long long launches = 0;
    float t = 0.f;
    while (t < 1e3 * seconds) {  // batches of 64 launches (~80 ms), timed as one train
        for (int i = 0; i < 64; ++i) fp64_fma_operand_kernel<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        launches += 64;
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t, a, b);
    }
    err = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *ms = t;
    *flops = 2.0 * 16.0 * iters * (double)blocks * threads * (double)launches;
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

static unsigned halo_blocks(long long total) {
    const long long b = (total + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 64 ? 64 : b));
}

cudaError_t launch_halo_push(double *e, double *h, double *s, long long plane, int words, long long l0,
                             long long count, double *slot, unsigned long long *flag, unsigned long long seq,
                             unsigned *ticket, cudaStream_t st) {
    const long long total = (long long)(2 + words) * count;
    halo_push_kernel<<<halo_blocks(total), 256, 0, st>>>(e, h, s, plane, words, l0, count, slot, flag, seq, ticket);
    return cudaGetLastError();
}

cudaError_t launch_halo_pull(double *e, double *h, double *s, long long plane, int words, long long l0,
                             long long count, const double *slot, const unsigned long long *flag,
                             unsigned long long seq, unsigned long long timeout_ns, unsigned *stall,
                             cudaStream_t st) {
    const long long total = (long long)(2 + words) * count;
    halo_pull_kernel<<<halo_blocks(total), 256, 0, st>>>(e, h, s, plane, words, l0, count, slot, flag, seq,
                                                        timeout_ns, stall);
    return cudaGetLastError();
}

}  // namespace mbg
