// C ABI of libmbgpu.so (declared in include/mbgpu.h).
//
// Owns the device state of one run (or of one slab of a multi-GPU run):
// ping-pong buffers for E, H and the density state planes, the per-step
// source samples, the record buffers and the non-finite flag.  mbg_advance
// is the replacement of FdtdSolver._run_serial (solver_fdtd.py:457-463): it
// issues one fused kernel per k time steps, computing on the host, per
// launch, which records sample and whether the non-finite scan runs at each
// fused step (solver_fdtd.py:386-393) so the kernels never divide in their
// inner loop.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/mbgpu.h"
#include "mbg_kernels.h"

using namespace mbg;

namespace {

struct QmHost {
    int n = 0;
    bool dense = false, rk4 = false;
    double bloch[15] = {};
    std::vector<double> pop, coh, bc, bf, h0, mu, popm, deph;  // complex interleaved where complex
    std::vector<double> pol_re, pol_im, pol_dv;
    double pol_factor = 0.0;
};

struct Rec {
    int q = 0, i = 0, j = 0;
    long long cell = -1, every = 1, rows = 0, cols = 0, col0 = 0;
    long long row0 = 0, cap = 0;  // device rows [row0, row0 + cap) (cap < rows: streamed)
    double *re = nullptr, *im = nullptr;
};

}  // namespace

struct mbg_solver {
    mbg_grid g{};
    int words = 0;
    bool bloch = false;
    int k = 1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    long long win_n = 0, plane = 0;
    double *e[2] = {nullptr, nullptr}, *h[2] = {nullptr, nullptr}, *s[2] = {nullptr, nullptr};
    int cur = 0;
    Regions rg{};
    bool have_regions = false;
    bool state_set = false;  // the density state was uploaded (or mapped into the frame)
    bool frame_on = false;   // the device state is in the relaxed frame (BlochFrame)
    std::vector<QmHost> qm;
    bool has_boundary = false;
    double bnd[6] = {};
    int n_src = 0;
    long long src_cell[kMaxSources] = {};
    int src_hard[kMaxSources] = {};
    double *src_values = nullptr;
    double *src_host = nullptr;  // pinned staging of the sample table (rows uploaded as they are sampled)
    size_t src_host_bytes = 0;
    std::vector<Rec> recs;
    unsigned long long *bad = nullptr;
    unsigned long long *inv = nullptr;  // running invariant keys (mbg_invariants_accumulate)
    long long inv_every = 0;            // two-level kernels fold the monitor every inv_every steps
    double *ck_e = nullptr, *ck_h = nullptr, *ck_s = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t marks[MBG_MAX_MARKS] = {};
    unsigned *wave = nullptr;  // persistent launch: [0] ticket, [1] stall, [2..] done flags
    long long wave_cap = 0;
    WaveItem *wave_items = nullptr;  // work items of one chunk (fixed per solver)
    long long wave_n = 0;
    unsigned *push_ticket = nullptr;  // peer-memory exchange: block ticket of the push kernel
    bool peer_used = false;           // a pull may have set the stall flag (bit 1)
    long long launches = 0;
    std::string err;
};

namespace {

int fail(mbg_solver *s, int code, const std::string &msg) {
    if (s) s->err = msg;
    return code;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t _e = (call);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return fail(s, MBG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));    \
    } while (0)

int default_tile_steps(int levels, int stepper) {
    if (levels <= 2 && stepper == MBG_STEPPER_SPLITTING) return 64;
    if (levels == 3 && stepper == MBG_STEPPER_SPLITTING) return 12;  // cfg3 sweep: k = 8..16 within 2 %, 12 best
    if (levels <= 3) return 16;
    return 4;
}

int tile_width(const mbg_solver *s) {
    if (s->bloch || s->g.levels == 0) return s->g.exact ? exact::bloch_cta_tile() : fast::bloch_cta_tile();
    return dense_tile_width(s->g.levels, s->g.stepper == MBG_STEPPER_RK4);
}

Launch base_launch(const mbg_solver *s) {
    Launch L;
    std::memset(&L, 0, sizeof(L));
    L.num_x = s->g.num_x;
    L.win_lo = s->g.win_lo;
    L.win_n = s->win_n;
    L.own_lo = s->g.own_lo;
    L.own_hi = s->g.own_hi;
    L.plane = s->plane;
    L.e_in = s->e[s->cur];
    L.h_in = s->h[s->cur];
    L.s_in = s->s[s->cur];
    L.e_out = s->e[1 - s->cur];
    L.h_out = s->h[1 - s->cur];
    L.s_out = s->s[1 - s->cur];
    L.has_boundary = s->has_boundary ? 1 : 0;
    // solver_fdtd.py:372-377: e_at = (1 - c) e0 + c e1; e = w * 0.5 * (...)
    L.l_omc = 1.0 - s->bnd[1];
    L.l_c = s->bnd[1];
    L.l_hw = s->bnd[0] * 0.5;
    L.l_z = s->bnd[2];
    L.r_omc = 1.0 - s->bnd[4];
    L.r_c = s->bnd[4];
    L.r_hw = s->bnd[3] * 0.5;
    L.r_z = s->bnd[5];
    L.n_src = s->n_src;
    for (int q = 0; q < s->n_src; ++q) {
        L.src_cell[q] = s->src_cell[q];
        L.src_hard[q] = s->src_hard[q];
    }
    L.src_values = s->src_values;
    L.words = s->words;
    L.num_t = s->g.num_t;
    L.n_rec = (int)s->recs.size();
    for (int r = 0; r < L.n_rec; ++r) {
        const Rec &R = s->recs[r];
        L.rec_q[r] = R.q;
        L.rec_i[r] = R.i;
        L.rec_j[r] = R.j;
        L.rec_cell[r] = R.cell;
        L.rec_every[r] = R.every;
        L.rec_cols[r] = R.cols;
        L.rec_col0[r] = R.col0;
        L.rec_row0[r] = R.row0;
        L.rec_re[r] = R.re;
        L.rec_im[r] = R.im;
        L.rec_len[r] = R.cap * R.cols;
    }
    L.bad_step = s->bad;
    L.inv = s->inv_every > 0 ? s->inv : nullptr;
    L.inv_every = s->inv_every;
    L.rg = s->rg;
    return L;
}

template <int N>
void fill_split(DenseQm<N> &d, const QmHost &h) {
    // B/2 = bc/2 + E bf/2 (exact halving): its inverse is 2 (I + iA)^-1
    for (int i = 0; i < N * N; ++i) {
        d.pop[i] = h.pop[i];
        d.coh[i] = h.coh[i];
        d.bc_re[i] = 0.5 * h.bc[2 * i];
        d.bc_im[i] = 0.5 * h.bc[2 * i + 1];
        d.bf_re[i] = 0.5 * h.bf[2 * i];
        d.bf_im[i] = 0.5 * h.bf[2 * i + 1];
    }
    for (int p = 0; p < N * (N - 1) / 2; ++p) {
        d.pol.pol_re[p] = h.pol_re[p];
        d.pol.pol_im[p] = h.pol_im[p];
    }
    for (int i = 0; i < N; ++i) d.pol.pol_dv[i] = h.pol_dv[i];
    d.pol.pol_factor = h.pol_factor;
}

// B = I + i a (H0 - E mu) with a real A = a (H0 - E mu): Re(b_const) = I and
// Re(b_field) = 0 exactly (real H0 and dipole; _kernels.py:437-439)
template <int N>
bool real_hamiltonian(const QmHost &h) {
    for (int i = 0; i < N * N; ++i)
        if (h.bc[2 * i] != (i % (N + 1) == 0 ? 1.0 : 0.0) || h.bf[2 * i] != 0.0) return false;
    return true;
}

// RK4 constants: H0 and the dipole real (_kernels.py:554-557)
template <int N>
bool real_operators(const QmHost &h) {
    for (int i = 0; i < N * N; ++i)
        if (h.h0[2 * i + 1] != 0.0 || h.mu[2 * i + 1] != 0.0) return false;
    return true;
}

// MBG_REAL_A=0: always the complex inversion (A/B timing)
inline bool disable_real_a() {
    static const bool off = [] {
        const char *v = std::getenv("MBG_REAL_A");
        return v && v[0] == '0';
    }();
    return off;
}

template <int N>
void fill_rk4(Rk4Qm<N> &d, const QmHost &h, double dt) {
    for (int i = 0; i < N * N; ++i) {
        d.h0_re[i] = h.h0[2 * i];
        d.h0_im[i] = h.h0[2 * i + 1];
        d.mu_re[i] = h.mu[2 * i];
        d.mu_im[i] = h.mu[2 * i + 1];
        d.popm[i] = h.popm[i];
        d.deph[i] = h.deph[i];
    }
    d.dt = dt;
    for (int p = 0; p < N * (N - 1) / 2; ++p) {
        d.pol.pol_re[p] = h.pol_re[p];
        d.pol.pol_im[p] = h.pol_im[p];
    }
    for (int i = 0; i < N; ++i) d.pol.pol_dv[i] = h.pol_dv[i];
    d.pol.pol_factor = h.pol_factor;
}

template <int N>
cudaError_t launch_dense_n(const mbg_solver *s, const Launch &L, long long tiles) {
    const bool rk4 = s->g.stepper == MBG_STEPPER_RK4;
    if (rk4) {
        auto *P = new DenseParams<N, Rk4Qm<N>>();
        P->L = L;
        P->n_qm = (int)s->qm.size();
        P->real_a = P->n_qm > 0 && !disable_real_a();
        for (int q = 0; q < P->n_qm; ++q) {
            fill_rk4<N>(P->qm[q], s->qm[q], s->g.dt);
            P->real_a &= real_operators<N>(s->qm[q]) ? 1 : 0;
        }
        cudaError_t e = s->g.exact ? exact::launch_dense_rk4(N, P, tiles, s->stream)
                                   : fast::launch_dense_rk4(N, P, tiles, s->stream);
        delete P;
        return e;
    }
    if constexpr (N >= 3) {
        auto *P = new DenseParams<N, DenseQm<N>>();
        P->L = L;
        P->n_qm = (int)s->qm.size();
        P->real_a = P->n_qm > 0 && !disable_real_a();
        for (int q = 0; q < P->n_qm; ++q) {
            fill_split<N>(P->qm[q], s->qm[q]);
            P->real_a &= real_hamiltonian<N>(s->qm[q]) ? 1 : 0;
        }
        cudaError_t e = s->g.exact ? exact::launch_dense_split(N, P, tiles, s->stream)
                                   : fast::launch_dense_split(N, P, tiles, s->stream);
        delete P;
        return e;
    }
    return cudaErrorInvalidValue;
}

// batched single points: the N-level parameter block (same constants and
// real-operator choice as the step kernels)
template <int N>
cudaError_t batch_dense_n(const mbg_solver *s, int B, const BatchRecs &R, const double *e_seq, double *state,
                          const int *medium, std::vector<void *> &dev_bufs) {
    const bool rk4 = s->g.stepper == MBG_STEPPER_RK4;
    auto go = [&](auto *P, auto fill, auto real) {
        using Q = std::remove_cv_t<std::remove_pointer_t<decltype(P->qm)>>;
        P->B = B;
        P->num_t = s->g.num_t;
        P->e_seq = e_seq;
        P->state = state;
        P->medium = medium;
        P->R = R;
        P->n_qm = (int)s->qm.size();
        P->real_a = P->n_qm > 0 && !disable_real_a();
        std::vector<Q> host(P->n_qm);
        for (int q = 0; q < P->n_qm; ++q) {
            fill(host[q], s->qm[q]);
            P->real_a &= real(s->qm[q]) ? 1 : 0;
        }
        Q *dq = nullptr;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&dq), sizeof(Q) * host.size(), s->stream);
        if (e == cudaSuccess) {
            dev_bufs.push_back(dq);
            e = cudaMemcpyAsync(dq, host.data(), sizeof(Q) * host.size(), cudaMemcpyHostToDevice, s->stream);
            // the pageable source must stay valid until the copy is staged
            if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
        }
        P->qm = dq;
        if (e == cudaSuccess)
            e = s->g.exact ? exact::launch_batch_dense(N, rk4, P, B, s->stream)
                           : fast::launch_batch_dense(N, rk4, P, B, s->stream);
        delete P;
        return e;
    };
    if (rk4)
        return go(new BatchParams<N, Rk4Qm<N>>(), [&](Rk4Qm<N> &d, const QmHost &h) { fill_rk4<N>(d, h, s->g.dt); },
                  [](const QmHost &h) { return real_operators<N>(h); });
    if constexpr (N >= 3)
        return go(new BatchParams<N, DenseQm<N>>(), [](DenseQm<N> &d, const QmHost &h) { fill_split<N>(d, h); },
                  [](const QmHost &h) { return real_hamiltonian<N>(h); });
    return cudaErrorInvalidValue;
}

// _kernels.py:481-494 components that vanish for a real dipole / diagonal H0
bool real_dipole(const BlochQm &b) {
    return b.ax_c == 0.0 && b.ay_c == 0.0 && b.ay_s == 0.0 && b.az_s == 0.0 && b.a0_s == 0.0 && b.mu_y == 0.0 &&
           b.mu_z == 0.0;
}

// the fast two-level path keeps its state in the relaxed frame when every
// medium has a real dipole and invertible half-step relaxation factors
BlochFrame frame_of(const mbg_solver *s) {
    BlochFrame F;
    std::memset(&F, 0, sizeof(F));
    if (s->g.exact || !(s->bloch || s->g.levels == 0) || s->qm.empty() || (int)s->qm.size() > kMaxQm) return F;
    for (size_t q = 0; q < s->qm.size(); ++q) {
        BlochQm b;
        std::memcpy(&b, s->qm[q].bloch, sizeof(BlochQm));
        if (!real_dipole(b) || !(b.fxy >= 1e-150) || !(b.kz >= 1e-150) || !std::isfinite(b.fxy) ||
            !std::isfinite(b.kz) || !std::isfinite(b.cz))
            return F;
        F.fxy[q] = b.fxy;
        F.kz[q] = b.kz;
        F.cz[q] = b.cz;
    }
    F.on = 1;
    return F;
}

// the frame the device state is in right now
BlochFrame state_frame(const mbg_solver *s) {
    BlochFrame F = frame_of(s);
    F.on = s->frame_on ? 1 : 0;
    return F;
}

BlochReal bloch_real(const BlochQm &b) {
    const double u = b.a0_c * b.a0_c;
    return BlochReal{u,
                     1.0 + u,
                     4.0 * u,
                     b.az_c * b.az_c,
                     b.pol_factor * b.mu_x * b.fxy,
                     b.fxy * b.fxy,
                     b.kz * b.kz,
                     b.kz * b.cz + b.cz,
                     0.5 * (1.0 + u)};
}

BlochParams bloch_params(const mbg_solver *s, const Launch &L) {
    BlochParams P;
    std::memset(&P, 0, sizeof(P));
    P.L = L;
    P.n_qm = (int)s->qm.size();
    P.real_dipole = P.n_qm > 0 ? 1 : 0;
    for (int q = 0; q < P.n_qm; ++q) {
        BlochQm &b = P.qm[q];
        std::memcpy(&b, s->qm[q].bloch, sizeof(BlochQm));
        P.real_dipole &= real_dipole(b) ? 1 : 0;
        P.rq[q] = bloch_real(b);
    }
    // the fast variant's real-dipole cell function works in the relaxed frame
    P.frame = state_frame(s);
    if (!s->g.exact && !P.frame.on) P.real_dipole = 0;
    return P;
}

cudaError_t launch_step(const mbg_solver *s, const Launch &L, long long tiles, int *kernels) {
    *kernels = 1;
    if (s->bloch || s->g.levels == 0) {
        const BlochParams P = bloch_params(s, L);
        return s->g.exact ? exact::launch_bloch(P, tiles, s->stream, kernels)
                          : fast::launch_bloch(P, tiles, s->stream, kernels);
    }
    switch (s->g.levels) {
        case 2: return launch_dense_n<2>(s, L, tiles);
        case 3: return launch_dense_n<3>(s, L, tiles);
        case 4: return launch_dense_n<4>(s, L, tiles);
        case 5: return launch_dense_n<5>(s, L, tiles);
        case 6: return launch_dense_n<6>(s, L, tiles);
        case 7: return launch_dense_n<7>(s, L, tiles);
        case 8: return launch_dense_n<8>(s, L, tiles);
        default: return cudaErrorInvalidValue;
    }
}

// Device memory comes from the device's default stream-ordered pool with an
// unbounded release threshold: a new solver for the same workload (every e2e
// run) reuses the previous one's blocks instead of paying cudaMalloc/cudaFree.
void configure_pool(int device) {
    static bool done[64] = {};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        unsigned long long threshold = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    done[device] = true;
}

cudaError_t dalloc(cudaStream_t st, double **p, size_t bytes) {
    return cudaMallocAsync(reinterpret_cast<void **>(p), bytes, st);
}

void dfree(cudaStream_t st, void *p) {
    if (p) cudaFreeAsync(p, st);
}

// Pinned host staging (the streamed source table) from a process-wide free
// list: page-locking costs milliseconds per call, and every run of the same
// workload asks for the same size again.  Blocks are returned only after the
// owner's stream has drained (mbg_destroy / mbg_set_sources synchronise first).
struct PinnedBlock {
    void *p;
    size_t bytes;
};
std::mutex g_pinned_mu;
std::vector<PinnedBlock> g_pinned_free;
constexpr size_t kPinnedKeep = 64;

cudaError_t pinned_get(double **p, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        for (size_t i = 0; i < g_pinned_free.size(); ++i) {
            if (g_pinned_free[i].bytes == bytes) {
                *p = static_cast<double *>(g_pinned_free[i].p);
                g_pinned_free.erase(g_pinned_free.begin() + (long)i);
                return cudaSuccess;
            }
        }
    }
    return cudaMallocHost(reinterpret_cast<void **>(p), bytes);
}

void pinned_put(void *p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (g_pinned_free.size() >= kPinnedKeep) {
        cudaFreeHost(g_pinned_free.front().p);
        g_pinned_free.erase(g_pinned_free.begin());
    }
    g_pinned_free.push_back({p, bytes});
}

bool window_ok(const mbg_grid *g) {
    return g->win_lo >= 0 && g->win_hi <= g->num_x && g->win_lo < g->win_hi && g->own_lo >= g->win_lo &&
           g->own_hi <= g->win_hi && g->own_lo < g->own_hi;
}

}  // namespace

extern "C" {

static int sync_frame(mbg_solver *s);


const char *mbg_version(void) { return "mbgpu 0.1 (sm_100a)"; }

int mbg_device_count(int *count) {
    mbg_solver *s = nullptr;
    CK(cudaGetDeviceCount(count));
    return MBG_OK;
}

const char *mbg_last_error(const mbg_solver *s) { return s ? s->err.c_str() : "null solver"; }

int mbg_create(const mbg_grid *grid, mbg_solver **out) {
    mbg_solver *s = nullptr;
    if (!grid || !out) return MBG_E_ARG;
    *out = nullptr;
    mbg_grid g = *grid;
    if (g.num_x < 1 || g.num_t < 2 || !(g.dt > 0)) return MBG_E_ARG;
    if (g.win_hi == 0 && g.win_lo == 0) {
        g.win_hi = g.num_x;
        g.own_lo = 0;
        g.own_hi = g.num_x;
    }
    if (!window_ok(&g)) return MBG_E_ARG;
    if (g.levels < 0 || g.levels > MBG_MAX_LEVELS || g.levels == 1) return MBG_E_UNSUPPORTED;
    if (g.stepper != MBG_STEPPER_SPLITTING && g.stepper != MBG_STEPPER_RK4) return MBG_E_ARG;
    s = new mbg_solver();
    s->g = g;
    s->bloch = g.levels == 2 && g.stepper == MBG_STEPPER_SPLITTING;
    s->words = g.levels == 0 ? 0 : (s->bloch ? 3 : g.levels * g.levels);
    s->win_n = g.win_hi - g.win_lo;
    s->plane = (s->win_n + 31) / 32 * 32;  // 256-byte aligned planes
    int k = g.tile_steps > 0 ? g.tile_steps : default_tile_steps(g.levels, g.stepper);
    const int w = tile_width(s);
    if (g.tile_steps <= 0 && !(s->bloch || g.levels == 0) && g.win_lo == 0 && g.win_hi == g.num_x &&
        !(g.flags & MBG_FLAG_DEFAULT_DEPTH)) {
        // small N-level domains (every tile on its own SM even at a deeper
        // chunk): fewer, deeper launches -- the per-launch overhead (~3.7 us)
        // is then paid every 32 steps instead of every 4 while the extra halo
        // work lands on idle SMs (tzenov2016-full, 8192 five-level cells:
        // 2.02 s at k = 4, 1.58 s at k = 32)
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g.device) != cudaSuccess || sms <= 0) sms = 148;
        for (int kk : {32, 16, 8}) {
            if (kk <= k || 2 * kk + 32 > w) continue;
            if ((s->win_n + (w - 2 * kk) - 1) / (w - 2 * kk) <= sms) {
                k = kk;
                break;
            }
        }
    }
    // every tile (and, for the two-level kernel, every warp tile of the edge
    // kernel) must keep at least 32 result cells
    const int wmin = (s->bloch || g.levels == 0) ? std::min(w, kBlochTile) : w;
    k = std::min(k, std::min(MBG_MAX_TILE_STEPS, (wmin - 32) / 2));
    s->k = std::max(k, 1);
    auto cleanup = [&](int code) {
        mbg_destroy(s);
        return code;
    };
    if (cudaSetDevice(g.device) != cudaSuccess) return cleanup(MBG_E_CUDA);
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) return cleanup(MBG_E_CUDA);
    s->own_stream = true;
    configure_pool(g.device);
    const size_t fb = sizeof(double) * (s->win_n + 1);
    const size_t sb = sizeof(double) * (size_t)std::max(1, s->words) * s->plane;
    for (int b = 0; b < 2; ++b) {
        if (dalloc(s->stream, &s->e[b], fb) != cudaSuccess || dalloc(s->stream, &s->h[b], fb) != cudaSuccess ||
            dalloc(s->stream, &s->s[b], sb) != cudaSuccess)
            return cleanup(MBG_E_CUDA);
        cudaMemsetAsync(s->e[b], 0, fb, s->stream);
        cudaMemsetAsync(s->h[b], 0, fb, s->stream);
        cudaMemsetAsync(s->s[b], 0, sb, s->stream);
    }
    // [0] first failing scan step (~0: none), [1] stall flag of the persistent
    // launches: sticky -- only check_stall clears it, after reporting it
    if (dalloc(s->stream, reinterpret_cast<double **>(&s->bad), 2 * sizeof(unsigned long long)) != cudaSuccess)
        return cleanup(MBG_E_CUDA);
    cudaMemsetAsync(s->bad, 0xff, sizeof(unsigned long long), s->stream);
    cudaMemsetAsync(s->bad + 1, 0, sizeof(unsigned long long), s->stream);
    cudaEventCreate(&s->ev0);
    cudaEventCreate(&s->ev1);
    if (cudaStreamSynchronize(s->stream) != cudaSuccess) return cleanup(MBG_E_CUDA);
    *out = s;
    return MBG_OK;
}

void mbg_destroy(mbg_solver *s) {
    if (!s) return;
    cudaSetDevice(s->g.device);
    cudaStream_t st = s->stream;
    if (st) cudaStreamSynchronize(st);
    for (int b = 0; b < 2; ++b) {
        dfree(st, s->e[b]);
        dfree(st, s->h[b]);
        dfree(st, s->s[b]);
    }
    dfree(st, s->bad);
    dfree(st, s->inv);
    dfree(st, s->wave);
    dfree(st, s->wave_items);
    dfree(st, s->push_ticket);
    dfree(st, s->ck_e);
    dfree(st, s->ck_h);
    dfree(st, s->ck_s);
    dfree(st, s->src_values);
    for (auto &r : s->recs) {
        dfree(st, r.re);
        dfree(st, r.im);
    }
    if (st) cudaStreamSynchronize(st);
    if (s->src_host) pinned_put(s->src_host, s->src_host_bytes);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    for (cudaEvent_t e : s->marks)
        if (e) cudaEventDestroy(e);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

int mbg_set_stream(mbg_solver *s, uint64_t stream) {
    if (!s) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    CK(cudaStreamSynchronize(s->stream));
    if (s->own_stream) cudaStreamDestroy(s->stream);
    if (stream == 0) {
        CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        s->own_stream = true;
    } else {
        s->stream = reinterpret_cast<cudaStream_t>(stream);
        s->own_stream = false;
    }
    return MBG_OK;
}

int mbg_tile_steps(const mbg_solver *s, int32_t *k) {
    if (!s || !k) return MBG_E_ARG;
    *k = s->k;
    return MBG_OK;
}

int mbg_set_regions(mbg_solver *s, int32_t n, const int64_t *e_start, const int64_t *h_start, const double *a,
                    const double *bg, const double *bdx, const double *ch, const int32_t *qm_index) {
    if (!s || n < 1) return fail(s, MBG_E_ARG, "need at least one region");
    if (n > kMaxRegions) return fail(s, MBG_E_UNSUPPORTED, "too many regions (max 128)");
    Regions &rg = s->rg;
    std::memset(&rg, 0, sizeof(rg));
    rg.n = n;
    for (int r = 0; r < n; ++r) {
        rg.e_start[r] = e_start[r];
        rg.h_start[r] = h_start[r];
        rg.a[r] = a[r];
        rg.bg[r] = bg[r];
        rg.bdx[r] = bdx[r];
        rg.ch[r] = ch[r];
        rg.qm[r] = qm_index[r];
        if (qm_index[r] >= kMaxQm) return fail(s, MBG_E_UNSUPPORTED, "too many quantum materials");
        if (r > 0 && (e_start[r] < e_start[r - 1] || h_start[r] < h_start[r - 1]))
            return fail(s, MBG_E_ARG, "region starts must be non-decreasing");
    }
    s->have_regions = true;
    return MBG_OK;
}

static QmHost &qm_slot(mbg_solver *s, int q) {
    if ((int)s->qm.size() <= q) s->qm.resize(q + 1);
    return s->qm[q];
}

int mbg_set_qm_bloch(mbg_solver *s, int32_t q, const double *c) {
    if (!s || q < 0 || q >= MBG_MAX_BATCH_QM || !c) return fail(s, MBG_E_ARG, "bad qm index");
    if (!s->bloch) return fail(s, MBG_E_STATE, "solver is not a two-level splitting solver");
    QmHost &h = qm_slot(s, q);
    h.n = 2;
    std::memcpy(h.bloch, c, sizeof(h.bloch));
    return MBG_OK;
}

static void set_pol(QmHost &h, int n, int npol, const int32_t *pi, const int32_t *pj, const double *pv, int ndpol,
                    const int32_t *pdi, const double *pdv, double pol_factor) {
    const int nu = n * (n - 1) / 2;
    h.pol_re.assign(std::max(nu, 1), 0.0);
    h.pol_im.assign(std::max(nu, 1), 0.0);
    h.pol_dv.assign(n, 0.0);
    for (int k = 0; k < npol; ++k) {
        const int i = pi[k], j = pj[k];
        const int p = i * n - i * (i + 1) / 2 + (j - i - 1);
        h.pol_re[p] = pv[2 * k];
        h.pol_im[p] = pv[2 * k + 1];
    }
    for (int k = 0; k < ndpol; ++k) h.pol_dv[pdi[k]] = pdv[k];
    h.pol_factor = pol_factor;
}

static bool pol_ok(int n, int npol, const int32_t *pi, const int32_t *pj, int ndpol, const int32_t *pdi) {
    for (int k = 0; k < npol; ++k)
        if (pi[k] < 0 || pj[k] <= pi[k] || pj[k] >= n) return false;
    for (int k = 0; k < ndpol; ++k)
        if (pdi[k] < 0 || pdi[k] >= n) return false;
    return true;
}

int mbg_set_qm_dense(mbg_solver *s, int32_t q, const double *pop, const double *coh, const double *bc,
                     const double *bf, int32_t npol, const int32_t *pi, const int32_t *pj, const double *pv,
                     int32_t ndpol, const int32_t *pdi, const double *pdv, double pol_factor) {
    if (!s || q < 0 || q >= MBG_MAX_BATCH_QM) return fail(s, MBG_E_UNSUPPORTED, "qm index beyond MBG_MAX_BATCH_QM");
    const int n = s->g.levels;
    if (s->bloch || s->g.stepper != MBG_STEPPER_SPLITTING || n < 3)
        return fail(s, MBG_E_STATE, "solver is not an N>=3 splitting solver");
    if (!pol_ok(n, npol, pi, pj, ndpol, pdi)) return fail(s, MBG_E_ARG, "bad dipole index list");
    QmHost &h = qm_slot(s, q);
    h.n = n;
    h.dense = true;
    h.pop.assign(pop, pop + n * n);
    h.coh.assign(coh, coh + n * n);
    h.bc.assign(bc, bc + 2 * n * n);
    h.bf.assign(bf, bf + 2 * n * n);
    set_pol(h, n, npol, pi, pj, pv, ndpol, pdi, pdv, pol_factor);
    return MBG_OK;
}

int mbg_set_qm_rk4(mbg_solver *s, int32_t q, const double *h0, const double *mu, const double *popm,
                   const double *deph, int32_t npol, const int32_t *pi, const int32_t *pj, const double *pv,
                   int32_t ndpol, const int32_t *pdi, const double *pdv, double pol_factor) {
    if (!s || q < 0 || q >= MBG_MAX_BATCH_QM) return fail(s, MBG_E_UNSUPPORTED, "qm index beyond MBG_MAX_BATCH_QM");
    const int n = s->g.levels;
    if (s->g.stepper != MBG_STEPPER_RK4 || n < 2) return fail(s, MBG_E_STATE, "solver is not an RK4 solver");
    if (!pol_ok(n, npol, pi, pj, ndpol, pdi)) return fail(s, MBG_E_ARG, "bad dipole index list");
    QmHost &h = qm_slot(s, q);
    h.n = n;
    h.rk4 = true;
    h.h0.assign(h0, h0 + 2 * n * n);
    h.mu.assign(mu, mu + 2 * n * n);
    h.popm.assign(popm, popm + n * n);
    h.deph.assign(deph, deph + n * n);
    set_pol(h, n, npol, pi, pj, pv, ndpol, pdi, pdv, pol_factor);
    return MBG_OK;
}

int mbg_set_boundary(mbg_solver *s, double wl, double cl, double zl, double wr, double cr, double zr) {
    if (!s) return MBG_E_ARG;
    s->has_boundary = s->g.num_x > 1;
    const double v[6] = {wl, cl, zl, wr, cr, zr};
    std::memcpy(s->bnd, v, sizeof(v));
    return MBG_OK;
}

int mbg_set_sources(mbg_solver *s, int32_t n, const int64_t *cell, const int32_t *hard, const double *values) {
    if (!s || n < 0) return MBG_E_ARG;
    if (n > kMaxSources) return fail(s, MBG_E_UNSUPPORTED, "too many sources (max 32)");
    cudaSetDevice(s->g.device);
    if (s->src_host) {
        CK(cudaStreamSynchronize(s->stream));  // no copy out of the old staging in flight
        pinned_put(s->src_host, s->src_host_bytes);
        s->src_host = nullptr;
    }
    dfree(s->stream, s->src_values);
    s->src_values = nullptr;
    s->n_src = n;
    for (int q = 0; q < n; ++q) {
        if (cell[q] < 0 || cell[q] >= s->g.num_x) return fail(s, MBG_E_ARG, "source cell outside the grid");
        s->src_cell[q] = cell[q];
        s->src_hard[q] = hard[q] ? 1 : 0;
    }
    if (n > 0) {
        const size_t bytes = sizeof(double) * (size_t)n * s->g.num_t;
        CK(dalloc(s->stream, &s->src_values, bytes));
        if (values) {
            CK(cudaMemcpyAsync(s->src_values, values, bytes, cudaMemcpyHostToDevice, s->stream));
            CK(cudaStreamSynchronize(s->stream));
        } else {
            // rows arrive later (mbg_set_source_rows) through a pinned staging copy
            CK(cudaMemsetAsync(s->src_values, 0, bytes, s->stream));
            CK(pinned_get(&s->src_host, bytes));
            s->src_host_bytes = bytes;
        }
    }
    return MBG_OK;
}

int mbg_set_source_rows(mbg_solver *s, int64_t lo, int64_t hi, const double *rows) {
    if (!s || lo < 0 || hi < lo || hi > s->g.num_t) return MBG_E_ARG;
    if (s->n_src == 0 || hi == lo) return MBG_OK;
    if (!s->src_host) return fail(s, MBG_E_STATE, "mbg_set_source_rows needs mbg_set_sources(..., values = NULL)");
    if (!rows) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    const size_t off = (size_t)lo * s->n_src, cnt = (size_t)(hi - lo) * s->n_src;
    // stream order: these rows reach the device before any later launch
    // reads them; the staging rows of earlier calls are never rewritten
    std::memcpy(s->src_host + off, rows, sizeof(double) * cnt);
    CK(cudaMemcpyAsync(s->src_values + off, s->src_host + off, sizeof(double) * cnt, cudaMemcpyHostToDevice,
                       s->stream));
    return MBG_OK;
}

int mbg_set_records(mbg_solver *s, int32_t n, const int32_t *q, const int64_t *cell, const int32_t *i,
                    const int32_t *j, const int64_t *every) {
    if (!s || n < 0) return MBG_E_ARG;
    if (n > kMaxRecords) return fail(s, MBG_E_UNSUPPORTED, "too many records (max 64)");
    cudaSetDevice(s->g.device);
    for (auto &r : s->recs) {
        dfree(s->stream, r.re);
        dfree(s->stream, r.im);
    }
    s->recs.assign(n, Rec());
    for (int r = 0; r < n; ++r) {
        Rec &R = s->recs[r];
        R.q = q[r];
        R.i = i[r];
        R.j = j[r];
        R.cell = cell[r];
        R.every = every[r];
        if (R.q < 0 || R.q > 3 || R.every < 1 || R.cell >= s->g.num_x ||
            (R.q == MBG_Q_D && (R.i < 0 || R.j < 0 || R.i >= std::max(1, s->g.levels) || R.j >= std::max(1, s->g.levels))))
            return fail(s, MBG_E_ARG, "bad record specification");
        R.rows = (s->g.num_t - 1) / R.every + 1;
        R.cols = R.cell >= 0 ? 1 : s->g.own_hi - s->g.own_lo;
        R.col0 = R.cell >= 0 ? R.cell : s->g.own_lo;
        R.row0 = 0;
        R.cap = R.rows;
        const size_t bytes = sizeof(double) * (size_t)R.rows * R.cols;
        CK(dalloc(s->stream, &R.re, bytes));
        CK(cudaMemsetAsync(R.re, 0, bytes, s->stream));
        if (R.q == MBG_Q_D && R.i != R.j) {
            CK(dalloc(s->stream, &R.im, bytes));
            CK(cudaMemsetAsync(R.im, 0, bytes, s->stream));
        }
    }
    return MBG_OK;
}

int mbg_upload_fields(mbg_solver *s, const double *e, const double *h) {
    if (!s || (!e) != (!h)) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    if (!e) {
        CK(cudaMemsetAsync(s->e[s->cur], 0, sizeof(double) * s->win_n, s->stream));
        CK(cudaMemsetAsync(s->h[s->cur], 0, sizeof(double) * (s->win_n + 1), s->stream));
        CK(cudaMemsetAsync(s->h[1 - s->cur] + s->win_n, 0, sizeof(double), s->stream));
        CK(cudaStreamSynchronize(s->stream));
        return MBG_OK;
    }
    // only the current buffer: every launch writes all of its result cells into
    // the other one, and node win_hi of H (never updated) is zeroed at create
    CK(cudaMemcpyAsync(s->e[s->cur], e, sizeof(double) * s->win_n, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->h[s->cur], h, sizeof(double) * (s->win_n + 1), cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->h[1 - s->cur] + s->win_n, h + s->win_n, sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

int mbg_upload_density(mbg_solver *s, const double *words) {
    if (!s || (!words && s->words)) return MBG_E_ARG;
    if (!s->have_regions) return fail(s, MBG_E_STATE, "set regions before the density state");
    if (s->words == 0) return MBG_OK;
    cudaSetDevice(s->g.device);
    double *w = nullptr;
    CK(dalloc(s->stream, &w, sizeof(double) * s->words));
    CK(cudaMemcpyAsync(w, words, sizeof(double) * s->words, cudaMemcpyHostToDevice, s->stream));
    CK(launch_broadcast_state(s->s[s->cur], s->plane, s->win_n, s->words, w, s->rg, s->g.win_lo, s->stream));
    dfree(s->stream, w);
    s->state_set = false;
    if (int rc = sync_frame(s)) return rc;
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

int mbg_upload_state(mbg_solver *s, const double *planes) {
    if (!s || !planes) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    for (int w = 0; w < s->words; ++w)
        CK(cudaMemcpyAsync(s->s[s->cur] + w * s->plane, planes + w * s->win_n, sizeof(double) * s->win_n,
                           cudaMemcpyHostToDevice, s->stream));
    s->state_set = false;
    if (s->have_regions)
        if (int rc = sync_frame(s)) return rc;
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

int mbg_download_fields(mbg_solver *s, double *e, double *h) {
    if (!s) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    if (e) CK(cudaMemcpyAsync(e, s->e[s->cur], sizeof(double) * s->win_n, cudaMemcpyDeviceToHost, s->stream));
    if (h) CK(cudaMemcpyAsync(h, s->h[s->cur], sizeof(double) * (s->win_n + 1), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

int mbg_download_state(mbg_solver *s, double *planes) {
    if (!s || !planes) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    if (s->frame_on) {  // true values out of the relaxed frame
        double *t = nullptr;
        const size_t bytes = sizeof(double) * s->words * s->win_n;
        CK(dalloc(s->stream, &t, bytes));
        CK(launch_frame(false, s->s[s->cur], s->plane, s->win_n, s->rg, s->g.win_lo, state_frame(s), t, s->stream));
        CK(cudaMemcpyAsync(planes, t, bytes, cudaMemcpyDeviceToHost, s->stream));
        dfree(s->stream, t);
        CK(cudaStreamSynchronize(s->stream));
        return MBG_OK;
    }
    for (int w = 0; w < s->words; ++w)
        CK(cudaMemcpyAsync(planes + w * s->win_n, s->s[s->cur] + w * s->plane, sizeof(double) * s->win_n,
                           cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

// every record row that steps [first, last] write lies in its device window
static bool rows_resident(const mbg_solver *s, long long first, long long last) {
    for (const Rec &R : s->recs) {
        if (R.cap >= R.rows || last < first) continue;
        const long long lo = (first + R.every - 1) / R.every, hi = last / R.every;  // rows written
        if (lo <= hi && (lo < R.row0 || hi >= R.row0 + R.cap)) return false;
    }
    return true;
}

int mbg_sample(mbg_solver *s, int64_t step) {
    if (!s) return MBG_E_ARG;
    if (!s->have_regions) return fail(s, MBG_E_STATE, "regions not set");
    if (!rows_resident(s, step, step)) return fail(s, MBG_E_ARG, "record row of this step is not device-resident");
    cudaSetDevice(s->g.device);
    if (int rc = sync_frame(s)) return rc;
    const Launch L = base_launch(s);
    CK(launch_sample(L, s->g.levels, s->bloch ? 1 : 0, step, state_frame(s), s->stream));
    ++s->launches;
    return MBG_OK;
}

// Map the device state into the relaxed frame if the medium calls for it and
// nothing was uploaded yet (a zero state); afterwards the medium may not
// change the frame (the stored words would be misread).
static int sync_frame(mbg_solver *s) {
    if (!s->have_regions || s->words == 0) return MBG_OK;
    const BlochFrame F = frame_of(s);
    if (!s->state_set) {
        if (F.on)
            CK(launch_frame(true, s->s[s->cur], s->plane, s->win_n, s->rg, s->g.win_lo, F, nullptr, s->stream));
        s->frame_on = F.on != 0;
        s->state_set = true;
    } else if ((F.on != 0) != s->frame_on) {
        return fail(s, MBG_E_STATE, "quantum constants changed after the density state was uploaded");
    }
    return MBG_OK;
}

// every quantum material a region refers to must have constants of the
// solver's stepper kind (otherwise a kernel would read an empty slot)
static int check_ready(mbg_solver *s) {
    if (!s->have_regions) return fail(s, MBG_E_STATE, "regions not set");
    const int limit = (s->bloch || s->g.levels == 0) ? kMaxQm : kMaxDenseQm;
    if ((int)s->qm.size() > limit) return fail(s, MBG_E_UNSUPPORTED, "too many quantum materials for this kernel");
    for (int r = 0; r < s->rg.n; ++r) {
        const int q = s->rg.qm[r];
        if (q < 0) continue;
        if (s->g.levels == 0) return fail(s, MBG_E_STATE, "region has a quantum material but levels == 0");
        if (q >= (int)s->qm.size() || s->qm[q].n != s->g.levels)
            return fail(s, MBG_E_STATE, "quantum constants not set for a material the regions use");
        const QmHost &h = s->qm[q];
        const bool ok = s->bloch ? (!h.dense && !h.rk4) : (s->g.stepper == MBG_STEPPER_RK4 ? h.rk4 : h.dense);
        if (!ok) return fail(s, MBG_E_STATE, "quantum constants do not match the stepper");
    }
    return sync_frame(s);
}

}  // extern "C"

namespace {

// the whole step range in one persistent launch (kernels_bloch.cu, BlochWave)
// the persistent wavefront pays off when a chunk has at least one tile per
// SM; a few-tile domain (cfg1: 17 tiles) is a dependency chain whose items
// run faster with a whole SM each, one launch per chunk (73 vs 200 ms)
bool wave_worthwhile(const mbg_solver *s, int tw) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->g.device) != cudaSuccess || sms <= 0)
        sms = 148;
    const long long tiles = s->win_n / std::max(1, tw - 2 * s->k);
    // edge ranges are one-cell-per-thread CTA items of kBlochTile - 2k cells and
    // every item must span >= k cells (dependencies j-1 .. j+1): beyond
    // k = kBlochTile / 3 they would be merged into ranges stepped by single
    // warps, a serial chain through the wavefront (k = 96: 951 ms against
    // 157 ms for one launch per chunk on cfg2) -- such depths go per launch
    if (kBlochTile - 2 * s->k < s->k) return false;
    return tiles >= sms;
}

int advance_wave(mbg_solver *s, long long first, long long n_steps, int tw) {
    const int k = s->k;
    Launch L = base_launch(s);
    L.n0 = first;
    L.k = k;
    // a window's result range loses k cells per side per chunk; its ghosts
    // (>= the steps between exchanges) absorb that (see mbg_advance)
    L.res_lo = s->g.win_lo == 0 ? 0 : s->g.win_lo + k;
    L.res_hi = s->g.win_hi == s->g.num_x ? s->g.num_x : s->g.win_hi - k;
    L.tile_own = tw - 2 * k;
    if (!s->wave_items) {
        // interior CTA tiles as they are; a non-interior tile split into items
        // of at most one round of warp ranges (host twin of the kernels'
        // classification, the same as launch_bloch's)
        const long long ct = (L.res_hi - L.res_lo + L.tile_own - 1) / L.tile_own;
        const long long warp_own = kBlochTile - 2 * k;
        std::vector<WaveItem> items;
        for (long long t = 0; t < ct; ++t) {
            const long long t_lo = L.res_lo + t * L.tile_own;
            const long long t_hi = std::min(t_lo + L.tile_own, L.res_hi);
            if (tile_is_interior(L, tile_base(L, t_lo), tw)) {
                items.push_back(WaveItem{t_lo, t_hi, 0, 0});
                continue;
            }
            // one item per edge range (flag 2: the CTA steps it one cell per
            // thread), the ranges of equal length (each >= k when possible)
            const long long len = t_hi - t_lo;
            const long long parts = (len + warp_own - 1) / warp_own;
            for (long long q = 0; q < parts; ++q)
                items.push_back(WaveItem{t_lo + len * q / parts, t_lo + len * (q + 1) / parts, 2, 0});
        }
        // every item but the last must span >= k cells (dependencies j-1 .. j+1)
        std::vector<WaveItem> merged;
        for (size_t j = 0; j < items.size(); ++j) {
            const bool last = j + 1 == items.size();
            if (!merged.empty() && (items[j].hi - items[j].lo < k && !last ||
                                    merged.back().hi - merged.back().lo < k)) {
                merged.back().hi = items[j].hi;
                merged.back().edge = 1;
            } else {
                merged.push_back(items[j]);
            }
        }
        CK(dalloc(s->stream, reinterpret_cast<double **>(&s->wave_items), sizeof(WaveItem) * merged.size()));
        CK(cudaMemcpyAsync(s->wave_items, merged.data(), sizeof(WaveItem) * merged.size(), cudaMemcpyHostToDevice,
                           s->stream));
        CK(cudaStreamSynchronize(s->stream));
        s->wave_n = (long long)merged.size();
    }
    const long long tiles = s->wave_n;
    const long long n_chunks = (n_steps + k - 1) / k;
    // [ticket, unused, done flags][masks (8 B per step)][checks (1 B per step)], in 4-byte words
    const long long flags = 2 + n_chunks * tiles;
    const long long mask_off = (flags + 1) / 2 * 2, check_off = mask_off + 2 * n_chunks * k;
    const long long need = check_off + (n_chunks * k + 3) / 4;
    if (need > s->wave_cap) {
        dfree(s->stream, s->wave);
        s->wave = nullptr;
        s->wave_cap = 0;
        CK(dalloc(s->stream, reinterpret_cast<double **>(&s->wave), sizeof(unsigned) * need));
        s->wave_cap = need;
    }
    CK(cudaMemsetAsync(s->wave, 0, sizeof(unsigned) * flags, s->stream));
    auto *masks = reinterpret_cast<unsigned long long *>(s->wave + mask_off);
    auto *checks = reinterpret_cast<unsigned char *>(s->wave + check_off);
    BlochWave V;
    std::memset(&V, 0, sizeof(V));
    V.n_chunks = (int)n_chunks;
    V.last_steps = (int)(n_steps - (n_chunks - 1) * k);
    V.tiles = tiles;
    V.items = s->wave_items;
    V.n0 = first;
    V.last_step = s->g.num_t - 1;
    V.masks = masks;
    V.checks = checks;
    for (int b = 0; b < 2; ++b) {
        V.e[b] = s->e[b];
        V.h[b] = s->h[b];
        V.s[b] = s->s[b];
    }
    V.cur = s->cur;
    V.ticket = s->wave;
    V.stall = reinterpret_cast<unsigned *>(s->bad + 1);  // sticky across launches
    V.done = s->wave + 2;
    CK(s->g.exact ? exact::launch_wave_masks(L, n_steps, V.last_step, masks, checks, s->stream)
                  : fast::launch_wave_masks(L, n_steps, V.last_step, masks, checks, s->stream));
    const BlochParams P = bloch_params(s, L);
    const char *trace_path = std::getenv("MBG_WAVE_TRACE");  // debug: per-item timeline
    const size_t trace_bytes = sizeof(unsigned long long) * 4 * n_chunks * tiles;
    if (trace_path) CK(cudaMalloc(reinterpret_cast<void **>(&V.trace), trace_bytes));
    CK(s->g.exact ? exact::launch_bloch_wave(P, V, s->stream) : fast::launch_bloch_wave(P, V, s->stream));
    if (trace_path) {
        std::vector<unsigned long long> h(trace_bytes / sizeof(unsigned long long));
        CK(cudaMemcpyAsync(h.data(), V.trace, trace_bytes, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        CK(cudaFree(V.trace));
        if (FILE *f = std::fopen(trace_path, "wb")) {
            const long long hdr[2] = {n_chunks, tiles};
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::fwrite(h.data(), 1, trace_bytes, f);
            std::fclose(f);
        }
    }
    s->launches += 2;  // step-mask pre-kernel + persistent step kernel
    if (n_chunks & 1) s->cur ^= 1;
    return MBG_OK;
}

// after a stream synchronize: a persistent launch that gave up waiting is an
// error.  The flag survives later launches (they are not allowed to clear it),
// so a timeout is reported at the first synchronisation after it, however
// many advances were enqueued in between; it is cleared once reported.
int check_stall(mbg_solver *s) {
    if (!s->wave && !s->peer_used) return MBG_OK;
    unsigned v = 0;
    CK(cudaMemcpy(&v, s->bad + 1, sizeof(v), cudaMemcpyDeviceToHost));
    if (v) {
        CK(cudaMemset(s->bad + 1, 0, sizeof(unsigned long long)));
        if (v & 2u)  // halo_pull_kernel: the ghosts of that period were left stale
            return fail(s, MBG_E_CUDA, "peer halo exchange: a neighbour's strip did not arrive within the timeout");
        return fail(s, MBG_E_CUDA, "persistent step kernel: dependency wait timed out");
    }
    return MBG_OK;
}

}  // namespace

extern "C" {

int mbg_advance(mbg_solver *s, int64_t first, int64_t n_steps) {
    if (!s) return MBG_E_ARG;
    if (int rc = check_ready(s)) return rc;
    if (first < 1 || n_steps < 0 || first + n_steps > s->g.num_t)
        return fail(s, MBG_E_ARG, "step range outside 1 .. num_t-1");
    if (!rows_resident(s, first, first + n_steps - 1))
        return fail(s, MBG_E_ARG, "record rows of this step range are not device-resident (streamed records)");
    const long long ghost_l = s->g.own_lo - s->g.win_lo, ghost_r = s->g.win_hi - s->g.own_hi;
    const bool windowed = s->g.win_lo > 0 || s->g.win_hi < s->g.num_x;
    if (windowed) {
        const long long gw = std::min(s->g.win_lo > 0 ? ghost_l : LLONG_MAX, s->g.win_hi < s->g.num_x ? ghost_r : LLONG_MAX);
        if (n_steps > gw)
            return fail(s, MBG_E_ARG, "a slab advances at most its ghost width in steps between exchanges");
    }
    cudaSetDevice(s->g.device);
    const int tw = tile_width(s);
    if ((s->bloch || s->g.levels == 0) && !(s->g.flags & MBG_FLAG_PER_LAUNCH) && n_steps > s->k &&
        ((s->g.flags & MBG_FLAG_PERSISTENT) || wave_worthwhile(s, tw)))
        return advance_wave(s, first, n_steps, tw);
    long long n = first;
    const long long end = first + n_steps;
    while (n < end) {
        const int kk = (int)std::min<long long>(s->k, end - n);
        Launch L = base_launch(s);
        L.n0 = n;
        L.k = kk;
        L.res_lo = s->g.win_lo == 0 ? 0 : s->g.win_lo + kk;
        L.res_hi = s->g.win_hi == s->g.num_x ? s->g.num_x : s->g.win_hi - kk;
        L.tile_own = tw - 2 * kk;
        for (int t = 0; t < kk; ++t) {
            const long long step = n + t;
            unsigned long long m = 0;
            for (size_t r = 0; r < s->recs.size(); ++r)
                if (step % s->recs[r].every == 0) m |= 1ull << r;
            L.step_mask[t] = m;
            L.check[t] = step_flags(L, step, s->g.num_t - 1);
        }
        const long long tiles = (L.res_hi - L.res_lo + L.tile_own - 1) / L.tile_own;
        int kernels = 0;
        CK(launch_step(s, L, tiles, &kernels));
        s->launches += kernels;
        s->cur ^= 1;
        n += kk;
    }
    return MBG_OK;
}

int mbg_stream_idle(mbg_solver *s, int32_t *idle) {
    if (!s || !idle) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    const cudaError_t e = cudaStreamQuery(s->stream);
    if (e == cudaErrorNotReady) {
        *idle = 0;
        return MBG_OK;
    }
    CK(e);
    *idle = 1;
    return MBG_OK;
}

int mbg_synchronize(mbg_solver *s) {
    if (!s) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    CK(cudaStreamSynchronize(s->stream));
    return check_stall(s);
}

int mbg_poll_nonfinite(mbg_solver *s, int64_t *bad_step) {
    if (!s || !bad_step) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, s->bad, sizeof(v), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *bad_step = v == ~0ull ? -1 : (int64_t)v;
    return check_stall(s);
}

static double from_key(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    std::memcpy(&v, &b, sizeof(v));
    return v;
}

int mbg_invariants(mbg_solver *s, double *out) {
    if (!s || !out) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    unsigned long long init[3] = {0, 0, ~0ull}, *d = nullptr;
    init[0] = init[1] = 0x8000000000000000ull;  // key of +0.0
    CK(dalloc(s->stream, reinterpret_cast<double **>(&d), sizeof(init)));
    CK(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, s->stream));
    const Launch L = base_launch(s);
    if (int rc = sync_frame(s)) return rc;
    if (s->words > 0) CK(launch_invariants(L, s->g.levels, s->bloch ? 1 : 0, state_frame(s), d, s->stream));
    unsigned long long h[3];
    CK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
    dfree(s->stream, d);
    CK(cudaStreamSynchronize(s->stream));
    out[0] = from_key(h[0]);
    out[1] = 0.0;  // Hermitian-packed state: exactly Hermitian
    out[2] = h[2] == ~0ull ? INFINITY : from_key(h[2]);
    return MBG_OK;
}

static const unsigned long long kInvInit[3] = {0x8000000000000000ull, 0x8000000000000000ull, ~0ull};

int mbg_invariants_accumulate(mbg_solver *s) {
    if (!s) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    if (!s->inv) {
        CK(dalloc(s->stream, reinterpret_cast<double **>(&s->inv), sizeof(kInvInit)));
        CK(cudaMemcpyAsync(s->inv, kInvInit, sizeof(kInvInit), cudaMemcpyHostToDevice, s->stream));
    }
    if (int rc = sync_frame(s)) return rc;
    const Launch L = base_launch(s);
    if (s->words > 0) CK(launch_invariants(L, s->g.levels, s->bloch ? 1 : 0, state_frame(s), s->inv, s->stream));
    ++s->launches;
    return MBG_OK;
}

int mbg_set_monitor(mbg_solver *s, int64_t every) {
    if (!s || every < 0) return MBG_E_ARG;
    if (every > 0 && !s->bloch) return fail(s, MBG_E_UNSUPPORTED, "the fused monitor is for two-level splitting media");
    cudaSetDevice(s->g.device);
    if (every > 0 && !s->inv) {
        CK(dalloc(s->stream, reinterpret_cast<double **>(&s->inv), sizeof(kInvInit)));
        CK(cudaMemcpyAsync(s->inv, kInvInit, sizeof(kInvInit), cudaMemcpyHostToDevice, s->stream));
    }
    s->inv_every = every;
    return MBG_OK;
}

int mbg_invariants_read(mbg_solver *s, double *out) {
    if (!s || !out) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    unsigned long long h[3] = {kInvInit[0], kInvInit[1], kInvInit[2]};
    if (s->inv) CK(cudaMemcpyAsync(h, s->inv, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    out[0] = from_key(h[0]);
    out[1] = 0.0;  // Hermitian-packed state: exactly Hermitian
    out[2] = h[2] == ~0ull ? INFINITY : from_key(h[2]);
    return MBG_OK;
}

int mbg_record_shape(const mbg_solver *s, int32_t r, int64_t *rows, int64_t *cols) {
    if (!s || r < 0 || r >= (int)s->recs.size()) return MBG_E_ARG;
    *rows = s->recs[r].rows;
    *cols = s->recs[r].cols;
    return MBG_OK;
}

int mbg_set_record_rows(mbg_solver *s, int32_t r, int64_t cap) {
    if (!s || r < 0 || r >= (int)s->recs.size()) return MBG_E_ARG;
    Rec &R = s->recs[r];
    if (cap < 1 || cap > R.rows) return fail(s, MBG_E_ARG, "record row capacity outside [1, rows]");
    cudaSetDevice(s->g.device);
    dfree(s->stream, R.re);
    dfree(s->stream, R.im);
    R.re = R.im = nullptr;
    R.row0 = 0;
    R.cap = cap;
    const size_t bytes = sizeof(double) * (size_t)cap * R.cols;
    CK(dalloc(s->stream, &R.re, bytes));
    CK(cudaMemsetAsync(R.re, 0, bytes, s->stream));
    if (R.q == MBG_Q_D && R.i != R.j) {
        CK(dalloc(s->stream, &R.im, bytes));
        CK(cudaMemsetAsync(R.im, 0, bytes, s->stream));
    }
    return MBG_OK;
}

int mbg_download_record_rows(mbg_solver *s, int32_t r, int64_t row_lo, int64_t row_hi, double *re, double *im) {
    if (!s || r < 0 || r >= (int)s->recs.size() || (!re && row_hi > row_lo)) return MBG_E_ARG;
    const Rec &R = s->recs[r];
    if (row_lo < R.row0 || row_hi < row_lo || row_hi > R.row0 + R.cap || row_hi > R.rows)
        return fail(s, MBG_E_ARG, "record rows outside the device-resident window");
    if (row_hi == row_lo) return MBG_OK;
    cudaSetDevice(s->g.device);
    const size_t off = (size_t)(row_lo - R.row0) * R.cols;
    const size_t bytes = sizeof(double) * (size_t)(row_hi - row_lo) * R.cols;
    CK(cudaMemcpyAsync(re, R.re + off, bytes, cudaMemcpyDeviceToHost, s->stream));
    if (R.im && im) CK(cudaMemcpyAsync(im, R.im + off, bytes, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

int mbg_set_record_row0(mbg_solver *s, int32_t r, int64_t row0) {
    if (!s || r < 0 || r >= (int)s->recs.size()) return MBG_E_ARG;
    Rec &R = s->recs[r];
    if (row0 < 0 || row0 > R.rows) return fail(s, MBG_E_ARG, "record window start outside [0, rows]");
    cudaSetDevice(s->g.device);
    R.row0 = row0;
    const size_t bytes = sizeof(double) * (size_t)R.cap * R.cols;
    CK(cudaMemsetAsync(R.re, 0, bytes, s->stream));
    if (R.im) CK(cudaMemsetAsync(R.im, 0, bytes, s->stream));
    return MBG_OK;
}

int mbg_download_record(mbg_solver *s, int32_t r, double *re, double *im) {
    if (!s || r < 0 || r >= (int)s->recs.size() || !re) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    const Rec &R = s->recs[r];
    if (R.cap < R.rows) return fail(s, MBG_E_STATE, "streamed record: use mbg_download_record_rows");
    const size_t bytes = sizeof(double) * (size_t)R.rows * R.cols;
    CK(cudaMemcpyAsync(re, R.re, bytes, cudaMemcpyDeviceToHost, s->stream));
    if (R.im && im) CK(cudaMemcpyAsync(im, R.im, bytes, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return MBG_OK;
}

int mbg_batch_points(mbg_solver *s, int32_t B, const int32_t *medium, const double *e_seq, double *state,
                     int32_t n_rec, const int32_t *quantity, const int32_t *ri, const int32_t *rj,
                     const int64_t *every, double *const *re, double *const *im) {
    if (!s || B < 1 || !medium || !e_seq || !state || n_rec < 0 || (n_rec && (!quantity || !ri || !rj || !every || !re)))
        return MBG_E_ARG;
    if (s->g.num_x != 1) return fail(s, MBG_E_ARG, "batched points need a single-grid-point solver (num_x = 1)");
    if (s->g.levels < 2 || s->qm.empty()) return fail(s, MBG_E_STATE, "quantum constants not set");
    if (n_rec > kMaxRecords) return fail(s, MBG_E_UNSUPPORTED, "too many records (max 64)");
    const int nq = (int)s->qm.size(), N = s->g.levels;
    for (int b = 0; b < B; ++b)
        if (medium[b] < 0 || medium[b] >= nq) return fail(s, MBG_E_ARG, "medium index out of range");
    BatchRecs R;
    std::memset(&R, 0, sizeof(R));
    R.n = n_rec;
    for (int r = 0; r < n_rec; ++r) {
        if ((quantity[r] != MBG_Q_D && quantity[r] != MBG_Q_INV) || every[r] < 1 || ri[r] < 0 || rj[r] < 0 ||
            ri[r] >= N || rj[r] >= N || (quantity[r] == MBG_Q_INV && N != 2))
            return fail(s, MBG_E_ARG, "batched records: density entries (or the two-level inversion) only");
        R.q[r] = quantity[r];
        R.i[r] = ri[r];
        R.j[r] = rj[r];
        R.every[r] = every[r];
        R.rows[r] = (s->g.num_t - 1) / every[r] + 1;
    }
    cudaSetDevice(s->g.device);
    const int words = s->words;
    double *d_e = nullptr, *d_s = nullptr;
    int *d_m = nullptr;
    std::vector<double *> bufs;
    std::vector<void *> qbufs;  // device constant sets of the media
    auto release = [&]() {
        dfree(s->stream, d_e);
        dfree(s->stream, d_s);
        dfree(s->stream, d_m);
        for (double *p : bufs) dfree(s->stream, p);
        for (void *p : qbufs) dfree(s->stream, p);
        cudaStreamSynchronize(s->stream);
    };
    auto step = [&](cudaError_t e, const char *what) {
        if (e == cudaSuccess) return true;
        s->err = std::string(what) + ": " + cudaGetErrorString(e);
        return false;
    };
    const size_t eb = sizeof(double) * (size_t)s->g.num_t * B, sb = sizeof(double) * (size_t)words * B;
    bool ok = step(dalloc(s->stream, &d_e, eb), "alloc") && step(dalloc(s->stream, &d_s, sb), "alloc") &&
              step(cudaMallocAsync(reinterpret_cast<void **>(&d_m), sizeof(int) * B, s->stream), "alloc") &&
              step(cudaMemcpyAsync(d_e, e_seq, eb, cudaMemcpyHostToDevice, s->stream), "copy") &&
              step(cudaMemcpyAsync(d_s, state, sb, cudaMemcpyHostToDevice, s->stream), "copy") &&
              step(cudaMemcpyAsync(d_m, medium, sizeof(int) * B, cudaMemcpyHostToDevice, s->stream), "copy");
    for (int r = 0; ok && r < n_rec; ++r) {
        const size_t rb = sizeof(double) * (size_t)R.rows[r] * B;
        ok = step(dalloc(s->stream, &R.re[r], rb), "alloc") &&
             step(cudaMemsetAsync(R.re[r], 0, rb, s->stream), "memset");
        bufs.push_back(R.re[r]);
        if (ok && R.q[r] == MBG_Q_D && R.i[r] != R.j[r]) {
            ok = step(dalloc(s->stream, &R.im[r], rb), "alloc") &&
                 step(cudaMemsetAsync(R.im[r], 0, rb, s->stream), "memset");
            bufs.push_back(R.im[r]);
        }
    }
    if (ok) {
        cudaError_t e;
        if (s->bloch) {
            BlochBatchParams P;
            std::memset(&P, 0, sizeof(P));
            P.B = B;
            P.num_t = s->g.num_t;
            P.e_seq = d_e;
            P.state = d_s;
            P.medium = d_m;
            P.R = R;
            P.n_qm = nq;
            P.real_dipole = 1;
            std::vector<BlochQm> hq(nq);
            std::vector<BlochReal> hr(nq);
            for (int q = 0; q < nq; ++q) {
                std::memcpy(&hq[q], s->qm[q].bloch, sizeof(BlochQm));
                hr[q] = bloch_real(hq[q]);
                P.real_dipole &= real_dipole(hq[q]) ? 1 : 0;
            }
            BlochQm *dq = nullptr;
            BlochReal *dr = nullptr;
            e = cudaMallocAsync(reinterpret_cast<void **>(&dq), sizeof(BlochQm) * nq, s->stream);
            if (e == cudaSuccess) {
                qbufs.push_back(dq);
                e = cudaMallocAsync(reinterpret_cast<void **>(&dr), sizeof(BlochReal) * nq, s->stream);
            }
            if (e == cudaSuccess) {
                qbufs.push_back(dr);
                e = cudaMemcpyAsync(dq, hq.data(), sizeof(BlochQm) * nq, cudaMemcpyHostToDevice, s->stream);
            }
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(dr, hr.data(), sizeof(BlochReal) * nq, cudaMemcpyHostToDevice, s->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);  // host vectors die at scope end
            P.qm = dq;
            P.rq = dr;
            if (e == cudaSuccess)
                e = s->g.exact ? exact::launch_batch_bloch(P, s->stream) : fast::launch_batch_bloch(P, s->stream);
        } else {
            switch (N) {
                case 2: e = batch_dense_n<2>(s, B, R, d_e, d_s, d_m, qbufs); break;
                case 3: e = batch_dense_n<3>(s, B, R, d_e, d_s, d_m, qbufs); break;
                case 4: e = batch_dense_n<4>(s, B, R, d_e, d_s, d_m, qbufs); break;
                case 5: e = batch_dense_n<5>(s, B, R, d_e, d_s, d_m, qbufs); break;
                case 6: e = batch_dense_n<6>(s, B, R, d_e, d_s, d_m, qbufs); break;
                case 7: e = batch_dense_n<7>(s, B, R, d_e, d_s, d_m, qbufs); break;
                case 8: e = batch_dense_n<8>(s, B, R, d_e, d_s, d_m, qbufs); break;
                default: e = cudaErrorInvalidValue;
            }
        }
        ok = step(e, "batch kernel");
        if (ok) ++s->launches;
    }
    for (int r = 0; ok && r < n_rec; ++r) {
        const size_t rb = sizeof(double) * (size_t)R.rows[r] * B;
        ok = step(cudaMemcpyAsync(re[r], R.re[r], rb, cudaMemcpyDeviceToHost, s->stream), "copy");
        if (ok && R.im[r] && im && im[r]) ok = step(cudaMemcpyAsync(im[r], R.im[r], rb, cudaMemcpyDeviceToHost, s->stream), "copy");
    }
    if (ok) ok = step(cudaMemcpyAsync(state, d_s, sb, cudaMemcpyDeviceToHost, s->stream), "copy");
    if (ok) ok = step(cudaStreamSynchronize(s->stream), "batch run");
    release();
    return ok ? MBG_OK : MBG_E_CUDA;
}

int mbg_halo_words(const mbg_solver *s, int32_t *words) {
    if (!s || !words) return MBG_E_ARG;
    *words = 2 + s->words;
    return MBG_OK;
}

static int halo(mbg_solver *s, bool pack, int64_t cell0, int64_t count, uint64_t buf) {
    if (!s || !buf || count < 0) return MBG_E_ARG;
    const long long l0 = cell0 - s->g.win_lo;
    if (l0 < 0 || l0 + count > s->win_n) return fail(s, MBG_E_ARG, "halo range outside the window");
    cudaSetDevice(s->g.device);
    CK(launch_halo(pack, s->e[s->cur], s->h[s->cur], s->s[s->cur], s->plane, s->words, l0, count,
                   reinterpret_cast<double *>(buf), s->stream));
    ++s->launches;
    return MBG_OK;
}

int mbg_pack_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t buf) { return halo(s, true, cell0, count, buf); }
int mbg_unpack_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t buf) { return halo(s, false, cell0, count, buf); }

/* ---- peer-memory ghost exchange (kernels_aux.cu: halo_push_kernel / halo_pull_kernel) ---- */

int mbg_mailbox_alloc(int32_t device, int64_t bytes, uint64_t *dev_ptr, unsigned char *ipc) {
    mbg_solver *s = nullptr;
    if (!dev_ptr || bytes <= 0) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    void *p = nullptr;
    CK(cudaMalloc(&p, (size_t)bytes));  // plain cudaMalloc: pool memory cannot be exported
    cudaError_t e = cudaMemset(p, 0, (size_t)bytes);
    if (e == cudaSuccess && ipc) {
        static_assert(sizeof(cudaIpcMemHandle_t) == MBG_IPC_HANDLE_BYTES, "IPC handle size");
        cudaIpcMemHandle_t hnd;
        e = cudaIpcGetMemHandle(&hnd, p);
        if (e == cudaSuccess) std::memcpy(ipc, &hnd, sizeof(hnd));
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(p);
        CK(e);
    }
    *dev_ptr = reinterpret_cast<uint64_t>(p);
    return MBG_OK;
}

int mbg_mailbox_free(int32_t device, uint64_t dev_ptr) {
    mbg_solver *s = nullptr;
    if (!dev_ptr) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    CK(cudaFree(reinterpret_cast<void *>(dev_ptr)));
    return MBG_OK;
}

int mbg_mailbox_map(int32_t device, const unsigned char *ipc, uint64_t *dev_ptr) {
    mbg_solver *s = nullptr;
    if (!ipc || !dev_ptr) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, ipc, sizeof(hnd));
    void *p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, hnd, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = reinterpret_cast<uint64_t>(p);
    return MBG_OK;
}

int mbg_mailbox_unmap(int32_t device, uint64_t dev_ptr) {
    mbg_solver *s = nullptr;
    if (!dev_ptr) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    CK(cudaIpcCloseMemHandle(reinterpret_cast<void *>(dev_ptr)));
    return MBG_OK;
}

static int halo_range(mbg_solver *s, int64_t cell0, int64_t count, long long *l0) {
    *l0 = cell0 - s->g.win_lo;
    if (*l0 < 0 || *l0 + count > s->win_n) return fail(s, MBG_E_ARG, "halo range outside the window");
    return MBG_OK;
}

int mbg_push_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t peer_slot, uint64_t peer_flag, uint64_t seq) {
    if (!s || !peer_slot || !peer_flag || count <= 0 || !seq) return MBG_E_ARG;
    long long l0 = 0;
    if (int rc = halo_range(s, cell0, count, &l0)) return rc;
    cudaSetDevice(s->g.device);
    if (!s->push_ticket) {
        CK(dalloc(s->stream, reinterpret_cast<double **>(&s->push_ticket), sizeof(double)));
        CK(cudaMemsetAsync(s->push_ticket, 0, sizeof(double), s->stream));
    }
    CK(launch_halo_push(s->e[s->cur], s->h[s->cur], s->s[s->cur], s->plane, s->words, l0, count,
                        reinterpret_cast<double *>(peer_slot), reinterpret_cast<unsigned long long *>(peer_flag),
                        seq, s->push_ticket, s->stream));
    ++s->launches;
    return MBG_OK;
}

int mbg_pull_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t slot, uint64_t flag, uint64_t seq,
                  int64_t timeout_ms) {
    if (!s || !slot || !flag || count <= 0 || !seq || timeout_ms <= 0) return MBG_E_ARG;
    long long l0 = 0;
    if (int rc = halo_range(s, cell0, count, &l0)) return rc;
    cudaSetDevice(s->g.device);
    s->peer_used = true;
    CK(launch_halo_pull(s->e[s->cur], s->h[s->cur], s->s[s->cur], s->plane, s->words, l0, count,
                        reinterpret_cast<const double *>(slot), reinterpret_cast<const unsigned long long *>(flag),
                        seq, (unsigned long long)timeout_ms * 1000000ull, reinterpret_cast<unsigned *>(s->bad + 1),
                        s->stream));
    ++s->launches;
    return MBG_OK;
}

int mbg_checkpoint_save(mbg_solver *s) {
    if (!s) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    const size_t fb = sizeof(double) * (s->win_n + 1);
    const size_t sb = sizeof(double) * (size_t)std::max(1, s->words) * s->plane;
    if (!s->ck_e) {
        CK(dalloc(s->stream, &s->ck_e, fb));
        CK(dalloc(s->stream, &s->ck_h, fb));
        CK(dalloc(s->stream, &s->ck_s, sb));
    }
    CK(cudaMemcpyAsync(s->ck_e, s->e[s->cur], fb, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->ck_h, s->h[s->cur], fb, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->ck_s, s->s[s->cur], sb, cudaMemcpyDeviceToDevice, s->stream));
    return MBG_OK;
}

int mbg_checkpoint_restore(mbg_solver *s) {
    if (!s) return MBG_E_ARG;
    if (!s->ck_e) return fail(s, MBG_E_STATE, "no checkpoint saved");
    cudaSetDevice(s->g.device);
    const size_t fb = sizeof(double) * (s->win_n + 1);
    const size_t sb = sizeof(double) * (size_t)std::max(1, s->words) * s->plane;
    CK(cudaMemcpyAsync(s->e[s->cur], s->ck_e, fb, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->h[s->cur], s->ck_h, fb, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->s[s->cur], s->ck_s, sb, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemsetAsync(s->bad, 0xff, sizeof(unsigned long long), s->stream));
    return MBG_OK;
}

int mbg_fp64_peak_sustained(int device, double seconds, double *tflops) {
    mbg_solver *s = nullptr;
    if (!tflops || !(seconds > 0)) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    double ms = 0.0, flops = 0.0;
    CK(measure_fp64_sustained(seconds, &ms, &flops));
    *tflops = flops / (ms * 1e-3) / 1e12;
    return MBG_OK;
}

int mbg_fp64_peak_operands(int device, int32_t mode, double *tflops) {
    mbg_solver *s = nullptr;
    if (!tflops || mode < 0 || mode > 3) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    double ms = 0.0, flops = 0.0;
    CK(measure_fp64_peak_operands(mode, &ms, &flops));
    *tflops = flops / (ms * 1e-3) / 1e12;
    return MBG_OK;
}

int mbg_fp64_peak(int device, double *tflops) {
    mbg_solver *s = nullptr;
    if (!tflops) return MBG_E_ARG;
    CK(cudaSetDevice(device));
    double ms = 0.0, flops = 0.0;
    CK(measure_fp64_peak(&ms, &flops));
    *tflops = flops / (ms * 1e-3) / 1e12;
    return MBG_OK;
}

int mbg_event_begin(mbg_solver *s) {
    if (!s) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    CK(cudaEventRecord(s->ev0, s->stream));
    return MBG_OK;
}

int mbg_event_end(mbg_solver *s, float *ms) {
    if (!s || !ms) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    CK(cudaEventRecord(s->ev1, s->stream));
    CK(cudaEventSynchronize(s->ev1));
    CK(cudaEventElapsedTime(ms, s->ev0, s->ev1));
    return MBG_OK;
}

int mbg_mark(mbg_solver *s, int32_t slot) {
    if (!s || slot < 0 || slot >= MBG_MAX_MARKS) return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    if (!s->marks[slot]) CK(cudaEventCreate(&s->marks[slot]));
    CK(cudaEventRecord(s->marks[slot], s->stream));
    return MBG_OK;
}

int mbg_mark_elapsed(mbg_solver *s, int32_t a, int32_t b, float *ms) {
    if (!s || !ms || a < 0 || b < 0 || a >= MBG_MAX_MARKS || b >= MBG_MAX_MARKS || !s->marks[a] || !s->marks[b])
        return MBG_E_ARG;
    cudaSetDevice(s->g.device);
    CK(cudaEventSynchronize(s->marks[b]));
    CK(cudaEventElapsedTime(ms, s->marks[a], s->marks[b]));
    return MBG_OK;
}

int mbg_launch_count(const mbg_solver *s, int64_t *launches) {
    if (!s || !launches) return MBG_E_ARG;
    *launches = s->launches;
    return MBG_OK;
}

}  // extern "C"
