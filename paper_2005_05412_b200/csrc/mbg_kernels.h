// Launchers of the step kernels.  Each kernel translation unit is compiled
// twice: MBG_VARIANT=fast (FMA contraction allowed) and MBG_VARIANT=exact
// (-fmad=false, IEEE operation order of the reference's numba loops, which
// makes the two-level path bit-identical to the reference).
#pragma once
#include <cuda_runtime.h>

#include "mbg_params.cuh"

namespace mbg {

#ifdef __CUDACC__
// a*b + c.  Fast variant: one fused multiply-add.  Exact variant: a rounded
// product then a rounded sum -- with IEEE commutativity this is exactly the
// reference's "c + a*b" / "a*b + c" for every place it is used.
__device__ __forceinline__ double mad(double a, double b, double c) {
#if defined(MBG_EXACT) && MBG_EXACT
    return __dadd_rn(__dmul_rn(a, b), c);
#else
    return fma(a, b, c);
#endif
}
#endif

// tile geometry of the N = 2 kernel: one warp per tile, C cells per lane
#ifndef MBG_BLOCH_C
#define MBG_BLOCH_C 8
#endif
constexpr int kBlochCellsPerLane = MBG_BLOCH_C;
constexpr int kBlochTile = 32 * kBlochCellsPerLane;  // one warp
#ifndef MBG_BLOCH_WARPS
#define MBG_BLOCH_WARPS 8
#endif
constexpr int kBlochWarpsPerBlock = MBG_BLOCH_WARPS;
// interior tiles are one CTA: the warps side by side exchange their seam cells
// through shared memory, so the redundant halo is paid once per CTA tile
constexpr int kBlochCtaTile = kBlochWarpsPerBlock * kBlochTile;
// dense kernels: one thread per cell, one CTA per tile
// dense kernels: one thread per cell, one CTA per tile; small N use wide tiles
// (less redundant halo) at 128 registers, large N narrow tiles (state in smem)
// (six-level RK4: 96-cell tiles, so two CTAs of three shared-memory state
// buffers fit an SM)
__host__ __device__ constexpr int dense_tile_width(int n, bool rk4) {
#ifdef MBG_DENSE_TW
    if (n >= 5 && !rk4) return MBG_DENSE_TW;  // tuning builds
#endif
#ifdef MBG_DENSE_TW3
    if (n == 3 && !rk4) return MBG_DENSE_TW3;
#endif
    return n <= 3 ? 256 : (rk4 && n == 6 ? 96 : (n <= 6 ? 128 : 64));
}
__host__ __device__ constexpr int dense_min_blocks(int n, bool rk4) {
#ifdef MBG_DENSE_MINB
    if (n >= 5 && !rk4) return MBG_DENSE_MINB;  // tuning builds
#endif
#ifdef MBG_DENSE_MINB3
    if (n == 3 && !rk4) return MBG_DENSE_MINB3;
#endif
    return n <= 3 ? 2 : 1;
}
// Four- and five-level splitting on large grids (at least two tiles per SM
// slot): a second instantiation with three CTAs per SM (168 registers, 12
// warps) beats two CTAs at 234 / 255 registers -- N = 4 1.58e10 -> 1.69e10
// (real media 1.89e10 -> 2.11e10), N = 5 8.05e9 -> 8.54e9 (1.009e10 ->
// 1.053e10); four CTAs at 128 registers spill and lose (N = 4: 1.55e10).
// Small domains (every tile on its own SM, e.g. the paper's QCL setups) are
// bound by one tile's latency and keep the spill-free variant (the
// three-CTA one: tzenov2016 0.76 -> 0.88 s).
__host__ __device__ constexpr int dense_min_blocks_large(int n, bool rk4) {
    return ((n == 4 || n == 5) && !rk4) ? 3 : dense_min_blocks(n, rk4);
}

// One persistent launch of the two-level kernel over many fused chunks
// (non-windowed solvers): work items (chunk c, tile t) are claimed in
// chunk-major ticket order; item (c, t) waits until (c-1, t-1..t+1) are done,
// so chunk c overlaps the tail of chunk c-1 and there is no launch gap or
// wave-quantisation tail per chunk.  Chunk c reads buffer (cur + c) & 1 and
// writes the other one.  Launch geometry (k, tile_own) is the one in P.L;
// chunk c runs steps n0 + c*k .. (the last chunk may be shorter).
// result range [lo, hi) of one work item: an interior CTA tile, or up to a
// few warp ranges of a non-interior tile (split so that those slower general
// path items do not become a serial chain through the wavefront); every item
// but the last is at least k cells long, so item j only reads cells of the
// previous chunk's items j-1 .. j+1
struct WaveItem {
    long long lo, hi;
    int edge, pad;
};

struct BlochWave {
    int n_chunks;
    int last_steps;              // steps of the last chunk (<= P.L.k)
    long long tiles;             // work items per chunk
    const WaveItem *items;       // [tiles]
    long long n0;                // first step of chunk 0
    long long last_step;         // num_t - 1 (always scanned)
    const unsigned long long *masks;  // [n_chunks * k] record masks of every step (wave_masks)
    const unsigned char *checks;      // [n_chunks * k] non-finite scan flags
    double *e[2], *h[2], *s[2];
    int cur;                     // buffer holding the state at step n0 - 1
    unsigned int *ticket;        // claim counter (zeroed before the launch)
    unsigned int *done;          // [n_chunks * tiles] completion flags (zeroed)
    unsigned int *stall;         // set if a dependency wait timed out
    unsigned long long *trace;   // debug: per item {claimed, deps met, done, sm} ns (null: off)
};

#define MBG_DECLARE_LAUNCHERS(NS)                                                             \
    namespace NS {                                                                            \
    int bloch_cta_tile();                                                                     \
    cudaError_t launch_bloch(const BlochParams &P, long long tiles, cudaStream_t st, int *kernels); \
    cudaError_t launch_bloch_wave(const BlochParams &P, const BlochWave &V, cudaStream_t st);     \
    cudaError_t launch_wave_masks(const Launch &L, long long n_steps, long long last_step,          \
                                  unsigned long long *masks, unsigned char *checks, cudaStream_t st); \
    cudaError_t launch_dense_split(int n, const void *params, long long tiles, cudaStream_t st); \
    cudaError_t launch_dense_rk4(int n, const void *params, long long tiles, cudaStream_t st);   \
    cudaError_t launch_batch_dense(int n, bool rk4, const void *params, int systems, cudaStream_t st); \
    cudaError_t launch_batch_bloch(const BlochBatchParams &P, cudaStream_t st);                   \
    }

MBG_DECLARE_LAUNCHERS(fast)
MBG_DECLARE_LAUNCHERS(exact)

// auxiliary kernels (variant independent)
cudaError_t launch_sample(const Launch &L, int levels, int bloch, long long step, const BlochFrame &F,
                          cudaStream_t st);
// relaxed-frame state: in place to the frame (to_frame), or out of it into `out`
cudaError_t launch_frame(bool to_frame, double *s, long long plane, long long win_n, const Regions &rg,
                         long long win_lo, const BlochFrame &F, double *out, cudaStream_t st);
cudaError_t launch_broadcast_state(double *s, long long plane, long long win_n, int words,
                                   const double *words_dev, const Regions &rg, long long win_lo,
                                   cudaStream_t st);
cudaError_t launch_halo(bool pack, double *e, double *h, double *s, long long plane, int words,
                        long long l0, long long count, double *buf, cudaStream_t st);

// peer-memory ghost exchange: store the cells into the receiver's mailbox slot
// and publish `seq` in its flag (push); wait for `seq`, copy the slot into the
// ghost cells (pull; sets bit 1 of *stall after timeout_ns without the strip)
cudaError_t launch_halo_push(double *e, double *h, double *s, long long plane, int words, long long l0,
                             long long count, double *slot, unsigned long long *flag, unsigned long long seq,
                             unsigned *ticket, cudaStream_t st);
cudaError_t launch_halo_pull(double *e, double *h, double *s, long long plane, int words, long long l0,
                             long long count, const double *slot, const unsigned long long *flag,
                             unsigned long long seq, unsigned long long timeout_ns, unsigned *stall,
                             cudaStream_t st);

// invariant monitor: out[0] max |trace - 1|, out[1] max Hermiticity deviation
// (0: packed storage), out[2] min eigenvalue, as order-preserving uint64 keys
cudaError_t launch_invariants(const Launch &L, int levels, int bloch, const BlochFrame &F, unsigned long long *out,
                              cudaStream_t st);

// FP64 roofline denominator: best-of-5 DFMA throughput (ms of the best launch, flops per launch)
cudaError_t measure_fp64_peak(double *ms, double *flops);
cudaError_t measure_fp64_sustained(double seconds, double *ms, double *flops);
// the same chains by operand pattern: mode 3 three distinct register operands per
// DFMA, 2 a multiplier register shared by consecutive DFMAs, 1 a uniform addend
cudaError_t measure_fp64_peak_operands(int mode, double *ms, double *flops);

}  // namespace mbg
