/*
 * mbgpu.h -- C ABI of the B200 time-stepping core (libmbgpu.so).
 *
 * The reference has no FFI: its hot loop is FdtdSolver.run()
 * (/root/reference/pkg/src/mblight/solver_fdtd.py:444-498) calling numba
 * loops per step.  This ABI is the seam a Python (ctypes) or any other host
 * binds to replace that loop; the setup arithmetic stays in the host
 * (paper_2005_05412_b200/plan.py builds it with the reference's own setup
 * functions and kernel constructors, FdtdSolver.__init__,
 * solver_fdtd.py:207-326) and is passed here as plain arrays.
 *
 * Entry point -> reference interface it replaces:
 *   mbg_create            FdtdSolver.__init__ state allocation      solver_fdtd.py:235-240
 *   mbg_set_regions       per-cell coefficient arrays              solver_fdtd.py:242-272
 *   mbg_set_qm_bloch      BlochSplittingKernel constants           _kernels.py:467-494
 *   mbg_set_qm_dense      VectorSplittingKernel constants          _kernels.py:431-439
 *   mbg_set_qm_rk4        VectorRk4Kernel constants                _kernels.py:552-557
 *   mbg_set_boundary      boundary precompute                      solver_fdtd.py:310-325
 *   mbg_set_sources       Source.value(n dt) per step              solver_fdtd.py:379-385
 *   mbg_set_source_rows   (same samples, streamed per run segment)  solver_fdtd.py:379-385
 *   mbg_set_records       _RecordPlan list                         solver_fdtd.py:136-172,300-305
 *   mbg_upload_fields     initial E / H                            solver_fdtd.py:237-239
 *   mbg_upload_density    DensityKernel.init_state                 _kernels.py:376-377, 496-500
 *   mbg_sample            _sample(0)                               solver_fdtd.py:449
 *   mbg_advance           the step loop (phase1/2 + after_*)       solver_fdtd.py:457-463
 *   mbg_poll_nonfinite    SolverError("non-finite ... at step n")  solver_fdtd.py:386-388
 *   mbg_download_record   plan.to_result                           solver_fdtd.py:164-172
 *   mbg_invariants        DensityKernel.invariant_stats            _kernels.py:394-401, 541-546
 *   mbg_batch_points      many Nx = 1 runs (ScalarKernel path)     solver_fdtd.py:89-96,347-349; _kernels.py:404-425
 *   mbg_pack_halo/unpack  (new) slab ghost exchange, no reference analogue
 *   mbg_push_halo/pull    (new) the same exchange through peer device memory (the worker
 *                         threads' shared arrays across the partition)  solver_fdtd.py:465-498
 *
 * Conventions: every function returns 0 on success or a negative MBG_E_*
 * code; mbg_last_error() gives the message.  All host pointers are plain
 * C arrays owned by the caller and only read during the call.  Device
 * memory is owned by the solver handle.  Cells are global grid indices.
 */
#ifndef MBGPU_H
#define MBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBG_OK 0
#define MBG_E_ARG (-1)
#define MBG_E_CUDA (-2)
#define MBG_E_UNSUPPORTED (-3)
#define MBG_E_STATE (-4)

#define MBG_STEPPER_SPLITTING 0
#define MBG_STEPPER_RK4 1

#define MBG_Q_E 0
#define MBG_Q_H 1
#define MBG_Q_D 2
#define MBG_Q_INV 3

#define MBG_MAX_REGIONS 128
#define MBG_MAX_QM 4
/* distinct quantum materials of one mbg_batch_points call (constant sets in device memory) */
#define MBG_MAX_BATCH_QM 65536
#define MBG_MAX_SOURCES 32
#define MBG_MAX_RECORDS 64
#define MBG_MAX_LEVELS 8
#define MBG_MAX_TILE_STEPS 128

/* mbg_grid.flags: one kernel launch per k fused steps instead of the
   persistent wavefront launch (two-level / classical, non-windowed solvers) */
#define MBG_FLAG_PER_LAUNCH 1
/* two-level / classical media: always the persistent wavefront launch (by
 * default it is used when a fused chunk has at least one tile per SM; a
 * narrower domain is a chain of few tiles, faster as one launch per chunk
 * with a whole SM per tile) */
#define MBG_FLAG_PERSISTENT 2
/* mbg_grid.flags: the kernels' default tile depth as such (no small-domain
   deepening, see mbg_create): what a slab of this scenario uses */
#define MBG_FLAG_DEFAULT_DEPTH 4

typedef struct mbg_solver mbg_solver;

typedef struct {
    int64_t num_x;      /* global grid points (>= 1) */
    int64_t num_t;      /* time levels; the run is steps 1 .. num_t-1 */
    double dt, dx;
    int32_t levels;     /* N of every quantum material, 0 if none */
    int32_t stepper;    /* MBG_STEPPER_* */
    int32_t tile_steps; /* k: time steps fused per kernel launch (0 = default) */
    int32_t exact;      /* 1: no FMA contraction (bit-exact to the reference for N = 2) */
    int32_t device;     /* CUDA device ordinal */
    int32_t flags;      /* MBG_FLAG_* */
    int64_t win_lo, win_hi; /* cells held on this device (slab incl. ghosts) */
    int64_t own_lo, own_hi; /* cells owned (recorded, scanned) by this device */
} mbg_grid;

/* lifecycle */
int mbg_create(const mbg_grid *grid, mbg_solver **out);
void mbg_destroy(mbg_solver *s);
const char *mbg_last_error(const mbg_solver *s);
const char *mbg_version(void);
int mbg_device_count(int *count);
/* stream: 0 = solver-owned stream; otherwise a cudaStream_t to launch on */
int mbg_set_stream(mbg_solver *s, uint64_t stream);
int mbg_tile_steps(const mbg_solver *s, int32_t *k);

/* setup (host arrays, copied) */
int mbg_set_regions(mbg_solver *s, int32_t n, const int64_t *e_start, const int64_t *h_start,
                    const double *coef_a, const double *coef_bg, const double *coef_bdx,
                    const double *coef_ch, const int32_t *qm_index);
/* c[15] = kz cz fxy ax_c ax_s ay_c ay_s az_c az_s a0_c a0_s mu_x mu_y mu_z pol_factor */
int mbg_set_qm_bloch(mbg_solver *s, int32_t qm, const double *c);
/* row-major N x N; complex arrays interleaved (re, im); pol lists as _kernels.py:360-374 */
int mbg_set_qm_dense(mbg_solver *s, int32_t qm, const double *pop_half, const double *coh_half,
                     const double *b_const, const double *b_field, int32_t npol,
                     const int32_t *pol_i, const int32_t *pol_j, const double *pol_v,
                     int32_t ndpol, const int32_t *pol_di, const double *pol_dv, double pol_factor);
int mbg_set_qm_rk4(mbg_solver *s, int32_t qm, const double *h0, const double *mu,
                   const double *pop_matrix, const double *deph_matrix, int32_t npol,
                   const int32_t *pol_i, const int32_t *pol_j, const double *pol_v,
                   int32_t ndpol, const int32_t *pol_di, const double *pol_dv, double pol_factor);
/* w = 1 - sqrt(R), c = v dt / dx, z = sqrt(mu / eps) of the edge materials */
int mbg_set_boundary(mbg_solver *s, double wl, double cl, double zl, double wr, double cr, double zr);
/* values: [num_t][n] samples Source.value(n dt) (row 0 unused); NULL: the
 * table starts zero and its rows come through mbg_set_source_rows */
int mbg_set_sources(mbg_solver *s, int32_t n, const int64_t *cell, const int32_t *hard,
                    const double *values);
/* rows [lo, hi) of the sample table (rows: (hi - lo) x n doubles), copied
 * stream-ordered through pinned staging: the run samples its sources segment
 * by segment while the device steps (Source.value inside the reference's
 * loop, solver_fdtd.py:379-385) */
int mbg_set_source_rows(mbg_solver *s, int64_t lo, int64_t hi, const double *rows);
/* *idle = 1 when every operation enqueued on the solver's stream has completed
 * (non-blocking; paces the host's source sampling against the device) */
int mbg_stream_idle(mbg_solver *s, int32_t *idle);
/* quantity MBG_Q_*, cell -1 = whole domain, i/j 0-based, every >= 1; complex for d with i != j */
int mbg_set_records(mbg_solver *s, int32_t n, const int32_t *quantity, const int64_t *cell,
                    const int32_t *i, const int32_t *j, const int64_t *every);

/* state: e has (win_hi - win_lo) entries, h has one more (node win_hi);
 * e == h == NULL sets both fields to zero on the device (no host copy) */
int mbg_upload_fields(mbg_solver *s, const double *e, const double *h);
/* one packed state vector (words per cell) broadcast to every quantum cell */
int mbg_upload_density(mbg_solver *s, const double *words);
/* full state planes [words][win cells] (tests, restarts) */
int mbg_upload_state(mbg_solver *s, const double *planes);
int mbg_download_fields(mbg_solver *s, double *e, double *h);
int mbg_download_state(mbg_solver *s, double *planes);

/* run */
int mbg_sample(mbg_solver *s, int64_t step);
/* steps first_step .. first_step + n_steps - 1, asynchronous on the solver
 * stream.  Two-level / classical media: one persistent wavefront launch for
 * the whole range (unless MBG_FLAG_PER_LAUNCH); N >= 3 and RK4: one launch per
 * k steps.  A windowed solver (slab) advances at most its ghost width. */
int mbg_advance(mbg_solver *s, int64_t first_step, int64_t n_steps);
/* waits for the stream; reports a persistent launch that gave up waiting */
int mbg_synchronize(mbg_solver *s);
int mbg_poll_nonfinite(mbg_solver *s, int64_t *bad_step); /* syncs; -1 when all finite */
/* invariant monitor of the current state (_kernels.py:394-401, solver_fdtd.py:428-440):
 * out[0] max |trace - 1|, out[1] max Hermiticity deviation, out[2] min eigenvalue
 * over the owned quantum cells (+inf when there are none) */
int mbg_invariants(mbg_solver *s, double *out);
/* the same statistics folded into device-resident running maxima / minima
 * without a host synchronisation (queued on the solver stream at every
 * monitored step); mbg_invariants_read syncs and returns them */
int mbg_invariants_accumulate(mbg_solver *s);
/* two-level splitting media: the step kernels fold the monitor themselves at
 * every step that is a multiple of `every` (0: off), in the same running
 * statistics -- no launch split at the monitored steps */
int mbg_set_monitor(mbg_solver *s, int64_t every);
int mbg_invariants_read(mbg_solver *s, double *out);
int mbg_record_shape(const mbg_solver *s, int32_t r, int64_t *rows, int64_t *cols);
int mbg_download_record(mbg_solver *s, int32_t r, double *re, double *im);
/* Streamed records (the reference keeps every row in host memory,
 * solver_fdtd.py:164-172, 398-424; here only a window of rows lives in HBM):
 * mbg_set_record_rows gives record r a device window of `cap` rows starting
 * at row 0 (after mbg_set_records); steps may only write rows inside the
 * window (mbg_advance / mbg_sample refuse otherwise); completed rows are
 * copied out with mbg_download_record_rows into the caller's host rows
 * [row_lo, row_hi) and the window is moved on with mbg_set_record_row0. */
int mbg_set_record_rows(mbg_solver *s, int32_t r, int64_t cap);
int mbg_download_record_rows(mbg_solver *s, int32_t r, int64_t row_lo, int64_t row_hi, double *re, double *im);
int mbg_set_record_row0(mbg_solver *s, int32_t r, int64_t row0);

/* Batched single-point systems (many Nx = 1 master-equation runs
 * of solver_fdtd.py:89-96, 347-349 per launch).  The handle is a num_x = 1
 * solver whose media (mbg_set_qm_*) the B systems index by medium[b]; at one
 * grid point the field is source-driven only, so e_seq [num_t][B] holds every
 * system's E at every step (computed by the caller from its sources), state
 * [words][B] the initial packed states (overwritten with the final ones).
 * Density records (MBG_Q_D with 0-based i, j; MBG_Q_INV for two-level media, either stepper)
 * of rows (num_t - 1)/every + 1 are written to re[r] / im[r] as [B][rows];
 * row 0 (the initial state) is left to the caller.  Blocking. */
int mbg_batch_points(mbg_solver *s, int32_t B, const int32_t *medium, const double *e_seq, double *state,
                     int32_t n_rec, const int32_t *quantity, const int32_t *i, const int32_t *j,
                     const int64_t *every, double *const *re, double *const *im);

/* multi-device slabs: pack/unpack `count` cells starting at global cell
 * `cell0` of E, H and every state plane into/out of a device buffer of
 * (2 + words) * count doubles (ordered on the solver's stream) */
int mbg_halo_words(const mbg_solver *s, int32_t *words);
int mbg_pack_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t dev_buf);
int mbg_unpack_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t dev_buf);

/* Peer-memory ghost exchange (multi-device slabs without a library collective
 * on the data path; the reference's counterpart is the shared arrays its
 * worker threads read across the partition bounds, solver_fdtd.py:465-498).
 * A mailbox is plain device memory owned by the RECEIVING rank, exported
 * through CUDA IPC and mapped by the neighbour (mbg_mailbox_map in the
 * neighbour's process; the same process passes the pointer itself).  The
 * caller lays it out: per interface two slots of (2 + words) * count doubles
 * and one zero-initialised 64-bit flag per slot.
 *   mbg_push_halo: store `count` cells from `cell0` (E, H, state planes, the
 *     mbg_pack_halo order) into the neighbour's slot and publish `seq` (> 0,
 *     increasing per slot) in its flag with a system-scope release -- NVLink
 *     stores on a multi-GPU box, ordered on the solver's stream.
 *   mbg_pull_halo: wait on the device until the flag reaches `seq`, then copy
 *     the slot into the ghost cells from `cell0`.  A strip that does not
 *     arrive within timeout_ms leaves the ghosts stale and sets the handle's
 *     sticky stall flag: the next mbg_synchronize / mbg_poll_nonfinite fails.
 * Slot reuse needs no acknowledgement with two slots used alternately: a
 * rank's push of period p + 2 is ordered after its pull of period p + 1, which
 * waited for the neighbour's push of p + 1, itself ordered after the
 * neighbour's pull of period p from the same slot. */
#define MBG_IPC_HANDLE_BYTES 64
int mbg_mailbox_alloc(int32_t device, int64_t bytes, uint64_t *dev_ptr, unsigned char *ipc_handle /* [64] or NULL */);
int mbg_mailbox_free(int32_t device, uint64_t dev_ptr);
int mbg_mailbox_map(int32_t device, const unsigned char *ipc_handle, uint64_t *dev_ptr);
int mbg_mailbox_unmap(int32_t device, uint64_t dev_ptr);
int mbg_push_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t peer_slot, uint64_t peer_flag, uint64_t seq);
int mbg_pull_halo(mbg_solver *s, int64_t cell0, int64_t count, uint64_t slot, uint64_t flag, uint64_t seq,
                  int64_t timeout_ms);

/* device-side checkpoint of E, H and the density state (save / restore the
 * current buffers; no reference analogue: FdtdSolver has no checkpointing) */
int mbg_checkpoint_save(mbg_solver *s);
int mbg_checkpoint_restore(mbg_solver *s);

/* measured FP64 FMA throughput of the device (TFLOP/s), the FP64 roofline
 * denominator: independent DFMA chains on every SM, timed with CUDA events */
int mbg_fp64_peak(int device, double *tflops);
/* the same measurement by operand pattern: mode 1 = two registers and a
 * uniform addend (the pipe's peak: what mbg_fp64_peak measures), 0 = multiplier
 * and addend registers shared by every instruction, 2 = one multiplier register
 * shared by consecutive DFMAs (operand reuse cache), 3 = three distinct register
 * operands per DFMA (matrix arithmetic with every operand fresh: limited by the
 * register file's operand bandwidth) */
int mbg_fp64_peak_operands(int device, int32_t mode, double *tflops);
/* the same DFMA chains back to back for at least `seconds` (sustained clocks
 * and power): the denominator for kernels timed inside a long run */
int mbg_fp64_peak_sustained(int device, double seconds, double *tflops);

/* timing helpers for bench.py: device time of the launches issued by
 * mbg_advance between mark_begin/mark_end (CUDA events on the solver stream) */
int mbg_event_begin(mbg_solver *s);
int mbg_event_end(mbg_solver *s, float *ms);
/* numbered events on the solver stream (slot < MBG_MAX_MARKS) for timing a
 * part of a timed region without synchronising inside it; mbg_mark_elapsed
 * waits for mark b and returns the device time from mark a to mark b */
#define MBG_MAX_MARKS 64
int mbg_mark(mbg_solver *s, int32_t slot);
int mbg_mark_elapsed(mbg_solver *s, int32_t a, int32_t b, float *ms);
/* kernels this handle has launched so far (step, edge, sample and halo kernels) */
int mbg_launch_count(const mbg_solver *s, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* MBGPU_H */
