"""Multi-GPU slab decomposition of the time-stepping core.

The 1D domain is cut into G contiguous slabs with the reference's own
partition rule (``np.linspace(0, Nx, G+1)``, solver_fdtd.py:468 -- there it
splits cells among CPU worker threads).  Each slab is held on its device as a
window [own_lo - g, own_hi + g) (clipped at the physical ends): g ghost cells
per side, g = the exchange period P = m * k steps (k = the temporal tile
depth; m = 32 chunks for the two-level / classical kernels, whose persistent
launch runs the m chunks back to back, 1 otherwise).  The valid region shrinks
by one cell per side per step, so after P steps exactly the owned cells are
current and the ghosts are refreshed by a point-to-point exchange with the two
neighbours -- E, H and every density plane of g cells per interface and
direction.  There is no other collective on the data path:
records are gathered once at the end and the non-finite flag is combined with
one MIN reduction per poll.

Every cell executes the same instruction sequence whatever slab or tile it
lands in, so results are bitwise independent of G (tested).

Transports:
  * :class:`LocalTransport` -- all slabs in one process on one device, ghost
    refresh by device-to-device pack/unpack (single-GPU tests of the slab
    path, no kernel ever waits on another).
  * :class:`TorchTransport` -- one process per GPU, ``torch.distributed``
    batched isend/irecv (NCCL over NVLink on the B200 box, gloo on CPU).
"""

from __future__ import annotations

import ctypes as C
from contextlib import nullcontext as _nullcontext
from dataclasses import dataclass

import numpy as np

from . import native
from .reference import mblight

SolverError = mblight.SolverError


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    own_lo: int
    own_hi: int
    win_lo: int
    win_hi: int

    @property
    def ghost_left(self) -> int:
        return self.own_lo - self.win_lo

    @property
    def ghost_right(self) -> int:
        return self.win_hi - self.own_hi


def partition(num_x: int, world: int, ghost: int) -> list[Slab]:
    """Contiguous slabs (reference rule, solver_fdtd.py:468) with ``ghost`` cells per side."""
    if world < 1 or world > num_x:
        raise ValueError("need 1 <= slabs <= cells")
    bounds = np.linspace(0, num_x, world + 1).astype(int)
    slabs = []
    for r in range(world):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        if hi - lo < ghost and world > 1:
            raise ValueError(f"slab {r} has {hi - lo} cells, fewer than the ghost width {ghost}")
        slabs.append(Slab(r, world, lo, hi, max(0, lo - ghost), min(num_x, hi + ghost)))
    return slabs


def exchange_plan(slab: Slab):
    """(send_left, recv_left, send_right, recv_right) as (cell0, count) or None.

    My left ghost [win_lo, own_lo) is the left neighbour's rightmost owned
    cells, and what I send left is my first cells [own_lo, own_lo + g) where
    g is the left neighbour's right ghost width (same partition, same k)."""
    sl = rl = sr = rr = None
    if slab.ghost_left:
        rl = (slab.win_lo, slab.ghost_left)
        sl = (slab.own_lo, slab.ghost_left)  # neighbour's right ghost has the same width
    if slab.ghost_right:
        rr = (slab.own_hi, slab.ghost_right)
        sr = (slab.own_hi - slab.ghost_right, slab.ghost_right)
    return sl, rl, sr, rr


class SlabState:
    """One slab on one device: the native handle plus its geometry."""

    def __init__(self, solver, slab: Slab, stream: int = 0):
        self.solver = solver
        self.slab = slab
        self.h = solver.open_handle(win=(slab.win_lo, slab.win_hi), own=(slab.own_lo, slab.own_hi))
        if stream:
            self.h.call("mbg_set_stream", stream)
        solver.upload_initial_state(self.h, win=(slab.win_lo, slab.win_hi))
        w = C.c_int32(0)
        self.h.call("mbg_halo_words", C.byref(w))
        self.words = w.value  # per cell: E, H, state planes

    def sample(self, step):
        self.h.call("mbg_sample", step)

    def advance(self, first, count):
        self.h.call("mbg_advance", first, count)

    def pack(self, cell0, count, ptr):
        self.h.call("mbg_pack_halo", cell0, count, ptr)

    def unpack(self, cell0, count, ptr):
        self.h.call("mbg_unpack_halo", cell0, count, ptr)

    # transport-facing: device tensors
    def pack_into(self, cell0, count, tensor):
        self.pack(cell0, count, tensor.data_ptr())

    def unpack_from(self, cell0, count, tensor):
        self.unpack(cell0, count, tensor.data_ptr())

    def poll(self) -> int:
        bad = C.c_int64(-1)
        self.h.call("mbg_poll_nonfinite", C.byref(bad))
        return bad.value

    def records(self):
        """Per record: (rows, cols) arrays of this slab's owned columns."""
        out = []
        for r, p in enumerate(self.solver.plan.plans):
            rows, cols = C.c_int64(0), C.c_int64(0)
            self.h.call("mbg_record_shape", r, C.byref(rows), C.byref(cols))
            re = np.zeros((rows.value, cols.value))
            im = np.zeros((rows.value, cols.value)) if p.is_complex else None
            self.h.call("mbg_download_record", r, native.ptr(re), native.ptr(im))
            out.append(re if im is None else re + 1j * im)
        return out

    def close(self):
        self.h.close()


def assemble(plan, slabs, per_slab_records):
    """Merge slab records into full records (point records from their owner)."""
    out = []
    for r, p in enumerate(plan.plans):
        if p.cell is None:
            out.append(np.concatenate([recs[r] for recs in per_slab_records], axis=1))
        else:
            owner = next(i for i, s in enumerate(slabs) if s.own_lo <= p.cell < s.own_hi)
            out.append(per_slab_records[owner][r])
    return out


# ---------------------------------------------------------------- transports --

class LocalTransport:
    """All slabs in this process on one device; ghosts refreshed device-to-device."""

    def __init__(self, states):
        import torch

        self.states = states
        words = max(s.words for s in states)
        k = max(max(s.slab.ghost_left, s.slab.ghost_right) for s in states)
        self.buf = torch.empty(max(1, words * k), dtype=torch.float64, device=f"cuda:{states[0].solver.gpu}")

    def exchange(self):
        # sequential per interface: pack the owner's cells, unpack into the ghost
        ptr = self.buf.data_ptr()
        for i, st in enumerate(self.states):
            sl, rl, sr, rr = exchange_plan(st.slab)
            if rl is not None:
                left = self.states[i - 1]
                left.pack(rl[0], rl[1], ptr)
                st.unpack(rl[0], rl[1], ptr)
            if rr is not None:
                right = self.states[i + 1]
                right.pack(rr[0], rr[1], ptr)
                st.unpack(rr[0], rr[1], ptr)
        for st in self.states:
            st.h.call("mbg_synchronize")


class TorchTransport:
    """One slab per process; neighbours exchange with batched isend/irecv."""

    def __init__(self, state: SlabState, device):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.state = state
        sl, rl, sr, rr = exchange_plan(state.slab)
        self.plan = (sl, rl, sr, rr)
        w = state.words

        def buf(spec):
            return None if spec is None else torch.empty(w * spec[1], dtype=torch.float64, device=device)

        self.send_l, self.recv_l, self.send_r, self.recv_r = buf(sl), buf(rl), buf(sr), buf(rr)
        # gloo moves host memory only: device buffers are staged through pinned
        # host copies (CPU tests, and several ranks sharing one GPU); NCCL
        # sends the device buffers directly
        self.stage = (torch.device(device).type == "cuda" and dist.get_backend() == "gloo")
        if self.stage:
            def host(b):
                return None if b is None else torch.empty(b.numel(), dtype=b.dtype, pin_memory=True)

            self.h_send_l, self.h_recv_l = host(self.send_l), host(self.recv_l)
            self.h_send_r, self.h_recv_r = host(self.send_r), host(self.recv_r)

    def exchange(self):
        sl, rl, sr, rr = self.plan
        st, dist = self.state, self.dist
        rank = st.slab.rank
        ops = []
        if self.stage:
            send_l, recv_l, send_r, recv_r = self.h_send_l, self.h_recv_l, self.h_send_r, self.h_recv_r
        else:
            send_l, recv_l, send_r, recv_r = self.send_l, self.recv_l, self.send_r, self.recv_r
        if sl is not None:
            st.pack_into(sl[0], sl[1], self.send_l)
            ops.append(dist.P2POp(dist.isend, send_l, rank - 1))
            ops.append(dist.P2POp(dist.irecv, recv_l, rank - 1))
        if sr is not None:
            st.pack_into(sr[0], sr[1], self.send_r)
            ops.append(dist.P2POp(dist.isend, send_r, rank + 1))
            ops.append(dist.P2POp(dist.irecv, recv_r, rank + 1))
        if self.stage:
            for d, h in ((self.send_l, send_l), (self.send_r, send_r)):
                if d is not None:
                    h.copy_(d)  # synchronous: the pack kernel has run
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self.stage:
            for d, h in ((self.recv_l, recv_l), (self.recv_r, recv_r)):
                if d is not None:
                    d.copy_(h)
        if rl is not None:
            st.unpack_from(rl[0], rl[1], self.recv_l)
        if rr is not None:
            st.unpack_from(rr[0], rr[1], self.recv_r)


# ---------------------------------------------------------------- drivers --

def _step_loop(grid, k, advance, exchange, poll, poll_every=1 << 14):
    n = 1
    since = 0
    while n < grid.num_t:
        cnt = min(k, grid.num_t - n)
        advance(n, cnt)
        exchange()
        n += cnt
        since += cnt
        if since >= poll_every or n >= grid.num_t:
            since = 0
            bad = poll()
            if bad >= 0:
                raise SolverError(f"non-finite electric field at step {bad}")


def run_slabs_local(solver, slabs_count: int, period=None):
    """Run ``solver``'s scenario as ``slabs_count`` slabs on one device (tests);
    ``period`` = steps between exchanges (default exchange_period)."""
    if solver._ran:
        raise SolverError("run() may only be called once per solver instance")
    solver._ran = True
    import torch

    k = tile_steps_of(solver)
    period = period or exchange_period(solver, k, slabs_count)
    slabs = partition(solver.grid.num_x, slabs_count, period)
    # one shared stream: every pack, unpack and launch runs in issue order
    stream = torch.cuda.Stream(device=f"cuda:{solver.gpu}")
    states = [SlabState(solver, s, stream=stream.cuda_stream) for s in slabs]
    try:
        tr = LocalTransport(states)
        for st in states:
            st.sample(0)

        def advance(n, cnt):
            for st in states:
                st.advance(n, cnt)

        def poll():
            bads = [b for b in (st.poll() for st in states) if b >= 0]
            return min(bads) if bads else -1

        _step_loop(solver.grid, period, advance, tr.exchange, poll)
        recs = assemble(solver.plan, slabs, [st.records() for st in states])
    finally:
        for st in states:
            st.close()
    solver.results = [p.to_result(solver.grid, d) for p, d in zip(solver.plan.plans, recs)]
    return solver.results


CHUNKS_PER_EXCHANGE = 32
# N-level / RK4 slabs: launches of k steps between exchanges (cfg5 per-rank
# rate flat from 4 to 32 launches per exchange, tools/slab_step.py, profiles/)
LAUNCHES_PER_EXCHANGE = 4


def exchange_period(solver, k: int, world: int) -> int:
    """Steps between halo exchanges (= ghost width): m fused chunks of k steps,
    at most the thinnest slab.  The two-level / classical kernels run the m
    chunks as one persistent launch; the N-level / RK4 kernels as m launches,
    each computing the window minus k cells per side (the valid region shrinks
    k cells per launch into the ghosts, as in the persistent kernel)."""
    dense = solver.plan.levels > 2 or (solver.plan.levels == 2 and solver.stepper == "rk4")
    period = (LAUNCHES_PER_EXCHANGE if dense else CHUNKS_PER_EXCHANGE) * k
    return max(1, min(period, solver.grid.num_x // max(1, world)))


def tile_steps_of(solver) -> int:
    """The k the native solver will use for this scenario (asks the library
    through a throw-away handle on a tiny window, so nothing big is allocated)."""
    w = min(solver.grid.num_x, 1024)
    h = native.Handle(solver._grid_struct(win=(0, w), own=(0, w)))
    try:
        k = C.c_int32(0)
        h.call("mbg_tile_steps", C.byref(k))
        return k.value
    finally:
        h.close()


def _reduce_scalar(value, op, device, dtype=None):
    """All-reduce one number: on the device under NCCL, on the host under gloo."""
    import torch
    import torch.distributed as dist

    dtype = torch.float64 if dtype is None else dtype
    where = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=dtype, device=where)
    dist.all_reduce(t, op=op)
    return t.item()


def slab_backend(local: int):
    """(backend, gpu) of a bench rank: NCCL on GPU ``local`` -- one process per
    GPU, the production shape.  ``MBG_SLAB_BACKEND=gloo MBG_SLAB_GPU=g`` puts
    every rank on GPU g with host-staged gloo exchanges instead: the whole
    multi-rank driver (partition, halo exchange, scan-flag reduction, record
    gather, timing) on a one-GPU box.  No kernel waits on another rank, since
    the ranks meet only on the host.  NCCL ranks sharing a GPU are refused."""
    import os

    backend = os.environ.get("MBG_SLAB_BACKEND", "nccl")
    if backend not in ("nccl", "gloo"):
        raise ValueError(f"MBG_SLAB_BACKEND must be nccl or gloo, not {backend!r}")
    shared = os.environ.get("MBG_SLAB_GPU")
    if shared is not None:
        if backend != "gloo":
            raise ValueError("MBG_SLAB_GPU (several ranks on one GPU) needs MBG_SLAB_BACKEND=gloo")
        local = int(shared)
    return backend, local


def run_slab_rank(solver, world: int, rank: int, device, state_factory=None, k=None, period=None):
    """This process's slab of a ``world``-way run (torch.distributed initialised).
    Returns the assembled records on rank 0 and None elsewhere.

    ``state_factory(solver, slab)`` replaces the native slab (tests drive the
    same host logic with a CPU slab stepper under gloo)."""
    import torch
    import torch.distributed as dist

    if k is None:
        k = tile_steps_of(solver)
    period = period or exchange_period(solver, k, world)
    slabs = partition(solver.grid.num_x, world, period)
    # the native launches, the pack/unpack kernels and torch's NCCL ops must
    # be ordered on one stream: a dedicated torch stream, made current, that
    # the native handle adopts (the legacy default stream cannot be adopted)
    stream = torch.cuda.Stream(device) if state_factory is None else None
    if state_factory is None:
        st = SlabState(solver, slabs[rank], stream=stream.cuda_stream)
    else:
        st = state_factory(solver, slabs[rank])
    try:
        with torch.cuda.stream(stream) if stream is not None else _nullcontext():
            tr = TorchTransport(st, device)
            st.sample(0)

            def poll():
                b = st.poll()
                v = int(_reduce_scalar(b if b >= 0 else 2**62, dist.ReduceOp.MIN, device, torch.int64))
                return -1 if v == 2**62 else v

            _step_loop(solver.grid, period, st.advance, tr.exchange, poll)
        mine = st.records()
    finally:
        st.close()
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    if rank != 0:
        return None
    return assemble(solver.plan, slabs, gathered)


def bench_rank(args, dev, sce, world, rank, local, metric, unit, clock_sampler=None, rebuild=None):
    """bench.py --gpus N under torchrun: weak-scaled cfg2, one slab per GPU,
    device time of K full runs, max over ranks.

    ``clock_sampler(gpu)``: context manager sampling clocks during the timed
    region (bench.py's ClockSampler); ``rebuild()``: fresh (device, scenario)
    for the end-to-end runs through run_slab_rank (the public multi-GPU call:
    window upload, exchanges, record download and gather), wall-clocked with
    barriers, max over ranks."""
    import json
    import os
    import time

    import torch
    import torch.distributed as dist

    from .solver import GpuFdtdSolver

    backend, local = slab_backend(local)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if not dist.is_initialized():
        dist.init_process_group(backend, device_id=device if backend == "nccl" else None)
    solver = GpuFdtdSolver(dev, sce, tile_steps=args.tile_steps, exact=args.exact, gpu=local)
    k = tile_steps_of(solver)
    period = exchange_period(solver, k, world)
    slabs = partition(solver.grid.num_x, world, period)
    # one stream for the native launches, the halo pack/unpack and NCCL (see run_slab_rank)
    stream = torch.cuda.Stream(device)
    st = SlabState(solver, slabs[rank], stream=stream.cuda_stream)
    ctx = torch.cuda.stream(stream)
    ctx.__enter__()
    tr = TorchTransport(st, device)
    st.h.call("mbg_checkpoint_save")
    grid = solver.grid

    def one_run():
        st.h.call("mbg_checkpoint_restore")
        st.sample(0)
        n = 1
        while n < grid.num_t:
            cnt = min(period, grid.num_t - n)
            st.advance(n, cnt)
            tr.exchange()
            n += cnt

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize(device)
    dist.barrier()
    l0 = C.c_int64(0)
    st.h.call("mbg_launch_count", C.byref(l0))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sampler = clock_sampler(local) if clock_sampler is not None else _nullcontext()
    with sampler:
        t0.record(stream)
        for _ in range(args.steps):
            one_run()
        t1.record(stream)
        torch.cuda.synchronize(device)
    dist.barrier()
    ms = _reduce_scalar(t0.elapsed_time(t1), dist.ReduceOp.MAX, device)
    l1 = C.c_int64(0)
    st.h.call("mbg_launch_count", C.byref(l1))
    bad = st.poll()
    st.close()
    ctx.__exit__(None, None, None)
    if bad >= 0:
        raise SolverError(f"non-finite electric field at step {bad}")
    ms = float(ms)
    cells = grid.num_x * (grid.num_t - 1) * args.steps

    e2e = None
    if rebuild is not None:
        walls = []
        for it in range(args.warmup + args.steps):
            d2, s2 = rebuild()
            sol = GpuFdtdSolver(d2, s2, tile_steps=args.tile_steps, exact=args.exact, gpu=local)
            torch.cuda.synchronize(device)
            dist.barrier()
            w0 = time.perf_counter()
            run_slab_rank(sol, world, rank, device)
            torch.cuda.synchronize(device)
            w = _reduce_scalar(time.perf_counter() - w0, dist.ReduceOp.MAX, device)
            if it >= args.warmup:
                walls.append(w)
        plan = solver.plan
        mine = slabs[rank]
        fields = 0 if plan.fields_zero else 2 * (mine.win_hi - mine.win_lo) + 1
        h2d = 8 * (fields + plan.state_words + plan.src_values.size)
        e2e = {"value": cells / sum(walls), "unit": unit, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(sum(p.rows * (mine.own_hi - mine.own_lo if p.cell is None else 1) *
                                             (16 if p.is_complex else 8) for p in plan.plans
                                             if p.cell is None or mine.own_lo <= p.cell < mine.own_hi)),
               "note": "rank 0's bytes; wall clock around run_slab_rank (window upload, exchanges, record "
                       "download + gather), max over ranks"}
    if rank == 0:
        launches = l1.value - l0.value
        line = {
            "metric": metric, "value": cells / (ms * 1e-3), "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"cfg2 weak-scaled: {world} copies of the cfg2 device, {world} slabs x 2^22 "
                                   f"cells, 20000 steps",
                       "num_x": grid.num_x, "tile_steps": k, "exchange_period": period,
                       "parallelism": f"slab{world}",
                       "exchange": f"NCCL batched isend/irecv of {period} ghost cells per interface every "
                                   f"{period} steps (one persistent launch of {period // k} chunks between)",
                       "l2": "inputs larger than L2 (~335 MB of state per GPU vs 126 MB L2)"},
            "e2e": e2e,
            # this rank's kernels (step, step-mask, sample, halo pack/unpack; library count)
            "gpu_launches": int(launches),
        }
        if backend != "nccl" or local != int(os.environ.get("LOCAL_RANK", local)):
            line["config"]["shared_gpu"] = (f"all {world} ranks on GPU {local}, {backend} exchanges staged "
                                            f"through the host: a functional run of the multi-rank path, "
                                            f"not a scaling measurement")
        if clock_sampler is not None:
            line["clocks"] = sampler.summary()
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
