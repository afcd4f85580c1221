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
  * :class:`PeerTransport` -- one process per GPU, no library collective on
    the data path: every rank owns a device mailbox per interface, exported
    through CUDA IPC; the neighbour's push kernel stores its edge cells
    straight into it (NVLink stores) and publishes a sequence flag, the
    owner's pull kernel acquires the flag and fills the ghosts
    (``mbg_push_halo`` / ``mbg_pull_halo``).  The default under NCCL.
"""

from __future__ import annotations

import ctypes as C
import sys
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

    def __init__(self, solver, slab: Slab, stream: int = 0, records: bool = True, stream_sources: bool = False):
        """``stream_sources``: the source samples (``Source.value`` per step, as
        the reference's loop calls it) are taken period by period while the
        device steps, as in ``GpuFdtdSolver.run`` -- for the one slab of a
        solver that steps alone (one rank per process, no edge strips)."""
        self.solver = solver
        self.slab = slab
        self.h = solver.open_handle(win=(slab.win_lo, slab.win_hi), own=(slab.own_lo, slab.own_hi),
                                    records=records, stream_sources=stream_sources)
        self.streaming = stream_sources and solver._fed < solver.grid.num_t
        if stream:
            self.h.call("mbg_set_stream", stream)
        solver.upload_initial_state(self.h, win=(slab.win_lo, slab.win_hi))
        w = C.c_int32(0)
        self.h.call("mbg_halo_words", C.byref(w))
        self.words = w.value  # per cell: E, H, state planes

    def sample(self, step):
        self.h.call("mbg_sample", step)

    def advance(self, first, count):
        if self.streaming:  # rows of this period, queued stream-ordered before its launch
            self.solver.plan.sample_sources(first + count)
            self.solver._feed_sources(self.h, first + count)
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


class EdgeStrips:
    """The cells a slab sends its neighbours, computed ahead of the slab itself
    so the halo exchange overlaps the slab's own advance.

    Per interface, the g cells a neighbour needs after one exchange period of
    P = g steps depend only on the 3g cells around them at the period's start
    (the dependency cone widens one cell per side per step).  A strip solver
    -- a second handle of the same solver with window [own_lo - g, own_lo + 2g)
    on the left (mirrored on the right), owned part the g sent cells, no
    records -- receives those 3g cells by a device copy, advances the period
    on a side stream and packs the g cells into the send buffer; the exchange
    then runs while the slab advances its whole window on the main stream.
    Every cell executes the same instruction sequence in the strip as in the
    slab, so the sent cells are bit-identical to the slab's own after the
    period, and the ghosts the slab unpacks are those of the serial path.

    Pays off for the N-level / RK4 kernels (launches of k steps that leave
    SM slots free between CTAs, short periods); the two-level persistent
    launch occupies every SM for its whole period, so its strips could not
    run beside it (and its 2048-step period already amortises the exchange).
    """

    def __init__(self, main: "SlabState", period: int, stream):
        import torch

        self.main, self.g, self.stream = main, period, stream
        sl = main.slab
        g = period
        if (sl.ghost_left or sl.ghost_right) and (sl.own_hi - sl.own_lo) < 2 * g:
            raise ValueError("edge strips need slabs of at least two exchange periods")
        self.sides = {}
        solver = main.solver
        for side in ("left", "right"):
            if side == "left" and sl.ghost_left:
                win, own = (sl.win_lo, sl.own_lo + 2 * g), (sl.own_lo, sl.own_lo + g)
            elif side == "right" and sl.ghost_right:
                win, own = (sl.own_hi - 2 * g, sl.win_hi), (sl.own_hi - g, sl.own_hi)
            else:
                continue
            h = solver.open_handle(win=win, own=own, records=False)
            h.call("mbg_set_stream", stream.cuda_stream)
            scratch = torch.empty(main.words * (win[1] - win[0]), dtype=torch.float64, device=stream.device)
            self.sides[side] = (h, win, own, scratch)
        # the strips' state is copied from the slab every period (opaque halo
        # words, already in the slab's storage frame): settle the handle's own
        # frame on an uploaded initial state first (mbg_sample without records
        # does only that), so no later call maps the copied words again
        for h, win, _, _ in self.sides.values():
            solver.upload_initial_state(h, win=win)
            h.call("mbg_sample", 0)

    def run(self, first: int, count: int, main_stream, send: dict):
        """Enqueue one period: copy the strips' 3g cells from the slab (main
        stream), then on the side stream advance them ``count`` steps and pack
        the sent cells into ``send[side]`` (device tensors) -- or, when
        ``send`` is a peer transport's sender, push them into the neighbour's
        mailbox (``send.push``)."""
        import torch

        for h, win, own, scratch in self.sides.values():
            self.main.pack(win[0], win[1] - win[0], scratch.data_ptr())
        ready = torch.cuda.Event()
        ready.record(main_stream)
        self.stream.wait_event(ready)
        for side, (h, win, own, scratch) in self.sides.items():
            h.call("mbg_unpack_halo", win[0], win[1] - win[0], scratch.data_ptr())
            h.call("mbg_advance", first, count)
            if hasattr(send, "push"):  # peer mailboxes: the strip stores into the neighbour's memory itself
                send.push(side, h, own[0], own[1] - own[0])
            else:
                h.call("mbg_pack_halo", own[0], own[1] - own[0], send[side].data_ptr())

    def close(self):
        for h, *_ in self.sides.values():
            h.close()
        self.sides = {}


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

    def exchange_from(self, sends):
        """Ghosts from the neighbours' edge-strip send buffers (``sends[i]``:
        side -> device tensor of slab i's strips)."""
        for i, st in enumerate(self.states):
            _, rl, _, rr = exchange_plan(st.slab)
            if rl is not None:
                st.unpack(rl[0], rl[1], sends[i - 1]["right"].data_ptr())
            if rr is not None:
                st.unpack(rr[0], rr[1], sends[i + 1]["left"].data_ptr())
        for st in self.states:
            st.h.call("mbg_synchronize")


class TorchTransport:
    """One slab per process; neighbours exchange with batched isend/irecv.

    ``exchange()`` = ``start()`` + ``finish()``: pack the slab's edge cells,
    send/receive, unpack the ghosts.  With edge strips (:class:`EdgeStrips`)
    the sent cells are packed by the strips on their side stream and
    ``start(packed=True)`` issues the transfer there; the slab's own advance
    is enqueued before ``finish()``, whose wait makes the main stream (not
    the host) wait for the transfer."""

    def __init__(self, state: SlabState, device, side_stream=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.state = state
        self.side_stream = side_stream
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
        self._reqs = []

    @property
    def send(self) -> dict:
        """Device send buffers by side (what EdgeStrips.run packs into)."""
        return {k: v for k, v in (("left", self.send_l), ("right", self.send_r)) if v is not None}

    def start(self, packed: bool = False):
        sl, rl, sr, rr = self.plan
        st, dist = self.state, self.dist
        rank = st.slab.rank
        if not packed:
            if sl is not None:
                st.pack_into(sl[0], sl[1], self.send_l)
            if sr is not None:
                st.pack_into(sr[0], sr[1], self.send_r)
        if self.stage:
            if packed and self.side_stream is not None:
                self.side_stream.synchronize()  # the strips packed on the side stream
            for d, h in ((self.send_l, self.h_send_l), (self.send_r, self.h_send_r)):
                if d is not None:
                    h.copy_(d)  # synchronous: the pack kernel has run
            send_l, recv_l, send_r, recv_r = self.h_send_l, self.h_recv_l, self.h_send_r, self.h_recv_r
        else:
            send_l, recv_l, send_r, recv_r = self.send_l, self.recv_l, self.send_r, self.recv_r
        ops = []
        if sl is not None:
            ops.append(dist.P2POp(dist.isend, send_l, rank - 1))
            ops.append(dist.P2POp(dist.irecv, recv_l, rank - 1))
        if sr is not None:
            ops.append(dist.P2POp(dist.isend, send_r, rank + 1))
            ops.append(dist.P2POp(dist.irecv, recv_r, rank + 1))
        if not ops:
            self._reqs = []
            return
        ctx = self.torch.cuda.stream(self.side_stream) if (packed and self.side_stream is not None
                                                          and not self.stage) else _nullcontext()
        with ctx:  # NCCL's stream waits for the stream current here
            self._reqs = dist.batch_isend_irecv(ops)

    def finish(self):
        sl, rl, sr, rr = self.plan
        st = self.state
        for req in self._reqs:
            req.wait()  # NCCL: the current (main) stream waits; gloo: the host waits
        self._reqs = []
        if self.stage:
            for d, h in ((self.recv_l, self.h_recv_l), (self.recv_r, self.h_recv_r)):
                if d is not None:
                    d.copy_(h)
        if rl is not None:
            st.unpack_from(rl[0], rl[1], self.recv_l)
        if rr is not None:
            st.unpack_from(rr[0], rr[1], self.recv_r)

    def exchange(self):
        self.start()
        self.finish()


class Mailbox:
    """Device memory a neighbour stores its ghost strips into (include/mbgpu.h,
    mbg_push_halo): a 128-byte header holding the two slot flags, then two
    slots of ``doubles`` doubles.  Owned (allocated here, exportable through
    CUDA IPC) or mapped from a neighbour's exported handle."""

    HEADER = 128

    def __init__(self, device: int, doubles: int, ipc: bytes | None = None):
        self.lib = native.load()
        self.device, self.doubles = int(device), int(doubles)
        ptr = C.c_uint64(0)
        self.owned = ipc is None
        if self.owned:
            buf = C.create_string_buffer(native.MBG_IPC_HANDLE_BYTES)
            rc = self.lib.mbg_mailbox_alloc(self.device, self.HEADER + 16 * self.doubles, C.byref(ptr), buf)
            self.ipc = buf.raw
        else:
            rc = self.lib.mbg_mailbox_map(self.device, ipc, C.byref(ptr))
            self.ipc = ipc
        if rc != 0:
            raise native.NativeError(f"peer mailbox {'allocation' if self.owned else 'mapping'} failed ({rc})")
        self.ptr = ptr.value

    def flag(self, slot: int) -> int:
        return self.ptr + 8 * slot

    def slot(self, slot: int) -> int:
        return self.ptr + self.HEADER + 8 * self.doubles * slot

    def close(self):
        if getattr(self, "ptr", 0):
            (self.lib.mbg_mailbox_free if self.owned else self.lib.mbg_mailbox_unmap)(self.device, self.ptr)
            self.ptr = 0


PULL_TIMEOUT_MS = 30000


def _pull_timeout() -> int:
    import os

    return int(os.environ.get("MBG_PULL_TIMEOUT_MS", PULL_TIMEOUT_MS))


class _PeerSender:
    """What EdgeStrips.run receives as ``send`` under a peer transport."""

    def __init__(self, push):
        self.push = push


class LocalPeerTransport:
    """All slabs in this process on one device, ghosts through peer mailboxes:
    the push / pull kernels and the slot and sequence protocol of
    :class:`PeerTransport` without a second process (every push is enqueued
    before the pull that waits for it, on one stream: no kernel ever waits)."""

    def __init__(self, states):
        self.states = states
        self.seq = 0
        dev = states[0].solver.gpu
        self.box = []  # per slab: side -> Mailbox it receives in
        for st in states:
            _, rl, _, rr = exchange_plan(st.slab)
            self.box.append({side: Mailbox(dev, st.words * spec[1])
                             for side, spec in (("left", rl), ("right", rr)) if spec is not None})

    def _push(self, i, side, handle, cell0, count):
        seq = self.seq + 1
        box = self.box[i - 1]["right"] if side == "left" else self.box[i + 1]["left"]
        handle.call("mbg_push_halo", cell0, count, box.slot(seq & 1), box.flag(seq & 1), seq)

    def sender(self, i):
        return _PeerSender(lambda side, handle, cell0, count: self._push(i, side, handle, cell0, count))

    def _pull_all(self):
        self.seq += 1
        for st, box in zip(self.states, self.box):
            _, rl, _, rr = exchange_plan(st.slab)
            for side, spec in (("left", rl), ("right", rr)):
                if spec is not None:
                    b = box[side]
                    st.h.call("mbg_pull_halo", spec[0], spec[1], b.slot(self.seq & 1), b.flag(self.seq & 1),
                              self.seq, _pull_timeout())
        for st in self.states:
            st.h.call("mbg_synchronize")

    def exchange(self):
        for i, st in enumerate(self.states):
            sl, _, sr, _ = exchange_plan(st.slab)
            if sl is not None:
                self._push(i, "left", st.h, sl[0], sl[1])
            if sr is not None:
                self._push(i, "right", st.h, sr[0], sr[1])
        self._pull_all()

    def exchange_from(self, sends):
        self._pull_all()  # the edge strips pushed through sender(i)

    def close(self):
        for box in self.box:
            for b in box.values():
                b.close()
        self.box = []


class PeerTransport:
    """One slab per process; ghost strips travel as stores into the
    neighbour's device memory, with no library collective on the data path.

    Setup (once): every rank allocates a :class:`Mailbox` per interface and the
    CUDA IPC handles go round with one ``all_gather_object``; each rank maps
    its neighbours' boxes (peer access over NVLink on a multi-GPU box, plain
    device memory when ranks share a GPU).  Per period: ``mbg_push_halo``
    stores the edge cells into the neighbour's slot ``seq & 1`` and publishes
    ``seq`` in its flag; ``mbg_pull_halo`` waits on the device for the flag and
    copies the slot into the ghosts.  Two slots need no acknowledgement (see
    include/mbgpu.h).  The host never waits inside the step loop.

    ``host_ordered`` (ranks sharing one GPU, tests and the one-GPU bench):
    every rank drains its device and meets the others on the host before the
    pulls are enqueued, so no kernel of one rank ever waits on a kernel of
    another rank on the same GPU."""

    def __init__(self, state: SlabState, device, side_stream=None, host_ordered: bool = False):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.state, self.side_stream, self.host_ordered = state, side_stream, host_ordered
        self.device = torch.device(device)
        self.plan = exchange_plan(state.slab)
        sl, rl, sr, rr = self.plan
        self.cuda = self.device.type == "cuda"  # (tests drive the protocol with host mailboxes on CPU)
        idx = self.device.index if self.device.index is not None else (torch.cuda.current_device() if self.cuda else 0)
        w = state.words
        self.box, self.peer = {}, {}
        try:  # a rank that cannot allocate still takes part in the gather (no rank may skip a collective)
            self.box = {side: Mailbox(idx, w * spec[1]) for side, spec in (("left", rl), ("right", rr))
                        if spec is not None}
            mine = {side: (b.ipc, b.doubles) for side, b in self.box.items()}
        except native.NativeError:
            mine = None
        every = [None] * dist.get_world_size()
        dist.all_gather_object(every, mine)
        if any(e is None for e in every):  # the same verdict on every rank
            self.close(abort=True)
            raise native.NativeError("a rank could not allocate its peer mailboxes")
        rank = state.slab.rank
        try:
            if sl is not None:  # what I send left lands in the left neighbour's right box
                ipc, doubles = every[rank - 1]["right"]
                self.peer["left"] = Mailbox(idx, doubles, ipc=ipc)
            if sr is not None:
                ipc, doubles = every[rank + 1]["left"]
                self.peer["right"] = Mailbox(idx, doubles, ipc=ipc)
        except native.NativeError:  # no IPC / peer access to that device: make_transport falls back on every rank
            self.close(abort=True)
            raise
        self.seq = 0

    @property
    def send(self):
        return _PeerSender(self.push)

    def push(self, side, handle, cell0, count):
        seq = self.seq + 1
        box = self.peer[side]
        handle.call("mbg_push_halo", cell0, count, box.slot(seq & 1), box.flag(seq & 1), seq)

    def start(self, packed: bool = False):
        sl, _, sr, _ = self.plan
        if not packed:
            if sl is not None:
                self.push("left", self.state.h, sl[0], sl[1])
            if sr is not None:
                self.push("right", self.state.h, sr[0], sr[1])
        self.seq += 1

    def finish(self):
        _, rl, _, rr = self.plan
        if self.host_ordered:
            if self.cuda:
                self.torch.cuda.synchronize(self.device)  # this rank's pushes have landed ...
            self.dist.barrier()                           # ... and so have everyone else's
        for side, spec in (("left", rl), ("right", rr)):
            if spec is not None:
                b = self.box[side]
                self.state.h.call("mbg_pull_halo", spec[0], spec[1], b.slot(self.seq & 1), b.flag(self.seq & 1),
                                  self.seq, _pull_timeout())

    def exchange(self):
        self.start()
        self.finish()

    def close(self, abort: bool = False):
        """Unmap the neighbours' boxes, then -- once every rank has -- free this
        rank's own.  ``abort`` (an exception is propagating, or the ranks did
        not all get their transport): no barrier, the run is over anyway."""
        if self.cuda:
            self.torch.cuda.synchronize(self.device)
        for b in self.peer.values():
            b.close()
        self.peer = {}
        if not abort:
            self.dist.barrier()  # nobody still maps a box when its owner frees it
        for b in self.box.values():
            b.close()
        self.box = {}


def exchange_mode(backend: str) -> str:
    """``MBG_SLAB_EXCHANGE`` = ``p2p`` (peer mailboxes) or ``nccl`` (batched
    isend/irecv; under gloo the host-staged send/recv).  Default: p2p under
    NCCL, send/recv under gloo."""
    import os

    mode = os.environ.get("MBG_SLAB_EXCHANGE", "p2p" if backend == "nccl" else "nccl")
    if mode not in ("p2p", "nccl"):
        raise ValueError(f"MBG_SLAB_EXCHANGE must be p2p or nccl, not {mode!r}")
    return mode


def make_transport(state: SlabState, device, side_stream=None):
    """The rank's ghost transport (torch.distributed initialised): peer
    mailboxes when asked for / by default under NCCL -- if every rank could
    set them up (CUDA IPC between the GPUs), else the send/recv transport."""
    import warnings

    import torch
    import torch.distributed as dist

    backend = dist.get_backend()
    if torch.device(device).type == "cuda" and dist.get_world_size() > 1 and exchange_mode(backend) == "p2p":
        tr, err = None, None
        try:
            tr = PeerTransport(state, device, side_stream=side_stream, host_ordered=(backend != "nccl"))
        except Exception as exc:  # IPC unavailable between these devices: every rank must agree
            err = exc
        ok = int(_reduce_scalar(0 if tr is None else 1, dist.ReduceOp.MIN, device, torch.int64))
        if ok:
            return tr
        if tr is not None:
            tr.close(abort=True)  # some rank has no transport: it would never reach a barrier
        warnings.warn(f"peer mailboxes unavailable ({err}); ghost exchange by send/recv")
    return TorchTransport(state, device, side_stream=side_stream)


# ---------------------------------------------------------------- drivers --

def _step_loop(grid, period, step_period, poll, poll_every=1 << 14):
    """Steps 1..num_t-1 in exchange periods: ``step_period(n, cnt)`` advances
    steps n..n+cnt-1 and refreshes the ghosts; the non-finite flag is polled
    every ``poll_every`` steps and at the end."""
    n = 1
    since = 0
    while n < grid.num_t:
        cnt = min(period, grid.num_t - n)
        step_period(n, cnt)
        n += cnt
        since += cnt
        if since >= poll_every or n >= grid.num_t:
            since = 0
            bad = poll()
            if bad >= 0:
                raise SolverError(f"non-finite electric field at step {bad}")


def _check_monitor(solver):
    if solver.monitor_invariants:
        raise NotImplementedError("the slab drivers do not run the invariant monitor; "
                                  "use GpuFdtdSolver.run() for a monitored run")


def run_slabs_local(solver, slabs_count: int, period=None, overlap: bool = False, exchange: str = "copy"):
    """Run ``solver``'s scenario as ``slabs_count`` slabs on one device (tests);
    ``period`` = steps between exchanges (default exchange_period);
    ``overlap``: the sent cells come from edge strips (EdgeStrips) on a side
    stream instead of the slabs themselves; ``exchange``: ``"copy"`` (pack /
    unpack through one scratch buffer) or ``"p2p"`` (peer mailboxes,
    :class:`LocalPeerTransport`)."""
    if solver._ran:
        raise SolverError("run() may only be called once per solver instance")
    _check_monitor(solver)
    solver._ran = True
    import torch

    k = tile_steps_of(solver)
    period = period or exchange_period(solver, k, slabs_count)
    slabs = partition(solver.grid.num_x, slabs_count, period)
    # one shared stream: every pack, unpack and launch runs in issue order
    device = torch.device("cuda", solver.gpu)
    stream = torch.cuda.Stream(device=device)
    states = [SlabState(solver, s, stream=stream.cuda_stream) for s in slabs]
    strips, sends = [], []
    try:
        tr = LocalPeerTransport(states) if exchange == "p2p" else LocalTransport(states)
        if overlap:
            side = torch.cuda.Stream(device=device, priority=-1)
            strips = [EdgeStrips(st, period, side) for st in states]
            if exchange == "p2p":
                sends = [tr.sender(i) for i in range(len(states))]
            else:
                sends = [{k2: torch.empty(st.words * period, dtype=torch.float64, device=device)
                          for k2 in sp.sides} for st, sp in zip(states, strips)]
        for st in states:
            st.sample(0)

        def step_period(n, cnt):
            if overlap:
                for sp, snd in zip(strips, sends):
                    sp.run(n, cnt, stream, snd)
            for st in states:
                st.advance(n, cnt)
            if overlap:
                done = torch.cuda.Event()
                done.record(side)
                stream.wait_event(done)
                tr.exchange_from(sends)
            else:
                tr.exchange()

        def poll():
            bads = [b for b in (st.poll() for st in states) if b >= 0]
            return min(bads) if bads else -1

        _step_loop(solver.grid, period, step_period, poll)
        recs = assemble(solver.plan, slabs, [st.records() for st in states])
    finally:
        for sp in strips:
            sp.close()
        for st in states:
            st.close()
        if exchange == "p2p" and "tr" in locals():
            tr.close()
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
    g = solver._grid_struct(win=(0, w), own=(0, w))
    g.flags |= native.MBG_FLAG_DEFAULT_DEPTH  # a slab's depth (slabs are windows: no small-domain deepening)
    h = native.Handle(g)
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


def overlaps_by_default(solver, backend: str) -> bool:
    """Edge strips for the N-level / RK4 kernels under NCCL (see EdgeStrips)."""
    dense = solver.plan.levels > 2 or (solver.plan.levels == 2 and solver.stepper == "rk4")
    return dense and backend == "nccl"


def run_slab_rank(solver, world: int, rank: int, device, state_factory=None, k=None, period=None, overlap=None,
                  transport=None):
    """This process's slab of a ``world``-way run (torch.distributed initialised).
    Returns the assembled records on rank 0 and None elsewhere.

    ``state_factory(solver, slab)`` replaces the native slab (tests drive the
    same host logic with a CPU slab stepper under gloo).  ``overlap``: send
    the edge strips' cells while the slab advances (default: N-level / RK4
    under NCCL, see :func:`overlaps_by_default`).  ``transport(state, device,
    side_stream)`` replaces :func:`make_transport` (tests)."""
    import torch
    import torch.distributed as dist

    _check_monitor(solver)
    if k is None:
        k = tile_steps_of(solver)
    period = period or exchange_period(solver, k, world)
    slabs = partition(solver.grid.num_x, world, period)
    if overlap is None:
        overlap = state_factory is None and overlaps_by_default(solver, dist.get_backend())
    if overlap and state_factory is not None:
        raise ValueError("edge strips need native slabs")
    # the native launches, the pack/unpack kernels and torch's NCCL ops must
    # be ordered on one stream: a dedicated torch stream, made current, that
    # the native handle adopts (the legacy default stream cannot be adopted)
    stream = torch.cuda.Stream(device) if state_factory is None else None
    side = torch.cuda.Stream(device, priority=-1) if overlap else None
    if state_factory is None:
        st = SlabState(solver, slabs[rank], stream=stream.cuda_stream, stream_sources=not overlap)
    else:
        st = state_factory(solver, slabs[rank])
    strips = None
    try:
        with torch.cuda.stream(stream) if stream is not None else _nullcontext():
            tr = (transport or make_transport)(st, device, side_stream=side)
            if overlap:
                strips = EdgeStrips(st, period, side)
            st.sample(0)

            def step_period(n, cnt):
                if strips is not None:
                    strips.run(n, cnt, stream, tr.send)
                    tr.start(packed=True)
                    st.advance(n, cnt)
                    tr.finish()
                else:
                    st.advance(n, cnt)
                    tr.exchange()

            def poll():
                b = st.poll()
                v = int(_reduce_scalar(b if b >= 0 else 2**62, dist.ReduceOp.MIN, device, torch.int64))
                return -1 if v == 2**62 else v

            _step_loop(solver.grid, period, step_period, poll)
        mine = st.records()
    finally:
        if strips is not None:
            strips.close()
        if hasattr(locals().get("tr"), "close"):
            tr.close(abort=sys.exc_info()[0] is not None)
        st.close()
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    if rank != 0:
        return None
    return assemble(solver.plan, slabs, gathered)


class SlabTimer:
    """Bounded, repeatable slab runs for the benchmark: this rank's slab (and
    edge strips) stay resident, every run restores the initial state from a
    device checkpoint and advances ``steps`` steps with an exchange every
    period.  ``time(reps)`` returns device milliseconds of ``reps`` runs
    (CUDA events on the launch stream), max over ranks.  World size 1 is a
    single slab without ghosts (no transport): the single-domain run."""

    def __init__(self, solver, world: int, rank: int, device, steps: int, period=None, k=None,
                 overlap: bool = False):
        import torch

        self.torch = torch
        self.world, self.rank, self.device = world, rank, device
        self.k = tile_steps_of(solver) if k is None else k
        self.period = period or (exchange_period(solver, self.k, world) if world > 1 else max(1, steps))
        self.steps = steps
        self.slabs = partition(solver.grid.num_x, world, self.period if world > 1 else 0)
        self.stream = torch.cuda.Stream(device)
        self.side = torch.cuda.Stream(device, priority=-1) if overlap else None
        self.st = SlabState(solver, self.slabs[rank], stream=self.stream.cuda_stream)
        self.tr = None
        self.strips = None
        with torch.cuda.stream(self.stream):
            if world > 1:
                self.tr = make_transport(self.st, device, side_stream=self.side)
                if overlap:
                    self.strips = EdgeStrips(self.st, self.period, self.side)
        self.st.h.call("mbg_checkpoint_save")
        self.grid = solver.grid

    def _period(self, n, cnt):
        st, tr = self.st, self.tr
        if tr is None:
            st.advance(n, cnt)
        elif self.strips is not None:
            self.strips.run(n, cnt, self.stream, tr.send)
            tr.start(packed=True)
            st.advance(n, cnt)
            tr.finish()
        else:
            st.advance(n, cnt)
            tr.exchange()

    def one_run(self):
        self.st.h.call("mbg_checkpoint_restore")
        self.st.sample(0)
        n = 1
        end = 1 + self.steps
        while n < end:
            cnt = min(self.period, end - n)
            self._period(n, cnt)
            n += cnt

    def launches(self) -> int:
        v = C.c_int64(0)
        self.st.h.call("mbg_launch_count", C.byref(v))
        return int(v.value)

    def time(self, reps: int, warmup: int = 1, sampler=None) -> float:
        torch = self.torch
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                self.one_run()
            torch.cuda.synchronize(self.device)
            self._barrier()
            l0 = self.launches()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            with sampler if sampler is not None else _nullcontext():
                t0.record(self.stream)
                for _ in range(reps):
                    self.one_run()
                t1.record(self.stream)
                torch.cuda.synchronize(self.device)
            self._barrier()
        self.timed_launches = self.launches() - l0
        ms = t0.elapsed_time(t1)
        if self.world > 1:
            import torch.distributed as dist

            ms = _reduce_scalar(ms, dist.ReduceOp.MAX, self.device)
        bad = self.st.poll()
        if bad >= 0:
            raise SolverError(f"non-finite electric field at step {bad}")
        return float(ms)

    def _barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def close(self):
        if self.strips is not None:
            self.strips.close()
        if hasattr(self.tr, "close"):
            self.tr.close()
        self.st.close()


def bench_rank(args, dev, sce, world, rank, local, metric, unit, clock_sampler=None, rebuild=None,
               samples=None, config=None):
    """bench.py --gpus N under torchrun: weak-scaled cfg2, one slab per GPU,
    device time of K full runs, max over ranks.

    ``clock_sampler(gpu)``: context manager sampling clocks during the timed
    region (bench.py's ClockSampler); ``rebuild()``: fresh (device, scenario)
    for the end-to-end runs through run_slab_rank (the public multi-GPU call:
    plan build, window upload, exchanges, record download and gather),
    wall-clocked with barriers, max over ranks; ``samples(world, rank,
    device)``: extra bounded multi-GPU workloads (bench.py: cfg4 strong
    scaling, cfg5 exchange-period sweep), reported under ``scaling_samples``."""
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
    grid = solver.grid
    timer = SlabTimer(solver, world, rank, device, steps=grid.num_t - 1)
    k, period, slabs = timer.k, timer.period, timer.slabs
    sampler = clock_sampler(local) if clock_sampler is not None else None
    ms = timer.time(args.steps, warmup=args.warmup, sampler=sampler)
    launches = timer.timed_launches
    peer = isinstance(timer.tr, PeerTransport)
    timer.close()
    cells = grid.num_x * (grid.num_t - 1) * args.steps

    e2e = None
    if rebuild is not None:
        walls = []
        for it in range(args.warmup + args.steps):
            torch.cuda.synchronize(device)
            dist.barrier()
            w0 = time.perf_counter()
            d2, s2 = rebuild()
            sol = GpuFdtdSolver(d2, s2, tile_steps=args.tile_steps, exact=args.exact, gpu=local)
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
               "note": "rank 0's bytes; wall clock around the public multi-GPU call (plan build with the "
                       "sources sampled by Source.value, window upload, exchanges, record download + "
                       "gather), max over ranks"}
    extra = samples(world, rank, device) if samples is not None else None
    if rank == 0:
        line = {
            "metric": metric, "value": cells / (ms * 1e-3), "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            # the workload (bench.py's, identical for the reference arm) and
            # the implementation knobs separately
            "config": dict(config) if config is not None else
                      {"workload": f"cfg2 weak-scaled: {world} copies of the cfg2 device, {world} slabs x 2^22 "
                                   f"cells, 20000 steps", "num_x": grid.num_x, "parallelism": f"slab{world}"},
            "implementation": {
                "tile_steps": k, "exchange_period": period,
                "exchange": (f"peer mailboxes (mbg_push_halo stores into the neighbour's device memory, "
                             f"mbg_pull_halo acquires the flag)" if peer else f"{backend} batched isend/irecv")
                            + f" of {period} ghost cells per interface every {period} steps (one persistent "
                              f"launch of {period // k} chunks between)"},
            "e2e": e2e,
            # this rank's kernels (step, step-mask, sample, halo pack/unpack; library count)
            "gpu_launches": int(launches),
            "scaling_samples": extra,
        }
        if backend != "nccl" or local != int(os.environ.get("LOCAL_RANK", local)):
            line["shared_gpu"] = (f"all {world} ranks on GPU {local}, {backend} exchanges staged "
                                            f"through the host: a functional run of the multi-rank path, "
                                            f"not a scaling measurement")
        if sampler is not None:
            line["clocks"] = sampler.summary()
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
