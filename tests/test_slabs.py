"""Slab decomposition: host logic on CPU (gloo, world size 2 and 3) and the
native windowed path on one GPU (all slabs in one process).

The multi-rank runs must be bit-identical to the single-domain CPU oracle:
every cell runs the same operation sequence whichever slab holds it.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp
from conftest import ROOT, build_case

import paper_2005_05412_b200 as gpu

from paper_2005_05412_b200.reference import mblight as mb
from paper_2005_05412_b200 import slabs


def test_partition_follows_reference_rule_and_ghosts():
    s = slabs.partition(1000, 3, 7)
    bounds = np.linspace(0, 1000, 4).astype(int)
    assert [(x.own_lo, x.own_hi) for x in s] == list(zip(bounds[:-1], bounds[1:]))
    assert (s[0].win_lo, s[0].win_hi) == (0, s[0].own_hi + 7)
    assert (s[2].win_lo, s[2].win_hi) == (s[2].own_lo - 7, 1000)
    assert s[1].ghost_left == s[1].ghost_right == 7


def test_exchange_plans_pair_up():
    parts = slabs.partition(500, 4, 5)
    for a, b in zip(parts, parts[1:]):
        _, _, send_r, recv_r = slabs.exchange_plan(a)
        send_l, recv_l, _, _ = slabs.exchange_plan(b)
        # what a sends right lands in b's left ghost, and vice versa
        assert send_r == recv_l and send_l == recv_r
        assert recv_l[0] == b.win_lo and recv_l[0] + recv_l[1] == b.own_lo


def test_partition_rejects_thin_slabs():
    with pytest.raises(ValueError):
        slabs.partition(20, 4, 8)


def test_exchange_mode_defaults_and_switch(monkeypatch):
    monkeypatch.delenv("MBG_SLAB_EXCHANGE", raising=False)
    assert slabs.exchange_mode("nccl") == "p2p" and slabs.exchange_mode("gloo") == "nccl"
    monkeypatch.setenv("MBG_SLAB_EXCHANGE", "nccl")
    assert slabs.exchange_mode("nccl") == "nccl"
    monkeypatch.setenv("MBG_SLAB_EXCHANGE", "shmem")
    with pytest.raises(ValueError):
        slabs.exchange_mode("nccl")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, k, period, out_path):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist
    from np_slab import NumpySlab

    import paper_2005_05412_b200 as gpu

    from paper_2005_05412_b200.reference import mblight as mbw
    from paper_2005_05412_b200 import slabs as sl

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import CASES

        build, stepper = CASES[case]
        mbw.clear_material_library()
        dev, sce = build(mbw)
        solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
        recs = sl.run_slab_rank(solver, world, rank, "cpu", state_factory=NumpySlab, k=k, period=period)
        if rank == 0:
            np.savez(out_path, *recs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,period,case", [(2, 7, None, "sit_hard_whole"), (3, 16, 16, "multi_material"),
                                                 (2, 5, None, "vacuum_sources"), (2, 3, 7, "sit_hard_whole"),
                                                 # N-level splitting and RK4 ranks (the density step of the
                                                 # twin is the oracle's own, on each window's quantum runs)
                                                 (2, 4, 12, "rand3_split"), (3, 4, 8, "rand6_split"),
                                                 (2, 4, 9, "rand4_rk4"), (2, 6, None, "rand2_rk4")])
def test_gloo_ranks_match_oracle_bitwise(world, k, period, case):
    """period: steps between exchanges (ghost width); None = m chunks of k."""
    import oracle as orc

    dev, sce, stepper = build_case(case)
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    ref, bad = orc.run_oracle(plan)
    assert bad == 0
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "recs.npz")
        mp.spawn(_worker, args=(world, _free_port(), case, k, period, out), nprocs=world, join=True)
        got = np.load(out)
        for r, (p, want) in enumerate(zip(plan.plans, ref)):
            have = got[f"arr_{r}"]
            assert have.shape == want.shape, p.record.name
            assert np.array_equal(have, want), (p.record.name, np.max(np.abs(have - want)))


def _peer_worker(rank, world, port, case, k, period, out_path, box_dir):
    """One gloo rank driving slabs.PeerTransport itself (handle exchange, which
    box a side's push lands in, slot and sequence numbers, close order) with
    host stand-ins for the device pieces: mailboxes are files mapped by both
    neighbours, the push / pull 'kernels' are numpy copies with the flag
    protocol of halo_push_kernel / halo_pull_kernel."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import time

    import torch
    import torch.distributed as dist
    from np_slab import NumpySlab

    import paper_2005_05412_b200 as gpu

    from paper_2005_05412_b200.reference import mblight as mbw
    from paper_2005_05412_b200 import slabs as sl

    class FileMailbox:
        HEADER = 128
        count = 0

        def __init__(self, device, doubles, ipc=None):
            self.doubles, self.owned = int(doubles), ipc is None
            if self.owned:
                FileMailbox.count += 1
                path = os.path.join(box_dir, f"box_{rank}_{FileMailbox.count}.bin")
                np.zeros(self.HEADER // 8 + 2 * self.doubles).tofile(path)
                self.ipc = path.encode()
            else:
                self.ipc = ipc
            self.mem = np.memmap(self.ipc.decode(), dtype=np.float64, mode="r+")

        def flag(self, slot):
            return (self.mem, slot)  # flag words at the head of the box

        def slot(self, slot):
            o = self.HEADER // 8 + slot * self.doubles
            return (self.mem, o)

        def close(self):
            self.mem.flush()

    class Handle:
        def __init__(self, slab):
            self.slab, self.calls = slab, []

        def call(self, name, cell0, count, slot, flag, seq, timeout_ms=None):
            self.calls.append((name, cell0, count, slot[1], flag[1], seq))
            mem, o = slot
            fmem, fo = flag
            n = self.slab.words * count
            if name == "mbg_push_halo":
                mem[o:o + n] = self.slab._pack(cell0, count)
                mem.flush()
                fmem.view(np.uint64)[fo] = seq  # published after the data
                fmem.flush()
            else:
                assert name == "mbg_pull_halo"
                t0 = time.time()
                while fmem.view(np.uint64)[fo] < seq:
                    assert time.time() - t0 < timeout_ms / 1e3, "strip did not arrive"
                    time.sleep(0.0005)
                self.slab.unpack_from(cell0, count, torch.from_numpy(np.array(mem[o:o + n])))

    class PeerSlab:  # the twin behind the attributes PeerTransport uses (state.h is the native handle there)
        def __init__(self, solver, slab):
            self.twin = NumpySlab(solver, slab)
            self.slab, self.words = slab, self.twin.words
            self.h = Handle(self.twin)

        def __getattr__(self, name):
            return getattr(self.twin, name)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import CASES

        sl.Mailbox = FileMailbox
        build, stepper = CASES[case]
        mbw.clear_material_library()
        dev, sce = build(mbw)
        solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
        made = []

        def transport(state, device, side_stream=None):
            made.append(sl.PeerTransport(state, device, side_stream=side_stream))
            return made[0]

        recs = sl.run_slab_rank(solver, world, rank, "cpu", state_factory=PeerSlab, k=k, period=period,
                                transport=transport)
        tr = made[0]
        calls = tr.state.h.calls
        # every exchange: pushes first (both sides), then the pulls, same sequence number, slot = seq & 1
        per = (2 if 0 < rank < world - 1 else 1) * 2
        assert len(calls) == tr.seq * per and tr.seq > 2
        for e in range(tr.seq):
            chunk = calls[e * per:(e + 1) * per]
            assert [c[0] for c in chunk] == ["mbg_push_halo"] * (per // 2) + ["mbg_pull_halo"] * (per // 2)
            assert all(c[5] == e + 1 and c[4] == (e + 1) & 1 for c in chunk)
        if rank == 0:
            np.savez(out_path, *recs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,period,case", [(3, 16, 16, "multi_material"), (2, 4, 12, "rand3_split")])
def test_peer_transport_protocol_between_gloo_ranks(world, k, period, case):
    """slabs.PeerTransport across processes on CPU: its own host logic with
    file-backed mailboxes and numpy push / pull, bit-identical to the oracle."""
    import oracle as orc

    dev, sce, stepper = build_case(case)
    plan = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).plan
    ref, bad = orc.run_oracle(plan)
    assert bad == 0
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "recs.npz")
        mp.spawn(_peer_worker, args=(world, _free_port(), case, k, period, out, d), nprocs=world, join=True)
        got = np.load(out)
        for r, (p, want) in enumerate(zip(plan.plans, ref)):
            have = got[f"arr_{r}"]
            assert have.shape == want.shape, p.record.name
            assert np.array_equal(have, want), (p.record.name, np.max(np.abs(have - want)))


@pytest.mark.gpu
@pytest.mark.parametrize("case,count,period", [("sit_hard_whole", 2, None), ("sit_hard_whole", 5, None),
                                               ("multi_material", 3, None), ("multi_material", 2, 64),
                                               ("cfg2_r16", 3, None), ("vacuum_sources", 2, 100),
                                               ("rand3_split", 2, None), ("rand6_split", 3, None),
                                               ("rand4_rk4", 2, None), ("cfg4_r14", 4, None),
                                               # N-level periods that are not one launch: 3 launches of k = 4,
                                               # and a period that is not a multiple of k
                                               ("rand6_split", 2, 12), ("cfg4_r14", 3, 10), ("rand3_split", 3, 29),
                                               # eight slabs, as on a full B200 box
                                               ("cfg2_r16", 8, None), ("cfg4_r14", 8, None)])
def test_native_slabs_on_one_gpu_match_single_domain(case, count, period):
    """Windowed solvers (persistent multi-chunk launches between exchanges for
    the two-level / classical kernels) bit-identical to the single domain."""
    dev, sce, stepper = build_case(case)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    mb.clear_material_library()
    dev, sce, stepper = build_case(case)
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    got = slabs.run_slabs_local(solver, count, period)
    for a, b in zip(ref, got):
        assert a.name == b.name and a.data.shape == b.data.shape
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


@pytest.mark.gpu
@pytest.mark.parametrize("case,count,period", [("rand6_split", 3, None), ("rand3_split", 2, 29), ("cfg4_r14", 4, None),
                                               ("rand4_rk4", 2, None), ("four_media", 3, 24)])
def test_edge_strips_match_single_domain(case, count, period):
    """Exchange overlapped with the slab's advance (EdgeStrips: the sent cells
    computed ahead by strip solvers on a side stream, the default under NCCL
    for N-level / RK4 slabs): bit-identical to the single domain."""
    dev, sce, stepper = build_case(case)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    mb.clear_material_library()
    dev, sce, stepper = build_case(case)
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    got = slabs.run_slabs_local(solver, count, period, overlap=True)
    for a, b in zip(ref, got):
        assert a.name == b.name and a.data.shape == b.data.shape
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


@pytest.mark.gpu
@pytest.mark.parametrize("case,count,period,overlap", [("cfg2_r16", 3, None, False), ("multi_material", 2, 64, False),
                                                       ("cfg4_r14", 4, None, False), ("rand3_split", 3, 29, False),
                                                       ("rand6_split", 3, None, True), ("rand4_rk4", 2, None, True),
                                                       ("cfg2_r16", 8, None, False)])
def test_peer_mailboxes_in_one_process_match_single_domain(case, count, period, overlap):
    """The peer-memory exchange (mbg_push_halo / mbg_pull_halo: slots, sequence
    flags, two-slot reuse) between slabs of one process, with and without edge
    strips pushing from their side stream: bit-identical to the single domain."""
    dev, sce, stepper = build_case(case)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    mb.clear_material_library()
    dev, sce, stepper = build_case(case)
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    got = slabs.run_slabs_local(solver, count, period, overlap=overlap, exchange="p2p")
    for a, b in zip(ref, got):
        assert a.name == b.name and a.data.shape == b.data.shape
        assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), a.name


@pytest.mark.gpu
def test_pull_without_a_push_times_out_and_is_reported():
    """A strip that never arrives: the pull kernel gives up after its timeout,
    leaves the ghosts alone and the next synchronisation raises."""
    import ctypes as C

    from paper_2005_05412_b200 import native

    dev, sce, stepper = build_case("multi_material")
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    slab = slabs.partition(solver.grid.num_x, 2, 64)[1]
    st = slabs.SlabState(solver, slab)
    box = slabs.Mailbox(solver.gpu, st.words * slab.ghost_left)
    try:
        st.h.call("mbg_pull_halo", slab.win_lo, slab.ghost_left, box.slot(1), box.flag(1), 1, 50)
        with pytest.raises(native.NativeError, match="did not arrive"):
            st.h.call("mbg_synchronize")
        st.h.call("mbg_synchronize")  # reported once, then cleared
        # a push with the awaited sequence number makes the same pull succeed
        st.h.call("mbg_push_halo", slab.own_lo, slab.ghost_left, box.slot(1), box.flag(1), 1)
        st.h.call("mbg_pull_halo", slab.win_lo, slab.ghost_left, box.slot(1), box.flag(1), 1, 50)
        st.h.call("mbg_synchronize")
    finally:
        st.close()
        box.close()


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [4, 5])
def test_occupancy_and_latency_instantiations_agree_bitwise(dim):
    """Four- and five-level splitting has two instantiations (three CTAs per SM
    from 888 tiles per launch on, the spill-free build below): a 2^17-cell
    single domain (1093 tiles) against the same run as two slabs (547 tiles
    each) and their edge strips (one tile): identical bits."""
    from cases import random_case

    nx = 1 << 17
    dt = 0.5 * (20e-6 / nx) / 299792458.0
    build, stepper = random_case(dim, 30 + dim, nx=nx, end=40.5 * dt, whole=True)  # every step, whole domain
    mb.clear_material_library()
    dev, sce = build(mb)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    for overlap in (False, True):
        mb.clear_material_library()
        dev, sce = build(mb)
        got = slabs.run_slabs_local(gpu.GpuFdtdSolver(dev, sce, stepper=stepper), 2, overlap=overlap)
        for a, b in zip(ref, got):
            assert a.data.shape == b.data.shape
            assert np.array_equal(a.data.view(np.float64), b.data.view(np.float64)), (a.name, overlap)


def _nccl_single(fn):
    """Run fn() inside a one-rank NCCL process group (the only NCCL shape one GPU allows)."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        return fn()
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.gpu
def test_run_slab_rank_nccl_world_one_matches_single_domain():
    """The torch.distributed driver of the native slab path (stream hand-off,
    TorchTransport, MIN reduction of the scan flag, gather of records)."""
    import torch

    dev, sce, stepper = build_case("multi_material")
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    mb.clear_material_library()
    dev, sce, stepper = build_case("multi_material")
    solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper)
    recs = _nccl_single(lambda: slabs.run_slab_rank(solver, 1, 0, torch.device("cuda", 0)))
    for a, b in zip(ref, recs):
        assert np.array_equal(a.data, b), a.name


@pytest.mark.gpu
def test_bench_rank_prints_a_line(capsys, monkeypatch):
    """bench.py's multi-GPU code path on one rank (NCCL world size 1)."""
    import json
    import types

    from paper_2005_05412_b200 import configs

    args = types.SimpleNamespace(tile_steps=None, exact=False, steps=1, warmup=1)
    mb.clear_material_library()
    dev, sce = configs.cfg2(mb, nx=1 << 16, steps=512)
    # bench_rank initialises (and destroys) its own process group
    for key, val in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", str(_free_port())), ("RANK", "0"),
                     ("WORLD_SIZE", "1")):
        monkeypatch.setenv(key, val)
    slabs.bench_rank(args, dev, sce, 1, 0, 0, "m", "cell-updates/s",
                     rebuild=lambda: configs.cfg2(mb, nx=1 << 16, steps=512))
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0


def _gpu_worker(rank, world, port, case, period, out_path, overlap=None):
    """One rank of a gloo run whose slabs all live on cuda:0 (native kernels,
    host-staged exchanges: the ranks only meet on the host)."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist

    import paper_2005_05412_b200 as gpu

    from paper_2005_05412_b200.reference import mblight as mbw
    from paper_2005_05412_b200 import slabs as sl

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import CASES

        build, stepper = CASES[case]
        mbw.clear_material_library()
        dev, sce = build(mbw)
        torch.cuda.set_device(0)
        solver = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, gpu=0)
        recs = sl.run_slab_rank(solver, world, rank, torch.device("cuda", 0), period=period, overlap=overlap)
        if rank == 0:
            np.savez(out_path, *[r.data for r in recs])
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,case,period,overlap", [(2, "multi_material", None, None), (3, "cfg2_r16", None, None),
                                                       (2, "rand3_split", None, None),
                                                       (2, "vacuum_sources", 100, None),
                                                       # the NCCL default for N-level slabs, edge strips on a
                                                       # side stream, here through the host-staged transport
                                                       (2, "rand6_split", None, True), (3, "rand3_split", 29, True)])
def test_native_ranks_sharing_one_gpu_match_single_domain(world, case, period, overlap):
    """run_slab_rank across processes with the native slab kernels: the
    TorchTransport exchange plan, pack/unpack on the adopted stream, scan-flag
    reduction and record gather, bit-identical to the single-domain run."""
    dev, sce, stepper = build_case(case)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "recs.npz")
        mp.spawn(_gpu_worker, args=(world, _free_port(), case, period, out, overlap), nprocs=world, join=True)
        got = np.load(out)
        for r, a in enumerate(ref):
            have = got[f"arr_{r}"]
            assert have.shape == a.data.shape, a.name
            assert np.array_equal(have, a.data), (a.name, np.max(np.abs(have - a.data)))


@pytest.mark.gpu
@pytest.mark.parametrize("world,case,period,overlap", [(2, "multi_material", None, None), (3, "cfg2_r16", None, None),
                                                       (2, "rand6_split", None, True), (3, "rand3_split", 29, None)])
def test_peer_mailboxes_across_processes_match_single_domain(world, case, period, overlap, monkeypatch):
    """PeerTransport between processes: mailboxes exported through CUDA IPC,
    mapped by the neighbour rank, strips stored into them by the neighbour's
    push kernel.  The ranks share cuda:0 here, so the transport runs host
    ordered (no kernel of one rank waits on another rank's kernel)."""
    monkeypatch.setenv("MBG_SLAB_EXCHANGE", "p2p")
    dev, sce, stepper = build_case(case)
    ref = gpu.GpuFdtdSolver(dev, sce, stepper=stepper).run()
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "recs.npz")
        mp.spawn(_gpu_worker, args=(world, _free_port(), case, period, out, overlap), nprocs=world, join=True)
        got = np.load(out)
        for r, a in enumerate(ref):
            have = got[f"arr_{r}"]
            assert have.shape == a.data.shape, a.name
            assert np.array_equal(have, a.data), (a.name, np.max(np.abs(have - a.data)))


@pytest.mark.gpu
def test_bench_under_torchrun_two_ranks_on_one_gpu():
    """bench.py --gpus 2 exactly as the driver launches it (torchrun), both
    ranks on cuda:0 with gloo (MBG_SLAB_GPU): one JSON line from rank 0."""
    import json
    import subprocess

    env = dict(os.environ, MBG_SLAB_BACKEND="gloo", MBG_SLAB_GPU="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "1"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["num_x"] == 2 << 22 and "shared_gpu" in line
    assert line["config"]["parallelism"] == "slab2" and "tile_steps" in line["implementation"]
