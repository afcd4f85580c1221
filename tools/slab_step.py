"""Per-rank cost of the slab path on one GPU (what one rank of `bench.py
--gpus G` does, minus the NCCL transfer): the middle slab of a G-way
weak-scaled run, advanced period steps at a time with both halos packed and
unpacked (into a scratch buffer, self-looped) after every period.

    python tools/slab_step.py [--config cfg2|cfg5] [--world 3] [--period P] [--tile-steps K] [--steps S]

cfg2: G copies of the two-level cfg2 device (2^22 cells per rank).  cfg5:
BASELINE configs[4], the six-level cfg4 medium on 2^22 cells per rank; the
exchange period P (= ghost width) may exceed the tile depth k (P/k fused
launches between exchanges).
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs, slabs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2", choices=("cfg2", "cfg5"))
ap.add_argument("--tile-steps", type=int, default=None)
ap.add_argument("--world", type=int, default=3)
ap.add_argument("--period", type=int, default=0)
ap.add_argument("--steps", type=int, default=20000)
a = ap.parse_args()
if a.config == "cfg2":
    dev, sce = configs.cfg2(mb, nx=(1 << 22) * a.world, steps=a.steps, replicas=a.world)
else:
    dev, sce = configs.cfg5(mb, gpus=a.world, steps=a.steps)
solver = gpu.GpuFdtdSolver(dev, sce, tile_steps=a.tile_steps)
k = slabs.tile_steps_of(solver)
period = a.period or slabs.exchange_period(solver, k, a.world)
part = slabs.partition(solver.grid.num_x, a.world, period)
mid = part[a.world // 2]
stream = torch.cuda.Stream(0)
torch.cuda.set_stream(stream)
st = slabs.SlabState(solver, mid, stream=stream.cuda_stream)
buf = torch.empty(st.words * period, dtype=torch.float64, device="cuda:0")
st.h.call("mbg_checkpoint_save")


def run():
    st.h.call("mbg_checkpoint_restore")
    st.sample(0)
    n = 1
    while n < solver.grid.num_t:
        cnt = min(period, solver.grid.num_t - n)
        st.advance(n, cnt)
        for cell0, ghost in ((mid.own_lo, mid.own_lo - mid.win_lo), (mid.own_hi - period, mid.win_hi - mid.own_hi)):
            st.pack_into(cell0, ghost, buf)
        st.unpack_from(mid.win_lo, mid.own_lo - mid.win_lo, buf)
        st.unpack_from(mid.own_hi, mid.win_hi - mid.own_hi, buf)
        n += cnt


run()
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
run()
t1.record()
torch.cuda.synchronize()
ms = t0.elapsed_time(t1)
cells = (mid.own_hi - mid.own_lo) * (solver.grid.num_t - 1)
print(f"slab {mid.rank}/{a.world}: own {mid.own_hi - mid.own_lo} cells, window {mid.win_hi - mid.win_lo}, k={k}, "
      f"period={period}: {ms:.1f} ms -> {cells / (ms * 1e-3):.3e} owned cell-updates/s per rank")
st.close()
