"""Cell-update rate of the N-level kernels on a random N-level medium
(tests/cases.py random_medium), one line per N and operator kind:

    python tools/nlevel_rate.py [--levels 3 4 5 6 7 8] [--nx 1048576] [--stepper splitting|rk4]

Times 8 launches of k steps with CUDA events through the C ABI (as
tools/prof_step.py does for the BASELINE configs).
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2005_05412_b200 as gpu  # noqa: E402
from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from cases import random_medium  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--levels", type=int, nargs="+", default=[3, 4, 5, 6, 7, 8])
ap.add_argument("--nx", type=int, default=1 << 20)
ap.add_argument("--stepper", default="splitting")
ap.add_argument("--launches", type=int, default=8)
a = ap.parse_args()

for dim in a.levels:
    for real in (False, True):
        mb.clear_material_library()
        rng = np.random.default_rng(100 + dim)
        desc = random_medium(mb, rng, dim, real=real)
        act = mb.ensure_material(mb.Material(f"Rate{dim}" + ("r" if real else ""), qm=desc))
        dev = mb.Device(f"rate{dim}")
        length = 20e-6
        dev.add_region(mb.Region("a", act.id, 0.0, length))
        dt = 0.5 * (length / a.nx) / 299792458.0
        rho0 = np.zeros(dim)
        rho0[0] = 1.0
        sce = mb.Scenario("s", a.nx, 400 * dt, mb.QmOperator(rho0))
        sce.add_source(mb.SechPulse("sech", 0.0, "hard", 1e9, 2e14, 5.0, 1e15))
        sce.add_record(mb.Record("e", quantity="e", interval=100 * dt, position=length / 2))
        sol = gpu.GpuFdtdSolver(dev, sce, stepper=a.stepper)
        h = sol.open_handle()
        sol.upload_initial_state(h)
        k = C.c_int32(0)
        h.call("mbg_tile_steps", C.byref(k))
        steps = a.launches * k.value
        h.call("mbg_sample", 0)
        h.call("mbg_checkpoint_save")
        h.call("mbg_advance", 1, steps)
        h.call("mbg_checkpoint_restore")
        h.call("mbg_event_begin")
        h.call("mbg_advance", 1, steps)
        ms = C.c_float(0)
        h.call("mbg_event_end", C.byref(ms))
        print(f"N={dim} {'real   ' if real else 'complex'} {a.stepper}: nx={sol.grid.num_x} k={k.value} steps={steps} "
              f"device {ms.value:.3f} ms -> {sol.grid.num_x * steps / (ms.value * 1e-3):.3e} cell-updates/s", flush=True)
        h.close()
