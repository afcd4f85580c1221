"""Short run of a BASELINE workload for profiling (ncu / compute-sanitizer).

    python tools/prof_step.py [cfg2|cfg3|cfg4|cfg5] [--steps S] [--tile-steps K] [--exact]

Builds the scenario, uploads it and runs S time steps (default 4 launches
worth) through the same C-ABI calls bench.py uses, then exits.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="cfg2")
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--tile-steps", type=int, default=None)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--stepper", default="splitting")
ap.add_argument("--nx", type=int, default=0)
ap.add_argument("--per-launch", action="store_true", help="one launch per k steps (no persistent kernel)")
ap.add_argument("--advance-steps", type=int, default=0, help="steps per mbg_advance call (0: all at once)")
ap.add_argument("--no-warm", action="store_true", help="single pass (for ncu)")
ap.add_argument("--real", action="store_true", help="cfg4: the real-Hamiltonian twin of the medium")
a = ap.parse_args()
kw = {"nx": a.nx} if a.nx else {}
if a.real:
    kw["real"] = True
total = max(400, a.steps)
if a.config == "cfg5":
    dev, sce = configs.cfg5(mb, steps=total)
else:
    dev, sce = getattr(configs, a.config)(mb, **kw, **({"steps": total} if a.config != "cfg1" else {}))
sol = gpu.GpuFdtdSolver(dev, sce, stepper=a.stepper, tile_steps=a.tile_steps, exact=a.exact,
                       persistent=False if a.per_launch else None)
h = sol.open_handle()
sol.upload_initial_state(h)
k = C.c_int32(0)
h.call("mbg_tile_steps", C.byref(k))
steps = a.steps or 4 * k.value
h.call("mbg_sample", 0)


def advance():
    per = a.advance_steps or steps
    n = 1
    while n < steps + 1:
        cnt = min(per, steps + 1 - n)
        h.call("mbg_advance", n, cnt)
        n += cnt


if not a.no_warm:  # ramp clocks / load modules outside the timed region
    h.call("mbg_checkpoint_save")
    advance()
    h.call("mbg_checkpoint_restore")
h.call("mbg_event_begin")
advance()
ms = C.c_float(0)
h.call("mbg_event_end", C.byref(ms))
print(f"{a.config}/{a.stepper}: nx={sol.grid.num_x} k={k.value} steps={steps} device {ms.value:.3f} ms "
      f"-> {sol.grid.num_x * steps / (ms.value * 1e-3):.3e} cell-updates/s")
h.close()
