"""Small N-level domains through the public call (default tile depth):
the reference's tzenov2016 / tzenov2016-full and the qcl5 / ladder6 golden cases."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2005_05412_b200 as gpu  # noqa: E402
from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from cases import CASES  # noqa: E402

jobs = [("tzenov2016", lambda: mb.builtin_setup("tzenov2016")), ("tzenov2016-full", lambda: mb.builtin_setup("tzenov2016-full"))]
for name in ("qcl5", "ladder6"):
    jobs.append((name, lambda n=name: CASES[n][0](mb)))
for name, build in jobs:
    for rep in range(2):
        mb.clear_material_library()
        dev, sce = build()
        s = gpu.GpuFdtdSolver(dev, sce)
        t = time.perf_counter()
        s.run()
        dt = time.perf_counter() - t
    print(f"{name:16s} {s.grid.num_x:6d} x {s.grid.num_t - 1:7d}: wall {dt:.3f} s device {s.kernel_ms / 1e3:.3f} s "
          f"launches {s.launches}", flush=True)
