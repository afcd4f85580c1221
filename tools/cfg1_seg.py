"""Public-call loop (GpuFdtdSolver.run) against the plain advance on the
small cfg1 and the large cfg2: wall and device time per run."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2005_05412_b200 as gpu  # noqa: E402
from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs  # noqa: E402

for name in ("cfg1", "cfg2"):
    for rep in range(4):
        mb.clear_material_library()
        dev, sce = getattr(configs, name)(mb)
        t = time.perf_counter()
        s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce)
        s.run()
        wall = time.perf_counter() - t
    print(f"{name}: run() wall {1e3 * wall:.1f} ms device {s.kernel_ms:.1f} ms launches {s.launches}", flush=True)
