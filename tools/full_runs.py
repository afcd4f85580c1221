"""The BASELINE configurations at their full size and length on one B200,
through the public solver API (GpuFdtdSolver.run with the invariant monitor):
wall time, device time, cell-updates/s, the invariant report (max |trace - 1|,
Hermiticity, min eigenvalue) and the record extrema.

    python tools/full_runs.py [cfg1 cfg2 cfg3 cfg4 cfg5]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs  # noqa: E402

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
for name in names:
    mb.clear_material_library()
    t0 = time.perf_counter()
    dev, sce = getattr(configs, name)(mb)
    sol = gpu.GpuFdtdSolver(dev, sce, monitor_invariants=True)
    t1 = time.perf_counter()
    res = sol.run()
    t2 = time.perf_counter()
    g = sol.grid
    cells = g.num_x * (g.num_t - 1)
    line = {
        "config": name, "num_x": g.num_x, "steps": g.num_t - 1, "levels": sol.plan.levels,
        "setup_s": round(t1 - t0, 2), "run_s": round(t2 - t1, 2), "device_ms": round(sol.kernel_ms, 1),
        "cell_updates_per_s_device": cells / (sol.kernel_ms * 1e-3), "cell_updates_per_s_wall": cells / (t2 - t1),
        "invariants": sol.invariant_report,
        "records": {r.name: [float(np.min(np.real(r.data))), float(np.max(np.real(r.data)))] for r in res},
        "finite": all(bool(np.all(np.isfinite(r.data))) for r in res),
    }
    print(json.dumps(line), flush=True)
