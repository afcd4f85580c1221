"""Generate golden records by running the REFERENCE solver (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [case ...]

Imports ``mblight`` from /root/reference/pkg/src, builds each case of
``tests/cases.py`` through the reference's own setup API, runs
``mblight.solver_fdtd.FdtdSolver`` and stores every ``Result`` in
``tests/golden/<case>.npz`` (data + axes).  The GPU box never reads
/root/reference; the tests only read these fixtures.
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

import mblight  # noqa: E402
from cases import BUILTIN_TWINS, CASES, SLOW  # noqa: E402


def generate(name, threads):
    build, stepper = CASES[name]
    mblight.clear_material_library()
    dev, sce = build(mblight)
    solver = mblight.FdtdSolver(dev, sce, stepper=stepper, threads=threads)
    t = time.perf_counter()
    results = solver.run()
    elapsed = time.perf_counter() - t
    arrays = {}
    meta = {"case": name, "stepper": stepper, "threads": solver.threads, "elapsed_s": elapsed,
            "grid": [solver.grid.num_x, solver.grid.dx, solver.grid.num_t, solver.grid.dt],
            "records": []}
    for k, r in enumerate(results):
        arrays[f"r{k}"] = r.data
        meta["records"].append({"name": r.name, "t0": r.t0, "dt_sample": r.dt_sample, "x0": r.x0, "dx": r.dx})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    if name in BUILTIN_TWINS:
        # the case restates one of the reference's built-in setups: its run
        # must equal builtin_setup's own, record for record and bit for bit
        (setup, gridpoints, end_time), shared = BUILTIN_TWINS[name]
        mblight.clear_material_library()
        bdev, bsce = mblight.builtin_setup(setup, gridpoints=gridpoints, end_time=end_time)
        twin = mblight.FdtdSolver(bdev, bsce, stepper=stepper, threads=threads).run()
        for a, b in zip(results[:shared], twin[:shared]):
            assert a.name == b.name and np.array_equal(a.data, b.data), (name, a.name)
        meta["builtin_twin"] = setup
        arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(f"{name}: {len(results)} records, {elapsed:.1f} s", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or [n for n in CASES if n not in SLOW]
    threads = int(os.environ.get("GOLDEN_THREADS", os.cpu_count() or 1))
    for n in names:
        generate(n, threads)
