"""Parity report: every golden case (records of the reference solver) vs the
GPU solver, fast and exact variants -> profiles/<tag>_parity.json.

    python tools/parity_report.py [--tag r1]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from cases import CASES  # noqa: E402
from conftest import load_golden, rel_err  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="r1")
a = ap.parse_args()
out = {}
for name in sorted(CASES):
    row = {}
    for exact in (False, True):
        mb.clear_material_library()
        build, stepper = CASES[name]
        dev, sce = build(mb)
        s = gpu.GpuFdtdSolver(dev, sce, stepper=stepper, exact=exact)
        t = time.perf_counter()
        res = s.run()
        wall = time.perf_counter() - t
        meta, recs = load_golden(name)
        errs = [rel_err(r.data, ref) for r, (_, ref, _) in zip(res, recs)]
        bit = all(np.array_equal(r.data, ref) for r, (_, ref, _) in zip(res, recs))
        key = "exact" if exact else "fast"
        row[key] = {"max_rel_err": max(errs), "bitwise": bit, "gpu_run_s": round(wall, 4)}
    g = s.grid
    row["grid"] = {"num_x": g.num_x, "steps": g.num_t - 1, "levels": s.plan.levels, "stepper": s.stepper}
    row["reference_cpu_s"] = round(meta.get("elapsed_s", float("nan")), 2)
    out[name] = row
    print(f"{name:22s} N={s.plan.levels} {g.num_x:>8d} x {g.num_t - 1:>6d}  fast {row['fast']['max_rel_err']:.2e}"
          f"  exact {row['exact']['max_rel_err']:.2e} bitwise={row['exact']['bitwise']}"
          f"  gpu {row['fast']['gpu_run_s']:.3f}s ref {row['reference_cpu_s']}s", flush=True)
(ROOT / "profiles" / f"{a.tag}_parity.json").write_text(json.dumps(out, indent=1))
