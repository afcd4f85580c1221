"""Throughput of the batched single-point mode: B song2005-type three-level
systems (pulse amplitudes swept over [0.1, 3] x the pi-pulse amplitude),
10000 steps each, one run_points call, against one single-point solver run.

    python tools/points_bench.py [--systems B] [--stepper splitting|rk4]
"""
import argparse
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200.points import LAST_RUN, run_points  # noqa: E402
from test_gpu_points import _song  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--systems", type=int, default=4096)
ap.add_argument("--stepper", default="splitting")
ap.add_argument("--fast-sources", action="store_true", help="run_points(fast_sources=True)")
ap.add_argument("--sweep", choices=("pulse", "media"), default="pulse",
                help="pulse: one three-level medium, pulse amplitudes swept; media: distinct two-level "
                     "media (T2 swept), one shared pulse")
a = ap.parse_args()
mb.clear_material_library()
if a.sweep == "pulse":
    scales = np.linspace(0.1, 3.0, a.systems)
    problems = [_song(scale=float(s)) for s in scales]
else:
    from test_gpu_points import _two_level  # noqa: E402

    problems = [_two_level(t2=float(t), tag=f"m{i}") for i, t in enumerate(np.linspace(2e11, 5e12, a.systems))]
run_points(problems[:8], stepper=a.stepper)  # warm (module load)
t0 = time.perf_counter()
res = run_points(problems, stepper=a.stepper, fast_sources=a.fast_sources)
t_batch = time.perf_counter() - t0
steps = problems[0][1].num_timesteps - 1 if problems[0][1].num_timesteps else 9999
sol = gpu.GpuFdtdSolver(*problems[0], stepper=a.stepper)
t0 = time.perf_counter()
sol.run()
t_one = time.perf_counter() - t0
t_dev = LAST_RUN["batch_s"]
print(f"{a.systems} systems x {steps} steps ({a.stepper}, {a.sweep} sweep{', fast sources' if a.fast_sources else ''}): run_points {t_batch:.3f} s = host "
      f"setup {LAST_RUN['host_setup_s']:.3f} s (plans, media, field sequences) + native batch call {t_dev:.3f} s "
      f"({a.systems * steps / t_dev:.3e} system-steps/s) + results {LAST_RUN['host_results_s']:.3f} s; "
      f"one single-point solver run {t_one:.3f} s ({steps / t_one:.3e} steps/s)")
