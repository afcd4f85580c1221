"""Where the e2e time of GpuFdtdSolver.run() goes (cfg2), phase by phase."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2005_05412_b200 as gpu  # noqa: E402
from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs  # noqa: E402

for rep in range(3):
    mb.clear_material_library()
    dev, sce = configs.cfg2(mb)
    s = gpu.GpuFdtdSolver(dev, sce)
    t = [time.perf_counter()]
    h = s.open_handle(); t.append(time.perf_counter())
    s.upload_initial_state(h); t.append(time.perf_counter())
    s._ran = True
    s._run_on(h); t.append(time.perf_counter())
    res = s.download_results(h); t.append(time.perf_counter())
    h.close(); t.append(time.perf_counter())
    names = ["open_handle", "upload", "run", "download", "close"]
    print(" ".join(f"{n}={1e3 * (b - a):.1f}ms" for n, a, b in zip(names, t, t[1:])), f"device={s.kernel_ms:.1f}ms")
