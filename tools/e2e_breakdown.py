"""Where the e2e time of the public call goes (cfg2), phase by phase:
create_solver (plan build), open_handle (device solver, constants, record
buffers, source table + pinned staging), upload of the initial state, the run
(sources sampled segment by segment while the device steps), record download
and close -- the same calls GpuFdtdSolver.run() makes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2005_05412_b200 as gpu  # noqa: E402,F401
from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs  # noqa: E402

for rep in range(4):
    mb.clear_material_library()
    dev, sce = configs.cfg2(mb)
    t = [time.perf_counter()]
    s = mb.create_solver("gpu-fdtd-reg-cayley", dev, sce); t.append(time.perf_counter())
    h = s.open_handle(stream_sources=True); t.append(time.perf_counter())
    s.upload_initial_state(h); t.append(time.perf_counter())
    s._ran = True
    s._run_on(h); t.append(time.perf_counter())
    res = s.download_results(h); t.append(time.perf_counter())
    h.close(); t.append(time.perf_counter())
    names = ["create_solver", "open_handle", "upload", "run", "download", "close"]
    print(" ".join(f"{n}={1e3 * (b - a):.2f}ms" for n, a, b in zip(names, t, t[1:])),
          f"total={1e3 * (t[-1] - t[0]):.1f}ms device={s.kernel_ms:.1f}ms launches={s.launches}", flush=True)
