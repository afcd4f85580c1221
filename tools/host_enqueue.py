"""Host-side cost of enqueueing the per-launch step sequence (cfg1): wall time
of mbg_advance's return (the launches are asynchronous) against the device
time of the same steps, on one handle reused and on a fresh handle per run."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2005_05412_b200 as gpu  # noqa: E402
from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from paper_2005_05412_b200 import configs  # noqa: E402


def run(h, s, label):
    h.call("mbg_synchronize")
    h.call("mbg_event_begin")
    t0 = time.perf_counter()
    h.call("mbg_advance", 1, s.grid.num_t - 1)
    t1 = time.perf_counter()
    ms = C.c_float(0)
    h.call("mbg_event_end", C.byref(ms))
    t2 = time.perf_counter()
    print(f"{label}: enqueue {1e3 * (t1 - t0):.2f} ms, until done {1e3 * (t2 - t0):.2f} ms, device {ms.value:.2f} ms",
          flush=True)


mb.clear_material_library()
dev, sce = configs.cfg1(mb)
s = gpu.GpuFdtdSolver(dev, sce)
h = s.open_handle()
s.upload_initial_state(h)
h.call("mbg_sample", 0)
h.call("mbg_checkpoint_save")
for rep in range(3):
    h.call("mbg_checkpoint_restore")
    run(h, s, "same handle")
h.close()
for rep in range(3):
    mb.clear_material_library()
    dev, sce = configs.cfg1(mb)
    s = gpu.GpuFdtdSolver(dev, sce)
    h = s.open_handle()
    s.upload_initial_state(h)
    h.call("mbg_sample", 0)
    run(h, s, "fresh handle")
    run(h, s, "  same fresh handle, second advance (state continues)")
    h.close()
