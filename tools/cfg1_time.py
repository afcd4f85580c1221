import sys, time
sys.path.insert(0, '.')
import paper_2005_05412_b200 as gpu
from paper_2005_05412_b200.reference import mblight as mb
from paper_2005_05412_b200 import configs
for k in (None, 8, 16, 32):
    for rep in range(2):
        mb.clear_material_library()
        dev, sce = configs.cfg1(mb)
        s = gpu.GpuFdtdSolver(dev, sce, tile_steps=k)
        t = time.perf_counter(); s.run(); dt = time.perf_counter() - t
    print(f"cfg1 k={k}: run() {dt*1e3:.1f} ms wall, device {s.kernel_ms:.1f} ms, launches {s.launches}, "
          f"{s.grid.num_x*(s.grid.num_t-1)/dt:.3e} cell-updates/s e2e")
