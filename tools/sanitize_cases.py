"""Small runs covering every kernel family, for compute-sanitizer (memcheck/racecheck)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402
from cases import CASES  # noqa: E402
from paper_2005_05412_b200 import slabs  # noqa: E402

for name in ["sit_hard_whole", "multi_material", "vacuum_sources", "rand3_split", "rand5_split", "rand8_split",
             "rand2_rk4", "rand4_rk4", "kernel6_split", "song_point", "point2", "tiny_group"]:
    mb.clear_material_library()
    build, stepper = CASES[name]
    dev, sce = build(mb)
    gpu.GpuFdtdSolver(dev, sce, stepper=stepper, monitor_invariants=True).run()
    print("ok", name, flush=True)
# the persistent wavefront kernel (cross-CTA acquire/release tickets): forced
# on small two-level runs, with and without records inside the wave
from paper_2005_05412_b200 import configs  # noqa: E402
for exact in (False, True):
    mb.clear_material_library()
    dev, sce = configs.cfg1(mb, nx=4096, steps=600, cells=(100, 2000, 4000))
    gpu.GpuFdtdSolver(dev, sce, persistent=True, tile_steps=16, exact=exact, monitor_invariants=True).run()
    print("ok persistent", "exact" if exact else "fast", flush=True)
mb.clear_material_library()
build, stepper = CASES["multi_material"]
dev, sce = build(mb)
slabs.run_slabs_local(gpu.GpuFdtdSolver(dev, sce, stepper=stepper), 3)
print("ok slabs", flush=True)
# peer-mailbox exchange (push / pull kernels), with and without edge strips
for case, count, overlap in (("multi_material", 3, False), ("rand6_split", 3, True)):
    mb.clear_material_library()
    build, stepper = CASES[case]
    dev, sce = build(mb)
    slabs.run_slabs_local(gpu.GpuFdtdSolver(dev, sce, stepper=stepper), count, overlap=overlap, exchange="p2p")
    print("ok slabs p2p", case, flush=True)
