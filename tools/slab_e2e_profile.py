"""The public multi-GPU call at world size 1 (NCCL) against GpuFdtdSolver.run() on cfg2: wall time of
run_slab_rank (window upload, streamed sources, the step loop, record gather) with a cProfile of
the third run -- the host overhead a rank adds to its device time.

    python tools/slab_e2e_profile.py
"""
import sys, time, os
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parent.parent))
import torch, torch.distributed as dist
import paper_2005_05412_b200 as gpu
from paper_2005_05412_b200.reference import mblight as mb
from paper_2005_05412_b200 import configs, slabs
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29544")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda",0))
dev0 = torch.device("cuda",0)
for it in range(3):
    mb.clear_material_library()
    t0=time.perf_counter(); dev,sce=configs.cfg2(mb); sol=gpu.GpuFdtdSolver(dev,sce); t1=time.perf_counter()
    import cProfile, pstats
    pr=cProfile.Profile(); pr.enable()
    recs=slabs.run_slab_rank(sol,1,0,dev0); torch.cuda.synchronize()
    pr.disable(); t2=time.perf_counter()
    print(f"iter {it}: build {t1-t0:.3f}s run_slab_rank {t2-t1:.3f}s")
    if it==2:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
for it in range(2):
    mb.clear_material_library()
    dev,sce=configs.cfg2(mb); sol=gpu.GpuFdtdSolver(dev,sce)
    t1=time.perf_counter(); sol.run(); t2=time.perf_counter()
    print(f"run(): {t2-t1:.3f}s")
dist.destroy_process_group()
