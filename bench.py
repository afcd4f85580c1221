"""Benchmark of the time-stepping core (BASELINE.json metric: cell-updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]

Workload (BASELINE.json configs[1], "cfg2"): two-level SIT medium, Nx = 2^22
cells (x N for --gpus N: weak scaling, 2^22 cells per GPU), 20000 time steps
with T1 = 1 ns / T2 = 1 ps relaxation, seeded synthetic initial inversion,
3 point records x 4 quantities every 100 steps.  One bench "step" is one full
20000-time-step run of that scenario from its initial condition: restore the
initial state (device-to-device), sample row 0, run every fused launch.

``value`` is device time (CUDA events on the launch stream, max over ranks)
with the state resident in HBM; ``e2e`` times the public API call
(``mblight.create_solver("gpu-fdtd-reg-cayley", ...).run()``: plan build with
the sources sampled by Source.value, initial-state upload, the run, record
download) every step.  ``--impl reference`` times the CPU restatement of the
reference loop (oracle/, OpenMP C port) on all host cores; both lines also
carry ``cpu_baseline_stock``: the reference's own numba solver
(``mblight.FdtdSolver``, installed unmodified in baseline/_ref) on the same
cores with all threads and with one, on bounded step samples.
Extra keys: ``roofline`` (sustained FP64 denominator, algorithmic and executed
fractions), ``n_level`` (BASELINE configs[2] / [3] samples), and
``scaling_samples`` (cfg4 strong scaling and the cfg5 exchange-period sweep
with efficiencies against one GPU; see scaling_samples()).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "cell-updates/sec (fp64, N-level) at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "cell-updates/s"


# ----------------------------------------------------------------- helpers --

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def build_workload(mb, gpus):
    from paper_2005_05412_b200 import configs

    mb.clear_material_library()
    if gpus == 1:
        return configs.cfg2(mb)
    # weak scaling: G copies of the cfg2 device side by side, 2^22 cells per
    # GPU, so each rank steps exactly cfg2's mix of medium and vacuum cells
    return configs.cfg2(mb, nx=(1 << 22) * gpus, replicas=gpus)


def algorithmic_per_cell(plan):
    """bytes B and flops F per cell-update (k = 1)."""
    nx = plan.grid.num_x
    qcells = sum(hi - lo for lo, hi, _ in plan.groups)
    fq = qcells / nx
    n = plan.levels
    sn = plan.state_words
    b = 32 + fq * 16 * sn
    if plan.stepper == "rk4" and n >= 2:
        fn = rk4_flops(n, int(np.count_nonzero(plan.qm[0].pol_v)), len(plan.qm[0].pol_di))
    elif n == 2:
        fn = 82
    elif n == 0:
        fn = 9
    else:
        nnz_off = int(np.count_nonzero(plan.qm[0].pol_v))
        nnz_d = len(plan.qm[0].pol_di)
        fn = 12 * n * n + 4 * n * n
        fn += sum(6 + (n - k - 1) * (6 + 8 * (n - k - 1) + 8 * n) for k in range(n))
        fn += sum(6 + n * (8 * (n - 1 - k) + 6) for k in range(n))
        fn += 8 * n ** 3 + 4 * n * n * (n + 1) + 10 * nnz_off + 3 * nnz_d + 1 + 9
    f = 9 + fq * (fn - 9)
    return b, f, fq


def rk4_flops(n, nnz_off, nnz_d):
    """Algorithmic flops of one RK4 cell-update in the reference's loop
    (_kernels.py:256-332; complex mul 6, add 2, real x complex 2), plus the
    FDTD's 9: H = h0 - E mu (4 n^2); per stage the commutator
    -i/hbar sum_k (H_ik S_kj - S_ik H_kj) (n^2 (14 n + 4)), dephasing
    (4 n (n - 1)) and population transfer (4 n^2); three stage states
    (4 n^2 each); the RK4 combination (14 n^2); symmetrisation (2 n (n - 1));
    the polarisation trace (10 per off-diagonal dipole, 3 per diagonal)."""
    stage = n * n * (14 * n + 4) + 4 * n * (n - 1) + 4 * n * n
    return (4 * n * n + 4 * stage + 3 * 4 * n * n + 14 * n * n + 2 * n * (n - 1) + 10 * nnz_off + 3 * nnz_d + 1
            + 9)


def measured_hbm_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_entry(config_key):
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(p.read_text()).get(config_key, {})
    except (OSError, ValueError):
        return {}


def ncu_traffic(config_key):
    return ncu_entry(config_key).get("dram_bytes_per_launch")


# -------------------------------------------------------------- reference --

def run_reference(args, world, rank):
    """CPU restatement of the reference loop (oracle/, kind 'port') on all host cores."""
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc

    import paper_2005_05412_b200 as gpu

    from paper_2005_05412_b200.reference import mblight as mb
    from paper_2005_05412_b200.plan import build_plan

    dev, sce = build_workload(mb, args.gpus)
    plan = build_plan(dev, sce)
    threads = os.cpu_count() or 1
    sample = args.cpu_steps
    nx = plan.grid.num_x
    for _ in range(args.warmup):
        orc.OracleRun(plan, threads=threads, step_limit=max(1, sample // 10)).run()
    t = 0.0
    for _ in range(args.steps):
        run = orc.OracleRun(plan, threads=threads, step_limit=sample)
        t0 = time.perf_counter()
        bad = run.run()
        t += time.perf_counter() - t0
        assert bad == 0
    value = nx * sample * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(plan, args),
        "implementation": {"kind": "CPU restatement of the reference loop (oracle/mb_oracle.c), OpenMP",
                           "threads": threads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} of {plan.grid.num_t - 1} time steps at full Nx={nx} per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline_stock": None if args.no_cpu_baseline else stock_reference(args.gpus),
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(plan, args):
    """The workload, identical for both arms (implementation knobs such as the
    GPU's temporal tile depth go under ``implementation``)."""
    return {
        "workload": "cfg2 (BASELINE configs[1]): two-level SIT, T1=1ns T2=1ps, Strang splitting, "
                    "soft sech source, 3 point records x 4 quantities every 100 steps",
        "num_x": plan.grid.num_x, "time_steps": plan.grid.num_t - 1, "levels": plan.levels,
        "exact": bool(args.exact),
        "parallelism": f"slab{args.gpus}" if args.gpus > 1 else "single-gpu",
        "l2": "inputs larger than L2 (E/H/Bloch state ping-pong ~335 MB per GPU vs 126 MB L2)",
    }


# ------------------------------------------------------------------- mine --

MARK_STEPS = 31  # per-step advance timing marks (mbg_mark slots 2..63)


def run_mine(args, world, rank, local):
    import ctypes as C

    import paper_2005_05412_b200 as gpu

    from paper_2005_05412_b200.reference import mblight as mb
    from paper_2005_05412_b200 import native

    dev, sce = build_workload(mb, args.gpus)
    if world > 1:
        from paper_2005_05412_b200 import slabs
        backend, _ = slabs.slab_backend(local)
        samples = None if args.no_scaling_samples else (
            lambda w, r, d: scaling_samples(w, r, d, backend=backend))
        from paper_2005_05412_b200.plan import build_plan

        cfg = workload_config(build_plan(dev, sce), args)
        return slabs.bench_rank(args, dev, sce, world, rank, local, METRIC, UNIT, clock_sampler=ClockSampler,
                                config=cfg,
                                rebuild=lambda: build_workload(mb, args.gpus), samples=samples)

    solver = gpu.GpuFdtdSolver(dev, sce, tile_steps=args.tile_steps, exact=args.exact, gpu=local)
    plan = solver.plan
    num_t = plan.grid.num_t
    nx = plan.grid.num_x
    h = solver.open_handle()
    solver.upload_initial_state(h)
    h.call("mbg_checkpoint_save")
    k = C.c_int32(0)
    h.call("mbg_tile_steps", C.byref(k))
    k = k.value

    def one_step(i=None):
        h.call("mbg_checkpoint_restore")
        h.call("mbg_sample", 0)
        if i is not None and i < MARK_STEPS:
            h.call("mbg_mark", 2 + 2 * i)
        h.call("mbg_advance", 1, num_t - 1)
        if i is not None and i < MARK_STEPS:
            h.call("mbg_mark", 3 + 2 * i)

    for _ in range(args.warmup):
        one_step()
    h.call("mbg_synchronize")
    l0 = C.c_int64(0)
    h.call("mbg_launch_count", C.byref(l0))
    with ClockSampler(local) as clocks:
        h.call("mbg_mark", 0)
        for i in range(args.steps):
            one_step(i)
        h.call("mbg_mark", 1)
        ms = C.c_float(0)
        h.call("mbg_mark_elapsed", 0, 1, C.byref(ms))
    ms = float(ms.value)
    # device time of the step launches alone (mbg_advance: the persistent
    # step kernel and its step-mask pre-kernel), from marks on the same stream
    adv_ms = []
    for i in range(min(args.steps, MARK_STEPS)):
        t = C.c_float(0)
        h.call("mbg_mark_elapsed", 2 + 2 * i, 3 + 2 * i, C.byref(t))
        adv_ms.append(float(t.value))
    l1 = C.c_int64(0)
    h.call("mbg_launch_count", C.byref(l1))
    launches = l1.value - l0.value
    bad = C.c_int64(0)
    h.call("mbg_poll_nonfinite", C.byref(bad))
    assert bad.value < 0, "non-finite field in the benchmark run"
    h.close()

    cell_updates = nx * (num_t - 1) * args.steps
    value = cell_updates / (ms * 1e-3)

    # e2e through the public API: plan, upload ICs, run, download records, every
    # step -- right after the device-timed region, before the FP64 peak train
    e2e_times = []
    h2d = d2h = 0
    for it in range(args.warmup + args.steps):
        mb.clear_material_library()
        d2, s2 = build_workload(mb, 1)
        t0 = time.perf_counter()
        # the call a user makes: create_solver(...) builds the plan and run()
        # uploads, steps (sampling the sources with Source.value as it goes, as
        # the reference's run() does per step), downloads the records
        sol = mb.create_solver("gpu-fdtd-reg-cayley", d2, s2, tile_steps=args.tile_steps, exact=args.exact,
                               gpu=local)
        res = sol.run()
        dt_run = time.perf_counter() - t0
        if it >= args.warmup:
            e2e_times.append(dt_run)
        if it == 0:
            p = sol.plan
            # initial E/H (skipped when identically zero: a device memset), rho0, source samples
            fields = 0 if p.fields_zero else p.grid.num_x + (p.grid.num_x + 1) + 1
            h2d = 8 * (fields + p.state_words + p.src_values.size)
            d2h = sum(r.data.size * (16 if r.is_complex else 8) for r in res) + 8 * max(1, (num_t - 1) // (1 << 14))
    e2e_value = cell_updates / sum(e2e_times)
    e2e_note = ("wall clock around mblight.create_solver('gpu-fdtd-reg-cayley', device, scenario).run(): plan "
                "build, initial-state upload, the run (the sources sampled with Source.value segment by segment "
                "while the device steps, rows copied through pinned staging), record download")

    # roofline of the dominant kernel: one persistent launch per run (two-level
    # medium, one GPU) working through ceil((Nt-1)/k) fused chunks
    b, f, fq = algorithmic_per_cell(plan)
    burst = C.c_double(0)
    native.load().mbg_fp64_peak(local, C.byref(burst))
    sustained = C.c_double(0)
    native.load().mbg_fp64_peak_sustained(local, 2.0, C.byref(sustained))
    # the same chains with three distinct register operands per DFMA (what
    # matrix-times-matrix FP64 code issues): the register file cannot feed
    # those at the pipe's full rate, so this is the ceiling of real FP64 code
    three_reg = C.c_double(0)
    native.load().mbg_fp64_peak_operands(local, 3, C.byref(three_reg))
    # the step kernel runs inside ~1 s of back-to-back runs: the sustained
    # DFMA figure (>= 2 s train, same clocks) is its denominator
    peak_fp64 = sustained.value
    bw, bw_src = measured_hbm_gbs()
    persistent = plan.levels <= 2 and solver.stepper == "splitting" and num_t - 1 > k
    chunks = (num_t - 1 + k - 1) // k
    per_launch_ms = sum(adv_ms) / len(adv_ms)
    cells_per_launch = nx * (num_t - 1)
    flops_launch = f * cells_per_launch
    bytes_launch = b * nx * chunks  # E, H and the state read + written once per fused chunk
    t_hbm = bytes_launch / (bw * 1e9)
    t_fp = flops_launch / (peak_fp64 * 1e12)
    bound = "fp64" if t_fp >= t_hbm else "hbm"
    if bound == "fp64":
        achieved = flops_launch / (per_launch_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": peak_fp64, "unit": "TFLOP/s",
                "frac": achieved / peak_fp64}
    else:
        achieved = bytes_launch / (per_launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": bw, "unit": "GB/s", "frac": achieved / bw}
    ncu_key = f"cfg2_wave_k{k}" if persistent else f"cfg2_k{k}"
    traffic = ncu_traffic(ncu_key)
    nc = ncu_entry(ncu_key)
    if nc.get("mix_per_cell_step"):
        mix = nc["mix_per_cell_step"]
        executed = 2 * mix.get("DFMA", 0.0) + mix.get("DMUL", 0.0) + mix.get("DADD", 0.0)
        roof["executed_frac"] = executed * cells_per_launch / (per_launch_ms * 1e-3) / 1e12 / peak_fp64
        roof["executed"] = {
            "source": f"profiles/ncu_summary.json[{ncu_key}] (ncu --set full of the same launch)",
            "fp64_instr_per_cell_step": nc.get("fp64_instr_per_cell_step"),
            "fp64_flops_per_cell_step": round(executed, 1),
            "fp64_pipe_pct": nc.get("fp64_pipe_pct"),
            "achieved_tflops": executed * cells_per_launch / (per_launch_ms * 1e-3) / 1e12,
            # FP64 instructions issued per second against the pipe's peak
            # instruction rate (one DFMA = 2 flops of the measured peak): the
            # pipe utilisation, independent of how few operations a step takes
            "fp64_instr_frac": (nc.get("fp64_instr_per_cell_step") or 0.0) * cells_per_launch
                               / (per_launch_ms * 1e-3) / (peak_fp64 * 1e12 / 2.0),
            # the same instruction rate against the measured rate of DFMAs
            # with three distinct register operands (mbg_fp64_peak_operands, mode 3)
            "fp64_instr_frac_of_3reg_rate": (nc.get("fp64_instr_per_cell_step") or 0.0) * cells_per_launch
                                            / (per_launch_ms * 1e-3) / (three_reg.value * 1e12 / 2.0),
            "note": ("frac counts SURVEY 8(d)'s algorithmic flops (the reference's 82-flop Bloch step); the fast "
                     "kernel evaluates the same step in fewer FP64 operations (Rodrigues-form rotation, fused "
                     "relaxations), so frac can exceed 1 -- the executed figures and the FP64 pipe share "
                     "say how busy the pipe really is"),
        }
    roof.update({
        "traffic": traffic,
        "kernel": ("bloch_wave_kernel (one persistent launch per run: ticketed (chunk, tile) items of k fused "
                   "steps, H + Bloch + E + boundary + sources + records)" if persistent else
                   "bloch_interior_kernel (fused H + Bloch + E + records, k steps/launch)"),
        "algorithmic_bytes_per_cell_update_k1": b, "algorithmic_flops_per_cell_update": f,
        "bytes_per_launch": bytes_launch, "flops_per_launch": flops_launch, "fused_chunks_per_launch": chunks,
        "launch_ms_avg": per_launch_ms, "launch_share_of_step": sum(adv_ms) / (ms * len(adv_ms) / args.steps),
        "hbm_achieved_gbs": bytes_launch / (per_launch_ms * 1e-3) / 1e9,
        "hbm_peak_gbs": bw, "hbm_peak_source": bw_src, "fp64_peak_tflops": peak_fp64,
        "fp64_peak_burst_tflops": burst.value,
        "fp64_peak_3reg_tflops": three_reg.value,
        "fp64_peak_source": ("measured in-run: mbg_fp64_peak_sustained (independent DFMA chains on every SM with "
                             "two register operands and a uniform addend -- the pattern that reaches the pipe's "
                             "nominal rate -- back to back for >= 2 s); burst = best single 1 ms launch "
                             "(mbg_fp64_peak); 3reg = the burst measurement with three distinct register operands "
                             "per DFMA (mbg_fp64_peak_operands, mode 3): the register-file-limited DFMA rate of "
                             "matrix arithmetic whose operands are all per-cell values"),
        "roofline_cell_updates_per_s": min(bw * 1e9 * k / b, peak_fp64 * 1e12 / f),
    })

    n_level = None if args.no_n_level else n_level_samples(local, peak_fp64, three_reg_tflops=three_reg.value)
    import torch

    samples = None if args.no_scaling_samples else scaling_samples(1, 0, torch.device("cuda", local))
    stock = None if args.no_cpu_baseline else stock_reference(1)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(plan, 3 * args.cpu_steps)  # ~10 s of host work

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(plan, args),
        "implementation": {"tile_steps": k, "kernel": "bloch_wave_kernel (persistent wavefront)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "note": e2e_note},
        "gpu_launches": int(launches),  # persistent step + step-mask + row-0 sample kernels (library count)
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        # the reference's own numba solver on the same host cores (the cpu_baseline is the C port)
        "cpu_baseline_stock": stock,
        # BASELINE configs[2], [3] (N = 3, N = 6) on one GPU, bounded samples beside the headline
        "n_level": n_level,
        # cfg4 strong / cfg5 exchange-period samples (at N = 1: the single-GPU rates they scale from)
        "scaling_samples": samples,
    }
    print(json.dumps(line), flush=True)
    return 0


def n_level_samples(local, peak_tflops, chunks=16, three_reg_tflops=None):
    """BASELINE configs[2] / [3] on one GPU (N = 3 on 2^23 cells, N = 6 on 2^24
    cells): device time of `chunks` fused launches from the initial state
    (bounded samples of the 50000- / 100000-step runs; reported beside the
    headline, not the headline), with the roofline of SURVEY 8(d)."""
    import ctypes as C

    import paper_2005_05412_b200 as gpu

    from paper_2005_05412_b200.reference import mblight as mb
    from paper_2005_05412_b200 import configs, native

    out = {}
    # the splitting headline media, and the six-level medium under the RK4
    # stepper (the second registered solver)
    for name, cfg, n, stepper in (("cfg3", "cfg3", 3, "splitting"), ("cfg4", "cfg4", 6, "splitting"),
                                  ("cfg4_rk4", "cfg4", 6, "rk4")):
        mb.clear_material_library()
        dev, sce = getattr(configs, cfg)(mb)
        sol = gpu.GpuFdtdSolver(dev, sce, gpu=local, stepper=stepper)
        h = sol.open_handle()
        sol.upload_initial_state(h)
        k = C.c_int32(0)
        h.call("mbg_tile_steps", C.byref(k))
        steps = chunks * k.value
        h.call("mbg_sample", 0)
        h.call("mbg_checkpoint_save")
        h.call("mbg_advance", 1, 2 * k.value)  # warm-up (clocks, modules)
        h.call("mbg_checkpoint_restore")
        h.call("mbg_event_begin")
        h.call("mbg_advance", 1, steps)
        ms = C.c_float(0)
        h.call("mbg_event_end", C.byref(ms))
        h.close()
        rate = sol.grid.num_x * steps / (ms.value * 1e-3)
        b, f, fq = algorithmic_per_cell(sol.plan)
        out[name] = {"levels": n, "stepper": stepper, "num_x": sol.grid.num_x, "tile_steps": k.value,
                     "sampled_steps": steps,
                     "of_steps": sol.grid.num_t - 1, "value": rate, "unit": UNIT,
                     "algorithmic_flops_per_cell_update": f, "achieved_tflops": rate * f / 1e12,
                     "fp64_peak_tflops": peak_tflops, "frac": rate * f / 1e12 / peak_tflops,
                     "launches": chunks}
        # executed FP64 instructions (ncu capture of the same kernel, profiles/) per second against
        # the measured rate of DFMAs with three distinct register operands
        nc = ncu_entry({"cfg3": "cfg3_k12", "cfg4": "cfg4_k4"}.get(name, ""))
        if nc.get("fp64_instr_per_cell_step") and three_reg_tflops:
            out[name]["fp64_instr_per_cell_step"] = nc["fp64_instr_per_cell_step"]
            out[name]["fp64_instr_frac_of_3reg_rate"] = (nc["fp64_instr_per_cell_step"] * rate
                                                         / (three_reg_tflops * 1e12 / 2.0))
    return out


def cpu_baseline(plan, steps):
    """The oracle (port of the reference loop) on this box's host cores, bounded sample."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc

    threads = os.cpu_count() or 1
    orc.OracleRun(plan, threads=threads, step_limit=5).run()  # warm
    run = orc.OracleRun(plan, threads=threads, step_limit=steps)
    t0 = time.perf_counter()
    bad = run.run()
    t = time.perf_counter() - t0
    assert bad == 0
    return {"value": plan.grid.num_x * steps / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{steps} of {plan.grid.num_t - 1} time steps of the same workload at full "
                      f"Nx={plan.grid.num_x} ({t:.1f} s, OpenMP C restatement, oracle/mb_oracle.c)"}


def stock_reference(gpus, steps_all=200, steps_one=40):
    """The reference's own solver, unmodified (``mblight.FdtdSolver``, numba,
    solver_fdtd.py:444-498, installed in baseline/_ref), on this box's host
    cores: threads = cpu_count and threads = 1, each on a bounded sample --
    the workload's grid and medium with the end time cut to a few steps (its
    run() has no step limit).  A first tiny run compiles the numba loops."""
    from paper_2005_05412_b200 import configs
    from paper_2005_05412_b200.reference import mblight as mb

    def sample(steps):
        mb.clear_material_library()
        if gpus == 1:
            return configs.cfg2(mb, steps=steps)
        return configs.cfg2(mb, nx=(1 << 22) * gpus, steps=steps, replicas=gpus)

    dev, sce = configs.cfg2(mb, nx=4096, steps=4, cells=(16, 2000))
    mb.FdtdSolver(dev, sce, threads=2).run()  # numba compile (cached in NUMBA_CACHE_DIR)
    out = {"kind": "reference", "impl": "mblight.FdtdSolver (numba, unmodified)"}
    for label, threads, steps in (("threads_all", os.cpu_count() or 1, steps_all), ("threads_1", 1, steps_one)):
        dev, sce = sample(steps)
        solver = mb.FdtdSolver(dev, sce, threads=threads)
        t0 = time.perf_counter()
        solver.run()
        t = time.perf_counter() - t0
        g = solver.grid
        out[label] = {"value": g.num_x * (g.num_t - 1) / t, "unit": UNIT, "cores": solver.threads,
                      "sample": f"cfg2 grid (Nx={g.num_x}) cut to {g.num_t - 1} time steps, {t:.1f} s "
                                f"including its per-step Source.value and record sampling"}
    return out


SAMPLE_STEPS = 128


def scaling_samples(world, rank, device, backend=None, reps=3):
    """north_star's multi-GPU targets as bounded samples:

    * ``cfg3_strong``: BASELINE configs[2] (three levels, 2^23 cells) split
      over the ranks (north_star: "run on 1/2/4 GPUs"), as cfg4 below;
    * ``cfg4_strong``: BASELINE configs[3] (six levels, 2^24 cells) split over
      the ranks, SAMPLE_STEPS steps per run with the halo exchange every
      period; efficiency = rate_N / (N * rate_1), rate_1 timed on rank 0
      alone on the whole grid;
    * ``cfg5_weak``: BASELINE configs[4] (cfg4's medium, 2^22 cells per rank)
      for exchange periods P in {1, 4, 16, 64} steps (tile depth k = min(P, 4));
      efficiency = per-rank rate / the single-domain rate of 2^22 cells at the
      same k (rank 0 alone).
    Device time, max over ranks; one warm-up run each."""
    import torch.distributed as dist

    import paper_2005_05412_b200 as gpu
    from paper_2005_05412_b200 import configs, slabs
    from paper_2005_05412_b200.reference import mblight as mb

    def timed(build, w, tile_steps=None, period=None):
        mb.clear_material_library()
        dev, sce = build()
        sol = gpu.GpuFdtdSolver(dev, sce, gpu=device.index, tile_steps=tile_steps)
        overlap = w > 1 and slabs.overlaps_by_default(sol, backend or "nccl")
        t = slabs.SlabTimer(sol, w, rank if w > 1 else 0, device, steps=SAMPLE_STEPS, period=period,
                            overlap=overlap)
        try:
            ms = t.time(reps)
        finally:
            t.close()
        return sol.grid.num_x * SAMPLE_STEPS * reps / (ms * 1e-3), t.k, t.period, overlap

    def single(build, tile_steps=None):
        """rank 0 alone: the 1-GPU rate of the same sample (broadcast)."""
        val = None
        if world == 1:
            return None
        if rank == 0:
            val = timed(build, 1, tile_steps)[0]
        box = [val]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    out = {"steps_per_run": SAMPLE_STEPS, "runs": reps}
    # BASELINE configs[2]: cfg3 (three levels, 2^23 cells) over the ranks
    rate, k, period, overlap = timed(lambda: configs.cfg3(mb), world)
    one = single(lambda: configs.cfg3(mb))
    out["cfg3_strong"] = {"num_x": 1 << 23, "levels": 3, "ranks": world, "tile_steps": k,
                          "exchange_period": period if world > 1 else None, "overlap": overlap,
                          "value": rate, "unit": UNIT, "single_gpu_value": one if world > 1 else rate,
                          "efficiency": rate / (world * one) if one else 1.0}
    rate, k, period, overlap = timed(lambda: configs.cfg4(mb), world)
    one = single(lambda: configs.cfg4(mb))
    out["cfg4_strong"] = {"num_x": 1 << 24, "levels": 6, "ranks": world, "tile_steps": k,
                          "exchange_period": period if world > 1 else None, "overlap": overlap,
                          "value": rate, "unit": UNIT, "single_gpu_value": one if world > 1 else rate,
                          "efficiency": rate / (world * one) if one else 1.0}
    sweep = []
    for p in (1, 4, 16, 64):
        kk = min(p, 4)
        rate, k, period, overlap = timed(lambda: configs.cfg5(mb, gpus=world), world, tile_steps=kk,
                                         period=p if world > 1 else None)
        one = single(lambda: configs.cfg5(mb, gpus=1), tile_steps=kk)
        per_rank = rate / world
        sweep.append({"exchange_period": p, "tile_steps": k, "overlap": overlap, "value": rate,
                      "per_rank_value": per_rank, "single_domain_value": one if world > 1 else per_rank,
                      "efficiency": per_rank / one if one else 1.0})
    out["cfg5_weak"] = {"num_x_per_rank": 1 << 22, "levels": 6, "ranks": world, "unit": UNIT, "sweep": sweep}
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("mine", "reference"), default="mine")
    ap.add_argument("--tile-steps", type=int, default=None)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-n-level", action="store_true", help="skip the N = 3 / N = 6 samples")
    ap.add_argument("--no-scaling-samples", action="store_true", help="skip the cfg4 / cfg5 multi-GPU samples")
    args = ap.parse_args(argv)
    world, rank, local = dist_env()
    if args.gpus != world:
        # one process per GPU: the driver launches --gpus N under torchrun
        if world == 1 and args.gpus > 1:
            print(f"bench.py: --gpus {args.gpus} needs torchrun --nproc-per-node {args.gpus}; "
                  "running the 1-GPU workload", file=sys.stderr)
        args.gpus = world
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_mine(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
