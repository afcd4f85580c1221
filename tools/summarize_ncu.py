"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py --tag r1 gpurun_out/prof_cfg2_r1b.ncu-rep:cfg2_k24 ... \
        --launches gpurun_out/launches_cfg2_r1b.csv

Writes profiles/ncu_summary.json (per workload: duration, DRAM bytes per
launch, FP64 pipe %, occupancy, registers, top stall reasons, instruction
mix per cell-step) and profiles/<tag>_ncu.md.
"""

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CELL_STEPS = {  # cell-steps per profiled launch (tools/prof_step.py defaults: k = 64 / 16 / 4)
    "cfg2": (1 << 22) * 64, "cfg3": (1 << 23) * 16, "cfg4": (1 << 24) * 4, "cfg5": (1 << 22) * 4,
}


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv(rep, "raw")
    hdr, vals = rows[0], rows[2]
    return dict(zip(hdr, vals))


def f(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def instruction_mix(rep, cell_steps):
    rows = ncu_csv(rep, "source", ("--print-source=sass",))
    hdr = rows[1]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    mix = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ei or not r[ei].isdigit():
            continue
        op = r[si].strip().split()
        if not op:
            continue
        m = op[1] if op[0].startswith("@") else op[0]
        mix[m.split(".")[0]] += int(r[ei])
    total = sum(mix.values())
    per = {k: round(v * 32 / cell_steps, 1) for k, v in mix.most_common(12)}
    fp64 = sum(v for k, v in mix.items() if k in ("DFMA", "DMUL", "DADD")) * 32 / cell_steps
    return per, round(total * 32 / cell_steps, 1), round(fp64, 1)


def summarize(rep, key):
    d = raw_metrics(rep)
    cfg = key.split("_")[0]
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
            stalls.append((f(d, k), name))
    stalls.sort(reverse=True)
    dur_unit = "ms"
    dram_r, dram_w = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
    out = {
        "kernel": d.get("Kernel Name", "?")[:120],
        "duration_us": f(d, "gpu__time_duration.sum") * (1000.0 if dur_unit == "ms" else 1.0),
        "registers": f(d, "launch__registers_per_thread"),
        "fp64_pipe_pct": f(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f(d, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "top_stalls": [(n, round(v, 3)) for v, n in stalls[:6]],
    }
    # units: ncu raw reports dram bytes in the unit row; normalise to bytes per launch
    rows = ncu_csv(rep, "raw")
    units = dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out["dram_read_bytes"] = dram_r * scale.get(units.get("dram__bytes_read.sum"), 1)
    out["dram_write_bytes"] = dram_w * scale.get(units.get("dram__bytes_write.sum"), 1)
    out["dram_bytes_per_launch"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    tu = units.get("gpu__time_duration.sum", "ns")
    out["duration_us"] = f(d, "gpu__time_duration.sum") * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                                           "msecond": 1e3, "nsecond": 1e-3}.get(tu, 1.0)
    if cfg in CELL_STEPS:
        try:
            per, total, fp64 = instruction_mix(rep, CELL_STEPS[cfg])
            out["instr_per_cell_step"] = total
            out["fp64_instr_per_cell_step"] = fp64
            out["mix_per_cell_step"] = per
        except Exception as exc:  # source page optional
            out["mix_error"] = str(exc)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": round(tot[k], 1), "share_pct": round(100 * tot[k] / total, 2),
             "avg_us": round(tot[k] / cnt[k], 2)} for k in sorted(tot, key=lambda k: -tot[k])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+", help="path.ncu-rep:key[:cell_steps of the profiled launch]")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    summ_path = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    md = [f"# ncu summary ({a.tag})\n"]
    for spec in a.reports:
        parts = spec.split(":")
        rep, key = parts[0], parts[1]
        if len(parts) > 2:
            CELL_STEPS[key.split("_")[0]] = int(float(parts[2]))
        s = summarize(rep, key)
        summ[key] = s
        md.append(f"## {key}\n\n```\n{json.dumps(s, indent=1)}\n```\n")
    if a.launches:
        ls = launches(a.launches)
        summ[f"launch_list_{a.tag}"] = ls
        md.append("## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n")
        md.append("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
        md += [f"| {x['kernel']} | {x['launches']} | {x['total_us']} | {x['share_pct']}% | {x['avg_us']} |" for x in ls]
    summ_path.write_text(json.dumps(summ, indent=1))
    (ROOT / "profiles" / f"{a.tag}_ncu.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
