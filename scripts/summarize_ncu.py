"""Summarize ncu outputs from gpurun_out/ into profiles/<round>_*.{md,json}.

  python scripts/summarize_ncu.py r01
Reads gpurun_out/launches.csv (gpu__time_duration launch list) and the
--set full reports gpurun_out/prof_<kernel>.ncu-rep (via `ncu -i`).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("NCU_OUT") or os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def launch_shares(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("::")[-1]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        tot[name] += ns
        cnt[name] += 1
    all_ns = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_ms": tot[k] / 1e6, "share": tot[k] / all_ns}
            for k in sorted(tot, key=lambda k: -tot[k])]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in METRICS or "issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                d[h] = (float(v.replace(",", "")), u)
            except ValueError:
                pass
    return d


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    summary = {"round": rnd}
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        summary["launch_list"] = launch_shares(os.path.join(OUT, "launches.csv"))
    kernels = {}
    for k in ("fnv_kernel", "pack_kernel", "replay_kernel", "fnv_witness_tc_kernel", "fnv_witness_kernel", "scope_kernel"):
        rep = os.path.join(OUT, f"prof_{k}.ncu-rep")
        if os.path.exists(rep):
            m = raw_metrics(rep)
            stalls = sorted(((h, v[0]) for h, v in m.items() if "issue_stalled" in h), key=lambda x: -x[1])[:6]
            kernels[k] = {h: v for h, v in m.items() if "issue_stalled" not in h}
            kernels[k]["top_stalls"] = [(h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""), round(v, 3)) for h, v in stalls]
            if "dram__bytes_read.sum" in m:
                rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                kernels[k]["traffic_bytes"] = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
    summary["full_captures"] = kernels
    with open(os.path.join(PROF, f"{rnd}_ncu_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1, default=str)
    lines = [f"# ncu summary ({rnd})", "",
             "Command: `python bench.py --steps 2 --warmup 3 --no-cpu --no-extras` (scripts/profile.sh); "
             "launch list = `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised); "
             "full captures = `--set full --clock-control none`, one launch each.", "",
             "## Launch list: share of device time", "", "| kernel | launches | total ms | share |",
             "|---|---|---|---|"]
    for r in summary.get("launch_list", []):
        lines.append(f"| {r['kernel']} | {r['launches']} | {r['total_ms']:.3f} | {100 * r['share']:.1f}% |")
    for k, m in kernels.items():
        lines += ["", f"## {k}", "", "| metric | value |", "|---|---|"]
        for h, v in m.items():
            if h in ("top_stalls",):
                continue
            lines.append(f"| {h} | {v if not isinstance(v, tuple) else f'{v[0]:g} {v[1]}'} |")
        lines.append(f"| top stall reasons (warps per issue) | {m.get('top_stalls')} |")
    with open(os.path.join(PROF, f"{rnd}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
