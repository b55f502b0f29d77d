"""Copy one measurement pass (tools/measure_r02.sh -> gpurun_out/r02final/)
into the tracked profiles/ files: bench lines, the launch list and its
summary, the blend kernels' traffic/counter capture, the ncu summary of the
full capture.  Usage: python tools/refresh_profiles.py [SRC_DIR] [TAG]"""
import csv
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SRC = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out" / "r02final"
TAG = sys.argv[2] if len(sys.argv) > 2 else "r02"
PROF = ROOT / "profiles"

TRAFFIC_METRICS = {
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__time_duration.sum": "us",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp_inst",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
}


def bench_lines():
    n = 0
    for f in sorted(SRC.glob("bench_*.json")):
        txt = f.read_text().strip().splitlines()
        if not txt:
            continue
        json.loads(txt[-1])  # (a valid line, or fail loudly)
        (PROF / f"{TAG}_{f.name}").write_text(txt[-1] + "\n")
        n += 1
    return n


def launches():
    src = SRC / "launches.csv"
    if not src.exists():
        return
    shutil.copy(src, PROF / f"{TAG}_launches_c3_softplus.csv")
    table = subprocess.run([sys.executable, str(ROOT / "tools" / "launch_table.py"), str(src), "20"],
                           capture_output=True, text=True, check=True).stdout
    head = (f"# {TAG} — ncu launch list, C3 softplus fwd+bwd (tools/measure_r02.sh)\n\n"
            "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv "
            "python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline` (every pass of the "
            "run: warm-up, timed, phase-timing and counting passes; cold-cache and serialised — "
            f"compare shares, not absolutes). Raw: `{TAG}_launches_c3_softplus.csv`.\n\n")
    (PROF / f"{TAG}_launches_summary.md").write_text(head + table)


def traffic():
    src = SRC / "ncu_traffic.csv"
    if not src.exists():
        return
    lines = [ln for ln in src.read_text().splitlines() if ln.startswith('"')]
    per = defaultdict(lambda: defaultdict(list))
    for row in csv.DictReader(lines):
        name = row["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("nxs::", "")
        key = TRAFFIC_METRICS.get(row["Metric Name"])
        if key is None:
            continue
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "")
        if key == "us":
            v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
        per[name][key].append(v)
    out = {}
    for k, d in per.items():
        out[k] = {m: round(sum(v) / len(v), 2) if m not in ("dram_read_bytes", "dram_write_bytes",
                                                            "warp_instructions")
                  else int(sum(v) / len(v)) for m, v in d.items()}
    path = PROF / f"{TAG}_blend_traffic.json"
    old = json.loads(path.read_text()) if path.exists() else {}
    old["per_step"] = out
    old["source"] = f"{src.relative_to(ROOT)} (tools/measure_r02.sh), mean over the captured launches"
    path.write_text(json.dumps(old, indent=1) + "\n")


def ncu_summary():
    rep = SRC / "blend_full.ncu-rep"
    if not rep.exists():
        return
    parts = [f"# {TAG} — ncu --set full of the Mode G blend kernels at C3 softplus "
             f"(tools/measure_r02.sh; report {rep.relative_to(ROOT)})\n"]
    for k in ("^k_blend_fwd$", "^k_blend_bwd$"):
        s = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep), k, "20"],
                           capture_output=True, text=True).stdout
        lines = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_lines.py"), str(rep), k, "25"],
                               capture_output=True, text=True).stdout
        parts.append(f"## {k}\n{s}\n### hottest source lines\n{lines}")
    (PROF / f"{TAG}_blend_ncu_summary.txt").write_text("\n".join(parts))


if __name__ == "__main__":
    print("bench lines:", bench_lines())
    launches()
    traffic()
    ncu_summary()
    print("profiles refreshed from", SRC)
