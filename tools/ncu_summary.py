"""Summarise one kernel of an .ncu-rep: key metrics, instruction mix and the
hottest SASS lines (by warp-stall samples).  Usage:
    python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX [top_n]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    det = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv", "-k",
                                          "regex:" + kre))))
    hdr = det[0]
    want = ("Duration", "Executed Instructions", "Registers Per Thread", "Achieved Occupancy",
            "Issue Slots Busy", "Executed Ipc Active", "DRAM Throughput", "L1/TEX Hit Rate",
            "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
            "Memory Throughput", "Compute (SM) Throughput")
    for r in det[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in want:
            print(f'{d["Metric Name"]:36s} {d["Metric Value"]:>14s} {d.get("Metric Unit", "")}')
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                           "--print-source", "sass", "-k", "regex:" + kre))))
    h = rows[1]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    st = h.index("Warp Stall Sampling (All Samples)")
    op, stall, tot, lines = Counter(), Counter(), 0, []
    for r in rows[2:]:
        try:
            n = int(r[ie] or 0)
            sm = int(r[st] or 0)
        except (ValueError, IndexError):
            continue
        s = r[src].strip()
        parts = s.split()
        mn = parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (
            parts[0] if parts else "")
        mn = mn.split(".")[0]
        op[mn] += n
        stall[mn] += sm
        tot += n
        lines.append((sm, n, r[0], s[:80]))
    tst = sum(stall.values()) or 1
    print(f"\ninstructions {tot}")
    for k, v in op.most_common(18):
        print(f"  {k:10s} {v / tot * 100:5.1f}%  stalls {stall[k] / tst * 100:5.1f}%")
    print("\nhottest lines (stall samples, executed, address, sass)")
    for sm, n, a, s in sorted(lines, reverse=True)[:top]:
        print(f"  {sm:6d} {n:10d} {a} {s}")


if __name__ == "__main__":
    main()
