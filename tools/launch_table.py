"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
into a markdown table of per-kernel total time, share and launch count.

    python tools/launch_table.py gpurun_out/launches.csv [top_n]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    tot, cnt = defaultdict(float), defaultdict(int)
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0]
        if len(name) > 60:
            name = name[:60]
        us = float(row["Metric Value"].replace(",", ""))
        if row.get("Metric Unit") == "ns":
            us /= 1e3
        elif row.get("Metric Unit") == "ms":
            us *= 1e3
        tot[name] += us
        cnt[name] += 1
    total = sum(tot.values())
    print("| kernel | total us | share | launches |")
    print("|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"| `{k}` | {v:.1f} | {100 * v / total:.1f}% | {cnt[k]} |")
    print(f"\nall kernels: {total:.1f} us over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()
