"""Per-kernel stall-reason breakdown, active threads per warp instruction and
warp instructions of an .ncu-rep (the VERDICT r01 item 3a figures), and —
given the algorithmic flops of one launch — instructions per algorithmic
flop.  Usage: python tools/ncu_stalls.py REPORT KERNEL_REGEX [flops_per_launch]"""
import csv
import io
import subprocess
import sys


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    flops = float(sys.argv[3]) if len(sys.argv) > 3 else None
    det = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv", "-k",
                                          "regex:" + kre))))
    hdr = det[0]
    vals = {}
    for r in det[1:]:
        d = dict(zip(hdr, r))
        vals.setdefault(d["Metric Name"], d["Metric Value"])
    inst = float(vals.get("Executed Instructions", "0").replace(",", ""))
    thr = vals.get("Avg. Active Threads Per Warp", "?")
    print(f"duration {vals.get('Duration', '?')} us, warp instructions {inst:.0f}, "
          f"active threads per warp instruction {thr}, issue slots busy "
          f"{vals.get('Issue Slots Busy', '?')} %")
    if flops:
        print(f"algorithmic flops {flops:.4g}: warp instructions per flop {inst / flops:.3f}, "
              f"thread instructions per flop {inst * float(thr) / flops:.2f}")
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                           "--print-source", "sass", "-k", "regex:" + kre))))
    h = rows[1]
    idx = {c: i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c}
    tot = {c: 0 for c in idx}
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        for c, i in idx.items():
            try:
                tot[c] += int(r[i] or 0)
            except ValueError:
                pass
    s = sum(tot.values()) or 1
    print("stall reasons (share of warp-state samples):")
    for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
        print(f"  {c[6:]:22s} {100 * v / s:5.1f} %")


if __name__ == "__main__":
    main()
