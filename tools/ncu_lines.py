"""Aggregate an .ncu-rep kernel's SASS metrics per CUDA source line
(--print-source cuda,sass).  Usage: python tools/ncu_lines.py REP REGEX [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(lambda: [0, 0, ""])
cur_file = None
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    # cuda rows have a line number in col 0; sass rows have '' in col 0?
    if r[0].strip():
        cur_line = (cur_file, r[0], r[1][:70])
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    if cur_line and not r[0].strip():
        a = agg[cur_line]
        a[0] += ie
        a[1] += st
tot_i = sum(a[0] for a in agg.values()) or 1
tot_s = sum(a[1] for a in agg.values()) or 1
print(f"instr {tot_i}  stall samples {tot_s}")
for k, (ie, st, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ie / tot_i * 100:5.1f}% instr {st / tot_s * 100:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
