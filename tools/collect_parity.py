"""Collect the per-case parity reports the GPU tests wrote
(gpurun_out/parity/<group>/<case>.json) into profiles/.
usage: python tools/collect_parity.py TAG   ->  profiles/TAG_parity_c3.json,
                                                profiles/TAG_parity_all.json"""
import json
import sys
from pathlib import Path

root = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = root / "gpurun_out" / "parity"
allrep = {}
for f in sorted(src.glob("*/*.json")):
    allrep.setdefault(f.parent.name, {})[f.stem] = json.loads(f.read_text())
keys = ("total", "strict", "strict_nc", "strict_budget", "budget_basis", "mass", "mass_c")
summary = {g: {c: {k: r.get(k) for k in keys} for c, r in cases.items()}
           for g, cases in allrep.items()}
c3 = allrep.get("c3", {})
out = {"protocol": "tests/test_gpu_parity_c3.py: C3 (1M Gaussians seed 5, 1920x1080), 256 random "
                   "pixels per case, third call on one reused view (device-sized first phase, "
                   "CUDA graph); tolerance 1e-6 + 1e-5|ref| (strict) and 1e-6 + 1e-5 S_c "
                   "(componentwise absolute-evaluation scale, the gate)",
       "cases": c3}
(root / "profiles" / f"{tag}_parity_c3.json").write_text(json.dumps(out, indent=1))
(root / "profiles" / f"{tag}_parity_all.json").write_text(json.dumps(summary, indent=1))
for g, cases in summary.items():
    for c, r in cases.items():
        print(f"{g:12s} {c:28s} strict {r['strict']:4d} nc {r['strict_nc']:4d} "
              f"budget {r['strict_budget']:4d} mass_c {r['mass_c']} normwise {r['mass']}")
