"""Compare two launch-list summaries (tools/summarize_launches.py --out) kernel by kernel.

    python tools/cmp_launches.py profiles/r01_launches_summary.json /tmp/new.json
"""
import json
import sys

a = json.load(open(sys.argv[1]))
b = json.load(open(sys.argv[2]))
A = {k["kernel"]: k for k in a["kernels"]}
B = {k["kernel"]: k for k in b["kernels"]}
keys = sorted(set(A) | set(B), key=lambda k: -(B.get(k, {}).get("ms_per_step", 0)))
ta = sum(k["ms_per_step"] for k in a["kernels"])
tb = sum(k["ms_per_step"] for k in b["kernels"])
print(f"total {ta:.3f} -> {tb:.3f} ms/step")
for k in keys:
    x, y = A.get(k, {}), B.get(k, {})
    print(f"{k[:62]:62s} {x.get('launches_per_step', 0):5.1f} {x.get('ms_per_step', 0):7.3f}  ->"
          f" {y.get('launches_per_step', 0):5.1f} {y.get('ms_per_step', 0):7.3f}")
