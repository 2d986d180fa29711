"""Attribute ncu warp-stall samples / executed instructions of one kernel to source lines.

    python tools/ncu_lines.py <report.ncu-rep> <kernel regex> <cubin> [--top 40]

ncu's SASS page (--page source --print-source sass) lists runtime addresses; offsets from
the function start match the cubin, whose line table nvdisasm -g prints.
"""
import argparse
import collections
import csv
import io
import re
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel")
ap.add_argument("cubin")
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()

out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + a.kernel], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
name = rows[0][1]
hdr = rows[1]
rows = [r for r in rows[2:] if len(r) == len(hdr)]
i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
num = lambda v: int(v) if v.strip().isdigit() else 0
base = int(rows[0][0], 16)

# mangled name from the cubin whose SASS length matches
dis = subprocess.run(["nvdisasm", "-g", a.cubin], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*\.text\.", dis)
best = None
for f in funcs:
    fname = f.split(":", 1)[0].strip()
    if not re.search(a.kernel, fname):
        continue
    cur = None
    lo = {}
    for ln in f.splitlines():
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m and "//##" in ln:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur is not None:
            lo[int(m.group(1), 16)] = cur
    n_inst = (max(lo) // 16 + 1) if lo else 0
    # the instantiation whose SASS length matches the profiled kernel's
    score = abs(n_inst - len(rows))
    if best is None or score < best[0]:
        best = (score, lo, fname)
line_of = best[1] if best else {}
agg = collections.Counter()
inst = collections.Counter()
stall_cols = [(h, i) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
reasons = collections.defaultdict(collections.Counter)
total_reasons = collections.Counter()
for r in rows:
    off = int(r[0], 16) - base
    ln = line_of.get(off, "?")
    agg[ln] += num(r[i_s])
    inst[ln] += num(r[i_e])
    for h, i in stall_cols:
        reasons[ln][h[6:]] += num(r[i])
        total_reasons[h[6:]] += num(r[i])
tot = sum(agg.values()) or 1
itot = sum(inst.values()) or 1
print(f"{name[:90]}\n total samples {tot}, warp-instructions {itot}, mapped lines {len(line_of)}")
rt = sum(total_reasons.values()) or 1
print(" stall reasons:", ", ".join(f"{k} {100 * v / rt:.1f}%" for k, v in total_reasons.most_common(8)))
for ln, v in agg.most_common(a.top):
    top = ", ".join(f"{k} {100 * c / max(1, sum(reasons[ln].values())):.0f}%" for k, c in reasons[ln].most_common(3))
    print(f"  {ln:28s}: {100 * v / tot:5.1f}% stalls  {100 * inst[ln] / itot:5.1f}% inst  [{top}]")
