"""Summarise an ncu launch list (gpu__time_duration.sum [+ dram__bytes_{read,write}.sum]).

    python tools/summarize_launches.py gpurun_out/launches.csv --steps 2 --out profiles/r01_launches_summary.json

Groups launches by kernel (template) name; prints each kernel's share of the total device
time (ncu times are cold-cache and serialised: compare shares, not absolutes) and its DRAM
bytes per launch.  Also writes profiles/traffic.json: DRAM bytes per launch for the bench's
dominant kernel class (ice_conv_wgrad = conv_gemm<.., WgradProb> + hwgrad_kernel).
"""
import argparse
import collections
import csv
import json
import os

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--steps", type=int, default=0, help="0: count head_ce_kernel launches (one per step)")
ap.add_argument("--out", default=None)
ap.add_argument("--traffic", default=None)
ap.add_argument("--after", default="adam_kernel",
                help="count only launches after the first launch whose name contains this (skips setup + step 1)")
ap.add_argument("--al-tiles", type=int, default=1024, help="tiles per autolabel256 launch (bench --corpus)")
a = ap.parse_args()

launch = collections.OrderedDict()
for r in csv.reader(open(a.csv)):
    if len(r) < 15 or not r[0].isdigit():
        continue
    key = (r[0], r[4])
    d = launch.setdefault(key, {"name": r[4], "ns": 0.0, "rd": 0.0, "wr": 0.0})
    unit, val = r[13], float(r[14].replace(",", "") or 0)
    scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    if r[12] == "gpu__time_duration.sum":
        d["ns"] = val * scale
    elif r[12] == "dram__bytes_read.sum":
        d["rd"] = val * scale
    elif r[12] == "dram__bytes_write.sum":
        d["wr"] = val * scale


def short(n):
    n = n.replace("<unnamed>::", "").replace("void ", "")
    return n.split("(")[0] if "(" in n and "<" not in n.split("(")[0][-2:] else n[: n.find(">(") + 1] if ">(" in n else n[:60]


if a.after:
    names = [d["name"] for d in launch.values()]
    first = next((i for i, n in enumerate(names) if a.after in n), None)
    if first is not None:
        launch = collections.OrderedDict(list(launch.items())[first + 1:])
if a.steps <= 0:
    a.steps = max(1, sum(1 for d in launch.values() if "head_ce_kernel" in d["name"]))
agg = collections.OrderedDict()
for d in launch.values():
    k = short(d["name"])
    g = agg.setdefault(k, {"launches": 0, "ns": 0.0, "dram_bytes": 0.0})
    g["launches"] += 1
    g["ns"] += d["ns"]
    g["dram_bytes"] += d["rd"] + d["wr"]
tot = sum(g["ns"] for g in agg.values()) or 1.0
rows = []
for k, g in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
    rows.append({"kernel": k, "launches_per_step": g["launches"] / a.steps, "ms_per_step": g["ns"] / 1e6 / a.steps,
                 "share": g["ns"] / tot, "dram_bytes_per_launch": g["dram_bytes"] / g["launches"]})
    print(f"{g['launches'] / a.steps:6.1f} x {g['ns'] / 1e6 / a.steps:8.3f} ms {100 * g['ns'] / tot:5.1f}%  "
          f"{g['dram_bytes'] / g['launches'] / 1e6:9.1f} MB/launch  {k}")
if a.out:
    json.dump({"source": a.csv, "steps": a.steps, "after_first": a.after, "kernels": rows}, open(a.out, "w"), indent=1)
fams = {"ice_conv_wgrad": lambda k: "WgradProb" in k or "hwgrad_kernel" in k,
        "ice_conv_dgrad": lambda k: "DgradProb" in k,
        "ice_conv_fprop": lambda k: "FpropProb" in k}
if a.traffic and any(g["dram_bytes"] for g in agg.values()):
    old = json.load(open(a.traffic)) if os.path.exists(a.traffic) else {}
    for fam, sel in fams.items():
        gs = [g for k, g in agg.items() if sel(k)]
        n = sum(g["launches"] for g in gs)
        if n:
            old[fam] = round(sum(g["dram_bytes"] for g in gs) / n)
    old["_note"] = ("DRAM read+write bytes per launch, averaged over each convolution family's kernels of the warm "
                    "steps (FpropProb / DgradProb / WgradProb + hwgrad template instances; the halving conv's "
                    "launches are included in their family), from " + a.csv)
    al = [g for k, g in agg.items() if "autolabel256" in k]
    if al and al[0]["dram_bytes"]:
        old["ice_autolabel_bytes_per_tile"] = round(al[0]["dram_bytes"] / al[0]["launches"] / a.al_tiles)
        old["_note_autolabel"] = (f"fastk::autolabel256_kernel over the {a.al_tiles}-tile corpus (one launch), DRAM "
                                  "read+write / tiles; algorithmic 458,752 B/tile")
    json.dump(old, open(a.traffic, "w"), indent=1)
    print("traffic:", old)
