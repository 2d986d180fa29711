"""Condense `ncu --set full` reports into a small JSON (per kernel launch): duration, DRAM
bytes, SOL throughputs, tensor-pipe activity, occupancy, and the top warp-stall reasons.

    python tools/summarize_ncu_full.py out.json rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}
out = []
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"report": rep.split("/")[-1], "kernel": r[hdr.index("Kernel Name")][:120]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                d[name] = r[i] + ("" if not units[i] else " " + units[i])
        stalls = {h[len("smsp__average_warp_latency_issue_stalled_"):].split(".")[0]: r[i]
                  for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  and h.endswith(".ratio")}
        try:
            top = sorted(((float(v), k) for k, v in stalls.items() if v), reverse=True)[:5]
            d["top_stalls_cycles_per_inst"] = {k: round(v, 2) for v, k in top}
        except ValueError:
            pass
        out.append(d)
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
