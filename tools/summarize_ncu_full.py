"""Condense `ncu --set full` reports into a small JSON (per kernel launch): duration, DRAM
bytes, SOL throughputs, the tcgen05 tensor-pipe figures, occupancy, and the top warp-stall
reasons.

    python tools/summarize_ncu_full.py out.json rep1.ncu-rep [rep2.ncu-rep ...] [--flops name=GFLOP ...]

Tensor-core evidence on sm_100a comes from the UTC (tcgen05) counters, not the legacy HMMA
pipe ones: `sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off` (bf16 dense MMA
ops: % of ncu's peak and ops/s) and `sm__pipe_tc_cycles_active` (cycles the tcgen05 pipe is
busy).  `--flops kernel_substring=GFLOP` adds the algorithmic FLOPs of a launch, so the JSON
carries achieved TFLOP/s (algorithmic / duration) next to ncu's own op rate and the DRAM
bytes next to the algorithmic bytes.
"""
import csv
import io
import json
import subprocess
import sys

UTC = "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off"
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    UTC + ".sum.pct_of_peak_sustained_elapsed": "utc_bf16_pct_of_peak",
    UTC + ".sum.per_second": "utc_bf16_ops_per_ns",
    UTC + ".sum": "utc_bf16_ops",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc_pipe_active_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}
STALL = "smsp__average_warps_issue_stalled_"


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main(argv):
    out_path, reps, flops = argv[0], [], {}
    i = 1
    while i < len(argv):
        if argv[i] == "--flops":
            k, v = argv[i + 1].split("=")
            flops[k] = float(v)
            i += 2
        else:
            reps.append(argv[i])
            i += 1
    out = []
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            d = {"report": rep.split("/")[-1], "kernel": name[:140]}
            for k, short in KEYS.items():
                if k in hdr:
                    j = hdr.index(k)
                    d[short] = r[j] + ("" if not units[j] else " " + units[j])
            stalls = {h[len(STALL):].replace("_per_issue_active.ratio", ""): to_num(r[j])
                      for j, h in enumerate(hdr) if h.startswith(STALL) and h.endswith("_per_issue_active.ratio")}
            top = sorted(((v, k) for k, v in stalls.items() if v), reverse=True)[:6]
            d["top_stalls_per_issue"] = {k: round(v, 3) for v, k in top}
            dur_ns = to_num(r[hdr.index("gpu__time_duration.sum")]) if "gpu__time_duration.sum" in hdr else None
            if dur_ns is not None and units[hdr.index("gpu__time_duration.sum")] in ("usecond", "us"):
                dur_ns *= 1e3
            elif dur_ns is not None and units[hdr.index("gpu__time_duration.sum")] in ("msecond", "ms"):
                dur_ns *= 1e6
            ops = to_num(r[hdr.index(UTC + ".sum")]) if UTC + ".sum" in hdr else None
            if ops and dur_ns:
                d["utc_bf16_tflops_executed"] = round(ops / dur_ns * 1e-3, 1)  # MMA ops actually issued / time
            for key, gflop in flops.items():
                if key in name and dur_ns:
                    d["algorithmic_gflop"] = gflop
                    d["achieved_tflops"] = round(gflop / dur_ns * 1e-3 * 1e3, 1)
            out.append(d)
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps(out, indent=1)[:4000])


if __name__ == "__main__":
    main(sys.argv[1:])
