#!/usr/bin/env python
"""Summarize an ncu --set full report into a small JSON (committed under profiles/).

    python profiles/summarize_ncu.py gpurun_out/k1_v5.ncu-rep --elements 268435456 \
        --algo-bytes-per-element 16.3125 > profiles/r01/k1_v5.json
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers_per_thread",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "pipe_tensor_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return float(val) * scale if scale else float(val)


def to_seconds(val, unit):
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3}.get(unit)
    return float(val) * scale if scale else float(val)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--elements", type=float, default=None)
    ap.add_argument("--algo-bytes-per-element", type=float, default=None)
    ap.add_argument("--kernel", default=None, help="substring of the kernel name to keep")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "")
        if a.kernel and a.kernel not in name:
            continue
        s = {"kernel": name[:160]}
        for k, short in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                v = d[k].replace(",", "")
                if short in ("dram_read", "dram_write"):
                    s[short + "_bytes"] = to_bytes(v, u[k])
                elif short == "duration":
                    s["duration_s"] = to_seconds(v, u[k])
                else:
                    try:
                        s[short] = float(v)
                    except ValueError:
                        s[short] = v
        stalls = {}
        for k in head:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(d[k])
                except ValueError:
                    pass
        s["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1])[:6])
        if "dram_read_bytes" in s and "duration_s" in s:
            s["dram_gbs"] = (s["dram_read_bytes"] + s["dram_write_bytes"]) / s["duration_s"] / 1e9
        if a.elements:
            s["elements"] = a.elements
            if "dram_read_bytes" in s:
                s["dram_bytes_per_element"] = (s["dram_read_bytes"] + s["dram_write_bytes"]) / a.elements
            if "warp_instructions" in s:
                s["lane_instructions_per_element"] = 32 * s["warp_instructions"] / a.elements
            if a.algo_bytes_per_element and "duration_s" in s:
                s["algorithmic_gbs"] = a.algo_bytes_per_element * a.elements / s["duration_s"] / 1e9
        out.append(s)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
