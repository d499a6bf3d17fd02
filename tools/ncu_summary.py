"""tools/ncu_summary.py REPORT.ncu-rep OUT.json [--elements N] [--bytes-per-element B]

Summarise an `ncu --set full` capture (one kernel per report row) into the
JSON kept under profiles/: duration, DRAM bytes and throughput, issue
utilisation, warps, registers, pipe utilisation and the stall reasons (cycles
per issued instruction).  With --elements the per-element DRAM bytes, lane
instructions and the algorithmic GB/s (B * N / duration) are added.
"""
import argparse
import csv
import io
import json
import subprocess


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--elements", type=float, default=None)
    ap.add_argument("--bytes-per-element", type=float, default=None)
    a = ap.parse_args()
    hdr, units, rows = raw_rows(a.report)
    res = []
    for r in rows:
        g = dict(zip(hdr, r))
        u = dict(zip(hdr, units))

        def val(k, scale_to=None):
            v = num(g.get(k, ""))
            if v is None:
                return None
            unit = u.get(k, "")
            mult = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
                    "nsecond": 1e-9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                    "Kbyte/block": 1e3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}
            return v * mult.get(unit, 1.0) if scale_to else v

        d = {
            "kernel": g.get("Kernel Name", "")[:160],
            "duration_s": val("gpu__time_duration.sum", True),
            "dram_read_bytes": val("dram__bytes_read.sum", True),
            "dram_write_bytes": val("dram__bytes_write.sum", True),
            "dram_pct_of_peak": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_slots_busy_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warp_instructions": val("smsp__inst_executed.sum"),
            "registers_per_thread": val("launch__registers_per_thread"),
            "shared_mem_per_block_bytes": val("launch__shared_mem_per_block_dynamic", True),
            "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "pipe_alu_pct": val("TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed"),
            "pipe_fp64_pct": val("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
            "pipe_tensor_pct": val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "lsu_wavefronts_pct": val("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            "grid": val("launch__grid_size"),
            "block": val("launch__block_size"),
            "sm_clock_hz": val("sm__cycles_elapsed.avg.per_second", True),
            "note": "ncu replay: cold caches, serialised launches -- absolute times are not bench values",
        }
        stalls = {}
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                v = num(g.get(k, ""))
                if v:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        d["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        if d["duration_s"] and d["dram_read_bytes"] is not None:
            d["dram_gbs"] = (d["dram_read_bytes"] + d["dram_write_bytes"]) / d["duration_s"] / 1e9
        if a.elements:
            d["elements"] = a.elements
            d["dram_bytes_per_element"] = (d["dram_read_bytes"] + d["dram_write_bytes"]) / a.elements
            if d["warp_instructions"]:
                d["lane_instructions_per_element"] = 32.0 * d["warp_instructions"] / a.elements
            if a.bytes_per_element and d["duration_s"]:
                d["algorithmic_gbs"] = a.bytes_per_element * a.elements / d["duration_s"] / 1e9
        res.append(d)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
