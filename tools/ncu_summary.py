"""Summarise an ncu report (raw page) into the metrics the roofline needs.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "time_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "ffma_thread_inst": "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "fadd_thread_inst": "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, m in WANT.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    f = float(v)
                    f *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "usecond": 1e3,
                          "ms": 1e6, "msecond": 1e6, "s": 1e9, "GHz": 1e9, "MHz": 1e6}.get(u, 1.0)
                    d[k] = f
                except ValueError:
                    d[k] = v
        if "dram_read" in d and "dram_write" in d and "time_ns" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            d["dram_gbs"] = d["dram_bytes"] / d["time_ns"]
        out.append(d)
    return out


if __name__ == "__main__":
    res = {p: summarise(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
