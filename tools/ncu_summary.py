#!/usr/bin/env python
"""Summarise one kernel of an `ncu --set full` report into the JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/<tag>/prof_attn_osp.ncu-rep --command "..." > profiles/<round>/x.json
"""
import argparse
import csv
import io
import json
import subprocess

FIELDS = {
    "gpu_time_ms": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
    "fma_pipe_pct_active": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct_active": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smem_tc_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "registers_per_thread": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "cluster_x": "launch__cluster_dim_x",
    "stall_long_scoreboard": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "stall_barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "stall_math_throttle": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "stall_mio_throttle": "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "stall_short_scoreboard": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_not_selected": "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--command", default="")
    ap.add_argument("--algorithmic-bytes-MB", type=float, default=None)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", ""), "command": args.command}
        for k, m in FIELDS.items():
            if m not in d:
                continue
            v = d[m].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                rec[k] = v
                continue
            unit = u.get(m, "")
            if k.endswith("_MB"):
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}.get(unit, 1.0)
            if k == "gpu_time_ms":
                x = x * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1.0)
            if k == "sm_clock_ghz":
                x = x * {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}.get(unit, 1.0)
            rec[k] = x
        if args.algorithmic_bytes_MB:
            rec["algorithmic_bytes_MB"] = args.algorithmic_bytes_MB
        res.append(rec)
    print(json.dumps(res[0] if len(res) == 1 else res, indent=1))


if __name__ == "__main__":
    main()
