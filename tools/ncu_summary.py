#!/usr/bin/env python3
"""Summarise an ncu --set full report into profiles/ncu_<workload>.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic).

  python tools/ncu_summary.py gpurun_out/prof_gemv.ncu-rep gemv [round]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_bytes.sum",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_not_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_selected_per_warp_active.pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    tag = sys.argv[3] if len(sys.argv) > 3 else "r01"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for row in data:
        rec = {"kernel": row[head.index("Kernel Name")] if "Kernel Name" in head else None}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                rec[k] = row[i]
                rec[k + ".unit"] = units[i]
        launches.append(rec)

    def val(rec, k):
        v = float(str(rec[k]).replace(",", ""))
        return v * SCALE.get(rec.get(k + ".unit", ""), 1.0)

    first = launches[0]
    traffic = val(first, "dram__bytes_read.sum") + val(first, "dram__bytes_write.sum")
    out = {
        "workload": workload,
        "round": tag,
        "source": f"ncu --set full --clock-control none ({Path(rep).name})",
        "kernel": first["kernel"],
        "duration_s": val(first, "gpu__time_duration.sum"),
        "dram_bytes_per_launch": traffic,
        "launches": launches,
    }
    dst = ROOT / "profiles" / f"ncu_{workload}.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: out[k] for k in ("workload", "kernel", "duration_s", "dram_bytes_per_launch")}))


if __name__ == "__main__":
    main()
