"""Summarise an ncu report into profiles/ (details page + key raw metrics).

    python tools/ncu_summary.py gpurun_out/r1_c4_star.ncu-rep profiles/r1_c4_star
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def main(rep: str, out: str) -> None:
    details = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(out + "_details.txt", "w").write(details)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    lines = ["metric,unit,value"]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    lines.append(f"Kernel Name,,\"{name}\"")
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k},{units[i]},{vals[i]}")
    stalls = []
    for i, h in enumerate(hdr):
        if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), h))
            except ValueError:
                pass
    for v, h in sorted(stalls, reverse=True)[:8]:
        lines.append(f"{h},ratio,{v}")
    open(out + "_metrics.csv", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
