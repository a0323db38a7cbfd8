"""Key metrics per kernel from an ncu report (raw page).  usage: python tools/ncu_summary.py rep [regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wf %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank confl"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wf"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld sectors"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "st:long_sb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "st:short_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "st:barrier"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "st:mio"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "st:wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "st:math"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "st:lg"),
]
ki = hdr.index("Kernel Name")
for r in rows[2:]:
    name = r[ki]
    if kre and not kre.search(name):
        continue
    parts = []
    for m, short in WANT:
        if m in hdr:
            i = hdr.index(m)
            parts.append(f"{short}={r[i]}{units[i] if units[i] in ('us','ms','Gbyte','Mbyte','%') else ''}")
    print(name[:60], "\n   ", "  ".join(parts))
