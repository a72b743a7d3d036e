"""Print the counters the DESIGN/profiles summaries cite from an ncu report (raw page)."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
data = rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_active.min",
        "sm__cycles_elapsed.max", "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__lsu_writeback_active.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_lg.sum", "smsp__inst_executed_op_shared_ld.sum"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s}", [r[i][:14] for r in data])
for h in hdr:
    m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio$", h)
    if m:
        i = hdr.index(h)
        v = [float(r[i] or 0) for r in data]
        if max(v) > 0.1:
            print(f"  stall {m.group(1):40s}", ["%.2f" % x for x in v])
