"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ci, cs, ce = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[cs]), r[ci], r[ce], r[0]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
for v, src, ex, addr in sorted(data, reverse=True)[:top]:
    print("%5.1f%%  %10s  %s" % (100 * v / tot, ex, src[:100]))
