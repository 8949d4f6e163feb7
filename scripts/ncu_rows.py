"""Key metrics of every kernel launch in an ncu report (one line per launch)."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
idx = [h.index(k) for k in want if k in h]
for r in rows[2:]:
    print(" | ".join(f"{h[i].split('.')[0]}={r[i]}{u[i] if u[i] not in ('', 'none') else ''}" for i in idx))
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("   stalls:", ", ".join(f"{k} {x / tot * 100:.1f}%" for x, k in sorted(st, reverse=True)[:8]))
