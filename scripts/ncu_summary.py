"""Summarise an ncu report: key pipe metrics, stall reasons, top stalled SASS lines, opcode mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]
for i, k in enumerate(h):
    if k in want:
        print(f"{k:90s} {u[i]:>8s} {v[i]}")
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st)
print("stalls:", ", ".join(f"{k} {x / tot * 100:.1f}%" for x, k in sorted(st, reverse=True)[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
hh = srows[1]
iS = hh.index("Warp Stall Sampling (All Samples)")
iE = hh.index("Instructions Executed")
# first kernel only: a multi-kernel report repeats the header row before each kernel's source table
data = []
for r in srows[2:]:
    if len(r) <= max(iS, iE) or r[iS] == "Warp Stall Sampling (All Samples)":
        break
    data.append(r)
tots = sum(float(r[iS] or 0) for r in data)
print("top stalled instructions:")
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {r[0][-5:]} {float(r[iS]) / tots * 100:5.1f}% exec {r[iE]:>12s}  {r[1][:80]}")
c = collections.Counter()
for r in data:
    ins = r[1].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    c[ins.split()[0] if ins else ""] += int(r[iE] or 0)
t = sum(c.values())
print("opcode mix (warp instr):", t)
print("  " + ", ".join(f"{op} {n / t * 100:.1f}%" for op, n in c.most_common(16)))
