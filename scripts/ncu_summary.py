"""Summarise an ncu report (raw page + source-page stall hot spots). Usage: ncu_summary.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, val = rows[0], rows[2]
d = dict(zip(hdr, val))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = []
for h, v in zip(hdr, val):
    if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    h = rows[1]
    ia, isrc, iw = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[iw] or 0), r[ia][-5:], r[isrc][:80]))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in data) or 1
    print("top stall sites:")
    for x in sorted(data, reverse=True)[:top]:
        print(f"  {100 * x[0] / tot:5.1f}%  {x[1]}  {x[2]}")


def stall_sites(rep, reason, top=12):
    """Instructions with the most samples of one stall reason (e.g. 'stall_long_sb')."""
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ia, isrc, ir = h.index("Address"), h.index("Source"), h.index(reason)
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ir] or 0), r[ia][-5:], r[isrc][:80]))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in data) or 1
    print(f"top {reason} sites ({tot} samples):")
    for x in sorted(data, reverse=True)[:top]:
        print(f"  {100 * x[0] / tot:5.1f}%  {x[1]}  {x[2]}")


if len(sys.argv) > 3:
    for reason in sys.argv[3].split(","):
        stall_sites(rep, reason)
