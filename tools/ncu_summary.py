"""Summarise an exported ncu raw page (CSV) of one kernel: time, DRAM bytes, occupancy, issue,
pipe use, cache hit rates and the top stall reasons.  usage: ncu_summary.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
v = rows[2] if len(rows) > 2 else rows[1]
units = rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
        "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
        "derived__memory_l1_wavefronts_shared_excessive", "sm__cycles_elapsed.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
out = {}
for i, n in enumerate(h):
    if n in want:
        out[n] = (v[i], units[i] if i < len(units) else "")
print("| metric | value |\n|---|---|")
for n in want:
    if n in out:
        print(f"| `{n}` | {out[n][0]} {out[n][1]} |")
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
tot = sum(x for x, _ in st)
print("\nstall reasons (warps stalled per issue; share of all stalls):\n")
for x, n in sorted(st, reverse=True)[:8]:
    print(f"- {n}: {x:.2f} ({x / tot * 100:.1f} %)")
