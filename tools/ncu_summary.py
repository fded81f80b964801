"""Key metrics of the first kernel in an ncu report: duration, pipe use, stall mix."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
def g(k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
print(d.get("Kernel Name", "")[:80])
for k in keys:
    if k in d:
        print(f"  {k:65s} {d[k]} {units[h.index(k)]}")
items = [(k, g(k)) for k in h if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
items = [(k, x) for k, x in items if x]
tot = sum(x for _, x in items)
print("  stall mix:", ", ".join(f"{k.split('stalled_')[1]} {100*x/tot:.1f}%" for k, x in sorted(items, key=lambda kv: -kv[1])[:8]))
