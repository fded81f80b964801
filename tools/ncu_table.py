"""One line per kernel of an ncu report: duration, DRAM bytes and GB/s,
issue / warps active, top stalls (development aid; summaries for profiles/)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
def f(d, k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return float("nan")
for v in rows[2:]:
    d = dict(zip(h, v))
    us = f(d, "gpu__time_duration.sum")
    ut = units[h.index("gpu__time_duration.sum")]
    us = us / 1000 if ut == "ns" else (us * 1000 if ut == "ms" else us)
    rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
    ub = units[h.index("dram__bytes_read.sum")]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ub, 1)
    rd, wr = rd * sc, wr * sc
    items = [(k, f(d, k)) for k in h if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
    items = [(k, x) for k, x in items if x == x and x > 0]
    tot = sum(x for _, x in items) or 1
    st = ", ".join(f"{k.split('stalled_')[1]} {100*x/tot:.0f}%" for k, x in sorted(items, key=lambda kv: -kv[1])[:4])
    print(f"{d.get('Kernel Name','')[:34]:34s} {us:8.1f}us dram {rd/1e6:8.1f}+{wr/1e6:8.1f} MB "
          f"{(rd+wr)/us/1e3:6.0f} GB/s issue {f(d,'smsp__issue_active.avg.pct_of_peak_sustained_active'):4.1f}% "
          f"warps {f(d,'sm__warps_active.avg.pct_of_peak_sustained_active'):4.1f}% regs {d.get('launch__registers_per_thread','')} | {st}")
