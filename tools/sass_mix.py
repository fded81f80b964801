"""Instruction mix (executed warp instructions and stall samples per opcode)
of one kernel from an ncu report's source page (development aid).
    python tools/sass_mix.py report.ncu-rep kernel_regex"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--kernel-name",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
c, s, tot = collections.Counter(), collections.Counter(), 0
h = None
for r in rows:
    if "Instructions Executed" in r:
        h = r
        ie, src, smp = r.index("Instructions Executed"), r.index("Source"), r.index("# Samples")
        continue
    if h is None or len(r) <= ie or not r[ie].isdigit():
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    n = int(r[ie])
    c[op] += n
    s[op] += int(r[smp] or 0)
    tot += n
ts = sum(s.values()) or 1
for op, n in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 24):
    print(f"{op:10s} {n:11d} {100 * n / tot:5.1f}%  samples {100 * s[op] / ts:5.1f}%")
print("total warp instructions", tot)
