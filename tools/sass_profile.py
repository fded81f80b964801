"""Summarise an ncu `--page source --print-source sass --csv` dump: instructions
executed and stall samples per opcode and per contiguous region."""
import csv, sys, re, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    ex = int(r[ix["Instructions Executed"]] or 0)
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    data.append((r[ix["Address"]], op, ex, st, src))
tot_ex = sum(d[2] for d in data); tot_st = sum(d[3] for d in data)
by = collections.defaultdict(lambda: [0, 0])
for _, op, ex, st, _ in data:
    k = op.split(".")[0]
    by[k][0] += ex; by[k][1] += st
print(f"total warp-instr executed {tot_ex:,}  stall samples {tot_st:,}")
for k, (ex, st) in sorted(by.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{k:10s} exec {ex:>14,} ({100*ex/tot_ex:5.1f}%)  stall {100*st/max(tot_st,1):5.1f}%")
print("\nregions (consecutive instrs with same exec count):")
reg = []
for i, d in enumerate(data):
    if reg and reg[-1][2] == d[2]:
        reg[-1][1] = i; reg[-1][3] += d[3]; reg[-1][4] += 1
    else:
        reg.append([i, i, d[2], d[3], 1])
reg.sort(key=lambda r: -(r[2] * r[4]))
for a, b, ex, st, cnt in reg[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    ops = collections.Counter(data[j][1].split(".")[0] for j in range(a, b + 1))
    print(f"[{a:5d}-{b:5d}] n={cnt:5d} exec/instr={ex:>10,} total={ex*cnt:>13,} stall={100*st/max(tot_st,1):5.1f}% ops={dict(ops.most_common(5))}")

# stall reasons per address range: python sass_profile.py dump.csv N lo-hi ...
reasons = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
for rng_ in sys.argv[3:]:
    lo, hi = map(int, rng_.split("-"))
    tot = collections.Counter()
    for r in rows[2 + lo: 2 + hi + 1]:
        for c in reasons:
            tot[c] += int(r[ix[c]] or 0)
    s = sum(tot.values()) or 1
    print(f"[{lo}-{hi}] samples {s}: " + ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in tot.most_common(6)))
