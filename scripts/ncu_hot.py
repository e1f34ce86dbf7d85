"""Summarise an ncu --page source --csv (SASS) dump: top stall instructions + opcode mix."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def f(x):
    try: return float(x)
    except: return 0.0
tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
print("total samples", tot, "instrs", len(data))
top = sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for d in top:
    print(f'{f(d["Warp Stall Sampling (All Samples)"])/tot*100:5.1f}% {d["Address"]:>6} exec={d["Instructions Executed"]:>8} {d["Source"][:90]}')
ops = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"] else "?"
    if op.startswith("@"): op = d["Source"].split()[1]
    ops[op.split(".")[0]] += f(d["Warp Stall Sampling (All Samples)"])
print("stall by opcode:", [(k, round(v / tot * 100, 1)) for k, v in ops.most_common(15)])
