"""Group an ncu SASS source dump (--print-source sass --csv) into runs of equal
execution count (~basic blocks) and print them by total warp instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
ix = hdr.index("Instructions Executed"); isrc = hdr.index("Source"); ith = hdr.index("Avg. Threads Executed")
ism = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ix]), float(r[ith]), float(r[ism]), r[isrc].strip()))
    except (ValueError, IndexError):
        pass
blocks, cur = [], None
for i, (n, th, smp, src) in enumerate(data):
    if cur and cur["n"] == n:
        cur["len"] += 1; cur["smp"] += smp; cur["last"] = src
    else:
        cur = {"start": i, "n": n, "len": 1, "th": th, "smp": smp, "first": src, "last": src}
        blocks.append(cur)
tot = sum(b["n"] * b["len"] for b in blocks); ts = sum(b["smp"] for b in blocks)
print(f"total warp instr {tot/1e6:.2f}M")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for b in sorted(blocks, key=lambda b: -b["n"] * b["len"])[:top]:
    print(f"@{b['start']:5d} len={b['len']:3d} n={b['n']:8.0f} tot={b['n']*b['len']/tot*100:5.1f}% smp={b['smp']/ts*100:4.1f}% thr={b['th']:4.1f} | {b['first'][:45]} .. {b['last'][:40]}")
