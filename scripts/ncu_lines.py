"""Per-CUDA-line view of an ncu source page (--print-source cuda,sass --csv):
stall samples, warp instructions and average active threads, hottest first.

    ncu -i rep --page source --csv --print-source cuda,sass -k regex:NAME --launch-count 1 > x.csv
    python scripts/ncu_lines.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = "?", None, []
for r in rows:
    if r and r[0] == "File Name":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0] or r[0] == "Function Name":
        continue
    try:
        samp = float(r[4]); inst = float(r[7]); thr = float(r[10])
    except (ValueError, IndexError):
        continue
    out.append((samp, inst, thr, f"{fname}:{r[0]}", r[1].strip()))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"samples {ts:.0f} warp-instr {ti:.0f}")
for s, i, t, loc, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{s/ts*100:5.1f}% inst {i/ti*100:5.1f}% thr {t:4.1f} {loc:<20} {src[:80]}")
