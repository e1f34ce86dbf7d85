"""Per-CUDA-line instruction counts from an ncu source CSV (same input as ncu_lines.py), by instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, out = None, []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        samp = float(r[4]); inst = float(r[7]); thr = float(r[10])
    except (ValueError, IndexError):
        continue
    out.append((samp, inst, thr, r[0], r[1].strip()))
ti = sum(o[1] for o in out) or 1
print(hdr[:12])
for s, i, t, loc, src in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"inst {i/ti*100:5.1f}% n={i:10.0f} thr={t:6.1f} L{loc:<5} {src[:90]}")
