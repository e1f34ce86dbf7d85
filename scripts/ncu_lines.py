"""Aggregate an ncu `--page source --print-source cuda,sass --csv` dump per CUDA
source line: warp instructions executed and stall samples (diagnostics)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ism, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        out.append((fname, int(r[0]), r[1].strip(), float(r[ism]), float(r[iex])))
    except (ValueError, IndexError):
        pass
ts = sum(o[3] for o in out) or 1.0
ti = sum(o[4] for o in out) or 1.0
print(f"total samples {ts:.0f}, warp instr {ti / 1e6:.2f}M")
print("-- by stall samples")
for f, ln, src, s, i in sorted(out, key=lambda o: -o[3])[:top]:
    print(f"{f}:{ln:4d} smp {s / ts * 100:5.1f}% ins {i / ti * 100:5.1f}% | {src[:70]}")
