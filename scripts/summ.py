"""Summarise gpurun_out: bench line essentials, ncu launch list, per-kernel details."""
import csv, collections, json, subprocess, sys
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
for k in ["value", "ms_per_step", "stage_ms", "e2e", "roofline", "clocks"]:
    print(k, d.get(k))
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r)); agg.setdefault(x["Kernel Name"][:50], []).append(float(x["Metric Value"]))
tot = 0
for n, v in agg.items():
    if n.startswith("void at::"): continue
    a = sum(v) / len(v) / 1000; tot += a
    print(f"  {n:52s} n={len(v):3d} avg={a:8.2f}us")
print(f"  sum of pf kernels {tot:.1f}us")
out = subprocess.run(["ncu", "-i", "gpurun_out/prof_full.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines())); h = r[0]
for row in r[2:]:
    name = row[h.index("Kernel Name")][:40]
    st = [(c.replace("smsp__pcsamp_warps_issue_stalled_", ""), row[i]) for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
    vals = [(k, float(v.replace(",", ""))) for k, v in st if v not in ("", "n/a")]
    t = sum(v for _, v in vals) or 1
    g = lambda m: row[h.index(m)] if m in h else "?"
    print(name, "dur", g("gpu__time_duration.sum"), "warps_active%", g("sm__warps_active.avg.pct_of_peak_sustained_active"),
          "dram R/W MB", g("dram__bytes_read.sum"), g("dram__bytes_write.sum"), "regs", g("launch__registers_per_thread"))
    print("    stalls", [(k, round(v / t * 100, 1)) for k, v in sorted(vals, key=lambda x: -x[1])[:7]])
