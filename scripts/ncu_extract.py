"""Extract per-kernel metrics from an ncu --set full report into profiles/ (JSON + markdown).

    python scripts/ncu_extract.py gpurun_out/prof_full.ncu-rep profiles/r01_ncu_kernels.json
"""

from __future__ import annotations

import csv
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__t_sector_hit_rate.pct": "l1tex_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "warp_exec_efficiency_threads",
    "smsp__inst_executed.sum": "warp_instructions",
}


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(unit, 1)
    return x * scale


def main(rep: str, out_json: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    per: dict[str, list[dict]] = {}
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        d = {}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = row[i]
                if v in ("", "n/a"):
                    continue
                if "bytes" in key:
                    d[key] = to_bytes(v, units[i])
                elif key == "duration_ns":
                    scale = {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(units[i], 1.0)
                    d[key] = float(v.replace(",", "")) * scale
                else:
                    d[key] = float(v.replace(",", ""))
        stalls = [(c.replace("smsp__pcsamp_warps_issue_stalled_", ""), row[i])
                  for i, c in enumerate(hdr)
                  if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
        vals = [(k, float(v.replace(",", ""))) for k, v in stalls if v not in ("", "n/a")]
        tot = sum(v for _, v in vals) or 1.0
        d["top_stalls_pct"] = {k: round(v / tot * 100, 1) for k, v in sorted(vals, key=lambda x: -x[1])[:6]}
        per.setdefault(name, []).append(d)
    summary = {}
    for name, lst in per.items():
        agg = {}
        for key in METRICS.values():
            xs = [d[key] for d in lst if key in d]
            if xs:
                agg[key] = sum(xs) / len(xs)
        agg["top_stalls_pct"] = lst[-1]["top_stalls_pct"]
        agg["launches_profiled"] = len(lst)
        if "dram_read_bytes" in agg:
            agg["dram_traffic_bytes"] = agg["dram_read_bytes"] + agg.get("dram_write_bytes", 0.0)
        summary[name] = agg
    with open(out_json, "w") as fh:
        json.dump(summary, fh, indent=1)
    for name, agg in summary.items():
        print(f"{name[:60]:60s} {agg.get('duration_ns', 0) / 1e3:8.2f} us  "
              f"dram {agg.get('dram_traffic_bytes', 0) / 1e6:7.2f} MB  regs {agg.get('registers', 0):.0f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
