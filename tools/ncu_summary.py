#!/usr/bin/env python
"""Summarise ncu reports (.ncu-rep) and launch lists into profiles/.

    python tools/ncu_summary.py OUT_PREFIX rep1.ncu-rep [rep2 ...] [--launches launches.csv]

Writes OUT_PREFIX.json (one record per profiled kernel: duration, DRAM
read/write bytes, DRAM/L2/SM throughput, tensor-pipe activity, achieved
occupancy, registers) and OUT_PREFIX.md (the same as a table, plus the
per-kernel share of the launch list).  Also merges the DRAM bytes per launch
into profiles/ncu_traffic.json, which bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import csv
import io
import json
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]

METRICS = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}

SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")], "report": pathlib.Path(rep).name}
        for key, name in METRICS.items():
            if key not in hdr:
                continue
            i = hdr.index(key)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if name == "duration_ms":
                v *= SCALE.get(u, 1.0)
            elif name.endswith("bytes"):
                v *= SCALE.get(u, 1.0)
            rec[name] = v
        recs.append(rec)
    return recs


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    per = {}
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        t = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-3 if r[ui] == "usecond" else 1.0)
        if r[ui] == "nsecond":
            t = float(r[vi].replace(",", "")) * 1e-6
        elif r[ui] == "usecond":
            t = float(r[vi].replace(",", "")) * 1e-3
        elif r[ui] == "msecond":
            t = float(r[vi].replace(",", ""))
        c, s = per.get(name, (0, 0.0))
        per[name] = (c + 1, s + t)
    total = sum(s for _, s in per.values())
    return total, sorted(((s, c, n) for n, (c, s) in per.items()), reverse=True)


def short(name):
    n = name.replace("void ", "").replace("glint::<unnamed>::", "").replace("(anonymous namespace)::", "")
    return n[:70]


def main():
    args = sys.argv[1:]
    lfile = None
    if "--launches" in args:
        i = args.index("--launches")
        lfile = args[i + 1]
        args = args[:i] + args[i + 2:]
    prefix = pathlib.Path(args[0])
    recs = []
    for rep in args[1:]:
        recs += raw(rep)
    out = {"kernels": recs}
    md = ["| kernel | ms | DRAM read GB | DRAM write GB | DRAM % peak | tensor pipe % | warps active % | regs |",
          "|---|---|---|---|---|---|---|---|"]
    for r in recs:
        md.append("| {} | {:.3f} | {:.2f} | {:.2f} | {:.1f} | {:.1f} | {:.1f} | {:.0f} |".format(
            short(r["kernel"]), r.get("duration_ms", 0), r.get("dram_read_bytes", 0) / 1e9,
            r.get("dram_write_bytes", 0) / 1e9, r.get("dram_pct_of_peak", 0),
            r.get("tensor_pipe_pct", 0), r.get("warps_active_pct", 0), r.get("registers", 0)))
    if lfile:
        total, per = launches(lfile)
        out["launch_list"] = {"total_ms": total,
                              "kernels": [{"kernel": n, "launches": c, "ms": s, "share": s / total}
                                          for s, c, n in per]}
        md += ["", f"Launch list ({lfile}): total {total:.2f} ms of kernel time (ncu, serialised, "
                   "cold caches; compare shares, not absolutes)", "",
               "| kernel | launches | ms | share |", "|---|---|---|---|"]
        for s, c, n in per[:15]:
            md.append(f"| {short(n)} | {c} | {s:.3f} | {100 * s / total:.1f}% |")
    prefix.with_suffix(".json").write_text(json.dumps(out, indent=1) + "\n")
    prefix.with_suffix(".md").write_text("\n".join(md) + "\n")
    traffic_path = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for key, stem in (("spmm_mean", "mean_kernel"), ("gat_aggregate", "gat_kernel")):
        hits = [r for r in recs if stem in r["kernel"]]
        if not hits:
            continue
        dram = sum(r.get("dram_read_bytes", 0) + r.get("dram_write_bytes", 0) for r in hits)
        traffic[key] = {"dram_bytes_per_launch": dram / len(hits), "launches": len(hits),
                        "dram_bytes_total": dram, "reports": sorted({r["report"] for r in hits}),
                        "duration_ms_total": sum(r.get("duration_ms", 0) for r in hits)}
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
