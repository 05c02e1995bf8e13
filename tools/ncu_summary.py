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
    md = (["| kernel | ms | DRAM read GB | DRAM write GB | DRAM % peak | tensor pipe % | warps active % | regs |",
           "|---|---|---|---|---|---|---|---|"] if recs else [])
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
    if lfile:
        step = step_traffic(lfile)
        if step:
            traffic_path = ROOT / "profiles" / "ncu_traffic.json"
            traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
            traffic.update(step)
            traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
            out["step_traffic"] = step
            prefix.with_suffix(".json").write_text(json.dumps(out, indent=1) + "\n")
    print("\n".join(md))


# K1 / K4 calls: the regular-row kernel plus its concurrent hub-row kernel
FAMILIES = {"spmm_mean": ("mean_async_kernel", "mean_kernel<", "mean_hub"),
            "gat_aggregate": ("gat_kernel<", "gat_async_kernel", "gat_hub"),
            "conv_mean": ("conv_mean_fused_kernel",)}


def step_traffic(lfile):
    """DRAM bytes per aggregation call of the LAST bench step in a launch list
    captured with dram__bytes_{read,write}.sum (bench.py --steps 1 --warmup 1:
    the second half of the calls).  A call = its regular-row launch (+ hub launch)."""
    rows = list(csv.reader(open(lfile)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"]
    if not hi:
        return {}
    h = rows[hi[0]]
    ii, ki, mi, vi = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = {}
    for r in rows[hi[0] + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(int(r[ii]), {"kernel": r[ki]})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    launches = [per[k] for k in sorted(per)]
    res = {}
    for key, stems in FAMILIES.items():
        fam = [x for x in launches if any(s in x["kernel"] for s in stems)]
        regular = [x for x in fam if "hub" not in x["kernel"]]
        if not regular or "dram__bytes_read.sum" not in regular[0]:
            continue
        calls = len(regular) // 2
        first = fam.index(regular[calls])          # first regular launch of the last step
        last = fam[first - 1] if first and "hub" in fam[first - 1]["kernel"] else None
        step = ([last] if last else []) + fam[first:]
        dram = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in step)
        res[key] = {"dram_bytes_per_launch": dram / calls, "launches": calls,
                    "dram_bytes_per_step": dram, "source": pathlib.Path(lfile).name,
                    "basis": "ncu launch list (gpu__time_duration, dram__bytes_*), last bench "
                             "step; a launch = one aggregation call (regular + hub kernels)"}
    return res


if __name__ == "__main__":
    main()
