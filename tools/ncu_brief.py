#!/usr/bin/env python
"""Print the headline metrics and the top stalled SASS lines of an ncu report.

  python tools/ncu_brief.py report.ncu-rep [--top 20]
"""
import csv
import subprocess
import sys

METRICS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
           'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
           'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
           'sm__warps_active.avg.pct_of_peak_sustained_active',
           'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
           'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
           'lts__throughput.avg.pct_of_peak_sustained_elapsed',
           'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
           'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
           'launch__registers_per_thread', 'sm__cycles_elapsed.avg.per_second']


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index('--top') + 1]) if '--top' in sys.argv else 20
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get('Kernel Name', '')[:100])
        for m in METRICS:
            if m in d:
                print(f'  {m:80s} {d[m]}')
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == 'Address':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    key = 'Warp Stall Sampling (All Samples)'
    tot = sum(float(d[key] or 0) for d in data) or 1.0
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:top]:
        print(f"{d['Address'][-5:]} {100 * float(d[key]) / tot:5.1f}% {d['Source'][:70]:70s} "
              f"x{d['Instructions Executed']}")


if __name__ == '__main__':
    main()
