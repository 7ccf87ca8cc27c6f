#!/usr/bin/env python
"""Summarise an .ncu-rep: key metrics per launch, stall reasons, and the
hottest SASS lines (instructions executed + stall samples).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--sass N]
"""
import csv
import io
import subprocess
import sys

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sectors.sum', 'lts__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__waves_per_multiprocessor']


def run(rep, page, extra=()):
    out = subprocess.run(['ncu', '-i', rep, '--page', page, '--csv', *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index('--sass') + 1]) if '--sass' in sys.argv else 40
    rows = run(rep, 'raw')
    hdr, units, data = rows[0], rows[1], rows[2:]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:60s} {units[i]:10s} {' '.join(d[i] for d in data)}")
    for i, h in enumerate(hdr):
        if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('per_issue_active.ratio'):
            v = [d[i] for d in data]
            if float(v[0] or 0) > 0.1:
                print(f"stall {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {' '.join(v)}")
    if nsass <= 0:
        return
    rows = run(rep, 'source', ['--print-source', 'sass'])
    hdr = rows[1]
    iS, iE, iW = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
    sass = []
    for r in rows[2:]:
        if r and r[0].startswith('0x'):
            sass.append(r)
        elif r and r[0] == 'Kernel Name' and sass:
            break
    tot = sum(int(r[iE] or 0) for r in sass)
    ws = sum(int(r[iW] or 0) for r in sass)
    print(f"warp instructions {tot}, stall samples {ws}")
    top = sorted(sass, key=lambda r: -int(r[iW] or 0))[:nsass]
    for r in top:
        print(f"{int(r[iE] or 0):9d} {int(r[iW] or 0):6d}  {r[0][-5:]}  {r[iS].strip()[:80]}")


if __name__ == '__main__':
    main()
