#!/usr/bin/env python
"""Summarise an ncu report (--set full) and a launch-list CSV into markdown for profiles/.

usage: summarize_ncu.py REPORT.ncu-rep [LAUNCHES.csv] > summary.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed.sum", "instructions (warp)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_active", "tensor (tmem) pipe %"),
]


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    rep = sys.argv[1]
    print(f"## ncu --set full: `{rep.split('/')[-1]}`\n")
    for d, u in ncu_raw(rep):
        print(f"### {d.get('Kernel Name', '?')[:120]}\n")
        print("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d:
                print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        print()
    if len(sys.argv) > 2:
        rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 5]
        hdr = rows[0]
        iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
        tot, cnt = collections.defaultdict(float), collections.Counter()
        for r in rows[1:]:
            name = r[iK].split("(")[0]
            tot[name] += float(r[iV].replace(",", ""))
            cnt[name] += 1
        allt = sum(tot.values())
        print(f"## launch list (`gpu__time_duration.sum`, cold-cache serialised; compare shares)\n")
        print("| kernel | launches | total ms | share |\n|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda t: -t[1]):
            print(f"| {k} | {cnt[k]} | {v / 1e6:.3f} | {v / allt * 100:.1f}% |")


if __name__ == "__main__":
    main()
