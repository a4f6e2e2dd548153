"""Per-source-line warp-instruction and stall-sample totals from an ncu source page
(--page source --print-source cuda,sass --csv), any kernel.  usage: ncu_srclines.py SRC.csv[.gz] [rows] [top]"""
import csv, gzip, sys
from collections import defaultdict
fn = sys.argv[1]
rows_n = float(sys.argv[2]) if len(sys.argv) > 2 else 65608366
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
op = gzip.open if fn.endswith('.gz') else open
f = None; per = []
for r in csv.reader(op(fn, 'rt')):
    if not r: continue
    if r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r[0] in ('Function Name', 'Line No') or not r[0].isdigit(): continue
    i = next((i for i in range(2, len(r) - 1) if r[i] == '-' and r[i + 1] == '-'), None)
    if i is None: continue
    try: st = float(r[i + 2]); ie = float(r[i + 5])
    except ValueError: continue
    src = ','.join(r[1:i]).strip()
    per.append((f, int(r[0]), ie, st, src))
te = sum(p[2] for p in per); ts = sum(p[3] for p in per)
print(f"total warp-instr {te:.4e} = {te / rows_n:.2f} per row; stall samples {ts:.0f}")
byf = defaultdict(lambda: [0, 0])
for p in per: byf[p[0]][0] += p[2]; byf[p[0]][1] += p[3]
for k, v in byf.items(): print(f"  {k:28s} {v[0] / rows_n:7.2f}/row  stalls {100 * v[1] / ts:5.1f}%")
for p in sorted(per, key=lambda p: -p[2])[:top]:
    print(f"{p[0][:14]:14s}:{p[1]:4d} {p[2] / rows_n:6.3f}/row st {100 * p[3] / ts:4.1f}%  {p[4][:90]}")
