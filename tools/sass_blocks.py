"""Summarise an ncu --page source --csv (SASS) dump: executed instructions per warp-batch,
hot blocks (runs of instructions with equal execution counts) and their stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
batches = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
data = rows[2:]
ia, isrc = hdr.index('Address'), hdr.index('Source')
iss, iex = hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot_s = sum(num(r[iss]) for r in data)
tot_e = sum(num(r[iex]) for r in data)
print(f"samples {tot_s:.0f}  warp-instr {tot_e:.0f}  per batch {tot_e / batches:.1f}")
blocks = []
for r in data:
    e = num(r[iex])
    op = r[isrc].split()[0] if r[isrc].split() else ''
    if op.startswith('@'):
        op = r[isrc].split()[1]
    if blocks and blocks[-1][1] == e:
        blocks[-1][2] += 1
        blocks[-1][3] += num(r[iss])
        blocks[-1][4].append(op)
    else:
        blocks.append([r[ia][-5:], e, 1, num(r[iss]), [op]])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
for b in blocks:
    if b[1] * b[2] > thr * tot_e or b[3] > 0.02 * tot_s:
        ops = {}
        for o in b[4]:
            ops[o] = ops.get(o, 0) + 1
        print(b[0], f"ex/batch={b[1] / batches:7.2f} n={b[2]:3d} share={b[1] * b[2] / tot_e * 100:5.1f}% "
              f"stall={b[3] / tot_s * 100:5.1f}%", ' '.join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:7]))
